"""GEMV work-unit size sweep for small-N_d plans (dev tool): F_q of config 2
(N_q=8, N_m=16384, N_t=128) and G* (N_d=64), F apply device time per unit_cols."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

for rows, label in [(8, "F_q"), (64, "G*")]:
    for uc in [0, 16384, 8192, 5462, 4096, 3277, 2731, 1786, 1024]:
        p = ltb.MatvecPlan.generated(rows, 16384, 128, seed=3, unit_cols=uc)
        s = ltb.MatvecPlan.Scratch(p, stream=torch.cuda.current_stream())
        m = torch.rand(16384 * 128, dtype=torch.float64, device="cuda")
        d = torch.empty(rows * 128, dtype=torch.float64, device="cuda")
        dd = torch.rand(rows * 128, dtype=torch.float64, device="cuda")
        mm = torch.empty(16384 * 128, dtype=torch.float64, device="cuda")
        s.timing(True)
        for _ in range(3):
            p.apply_raw(m, d, s)
            p.apply_adjoint_raw(dd, mm, s)
        s.timing(True)
        for _ in range(10):
            p.apply_raw(m, d, s)
            p.apply_adjoint_raw(dd, mm, s)
        st = s.stage_ms()
        print("%s unit_cols=%5d  gemv_n %.1f us  gemv_h %.1f us" %
              (label, uc, st["F"][1] / 10 * 1e3, st["Fstar"][1] / 10 * 1e3))
        s.close()
        p.close()
