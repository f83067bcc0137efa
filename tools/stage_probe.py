"""Per-stage device times (CUDA events inside libltb) of F m and F* d for a
set of shapes; a development probe, not part of the product."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402


def probe(nd, nm, nt, reps=20):
    plan = ltb.MatvecPlan.generated(nd, nm, nt, seed=1)
    s = ltb.MatvecPlan.Scratch(plan)
    m = torch.rand(nm * nt, dtype=torch.float64, device="cuda")
    d = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
    dm = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
    mm = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
    for _ in range(3):
        plan.apply_raw(m, dm, s)
        plan.apply_adjoint_raw(d, mm, s)
    s.timing(True)
    for _ in range(reps):
        plan.apply_raw(m, dm, s)
        plan.apply_adjoint_raw(d, mm, s)
    st = s.stage_ms()
    gb = 16 * (nt + 1) * nd * nm
    out = {"shape": [nd, nm, nt],
           "F_us": [round(x / reps * 1e3, 1) for x in st["F"]],
           "Fstar_us": [round(x / reps * 1e3, 1) for x in st["Fstar"]],
           "gemv_n_gbs": round(gb / (st["F"][1] / reps * 1e-3) / 1e9, 1),
           "gemv_h_gbs": round(gb / (st["Fstar"][1] / reps * 1e-3) / 1e9, 1)}
    print(json.dumps(out), flush=True)
    del s, plan


if __name__ == "__main__":
    shapes = [(8, 1024, 64), (8, 16384, 128), (21, 16384, 420), (64, 16384, 128),
              (600, 2048, 420), (600, 8192, 420)]
    for sh in shapes:
        probe(*sh)
