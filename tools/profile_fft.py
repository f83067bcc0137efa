"""ncu driver for the time-axis transform kernels (dev tool): F m and F* d
on (Nd, Nm, Nt) = (8, 16384, 128) and (600, 4096, 420)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

for nd, nm, nt in [(8, 16384, 128), (600, 4096, 420)]:
    plan = ltb.MatvecPlan.generated(nd, nm, nt, seed=3)
    s = ltb.MatvecPlan.Scratch(plan)
    m = torch.rand(nm * nt, dtype=torch.float64, device="cuda")
    d = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
    dm = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
    mm = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
    for _ in range(2):
        plan.apply_raw(m, dm, s)
        plan.apply_adjoint_raw(d, mm, s)
    s.sync()
    del s, plan
print("ok")
