"""Small driver for ncu captures of the hot kernels: a Cascadia-shaped plan
with fewer columns (Nd=600, Nt=420, Nm=2048 -> F-hat 8.3 GB, still far larger
than L2), a few F m / F* d applies.  Development tool, not part of the
product."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

nd, nm, nt = 600, int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 420
plan = ltb.MatvecPlan.generated(nd, nm, nt, seed=20250810)
s = ltb.MatvecPlan.Scratch(plan)
m = torch.rand(nm * nt, dtype=torch.float64, device="cuda")
d = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
dm = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
mm = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
for _ in range(3):
    plan.apply_raw(m, dm, s)
    plan.apply_adjoint_raw(d, mm, s)
s.sync()
print("ok", float(dm.abs().sum()), float(mm.abs().sum()))
