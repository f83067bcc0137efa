"""Driver for ncu captures of the time-axis transforms at the Cascadia row
count (dev tool): a thin generated plan (Nd=8) over Nm columns of Nt=420, so
F m runs the r2c over Nm rows and F* d the c2r over Nm rows; prints device
times of a few applies (F-hat of this plan is small, the transforms dominate)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nm = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
nt = int(sys.argv[3]) if len(sys.argv) > 3 else 420
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
import time

plan = ltb.MatvecPlan.generated(nd, nm, nt, seed=7)
sc = ltb.MatvecPlan.Scratch(plan)
m = torch.rand(nm * nt, dtype=torch.float64, device="cuda")
d = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
mo = torch.empty_like(m)
gb = (nm * nt * 8 + nm * (nt + 1) * 16) / 1e9
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.apply_raw(m, d, sc)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan.apply_adjoint_raw(d, mo, sc)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("rep %d F %.3f ms  F* %.3f ms  (wall, incl. launch; r2c/c2r bytes %.3f GB each)"
          % (i, (t1 - t0) * 1e3, (t2 - t1) * 1e3, gb))
