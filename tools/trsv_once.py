"""One K^{-1} apply at config 2 (dev tool, for ncu)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

g = ltb.MatvecPlan.generated(64, 64, 128, seed=1, tag=ltb.KernelTag.Gstar)
eng = ltb.InferenceEngine(g)
eng.set_factor_generated(4321)
y = torch.rand(64 * 128, dtype=torch.float64, device="cuda")
for _ in range(2):
    eng.solve_k_inplace(y)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()))
