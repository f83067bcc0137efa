"""Driver for an ncu launch list of the online path at config 2 (dev tool):
generated G* / F_q plans, generated factor, a few infer_map + forecast."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

nd, nm, nt, nq, seed = 64, 16384, 128, 8, 4321
g = ltb.MatvecPlan.generated(nd, nm, nt, seed=seed, tag=ltb.KernelTag.Gstar)
fq = ltb.MatvecPlan.generated(nq, nm, nt, seed=seed, tag=ltb.KernelTag.Fq)
eng = ltb.InferenceEngine(g, fq)
eng.set_factor_generated(seed)
d = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
m = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
q = torch.empty(nq * nt, dtype=torch.float64, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ts = sorted(eng.infer_raw(d, m, q) for _ in range(reps))
print("infer+forecast median %.3f ms (min %.3f, %d reps)" % (ts[len(ts) // 2] * 1e3, ts[0] * 1e3, reps))
