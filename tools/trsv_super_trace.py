"""Timeline of the one-GPU super-block K^{-1} kernel (dev tool): kernel start,
grid barrier, per chain step the time its inputs were resolved and the time
it published, end -- plus the device time of solve_k_inplace.
    python tools/trsv_super_trace.py [nd nt]"""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402
from paper_2504_16344_b200 import _lib  # noqa: E402

nd, nt = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (64, 128)
g = ltb.MatvecPlan.generated(nd, 64, nt, seed=1, tag=ltb.KernelTag.Gstar)
eng = ltb.InferenceEngine(g)
eng.set_factor_generated(4321)
L = _lib.load()
L.ltb_engine_trsv_trace(eng._h, 1, None, 0)
y = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
for _ in range(5):
    eng.solve_k_inplace(y)
torch.cuda.synchronize()
nb = (nd * nt + 63) // 64
ns = (nb + 7) // 8
buf = (C.c_ulonglong * (8 * nb + 1))()
L.ltb_engine_trsv_trace(eng._h, 1, buf, 8 * nb + 1)
a = np.array(buf[:], dtype=np.float64)
t0 = a[0]
pub = (a[2:2 + 2 * ns] - t0) / 1e3
inp = (a[2 + 2 * ns:2 + 4 * ns] - t0) / 1e3
print(json.dumps({"n": nd * nt, "nb": nb, "ns": ns, "barrier_us": (a[1] - t0) / 1e3, "end_us": (a[2 + 4 * ns] - t0) / 1e3,
                  "step_inputs_us": [round(v, 2) for v in inp], "step_published_us": [round(v, 2) for v in pub],
                  "compute_us_median": float(np.median(pub - inp))}))
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.solve_k_inplace(y)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("solve_k_inplace device ms: median %.3f min %.3f" % (sorted(ts)[5], min(ts)))
