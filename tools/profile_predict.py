"""predict_qoi (Q d + credible intervals) at the Cascadia QoI shape (dev
tool): Nd=600, Nq=21, Nt=420 -> Q is 8820 x 252000 FP64 = 17.8 GB, built on
the device (torch.rand) and installed through ltb_engine_set_phase3 with
device pointers; prints the device time of Q d and its GB/s."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402
from paper_2504_16344_b200 import _lib  # noqa: E402

nd, nq, nt = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (600, 21, 420)
g = ltb.MatvecPlan.generated(nd, 64, nt, seed=1, tag=ltb.KernelTag.Gstar)
fq = ltb.MatvecPlan.generated(nq, 64, nt, seed=1, tag=ltb.KernelTag.Fq)
eng = ltb.InferenceEngine(g, fq)
rows, cols = nq * nt, nd * nt
Q = torch.rand(cols, rows, dtype=torch.float64, device="cuda").t()  # column-major rows x cols
gd = torch.rand(rows, dtype=torch.float64, device="cuda")
L = _lib.load()
ltb.matvec.check(L.ltb_engine_set_phase3(eng._h, C.c_void_p(Q.data_ptr()), rows, C.c_void_p(gd.data_ptr()), 1))
del Q
torch.cuda.empty_cache()
d = torch.rand(cols, dtype=torch.float64, device="cuda")
q, lo, hi = (torch.empty(rows, dtype=torch.float64, device="cuda") for _ in range(3))
secs = C.c_double()
ts = []
for r in range(8):
    ltb.matvec.check(L.ltb_engine_predict_qoi(eng._h, eng._scratch._h, C.c_void_p(d.data_ptr()), 0.95,
                                               C.c_void_p(q.data_ptr()), C.c_void_p(lo.data_ptr()),
                                               C.c_void_p(hi.data_ptr()), C.byref(secs), 1))
    ts.append(secs.value)
t = sorted(ts[2:])[len(ts[2:]) // 2]
gb = rows * cols * 8 / 1e9
print("predict_qoi Q %dx%d (%.1f GB): %.3f ms  %.0f GB/s" % (rows, cols, gb, t * 1e3, gb / t))
