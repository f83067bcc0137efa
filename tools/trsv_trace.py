"""TRSV chain/worker timeline on config 2 (dev tool)."""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402
from paper_2504_16344_b200 import _lib  # noqa: E402

nd, nm, nt, seed = 64, 16384, 128, 4321
g = ltb.MatvecPlan.generated(nd, nm, nt, seed=seed, tag=ltb.KernelTag.Gstar)
eng = ltb.InferenceEngine(g)
eng.set_factor_generated(seed)
L = _lib.load()
L.ltb_engine_trsv_trace(eng._h, 1, None, 0)
y = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
for _ in range(5):
    eng.solve_k_inplace(y)
nb = (nd * nt + 63) // 64
buf = (C.c_ulonglong * (8 * nb + 1))()
L.ltb_engine_trsv_trace(eng._h, 1, buf, 8 * nb + 1)
a = np.array(buf[:], dtype=np.float64)
t0 = a[4 * nb]
cf, cb, wf, wb = a[:nb] - t0, a[nb:2 * nb] - t0, a[2 * nb:3 * nb] - t0, a[3 * nb:4 * nb] - t0
det = np.array(buf[4 * nb + 1:8 * nb + 1], dtype=np.float64).reshape(nb, 4)  # SM cycles
ph = np.stack([det[:, 1] - det[:, 0], det[:, 2] - det[:, 1], det[:, 3] - det[:, 2],
               np.concatenate([det[1:, 0] - det[:-1, 3], [np.nan]])], 1)[3:-1]
detail = {"unit": "SM cycles (median)", "tile_wait": float(np.median(ph[:, 0])), "peer_fma_bar1": float(np.median(ph[:, 1])),
          "c_resolve": float(np.median(ph[:, 2])), "push_bar2_next_issue": float(np.median(ph[:, 3])),
          "step_total": float(np.median(np.diff(det[:, 0])))}
out = {"nb": nb, "fwd_detail": detail, "fwd_chain_end_us": cf[-1] / 1e3, "bwd_chain_end_us": cb[0] / 1e3,
       "fwd_step_us_median": float(np.median(np.diff(cf))) / 1e3,
       "bwd_step_us_median": float(np.median(-np.diff(cb))) / 1e3,
       "fwd_worker_lead_us": [round((cf[i] - wf[i]) / 1e3, 2) for i in range(0, nb, 8)],
       "bwd_worker_lead_us": [round((cb[i] - wb[i]) / 1e3, 2) for i in range(0, nb, 8)],
       "fwd_chain_us": [round(x / 1e3, 2) for x in cf[::8]],
       "fwd_worker_done_us": [round(x / 1e3, 2) for x in wf[::8]]}
print(json.dumps(out))
