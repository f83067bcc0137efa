"""Offline phase 2 at sizes beyond config 2 (dev tool): form_K of the
generated prior-premultiplied G, factorize, and the round trip
K^{-1} (K x) == x with K x = F (G* x) + x applied through the plans.
    python tools/offline_scale_check.py"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

PRIOR = (1.0, 2.0, 1.0)
for nd, nm, nt in [(128, 8192, 128), (96, 4096, 100)]:
    pg = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, 4321, PRIOR)
    pf = ltb.MatvecPlan.generated(nd, nm, nt, seed=4321, tag=ltb.KernelTag.F)
    eng = ltb.InferenceEngine(pg)
    eng.form_K_generated(4321, 1, PRIOR, 1.0)
    eng.factorize()
    fk, fz = eng.offline_ms()
    n = nd * nt
    sg, sf = ltb.MatvecPlan.Scratch(pg), ltb.MatvecPlan.Scratch(pf)
    x = np.random.default_rng(1).standard_normal(n)
    m, kx = np.empty(nm * nt), np.empty(n)
    pg.apply_adjoint_raw(x, m, sg)
    pf.apply_raw(m, kx, sf)
    kx += x
    y = eng.solve_k_inplace(kx.copy())
    print("n=%d form_K %.1f ms (%.1f TFLOP/s) factorize %.2f ms (%.1f TFLOP/s)  |K^-1 (K x) - x| / |x| = %.2e"
          % (n, fk, n * n * nm / fk / 1e9, fz, n ** 3 / 3 / fz / 1e9, np.linalg.norm(y - x) / np.linalg.norm(x)))
    sg.close()
    sf.close()
    eng.close()
