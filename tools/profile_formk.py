"""Driver for ncu captures of the offline phase-2 kernels at config 2
(N_d=64, N_m=16384, N_t=128, n=8192): form_K of the generated kernel and
the tile Cholesky.  Development tool, not part of the product."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

nd, nm, nt = 64, int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prior = (1.0, 2.0, 1.0)
pg = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, 4321, prior)
eng = ltb.InferenceEngine(pg)
n = nd * nt
for r in range(reps):
    t0 = time.time()
    eng.form_K_generated(4321, 1, prior, 1.0)
    eng.factorize()
    fk, fz = eng.offline_ms()
    print("rep %d form_K %.2f ms (%.1f TFLOP/s) factorize %.2f ms (%.1f TFLOP/s) wall %.2f s" %
          (r, fk, n * n * nm / fk / 1e9, fz, n ** 3 / 3 / fz / 1e9, time.time() - t0))
