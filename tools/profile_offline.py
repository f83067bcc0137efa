"""Driver for ncu captures of the offline DMMA kernels at config 2 (dev
tool): form_K, factorize, form_Q of the generated model."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

nd, nm, nt, nq, seed = 64, 16384, 128, 8, 4321
prior = (1.0, 2.0, 1.0)
pg = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, seed, prior)
pq = ltb.MatvecPlan.generated(nq, nm, nt, seed, tag=ltb.KernelTag.Fq)
eng = ltb.InferenceEngine(pg, pq)
eng.form_K_generated(seed, 1, prior, 1.0)
eng.factorize()
eng.form_Q_generated(seed, nq, prior)
print("offline ms", eng.offline_ms(), eng.form_Q_ms())
