"""Small end-to-end exercise of every kernel family (e.g. for a sanitizer or
a quick smoke on a new box; dev tool): plans (generated, premultiplied, four-step FFT), host/device
applies incl. the pipelined host path, form_K / factorize / form_Q, infer
with the fused forecast, predict_qoi, residual, writers."""
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

rng = np.random.default_rng(0)
nd, nq, nm, nt = 3, 2, 24, 10
prior, s2 = (1.0, 2.0, 1.0), 0.3
f = rng.standard_normal((nd, nm, nt))
fq = rng.standard_normal((nq, nm, nt))
kf = ltb.BlockToeplitzKernel(nd, nm, nt, tag=ltb.KernelTag.F, data=f)
pf = ltb.MatvecPlan(kf)
pg = ltb.MatvecPlan.premultiplied(kf, prior)
pq = ltb.MatvecPlan(ltb.BlockToeplitzKernel(nq, nm, nt, tag=ltb.KernelTag.Fq, data=fq))
d = pf.apply_adjoint(ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, rng.standard_normal(nd * nt)))
eng = ltb.InferenceEngine(pg, pq)
eng.form_K(f, prior=prior, sigma2=s2)
eng.factorize()
eng.form_Q(f, fq, prior=prior)
eng.set_residual_model(pf, s2, prior)
obs = ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, rng.standard_normal(nd * nt))
r = eng.infer_map(obs, with_forecast=True)
p = eng.predict_qoi(obs)
with tempfile.TemporaryDirectory() as t:
    ltb.write_engine_artifacts(t, eng, f_kernel=kf)
# pipelined host path (>= 16 MB field) and the four-step FFT
big = ltb.MatvecPlan.generated(4, 16500, 128, seed=1)
m = rng.standard_normal(16500 * 128)
dd = np.empty(4 * 128)
big.apply_raw(m, dd, ltb.MatvecPlan.Scratch(big))
mm = np.empty(16500 * 128)
big.apply_adjoint_raw(dd, mm, ltb.MatvecPlan.Scratch(big))
long = ltb.MatvecPlan(ltb.BlockToeplitzKernel(2, 3, 4096, data=rng.standard_normal((2, 3, 4096))))
long.apply(ltb.SpaceTimeField(3, 4096, ltb.Layout.SpaceMajorRows, rng.standard_normal(3 * 4096)))
torch.cuda.synchronize()
print("sanitize run ok", float(np.abs(r.m_map.values).sum()), float(np.abs(mm).sum()))
