"""The distributed offline phase 2 (form_K + factorize into the row-cyclic
layout of the distributed K^{-1}, ltb_engine_form_k_generated_dist /
ltb_engine_factorize_dist) on ONE GPU (world 1: the same kernels, no NCCL),
against the one-GPU path (itself checked against the oracle in
test_formk.py) -- K, L and the online result -- plus the column-sharded
prior-premultiplied G* plan the distributed online phase uses.  The
multi-GPU run of the same code is tests/dist_offline_check.py."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
PRIOR = (1.0, 2.0, 1.0)


@pytest.fixture(scope="module")
def ltb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_16344_b200 as ltb
    ltb.load()
    return ltb


@pytest.mark.parametrize("nd,nm,nt", [(16, 300, 64), (10, 200, 50), (7, 96, 37), (64, 2048, 128)])
def test_distributed_path_matches_one_gpu(ltb, nd, nm, nt):
    seed, s2 = 31 + nd, 0.7
    pg = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, seed, PRIOR)
    one = ltb.InferenceEngine(pg)
    one.form_K_generated(seed, 1, PRIOR, s2)
    K1 = one.K_lower()
    one.factorize()
    L1 = one.chol_lower()
    dst = ltb.InferenceEngine(pg)
    dst.form_K_generated(seed, 1, PRIOR, s2, distributed=True)
    K2 = dst.K_lower()
    assert orc.rel_err(K2, K1) <= 1e-14
    dst.factorize()
    L2 = dst.chol_lower()
    assert np.all(np.triu(L2, 1) == 0.0)
    assert orc.rel_err(L2, L1) <= 1e-13
    d = np.random.default_rng(nd).standard_normal(nd * nt)
    m1, m2 = np.empty(nm * nt), np.empty(nm * nt)
    one.infer_raw(d, m1)
    dst.infer_raw(d, m2)
    assert orc.rel_err(m2, m1) <= 1e-12
    # and the factor solves: K^{-1} (K x) == x through the oracle's K
    x = np.random.default_rng(1).standard_normal(nd * nt)
    K = K1 + np.tril(K1, -1).T
    assert orc.rel_err(dst.solve_k_inplace(K @ x), x) <= 1e-9
    one.close()
    dst.close()


def test_sharded_premultiplied_plan(ltb):
    nd, nm, nt, seed = 8, 500, 40, 5
    full = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, seed, PRIOR)
    d = np.random.default_rng(2).standard_normal(nd * nt)
    ref = full.apply_adjoint(ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, d)).values.reshape(nm, nt)
    for c0, c1 in [(0, 167), (167, 334), (334, 500), (17, 18)]:
        sh = ltb.MatvecPlan.generated_premultiplied(nd, c1 - c0, nt, seed, PRIOR, nm_total=nm, c0=c0)
        got = sh.apply_adjoint(ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, d)).values.reshape(c1 - c0, nt)
        assert orc.rel_err(got, ref[c0:c1]) <= 1e-14
    g = orc.prior_premultiply(orc.gen_kernel(seed, nd, nm, nt, stream=1), *PRIOR)
    assert orc.rel_err(ref.ravel(), orc.OraclePlan(g).apply_adjoint(d)) <= 1e-12


def test_distributed_path_not_positive_definite(ltb):
    """A K that is not SPD (sigma2 far below zero) fails the distributed
    factorisation with NumericalError, as the one-GPU path (bayes_engine.cpp:
    176-209 throws on a failed dpotrf / LLT)."""
    nd, nm, nt, seed = 6, 64, 32, 3
    pg = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, seed, PRIOR)
    eng = ltb.InferenceEngine(pg)
    eng.form_K_generated(seed, 1, PRIOR, -1e6, distributed=True)
    with pytest.raises(ltb.NumericalError):
        eng.factorize()
    with pytest.raises(ltb.StateError):  # K was consumed; no factor
        eng.infer_raw(np.zeros(nd * nt), np.empty(nm * nt))
    eng.close()
