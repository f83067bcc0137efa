"""The one-GPU super-block K^{-1} chain (ltb_trsv.cu trsv_super_kernel, every
one-GPU factor with nb <= 512): solves through set_factor against the
oracle's substitution (orc_solve_k, the reference's two TRSVs,
bayes_engine.cpp:236-240) at sizes spanning partial and full super blocks,
on the synthetic factor and on factors with a graded diagonal (condition
numbers of L up to ~1e4), where the tolerance scales with kappa(K) as the
error of any backward-stable solve does."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ltb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_16344_b200 as ltb
    ltb.load()
    return ltb


def engine(ltb, n):
    ident = np.zeros((n, n, 1))
    ident[np.arange(n), np.arange(n), 0] = 1.0
    return ltb.InferenceEngine(ltb.MatvecPlan(ltb.BlockToeplitzKernel(n, n, 1, tag=ltb.KernelTag.Gstar, data=ident)))


def identity_engine_nt(ltb, nd, nt):
    """n = nd * nt without an n x n x 1 dense kernel (large n): a G* plan of
    nd sensors x nt lags whose values never matter for solve_k_inplace."""
    return ltb.InferenceEngine(ltb.MatvecPlan.generated(nd, 8, nt, seed=1, tag=ltb.KernelTag.Gstar))


@pytest.mark.parametrize("n", [511, 512, 513, 1536, 4096, 4097, 6000])
def test_super_chain_vs_substitution(ltb, n):
    L = orc.gen_factor(7 + n % 97, n)
    eng = engine(ltb, n)
    eng.set_factor(L)
    y = np.random.default_rng(n).standard_normal(n)
    x = eng.solve_k_inplace(y.copy())
    assert orc.rel_err(x, orc.solve_k(L, y)) <= 1e-12
    eng.close()


@pytest.mark.parametrize("nd,nt", [(64, 128), (128, 128), (256, 128)])
def test_super_chain_generated_factor_large(ltb, nd, nt):
    """n = 8192 (config 2), 16384, 32768 (nb = 512, the largest super-chain
    size) on the generated factor against the oracle's blocked substitution."""
    n = nd * nt
    eng = identity_engine_nt(ltb, nd, nt)
    eng.set_factor_generated(4321)
    y = np.random.default_rng(n).standard_normal(n)
    x = eng.solve_k_inplace(y.copy())
    assert orc.rel_err(x, orc.solve_k_gen(4321, y)) <= 1e-12
    eng.close()


@pytest.mark.parametrize("n,grade", [(2048, 1e2), (3000, 1e3), (4096, 1e4)])
def test_super_chain_graded_diagonal(ltb, n, grade):
    """L = D (I + strictly lower noise) with D graded from 1 to 1/grade:
    kappa(L) ~ grade.  Both the explicit 512-block inverses and the
    row-by-row substitution are backward stable here, so they agree to
    O(kappa(K) eps); held to 50 kappa(K) eps."""
    rng = np.random.default_rng(n)
    d = np.geomspace(1.0, 1.0 / grade, n)
    rng.shuffle(d)
    L = np.tril(rng.standard_normal((n, n)) * 0.3 / np.sqrt(n), -1) + np.eye(n)
    L = L * d[:, None]
    eng = engine(ltb, n)
    eng.set_factor(L)
    y = rng.standard_normal(n)
    x = eng.solve_k_inplace(y.copy())
    ref = orc.solve_k(L, y)
    kappa_k = np.linalg.cond(L) ** 2
    err = orc.rel_err(x, ref)
    assert err <= 50 * kappa_k * np.finfo(float).eps, (err, kappa_k)
    eng.close()
