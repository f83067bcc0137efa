"""Seeded random sweep over shapes (GPU): every path against the oracle on
shapes the targeted tests do not pin -- prime / odd / ragged N_t, N_d, N_m,
n not a multiple of the 64-blocks, unit sizes, host and device pointers."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def ltb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_16344_b200 as ltb
    ltb.load()
    return ltb


def shapes(seed, count, nd_max, nm_max, nt_max):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(1, nd_max + 1)), int(rng.integers(1, nm_max + 1)), int(rng.integers(1, nt_max + 1)),
             int(rng.integers(0, 2**31))) for _ in range(count)]


@pytest.mark.parametrize("nd,nm,nt,seed", shapes(101, 24, 40, 700, 300))
def test_matvec_random_shapes(ltb, nd, nm, nt, seed):
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((nd, nm, nt))
    plan = ltb.MatvecPlan(ltb.BlockToeplitzKernel(nd, nm, nt, data=k),
                          unit_cols=int(rng.choice([0, 1, 7, 64])))
    op = orc.OraclePlan(k)
    m = rng.standard_normal(nm * nt)
    d = rng.standard_normal(nd * nt)
    s = ltb.MatvecPlan.Scratch(plan)
    fm, fd = np.empty(nd * nt), np.empty(nm * nt)
    plan.apply_raw(m, fm, s)
    plan.apply_adjoint_raw(d, fd, s)
    assert orc.rel_err(fm, op.apply(m)) <= TOL
    assert orc.rel_err(fd, op.apply_adjoint(d)) <= TOL


def reg_shapes(seed, count):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(1, 24)), int(rng.integers(1, 3000)), int(rng.choice([64, 128, 256, 420, 512])),
             int(rng.integers(0, 2**31))) for _ in range(count)]


@pytest.mark.parametrize("nd,nm,nt,seed", reg_shapes(303, 12))
def test_register_fft_random_shapes(ltb, nd, nm, nt, seed):
    """The register two-pass transforms (2 N_t in {128, 256, 512, 840, 1024})
    on random row counts, unit sizes and both pointer kinds."""
    import torch
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((nd, nm, nt))
    plan = ltb.MatvecPlan(ltb.BlockToeplitzKernel(nd, nm, nt, data=k),
                          unit_cols=int(rng.choice([0, 1, 7, 64])))
    op = orc.OraclePlan(k)
    m = rng.standard_normal(nm * nt)
    d = rng.standard_normal(nd * nt)
    s = ltb.MatvecPlan.Scratch(plan, stream=torch.cuda.current_stream())
    if rng.integers(0, 2):
        fm, fd = np.empty(nd * nt), np.empty(nm * nt)
        plan.apply_raw(m, fm, s)
        plan.apply_adjoint_raw(d, fd, s)
    else:
        fm_t = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
        fd_t = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
        plan.apply_raw(torch.from_numpy(m).cuda(), fm_t, s)
        plan.apply_adjoint_raw(torch.from_numpy(d).cuda(), fd_t, s)
        torch.cuda.synchronize()
        fm, fd = fm_t.cpu().numpy(), fd_t.cpu().numpy()
    assert orc.rel_err(fm, op.apply(m)) <= TOL
    assert orc.rel_err(fd, op.apply_adjoint(d)) <= TOL


@pytest.mark.parametrize("nd,nm,nt,seed", shapes(202, 8, 9, 90, 40))
def test_offline_random_shapes(ltb, nd, nm, nt, seed):
    rng = np.random.default_rng(seed)
    prior, s2 = (1.0, float(rng.uniform(0.0, 3.0)), 1.0), float(rng.uniform(0.2, 2.0))
    f = rng.standard_normal((nd, nm, nt)) * 0.8 ** np.arange(nt)
    fq = rng.standard_normal((2, nm, nt)) * 0.8 ** np.arange(nt)
    g = orc.prior_premultiply(f, *prior)
    gq = orc.prior_premultiply(fq, *prior)
    kf = ltb.BlockToeplitzKernel(nd, nm, nt, tag=ltb.KernelTag.F, data=f)
    eng = ltb.InferenceEngine(ltb.MatvecPlan.premultiplied(kf, prior),
                              ltb.MatvecPlan(ltb.BlockToeplitzKernel(2, nm, nt, tag=ltb.KernelTag.Fq, data=fq)))
    eng.form_K(f, prior=prior, sigma2=s2)
    K_orc, _ = orc.form_k(f, g, s2, mode=1)
    assert orc.rel_err(eng.K(), K_orc) <= TOL
    eng.factorize()
    L_orc = orc.cholesky(K_orc)
    assert orc.rel_err(eng.chol_lower(), L_orc) <= TOL
    eng.form_Q(f, fq, prior=prior)
    Q, gp, pc = orc.form_q(f, fq, gq, L_orc)
    assert orc.rel_err(eng.Q(), Q) <= TOL
    assert orc.rel_err(eng.prior_qoi_cov(), pc) <= TOL


@pytest.mark.parametrize("n,seed", [(int(n), int(s)) for n, s in zip(
    np.random.default_rng(303).integers(1, 2500, 8), np.random.default_rng(304).integers(0, 2**31, 8))])
def test_solve_random_sizes(ltb, n, seed):
    import scipy.linalg as sl
    ident = np.zeros((n, n, 1))
    for i in range(n):
        ident[i, i, 0] = 1.0
    eng = ltb.InferenceEngine(ltb.MatvecPlan(ltb.BlockToeplitzKernel(n, n, 1, tag=ltb.KernelTag.Gstar, data=ident)))
    L = orc.gen_factor(seed % 1000, n)
    eng.set_factor(L)
    y = np.random.default_rng(seed).standard_normal(n)
    x = eng.solve_k_inplace(y.copy())
    ref = sl.solve_triangular(L.T, sl.solve_triangular(L, y, lower=True), lower=False)
    assert orc.rel_err(x, ref) <= TOL
