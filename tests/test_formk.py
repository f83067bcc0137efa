"""form_K + factorize (offline phase 2, bayes_engine.cpp:136-209) on the
device vs the oracle, restating proj/tests/test_bayes_engine.cpp:
identity maps (:86-107), diagonal examples + random SPD (:109-124), column
vs fused paths + dense oracle + asymmetry (:126-143), and the full pipeline
(form_K -> factorize -> infer_map)."""
import numpy as np
import pytest

from oracle import oracle as orc

PRIOR = (1.0, 2.0, 1.0)  # (h_x, gamma, delta) as random_instance (:40)


def gamma_x(nm, h_x, gamma, delta):
    """Dense Gamma_x = A_x^{-2}, A_x = delta I - gamma L_Neumann / h_x^2
    (prior.cpp:9-39), built independently of the oracle."""
    w = gamma / (h_x * h_x)
    A = np.zeros((nm, nm))
    for i in range(nm):
        A[i, i] = delta + w * ((i > 0) + (i + 1 < nm))
        if i > 0:
            A[i, i - 1] = A[i - 1, i] = -w
    Ai = np.linalg.inv(A)
    return Ai @ Ai


def dense_f(f):
    """materialize_dense: (nd nt) x (nm nt), SpaceMajorRows both sides."""
    nd, nm, nt = f.shape
    Fd = np.zeros((nd * nt, nm * nt))
    for r in range(nd):
        for x in range(nm):
            for t in range(nt):
                for tau in range(t + 1):
                    Fd[r * nt + t, x * nt + tau] = f[r, x, t - tau]
    return Fd


def lti_like(rng, nd, nm, nt):
    """Decaying impulse responses (lti_impulse_kernel flavour)."""
    decay = 0.85 ** np.arange(nt)
    return rng.standard_normal((nd, nm, nt)) * decay


# ---------------------------------------------------------------- CPU (oracle)
def test_oracle_form_k_paths_and_dense():
    """:126-143 -- column and fused assembly agree, asymmetry tiny, and K
    equals sigma2 I + F Gamma_prior F^T (dense)."""
    rng = np.random.default_rng(1234)
    nd, nm, nt, s2 = 3, 4, 6, 0.3
    f = lti_like(rng, nd, nm, nt)
    g = orc.prior_premultiply(f, *PRIOR)
    K1, asym = orc.form_k(f, g, s2, mode=0)
    K2, _ = orc.form_k(f, g, s2, mode=1)
    assert orc.rel_err(K2, K1) <= 1e-12
    assert asym <= 1e-11
    Fd = dense_f(f)
    Gp = np.kron(gamma_x(nm, *PRIOR), np.eye(nt))  # SpaceMajorRows: x major, t minor
    K_ref = s2 * np.eye(nd * nt) + Fd @ Gp @ Fd.T
    assert orc.rel_err(K1, K_ref) <= 1e-10


def test_oracle_cholesky():
    rng = np.random.default_rng(77)
    M = rng.standard_normal((40, 40))
    K = M @ M.T + 40 * np.eye(40)
    L = orc.cholesky(K)
    assert np.all(np.triu(L, 1) == 0.0)
    assert orc.rel_err(L @ L.T, K) <= 1e-14
    assert orc.rel_err(L, np.linalg.cholesky(K)) <= 1e-13
    with pytest.raises(ValueError):
        orc.cholesky(-np.eye(3))


# ---------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def ltb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_16344_b200 as ltb
    ltb.load()
    return ltb


def engine_for(ltb, f, prior=PRIOR):
    kern = ltb.BlockToeplitzKernel(*f.shape, tag=ltb.KernelTag.F, data=f)
    plan_g = ltb.MatvecPlan.premultiplied(kern, prior)
    return ltb.InferenceEngine(plan_g), plan_g


@pytest.mark.gpu
def test_identity_maps(ltb):
    """:86-107 -- F = I, Gamma = I: K = (1 + s2) I, chol = sqrt(1 + s2) I,
    m_map = d / (1 + s2)."""
    n, nt, s2 = 3, 4, 0.25
    f = np.zeros((n, n, nt))
    for i in range(n):
        f[i, i, 0] = 1.0
    eng, _pg = engine_for(ltb, f, prior=(1.0, 0.0, 1.0))
    eng.form_K(f, prior=(1.0, 0.0, 1.0), sigma2=s2)
    assert np.linalg.norm(eng.K() - (1 + s2) * np.eye(n * nt)) <= 1e-12
    eng.factorize()
    assert np.linalg.norm(eng.chol_lower() - np.sqrt(1 + s2) * np.eye(n * nt)) <= 1e-12
    d = np.random.default_rng(2).standard_normal(n * nt)
    res = eng.infer_map(ltb.ObsSeries(n, nt, ltb.Layout.SpaceMajorRows, d))
    assert np.allclose(res.m_map.values, d / (1 + s2), rtol=1e-12, atol=0)


@pytest.mark.gpu
def test_factorize_diagonal_and_state(ltb):
    """:109-124 -- K = 4 I -> L = 2 I; factorize before form_K is a
    StateError; a K that is not SPD raises NumericalError."""
    n, nt = 2, 3
    f = np.zeros((n, n, nt))
    for i in range(n):
        f[i, i, 0] = 1.0
    eng, _pg = engine_for(ltb, f, prior=(1.0, 0.0, 1.0))
    with pytest.raises(ltb.StateError):
        eng.factorize()
    with pytest.raises(ltb.StateError):
        eng.K()
    eng.form_K(f, prior=(1.0, 0.0, 1.0), sigma2=3.0)
    eng.factorize()
    assert np.linalg.norm(eng.chol_lower() - 2.0 * np.eye(n * nt)) <= 1e-12
    with pytest.raises(ltb.StateError):  # K was overwritten in place
        eng.factorize()
    eng.form_K(f, prior=(1.0, 0.0, 1.0), sigma2=-5.0)
    with pytest.raises(ltb.NumericalError):
        eng.factorize()


@pytest.mark.gpu
@pytest.mark.parametrize("nd,nm,nt", [(3, 4, 6), (8, 300, 50), (5, 64, 33), (16, 1024, 64),
                                      (2, 40, 129), (20, 64, 128)])
def test_form_k_factorize_vs_oracle(ltb, nd, nm, nt):
    """K (DMMA lag Gram + diagonal recurrence) vs the oracle's column-by-
    column FFT assembly; L vs the oracle Cholesky; ragged n, odd N_t (8-byte
    operand path), N_m not a multiple of the 16-wide k-stage, and (n = 2560:
    210 CTA tiles) the split-k last wave."""
    rng = np.random.default_rng(nd * 1000 + nm + nt)
    s2 = 0.3
    f = lti_like(rng, nd, nm, nt)
    g = orc.prior_premultiply(f, *PRIOR)
    K_orc, _ = orc.form_k(f, g, s2, mode=1)
    eng, _pg = engine_for(ltb, f)
    eng.form_K(f, prior=PRIOR, sigma2=s2)
    K = eng.K()
    assert orc.rel_err(K, K_orc) <= 1e-12
    # explicit G kernel (host) gives the same K
    eng.form_K(f, g_kernel=g, sigma2=s2)
    assert orc.rel_err(eng.K(), K_orc) <= 1e-12
    eng.factorize()
    L = eng.chol_lower()
    L_orc = orc.cholesky(K_orc)
    assert np.all(np.triu(L, 1) == 0.0)
    assert orc.rel_err(L, L_orc) <= 1e-12
    assert orc.rel_err(L @ L.T, K_orc) <= 1e-12
    # the factor drives the online solve
    y = rng.standard_normal(nd * nt)
    x = eng.solve_k_inplace(y.copy())
    assert orc.rel_err(x, orc.solve_k(L_orc, y)) <= 1e-12
    fk, fz = eng.offline_ms()
    assert fk > 0 and fz > 0


@pytest.mark.gpu
def test_device_kernels_and_pipeline(ltb):
    """CUDA-tensor kernels; form_K -> factorize -> infer_map vs the oracle
    chain (oracle K, oracle Cholesky, oracle infer_map) within 1e-10."""
    import torch
    nd, nm, nt, s2 = 4, 96, 32, 0.3
    rng = np.random.default_rng(5)
    f = lti_like(rng, nd, nm, nt)
    g = orc.prior_premultiply(f, *PRIOR)
    eng, plan_g = engine_for(ltb, f)
    ft = torch.from_numpy(f).cuda()
    gt = torch.from_numpy(g).cuda()
    eng.form_K(ft, g_kernel=gt, sigma2=s2)
    eng.factorize()
    K_orc, _ = orc.form_k(f, g, s2, mode=0)
    L_orc = orc.cholesky(K_orc)
    d = rng.standard_normal(nd * nt)
    res = eng.infer_map(ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, d))
    m_orc = orc.OraclePlan(g).apply_adjoint(orc.solve_k(L_orc, d))
    assert orc.rel_err(res.m_map.values, m_orc) <= 1e-10


@pytest.mark.gpu
def test_generated_small_inversion_config(ltb):
    """Config 2 (N_d=64, N_m=16384, N_t=128, n=8192) fully on the device:
    form_K of the generated F, factorize, then size-independent checks
    against the (oracle-verified) matvec path: L L^T x == F G* x + s2 x and
    K^{-1} (K x) == x."""
    nd, nm, nt, seed, s2 = 64, 16384, 128, 4321, 1.0
    prior = (1.0, 2.0, 1.0)
    pf = ltb.MatvecPlan.generated(nd, nm, nt, seed, tag=ltb.KernelTag.F)
    pg = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, seed, prior, tag=ltb.KernelTag.F)
    eng = ltb.InferenceEngine(pg)
    eng.form_K_generated(seed, 1, prior, s2)
    n = nd * nt
    rng = np.random.default_rng(9)
    x = rng.standard_normal(n)
    Kx = pf.apply(ltb.SpaceTimeField(nm, nt, ltb.Layout.SpaceMajorRows,
                                      pg.apply_adjoint(ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows,
                                                                     x)).values)).values + s2 * x
    Kl = eng.K_lower()
    Kx_dev = Kl @ x + np.tril(Kl, -1).T @ x
    assert orc.rel_err(Kx_dev, Kx) <= 1e-12
    del Kl
    eng.factorize()
    L = eng.chol_lower()
    assert orc.rel_err(L @ (L.T @ x), Kx) <= 1e-12
    del L
    back = eng.solve_k_inplace(Kx.copy())
    assert orc.rel_err(back, x) <= 1e-9
    fk, fz = eng.offline_ms()
    print("config2 form_K %.2f ms (%.1f TFLOP/s lag Gram), factorize %.2f ms" %
          (fk, n * n * nm / fk / 1e9, fz))


# ---------------------------------------------------------------- form_Q
@pytest.mark.gpu
@pytest.mark.parametrize("nd,nq,nm,nt", [(2, 2, 4, 5), (4, 3, 40, 33), (8, 2, 300, 64), (16, 4, 256, 48)])
def test_form_q_vs_oracle(ltb, nd, nq, nm, nt):
    """form_Q + form_qoi_cov (bayes_engine.cpp:242-285) on the device vs the
    oracle (column-by-column FFT assembly, per-column solve_k): Q, Gamma_post_q
    and the prior QoI covariance within 1e-12; then predict_qoi with the
    device-made artifacts equals F_q m_map (the Phase-4 chain identity)."""
    rng = np.random.default_rng(nd * 100 + nq * 10 + nt)
    s2 = 0.3
    f = lti_like(rng, nd, nm, nt)
    fq = lti_like(rng, nq, nm, nt)
    g = orc.prior_premultiply(f, *PRIOR)
    gq = orc.prior_premultiply(fq, *PRIOR)
    kern_fq = ltb.BlockToeplitzKernel(*fq.shape, tag=ltb.KernelTag.Fq, data=fq)
    plan_fq = ltb.MatvecPlan(kern_fq)
    kern = ltb.BlockToeplitzKernel(*f.shape, tag=ltb.KernelTag.F, data=f)
    plan_g = ltb.MatvecPlan.premultiplied(kern, PRIOR)
    eng = ltb.InferenceEngine(plan_g, plan_fq)
    with pytest.raises(ltb.StateError):  # needs the factor
        eng.form_Q(f, fq, prior=PRIOR)
    eng.form_K(f, prior=PRIOR, sigma2=s2)
    eng.factorize()
    eng.form_Q(f, fq, prior=PRIOR)
    L = eng.chol_lower()
    Q_o, gp_o, pc_o = orc.form_q(f, fq, gq, L)
    assert orc.rel_err(eng.Q(), Q_o) <= 1e-12
    assert orc.rel_err(eng.prior_qoi_cov(), pc_o) <= 1e-12
    assert orc.rel_err(eng.gamma_post_q(), gp_o) <= 1e-12
    # explicit Gq kernel gives the same operator
    eng.form_Q(f, fq, gq_kernel=gq)
    assert orc.rel_err(eng.Q(), Q_o) <= 1e-12
    assert eng.form_Q_ms() > 0
    d = rng.standard_normal(nd * nt)
    obs = ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, d)
    pred = eng.predict_qoi(obs)
    res = eng.infer_map(obs, with_forecast=True)
    assert orc.rel_err(pred.q_map.values, res.q_map.values) <= 1e-10  # Q d == F_q m_map
    sd = np.sqrt(np.maximum(np.diag(gp_o), 0))
    assert np.allclose(pred.ci_upper.values - pred.q_map.values, 1.96 * sd, rtol=1e-10, atol=1e-14)


@pytest.mark.gpu
def test_form_q_generated_small_inversion(ltb):
    """Config 2 with N_q = 8 fully on the device (form_K -> factorize ->
    form_Q -> predict_qoi); size-independent checks: Q d == F_q m_map and
    diag(Gamma_post_q) <= diag(prior QoI covariance) (data only reduces
    variance)."""
    nd, nm, nt, nq, seed, s2 = 64, 16384, 128, 8, 4321, 1.0
    prior = (1.0, 2.0, 1.0)
    pg = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, seed, prior, tag=ltb.KernelTag.F)
    fq = ltb.MatvecPlan.generated(nq, nm, nt, seed, tag=ltb.KernelTag.Fq)
    eng = ltb.InferenceEngine(pg, fq)
    eng.form_K_generated(seed, 1, prior, s2)
    eng.factorize()
    eng.form_Q_generated(seed, nq, prior)
    rng = np.random.default_rng(3)
    obs = ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, rng.standard_normal(nd * nt))
    pred = eng.predict_qoi(obs)
    res = eng.infer_map(obs, with_forecast=True)
    assert orc.rel_err(pred.q_map.values, res.q_map.values) <= 1e-9
    gp, pc = eng.gamma_post_q(), eng.prior_qoi_cov()
    assert np.all(np.diag(gp) <= np.diag(pc) * (1 + 1e-12))
    assert np.all(np.diag(gp) > 0)
    print("config2 form_Q (N_q=8) %.2f ms" % eng.form_Q_ms())
