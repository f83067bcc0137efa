"""Device plan build from time-domain kernels with the prior premultiply
(G* = Gamma_prior F*, prior.cpp:108-134) and the BTPZ1 kernel-archive
loader (io.cpp:71-100), against the oracle."""
import struct

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


def write_btpz(path, k, tag=0):
    """io.cpp:71-82 byte layout."""
    with open(path, "wb") as fh:
        fh.write(b"BTPZ1")
        fh.write(struct.pack("<4Q", k.shape[0], k.shape[1], k.shape[2], tag))
        fh.write(np.ascontiguousarray(k, dtype="<f8").tobytes())


@pytest.mark.parametrize("rows,cols,nt,prior", [(3, 12, 5, (1.0, 2.0, 1.0)), (20, 300, 24, (1000.0, 16e6, 1.0)),
                                                (40, 64, 9, (0.5, 0.0, 3.0))])
def test_premultiplied_plan_vs_oracle(ltb, rows, cols, nt, prior):
    rng = np.random.default_rng(rows + cols)
    f = rng.standard_normal((rows, cols, nt))
    g = orc.prior_premultiply(f, *prior)
    gp = ltb.MatvecPlan.premultiplied(ltb.BlockToeplitzKernel(rows, cols, nt, tag=ltb.KernelTag.F, data=f), prior)
    assert gp.tag() == ltb.KernelTag.Gstar
    ref = orc.OraclePlan(g)
    assert orc.rel_err(gp.kernel_hat().view(np.float64), ref.khat().view(np.float64)) <= 1e-12
    d = rng.standard_normal(rows * nt)
    s = ltb.MatvecPlan.Scratch(gp)
    out = np.empty(cols * nt)
    gp.apply_adjoint_raw(d, out, s)
    assert orc.rel_err(out, ref.apply_adjoint(d)) <= 1e-12


def test_generated_premultiplied_vs_oracle(ltb):
    rows, cols, nt, seed, prior = 6, 40, 16, 77, (1.0, 2.0, 1.0)
    gp = ltb.MatvecPlan.generated_premultiplied(rows, cols, nt, seed, prior, tag=ltb.KernelTag.Fq)
    assert gp.tag() == ltb.KernelTag.Gqstar
    g = orc.prior_premultiply(orc.gen_kernel(seed, rows, cols, nt, stream=2), *prior)
    assert orc.rel_err(gp.kernel_hat().view(np.float64), orc.OraclePlan(g).khat().view(np.float64)) <= 1e-12


def test_premultiply_contract(ltb):
    k = ltb.BlockToeplitzKernel(2, 5, 4, tag=ltb.KernelTag.Gstar, data=np.ones((2, 5, 4)))
    with pytest.raises(ltb.ConfigError):
        ltb.MatvecPlan.premultiplied(k, (1.0, 1.0, 1.0))
    k = ltb.BlockToeplitzKernel(2, 5, 4, data=np.ones((2, 5, 4)))
    for bad in [(0.0, 1.0, 1.0), (1.0, -1.0, 1.0), (1.0, 1.0, 0.0)]:
        with pytest.raises(ltb.ConfigError):
            ltb.MatvecPlan.premultiplied(k, bad)


def test_btpz_loader_roundtrip(ltb, tmp_path):
    rng = np.random.default_rng(4)
    k = rng.standard_normal((7, 33, 11))
    path = tmp_path / "f.btpz"
    write_btpz(path, k, tag=1)
    lp = ltb.MatvecPlan.load(path)
    assert lp.tag() == ltb.KernelTag.Fq and (lp.rows_out(), lp.n_cols(), lp.n_time()) == (7, 33, 11)
    ref = ltb.MatvecPlan(ltb.BlockToeplitzKernel(7, 33, 11, tag=1, data=k))
    assert np.array_equal(lp.kernel_hat(), ref.kernel_hat())  # same bits in, same FFT
    lg = ltb.MatvecPlan.load(path, prior=(1.0, 2.0, 1.0))
    assert lg.tag() == ltb.KernelTag.Gqstar
    g = orc.prior_premultiply(k, 1.0, 2.0, 1.0)
    assert orc.rel_err(lg.kernel_hat().view(np.float64), orc.OraclePlan(g).khat().view(np.float64)) <= 1e-12


def test_btpz_loader_errors(ltb, tmp_path):
    bad = tmp_path / "bad.btpz"
    bad.write_bytes(b"XXXXX" + b"\0" * 40)
    with pytest.raises(ltb.IoError):
        ltb.MatvecPlan.load(bad)
    with pytest.raises(ltb.IoError):
        ltb.MatvecPlan.load(tmp_path / "missing.btpz")
    k = np.ones((2, 3, 4))
    trunc = tmp_path / "trunc.btpz"
    write_btpz(trunc, k)
    trunc.write_bytes(trunc.read_bytes()[:-8])
    with pytest.raises(ltb.IoError):
        ltb.MatvecPlan.load(trunc)
    nan = tmp_path / "nan.btpz"
    k[1, 2, 3] = np.nan
    write_btpz(nan, k)
    with pytest.raises(ltb.NumericalError):
        ltb.MatvecPlan.load(nan)


def write_dnsm(path, m, symmetric=False):
    """io.cpp:102-115 byte layout (row-major)."""
    m = np.asarray(m, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(b"DNSM1")
        fh.write(struct.pack("<3Q", m.shape[0], m.shape[1], int(symmetric)))
        fh.write(np.ascontiguousarray(m).tobytes())


def fnv1a64(data):
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def test_dnsm_factor_and_phase3_loaders(ltb, tmp_path):
    import ctypes as C
    import scipy.linalg as sl
    from paper_2504_16344_b200 import _lib
    nd, nq, nm, nt = 3, 2, 5, 30  # n = 90: two 64-blocks, ragged
    n = nd * nt
    g = ltb.MatvecPlan.generated(nd, nm, nt, seed=2, tag=ltb.KernelTag.Gstar)
    fq = ltb.MatvecPlan.generated(nq, nm, nt, seed=2, tag=ltb.KernelTag.Fq)
    eng = ltb.InferenceEngine(g, fq)
    rng = np.random.default_rng(0)
    L = orc.gen_factor(5, n)
    stored = L + np.triu(rng.standard_normal((n, n)), 1)  # upper part must be ignored
    write_dnsm(tmp_path / "chol.dnsm", stored)
    eng.load_factor(tmp_path / "chol.dnsm")
    y = rng.standard_normal(n)
    ref = sl.solve_triangular(L, sl.solve_triangular(L, y, lower=True), lower=True, trans="T")
    assert orc.rel_err(eng.solve_k_inplace(y.copy()), ref) <= 1e-12
    Q = rng.standard_normal((nq * nt, n))
    G = rng.standard_normal((nq * nt, nq * nt))
    G = G @ G.T
    write_dnsm(tmp_path / "Q.dnsm", Q)
    write_dnsm(tmp_path / "Gpost.dnsm", G, symmetric=True)
    eng.load_phase3(tmp_path / "Q.dnsm", tmp_path / "Gpost.dnsm")
    res = eng.predict_qoi(ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, y))
    assert orc.rel_err(res.q_map.values, Q @ y) <= 1e-13
    assert np.allclose(res.ci_upper.values - res.q_map.values, 1.96 * np.sqrt(np.diag(G)), rtol=1e-12)
    # FNV-1a over the archive bytes (io.cpp:198-219)
    h = C.c_uint64()
    assert _lib.load().ltb_fnv1a64_file(str(tmp_path / "Q.dnsm").encode(), C.byref(h)) == 0
    assert h.value == fnv1a64((tmp_path / "Q.dnsm").read_bytes())
    with pytest.raises(ltb.DimensionError):
        write_dnsm(tmp_path / "small.dnsm", np.eye(4))
        eng.load_factor(tmp_path / "small.dnsm")
    with pytest.raises(ltb.IoError):
        eng.load_factor(tmp_path / "none.dnsm")


def test_device_built_artifacts_roundtrip(ltb, tmp_path):
    """form_K -> factorize -> form_Q on the device, the reference's artifact
    set written (workflow.cpp:256-264 names), then a fresh engine built from
    those files (MatvecPlan.load, load_factor, load_phase3) predicts the same
    posterior mean and QoI intervals."""
    nd, nq, nm, nt, s2, prior = 4, 2, 48, 16, 0.3, (1.0, 2.0, 1.0)
    rng = np.random.default_rng(21)
    f = rng.standard_normal((nd, nm, nt)) * 0.9 ** np.arange(nt)
    fq = rng.standard_normal((nq, nm, nt)) * 0.9 ** np.arange(nt)
    kf = ltb.BlockToeplitzKernel(nd, nm, nt, tag=ltb.KernelTag.F, data=f)
    kq = ltb.BlockToeplitzKernel(nq, nm, nt, tag=ltb.KernelTag.Fq, data=fq)
    eng = ltb.InferenceEngine(ltb.MatvecPlan.premultiplied(kf, prior), ltb.MatvecPlan(kq))
    eng.form_K(f, prior=prior, sigma2=s2)
    K = eng.K()
    eng.factorize()
    eng.form_Q(f, fq, prior=prior)
    ltb.write_engine_artifacts(tmp_path, eng, f_kernel=kf, fq_kernel=kq, K=K)
    assert sorted(p.name for p in tmp_path.iterdir()) == sorted(
        ["K.dnsm", "chol.dnsm", "Q.dnsm", "gamma_post_q.dnsm", "prior_qoi_cov.dnsm", "f.btpz", "fq.btpz",
         "manifest.txt"])
    man = ltb.read_manifest(tmp_path / "manifest.txt")
    assert [e[0] for e in man.artifacts] == ["f.btpz", "fq.btpz", "K.dnsm", "chol.dnsm", "Q.dnsm",
                                             "gamma_post_q.dnsm", "prior_qoi_cov.dnsm"]
    assert ltb.verify_manifest(tmp_path, man) is None
    eng2 = ltb.InferenceEngine(ltb.MatvecPlan.load(tmp_path / "f.btpz", prior=prior),
                               ltb.MatvecPlan.load(tmp_path / "fq.btpz"))
    eng2.load_factor(tmp_path / "chol.dnsm")
    eng2.load_phase3(tmp_path / "Q.dnsm", tmp_path / "gamma_post_q.dnsm")
    d = ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, rng.standard_normal(nd * nt))
    a, b = eng.infer_map(d, with_forecast=True), eng2.infer_map(d, with_forecast=True)
    assert np.array_equal(a.m_map.values, b.m_map.values)
    assert np.array_equal(a.q_map.values, b.q_map.values)
    pa, pb = eng.predict_qoi(d), eng2.predict_qoi(d)
    assert np.array_equal(pa.q_map.values, pb.q_map.values)
    assert np.array_equal(pa.ci_upper.values, pb.ci_upper.values)


def test_infer_from_artifacts_like_cmd_infer(ltb, tmp_path):
    """workflow.cpp:300-380 (cmd_infer) over the library: artifacts written
    from a device-built engine + a d_obs series file -> m_map.f64, the
    displacement / QoI CSVs and latency.txt, equal to the engine's own
    results."""
    nd, nq, nm, nt, s2, prior, dt = 3, 2, 40, 12, 0.3, (1.0, 2.0, 1.0), 0.5
    rng = np.random.default_rng(33)
    f = rng.standard_normal((nd, nm, nt)) * 0.9 ** np.arange(nt)
    fq = rng.standard_normal((nq, nm, nt)) * 0.9 ** np.arange(nt)
    kf = ltb.BlockToeplitzKernel(nd, nm, nt, tag=ltb.KernelTag.F, data=f)
    kq = ltb.BlockToeplitzKernel(nq, nm, nt, tag=ltb.KernelTag.Fq, data=fq)
    eng = ltb.InferenceEngine(ltb.MatvecPlan.premultiplied(kf, prior), ltb.MatvecPlan(kq))
    eng.form_K(f, prior=prior, sigma2=s2)
    eng.factorize()
    eng.form_Q(f, fq, prior=prior)
    ltb.write_engine_artifacts(tmp_path, eng, f_kernel=kf, fq_kernel=kq, meta=[("sigma2", repr(s2))])
    d = ltb.ObsSeries(nd, nt, ltb.Layout.SpaceMajorRows, rng.standard_normal(nd * nt))
    ltb.write_series(tmp_path / "d_obs.f64", ltb.reindex(d, ltb.Layout.TimeMajorBlocks))
    out = ltb.infer_from_artifacts(str(tmp_path), tmp_path / "d_obs.f64", None, prior, dt)  # sigma2 from meta
    ref = eng.infer_map(d)
    assert np.array_equal(out["m_map"].values, ref.m_map.values)
    m = ltb.read_series(tmp_path / "m_map.f64", ltb.SpaceTimeField)
    assert np.array_equal(m.values, ref.m_map.values)
    assert out["smw_rel_residual"] <= 1e-8
    disp = np.loadtxt(tmp_path / "map_displacement.csv", delimiter=",", skiprows=1, usecols=(0, 1))
    assert np.allclose(disp[:, 1], dt * ref.m_map.values.reshape(nm, nt).sum(axis=1), rtol=1e-13, atol=1e-15)
    qcsv = np.loadtxt(tmp_path / "qoi_forecast.csv", delimiter=",", skiprows=1)
    assert qcsv.shape == (nq * nt, 5)
    assert np.allclose(qcsv[:, 2], eng.predict_qoi(d).q_map.values, rtol=1e-15, atol=0)
    assert "smw_rel_residual" in (tmp_path / "latency.txt").read_text()
    # an artifact altered after the manifest was written: stale, as cmd_infer
    q = bytearray((tmp_path / "Q.dnsm").read_bytes())
    q[-1] ^= 0x10
    (tmp_path / "Q.dnsm").write_bytes(bytes(q))
    with pytest.raises(ltb.StateError, match="Q.dnsm"):
        ltb.infer_from_artifacts(str(tmp_path), tmp_path / "d_obs.f64", s2, prior, dt)
