"""Re-entrancy and robustness of the online engine (the reference's const
contract): InferenceEngine::solve_k_inplace / infer_map are const and are
called concurrently from parallel_for workers -- form_Q
(bayes_engine.cpp:252-256) and the Hutchinson pointwise std (:386-389) -- so
concurrent calls on one engine, two engines on two streams at once, and
NaN / Inf data (the reference's Eigen TRSV just propagates them) must all give
the oracle's answer (<= 1e-12) promptly, with no dependency-wait timeouts."""
import threading
import time

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


def engine(ltb, nd, nm, nt, seed, nq=0, stream=None):
    g = ltb.MatvecPlan.generated(nd, nm, nt, seed=seed, tag=ltb.KernelTag.Gstar)
    fq = ltb.MatvecPlan.generated(nq, nm, nt, seed=seed, tag=ltb.KernelTag.Fq) if nq else None
    eng = ltb.InferenceEngine(g, fq, stream=stream)
    eng.set_factor_generated(seed)
    return eng, g, fq


def run_threads(fn, n):
    errs, res = [], [None] * n

    def body(i):
        try:
            res[i] = fn(i)
        except BaseException as exc:  # noqa: BLE001 -- reported below
            errs.append(exc)

    ts = [threading.Thread(target=body, args=(i,)) for i in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not errs, errs
    return res


def test_eight_threads_solve_k_one_engine(ltb):
    """The form_Q / pointwise_param_std pattern: 8 host threads, one engine,
    each solving its own right-hand sides repeatedly."""
    nd, nm, nt, seed = 32, 64, 64, 77  # n = 2048
    eng, _g, _fq = engine(ltb, nd, nm, nt, seed)
    n = nd * nt
    ys = [np.random.default_rng(100 + i).standard_normal(n) for i in range(8)]
    refs = [orc.solve_k_gen(seed, y) for y in ys]

    def work(i):
        worst = 0.0
        for _ in range(6):
            x = eng.solve_k_inplace(ys[i].copy())
            worst = max(worst, orc.rel_err(x, refs[i]))
        return worst

    t0 = time.time()
    errs = run_threads(work, 8)
    assert max(errs) <= TOL, errs
    assert time.time() - t0 < 60
    eng.close()


def test_threads_with_own_scratch_infer_and_forecast(ltb):
    """Concurrent infer_map + forecast, one Scratch (stream) per thread, as a
    parallel_for worker holds its own MatvecPlan::Scratch."""
    nd, nm, nt, nq, seed = 16, 300, 64, 4, 78
    eng, g, _fq = engine(ltb, nd, nm, nt, seed, nq=nq)
    ds = [np.random.default_rng(200 + i).standard_normal(nd * nt) for i in range(4)]
    gop = orc.OraclePlan(orc.gen_kernel(seed, nd, nm, nt, stream=3))
    fop = orc.OraclePlan(orc.gen_kernel(seed, nq, nm, nt, stream=2))
    refs = []
    for d in ds:
        m = gop.apply_adjoint(orc.solve_k_gen(seed, d))
        refs.append((m, fop.apply(m)))

    def work(i):
        sc = ltb.MatvecPlan.Scratch(g)
        worst = 0.0
        m, q = np.empty(nm * nt), np.empty(nq * nt)
        for _ in range(5):
            eng.infer_raw(ds[i], m, q, scratch=sc)
            worst = max(worst, orc.rel_err(m, refs[i][0]), orc.rel_err(q, refs[i][1]))
        sc.close()
        return worst

    errs = run_threads(work, 4)
    assert max(errs) <= TOL, errs
    eng.close()


def test_two_engines_two_streams_at_once(ltb):
    """Two engines (two persistent K^{-1} kernels that each fill the GPU),
    each driven from its own thread on its own stream."""
    import torch
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    e1, *_ = engine(ltb, 24, 40, 128, 81, stream=s1)   # n = 3072
    e2, *_ = engine(ltb, 40, 40, 120, 82, stream=s2)   # n = 4800
    y1 = np.random.default_rng(1).standard_normal(24 * 128)
    y2 = np.random.default_rng(2).standard_normal(40 * 120)
    r1, r2 = orc.solve_k_gen(81, y1), orc.solve_k_gen(82, y2)
    # device-pointer inputs as well (async on the engine's stream)
    t1 = torch.from_numpy(y1).cuda()
    t2 = torch.from_numpy(y2).cuda()

    def work(i):
        eng, y, r, t = (e1, y1, r1, t1) if i == 0 else (e2, y2, r2, t2)
        worst = 0.0
        for k in range(10):
            if k % 2:
                x = eng.solve_k_inplace(y.copy())
            else:
                tt = t.clone()
                eng.solve_k_inplace(tt)
                torch.cuda.synchronize()
                x = tt.cpu().numpy()
            worst = max(worst, orc.rel_err(x, r))
        return worst

    errs = run_threads(work, 2)
    assert max(errs) <= TOL, errs
    e1.close()
    e2.close()


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_data_propagates_promptly(ltb, bad):
    """A NaN / Inf in d reaches the result as in the reference's Eigen TRSV
    (forward substitution spreads it to every later entry) -- no 4 s
    dependency-wait timeout, no error -- and the engine stays usable."""
    nd, nm, nt, seed = 16, 64, 64, 83  # n = 1024: 16 blocks, 8-CTA chain
    eng, _g, _fq = engine(ltb, nd, nm, nt, seed)
    n = nd * nt
    y = np.random.default_rng(5).standard_normal(n)
    for pos in (0, 517, n - 1):
        yb = y.copy()
        yb[pos] = bad
        ref = orc.solve_k_gen(seed, yb)
        t0 = time.time()
        x = eng.solve_k_inplace(yb.copy())
        assert time.time() - t0 < 2.0
        # same non-finite pattern as the oracle (both sweeps spread it)
        assert np.array_equal(np.isfinite(x), np.isfinite(ref)), pos
        assert not np.all(np.isfinite(x))
        fin = np.isfinite(ref)
        if fin.any():
            assert orc.rel_err(x[fin], ref[fin]) <= TOL
    x = eng.solve_k_inplace(y.copy())  # still healthy
    assert orc.rel_err(x, orc.solve_k_gen(seed, y)) <= TOL
    eng.close()


def test_nan_in_infer_map_gives_nan_m(ltb):
    nd, nm, nt, seed = 8, 100, 32, 84
    eng, _g, _fq = engine(ltb, nd, nm, nt, seed)
    d = np.random.default_rng(6).standard_normal(nd * nt)
    d[3] = np.nan
    m = np.empty(nm * nt)
    eng.infer_raw(d, m)
    assert np.isnan(m).any()
    d[3] = 0.0
    eng.infer_raw(d, m)
    ref = orc.OraclePlan(orc.gen_kernel(seed, nd, nm, nt, stream=3)).apply_adjoint(orc.solve_k_gen(seed, d))
    assert orc.rel_err(m, ref) <= TOL
    eng.close()
