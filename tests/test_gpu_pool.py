"""Scratch reuse: the reference builds a fresh MatvecPlan::Scratch for every
apply(m) (fft_matvec.cpp:232-235), infer_map (bayes_engine.cpp:317) and
form_K column (:144).  ltb_scratch_destroy parks the workspaces in the plan's
pool and ltb_scratch_create hands them back, fenced by an event on the
previous owner's stream -- results must not change, a Scratch may outlive its
plan (as in the reference), and a reference-style call must cost about what
a reused Scratch costs."""
import time

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


def test_fresh_scratch_per_call_is_bit_identical(ltb):
    import torch
    nd, nm, nt, seed = 16, 4000, 128, 5
    plan = ltb.MatvecPlan.generated(nd, nm, nt, seed=seed)
    m = orc.gen_fill(seed, 10, nm * nt)
    d = orc.gen_fill(seed, 11, nd * nt)
    s0 = ltb.MatvecPlan.Scratch(plan)
    f0, a0 = np.empty(nd * nt), np.empty(nm * nt)
    plan.apply_raw(m, f0, s0)
    plan.apply_adjoint_raw(d, a0, s0)
    s0.close()
    side = torch.cuda.Stream()
    for i in range(20):
        # alternate private streams and a caller stream across pool reuses
        s = ltb.MatvecPlan.Scratch(plan, stream=side if i % 3 == 0 else None)
        f, a = np.empty(nd * nt), np.empty(nm * nt)
        plan.apply_raw(m, f, s)
        plan.apply_adjoint_raw(d, a, s)
        s.close()
        assert np.array_equal(f, f0) and np.array_equal(a, a0), i
    # device-pointer work still queued when the scratch is released: the next
    # owner (another stream) must wait for it
    mt = torch.from_numpy(m).cuda()
    outs = []
    for i in range(4):
        s = ltb.MatvecPlan.Scratch(plan, stream=side if i % 2 else None)
        o = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
        plan.apply_raw(mt, o, s)
        s.close()  # no sync: released with the work in flight
        outs.append(o)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), f0)
    assert orc.rel_err(f0, orc.OraclePlan(orc.gen_kernel(seed, nd, nm, nt)).apply(m)) <= 1e-12


def test_scratch_outlives_plan(ltb):
    plan = ltb.MatvecPlan.generated(4, 100, 16, seed=1)
    s = ltb.MatvecPlan.Scratch(plan)
    s2 = ltb.MatvecPlan.Scratch(plan)
    s2.close()  # pooled
    plan.close()  # frees the pooled one, detaches the pool
    s.close()  # plan gone: freed, not pooled


def test_reference_style_call_cost(ltb):
    """apply(m) with a fresh Scratch (typed API, no scratch argument) costs
    about the same as with a reused one once the pool is warm."""
    nd, nm, nt = 64, 16384, 128  # config 2 shape
    plan = ltb.MatvecPlan.generated(nd, nm, nt, seed=4321)
    m = ltb.SpaceTimeField(nm, nt, ltb.Layout.SpaceMajorRows, orc.gen_fill(4321, 10, nm * nt))
    s = ltb.MatvecPlan.Scratch(plan)
    for _ in range(3):
        plan.apply(m, s)
        plan.apply(m)

    def best(fn, n=15):
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    reused = best(lambda: plan.apply(m, s))
    fresh = best(lambda: plan.apply(m))
    print("apply(m): reused scratch %.3f ms, fresh scratch %.3f ms" % (reused * 1e3, fresh * 1e3))
    assert fresh <= reused * 1.10 + 2e-4
