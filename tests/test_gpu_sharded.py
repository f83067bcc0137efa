"""MatvecPlan sharded over the GPUs of one process (ltb_plan_create_sharded,
SURVEY 8(b)/(e)) against the oracle: column shards on devs[k], F m summed
on the home device over NVLink peer mappings, F* d with d handed to every
shard.  On a one-GPU box the shards repeat device 0 (same code path, peer
reads of the same device); with >= 2 GPUs they span real devices."""
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


def device_sets():
    import torch
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    sets = [[0, 0], [0, 0, 0]]
    if n >= 2:
        sets += [[0, 1], [1, 0, 1]]
    if n >= 4:
        sets += [[0, 1, 2, 3]]
    return sets


@pytest.mark.parametrize("nd,nm,nt", [(8, 1024, 64), (5, 37, 17), (24, 1001, 100), (3, 20000, 112)])
def test_sharded_vs_oracle_host_pointers(ltb, nd, nm, nt):
    rng = np.random.default_rng(nd * 7 + nm + nt)
    k = rng.standard_normal((nd, nm, nt))
    m, d = rng.standard_normal(nm * nt), rng.standard_normal(nd * nt)
    op = orc.OraclePlan(k)
    fm_ref, ftd_ref = op.apply(m), op.apply_adjoint(d)
    single = ltb.MatvecPlan(ltb.BlockToeplitzKernel(nd, nm, nt, ltb.KernelTag.F, k))
    for devs in device_sets():
        sp = ltb.ShardedMatvecPlan(ltb.BlockToeplitzKernel(nd, nm, nt, ltb.KernelTag.F, k), devs)
        sh = sp.shards()
        assert [s[0] for s in sh] == devs and sh[0][1] == 0 and sh[-1][2] == nm
        assert all(sh[i][2] == sh[i + 1][1] for i in range(len(sh) - 1))
        s = ltb.ShardedMatvecPlan.Scratch(sp)
        fm, ftd = np.empty(nd * nt), np.empty(nm * nt)
        sp.apply_raw(m, fm, s)
        sp.apply_adjoint_raw(d, ftd, s)
        assert orc.rel_err(fm, fm_ref) <= TOL, devs
        assert orc.rel_err(ftd, ftd_ref) <= TOL, devs
        # repeat: bit-identical (fixed shard-order reduction)
        fm2 = np.empty_like(fm)
        sp.apply_raw(m, fm2, s)
        assert np.array_equal(fm, fm2)
        assert sp.kernel_hat_sqnorm() == pytest.approx(single.kernel_hat_sqnorm(), rel=1e-12)
        s.close()
        sp.close()


def test_sharded_device_pointers(ltb):
    """Device buffers on the home device: async on the home stream; F* d
    equals the host-pointer result bit for bit, F m to rounding."""
    import torch
    nd, nm, nt = 16, 3000, 96
    rng = np.random.default_rng(4)
    k = rng.standard_normal((nd, nm, nt))
    m, d = rng.standard_normal(nm * nt), rng.standard_normal(nd * nt)
    op = orc.OraclePlan(k)
    for devs in device_sets():
        sp = ltb.ShardedMatvecPlan(ltb.BlockToeplitzKernel(nd, nm, nt, ltb.KernelTag.F, k), devs)
        s = ltb.ShardedMatvecPlan.Scratch(sp)
        with torch.cuda.device(devs[0]):
            mt = torch.from_numpy(m).cuda()
            dt = torch.from_numpy(d).cuda()
            fo = torch.empty(nd * nt, dtype=torch.float64, device="cuda")
            ao = torch.empty(nm * nt, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            sp.apply_raw(mt, fo, s)
            sp.apply_adjoint_raw(dt, ao, s)
            s.sync()
            fo, ao = fo.cpu().numpy(), ao.cpu().numpy()
        assert orc.rel_err(fo, op.apply(m)) <= TOL
        assert orc.rel_err(ao, op.apply_adjoint(d)) <= TOL
        ah = np.empty(nm * nt)
        sp.apply_adjoint_raw(d, ah, s)
        assert np.array_equal(ah, ao)
        s.close()
        sp.close()


def test_sharded_generated_matches_single_plan(ltb):
    """Generated sharded plan (each shard its column range of one global
    generated kernel) == the single-device generated plan to rounding, and
    F* d on sampled columns vs the single-column oracle."""
    nd, nm, nt, seed = 32, 9000, 128, 21
    single = ltb.MatvecPlan.generated(nd, nm, nt, seed=seed)
    ss = ltb.MatvecPlan.Scratch(single)
    m = orc.gen_fill(seed, 10, nm * nt)
    d = orc.gen_fill(seed, 11, nd * nt)
    f1, a1 = np.empty(nd * nt), np.empty(nm * nt)
    single.apply_raw(m, f1, ss)
    single.apply_adjoint_raw(d, a1, ss)
    for devs in device_sets():
        sp = ltb.ShardedMatvecPlan.generated(nd, nm, nt, seed, devs)
        s = ltb.ShardedMatvecPlan.Scratch(sp)
        f2, a2 = np.empty(nd * nt), np.empty(nm * nt)
        sp.apply_raw(m, f2, s)
        sp.apply_adjoint_raw(d, a2, s)
        assert orc.rel_err(f2, f1) <= 1e-14
        assert orc.rel_err(a2, a1) <= 1e-14
        for c in [0, nm // len(devs), nm - 1]:
            opc = orc.OraclePlan(orc.gen_kernel(seed, nd, nm, nt, c0=c, cols=1))
            assert orc.rel_err(a2.reshape(nm, nt)[c], opc.apply_adjoint(d)) <= TOL
        s.close()
        sp.close()


def test_sharded_contract(ltb):
    k = np.ones((2, 3, 4))
    with pytest.raises(ltb.DimensionError):  # more shards than columns
        ltb.ShardedMatvecPlan(ltb.BlockToeplitzKernel(2, 3, 4, ltb.KernelTag.F, k), [0, 0, 0, 0])
    with pytest.raises(ValueError):
        ltb.ShardedMatvecPlan(ltb.BlockToeplitzKernel(2, 3, 4, ltb.KernelTag.F, k), [0, 99])
    sp = ltb.ShardedMatvecPlan(ltb.BlockToeplitzKernel(2, 3, 4, ltb.KernelTag.F, k), [0, 0])
    sp2 = ltb.ShardedMatvecPlan(ltb.BlockToeplitzKernel(2, 3, 4, ltb.KernelTag.F, k), [0, 0])
    s2 = ltb.ShardedMatvecPlan.Scratch(sp2)
    with pytest.raises(ValueError):  # scratch of another plan -> LTB_INVALID
        sp.apply_raw(np.zeros(12), np.zeros(8), s2)


def test_cascadia_sharded_two_gpus(ltb):
    """Config 4's layout at 2 GPUs: Nd=600, Nt=420, Nm=65536 (32768 columns,
    132.4 GB of F-hat per GPU) in one process; F* d on sampled columns of
    both shards and F m on column-supported m vs the oracle."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    nd, nm, nt, seed = 600, 65536, 420, 20250810
    sp = ltb.ShardedMatvecPlan.generated(nd, nm, nt, seed, [0, 1])
    s = ltb.ShardedMatvecPlan.Scratch(sp)
    d = orc.gen_fill(seed, 11, nd * nt)
    ftd = np.empty(nm * nt)
    sp.apply_adjoint_raw(d, ftd, s)
    ftd = ftd.reshape(nm, nt)
    for c in [0, 436, 32767, 32768, 40000, nm - 1]:
        opc = orc.OraclePlan(orc.gen_kernel(seed, nd, nm, nt, c0=c, cols=1))
        assert orc.rel_err(ftd[c], opc.apply_adjoint(d)) <= TOL, c
    sub = [7, 32768, 65535]
    rng = np.random.default_rng(2)
    msub = rng.standard_normal((len(sub), nt))
    m = np.zeros((nm, nt))
    m[sub] = msub
    fm = np.empty(nd * nt)
    sp.apply_raw(m.ravel(), fm, s)
    ker = np.concatenate([orc.gen_kernel(seed, nd, nm, nt, c0=c, cols=1) for c in sub], axis=1)
    assert orc.rel_err(fm, orc.OraclePlan(ker).apply(msub.ravel())) <= TOL
    s.close()
    sp.close()
