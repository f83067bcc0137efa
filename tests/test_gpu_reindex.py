"""reindex (core.cpp:40-51) on the device: the TimeMajorBlocks <->
SpaceMajorRows permutation through ltb_reindex, bit-exact against the
oracle's restatement on ragged, tiny and Cascadia-sized series (the shape
cmd_infer reindexes on load, workflow.cpp:333), round trips exact, and the
layout contract of the reference (same layout -> copy)."""
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


@pytest.mark.parametrize("rows,nt", [(1, 1), (7, 5), (1, 37), (33, 1), (31, 33), (64, 128), (600, 420),
                                     (32768, 420)])
def test_reindex_bit_exact_vs_oracle(ltb, rows, nt):
    rng = np.random.default_rng(rows * 1000 + nt)
    v = ltb.SpaceTimeField(rows, nt, ltb.Layout.SpaceMajorRows, rng.standard_normal(rows * nt))
    tm = ltb.reindex(v, ltb.Layout.TimeMajorBlocks)
    assert tm.layout == ltb.Layout.TimeMajorBlocks
    assert np.array_equal(tm.values, orc.reindex(v.values, rows, nt, True))
    back = ltb.reindex(tm, ltb.Layout.SpaceMajorRows)
    assert np.array_equal(back.values, v.values)
    for r, j in [(0, 0), (rows - 1, nt - 1), (rows // 2, nt // 3)]:
        assert tm.values[tm.index(r, j)] == v.values[v.index(r, j)]
    same = ltb.reindex(v, ltb.Layout.SpaceMajorRows)  # same layout: a copy
    assert np.array_equal(same.values, v.values) and same.values is not v.values


def test_reindex_device_tensors(ltb):
    import torch
    rows, nt = 600, 420
    x = torch.randn(rows * nt, dtype=torch.float64, device="cuda")
    tm = ltb.reindex_device(x, rows, nt, ltb.Layout.SpaceMajorRows, ltb.Layout.TimeMajorBlocks)
    back = ltb.reindex_device(tm, rows, nt, ltb.Layout.TimeMajorBlocks, ltb.Layout.SpaceMajorRows)
    torch.cuda.synchronize()
    assert torch.equal(back, x)
    assert np.array_equal(tm.cpu().numpy(), orc.reindex(x.cpu().numpy(), rows, nt, True))


def test_reindex_contract(ltb):
    with pytest.raises(ltb.DimensionError):
        ltb.reindex(ltb.SpaceTimeField(3, 4, ltb.Layout.SpaceMajorRows, np.zeros(11)), ltb.Layout.TimeMajorBlocks)
