"""World-size-2 gloo test (CPU) of the Nm-sharding host logic in
paper_2504_16344_b200/dist.py: shard ranges, the all-reduce of F m and the
broadcast of d for F* d reproduce the unsharded operator.  The local shard
operator is the CPU oracle (the GPU shard is exercised by bench.py on the
box); this checks the decomposition and collectives, not the kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_2504_16344_b200.dist import ShardedMatvec, shard_range

ND, NM, NT, SEED = 5, 23, 12, 77


class OracleShard:
    """CPU stand-in for a MatvecPlan shard (test only)."""

    def __init__(self, c0, c1):
        self.plan = orc.OraclePlan(orc.gen_kernel(SEED, ND, NM, NT, c0=c0, cols=c1 - c0))

    def apply_raw(self, m, out, scratch):
        out.copy_(torch.from_numpy(self.plan.apply(m.numpy())))

    def apply_adjoint_raw(self, d, out, scratch):
        out.copy_(torch.from_numpy(self.plan.apply_adjoint(d.numpy())))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c0, c1 = shard_range(NM, world, rank)
        sm = ShardedMatvec(ND, NM, NT, SEED, local=OracleShard(c0, c1))
        m = torch.from_numpy(orc.gen_fill(SEED, 10, NM * NT))
        d_out = torch.empty(ND * NT, dtype=torch.float64)
        sm.apply(m[c0 * NT:c1 * NT].clone(), d_out)
        d = torch.from_numpy(orc.gen_fill(SEED, 11, ND * NT)) if rank == 0 else torch.zeros(ND * NT, dtype=torch.float64)
        m_out = torch.empty((c1 - c0) * NT, dtype=torch.float64)
        sm.apply_adjoint(d, m_out)
        parts = [None] * world
        dist.all_gather_object(parts, (c0, c1, m_out.numpy()))
        q.put((rank, d_out.numpy(), parts))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover_exactly():
    for nm in (1, 7, 23, 32768):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(nm, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == nm
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_sharded_matches_unsharded_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = orc.OraclePlan(orc.gen_kernel(SEED, ND, NM, NT))
    m = orc.gen_fill(SEED, 10, NM * NT)
    d = orc.gen_fill(SEED, 11, ND * NT)
    ref_f, ref_a = full.apply(m), full.apply_adjoint(d)
    for rank, d_out, parts in res:
        assert orc.rel_err(d_out, ref_f) <= 1e-13
        m_all = np.concatenate([p[2] for p in sorted(parts, key=lambda t: t[0])])
        assert orc.rel_err(m_all, ref_a) <= 1e-14
