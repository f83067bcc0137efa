"""Distributed online phase vs the oracle (run under torchrun, one rank per
GPU; invoked by tests/test_gpu_dist.py when >= 2 GPUs are visible, or by
hand:  python -m torch.distributed.run --nproc-per-node 2 tests/dist_online_check.py).

Each rank holds a column shard of generated G* / F_q kernels and its
row-cyclic share of the synthetic Cholesky factor; m_map = G* K^{-1} d is
checked shard by shard against the oracle, q = F_q m_map (all-reduced)
against the oracle F_q applied to the oracle m_map.  Prints PASS / FAIL.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_16344_b200 as ltb  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (checker)
from paper_2504_16344_b200.dist import shard_range  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok = True
    for nd, nm, nt, nq, seed in [(16, 300, 64, 4, 11), (24, 130, 100, 3, 12)]:
        c0, c1 = shard_range(nm, world, rank)
        g = ltb.MatvecPlan.generated(nd, c1 - c0, nt, seed=seed, tag=ltb.KernelTag.Gstar,
                                     nm_total=nm, c0=c0)
        fq = ltb.MatvecPlan.generated(nq, c1 - c0, nt, seed=seed, tag=ltb.KernelTag.Fq,
                                      nm_total=nm, c0=c0)
        eng = ltb.InferenceEngine(g, fq, world=world, rank=rank)
        eng.set_factor_generated(seed)
        d = torch.from_numpy(orc.gen_fill(seed, 11, nd * nt)).cuda()
        m = torch.empty((c1 - c0) * nt, dtype=torch.float64, device="cuda")
        q = torch.empty(nq * nt, dtype=torch.float64, device="cuda")
        for _ in range(3):  # repeated solves exercise the epoch / sentinel re-arm
            eng.infer_raw(d, m, q)
            dist.all_reduce(q)
        y = orc.solve_k_gen(seed, orc.gen_fill(seed, 11, nd * nt))
        m_ref = orc.OraclePlan(orc.gen_kernel(seed, nd, nm, nt, stream=3)).apply_adjoint(y)
        q_ref = orc.OraclePlan(orc.gen_kernel(seed, nq, nm, nt, stream=2)).apply(m_ref)
        e_m = orc.rel_err(m.cpu().numpy(), m_ref[c0 * nt:c1 * nt])
        e_q = orc.rel_err(q.cpu().numpy(), q_ref)
        ok &= e_m <= 1e-12 and e_q <= 1e-12
        print("rank %d world %d n=%d: m shard %.2e  q %.2e" % (rank, world, nd * nt, e_m, e_q), flush=True)
        eng.close()
    flags = torch.tensor([1.0 if ok else 0.0], device="cuda")
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("PASS" if flags.item() == 1.0 else "FAIL", flush=True)
    dist.destroy_process_group()
    return 0 if flags.item() == 1.0 else 1


if __name__ == "__main__":
    sys.exit(main())
