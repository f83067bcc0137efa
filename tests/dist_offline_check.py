"""Distributed offline phase 2 + online phase on P GPUs (torchrun, one rank
per GPU; invoked by tests/test_gpu_dist.py when >= 2 GPUs are visible):
every rank forms its block rows of K = F G* + s2 I (lag Gram + the
recurrence carried rank to rank), the ranks factorize it together (panel
broadcast / all-gather over NCCL), and the distributed K^{-1} + sharded G* /
F_q run on that real factor.  Checked against the one-GPU path on every
rank (m_map shard, q after the all-reduce) and, on rank 0, the factor's
block rows against the one-GPU factor.  Prints PASS / FAIL."""
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

PRIOR = (1.0, 2.0, 1.0)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok = True
    for nd, nm, nt, nq, seed, s2 in [(16, 300, 64, 4, 41, 0.7), (10, 200, 50, 3, 42, 1.3), (24, 512, 96, 2, 43, 0.5)]:
        c0, c1 = shard_range(nm, world, rank)
        g = ltb.MatvecPlan.generated_premultiplied(nd, c1 - c0, nt, seed, PRIOR, nm_total=nm, c0=c0)
        fq = ltb.MatvecPlan.generated(nq, c1 - c0, nt, seed=seed, tag=ltb.KernelTag.Fq, nm_total=nm, c0=c0)
        eng = ltb.InferenceEngine(g, fq, world=world, rank=rank)
        eng.form_K_generated(seed, 1, PRIOR, s2, nm_total=nm)
        eng.factorize()
        d = torch.from_numpy(np.random.default_rng(seed).standard_normal(nd * nt)).cuda()
        m = torch.empty((c1 - c0) * nt, dtype=torch.float64, device="cuda")
        q = torch.empty(nq * nt, dtype=torch.float64, device="cuda")
        for _ in range(2):
            eng.infer_raw(d, m, q)
            dist.all_reduce(q)
        # the one-GPU reference on this rank
        gf = ltb.MatvecPlan.generated_premultiplied(nd, nm, nt, seed, PRIOR)
        fqf = ltb.MatvecPlan.generated(nq, nm, nt, seed=seed, tag=ltb.KernelTag.Fq)
        one = ltb.InferenceEngine(gf, fqf)
        one.form_K_generated(seed, 1, PRIOR, s2)
        one.factorize()
        mh, qh = np.empty(nm * nt), np.empty(nq * nt)
        one.infer_raw(d.cpu().numpy(), mh, qh)
        e_m = orc.rel_err(m.cpu().numpy(), mh[c0 * nt:c1 * nt])
        e_q = orc.rel_err(q.cpu().numpy(), qh)
        ok &= e_m <= 1e-12 and e_q <= 1e-12
        print("rank %d world %d n=%d: real distributed factor -> m shard %.2e  q %.2e" % (rank, world, nd * nt,
                                                                                         e_m, e_q), flush=True)
        for x in (eng, one):
            x.close()
    flags = torch.tensor([1.0 if ok else 0.0], device="cuda")
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("PASS" if flags.item() == 1.0 else "FAIL", flush=True)
    dist.destroy_process_group()
    return 0 if flags.item() == 1.0 else 1


if __name__ == "__main__":
    sys.exit(main())
