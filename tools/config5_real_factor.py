"""BASELINE config 5 on a REAL factor (dev tool; torchrun, one rank per GPU,
>= 4 GPUs for the 254 GB packed factor next to the F / G kernels):

  offline: form_K of the generated F and its prior-premultiplied G
           (Nd=600, Nt=420, Nm=16384, sigma2=1) straight into the row-cyclic
           factor layout, distributed tile Cholesky, K^{-1} preparation;
  online:  infer_map + forecast latency through the distributed K^{-1} and
           the column-sharded G* / F_q (max over ranks, CUDA events);
  checks:  backward error of the solve at full size, ||K y - b|| / (||K|| ||y||)
           with K applied through the sharded F and G* plans (F G* + s2 I),
           and m_map == G* (K^{-1} d).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/config5_real_factor.py [nm [nd nt]]
Prints one JSON line (rank 0)."""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402
from paper_2504_16344_b200.dist import shard_range  # noqa: E402

PRIOR = (1.0, 2.0, 1.0)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nd, nt, nq, seed, s2 = 600, 420, 21, 20250810, 1.0
    nm = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    if len(sys.argv) > 3:  # smaller shapes for a quick check of the same pipeline
        nd, nt = int(sys.argv[2]), int(sys.argv[3])
    n = nd * nt
    c0, c1 = shard_range(nm, world, rank)
    t0 = time.time()
    g = ltb.MatvecPlan.generated_premultiplied(nd, c1 - c0, nt, seed, PRIOR, nm_total=nm, c0=c0)
    fq = ltb.MatvecPlan.generated(nq, c1 - c0, nt, seed=seed, tag=ltb.KernelTag.Fq, nm_total=nm, c0=c0)
    eng = ltb.InferenceEngine(g, fq, world=world, rank=rank)
    torch.cuda.synchronize()
    t_plans = time.time() - t0
    dist.barrier()
    t0 = time.time()
    eng.form_K_generated(seed, 1, PRIOR, s2, nm_total=nm)
    torch.cuda.synchronize()
    dist.barrier()
    t_formk = time.time() - t0
    t0 = time.time()
    eng.factorize()
    torch.cuda.synchronize()
    dist.barrier()
    t_fact = time.time() - t0
    fk_ms, fz_ms = eng.offline_ms()
    # online latency on the real factor (max over ranks of the device time)
    d = torch.from_numpy(np.random.default_rng(5).standard_normal(n)).cuda()
    m = torch.empty((c1 - c0) * nt, dtype=torch.float64, device="cuda")
    q = torch.empty(nq * nt, dtype=torch.float64, device="cuda")
    for _ in range(2):
        dist.barrier()
        eng.infer_raw(d, m, q)
    lat = []
    for _ in range(5):
        dist.barrier()
        torch.cuda.synchronize()
        sec = eng.infer_raw(d, m, q)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dist.all_reduce(q)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([sec * 1e3 + e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        lat.append(float(t.item()))
    lat.sort()
    # checks at full size through the (oracle-verified) sharded matvec path
    f = ltb.MatvecPlan.generated(nd, c1 - c0, nt, seed=seed, tag=ltb.KernelTag.F, nm_total=nm, c0=c0)
    sf, sg = ltb.MatvecPlan.Scratch(f), ltb.MatvecPlan.Scratch(g)

    def apply_k(x):  # F G* x + s2 x, G* column-sharded, F m all-reduced
        mm = torch.empty((c1 - c0) * nt, dtype=torch.float64, device="cuda")
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        g.apply_adjoint_raw(x, mm, sg)
        sg.sync()
        f.apply_raw(mm, out, sf)
        sf.sync()
        dist.all_reduce(out)
        return out + s2 * x

    b = torch.from_numpy(np.random.default_rng(7).standard_normal(n)).cuda()
    y = b.clone()
    eng.solve_k_inplace(y)
    torch.cuda.synchronize()
    r = apply_k(y) - b
    kb = apply_k(b)
    back = float(torch.linalg.norm(r) / torch.linalg.norm(b))
    # ||K|| lower bound from one product: ||K b|| / ||b||
    knorm = float(torch.linalg.norm(kb) / torch.linalg.norm(b))
    berr = float(torch.linalg.norm(r) / (knorm * torch.linalg.norm(y)))
    # m_map == G* (K^{-1} d)
    yd = d.clone()
    eng.solve_k_inplace(yd)
    mg = torch.empty_like(m)
    g.apply_adjoint_raw(yd, mg, sg)
    sg.sync()
    eng.infer_raw(d, m, q)
    torch.cuda.synchronize()
    e_m = float(torch.linalg.norm(m - mg) / torch.linalg.norm(mg))
    stats = torch.tensor([e_m, berr, back], dtype=torch.float64, device="cuda")
    dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    if rank == 0:
        fac_bytes = 8 * n * (n + 1) // 2
        print(json.dumps({
            "config": "5: Nd=%d, Nt=%d, Nq=21, n=%d, Nm=%d, %d GPUs, REAL factor (K = F G* + I formed and "
                      "factorized on the GPUs, Gamma_x-premultiplied generated F)" % (nd, nt, n, nm, world),
            "offline": {"plans_s": t_plans, "form_k_s": t_formk, "form_k_device_ms": fk_ms,
                        "form_k_tflops_aggregate": n * n * nm / (fk_ms * 1e-3) / 1e12,
                        "factorize_s": t_fact, "factorize_device_ms": fz_ms,
                        "factorize_tflops_aggregate": n ** 3 / 3 / (fz_ms * 1e-3) / 1e12,
                        "factor_bytes": fac_bytes},
            "online": {"latency_ms": lat[len(lat) // 2], "latency_min_ms": lat[0],
                       "achieved_gbs": (2 * fac_bytes + 16 * (nt + 1) * (nd + nq) * nm) / (lat[len(lat) // 2] * 1e-3)
                                       / 1e9},
            "checks": {"m_map_vs_gstar_of_solve": float(stats[0]),
                       "solve_backward_error": float(stats[1]), "solve_relative_residual": float(stats[2]),
                       "what": "||K y - b|| / (||K|| ||y||) with K = F G* + I applied through the sharded plans, "
                               "||K|| estimated by ||K b|| / ||b||; m_map vs G* applied to the solve"},
        }), flush=True)
    for x in (sf, sg):
        x.close()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
