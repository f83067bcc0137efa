"""K^{-1} apply latency at config 2 (n = 8192) and a larger n (dev tool):
device time of solve_k_inplace on a CUDA tensor (CUDA events, median).
    python tools/solve_bench.py [nd:nt ...]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

shapes = [(64, 128), (600, 64)]
if len(sys.argv) > 1:  # nd:nt pairs
    shapes = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]]
for nd, nt in shapes:
    g = ltb.MatvecPlan.generated(nd, 64, nt, seed=1, tag=ltb.KernelTag.Gstar)
    eng = ltb.InferenceEngine(g)
    eng.set_factor_generated(4321)
    y = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    s = ltb.MatvecPlan.Scratch(g, stream=st)
    for _ in range(3):
        eng.solve_k_inplace(y, scratch=s)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.solve_k_inplace(y, scratch=s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    n = nd * nt
    print("n=%d nb=%d solve_k %.3f ms (min %.3f)  %.2f us/block-step  %.0f GB/s" %
          (n, (n + 63) // 64, ts[10], ts[0], ts[10] * 1e3 / (2 * ((n + 63) // 64)), 8 * n * n / ts[10] / 1e6))
    s.close()
    eng.close()
