"""GEMV-H work-unit sweep for G* of config 2 (dev tool): adjoint apply in
stage-timing mode (events around each stage) per unit_cols, three trials.
Note: stage-timing mode isolates the kernel; the pipelined online path can
rank the shapes differently (round 1: equal 10-unit splits won here by
~15 us but lost ~7 us inside infer_map + forecast, so the default stayed)."""
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2504_16344_b200 as ltb
res = {}
for trial in range(3):
    for uc in [0, 1024, 1365, 2048, 2731, 4096]:
        p = ltb.MatvecPlan.generated(64, 16384, 128, seed=3, unit_cols=uc)
        s = ltb.MatvecPlan.Scratch(p, stream=torch.cuda.current_stream())
        dd = torch.rand(64 * 128, dtype=torch.float64, device="cuda")
        mm = torch.empty(16384 * 128, dtype=torch.float64, device="cuda")
        s.timing(True)
        for _ in range(3):
            p.apply_adjoint_raw(dd, mm, s)
        s.timing(True)
        for _ in range(20):
            p.apply_adjoint_raw(dd, mm, s)
        st = s.stage_ms()
        res.setdefault(uc, []).append(st["Fstar"][1] / 20 * 1e3)
        s.close(); p.close()
for uc, v in res.items():
    print("unit_cols=%5d gemv_h %s" % (uc, " ".join("%.1f" % x for x in v)))
