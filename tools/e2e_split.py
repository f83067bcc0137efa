"""Host-pointer (e2e) vs device-pointer matvec time per direction at the
Cascadia shape (dev tool): where the e2e overhead of the bench step goes."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2504_16344_b200 as ltb  # noqa: E402

nd, nm, nt = 600, 32768, 420
plan = ltb.MatvecPlan.generated(nd, nm, nt, seed=20250810)
s = ltb.MatvecPlan.Scratch(plan, stream=torch.cuda.current_stream())
m = torch.rand(nm * nt, dtype=torch.float64, device="cuda")
d = torch.rand(nd * nt, dtype=torch.float64, device="cuda")
mo = torch.empty_like(m)
do = torch.empty_like(d)
mh, dh = m.cpu().pin_memory(), d.cpu().pin_memory()
moh, doh = torch.empty_like(mh).pin_memory(), torch.empty_like(dh).pin_memory()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[reps // 2] * 1e3


print("F  device %.3f ms  host %.3f ms" % (t(lambda: plan.apply_raw(m, do, s)), t(lambda: plan.apply_raw(mh.numpy(), doh.numpy(), s))))
print("F* device %.3f ms  host %.3f ms" % (t(lambda: plan.apply_adjoint_raw(d, mo, s)),
                                         t(lambda: plan.apply_adjoint_raw(dh.numpy(), moh.numpy(), s))))
