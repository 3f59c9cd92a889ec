"""Ad-hoc timing: dense vs coherence-block forward (fidelity only) on the configs[2] workload."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_13330_b200 import qal, inputs as qi

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
N = 1024
p = qi.cfg2(batch=B, N=N)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
L0, Lc, _ = qal.qal_build_liouvillian(d(p.H0), d(p.Hc), d(p.C))
u, V = d(p.u), d(p.V)
plan = qal.qal_block_plan_build(torch.cat([L0[:1], Lc]), mirror=True)
L0p, f0 = qal.qal_block_pack(plan, L0)
Lcp, f1 = qal.qal_block_pack(plan, Lc)
print("flags", f0.item(), f1.item(), "groups", plan.groups())
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): out = fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out
ms_d, (Fd, _, _) = timeit(lambda: qal.qal_fidelity_grad(L0, Lc, u, p.T, N, V, want_grad=False))
ms_b, (Fb, _, _) = timeit(lambda: qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, p.T, N, V, want_grad=False))
err = (Fb - Fd).abs().max().item() / Fd.abs().max().item()
print(f"dense fwd {ms_d:.1f} ms  {B*N/ms_d/1e3:.3f} M slices/s")
print(f"block fwd {ms_b:.1f} ms  {B*N/ms_b/1e3:.3f} M slices/s  speedup {ms_d/ms_b:.1f}x  maxrelF {err:.2e}")
Bg = min(B, 296)
ug = u[:Bg].contiguous()
ms_dg, (Fdg, gd, _) = timeit(lambda: qal.qal_fidelity_grad(L0[:Bg].contiguous(), Lc, ug, p.T, N, V), reps=1)
ms_bg, (Fbg, gb, _) = timeit(lambda: qal.qal_block_fidelity_grad(plan, L0p[:Bg].contiguous(), Lcp, ug, p.T, N, V), reps=1)
eg = ((gb - gd).reshape(Bg, -1).norm(dim=1) / gd.reshape(Bg, -1).norm(dim=1)).max().item()
print(f"dense fwd+grad {ms_dg:.1f} ms  {Bg*N/ms_dg/1e3:.3f} M slices/s")
print(f"block fwd+grad {ms_bg:.1f} ms  {Bg*N/ms_bg/1e3:.3f} M slices/s  speedup {ms_dg/ms_bg:.1f}x  max rel grad err {eg:.2e}")
qal.qal_profile_begin()
qal.qal_block_fidelity_grad(plan, L0p[:Bg].contiguous(), Lcp, ug, p.T, N, V)
torch.cuda.synchronize()
print({k: v for k, v in qal.qal_profile_end().items() if v[1]})
