"""Forward-only block path timing at small item counts (one chunk per pulse) vs the bench sizes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_13330_b200 import qal, inputs as qi

for B, N in ((296, 256), (888, 1024)):
    p = qi.cfg2(batch=B, N=N, T=200.0 * N / 1024)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    L0, Lc, _ = qal.qal_build_liouvillian(d(p.H0), d(p.Hc), d(p.C))
    plan = qal.qal_block_plan_build(torch.cat([L0[:1], Lc]), mirror=True)
    L0p, _ = qal.qal_block_pack(plan, L0)
    Lcp, _ = qal.qal_block_pack(plan, Lc)
    u, V = d(p.u), d(p.V)
    f = lambda: qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, p.T, N, V, want_grad=False)  # noqa: E731
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"B={B} N={N}: forward+fidelity {ms:.2f} ms, {B * N / ms / 1e3:.2f} M slices/s")
