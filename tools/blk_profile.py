"""One block-path fwd+grad call on a configs[2]-recipe batch, for ncu captures."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_13330_b200 import qal, inputs as qi

B = int(sys.argv[1]) if len(sys.argv) > 1 else 296
N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
p = qi.cfg2(batch=B, N=N, T=200.0 * N / 1024)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
L0, Lc, _ = qal.qal_build_liouvillian(d(p.H0), d(p.Hc), d(p.C))
plan = qal.qal_block_plan_build(torch.cat([L0[:1], Lc]), mirror=True)
L0p, _ = qal.qal_block_pack(plan, L0)
Lcp, _ = qal.qal_block_pack(plan, Lc)
u, V = d(p.u), d(p.V)
for _ in range(2):
    F, g, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, p.T, N, V)
torch.cuda.synchronize()
print("ok", F[:2].tolist())
