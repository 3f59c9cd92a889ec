"""A few slices of the configs[4] (or Hubbard) block-tiled path, for ncu captures of k_bb_gemm."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_13330_b200 import qal, inputs as qi

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = qi.hubbard3() if "hubbard" in sys.argv else qi.cfg4()
to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
L0, Lc, _ = qal.qal_build_liouvillian(to(prob.H0), to(prob.Hc), to(prob.C))
u = to(prob.u[0:1, :S])
lib = qal.load()
plan = qal.qal_bigblock_plan_build(torch.cat([L0[:1], Lc]), mirror=True)
ws = torch.empty(lib.qal_bigblock_workspace_bytes(ctypes.byref(plan)), dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
P = torch.empty((1, 1, 4096, 4096), dtype=torch.complex128, device="cuda")
for _ in range(2):
    rc = lib.qal_bigblock_expm_slices(ctypes.byref(plan), prob.N, prob.T, S, prob.J, qal._ptr(u[0]), qal._ptr(L0),
                                      qal._ptr(Lc), S, qal._ptr(P), None, qal._ptr(flag), qal._ptr(ws), ws.numel(),
                                      qal._stream(None))
    qal._check(rc, "qal_bigblock_expm_slices")
torch.cuda.synchronize()
print("ok", plan.sizes(), flag.item())
