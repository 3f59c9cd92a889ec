#!/usr/bin/env python
"""A cfg0-sized pass over every kernel family of libqal.so, for compute-sanitizer (memcheck / racecheck /
synccheck): dense forward + gradient (K1-K6), the ordered product / scan / batched products, the fidelity
(n = 64 and n = 4096), the coherence-block path in its three launch layouts (forward, suffix chain,
gradient, tree, scans, pack / unpack / check), NODES mode with the commutator basis, the block VJP, and the
n = 4096 block path on one slice.  usage: python tools/sanitize_run.py [--no-big] [--save out.npz]
(--save: every output, for the bit-for-bit comparison of tools/stress_check.py)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13330_b200 import _build, driver, inputs as qi, qal  # noqa: E402


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


OUT = {}


def keep(name, t):
    if t is not None:
        OUT[name] = (torch.view_as_real(t) if t.is_complex() else t).detach().cpu().numpy().copy()
    return t


def main():
    if not os.environ.get("QAL_LIB"):
        _build.build()
    big = "--no-big" not in sys.argv
    p = qi.cfg2(batch=5, N=12, T=200.0 * 12 / 1024)
    L0, Lc, _ = qal.qal_build_liouvillian(d(p.H0), d(p.Hc), d(p.C))
    u, V = d(p.u), d(p.V)
    # dense: fidelity + gradient, forward chunks + tree, scan, batched products
    F, g, Lam = qal.qal_fidelity_grad(L0, Lc, u, p.T, p.N, V, want_Lambda=True)
    keep('dense_F', F); keep('dense_g', g); keep('dense_Lam', Lam)
    _, parts = qal.qal_magnus_expm_slices(L0, Lc, u, p.T, p.N, chunk=4)
    keep('dense_parts', parts); keep('dense_prod', qal.qal_ordered_product(parts))
    pre, suf = qal.qal_ordered_scan(parts)
    keep('dense_pre', pre); keep('dense_suf', suf); keep('dense_bmm', qal.qal_batched_matmul(pre[0], suf[0]))
    keep('dense_fid', qal.qal_fidelity(Lam, V))
    # NODES mode with the commutator basis (configs[3] recipe, a short horizon)
    p3 = qi.cfg3(N=64, T=10.0)
    L03, Lc3, Lcomm3 = qal.qal_build_liouvillian(d(p3.H0), d(p3.Hc), d(p3.C), want_comm=True)
    u3 = qal.qal_sample_controls_sines(d(p3.sines), p3.u_max, p3.N, p3.T).unsqueeze(0).contiguous()
    r3 = qal.qal_fidelity_grad(L03, Lc3, u3, p3.T, p3.N, d(p3.V), ctrl_mode=1, Lcomm=Lcomm3)
    keep('nodes_F', r3[0]); keep('nodes_g', r3[1])
    # coherence blocks, every launch layout
    plan = qal.qal_block_plan_build(torch.cat([L0[:1], Lc]), mirror=True)
    L0p, f0 = qal.qal_block_pack(plan, L0)
    Lcp, f1 = qal.qal_block_pack(plan, Lc)
    st = torch.zeros(p.u.shape[0], dtype=torch.int32, device="cuda")
    qal.qal_block_check(plan, L0, st)
    qal.qal_block_check(plan, Lc, st, broadcast=True)
    for sets in (qal.QAL_BLK_SETS_DEFAULT, qal.QAL_BLK_SETS_FUSED, qal.QAL_BLK_SETS_PAIRS):
        plan.launch_sets = sets
        Fb, gb, Lp = qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, p.T, p.N, V, want_Lambda=True)
        keep(f'blk{sets}_F', Fb); keep(f'blk{sets}_g', gb); keep(f'blk{sets}_Lam', Lp)
    plan.launch_sets = qal.QAL_BLK_SETS_DEFAULT
    keep('blk_unpack', qal.qal_block_unpack(plan, Lp))
    # the fused forward layout of the gradient path (>= 8 x SMs pulses) and s > 0 squarings (long slices)
    pb = qi.cfg2(batch=1200, N=4, T=200.0 * 4 / 1024)
    L0b = qal.qal_build_liouvillian(d(pb.H0), d(pb.Hc), d(pb.C))[0]
    L0bp, _ = qal.qal_block_pack(plan, L0b)
    Fz, gz, _ = qal.qal_block_fidelity_grad(plan, L0bp, Lcp, d(pb.u), pb.T, pb.N, V)
    keep('blk_fused_F', Fz); keep('blk_fused_g', gz)
    Fs, gs, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, 40.0 * p.T, p.N, V)
    keep('blk_long_F', Fs); keep('blk_long_g', gs)
    bparts = qal.qal_block_expm_slices(plan, L0p, Lcp, u, p.T, p.N, chunk=4)
    keep('blk_parts', bparts); keep('blk_prod', qal.qal_block_ordered_product(plan, bparts))
    bpre, bsuf = qal.qal_block_ordered_scan(plan, bparts)
    keep('blk_pre', bpre); keep('blk_suf', bsuf); keep('blk_bmm', qal.qal_block_batched_matmul(plan, bpre[0], bsuf[0]))
    cot = qal.qal_block_fidelity_cotangent(plan, V)
    keep('blk_vjp', qal.qal_block_propagator_vjp(plan, L0p, Lcp, u, p.T, p.N,
                                                   cot.unsqueeze(0).expand(u.shape[0], -1).contiguous())[0])
    keep('blk_fid', qal.qal_block_fidelity(plan, Lp, V))
    # blocks in NODES mode (commutators packed)
    plan3 = qal.qal_block_plan_build(torch.cat([L03, Lc3, Lcomm3.reshape(-1, 64, 64)]), mirror=True)
    m3 = [qal.qal_block_pack(plan3, m, check=True)[0] for m in (L03, Lc3, Lcomm3)]
    r3b = qal.qal_block_fidelity_grad(plan3, m3[0], m3[1], u3, p3.T, p3.N, d(p3.V), ctrl_mode=1, Lcommp=m3[2])
    keep('blk_nodes_F', r3b[0]); keep('blk_nodes_g', r3b[1])
    torch.cuda.synchronize()
    if big:
        p4 = qi.cfg4(batch=1, N=2, T=100.0 * 2 / 512)
        L04, Lc4, _ = qal.qal_build_liouvillian(d(p4.H0), d(p4.Hc), d(p4.C))
        plan4 = qal.qal_bigblock_plan_build(torch.cat([L04, Lc4]), mirror=True)
        P4, _ = qal.qal_bigblock_expm_slices(plan4, L04, Lc4, d(p4.u[0, :1]), p4.T, p4.N, count=1)
        ws = torch.empty(qal.workspace_bytes(qal.QAL_OP_FIDELITY_REDUCE, 4096, 1, 1), dtype=torch.uint8,
                         device="cuda")
        keep('big_P_rows', P4[:, :96].contiguous()); keep('big_P_sum', torch.view_as_real(P4).sum(dim=(1, 2))); keep('big_fid_ws', qal.qal_fidelity(P4, d(p4.V), ws=ws))
        keep('big_fid', qal.qal_fidelity(P4, d(p4.V)))
        torch.cuda.synchronize()
    if "--save" in sys.argv:
        np.savez(sys.argv[sys.argv.index("--save") + 1], **OUT)
    print("sanitize_run ok", float(F[0]), float(Fb[0]), len(OUT), "outputs")


if __name__ == "__main__":
    main()
