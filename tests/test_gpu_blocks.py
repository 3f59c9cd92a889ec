"""GPU parity of the coherence-block path (pin P-13) against the CPU oracle.

The block path computes the same Omega_k, U_k, Lambda, F (and dF/du) as the dense path, restricted to
the coherence-order blocks found by qal_block_plan_build; every expected value here comes from
oracle/ (dense, sequential, no structure), so these tests pin the block path to the definition.
Tolerances as tests/test_gpu_parity.py (BASELINE north_star).
"""
import numpy as np
import pytest

from paper_2511_13330_b200 import inputs as qi

pytestmark = pytest.mark.gpu

TOL_PROP = 1e-10
TOL_GRAD = 1e-8


def relfro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return torch


@pytest.fixture(scope="module")
def qal(torch_cuda):
    from paper_2511_13330_b200 import _build, qal as q
    _build.build()
    q.load()
    return q


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def packed_basis(torch, qal, prob, mirror=True, want_comm=False):
    """Dense basis on the GPU (K1), plan from it, packed copies (with the device structure check)."""
    C = prob.C if prob.C.shape[0] > 0 else None
    L0, Lc, Lcomm = qal.qal_build_liouvillian(dev(torch, prob.H0), dev(torch, prob.Hc),
                                              None if C is None else dev(torch, C), want_comm=want_comm)
    mats = [L0, Lc] + ([Lcomm.reshape(-1, 64, 64)] if want_comm else [])
    plan = qal.qal_block_plan_build(torch.cat([m.reshape(-1, 64, 64) for m in mats]), mirror=mirror)
    L0p, f0 = qal.qal_block_pack(plan, L0)
    Lcp, f1 = qal.qal_block_pack(plan, Lc)
    Lcommp = None
    if want_comm:
        Lcommp, f2 = qal.qal_block_pack(plan, Lcomm)
        assert f2.item() == 0
    assert f0.item() == 0 and f1.item() == 0
    return plan, L0p, Lcp, Lcommp


@pytest.mark.parametrize("mirror", [True, False])
def test_pack_unpack_roundtrip_of_oracle_lambda(torch_cuda, qal, oracle, mirror):
    torch = torch_cuda
    p = qi.cfg0(N=16, T=100.0 * 16 / 256)
    plan, _, _, _ = packed_basis(torch, qal, p, mirror)
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(L0, Lc, p.u[0], p.T, p.N)
    pk, flag = qal.qal_block_pack(plan, dev(torch, Lam[None]))
    assert flag.item() == 0                        # the oracle's Lambda is block diagonal (P-13)
    back = qal.qal_block_unpack(plan, pk)[0].cpu().numpy()
    assert relfro(back, Lam) <= 1e-14              # mirror fill = Hermiticity preservation (P-5)


def test_structure_check_flags_off_block_entry(torch_cuda, qal):
    torch = torch_cuda
    p = qi.cfg0(N=4, T=1.0)
    plan, _, _, _ = packed_basis(torch, qal, p)
    M = torch.zeros((2, 64, 64), dtype=torch.complex128, device="cuda")
    M[1, 0, 1] = 1e-300                            # couples natural indices 0 and 1 (q = 0 and q = 1)
    _, flag = qal.qal_block_pack(plan, M)
    assert flag.item() == qal.QAL_ERR_STRUCTURE


@pytest.mark.parametrize("mirror", [True, False])
def test_cfg0_forward_block_path(torch_cuda, qal, oracle, mirror):
    torch = torch_cuda
    p = qi.cfg0()
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p, mirror)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(rL0, rLc, p.u[0], p.T, p.N)
    F, _, Lp = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V),
                                           want_grad=False, want_Lambda=True)
    got = qal.qal_block_unpack(plan, Lp)[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP, relfro(got, Lam)
    Fr = oracle.fidelity(Lam, p.V)
    assert abs(F.item() - Fr) / abs(Fr) <= TOL_PROP
    Fb = qal.qal_block_fidelity(plan, Lp, dev(torch, p.V)).item()
    assert abs(Fb - Fr) / abs(Fr) <= TOL_PROP


@pytest.mark.parametrize("chunk", [1, 4, 64, 256])
def test_chunk_fold_and_block_tree(torch_cuda, qal, oracle, chunk):
    torch = torch_cuda
    p = qi.cfg0()
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(rL0, rLc, p.u[0], p.T, p.N)
    parts = qal.qal_block_expm_slices(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, chunk=chunk)
    got = qal.qal_block_unpack(plan, qal.qal_block_ordered_product(plan, parts))[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP


@pytest.mark.parametrize("count", [1, 2, 3, 5, 13])
def test_block_ordered_product_ragged(torch_cuda, qal, oracle, count):
    """Tree over `count` packed slice exponentials vs the oracle's sequential left fold (A4)."""
    torch = torch_cuda
    p = qi.cfg0(N=count, T=100.0 * count / 256)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(rL0, rLc, p.u[0], p.T, p.N)
    Us = qal.qal_block_expm_slices(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, chunk=1)
    got = qal.qal_block_unpack(plan, qal.qal_block_ordered_product(plan, Us))[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP


def test_cfg2_recipe_per_pulse_drift(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.cfg2(batch=3, N=32, T=200.0 * 32 / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    F, _, Lp = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V),
                                           want_grad=False, want_Lambda=True)
    got = qal.qal_block_unpack(plan, Lp).cpu().numpy()
    for b in range(3):
        rL0, rLc = oracle.build_liouvillian(p.H0[b], p.Hc, p.C)
        Lam = oracle.propagate(rL0, rLc, p.u[b], p.T, p.N)
        assert relfro(got[b], Lam) <= TOL_PROP
        Fr = oracle.fidelity(Lam, p.V)
        assert abs(F[b].item() - Fr) / abs(Fr) <= TOL_PROP


@pytest.mark.parametrize("order", [2, 4])
def test_nodes_mode_block_forward(torch_cuda, qal, oracle, order):
    """cfg3 recipe: Magnus-4 commutator basis, packed (the commutators are block diagonal too)."""
    torch = torch_cuda
    p = qi.cfg3()
    N, T = 256, 200.0
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)[None]
    plan, L0p, Lcp, Lcommp = packed_basis(torch, qal, p, want_comm=True)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(rL0, rLc, u[0], T, N, mode=1, order=order)
    parts = qal.qal_block_expm_slices(plan, L0p, Lcp, dev(torch, u), T, N, chunk=16, magnus_order=order,
                                      ctrl_mode=1, Lcommp=Lcommp)
    got = qal.qal_block_unpack(plan, qal.qal_block_ordered_product(plan, parts))[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP


def test_block_slice_range_k0(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.cfg3()
    N, T = 256, 200.0
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)[None]
    plan, L0p, Lcp, Lcommp = packed_basis(torch, qal, p, want_comm=True)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    k0, cnt = 96, 64
    Lam = oracle.propagate(rL0, rLc, u[0], T, N, mode=1, k0=k0, k1=k0 + cnt)
    parts = qal.qal_block_expm_slices(plan, L0p, Lcp, dev(torch, u[:, k0:k0 + cnt]), T, N, k0=k0, count=cnt,
                                      chunk=cnt, ctrl_mode=1, Lcommp=Lcommp)
    got = qal.qal_block_unpack(plan, parts[:, 0])[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP


@pytest.mark.parametrize("T,N", [(100.0, 4), (1000.0, 2), (3.0, 8), (100.0, 64)])
def test_block_norm_regimes(torch_cuda, qal, oracle, T, N):
    """Per-block (m, s) choices: squarings (s > 0) and the T8 scheme."""
    torch = torch_cuda
    p = qi.cfg0(N=N, T=T)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(rL0, rLc, p.u[0], T, N)
    F, _, Lp = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), T, N, dev(torch, p.V),
                                           want_grad=False, want_Lambda=True)
    got = qal.qal_block_unpack(plan, Lp)[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP


# ------------------------------------------------------------------ gradient (a7) on the blocks
@pytest.mark.parametrize("mirror", [True, False])
def test_cfg1_block_gradient(torch_cuda, qal, oracle, mirror):
    torch = torch_cuda
    p = qi.cfg1()
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p, mirror)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, Lam = oracle.gradient(rL0, rLc, p.u[0], p.T, p.N, p.V)
    F, g, Lp = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V),
                                           want_Lambda=True)
    assert relfro(qal.qal_block_unpack(plan, Lp)[0].cpu().numpy(), Lam) <= TOL_PROP
    assert abs(F.item() - Fr) / abs(Fr) <= TOL_PROP
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD, relfro(g[0].cpu().numpy(), gr)


def test_cfg2_recipe_block_gradient(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.cfg2(batch=3, N=32, T=200.0 * 32 / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    F, g, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V))
    for b in range(3):
        rL0, rLc = oracle.build_liouvillian(p.H0[b], p.Hc, p.C)
        Fr, gr, _ = oracle.gradient(rL0, rLc, p.u[b], p.T, p.N, p.V)
        assert abs(F[b].item() - Fr) / abs(Fr) <= TOL_PROP
        assert relfro(g[b].cpu().numpy(), gr) <= TOL_GRAD


def test_nodes_mode_block_gradient(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.cfg3()
    N, T = 64, 300.0
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)[None]
    plan, L0p, Lcp, Lcommp = packed_basis(torch, qal, p, want_comm=True)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, _ = oracle.gradient(rL0, rLc, u[0], T, N, p.V, mode=1)
    F, g, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, u), T, N, dev(torch, p.V), ctrl_mode=1,
                                          Lcommp=Lcommp)
    assert abs(F.item() - Fr) / abs(Fr) <= TOL_PROP
    assert g.shape == (1, N, 2, 2)
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD


@pytest.mark.parametrize("T,N", [(100.0, 4), (1000.0, 2), (3.0, 8), (100.0, 64)])
def test_block_gradient_norm_regimes(torch_cuda, qal, oracle, T, N):
    torch = torch_cuda
    p = qi.cfg0(N=N, T=T)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, _ = oracle.gradient(rL0, rLc, p.u[0], T, N, p.V)
    F, g, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), T, N, dev(torch, p.V))
    assert abs(F.item() - Fr) <= TOL_PROP * max(abs(Fr), 1e-3)
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD


def test_block_gradient_matches_dense_path_bitwise_shape(torch_cuda, qal):
    """Same layout and values (within rounding) as the dense qal_fidelity_grad on a larger batch."""
    torch = torch_cuda
    p = qi.cfg2(batch=64, N=128, T=200.0 * 128 / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    L0, Lc, _ = qal.qal_build_liouvillian(dev(torch, p.H0), dev(torch, p.Hc), dev(torch, p.C))
    Fd, gd, _ = qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), p.T, p.N, dev(torch, p.V))
    Fb, gb, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V))
    assert gb.shape == gd.shape
    assert ((Fb - Fd).abs() / Fd.abs()).max().item() <= 1e-12
    err = ((gb - gd).reshape(64, -1).norm(dim=1) / gd.reshape(64, -1).norm(dim=1)).max().item()
    assert err <= 1e-11, err


def test_pulse_batch_block_structure_matches_oracle(torch_cuda, qal, oracle):
    """The bench engine (driver.PulseBatch, structure='blocks', sub-batched) vs the oracle on sampled
    pulses of a configs[2]-recipe batch, and vs the dense engine on every pulse."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg2(batch=40, N=64, T=200.0 * 64 / 1024)
    args = [dev(torch, a) for a in (p.H0, p.Hc, p.C, p.u, p.V)]
    eb = driver.PulseBatch(*args, p.T, sub_batch=16, structure="blocks")
    Fb, gb = eb.step()
    assert eb.structure_ok()
    ed = driver.PulseBatch(*args, p.T, sub_batch=16, structure="dense")
    Fd, gd = ed.step()
    assert ((Fb - Fd).abs() / Fd.abs()).max().item() <= 1e-12
    assert ((gb - gd).reshape(40, -1).norm(dim=1) / gd.reshape(40, -1).norm(dim=1)).max().item() <= 1e-11
    for b in (0, 17, 39):
        rL0, rLc = oracle.build_liouvillian(p.H0[b], p.Hc, p.C)
        Fr, gr, _ = oracle.gradient(rL0, rLc, p.u[b], p.T, p.N, p.V)
        assert abs(Fb[b].item() - Fr) / abs(Fr) <= TOL_PROP
        assert relfro(gb[b].cpu().numpy(), gr) <= TOL_GRAD


def test_time_shard_propagator_blocks_matches_oracle(torch_cuda, qal, oracle):
    """configs[3] recipe through driver.time_shard_propagator with a block plan (G = 1 on one GPU):
    packed chunk fold + tree + ordered combine vs the oracle's sequential fold."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg3()
    N, T = 512, 400.0
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)[None]
    plan, L0p, Lcp, Lcommp = packed_basis(torch, qal, p, want_comm=True)
    Lam_p = driver.time_shard_propagator(L0p, Lcp, Lcommp, dev(torch, u), T, N, 0, ctrl_mode=1, plan=plan)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(rL0, rLc, u[0], T, N, mode=1)
    got = qal.qal_block_unpack(plan, Lam_p.unsqueeze(0))[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP
    F = qal.qal_block_fidelity(plan, Lam_p.unsqueeze(0), dev(torch, p.V)).item()
    Fr = oracle.fidelity(Lam, p.V)
    assert abs(F - Fr) / abs(Fr) <= TOL_PROP


# ------------------------------------------------------------------ general cotangent (f1/f2 on the blocks)
def test_block_vjp_with_fidelity_cotangent_equals_fidelity_gradient(torch_cuda, qal):
    torch = torch_cuda
    p = qi.cfg2(batch=5, N=48, T=200.0 * 48 / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    V = dev(torch, p.V)
    _, gF, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, V)
    C = qal.qal_block_fidelity_cotangent(plan, V).unsqueeze(0).repeat(5, 1).contiguous()
    gC, _ = qal.qal_block_propagator_vjp(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, C)
    err = ((gC - gF).reshape(5, -1).norm(dim=1) / gF.reshape(5, -1).norm(dim=1)).max().item()
    assert err <= 1e-13, err


def test_block_vjp_general_cotangent_matches_oracle(torch_cuda, qal, oracle):
    """A Hermiticity-preserving cotangent (C = Lambda_target^dag, the superoperator of a CPTP map)
    packed with qal_block_pack vs the oracle's per-direction vjp (O7 with a general seed)."""
    torch = torch_cuda
    p = qi.cfg0(N=32, T=100.0 * 32 / 256)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    q = qi.cfg0(N=8, T=37.0)
    Lt = oracle.propagate(rL0, rLc, q.u[0], q.T, q.N)            # a CPTP superoperator: HP
    Cn = Lt.conj().T.copy()
    gr, _ = oracle.vjp(rL0, rLc, p.u[0], p.T, p.N, Cn)
    Cp, flag = qal.qal_block_pack(plan, dev(torch, Cn[None]))
    assert flag.item() == 0
    g, _ = qal.qal_block_propagator_vjp(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, Cp)
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD


def test_fused_and_split_forward_layouts_are_bit_identical(torch_cuda, qal):
    """The gradient path's forward runs fused (one slot per pulse: expm + prefix fold per slice) for large
    batches and split (persistent expm over all slices, then the prefix chain beside the suffix chain)
    for batches below 8 x SMs: the same arithmetic, so 1200 pulses in one call (fused) equal the same
    pulses in two calls of 600 (split) bit for bit."""
    torch = torch_cuda
    B = 1200
    assert B >= 8 * torch.cuda.get_device_properties(0).multi_processor_count
    p = qi.cfg2(batch=B, N=6, T=200.0 * 6 / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    u, V = dev(torch, p.u), dev(torch, p.V)
    F1, g1, L1 = qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, p.T, p.N, V, want_Lambda=True)
    parts = [qal.qal_block_fidelity_grad(plan, L0p[i:i + 600].contiguous(), Lcp, u[i:i + 600].contiguous(), p.T, p.N,
                                         V, want_Lambda=True) for i in (0, 600)]
    F2, g2, L2 = (torch.cat([a[k] for a in parts]) for k in range(3))
    assert torch.equal(L1, L2) and torch.equal(F1, F2) and torch.equal(g1, g2)


def test_block_forward_backward_session_equals_one_call_vjp_and_oracle(torch_cuda, qal, oracle):
    """qal_block_propagator_forward + _backward (the stored forward of the time-sharded gradient) give
    bit for bit the Lambda and gradient of the one-call qal_block_propagator_vjp, and the oracle's
    per-direction vjp; the cotangent is built from the forward's Lambda in between (NODES mode with the
    commutator basis, so the stored (m, s) codes and the commutator traces are exercised)."""
    torch = torch_cuda
    p = qi.cfg3(N=96, T=40.0)
    plan, L0p, Lcp, Lcommp = packed_basis(torch, qal, p, want_comm=True)
    un = oracle.sines_nodes(p.sines, p.u_max, p.N, p.T).reshape(3, 32, 2, 2)   # host controls, both sides
    u = dev(torch, un)
    sess = qal.BlockGradientSession(plan, L0p, Lcp, u, p.T, p.N, ctrl_mode=1, Lcommp=Lcommp)
    Lam = sess.forward()
    C = qal.qal_block_fidelity_cotangent(plan, dev(torch, p.V)).unsqueeze(0).repeat(3, 1).contiguous()
    C = qal.qal_block_batched_matmul(plan, C, Lam)      # a cotangent that depends on the forward's Lambda
    g = sess.vjp(C)
    g1, L1 = qal.qal_block_propagator_vjp(plan, L0p, Lcp, u, p.T, p.N, C, ctrl_mode=1, Lcommp=Lcommp,
                                          want_Lambda=True)
    assert torch.equal(Lam, L1) and torch.equal(g, g1)
    # the oracle's reference: its own Lambda and cotangent (no GPU value enters the oracle)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Cf = oracle.fidelity_cotangent(p.V)
    for b in range(3):
        Lr = oracle.propagate(rL0, rLc, un[b], p.T * 32 / p.N, 32, mode=1)
        gr, _ = oracle.vjp(rL0, rLc, un[b], p.T * 32 / p.N, 32, oracle.matmul(Cf, Lr), mode=1)
        assert relfro(g[b].cpu().numpy(), gr) <= TOL_GRAD


def test_block_scan_and_batched_matmul(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.cfg0(N=11, T=100.0 * 11 / 256)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    Us = qal.qal_block_expm_slices(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, chunk=1)        # [1][11][packed]
    pre, suf = qal.qal_block_ordered_scan(plan, Us)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    _, Un = oracle.propagate(rL0, rLc, p.u[0], p.T, p.N, store=True)
    for s in (0, 4, 10):
        ref_pre = oracle.ordered_product(Un[:s]) if s > 0 else np.eye(64)
        ref_suf = oracle.ordered_product(Un[s + 1:]) if s + 1 < 11 else np.eye(64)
        assert relfro(qal.qal_block_unpack(plan, pre[0, s:s + 1])[0].cpu().numpy(), ref_pre) <= 1e-12
        assert relfro(qal.qal_block_unpack(plan, suf[0, s:s + 1])[0].cpu().numpy(), ref_suf) <= 1e-12
    AB = qal.qal_block_batched_matmul(plan, Us[0, 3:4], Us[0, 2:3])
    assert relfro(qal.qal_block_unpack(plan, AB)[0].cpu().numpy(), Un[3] @ Un[2]) <= 1e-13


def test_time_sharded_gradient_blocks_matches_oracle(torch_cuda, qal, oracle):
    """NEXT f2 on the block path (G = 1): segmented, scanned, one batched block VJP."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg3()
    N, T = 256, 150.0
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)[None]
    plan, L0p, Lcp, Lcommp = packed_basis(torch, qal, p, want_comm=True)
    V = dev(torch, p.V)
    Lam, g = driver.time_sharded_gradient(L0p, Lcp, Lcommp, dev(torch, u), T, N, 0, ctrl_mode=1, sub=32, plan=plan,
                                          cotangent=lambda Lm: qal.qal_block_fidelity_cotangent(plan, V))
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, Lr = oracle.gradient(rL0, rLc, u[0], T, N, p.V, mode=1)
    assert relfro(qal.qal_block_unpack(plan, Lam.unsqueeze(0))[0].cpu().numpy(), Lr) <= TOL_PROP
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD


# ------------------------------------------------------------------ status flags, determinism, structure check
def test_block_status_flags_nonfinite_input(torch_cuda, qal):
    torch = torch_cuda
    p = qi.cfg0(N=8)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    u = np.concatenate([p.u, p.u], axis=0)
    u[1, 3, 0] = np.nan
    V = dev(torch, p.V)
    for want_grad in (False, True):
        status = torch.full((2,), 7, dtype=torch.int32, device="cuda")
        qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, u), p.T, p.N, V, want_grad=want_grad, status=status)
        assert status.cpu().tolist() == [0, qal.QAL_ERR_NONFINITE]


def test_block_path_bit_identical_runs(torch_cuda, qal):
    torch = torch_cuda
    p = qi.cfg2(batch=7, N=64, T=200.0 * 64 / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    outs = [qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V), want_Lambda=True)
            for _ in range(2)]
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_pulse_batch_reports_a_broken_structure(torch_cuda, qal):
    """A transverse drift term (sigma_x on spin 1) breaks total S_z: the per-step device check of the
    bench engine reports it as QAL_ERR_STRUCTURE (-8) in status[b] of exactly that pulse (the plan was
    detected from the symmetric basis of pulse 0), and a clean step clears it again."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg2(batch=3, N=8, T=2.0)
    args = [dev(torch, a) for a in (p.H0, p.Hc, p.C, p.u, p.V)]
    eng = driver.PulseBatch(*args, p.T, structure="blocks")
    eng.step()
    assert eng.structure_ok() and eng.status.cpu().tolist() == [0, 0, 0]
    H0_clean = eng.H0.clone()
    sx = np.kron(np.array([[0, 1], [1, 0]], dtype=complex), np.eye(4))
    eng.H0[2] += dev(torch, 0.01 * sx)
    eng.H0 = eng.H0.contiguous()
    eng.step()
    assert not eng.structure_ok()
    assert eng.status.cpu().tolist() == [0, 0, qal.QAL_ERR_STRUCTURE]
    eng.H0 = H0_clean
    eng.step()
    assert eng.structure_ok() and eng.status.cpu().tolist() == [0, 0, 0]


def test_block_check_broadcasts_a_broken_shared_basis(torch_cuda, qal):
    """A shared control operator that breaks the structure flags every pulse (broadcast mode)."""
    torch = torch_cuda
    p = qi.cfg2(batch=4, N=4, T=1.0)
    plan, _, _, _ = packed_basis(torch, qal, p, True)
    Hc = p.Hc.copy()
    Hc[1] = Hc[1] + 0.3 * np.kron(np.array([[0, 1], [1, 0]], dtype=complex), np.eye(4))
    _, Lc, _ = qal.qal_build_liouvillian(dev(torch, p.H0[:1]), dev(torch, Hc), dev(torch, p.C))
    status = torch.zeros(4, dtype=torch.int32, device="cuda")
    qal.qal_block_check(plan, Lc[:1], status, broadcast=True)
    assert status.cpu().tolist() == [0, 0, 0, 0]               # L_1 alone still conserves S_z
    qal.qal_block_check(plan, Lc, status, broadcast=True)
    assert status.cpu().tolist() == [qal.QAL_ERR_STRUCTURE] * 4


@pytest.mark.parametrize("mirror", [True, False])
def test_launch_sets_fused_vs_group_specialised(torch_cuda, qal, mirror):
    """The forward / suffix-chain / gradient kernels run one launch per group (slots, role-compiled
    kernels) by default; the plan's launch_sets option selects one fused CTA per item (every group) or
    two items per CTA.  The forward and the suffix chain are identical (the same arithmetic per group),
    the gradient equal up to the order of the per-group trace sums.  An invalid option is refused
    before any launch."""
    torch = torch_cuda
    p = qi.cfg2(batch=40, N=96, T=200.0 * 96 / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p, mirror)
    u, V = dev(torch, p.u), dev(torch, p.V)

    def run(sets):
        plan.launch_sets = sets
        F, g, Lam = qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, p.T, p.N, V, want_Lambda=True)
        torch.cuda.synchronize()
        return F.cpu().numpy(), g.cpu().numpy(), Lam.cpu().numpy()

    Fd, gd, Ld = run(qal.QAL_BLK_SETS_DEFAULT)
    Ff, gf, Lf = run(qal.QAL_BLK_SETS_FUSED)
    F2, g2, L2 = run(qal.QAL_BLK_SETS_PAIRS)
    assert np.array_equal(Ld, Lf) and np.array_equal(Fd, Ff)
    assert np.array_equal(L2, Ld) and np.array_equal(g2, gd)
    rel = np.linalg.norm((gd - gf).reshape(len(gd), -1), axis=1) / np.linalg.norm(gf.reshape(len(gf), -1), axis=1)
    assert np.max(rel) <= 1e-13
    plan.launch_sets = 5
    with pytest.raises(RuntimeError):
        qal.qal_block_fidelity_grad(plan, L0p, Lcp, u, p.T, p.N, V)
    plan.launch_sets = qal.QAL_BLK_SETS_DEFAULT


@pytest.mark.parametrize("batch,N", [(1, 1), (3, 5), (5, 2), (7, 3)])
def test_block_gradient_degenerate_and_ragged_sizes(torch_cuda, qal, oracle, batch, N):
    """Item counts below and not divisible by the slots per CTA (group-specialised launches leave
    slots empty), a single slice, and pulse counts that are not multiples of anything, vs the oracle."""
    torch = torch_cuda
    p = qi.cfg2(batch=batch, N=N, T=200.0 * N / 1024)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, qi.cfg2(batch=1, N=2), True)
    L0 = qal.qal_build_liouvillian(dev(torch, p.H0), dev(torch, p.Hc), dev(torch, p.C))[0]
    L0p, f0 = qal.qal_block_pack(plan, L0)
    assert f0.item() == 0
    F, g, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V))
    torch.cuda.synchronize()
    F, g = F.cpu().numpy(), g.cpu().numpy()
    for b in range(batch):
        rL0, rLc = oracle.build_liouvillian(p.H0[b], p.Hc, p.C)
        Fr, gr, _ = oracle.gradient(rL0, rLc, p.u[b], p.T, p.N, p.V)
        assert abs(F[b] - Fr) / abs(Fr) <= TOL_PROP
        assert relfro(g[b], gr) <= TOL_GRAD


def _with_controls(p, J):
    """The cfg0 problem with J control Hamiltonians: the first one only, or the two exchange terms plus a
    third S_z-conserving one (the 1-3 exchange), with seeded piecewise-constant amplitudes."""
    import dataclasses
    sx = np.array([[0, 1], [1, 0]], dtype=complex)
    sy = np.array([[0, -1j], [1j, 0]], dtype=complex)
    sz = np.array([[1, 0], [0, -1]], dtype=complex)
    i2 = np.eye(2, dtype=complex)
    if J == 1:
        Hc = p.Hc[:1].copy()
    else:
        H13 = sum(np.kron(np.kron(s, i2), s) for s in (sx, sy, sz)) / 4.0
        Hc = np.concatenate([p.Hc, H13[None]], axis=0)
    rng = np.random.default_rng(1234 + J)
    u = rng.uniform(0.0, 2 * np.pi * 0.05, size=(1, p.N, J))
    return dataclasses.replace(p, Hc=Hc, u=u)


@pytest.mark.parametrize("J", [1, 3])
def test_block_gradient_other_control_counts(torch_cuda, qal, oracle, J):
    """The gradient role kernels are compiled in variants (Omega basis cache + stored (m, s) codes, PWC
    trace-basis cache, J = 2 unrolled); J = 1 takes the variant without the unrolled loops and J = 3 the one
    without the trace-basis cache.  Same parity bar as J = 2."""
    torch = torch_cuda
    p = _with_controls(qi.cfg0(N=24, T=100.0 * 24 / 256), J)
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, Lam = oracle.gradient(rL0, rLc, p.u[0], p.T, p.N, p.V)
    F, g, Lp = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, p.u), p.T, p.N, dev(torch, p.V),
                                           want_Lambda=True)
    assert g.shape == (1, p.N, J)
    assert relfro(qal.qal_block_unpack(plan, Lp)[0].cpu().numpy(), Lam) <= TOL_PROP
    assert abs(F.item() - Fr) <= TOL_PROP * max(abs(Fr), 1e-3)
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD, relfro(g[0].cpu().numpy(), gr)


def test_nodes_mode_order2_block_gradient(torch_cuda, qal, oracle):
    """Node-sampled controls at Magnus order 2 (no commutator terms): the cached-basis variants with two
    control values per slice."""
    torch = torch_cuda
    p = qi.cfg3()
    N, T = 48, 200.0
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)[None]
    plan, L0p, Lcp, _ = packed_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, _ = oracle.gradient(rL0, rLc, u[0], T, N, p.V, mode=1, order=2)
    F, g, _ = qal.qal_block_fidelity_grad(plan, L0p, Lcp, dev(torch, u), T, N, dev(torch, p.V), ctrl_mode=1,
                                          magnus_order=2)
    assert abs(F.item() - Fr) / abs(Fr) <= TOL_PROP
    assert g.shape == (1, N, 2, 2)
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD
