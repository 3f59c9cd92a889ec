"""GPU parity: libqal.so (through the C ABI) vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): relative Frobenius error
<= 1e-10 on propagators and fidelities, relative L2 <= 1e-8 on gradients.  Every
reference value comes from oracle/ (never from the CUDA path).
"""
import math

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


def dev(torch, a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def build_basis(torch, qal, prob, want_comm=False):
    C = prob.C if prob.C.shape[0] > 0 else None
    return qal.qal_build_liouvillian(dev(torch, prob.H0), dev(torch, prob.Hc),
                                     None if C is None else dev(torch, C), want_comm=want_comm)


# ------------------------------------------------------------------ K1
def test_liouvillian_matches_oracle(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.cfg2(batch=3, N=8)
    L0, Lc, Lcomm = build_basis(torch, qal, p, want_comm=True)
    for b in range(3):
        rL0, rLc = oracle.build_liouvillian(p.H0[b], p.Hc, p.C)
        assert np.max(np.abs(L0[b].cpu().numpy() - rL0)) <= 1e-15
        assert np.max(np.abs(Lc.cpu().numpy() - rLc)) <= 1e-15
        # commutator basis [L0, L_j], [L_1, L_2] vs the oracle's plain products
        got = Lcomm[b].cpu().numpy()
        for j in range(2):
            ref = oracle.matmul(rL0, rLc[j]) - oracle.matmul(rLc[j], rL0)
            assert relfro(got[j], ref) <= 1e-14
        ref = oracle.matmul(rLc[0], rLc[1]) - oracle.matmul(rLc[1], rLc[0])
        assert relfro(got[2], ref) <= 1e-14


# ------------------------------------------------------------------ K3 per slice
@pytest.fixture(scope="module")
def cfg0_ref(oracle):
    p = qi.cfg0()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam, Us = oracle.propagate(L0, Lc, p.u[0], p.T, p.N, store=True)
    return p, L0, Lc, Lam, Us


def test_slice_exponentials_match_oracle(torch_cuda, qal, cfg0_ref):
    torch = torch_cuda
    p, _, _, _, Us = cfg0_ref
    L0, Lc, _ = build_basis(torch, qal, p)
    U, _ = qal.qal_magnus_expm_slices(L0, Lc, dev(torch, p.u), p.T, p.N, want_U=True)
    U = U[0].cpu().numpy()
    errs = [relfro(U[k], Us[k]) for k in range(p.N)]
    assert max(errs) <= 1e-13, max(errs)


@pytest.mark.parametrize("chunk", [1, 4, 16, 64, 256])
def test_chunk_fold_and_tree_match_oracle(torch_cuda, qal, cfg0_ref, chunk):
    torch = torch_cuda
    p, _, _, Lam, _ = cfg0_ref
    L0, Lc, _ = build_basis(torch, qal, p)
    _, P = qal.qal_magnus_expm_slices(L0, Lc, dev(torch, p.u), p.T, p.N, chunk=chunk)
    got = qal.qal_ordered_product(P)[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP


@pytest.mark.parametrize("count", [1, 2, 3, 5, 7, 13, 16])
def test_ordered_product_ragged_counts(torch_cuda, qal, oracle, count):
    torch = torch_cuda
    rng = np.random.default_rng(count)
    U = (rng.standard_normal((2, count, 64, 64)) + 1j * rng.standard_normal((2, count, 64, 64))) / 8.0
    got = qal.qal_ordered_product(dev(torch, U)).cpu().numpy()
    for b in range(2):
        assert relfro(got[b], oracle.ordered_product(U[b])) <= 1e-13


def test_ordering_later_slice_on_the_left(torch_cuda, qal, oracle):
    """S:264 analog: A (earlier) then B (later) gives B A, not A B."""
    torch = torch_cuda
    rng = np.random.default_rng(7)
    A = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
    B = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
    got = qal.qal_ordered_product(dev(torch, np.stack([A, B])[None]))[0].cpu().numpy()
    assert relfro(got, oracle.matmul(B, A)) <= 1e-14
    assert relfro(got, oracle.matmul(A, B)) > 1e-3


# ------------------------------------------------------------------ K5 + whole path, cfg0
def test_fidelity_matches_oracle(torch_cuda, qal, oracle, cfg0_ref):
    torch = torch_cuda
    p, _, _, Lam, _ = cfg0_ref
    F = qal.qal_fidelity(dev(torch, Lam[None]), dev(torch, p.V)).cpu().numpy()[0]
    Fr = oracle.fidelity(Lam, p.V)
    assert abs(F - Fr) <= 1e-13 * abs(Fr) + 1e-16


def test_cfg0_forward_path(torch_cuda, qal, oracle, cfg0_ref):
    torch = torch_cuda
    p, _, _, Lam, _ = cfg0_ref
    L0, Lc, _ = build_basis(torch, qal, p)
    F, g, Lg = qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), p.T, p.N, dev(torch, p.V), want_grad=False,
                                     want_Lambda=True)
    assert relfro(Lg[0].cpu().numpy(), Lam) <= TOL_PROP
    Fr = oracle.fidelity(Lam, p.V)
    assert abs(F.cpu().item() - Fr) / abs(Fr) <= TOL_PROP


# ------------------------------------------------------------------ K6, cfg1
@pytest.fixture(scope="module")
def cfg1_ref(oracle):
    p = qi.cfg1()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    F, g, Lam = oracle.gradient(L0, Lc, p.u[0], p.T, p.N, p.V)
    return p, F, g, Lam


def test_cfg1_gradient_matches_oracle(torch_cuda, qal, cfg1_ref):
    torch = torch_cuda
    p, Fr, gr, Lam = cfg1_ref
    L0, Lc, _ = build_basis(torch, qal, p)
    F, g, Lg = qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), p.T, p.N, dev(torch, p.V), want_Lambda=True)
    assert relfro(Lg[0].cpu().numpy(), Lam) <= TOL_PROP
    assert abs(F.cpu().item() - Fr) / abs(Fr) <= TOL_PROP
    g = g[0].cpu().numpy()
    assert g.shape == gr.shape
    assert relfro(g, gr) <= TOL_GRAD, relfro(g, gr)


# ------------------------------------------------------------------ batch with per-pulse drift (cfg2 recipe)
def test_cfg2_small_batch_forward_and_gradient(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.cfg2(batch=3, N=32, T=200.0 * 32 / 1024)
    L0, Lc, _ = build_basis(torch, qal, p)
    F, g, Lg = qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), p.T, p.N, dev(torch, p.V), want_Lambda=True)
    for b in range(3):
        rL0, rLc = oracle.build_liouvillian(p.H0[b], p.Hc, p.C)
        Fr, gr, Lam = oracle.gradient(rL0, rLc, p.u[b], p.T, p.N, p.V)
        assert relfro(Lg[b].cpu().numpy(), Lam) <= TOL_PROP
        assert abs(F[b].item() - Fr) / abs(Fr) <= TOL_PROP
        assert relfro(g[b].cpu().numpy(), gr) <= TOL_GRAD


# ------------------------------------------------------------------ NODES (cfg3 recipe), Magnus-4 commutator
def cfg3_short(oracle, N=512, T=10_000.0 * 512 / (1 << 20) * 8):
    p = qi.cfg3()
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)
    return p, u[None], N, T


def test_nodes_mode_forward_and_gradient(torch_cuda, qal, oracle):
    torch = torch_cuda
    p, u, N, T = cfg3_short(oracle, N=64, T=300.0)
    L0, Lc, Lcomm = build_basis(torch, qal, p, want_comm=True)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, Lam = oracle.gradient(rL0, rLc, u[0], T, N, p.V, mode=1)
    F, g, Lg = qal.qal_fidelity_grad(L0, Lc, dev(torch, u), T, N, dev(torch, p.V), ctrl_mode=1, Lcomm=Lcomm,
                                     want_Lambda=True)
    assert relfro(Lg[0].cpu().numpy(), Lam) <= TOL_PROP
    assert abs(F.item() - Fr) / abs(Fr) <= TOL_PROP
    assert g.shape == (1, N, 2, 2)
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD


@pytest.mark.parametrize("order", [2, 4])
def test_nodes_mode_chunked_forward(torch_cuda, qal, oracle, order):
    torch = torch_cuda
    p, u, N, T = cfg3_short(oracle)
    L0, Lc, Lcomm = build_basis(torch, qal, p, want_comm=True)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(rL0, rLc, u[0], T, N, mode=1, order=order)
    _, P = qal.qal_magnus_expm_slices(L0, Lc, dev(torch, u), T, N, magnus_order=order, ctrl_mode=1,
                                      Lcomm=Lcomm, chunk=64)
    got = qal.qal_ordered_product(P)[0].cpu().numpy()
    assert relfro(got, Lam) <= TOL_PROP


def test_slice_range_k0(torch_cuda, qal, oracle):
    """Time sharding: slices [k0, k0+count) of the global grid (cfg3 per-rank call)."""
    torch = torch_cuda
    p, u, N, T = cfg3_short(oracle, N=256, T=200.0)
    L0, Lc, Lcomm = build_basis(torch, qal, p, want_comm=True)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    k0, cnt = 96, 64
    Lam = oracle.propagate(rL0, rLc, u[0], T, N, mode=1, k0=k0, k1=k0 + cnt)
    _, P = qal.qal_magnus_expm_slices(L0, Lc, dev(torch, u[:, k0:k0 + cnt]), T, N, k0=k0, count=cnt,
                                      ctrl_mode=1, Lcomm=Lcomm, chunk=cnt)
    assert relfro(P[0, 0].cpu().numpy(), Lam) <= TOL_PROP


# ------------------------------------------------------------------ scaling and squaring (s > 0), m = 8 / 12
@pytest.mark.parametrize("T,N", [(100.0, 4), (100.0, 16), (100.0, 64), (1000.0, 2), (3.0, 8)])
def test_norm_regimes_match_oracle(torch_cuda, qal, oracle, T, N):
    """Large ||Omega|| (s > 0 squarings) and small ones (m = 8, 12), forward and gradient."""
    torch = torch_cuda
    p = qi.cfg0(N=N, T=T)
    L0, Lc, _ = build_basis(torch, qal, p)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, Lam = oracle.gradient(rL0, rLc, p.u[0], T, N, p.V)
    F, g, Lg = qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), T, N, dev(torch, p.V), want_Lambda=True)
    assert relfro(Lg[0].cpu().numpy(), Lam) <= TOL_PROP
    assert abs(F.item() - Fr) <= TOL_PROP * max(abs(Fr), 1e-3)
    assert relfro(g[0].cpu().numpy(), gr) <= TOL_GRAD


# ------------------------------------------------------------------ invariants on the GPU result
def test_zero_dissipation_is_conj_u_kron_u(torch_cuda, qal, oracle):
    """P-3: without collapse ops Lambda = conj(U) (x) U with U unitary (Hilbert-space Magnus)."""
    torch = torch_cuda
    p = qi.cfg0(N=64)
    p.C = np.zeros((0, 8, 8), np.complex128)
    L0, Lc, _ = build_basis(torch, qal, p)
    F, _, Lg = qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), p.T, p.N, dev(torch, p.V), want_grad=False,
                                     want_Lambda=True)
    Lam = Lg[0].cpu().numpy()
    # Hilbert-space propagator from the oracle's expm on -i h H_k (PWC: Magnus-4 exact per slice)
    h = p.T / p.N
    U = np.eye(8, dtype=np.complex128)
    for k in range(p.N):
        Hk = p.H0[0] + sum(p.u[0, k, j] * p.Hc[j] for j in range(2))
        U = oracle.expm(-1j * h * Hk) @ U
    assert np.linalg.norm(U.conj().T @ U - np.eye(8)) <= 1e-13
    assert relfro(Lam, np.kron(U.conj(), U)) <= TOL_PROP


def test_trace_and_hermiticity_preservation(torch_cuda, qal, cfg0_ref):
    """P-4, P-5 on the GPU propagator."""
    torch = torch_cuda
    p = cfg0_ref[0]
    L0, Lc, _ = build_basis(torch, qal, p)
    _, _, Lg = qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), p.T, p.N, dev(torch, p.V), want_grad=False,
                                     want_Lambda=True)
    Lam = Lg[0].cpu().numpy()
    vecI = np.eye(8).reshape(-1, order="F")
    assert np.max(np.abs(vecI @ Lam - vecI)) <= 1e-13
    d = 8
    idx = np.arange(64)
    sw = (idx // d) + d * (idx % d)        # i + d j  ->  j + d i
    assert np.max(np.abs(Lam - Lam[sw][:, sw].conj())) <= 1e-13


def test_status_flags_nonfinite_input(torch_cuda, qal):
    torch = torch_cuda
    p = qi.cfg0(N=8)
    L0, Lc, _ = build_basis(torch, qal, p)
    u = p.u.copy()
    u = np.concatenate([u, u], axis=0)
    u[1, 3, 0] = np.nan
    status = torch.full((2,), 7, dtype=torch.int32, device="cuda")
    qal.qal_magnus_expm_slices(L0, Lc, dev(torch, u), p.T, p.N, chunk=8, status=status)
    assert status.cpu().tolist() == [0, -4]


def test_determinism_bit_identical(torch_cuda, qal, cfg0_ref):
    torch = torch_cuda
    p = cfg0_ref[0]
    L0, Lc, _ = build_basis(torch, qal, p)
    outs = [qal.qal_fidelity_grad(L0, Lc, dev(torch, p.u), p.T, p.N, dev(torch, p.V)) for _ in range(2)]
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


# ------------------------------------------------------------------ a1, NODES controls on the device
@pytest.mark.parametrize("k0,count", [(0, 4096), ((1 << 20) - 777, 777), (123456, 1)])
def test_sines_sampler_matches_oracle(torch_cuda, qal, oracle, k0, count):
    torch = torch_cuda
    p = qi.cfg3()
    got = qal.qal_sample_controls_sines(dev(torch, p.sines), p.u_max, p.N, p.T, k0, count).cpu().numpy()
    ref = oracle.sines_nodes(p.sines, p.u_max, p.N, p.T, k0, k0 + count)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) <= 1e-13 * p.u_max


# ------------------------------------------------------------------ log-depth scans
@pytest.mark.parametrize("count", [1, 2, 5, 13, 64])
def test_ordered_scan_matches_oracle(torch_cuda, qal, oracle, count):
    torch = torch_cuda
    rng = np.random.default_rng(count)
    U = (rng.standard_normal((2, count, 64, 64)) + 1j * rng.standard_normal((2, count, 64, 64))) / 8.0
    pre, suf = qal.qal_ordered_scan(dev(torch, U))
    pre, suf = pre.cpu().numpy(), suf.cpu().numpy()
    I = np.eye(64)
    for b in range(2):
        for s in range(count):
            rp = oracle.ordered_product(U[b, :s]) if s > 0 else I
            rs = oracle.ordered_product(U[b, s + 1:]) if s + 1 < count else I
            assert relfro(pre[b, s], rp) <= 1e-12 and relfro(suf[b, s], rs) <= 1e-12


def test_batched_matmul_broadcast(torch_cuda, qal, oracle):
    torch = torch_cuda
    rng = np.random.default_rng(3)
    A = rng.standard_normal((1, 64, 64)) + 1j * rng.standard_normal((1, 64, 64))
    B = rng.standard_normal((4, 64, 64)) + 1j * rng.standard_normal((4, 64, 64))
    C = qal.qal_batched_matmul(dev(torch, A), dev(torch, B)).cpu().numpy()
    for i in range(4):
        assert relfro(C[i], oracle.matmul(A[0], B[i])) <= 1e-14
