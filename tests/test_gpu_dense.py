"""configs[4] (six spins, d = 64, n = 4096): the dense tiled DMMA path vs the oracle.

The oracle cannot form a 4096^2 propagator in test time, so the checks are: the
Liouvillian element by element (the oracle's literal Kronecker build is O(n^2)); sampled
rows of dense products; the zero-dissipation identity Lambda = conj(U) (x) U with U from
the oracle's 64 x 64 exponentials (P-3); the dissipative propagator applied to density
matrices vs the oracle's RK4 of Eq. 6 on rho itself; the fidelity; trace / Hermiticity
preservation (P-4, P-5) at full pulse length."""
import numpy as np
import pytest

from paper_2511_13330_b200 import inputs as qi

pytestmark = pytest.mark.gpu


def relfro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def qal(torch_cuda):
    from paper_2511_13330_b200 import _build, qal as q
    _build.build()
    q.load()
    return q


def to(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def cfg4(torch_cuda, qal):
    torch = torch_cuda
    p = qi.cfg4(batch=2)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    return p, L0, Lc


def test_dense_liouvillian_matches_oracle(cfg4, oracle):
    p, L0, Lc = cfg4
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    assert np.max(np.abs(L0[0].cpu().numpy() - rL0)) <= 1e-15
    assert np.max(np.abs(Lc[2].cpu().numpy() - rLc[2])) <= 1e-15


@pytest.mark.parametrize("count", [2, 3])
def test_dense_products_sampled_rows(torch_cuda, qal, oracle, count):
    torch = torch_cuda
    rng = np.random.default_rng(count)
    U = (rng.standard_normal((1, count, 4096, 4096)) + 1j * rng.standard_normal((1, count, 4096, 4096))) / 64.0
    got = qal.qal_ordered_product(to(torch, U))[0].cpu().numpy()
    rows = [0, 1, 2047, 4095]
    if count == 2:
        ref = np.concatenate([oracle.matmul_rows(U[0, 1], U[0, 0], r, r + 1) for r in rows])
    else:  # U2 U1 U0 row by row on the host: rows r of U2 U1 (oracle), then those rows times U0 (oracle);
        # associativity makes this the tree's (U2 carried) * (U1 U0) up to rounding, with no GPU value in it
        W = np.zeros((4096, 4096), np.complex128)
        for i, r in enumerate(rows):
            W[i] = oracle.matmul_rows(U[0, 2], U[0, 1], r, r + 1)[0]
        ref = oracle.matmul_rows(W, U[0, 0], 0, len(rows))
    for i, r in enumerate(rows):
        assert relfro(got[r], ref[i]) <= 1e-13


def test_dense_zero_dissipation_is_conj_u_kron_u(torch_cuda, qal, oracle):
    torch = torch_cuda
    N = 8
    p = qi.cfg4(batch=1, N=N, T=100.0 * N / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), None)
    _, P = qal.qal_magnus_expm_slices(L0, Lc, to(torch, p.u), p.T, N, chunk=N)
    Lam = P[0, 0].cpu().numpy()
    h = p.T / N
    U = np.eye(64, dtype=np.complex128)
    for k in range(N):
        Hk = p.H0[0] + sum(p.u[0, k, j] * p.Hc[j] for j in range(5))
        U = oracle.matmul(oracle.expm(-1j * h * Hk), U)
    assert np.linalg.norm(U.conj().T @ U - np.eye(64)) <= 1e-13
    assert relfro(Lam, np.kron(U.conj(), U)) <= 1e-10


@pytest.fixture(scope="module")
def dissipative_short(torch_cuda, qal):
    torch = torch_cuda
    N = 2
    p = qi.cfg4(batch=1, N=N, T=100.0 * N / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    _, P = qal.qal_magnus_expm_slices(L0, Lc, to(torch, p.u), p.T, N, chunk=N)
    return p, P[0, 0].cpu().numpy()


def test_dense_dissipative_propagator_vs_rk4_on_rho(dissipative_short, oracle):
    p, Lam = dissipative_short
    rng = np.random.default_rng(9)
    for _ in range(2):
        a = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
        rho0 = a @ a.conj().T
        rho0 /= np.trace(rho0)
        ref = oracle.evolve_rho(p.H0[0], p.Hc, p.C, p.u[0], p.T, p.N, 256, rho0)
        got = (Lam @ rho0.reshape(-1, order="F")).reshape(64, 64, order="F")
        assert relfro(got, ref) <= 1e-10


def test_dense_fidelity_matches_oracle(dissipative_short, qal, oracle, torch_cuda):
    torch = torch_cuda
    p, Lam = dissipative_short
    F = qal.qal_fidelity(to(torch, Lam[None]), to(torch, p.V)).item()
    Fr = oracle.fidelity(Lam, p.V)
    assert abs(F - Fr) <= 1e-12 * abs(Fr) + 1e-17


def test_dense_fidelity_concurrent_streams_are_bit_identical(torch_cuda, qal):
    """SURVEY 8(b) reentrancy: the n = 4096 fidelity keeps no library-held scratch, so two calls on two
    streams at once (each with its own workspace for the slab reduction, and the no-workspace form)
    return exactly the serial results."""
    torch = torch_cuda
    V = to(torch, qi.haar_unitary(64, 5))
    gen = torch.Generator(device="cuda").manual_seed(11)
    lams = [torch.complex(torch.randn(2, 4096, 4096, dtype=torch.float64, device="cuda", generator=gen),
                          torch.randn(2, 4096, 4096, dtype=torch.float64, device="cuda", generator=gen))
            for _ in range(2)]
    wsb = qal.workspace_bytes(qal.QAL_OP_FIDELITY_REDUCE, 4096, 2, 1)
    assert wsb == 2 * 512 * 8
    ws = [torch.empty(wsb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    serial = [qal.qal_fidelity(L, V, ws=w) for L, w in zip(lams, ws)]
    serial1 = [qal.qal_fidelity(L, V) for L in lams]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            a = qal.qal_fidelity(lams[0], V, ws=ws[0], stream=s1)
            a1 = qal.qal_fidelity(lams[0], V, stream=s1)
        with torch.cuda.stream(s2):
            b = qal.qal_fidelity(lams[1], V, ws=ws[1], stream=s2)
            b1 = qal.qal_fidelity(lams[1], V, stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(a, serial[0]) and torch.equal(b, serial[1])
        assert torch.equal(a1, serial1[0]) and torch.equal(b1, serial1[1])
    # the two reductions (512 slabs + fixed-order sum vs one CTA) agree to rounding
    for x, y in zip(serial, serial1):
        assert torch.allclose(x, y, rtol=1e-12, atol=1e-12)


def check_cptp_invariants(Lam, tol):
    d = 64
    vecI = np.eye(d).reshape(-1, order="F")
    assert np.max(np.abs(vecI @ Lam - vecI)) <= tol
    idx = np.arange(d * d)
    sw = (idx // d) + d * (idx % d)
    assert np.max(np.abs(Lam - Lam[sw][:, sw].conj())) <= tol


def test_dense_full_pulse_invariants_and_fidelity_path(cfg4, qal, torch_cuda):
    """configs[4] pulse 0 at full length (512 slices), in bench.py's launch configuration."""
    torch = torch_cuda
    p, L0, Lc = cfg4
    F, _, Lg = qal.qal_fidelity_grad(L0[:1].contiguous(), Lc, to(torch, p.u[:1]), p.T, p.N, to(torch, p.V),
                                     want_grad=False, want_Lambda=True)
    Lam = Lg[0].cpu().numpy()
    check_cptp_invariants(Lam, 1e-10)
    assert 0.0 < F.item() < 1.0


# ------------------------------------------------------------------ NEXT f3: 3-dot Hubbard model (Eq. 1)
@pytest.fixture(scope="module")
def hub(torch_cuda, qal):
    torch = torch_cuda
    p = qi.hubbard3(N=2, T=100.0 * 2 / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    return p, L0, Lc


def test_hubbard_liouvillian_matches_oracle(hub, oracle):
    p, L0, Lc = hub
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    assert np.max(np.abs(L0[0].cpu().numpy() - rL0)) <= 1e-13
    assert np.max(np.abs(Lc.cpu().numpy() - rLc)) <= 1e-13


def test_hubbard_zero_dissipation_is_conj_u_kron_u(torch_cuda, qal, oracle):
    torch = torch_cuda
    p = qi.hubbard3(N=4, T=100.0 * 4 / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), None)
    _, P = qal.qal_magnus_expm_slices(L0, Lc, to(torch, p.u), p.T, p.N, chunk=p.N)
    h = p.T / p.N
    U = np.eye(64, dtype=np.complex128)
    for k in range(p.N):
        Hk = p.H0[0] + sum(p.u[0, k, j] * p.Hc[j] for j in range(2))
        U = oracle.matmul(oracle.expm(-1j * h * Hk), U)
    assert relfro(P[0, 0].cpu().numpy(), np.kron(U.conj(), U)) <= 1e-10


def test_hubbard_dissipative_slice_vs_rk4_on_rho(torch_cuda, qal, oracle):
    """one slice (||Omega||_1 ~ 25: s = 5 squarings on the device) applied to a density matrix vs the
    oracle's RK4 of Eq. 6 with 8192 sub-steps (global RK4 error ~ 2e-11)."""
    torch = torch_cuda
    p = qi.hubbard3(N=1, T=100.0 / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    _, P = qal.qal_magnus_expm_slices(L0, Lc, to(torch, p.u), p.T, 1, chunk=1)
    Lam = P[0, 0].cpu().numpy()
    phis = qi.hubbard_logical_states()
    rho0 = 0.7 * np.outer(phis[0], phis[0].conj()) + 0.3 * np.outer(phis[1], phis[1].conj())
    rho0 += 0.2 * (np.outer(phis[0], phis[1].conj()) + np.outer(phis[1], phis[0].conj()))
    ref = oracle.evolve_rho(p.H0[0], p.Hc, p.C, p.u[0], p.T, 1, 8192, rho0)
    got = (Lam @ rho0.reshape(-1, order="F")).reshape(64, 64, order="F")
    assert relfro(got, ref) <= 1e-10
    check_cptp_invariants(Lam, 1e-10)
