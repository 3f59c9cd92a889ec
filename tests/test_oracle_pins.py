"""Pins of the CPU oracle against things other than itself.

Independent references used here: closed forms, scipy.linalg.expm /
expm_frechet, numpy eigendecompositions, scipy.integrate.solve_ivp on Eq. 6
written in matrix form, and mathematical invariants.  No CUDA involved.
"""
import math

import numpy as np
import pytest
import scipy.integrate
import scipy.linalg

from paper_2511_13330_b200 import inputs as qi


def vec(rho):
    """column stacking: vec(rho)[i + d j] = rho[i, j]   (A5)"""
    return rho.reshape(-1, order="F")


def unvec(v, d):
    return v.reshape(d, d, order="F")


def rand_c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def rand_herm(rng, d):
    a = rand_c(rng, d, d)
    return (a + a.conj().T) / 2


def rand_rho(rng, d):
    a = rand_c(rng, d, d)
    r = a @ a.conj().T
    return r / np.trace(r)


def eq6_numpy(H, C, rho):
    """Eq. 6 in matrix form, written independently of the oracle."""
    out = -1j * (H @ rho - rho @ H)
    for c in C:
        cd = c.conj().T
        out += c @ rho @ cd - 0.5 * (cd @ c @ rho + rho @ cd @ c)
    return out


# ---------------------------------------------------------------- layout / Eq. 8
def test_vectorization_convention(oracle):
    # vec([[a,b],[c,d]]) = (a,c,b,d) and vec(H rho) = (I (x) H) vec(rho)
    assert np.array_equal(vec(np.array([[1, 2], [3, 4]])), [1, 3, 2, 4])
    rng = np.random.default_rng(1)
    H = rand_herm(rng, 3)
    L0, _ = oracle.build_liouvillian(H, np.zeros((0, 3, 3)), np.zeros((0, 3, 3)))
    rho = rand_c(rng, 3, 3)
    assert np.allclose(L0 @ vec(rho), vec(-1j * (H @ rho - rho @ H)), atol=1e-14)


@pytest.mark.parametrize("d", [2, 3, 8])
def test_eq8_matches_eq6(oracle, d):
    rng = np.random.default_rng(d)
    H = rand_herm(rng, d)
    C = rand_c(rng, 3, d, d) * 0.3
    Hc = np.stack([rand_herm(rng, d)])
    L0, Lc = oracle.build_liouvillian(H, Hc, C)
    rho = rand_rho(rng, d)
    want = eq6_numpy(H, C, rho)
    assert np.abs(L0 @ vec(rho) - vec(want)).max() < 1e-13
    assert np.abs(unvec(L0 @ vec(rho), d) - oracle.lindblad_rhs(H, C, rho)).max() < 1e-13
    # control Liouvillian has no dissipator: L_j vec(rho) = vec(-i[H_j, rho])
    assert np.abs(Lc[0] @ vec(rho) - vec(-1j * (Hc[0] @ rho - rho @ Hc[0]))).max() < 1e-13
    # spectrum of a Lindblad generator: Re(lambda) <= 0
    assert np.linalg.eigvals(L0).real.max() < 1e-9


def test_liouvillian_zero(oracle):
    L0, Lc = oracle.build_liouvillian(np.zeros((2, 2)), np.zeros((1, 2, 2)), np.zeros((0, 2, 2)))
    assert not L0.any() and not Lc.any()


# ---------------------------------------------------------------- expm (Eq. 14), P-11
@pytest.mark.parametrize("n,scale", [(4, 1e-3), (4, 3.0), (16, 0.7), (64, 0.05), (64, 0.9), (64, 12.0)])
def test_expm_vs_scipy(oracle, n, scale):
    rng = np.random.default_rng(n)
    A = rand_c(rng, n, n)
    A *= scale / np.abs(A).sum(0).max()
    E = oracle.expm(A)
    R = scipy.linalg.expm(A)
    assert np.linalg.norm(E - R) / np.linalg.norm(R) < 5e-14


def test_expm_closed_forms(oracle):
    assert np.array_equal(oracle.expm(np.zeros((5, 5), complex)), np.eye(5))
    dg = np.array([0.1, -2.0, 3.5 + 1j, -0.7j])
    assert np.allclose(oracle.expm(np.diag(dg)), np.diag(np.exp(dg)), rtol=1e-14, atol=0)
    assert np.array_equal(oracle.expm(np.array([[0, 1], [0, 0]], complex)), [[1, 1], [0, 1]])
    # e^{-iHt} for Hermitian H via the eigendecomposition (independent of any expm)
    rng = np.random.default_rng(7)
    H = rand_herm(rng, 8)
    w, Q = np.linalg.eigh(H)
    want = (Q * np.exp(-1j * w * 1.7)) @ Q.conj().T
    assert np.abs(oracle.expm(-1j * 1.7 * H) - want).max() < 1e-13


# ---------------------------------------------------------------- Frechet, P-9
def test_frechet_vs_scipy(oracle):
    rng = np.random.default_rng(3)
    for n, s in [(4, 0.5), (16, 1.3), (64, 0.4)]:
        A = rand_c(rng, n, n)
        A *= s / np.abs(A).sum(0).max()
        E = rand_c(rng, n, n)
        L, X = oracle.frechet(A, E)
        Xs, Ls = scipy.linalg.expm_frechet(A, E)
        assert np.linalg.norm(L - Ls) / np.linalg.norm(Ls) < 1e-13
        assert np.linalg.norm(X - Xs) / np.linalg.norm(Xs) < 1e-13
        # commuting case L(A, A) = A e^A
        L2, _ = oracle.frechet(A, A)
        assert np.linalg.norm(L2 - A @ Xs) / np.linalg.norm(L2) < 1e-13


# ---------------------------------------------------------------- RK4 oracle (O8)
def test_rk4_precession_and_order(oracle):
    b, T = 2.0, math.pi
    H0 = (b / 2) * qi.SZ
    L0, Lc = oracle.build_liouvillian(H0, np.zeros((1, 2, 2)), np.zeros((0, 2, 2)))
    rho0 = np.array([[0.5, 0.5], [0.5, 0.5]], complex)
    errs = []
    for sub in (8, 16):
        Lam = oracle.rk4(L0, Lc, T, 4, sub, u=np.zeros((4, 1)))
        rho = unvec(Lam @ vec(rho0), 2)
        errs.append(abs(rho[0, 1] - 0.5 * np.exp(-1j * b * T)))
    Lam = oracle.rk4(L0, Lc, T, 4, 256, u=np.zeros((4, 1)))
    assert abs(unvec(Lam @ vec(rho0), 2)[0, 1] - 0.5 * np.exp(-1j * b * T)) < 1e-8
    assert 4 - 0.3 < math.log2(errs[0] / errs[1]) < 4 + 0.3


# ---------------------------------------------------------------- P-1, P-2, P-12
def test_p1_identity(oracle):
    L0, Lc = oracle.build_liouvillian(np.zeros((8, 8)), np.zeros((2, 8, 8)), np.zeros((0, 8, 8)))
    Lam = oracle.propagate(L0, Lc, np.zeros((16, 2)), 10.0, 16)
    assert np.array_equal(Lam, np.eye(64))


def test_p2_constant_controls(oracle):
    p = qi.cfg0()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    T = 25.0
    uc = np.array([0.1, 0.2])
    L = L0 + uc[0] * Lc[0] + uc[1] * Lc[1]
    ref = scipy.linalg.expm(T * L)
    lam1 = oracle.propagate(L0, Lc, np.tile(uc, (1, 1)), T, 1)
    lam8 = oracle.propagate(L0, Lc, np.tile(uc, (8, 1)), T, 8)
    assert np.linalg.norm(lam1 - ref) / np.linalg.norm(ref) < 1e-12
    assert np.linalg.norm(lam8 - lam1) / np.linalg.norm(ref) < 1e-12


def test_p12_ordering_and_semigroup(oracle):
    p = qi.cfg0()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    u = np.array([[0.3, 0.0], [0.0, 0.3]])          # slice 0 (earlier) then slice 1 (later)
    h = 3.0
    A = scipy.linalg.expm(h * (L0 + 0.3 * Lc[0]))
    B = scipy.linalg.expm(h * (L0 + 0.3 * Lc[1]))
    assert np.linalg.norm(A @ B - B @ A) > 1e-3        # non-commuting fixture
    Lam = oracle.propagate(L0, Lc, u, 2 * h, 2)
    assert np.linalg.norm(Lam - B @ A) < 1e-12
    assert np.linalg.norm(Lam - A @ B) > 1e-3
    # [0, T] = [T/2, T] o [0, T/2]
    N = 32
    full = oracle.propagate(L0, Lc, p.u[0, :N], 12.5, N)
    first = oracle.propagate(L0, Lc, p.u[0, :N], 12.5, N, k1=N // 2)
    second = oracle.propagate(L0, Lc, p.u[0, :N], 12.5, N, k0=N // 2)
    assert np.linalg.norm(second @ first - full) / np.linalg.norm(full) < 1e-13
    # ordered product helper: earlier on the right
    assert np.allclose(oracle.ordered_product(np.stack([A, B])), B @ A, atol=1e-14)


# ---------------------------------------------------------------- P-3, P-4, P-5, P-13
def hilbert_magnus4(H1, H2, h):
    """Hilbert-space 4th-order Magnus generator for one slice (test's own Hilbert-space form)."""
    A1, A2 = -1j * H1, -1j * H2
    return 0.5 * h * (A1 + A2) - math.sqrt(3) * h * h / 12 * (A1 @ A2 - A2 @ A1)


@pytest.mark.parametrize("mode", [0, 1])
def test_p3_zero_dissipation(oracle, mode):
    p = qi.cfg0()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, np.zeros((0, 8, 8)))
    N, T = 64, 25.0
    h = T / N
    rng = np.random.default_rng(11)
    if mode == 0:
        u = p.u[0, :N]
        nodes = np.stack([u, u], axis=1)
    else:
        nodes = rng.uniform(0, qi.U_MAX, (N, 2, 2))
        u = nodes
    Lam = oracle.propagate(L0, Lc, u, T, N, mode=mode)
    U = np.eye(8, dtype=complex)
    for k in range(N):
        H1 = p.H0[0] + nodes[k, 0, 0] * p.Hc[0] + nodes[k, 0, 1] * p.Hc[1]
        H2 = p.H0[0] + nodes[k, 1, 0] * p.Hc[0] + nodes[k, 1, 1] * p.Hc[1]
        U = scipy.linalg.expm(hilbert_magnus4(H1, H2, h)) @ U
    assert np.abs(U.conj().T @ U - np.eye(8)).max() < 1e-13
    want = np.kron(U.conj(), U)
    assert np.linalg.norm(Lam - want) / np.linalg.norm(want) < 1e-12


def test_p4_p5_p13_invariants(oracle):
    p = qi.cfg0()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(L0, Lc, p.u[0], p.T, p.N)
    d = 8
    vI = vec(np.eye(d))
    assert np.abs(vI.conj() @ Lam - vI.conj()).max() < 1e-13               # P-4 trace
    idx = np.arange(64)
    i, j = idx % d, idx // d
    swap = j + d * i                                                          # (i,j) -> (j,i)
    assert np.abs(Lam - Lam[np.ix_(swap, swap)].conj()).max() < 1e-13         # P-5 Hermiticity
    # P-13 coherence-order blocks: m(i) = magnetisation of basis state i
    m = np.array([sum(1 if ((s >> (2 - q)) & 1) == 0 else -1 for q in range(3)) for s in range(d)])
    q = m[i] - m[j]
    off = q[:, None] != q[None, :]
    assert np.count_nonzero(Lam[off]) == 0
    assert np.count_nonzero(L0[off]) == 0 and np.count_nonzero(Lc[:, off]) == 0
    sizes = sorted(np.bincount(q + 6)[np.bincount(q + 6) > 0].tolist(), reverse=True)
    assert sizes == [20, 15, 15, 6, 6, 1, 1]


# ---------------------------------------------------------------- P-6 single-spin closed forms
def _spin_lam(oracle, H0, Hx, C, T, N, W=0.0):
    L0, Lc = oracle.build_liouvillian(H0, Hx[None], C)
    return oracle.propagate(L0, Lc, np.full((N, 1), W), T, N)


def test_p6_precession_and_decay(oracle):
    b, t1, t2, T = 0.9, 50.0, 20.0, 7.3
    C = np.stack([qi.SMINUS / math.sqrt(t1), qi.SZ * math.sqrt(1 / (2 * t2))])
    Lam = _spin_lam(oracle, (b / 2) * qi.SZ, 0.5 * qi.SX, C, T, 4)
    rho0 = np.array([[0.6, 0.3 - 0.2j], [0.3 + 0.2j, 0.4]])
    rho = unvec(Lam @ vec(rho0), 2)
    assert abs(rho[0, 1] - rho0[0, 1] * np.exp(-1j * b * T - T / t2 - T / (2 * t1))) < 1e-14
    assert abs(rho[0, 0] - rho0[0, 0] * np.exp(-T / t1)) < 1e-14


def test_p6_rabi_with_dephasing(oracle):
    W, t2, T = 1.3, 4.0, 6.0
    C = np.stack([qi.SZ * math.sqrt(1 / (2 * t2))])
    Lam = _spin_lam(oracle, np.zeros((2, 2)), 0.5 * qi.SX, C, T, 16, W=W)
    rho = unvec(Lam @ vec(np.array([[1, 0], [0, 0]], complex)), 2)
    kap = 1 / (2 * t2)
    mu = math.sqrt(W * W - kap * kap)
    want = math.exp(-kap * T) * (math.cos(mu * T) + kap / mu * math.sin(mu * T))
    assert abs((rho[0, 0] - rho[1, 1]).real - want) < 1e-13


# ---------------------------------------------------------------- P-7 order 4 (A1, A2)
def _smooth_case():
    p = qi.cfg0()
    C = qi.collapse_ops(3, t1=200.0, t2=50.0)        # stronger dissipation: exercise the dissipator
    prm = qi.sine_params(9, 2, nterm=4)
    prm[:, :, 1] *= 4.0                                # faster controls: visible time dependence
    return p, C, prm


def _ivp_reference(p, C, prm, T, rho0, oracle):
    def rhs(t, y):
        u = oracle.sines_eval(prm, qi.U_MAX, t)
        H = p.H0[0] + u[0] * p.Hc[0] + u[1] * p.Hc[1]
        return eq6_numpy(H, C, y.reshape(8, 8)).reshape(-1)
    sol = scipy.integrate.solve_ivp(rhs, (0, T), rho0.reshape(-1).astype(complex), method="DOP853",
                                    rtol=1e-13, atol=1e-15)
    return sol.y[:, -1].reshape(8, 8)


def test_p7_magnus4_order(oracle):
    p, C, prm = _smooth_case()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, C)
    T = 12.0
    rho0 = rand_rho(np.random.default_rng(5), 8)
    ref = _ivp_reference(p, C, prm, T, rho0, oracle)
    errs = {}
    for order in (4, 2):
        e = []
        for N in (8, 16, 32):
            u = oracle.sines_nodes(prm, qi.U_MAX, N, T)
            Lam = oracle.propagate(L0, Lc, u, T, N, mode=1, order=order)
            e.append(np.abs(unvec(Lam @ vec(rho0), 8) - ref).max())
        errs[order] = e
    o4 = [math.log2(errs[4][i] / errs[4][i + 1]) for i in range(2)]
    o2 = [math.log2(errs[2][i] / errs[2][i + 1]) for i in range(2)]
    assert all(3.7 < o < 4.3 for o in o4), o4
    assert all(1.7 < o < 2.3 for o in o2), o2


def test_p7_magnus4_sign_is_detected(oracle):
    """The flipped commutator sign must NOT give order 4 (sign detector, A2)."""
    p, C, prm = _smooth_case()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, C)
    T = 12.0
    rho0 = rand_rho(np.random.default_rng(5), 8)
    ref = _ivp_reference(p, C, prm, T, rho0, oracle)
    e = []
    for N in (8, 16, 32):
        h = T / N
        u = oracle.sines_nodes(prm, qi.U_MAX, N, T)
        Lam = np.eye(64, dtype=complex)
        for k in range(N):
            A1 = L0 + u[k, 0, 0] * Lc[0] + u[k, 0, 1] * Lc[1]
            A2 = L0 + u[k, 1, 0] * Lc[0] + u[k, 1, 1] * Lc[1]
            Om = 0.5 * h * (A1 + A2) + math.sqrt(3) * h * h / 12 * (A1 @ A2 - A2 @ A1)
            Lam = scipy.linalg.expm(Om) @ Lam
        e.append(np.abs(unvec(Lam @ vec(rho0), 8) - ref).max())
    assert math.log2(e[1] / e[2]) < 3.0


def test_p7_pwc_matches_rk4(oracle):
    p = qi.cfg0()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    N, T = 8, 4.0
    u = p.u[0, :N]
    Lam = oracle.propagate(L0, Lc, u, T, N)
    e1 = np.abs(oracle.rk4(L0, Lc, T, N, 32, u=u) - Lam).max()
    e2 = np.abs(oracle.rk4(L0, Lc, T, N, 64, u=u) - Lam).max()
    assert e2 < 1e-8 and 14 < e1 / e2 < 18


def test_rk4_sinusoid_mode_matches_solve_ivp_and_is_order_4(oracle):
    """O8 with continuous controls (cmode 2): the RK4 of Eq. 9 evaluating u(t) at every stage agrees
    with an independent DOP853 integration of Eq. 6 (matrix form, tight tolerances), and halving its
    step divides the error by ~16."""
    p, C, prm = _smooth_case()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, C)
    T = 12.0
    rho0 = rand_rho(np.random.default_rng(5), 8)
    ref = _ivp_reference(p, C, prm, T, rho0, oracle)
    errs = []
    for sub in (32, 64):
        Lam = oracle.rk4(L0, Lc, T, 8, sub, prm=prm, umax=qi.U_MAX)
        errs.append(np.abs(unvec(Lam @ vec(rho0), 8) - ref).max())
    assert errs[1] <= 3e-8, errs
    assert 13.0 < errs[0] / errs[1] < 19.0, errs


# ---------------------------------------------------------------- P-10 fidelity
def test_p10_fidelity(oracle):
    V = qi.haar_unitary(8, 0)
    assert abs(oracle.fidelity(np.kron(V.conj(), V), V) - 1.0) < 1e-14
    U = qi.haar_unitary(8, 1)
    want = abs(np.trace(V.conj().T @ U)) ** 2 / 64
    assert abs(oracle.fidelity(np.kron(U.conj(), U), V) - want) < 1e-15
    # CPTP Lambda: F in [0, 1]
    p = qi.cfg0()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    F = oracle.fidelity(oracle.propagate(L0, Lc, p.u[0, :32], 12.5, 32), V)
    assert 0.0 <= F <= 1.0


# ---------------------------------------------------------------- P-8 gradient vs FD
def _fd(oracle, L0, Lc, u, T, N, V, mode, eps=1e-6, entries=None):
    g = np.zeros(u.shape)
    flat = list(np.ndindex(*u.shape)) if entries is None else entries
    for ix in flat:
        up, um = u.copy(), u.copy()
        up[ix] += eps
        um[ix] -= eps
        Fp = oracle.fidelity(oracle.propagate(L0, Lc, up, T, N, mode=mode), V)
        Fm = oracle.fidelity(oracle.propagate(L0, Lc, um, T, N, mode=mode), V)
        g[ix] = (Fp - Fm) / (2 * eps)
    return g


@pytest.mark.parametrize("mode", [0, 1])
def test_p8_gradient_vs_fd_d8(oracle, mode):
    p = qi.cfg0()
    C = qi.collapse_ops(3, t1=300.0, t2=60.0)
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, C)
    N, T = 6, 9.0
    rng = np.random.default_rng(21 + mode)
    u = p.u[0, :N] if mode == 0 else rng.uniform(0, qi.U_MAX, (N, 2, 2)) * 5
    F, g, Lam = oracle.gradient(L0, Lc, u, T, N, p.V, mode=mode)
    assert abs(F - oracle.fidelity(oracle.propagate(L0, Lc, u, T, N, mode=mode), p.V)) < 1e-15
    gfd = _fd(oracle, L0, Lc, u, T, N, p.V, mode)
    assert np.linalg.norm(g - gfd) / np.linalg.norm(gfd) < 1e-6


def test_p8_gradient_d2_and_small_T(oracle):
    C = np.stack([qi.SMINUS / math.sqrt(30.0), qi.SZ * math.sqrt(1 / 20.0)])
    L0, Lc = oracle.build_liouvillian(0.4 * qi.SZ, (0.5 * qi.SX)[None], C)
    V = qi.haar_unitary(2, 3)
    u = np.random.default_rng(2).uniform(0, 2, (5, 1))
    F, g, _ = oracle.gradient(L0, Lc, u, 3.0, 5, V)
    gfd = _fd(oracle, L0, Lc, u, 3.0, 5, V, 0)
    assert np.linalg.norm(g - gfd) / np.linalg.norm(gfd) < 1e-6
    # T -> 0: gradient -> 0 linearly in h
    _, g1, _ = oracle.gradient(L0, Lc, u, 1e-4, 5, V)
    _, g2, _ = oracle.gradient(L0, Lc, u, 2e-4, 5, V)
    assert np.abs(g1).max() < 1e-4 and abs(np.linalg.norm(g2) / np.linalg.norm(g1) - 2) < 1e-3


# ---------------------------------------------------------------- controls of configs[3] (A11)
def test_sines_controls_clip_and_nodes(oracle):
    prm = qi.sine_params(3, 2)
    ts = np.linspace(0, 2000, 4001)
    vals = np.array([oracle.sines_eval(prm, qi.U_MAX, t) for t in ts])
    assert vals.min() >= 0.0 and vals.max() <= qi.U_MAX
    clipped = np.mean((vals == 0.0) | (vals == qi.U_MAX))
    assert 0.0 < clipped < 0.2
    # node sampling = function at t_k + (1/2 -+ sqrt(3)/6) h
    N, T = 10, 50.0
    nodes = oracle.sines_nodes(prm, qi.U_MAX, N, T)
    h = T / N
    k = 7
    assert np.allclose(nodes[k, 0], oracle.sines_eval(prm, qi.U_MAX, k * h + (0.5 - math.sqrt(3) / 6) * h))
    assert np.allclose(nodes[k, 1], oracle.sines_eval(prm, qi.U_MAX, k * h + (0.5 + math.sqrt(3) / 6) * h))


def test_sines_single_term_extremes_and_period(oracle):
    """A11 pins from the mathematics of the normalised sum, not its formula: with one term the
    normalisation a / sqrt(a^2 / 2) makes s = sqrt(2) sin(.), so u never clips, has period 1/f, and
    reaches exactly u_max/2 (1 +- 1/sqrt(2)) where the sine peaks."""
    a, f, phi = 0.37, 0.0125, 0.9
    prm = np.array([[[a, f, phi]]])
    umax = qi.U_MAX
    t_peak = (0.25 - phi / (2 * math.pi)) / f            # 2 pi f t + phi = pi / 2
    t_trough = t_peak + 0.5 / f
    assert abs(oracle.sines_eval(prm, umax, t_peak)[0] - umax / 2 * (1 + 2 ** -0.5)) <= 1e-15 * umax
    assert abs(oracle.sines_eval(prm, umax, t_trough)[0] - umax / 2 * (1 - 2 ** -0.5)) <= 1e-15 * umax
    ts = np.linspace(0.0, 1.0 / f, 777)
    v = np.array([oracle.sines_eval(prm, umax, t)[0] for t in ts])
    v2 = np.array([oracle.sines_eval(prm, umax, t + 3.0 / f)[0] for t in ts])
    assert np.max(np.abs(v - v2)) <= 1e-13 * umax
    assert umax / 2 * (1 - 2 ** -0.5) - 1e-15 <= v.min() and v.max() <= umax / 2 * (1 + 2 ** -0.5) + 1e-15
    # a second control channel is independent of the first
    prm2 = np.array([[[a, f, phi]], [[1.0, 0.0, math.pi / 2]]])   # f = 0: s = sqrt(2), constant
    out = oracle.sines_eval(prm2, umax, 123.0)
    assert abs(out[1] - umax / 2 * (1 + 2 ** -0.5)) <= 1e-15 * umax


def test_sines_unit_rms_and_clipping(oracle):
    """The normalisation gives s unit RMS for incommensurate frequencies (mean sin^2 = 1/2, cross
    terms average out): two equal-amplitude terms never clip (|s| <= 2) and mean(s^2) -> 1; amplitudes
    pushing s beyond +-2 clip to exactly 0 and u_max."""
    umax = qi.U_MAX
    prm = np.array([[[0.5, 0.0101, 0.3], [0.5, 0.0163, 1.7]]])
    ts = np.linspace(0.0, 40000.0, 200001)
    u = np.array([oracle.sines_eval(prm, umax, t)[0] for t in ts])
    s = 4.0 * u / umax - 2.0                               # invert u = u_max/2 (1 + s/2) (no clipping)
    assert np.all((u > 0.0) & (u < umax))
    assert abs(np.mean(s * s) - 1.0) < 5e-3 and abs(np.mean(s)) < 5e-3
    # two equal terms: s = sin + sin, |s| <= 2 (Cauchy-Schwarz bound sqrt(2 n) with n = 2)
    assert np.max(np.abs(s)) <= 2.0 + 1e-12
    # a constant (f = 0) term at phase pi/2 plus a sinusoid: s = 1 + sin(.), reaching the bound 2
    prm_c = np.array([[[1.0, 0.0, math.pi / 2], [1.0, 0.02, 0.0]]])   # s = sin(.) + 1 over sqrt(1)
    t_hi = 0.25 / 0.02                                      # s = 2 (edge), u = u_max exactly
    t_lo = 0.75 / 0.02                                      # s = 0, u = u_max / 2
    assert abs(oracle.sines_eval(prm_c, umax, t_hi)[0] - umax) <= 1e-15 * umax
    assert abs(oracle.sines_eval(prm_c, umax, t_lo)[0] - umax / 2) <= 1e-15 * umax
    # Cauchy-Schwarz: |s| <= sqrt(2 n); three equal constant terms give s = 3 / sqrt(3/2) = sqrt(6) > 2
    prm_x = np.array([[[1.0, 0.0, math.pi / 2]] * 3])
    assert oracle.sines_eval(prm_x, umax, 5.0)[0] == umax
    prm_y = np.array([[[1.0, 0.0, -math.pi / 2]] * 3])
    assert oracle.sines_eval(prm_y, umax, 5.0)[0] == 0.0


def test_sines_nodes_are_gauss_legendre(oracle):
    """Node sampling pinned to numpy's Gauss-Legendre rule (leggauss(2) mapped onto each slice), and
    the 2-point rule's exactness for cubics: integrating the sampled slice values reproduces the
    exact integral of u over [0, T] up to the rule's O(h^4) error."""
    prm = qi.sine_params(3, 2)
    umax = qi.U_MAX
    N, T = 40, 200.0
    h = T / N
    xi, wts = np.polynomial.legendre.leggauss(2)
    nodes = oracle.sines_nodes(prm, umax, N, T)
    for k in (0, 17, N - 1):
        for a in range(2):
            t = k * h + h * (1.0 + xi[a]) / 2.0
            assert np.array_equal(nodes[k, a], oracle.sines_eval(prm, umax, t)) or \
                np.max(np.abs(nodes[k, a] - oracle.sines_eval(prm, umax, t))) <= 1e-15 * umax
    # composite 2-point Gauss vs a fine composite Simpson integral of the same function
    gauss = (h / 2.0) * np.einsum("a,kaj->j", wts, nodes)
    tf = np.linspace(0.0, T, 20001)
    uf = np.array([oracle.sines_eval(prm, umax, t) for t in tf])
    from scipy.integrate import simpson
    ref = simpson(uf, x=tf, axis=0)
    assert np.max(np.abs(gauss - ref)) <= 1e-3 * T * umax   # clipped kinks make u only C^0


# ---------------------------------------------------------------- helpers used by the d = 64 checks
def test_matmul_rows_is_the_matrix_product(oracle):
    rng = np.random.default_rng(11)
    A = rand_c(rng, 96, 96)
    B = rand_c(rng, 96, 96)
    got = oracle.matmul_rows(A, B, 17, 29)
    assert np.allclose(got, (A @ B)[17:29], rtol=0, atol=1e-12)


def test_evolve_rho_t1_decay_closed_form(oracle):
    """P-6(ii) on the density-matrix integrator: rho_upup(t) = e^{-t/T1}."""
    T1 = 7.0
    p = qi.single_spin("t1", T=5.0, N=5, t1=T1)
    rho0 = np.array([[1, 0], [0, 0]], dtype=np.complex128)
    rho = oracle.evolve_rho(p.H0[0], p.Hc, p.C, p.u[0], p.T, p.N, 64, rho0)
    assert abs(rho[0, 0] - math.exp(-5.0 / T1)) <= 1e-12
    assert abs(np.trace(rho) - 1.0) <= 1e-14


def test_evolve_rho_matches_solve_ivp_d8(oracle):
    """Eq. 6 with PWC controls on the 3-spin model vs scipy's adaptive integrator."""
    p = qi.cfg0(N=4, T=100.0 * 4 / 256)
    rng = np.random.default_rng(5)
    rho0 = rand_rho(rng, 8)
    got = oracle.evolve_rho(p.H0[0], p.Hc, p.C, p.u[0], p.T, p.N, 256, rho0)
    h = p.T / p.N
    rho = rho0.copy()
    for k in range(p.N):
        H = p.H0[0] + sum(p.u[0, k, j] * p.Hc[j] for j in range(2))
        f = lambda t, y, H=H: eq6_numpy(H, p.C, y.reshape(8, 8)).reshape(-1)  # noqa: E731
        sol = scipy.integrate.solve_ivp(f, (0.0, h), rho.reshape(-1), method="DOP853", rtol=1e-13, atol=1e-15)
        rho = sol.y[:, -1].reshape(8, 8)
    assert np.max(np.abs(got - rho)) <= 1e-13


# ---------------------------------------------------------------- calibration objective (NEXT f1)
def test_projection_matrix_is_orthonormal_and_literal():
    """S:101-103 adapted to the spin basis: P^dag P = I_2; column 0 = vec(|phi0><phi0|)."""
    for variant in ("standard-dfs", "as-printed"):
        P = qi.projection_matrix(variant)
        assert P.shape == (64, 2)
        assert np.allclose(P.conj().T @ P, np.eye(2), atol=1e-15)
    P = qi.projection_matrix()
    # |phi0> = (|uud> - |duu>)/sqrt2 -> indices 1 and 4; vec index i + 8 j
    assert abs(P[1 + 8 * 1, 0] - 0.5) < 1e-15 and abs(P[1 + 8 * 4, 0] + 0.5) < 1e-15
    phis = qi.logical_states()
    sz = np.diag(sum(qi.site_op(qi.SZ, i, 3) for i in range(3))).real
    for p in phis:                                    # both states in the S_z = +1/2 sector (A22)
        assert abs(np.vdot(p, sz * p).real - 1.0) < 1e-15


def test_logical_loss_identity_swap_and_cotangent(oracle):
    P = qi.projection_matrix()
    # Lambda = I -> Pi = I_2
    loss, _ = oracle.logical_loss(np.eye(64, dtype=np.complex128), P, np.eye(2, dtype=np.complex128))
    assert loss < 1e-30
    # logical swap: the unitary exchanging phi0 <-> phi1 and fixing their complement
    phis = qi.logical_states()
    W = np.eye(8, dtype=np.complex128) - np.outer(phis[0], phis[0].conj()) - np.outer(phis[1], phis[1].conj())
    W += np.outer(phis[0], phis[1].conj()) + np.outer(phis[1], phis[0].conj())
    Lsw = np.kron(W.conj(), W)
    loss, _ = oracle.logical_loss(Lsw, P, qi.LOGICAL_GATES["X"])
    assert loss < 1e-28
    # normalisation (A22: 1/4 ||Pi - G||_F^2, "mean" over the 4 entries of the 2x2 matrices): Lambda = I
    # gives Pi = P^dag P = I_2 exactly, so against G = X the residual is [[1, -1], [-1, 1]] with
    # ||.||_F^2 = 4 -> loss = 1; against G = 0, ||I_2||_F^2 = 2 -> loss = 1/2
    loss, _ = oracle.logical_loss(np.eye(64, dtype=np.complex128), P, qi.LOGICAL_GATES["X"])
    assert abs(loss - 1.0) <= 1e-14
    loss, _ = oracle.logical_loss(np.eye(64, dtype=np.complex128), P, np.zeros((2, 2), np.complex128))
    assert abs(loss - 0.5) <= 1e-14
    # cotangent: d loss along E equals Re Tr(C E) (central difference)
    rng = np.random.default_rng(3)
    Lam = rand_c(rng, 64, 64) / 8.0
    G = rand_c(rng, 2, 2)
    E = rand_c(rng, 64, 64)
    l0, C = oracle.logical_loss(Lam, P, G)
    eps = 1e-6
    lp, _ = oracle.logical_loss(Lam + eps * E, P, G)
    lm, _ = oracle.logical_loss(Lam - eps * E, P, G)
    fd = (lp - lm) / (2 * eps)
    assert abs(fd - np.trace(C @ E).real) <= 1e-8 * max(1.0, abs(fd))


def test_vjp_reduces_to_the_fidelity_gradient_and_matches_fd(oracle):
    p = qi.cfg0(N=6, T=100.0 * 6 / 256)
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    F, g, Lam = oracle.gradient(L0, Lc, p.u[0], p.T, p.N, p.V)
    SV = np.kron(p.V.conj(), p.V)
    gv, Lv = oracle.vjp(L0, Lc, p.u[0], p.T, p.N, SV.conj().T / 64.0)
    assert np.allclose(gv, g, rtol=0, atol=1e-16 + 1e-12 * np.abs(g).max())
    assert np.array_equal(Lv, Lam)
    rng = np.random.default_rng(8)
    C = rand_c(rng, 64, 64)
    gC, _ = oracle.vjp(L0, Lc, p.u[0], p.T, p.N, C)
    eps = 1e-6
    for k, j in [(0, 0), (3, 1), (5, 0)]:
        up, um = p.u[0].copy(), p.u[0].copy()
        up[k, j] += eps
        um[k, j] -= eps
        fp = np.trace(C @ oracle.propagate(L0, Lc, up, p.T, p.N)).real
        fm = np.trace(C @ oracle.propagate(L0, Lc, um, p.T, p.N)).real
        assert abs((fp - fm) / (2 * eps) - gC[k, j]) <= 1e-6 * np.abs(gC).max()


def test_adam_closed_forms(oracle):
    rng = np.random.default_rng(2)
    g = rng.standard_normal(7)
    th = np.zeros(7)
    m = np.zeros(7)
    v = np.zeros(7)
    oracle.adam_step(th, g, m, v, 1, lr=0.1, eps=0.0)
    assert np.allclose(th, -0.1 * np.sign(g), atol=1e-15)        # first step: lr * sign(g)
    for t in range(2, 6):                                          # constant gradient: every step lr sign(g)
        oracle.adam_step(th, g, m, v, t, lr=0.1, eps=0.0)
        assert np.allclose(th, -0.1 * t * np.sign(g), atol=1e-13)
