"""Seeded synthetic inputs for the Qalibrate hot path (arxiv 2511.13330).

This module is shared by the oracle side (tests, ``bench.py --impl reference``)
and the CUDA side (``bench.py``, ``smoke()``).  It holds NONE of the method's
arithmetic (no Liouvillian, no Magnus generator, no exponential, no product,
no fidelity): only

* a counter-based SplitMix64 generator (uniform and Box-Muller normal draws),
* the problem statement's operators -- the spin-model Hamiltonians H0, H_j and
  the collapse operators c_k (BASELINE.json configs[0], configs[4]; PAPER.md
  P:59 "eight-dimensional Hilbert space", P:85 jump operators from T1/T2),
* the seeded draws each config names (control tables, Zeeman offsets, the Haar
  target, the sinusoid parameters of configs[3]).

Readings:
  A6  collapse ops: sigma-_i / sqrt(T1) and sigma_z_i * sqrt(1/(2 T2)).
  A7  spin basis: index = sum_i s_i 2^(n-1-i), s = 0 for up (spin 1 most significant);
      sigma_z = diag(+1, -1) in (up, down); sigma- = [[0,0],[1,0]] (lowers up -> down).
  A9  Haar: Ginibre Z = (X + iY)/sqrt(2) row-major, QR, V = Q diag(R_ii/|R_ii|).
  A10 RNG: SplitMix64 streams keyed by (config seed, purpose tag, pulse index).
  A11 configs[3] controls: sum of 16 sinusoids, parameters drawn here; the
      function itself is evaluated by each side (oracle / CUDA kernel).
  A12 configs[2] Zeeman offsets delta b_i ~ N(0, (2 pi 0.002)^2) per pulse.
  A18 units: hbar = 1, t in ns, energies in rad/ns.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1

TWO_PI = 2.0 * math.pi
U_MAX = TWO_PI * 0.05            # rad/ns, BASELINE configs[0]: controls on [0, 2 pi 0.05]
T1_NS = 1.0e5                    # configs[0]
T2_NS = 1.0e4                    # configs[0]


# --------------------------------------------------------------------------
# SplitMix64 (counter form: output i of the stream seeded with s is mix(s + (i+1) gamma))
# --------------------------------------------------------------------------
def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix64(state: int, count: int, offset: int = 0) -> np.ndarray:
    """Outputs offset..offset+count-1 of the SplitMix64 stream with initial state ``state``."""
    i = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state & _MASK) + i * _GOLDEN
    return _mix64(z)


def _fnv1a(tag: str) -> int:
    h = 0xCBF29CE484222325
    for ch in tag.encode():
        h ^= ch
        h = (h * 0x100000001B3) & _MASK
    return h


def stream_state(seed: int, purpose: str, index: int = 0) -> int:
    """Per-(seed, purpose, index) stream state (A10)."""
    x = (seed * 0x9E3779B97F4A7C15) ^ _fnv1a(purpose) ^ ((index + 1) * 0xD1B54A32D192ED03)
    return int(_mix64(np.array([x & _MASK], dtype=np.uint64))[0])


def uniform(seed: int, purpose: str, index: int, count: int) -> np.ndarray:
    """count draws on [0, 1): (x >> 11) * 2^-53."""
    x = splitmix64(stream_state(seed, purpose, index), count)
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed: int, purpose: str, index: int, count: int) -> np.ndarray:
    """count N(0,1) draws, Box-Muller on consecutive uniform pairs (u1 in (0,1])."""
    m = (count + 1) // 2
    u = uniform(seed, purpose, index, 2 * m)
    u1 = 1.0 - u[0::2]
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * m)
    z[0::2] = r * np.cos(TWO_PI * u2)
    z[1::2] = r * np.sin(TWO_PI * u2)
    return z[:count]


# --------------------------------------------------------------------------
# Spin operators (A7) and the configs' physical model
# --------------------------------------------------------------------------
SX = np.array([[0, 1], [1, 0]], dtype=np.complex128)
SY = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
SZ = np.array([[1, 0], [0, -1]], dtype=np.complex128)
SMINUS = np.array([[0, 0], [1, 0]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)


def site_op(op: np.ndarray, i: int, nspin: int) -> np.ndarray:
    """op acting on spin i (0-based, spin 0 most significant) of nspin spins."""
    out = np.ones((1, 1), dtype=np.complex128)
    for s in range(nspin):
        out = np.kron(out, op if s == i else I2)
    return out


def exchange_op(i: int, j: int, nspin: int) -> np.ndarray:
    """(sigma_i . sigma_j) / 4."""
    return sum(site_op(P, i, nspin) @ site_op(P, j, nspin) for P in (SX, SY, SZ)) / 4.0


def zeeman_h0(b: np.ndarray) -> np.ndarray:
    """H0 = sum_i (b_i/2) sigma_z_i."""
    n = len(b)
    return sum((b[i] / 2.0) * site_op(SZ, i, n) for i in range(n))


def collapse_ops(nspin: int, t1: float = T1_NS, t2: float = T2_NS) -> np.ndarray:
    """[sigma-_i/sqrt(T1) for i] + [sigma_z_i sqrt(1/(2 T2)) for i]  (A6)."""
    ops = [site_op(SMINUS, i, nspin) / math.sqrt(t1) for i in range(nspin)]
    ops += [site_op(SZ, i, nspin) * math.sqrt(1.0 / (2.0 * t2)) for i in range(nspin)]
    return np.stack(ops)


def haar_unitary(dim: int, seed: int, purpose: str = "haar") -> np.ndarray:
    """Haar-random unitary (A9)."""
    g = normal(seed, purpose, 0, 2 * dim * dim)
    z = (g[0::2] + 1j * g[1::2]).reshape(dim, dim) / math.sqrt(2.0)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return np.ascontiguousarray(q * ph[None, :])


# --------------------------------------------------------------------------
# Problem instances
# --------------------------------------------------------------------------
CTRL_PWC = 0      # u[B][N][J]
CTRL_NODES = 1    # u[B][N][2][J]  (values at the two Gauss-Legendre nodes)


@dataclass
class Problem:
    """One instance of the propagator problem (all arrays C-contiguous)."""
    name: str
    d: int
    H0: np.ndarray            # [B or 1][d][d] complex128
    Hc: np.ndarray            # [J][d][d]
    C: np.ndarray             # [ncops][d][d]  (sqrt(rate) folded in)
    T: float
    N: int
    u: np.ndarray | None      # PWC: [B][N][J]; NODES: filled by the control sampler
    ctrl_mode: int
    V: np.ndarray             # [d][d] target unitary
    magnus_order: int = 4
    sines: np.ndarray | None = None   # [J][16][3] (a, f, phi) for configs[3]
    u_max: float = U_MAX
    extra: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return self.H0.shape[0] if self.u is None else self.u.shape[0]

    @property
    def J(self) -> int:
        return self.Hc.shape[0]

    @property
    def n(self) -> int:
        return self.d * self.d


def spin_chain(nspin: int, b: np.ndarray):
    H0 = zeeman_h0(np.asarray(b, dtype=np.float64))
    Hc = np.stack([exchange_op(i, i + 1, nspin) for i in range(nspin - 1)])
    return H0, Hc, collapse_ops(nspin)


B3 = TWO_PI * np.array([0.10, 0.12, 0.09])


def pwc_controls(seed: int, batch: int, N: int, J: int, first_pulse: int = 0) -> np.ndarray:
    u = np.empty((batch, N, J))
    for p in range(batch):
        u[p] = U_MAX * uniform(seed, "controls", first_pulse + p, N * J).reshape(N, J)
    return u


def cfg0(seed: int = 0, N: int = 256, T: float = 100.0) -> Problem:
    """BASELINE configs[0]: single pulse, d = 8, PWC controls on [0, u_max), Haar target."""
    H0, Hc, C = spin_chain(3, B3)
    return Problem("cfg0", 8, H0[None].copy(), Hc, C, T, N, pwc_controls(seed, 1, N, 2),
                   CTRL_PWC, haar_unitary(8, seed))


def cfg1(seed: int = 0) -> Problem:
    """BASELINE configs[1]: configs[0] plus the gradient (same inputs)."""
    p = cfg0(seed)
    p.name = "cfg1"
    p.extra["fd_eps"] = 1e-6
    return p


def cfg2(batch: int = 4096, N: int = 1024, T: float = 200.0, seed: int = 2,
         first_pulse: int = 0) -> Problem:
    """BASELINE configs[2]: robustness batch with quasistatic Zeeman offsets (A12)."""
    _, Hc, C = spin_chain(3, B3)
    H0 = np.empty((batch, 8, 8), dtype=np.complex128)
    db = np.empty((batch, 3))
    for p in range(batch):
        db[p] = (TWO_PI * 0.002) * normal(seed, "zeeman", first_pulse + p, 3)
        H0[p] = zeeman_h0(B3 + db[p])
    u = pwc_controls(seed, batch, N, 2, first_pulse)
    V = haar_unitary(8, seed)      # one shared target (A13)
    return Problem("cfg2", 8, H0, Hc, C, T, N, u, CTRL_PWC, V, extra={"delta_b": db})


def sine_params(seed: int, J: int, nterm: int = 16) -> np.ndarray:
    """(a, f, phi)[J][nterm]: a ~ U[0,1), f ~ U[0, 0.05) GHz, phi ~ U[0, 2 pi)  (A11)."""
    out = np.empty((J, nterm, 3))
    for j in range(J):
        r = uniform(seed, "sines", j, 3 * nterm).reshape(nterm, 3)
        out[j, :, 0] = r[:, 0]
        out[j, :, 1] = 0.05 * r[:, 1]
        out[j, :, 2] = TWO_PI * r[:, 2]
    return out


def cfg3(N: int = 1 << 20, T: float = 10_000.0, seed: int = 3) -> Problem:
    """BASELINE configs[3]: long horizon, smooth sinusoid-sum controls sampled at GL nodes."""
    H0, Hc, C = spin_chain(3, B3)
    return Problem("cfg3", 8, H0[None].copy(), Hc, C, T, N, None, CTRL_NODES,
                   haar_unitary(8, seed), sines=sine_params(seed, 2))


def cfg4(batch: int = 32, N: int = 512, T: float = 100.0, seed: int = 4) -> Problem:
    """BASELINE configs[4]: 6 spins, d = 64, 5 exchange controls, 12 collapse ops."""
    b6 = TWO_PI * (0.09 + 0.01 * np.arange(1, 7))
    H0, Hc, C = spin_chain(6, b6)
    return Problem("cfg4", 64, H0[None].copy(), Hc, C, T, N, pwc_controls(seed, batch, N, 5),
                   CTRL_PWC, haar_unitary(64, seed))


def single_spin(kind: str, T: float, N: int, b: float = 0.0, W: float = 0.0,
                t1: float = 1e30, t2: float = 1e30) -> Problem:
    """d = 2 closed-form cases (pins P-6): H0 = (b/2) sigma_z, one control (W/2) sigma_x held at 1."""
    H0 = (b / 2.0) * SZ
    Hc = ((1.0 / 2.0) * SX)[None]
    ops = []
    if t1 < 1e29:
        ops.append(SMINUS / math.sqrt(t1))
    if t2 < 1e29:
        ops.append(SZ * math.sqrt(1.0 / (2.0 * t2)))
    C = np.stack(ops) if ops else np.zeros((0, 2, 2), dtype=np.complex128)
    u = np.full((1, N, 1), W)
    return Problem(f"spin1-{kind}", 2, H0[None].copy(), Hc, C, T, N, u, CTRL_PWC, np.eye(2, dtype=np.complex128))


# --------------------------------------------------------------------------
# Logical encoding of the exchange-only qubit (Eqs. 2-3) and the projection of Eq. 16
# (P:145-151): P = [vec(rho_0) vec(rho_1)], rho_k = |phi_k><phi_k|, column stacking (A5).
# A22: Eq. 3 as printed, 2|uuu> - |uud> - |duu>, mixes S_z sectors (|uuu> has S_z = 3/2); the
# default is the standard decoherence-free-subspace state 2|udu> - |uud> - |duu> (S_z = 1/2,
# orthogonal to phi_0); variant="as-printed" reproduces the printed equation.
# --------------------------------------------------------------------------
def _ket(bits: str) -> np.ndarray:
    """|s1 s2 s3> with 'u' = up (0), 'd' = down (1); index = 4 s1 + 2 s2 + s3 (A7)."""
    v = np.zeros(8, dtype=np.complex128)
    v[int("".join("0" if c == "u" else "1" for c in bits), 2)] = 1.0
    return v


def logical_states(variant: str = "standard-dfs") -> np.ndarray:
    phi0 = (_ket("uud") - _ket("duu")) / math.sqrt(2.0)
    top = _ket("uuu") if variant == "as-printed" else _ket("udu")
    phi1 = (2.0 * top - _ket("uud") - _ket("duu")) / math.sqrt(6.0)
    return np.stack([phi0, phi1])


def projection_matrix(variant: str = "standard-dfs") -> np.ndarray:
    """[n][2] complex: columns vec(|phi_k><phi_k|) (column stacking)."""
    phis = logical_states(variant)
    return np.ascontiguousarray(np.stack([np.outer(p, p.conj()).reshape(-1, order="F") for p in phis], axis=1))


LOGICAL_GATES = {
    "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "I": np.eye(2, dtype=np.complex128),
}


# --------------------------------------------------------------------------
# NEXT f3: the paper's own model -- the Hubbard Hamiltonian of Eq. 1 on a chain of
# quantum dots, each with the 4-dim Fock space {|>, |u>, |d>, |ud>}.
# A23 (basis): index = base-4 number with digit map {empty 0, up 1, down 2, updown 3},
#     dot 1 most significant.  A24 (signs): Jordan-Wigner over fermionic modes ordered
#     (dot-major, up before down), so the operators anticommute exactly.
# A25 (unstated parameters; synthetic, rad/ns): U~ = 2pi 2.0, V_i = -2pi (0.30, 0.25, 0.30),
#     U_C = 2pi 0.5; controls are the hoppings t_{i,i+1} in [0, 2pi 0.5].  Jump operators of P:85
#     with the logical-subspace lowering a = phi_0 phi_1^dag: L1 = a/sqrt(T1), L2 = a^dag a/sqrt(T2).
# --------------------------------------------------------------------------
def fock_creation(dot: int, spin: int, n_dots: int) -> np.ndarray:
    """c^dag_{dot, spin} (spin 0 = up, 1 = down) as a 4^N x 4^N matrix (A23, A24)."""
    D = 4 ** n_dots
    mode = 2 * dot + spin
    out = np.zeros((D, D), dtype=np.complex128)
    for idx in range(D):
        digits = [(idx // 4 ** (n_dots - 1 - i)) % 4 for i in range(n_dots)]
        occ = []
        for dgt in digits:                      # digit -> (n_up, n_down)
            occ += [1 if dgt in (1, 3) else 0, 1 if dgt in (2, 3) else 0]
        if occ[mode]:
            continue
        sign = -1.0 if sum(occ[:mode]) % 2 else 1.0
        occ[mode] = 1
        new = 0
        for i in range(n_dots):
            nu, nd = occ[2 * i], occ[2 * i + 1]
            new = new * 4 + (0 if (nu, nd) == (0, 0) else 1 if (nu, nd) == (1, 0) else 2 if (nu, nd) == (0, 1) else 3)
        out[new, idx] = sign
    return out


def fock_number(dot: int, n_dots: int) -> np.ndarray:
    n = np.zeros((4 ** n_dots,) * 2, dtype=np.complex128)
    for s in (0, 1):
        c = fock_creation(dot, s, n_dots)
        n += c @ c.conj().T
    return n


def hubbard_terms(n_dots: int, U: float, V, UC: float):
    """(H0, [H_j]): H0 = sum_i [U/2 n_i(n_i - 1) + V_i n_i] + sum_<ij> U_C n_i n_j and the hopping
    terms H_j = sum_sigma (c^dag_{j sigma} c_{j+1 sigma} + h.c.) whose coefficients t_{j,j+1} are the controls."""
    D = 4 ** n_dots
    I = np.eye(D, dtype=np.complex128)
    ns = [fock_number(i, n_dots) for i in range(n_dots)]
    H0 = sum(0.5 * U * n @ (n - I) + V[i] * n for i, n in enumerate(ns))
    H0 = H0 + sum(UC * ns[i] @ ns[i + 1] for i in range(n_dots - 1))
    Hc = []
    for j in range(n_dots - 1):
        h = np.zeros((D, D), dtype=np.complex128)
        for s in (0, 1):
            cd_j, cd_k = fock_creation(j, s, n_dots), fock_creation(j + 1, s, n_dots)
            h += cd_j @ cd_k.conj().T
        Hc.append(h + h.conj().T)
    return H0, (np.stack(Hc) if Hc else np.zeros((0, D, D), dtype=np.complex128))


def hubbard_logical_states() -> np.ndarray:
    """Eqs. 2-3 in the 3-dot Fock space (one electron per dot): phi_0 = (|u u d> - |d u u>)/sqrt2,
    phi_1 (A22 standard DFS) = (2|u d u> - |u u d> - |d u u>)/sqrt6; base-4 indices per A23."""
    def ket(s):
        v = np.zeros(64, dtype=np.complex128)
        v[sum((1 if c == "u" else 2) * 4 ** (2 - i) for i, c in enumerate(s))] = 1.0
        return v
    phi0 = (ket("uud") - ket("duu")) / math.sqrt(2.0)
    phi1 = (2.0 * ket("udu") - ket("uud") - ket("duu")) / math.sqrt(6.0)
    return np.stack([phi0, phi1])


def hubbard3(seed: int = 7, N: int = 512, T: float = 100.0, batch: int = 1) -> Problem:
    """NEXT f3: the paper's 3-dot Hubbard workload (D = 64, 4096 x 4096 superoperators, Fig. 1 /
    P:147); T and M are unstated in the paper (A25), chosen like configs[4]."""
    H0, Hc = hubbard_terms(3, TWO_PI * 2.0, -TWO_PI * np.array([0.30, 0.25, 0.30]), TWO_PI * 0.5)
    phi0, phi1 = hubbard_logical_states()
    a = np.outer(phi0, phi1.conj())
    C = np.stack([a / math.sqrt(T1_NS), (a.conj().T @ a) / math.sqrt(T2_NS)])
    u = np.empty((batch, N, 2))
    for p in range(batch):
        u[p] = TWO_PI * 0.5 * uniform(seed, "hubbard", p, 2 * N).reshape(N, 2)
    return Problem("hubbard3", 64, H0[None].copy(), Hc, C, T, N, u, CTRL_PWC, haar_unitary(64, seed))


CONFIGS = {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "hubbard3": hubbard3}
