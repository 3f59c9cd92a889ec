"""ctypes wrapper of the CPU oracle ``oracle/libqalref.so`` (built from qalref.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs are the only callers.  Nothing under
paper_2511_13330_b200/ imports this package.  See qalref.c for the citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libqalref.so")
_SRC = os.path.join(_HERE, "qalref.c")

CFLAGS = ["-O2", "-fcx-limited-range", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-D_GNU_SOURCE"]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc).  Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        _lib.qalref_fidelity.restype = ctypes.c_double
    return _lib


def set_threads(n: int):
    """OpenMP threads of the oracle's parallel loops (libgomp, linked into libqalref.so)."""
    lib().omp_set_num_threads(int(n))


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.c_void_p)


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"oracle error {rc}")


def build_liouvillian(H0, Hc, C):
    """Eq. 8.  Returns (L0 [n][n], Lc [J][n][n])."""
    H0, pH0 = _c(H0, np.complex128)
    d = H0.shape[-1]
    Hc, pHc = _c(np.asarray(Hc).reshape(-1, d, d), np.complex128)
    C, pC = _c(np.asarray(C).reshape(-1, d, d), np.complex128)
    n = d * d
    L0 = np.zeros((n, n), np.complex128)
    Lc = np.zeros((Hc.shape[0], n, n), np.complex128)
    _chk(lib().qalref_build_liouvillian(d, pH0, Hc.shape[0], pHc, C.shape[0], pC,
                                        L0.ctypes.data_as(ctypes.c_void_p),
                                        Lc.ctypes.data_as(ctypes.c_void_p)))
    return L0, Lc


def lindblad_rhs(H, C, rho):
    """Eq. 6 directly."""
    H, pH = _c(H, np.complex128)
    d = H.shape[0]
    C, pC = _c(np.asarray(C).reshape(-1, d, d), np.complex128)
    rho, pr = _c(rho, np.complex128)
    out = np.zeros((d, d), np.complex128)
    _chk(lib().qalref_lindblad_rhs(d, pH, C.shape[0], pC, pr, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def expm(A):
    A, pA = _c(A, np.complex128)
    E = np.zeros_like(A)
    _chk(lib().qalref_expm(A.shape[0], pA, E.ctypes.data_as(ctypes.c_void_p)))
    return E


def frechet(A, E):
    """(L(A, E), e^A) via the 2n x 2n augmented exponential."""
    A, pA = _c(A, np.complex128)
    E, pE = _c(E, np.complex128)
    L = np.zeros_like(A)
    X = np.zeros_like(A)
    _chk(lib().qalref_frechet(A.shape[0], pA, pE, L.ctypes.data_as(ctypes.c_void_p),
                              X.ctypes.data_as(ctypes.c_void_p)))
    return L, X


def magnus_generator(L0, Lc, h, u1, u2, order=4):
    L0, p0 = _c(L0, np.complex128)
    Lc, pc = _c(Lc, np.complex128)
    u1, p1 = _c(u1, np.float64)
    u2, p2 = _c(u2, np.float64)
    Om = np.zeros_like(L0)
    _chk(lib().qalref_magnus_generator(L0.shape[0], order, ctypes.c_double(h), Lc.shape[0], p0, pc,
                                       p1, p2, Om.ctypes.data_as(ctypes.c_void_p)))
    return Om


def propagate(L0, Lc, u, T, N, mode=0, order=4, k0=0, k1=None, store=False):
    """Lambda = U_{k1-1} ... U_{k0} (Eq. 15), sequential left fold.  u is one pulse."""
    L0, p0 = _c(L0, np.complex128)
    Lc, pc = _c(Lc, np.complex128)
    u, pu = _c(u, np.float64)
    n = L0.shape[0]
    k1 = N if k1 is None else k1
    Lam = np.zeros((n, n), np.complex128)
    Us = np.zeros((k1 - k0, n, n), np.complex128) if store else None
    _chk(lib().qalref_propagate(n, N, ctypes.c_double(T), order, mode, Lc.shape[0], pu, p0, pc, k0, k1,
                                Lam.ctypes.data_as(ctypes.c_void_p),
                                Us.ctypes.data_as(ctypes.c_void_p) if store else None))
    return (Lam, Us) if store else Lam


def fidelity(Lam, V):
    Lam, pl = _c(Lam, np.complex128)
    V, pv = _c(V, np.complex128)
    return lib().qalref_fidelity(V.shape[0], pl, pv)


def gradient(L0, Lc, u, T, N, V, mode=0, order=4):
    """(F, grad with the layout of u, Lambda) -- O7, per-direction augmented exponential."""
    L0, p0 = _c(L0, np.complex128)
    Lc, pc = _c(Lc, np.complex128)
    u, pu = _c(u, np.float64)
    V, pv = _c(V, np.complex128)
    d = V.shape[0]
    n = d * d
    F = ctypes.c_double(0.0)
    g = np.zeros(u.shape, np.float64)
    Lam = np.zeros((n, n), np.complex128)
    _chk(lib().qalref_gradient(d, N, ctypes.c_double(T), order, mode, Lc.shape[0], pu, p0, pc, pv,
                               ctypes.byref(F), g.ctypes.data_as(ctypes.c_void_p),
                               Lam.ctypes.data_as(ctypes.c_void_p)))
    return F.value, g, Lam


def vjp(L0, Lc, u, T, N, C, mode=0, order=4):
    """dL/du for dL = Re Tr(C dLambda) (per-direction augmented exponentials); returns (grad, Lambda)."""
    L0, p0 = _c(L0, np.complex128)
    Lc, pc = _c(Lc, np.complex128)
    u, pu = _c(u, np.float64)
    C, pC = _c(C, np.complex128)
    n = L0.shape[0]
    g = np.zeros(u.shape, np.float64)
    Lam = np.zeros((n, n), np.complex128)
    _chk(lib().qalref_vjp(n, N, ctypes.c_double(T), order, mode, Lc.shape[0], pu, p0, pc, pC,
                          g.ctypes.data_as(ctypes.c_void_p), Lam.ctypes.data_as(ctypes.c_void_p)))
    return g, Lam


def fidelity_cotangent(V):
    V, pv = _c(V, np.complex128)
    d = V.shape[0]
    C = np.zeros((d * d, d * d), np.complex128)
    lib().qalref_fidelity_cotangent(d, pv, C.ctypes.data_as(ctypes.c_void_p))
    return C


def logical_loss(Lam, P, G):
    """Eqs. 16-17: (loss, cotangent C)."""
    Lam, pl = _c(Lam, np.complex128)
    P, pp = _c(P, np.complex128)
    G, pg = _c(G, np.complex128)
    n = Lam.shape[0]
    loss = ctypes.c_double(0.0)
    C = np.zeros((n, n), np.complex128)
    _chk(lib().qalref_logical_loss(n, pl, pp, pg, ctypes.byref(loss), C.ctypes.data_as(ctypes.c_void_p)))
    return loss.value, C


def adam_step(theta, g, m, v, t, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8):
    """in place on theta, m, v (float64 contiguous arrays)."""
    for a in (theta, g, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    lib().qalref_adam_step(theta.size, theta.ctypes.data_as(ctypes.c_void_p), g.ctypes.data_as(ctypes.c_void_p),
                           m.ctypes.data_as(ctypes.c_void_p), v.ctypes.data_as(ctypes.c_void_p), t,
                           ctypes.c_double(lr), ctypes.c_double(b1), ctypes.c_double(b2), ctypes.c_double(eps))


def sines_eval(prm, umax, t):
    prm, pp = _c(prm, np.float64)
    J, nterm = prm.shape[0], prm.shape[1]
    out = np.zeros(J)
    lib().qalref_sines_eval(J, nterm, pp, ctypes.c_double(umax), ctypes.c_double(t),
                            out.ctypes.data_as(ctypes.c_void_p))
    return out


def sines_nodes(prm, umax, N, T, k0=0, k1=None):
    """u[k][a][j] at the Gauss-Legendre nodes of slices k0..k1-1."""
    prm, pp = _c(prm, np.float64)
    J, nterm = prm.shape[0], prm.shape[1]
    k1 = N if k1 is None else k1
    out = np.zeros((k1 - k0, 2, J))
    lib().qalref_sines_nodes(J, nterm, pp, ctypes.c_double(umax), N, ctypes.c_double(T), k0, k1,
                             out.ctypes.data_as(ctypes.c_void_p))
    return out


def rk4(L0, Lc, T, N, sub, u=None, prm=None, umax=0.0):
    """Fixed-step RK4 of dLambda/dt = L(t) Lambda (O8); PWC table u[N][J] or sinusoid prm."""
    L0, p0 = _c(L0, np.complex128)
    Lc, pc = _c(Lc, np.complex128)
    n = L0.shape[0]
    J = Lc.shape[0]
    if u is not None:
        u, pu = _c(u, np.float64)
        cmode, pp, nterm = 0, None, 0
    else:
        prm, pp = _c(prm, np.float64)
        cmode, pu, nterm = 2, None, prm.shape[1]
    Lam = np.zeros((n, n), np.complex128)
    _chk(lib().qalref_rk4(n, N, ctypes.c_double(T), sub, cmode, J, pu, pp, nterm, ctypes.c_double(umax),
                          p0, pc, Lam.ctypes.data_as(ctypes.c_void_p)))
    return Lam


def matmul(A, B):
    A, pa = _c(A, np.complex128)
    B, pb = _c(B, np.complex128)
    C = np.zeros_like(A)
    lib().qalref_matmul(A.shape[0], pa, pb, C.ctypes.data_as(ctypes.c_void_p))
    return C


def matmul_rows(A, B, r0, r1):
    """rows r0..r1-1 of A B (plain sums)."""
    A, pa = _c(A, np.complex128)
    B, pb = _c(B, np.complex128)
    n = A.shape[0]
    C = np.zeros((r1 - r0, n), np.complex128)
    lib().qalref_matmul_rows(n, pa, pb, r0, r1, C.ctypes.data_as(ctypes.c_void_p))
    return C


def evolve_rho(H0, Hc, C, u, T, N, sub, rho0):
    """RK4 of Eq. 6 on the density matrix with PWC controls u[N][J] (no superoperator)."""
    H0, p0 = _c(H0, np.complex128)
    d = H0.shape[-1]
    Hc, pc = _c(np.asarray(Hc).reshape(-1, d, d), np.complex128)
    C, pC = _c(np.asarray(C).reshape(-1, d, d), np.complex128)
    u, pu = _c(u, np.float64)
    rho0, pr = _c(rho0, np.complex128)
    rho = np.zeros_like(rho0)
    _chk(lib().qalref_evolve_rho(d, p0, Hc.shape[0], pc, C.shape[0], pC, N, ctypes.c_double(T), sub, pu, pr,
                                 rho.ctypes.data_as(ctypes.c_void_p)))
    return rho


def ordered_product(Us):
    """U[count-1] ... U[0] by a sequential left fold (Eq. 15)."""
    P = np.eye(Us.shape[-1], dtype=np.complex128)
    for U in Us:
        P = matmul(U, P)
    return P
