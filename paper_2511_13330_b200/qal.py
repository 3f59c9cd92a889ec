"""Thin ctypes binding of libqal.so (include/qal.h), same names as the C ABI.

Argument marshalling only: torch tensors (device memory) are passed as raw
pointers together with the current CUDA stream; every step of the hot path runs
in the library's sm_100a kernels.  There is no CPU fallback: if the library or a
GPU is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QAL_LIB") or os.path.join(_HERE, "libqal.so")   # QAL_LIB: experiment builds only

QAL_OK = 0
QAL_CTRL_PWC = 0
QAL_CTRL_NODES = 1
QAL_OP_ORDERED_PRODUCT = 1
QAL_OP_FIDELITY = 2
QAL_OP_FIDELITY_GRAD = 3
QAL_OP_EXPM_SLICES = 4
QAL_OP_VJP = 5
QAL_OP_FIDELITY_REDUCE = 6
QAL_BLK_SETS_DEFAULT, QAL_BLK_SETS_FUSED, QAL_BLK_SETS_PAIRS = 0, 1, 2
QAL_MAX_CTRL = 8
STAGES = ["liouvillian", "commutators", "expm_fold", "tree", "fidelity", "prefix_chain", "suffix_chain",
          "grad_slices", "dense_gemm", "blk_expm_fold", "blk_tree", "blk_prefix_chain", "blk_suffix_chain",
          "blk_grad_slices", "blk_gemm", "blk_fold"]
# stages whose device counter holds algorithmic FLOPs (coherence-block path), not product counts
FLOP_STAGES = {"blk_expm_fold", "blk_tree", "blk_prefix_chain", "blk_suffix_chain", "blk_grad_slices", "blk_gemm", "blk_fold"}
KERNELS = {"liouvillian": "k_liouvillian", "commutators": "k_commutators", "expm_fold": "k_expm_fold",
           "tree": "k_tree_level", "fidelity": "k_fidelity", "prefix_chain": "k_prefix_chain",
           "suffix_chain": "k_suffix_chain", "grad_slices": "k_grad_slices", "dense_gemm": "k_dense_gemm",
           "blk_expm_fold": "k_blk_expm_fold", "blk_tree": "k_blk_tree_level", "blk_prefix_chain": "k_blk_prefix_chain",
           "blk_suffix_chain": "k_blk_suffix_chain", "blk_grad_slices": "k_blk_grad_slices", "blk_gemm": "k_bb_gemm",
           "blk_fold": "k_blk_expm_fold"}

_EXPORTS = {
    "qal_abi_version": (ctypes.c_int, []),
    "qal_real_mults_per_complex_product": (ctypes.c_int, []),
    "qal_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "qal_last_cuda_error": (ctypes.c_char_p, []),
    "qal_last_launch_count": (ctypes.c_int, []),
    "qal_default_chunk": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "qal_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int] * 6),
    "qal_build_liouvillian": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "qal_magnus_expm_slices": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                                               ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_ordered_product": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_fidelity": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p]),
    "qal_fidelity_ws": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_fidelity_grad": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_sample_controls_sines": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_double,
                                                  ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_void_p, ctypes.c_void_p]),
    "qal_propagator_forward": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_propagator_vjp": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_ordered_scan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_batched_matmul": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong,
                                           ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]),
    "qal_fidelity_cotangent": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "qal_logical_loss": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "qal_adam_step": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_void_p]),
    "qal_block_plan_build": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_void_p]),
    "qal_block_pack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "qal_block_unpack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]),
    "qal_block_check": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "qal_block_expm_slices": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p]),
    "qal_block_ordered_product": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                                  ctypes.c_void_p]),
    "qal_block_fidelity": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]),
    "qal_block_fidelity_grad": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                                ctypes.c_void_p]),
    "qal_block_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "qal_block_propagator_forward": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_block_propagator_backward": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                      ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                                      ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                                      ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                                      ctypes.c_void_p]),
    "qal_block_propagator_vjp": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                                 ctypes.c_void_p]),
    "qal_block_ordered_scan": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.c_void_p]),
    "qal_block_batched_matmul": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong,
                                                 ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]),
    "qal_block_fidelity_cotangent": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_void_p]),
    "qal_bigblock_plan_workspace_bytes": (ctypes.c_size_t, []),
    "qal_bigblock_plan_build": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_bigblock_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p]),
    "qal_bigblock_expm_slices": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                                 ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "qal_profile_begin": (ctypes.c_int, [ctypes.c_void_p]),
    "qal_profile_end": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]),
    "qal_fp64_peak_probe": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_double), ctypes.c_void_p, ctypes.c_void_p]),
}

_lib = None


class QalError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load libqal.so and declare every exported symbol (fails loudly if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise QalError(f"libqal.so not built ({path}); run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int, what: str):
    if rc != QAL_OK:
        msg = f"{what}: {load().qal_status_string(rc).decode()} ({rc})"
        if rc == -7:
            msg += f": {load().qal_last_cuda_error().decode()}"
        raise QalError(msg)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t, dtype, name):
    if t is None:
        return None
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise QalError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise QalError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise QalError(f"{name} must be contiguous")
    return t


def abi_version() -> int:
    return load().qal_abi_version()


def real_mults_per_complex_product() -> int:
    """4 (default build), 3 for a -DQAL_USE_3M build (Gauss complex product)."""
    return load().qal_real_mults_per_complex_product()


def last_launch_count() -> int:
    return load().qal_last_launch_count()


def default_chunk(batch: int, n_slices: int) -> int:
    return load().qal_default_chunk(batch, n_slices)


def workspace_bytes(op: int, n: int, batch: int, n_slices: int, n_ctrl: int = 0, flags: int = 0) -> int:
    return load().qal_workspace_bytes(op, n, batch, n_slices, n_ctrl, flags)


def n_comm(J: int) -> int:
    return J + J * (J - 1) // 2


def qal_build_liouvillian(H0, Hc, C, want_comm=False, stream=None):
    """Eq. 8: returns (L0 [B][n][n], Lc [J][n][n], Lcomm [B][ncomm][n][n] or None)."""
    c128 = torch.complex128
    H0 = _dev(H0, c128, "H0")
    Hc = _dev(Hc, c128, "Hc")
    C = _dev(C, c128, "C") if C is not None and C.shape[0] > 0 else None
    d = H0.shape[-1]
    B = H0.shape[0]
    J = Hc.shape[0]
    n = d * d
    dev = H0.device
    L0 = torch.empty((B, n, n), dtype=c128, device=dev)
    Lc = torch.empty((J, n, n), dtype=c128, device=dev)
    Lcomm = torch.empty((B, n_comm(J), n, n), dtype=c128, device=dev) if want_comm else None
    rc = load().qal_build_liouvillian(d, B, _ptr(H0), J, _ptr(Hc), 0 if C is None else C.shape[0], _ptr(C),
                                      int(bool(want_comm)), _ptr(L0), _ptr(Lc), _ptr(Lcomm), _stream(stream))
    _check(rc, "qal_build_liouvillian")
    return L0, Lc, Lcomm


def qal_magnus_expm_slices(L0, Lc, u, T, n_slices, *, k0=0, count=None, magnus_order=4,
                           ctrl_mode=QAL_CTRL_PWC, Lcomm=None, want_U=False, chunk=None, status=None,
                           stream=None):
    """Eqs. 13-15: per-slice U_k and/or chunk products.  Returns (U or None, chunk_prod or None)."""
    c128 = torch.complex128
    L0 = _dev(L0, c128, "L0")
    Lc = _dev(Lc, c128, "Lc")
    u = _dev(u, torch.float64, "u")
    B = u.shape[0]
    J = Lc.shape[0]
    n = L0.shape[-1]
    count = n_slices - k0 if count is None else count
    dev = u.device
    U = torch.empty((B, count, n, n), dtype=c128, device=dev) if want_U else None
    P = None
    if chunk is not None:
        P = torch.empty((B, count // chunk, n, n), dtype=c128, device=dev)
    L0s = 0 if L0.shape[0] == 1 else n * n
    Lcs = 0
    if Lcomm is not None:
        Lcomm = _dev(Lcomm, c128, "Lcomm")
        Lcs = 0 if Lcomm.shape[0] == 1 else n_comm(J) * n * n
    wsb = workspace_bytes(QAL_OP_EXPM_SLICES, n, B, count)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
    rc = load().qal_magnus_expm_slices(n, B, n_slices, float(T), k0, count, magnus_order, ctrl_mode, J, _ptr(u),
                                       _ptr(L0), L0s, _ptr(Lc), _ptr(Lcomm), Lcs, _ptr(U),
                                       1 if chunk is None else chunk, _ptr(P), _ptr(status), _ptr(ws), wsb,
                                       _stream(stream))
    _check(rc, "qal_magnus_expm_slices")
    return U, P


def qal_ordered_product(U, stream=None):
    """Eq. 15 / P:141 balanced tree: U [B][count][n][n] -> U[count-1] ... U[0]."""
    U = _dev(U, torch.complex128, "U")
    B, count, n = U.shape[0], U.shape[1], U.shape[2]
    out = torch.empty((B, n, n), dtype=U.dtype, device=U.device)
    wsb = workspace_bytes(QAL_OP_ORDERED_PRODUCT, n, B, count)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=U.device)
    rc = load().qal_ordered_product(n, B, count, _ptr(U), _ptr(out), _ptr(ws), wsb, _stream(stream))
    _check(rc, "qal_ordered_product")
    return out


def qal_ordered_scan(U, want_prefix=True, want_suffix=True, stream=None):
    """Exclusive prefix / suffix products of U [B][count][n][n] (later on the LEFT)."""
    U = _dev(U, torch.complex128, "U")
    B, cnt, n = U.shape[0], U.shape[1], U.shape[2]
    pre = torch.empty_like(U) if want_prefix else None
    suf = torch.empty_like(U) if want_suffix else None
    ws = torch.empty(4 * B * cnt * n * n * 16, dtype=torch.uint8, device=U.device)
    rc = load().qal_ordered_scan(n, B, cnt, _ptr(U), _ptr(pre), _ptr(suf), _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "qal_ordered_scan")
    return pre, suf


def qal_batched_matmul(A, B, stream=None):
    """A [count|1][n][n] @ B [count|1][n][n] -> [count][n][n] (broadcast a leading 1)."""
    A = _dev(A, torch.complex128, "A")
    B = _dev(B, torch.complex128, "B")
    cnt = max(A.shape[0], B.shape[0])
    n = A.shape[-1]
    out = torch.empty((cnt, n, n), dtype=torch.complex128, device=A.device)
    rc = load().qal_batched_matmul(n, cnt, _ptr(A), 0 if A.shape[0] == 1 else n * n, _ptr(B),
                                   0 if B.shape[0] == 1 else n * n, _ptr(out), _stream(stream))
    _check(rc, "qal_batched_matmul")
    return out


def qal_fidelity(Lam, V, ws=None, stream=None):
    """A8: F[b] = Re Tr(S_V^dag Lambda_b) / d^2.  With `ws` (a device byte tensor of at least
    qal_workspace_bytes(QAL_OP_FIDELITY_REDUCE, n, B)) the d = 64 reduction runs over 512 row slabs
    per pulse (qal_fidelity_ws); without it one CTA per pulse (qal_fidelity)."""
    Lam = _dev(Lam, torch.complex128, "Lambda")
    V = _dev(V, torch.complex128, "V")
    F = torch.empty(Lam.shape[0], dtype=torch.float64, device=Lam.device)
    if ws is None:
        rc = load().qal_fidelity(V.shape[0], Lam.shape[0], _ptr(Lam), _ptr(V), _ptr(F), _stream(stream))
    else:
        rc = load().qal_fidelity_ws(V.shape[0], Lam.shape[0], _ptr(Lam), _ptr(V), _ptr(F), _ptr(ws), ws.numel(),
                                    _stream(stream))
    _check(rc, "qal_fidelity")
    return F


def qal_fidelity_grad(L0, Lc, u, T, n_slices, V, *, magnus_order=4, ctrl_mode=QAL_CTRL_PWC, Lcomm=None,
                      want_grad=True, want_Lambda=False, status=None, ws=None, stream=None):
    """The whole hot path: returns (F [B], grad (layout of u) or None, Lambda or None)."""
    c128 = torch.complex128
    L0 = _dev(L0, c128, "L0")
    Lc = _dev(Lc, c128, "Lc")
    u = _dev(u, torch.float64, "u")
    V = _dev(V, c128, "V")
    B = u.shape[0]
    J = Lc.shape[0]
    n = L0.shape[-1]
    d = V.shape[0]
    dev = u.device
    F = torch.empty(B, dtype=torch.float64, device=dev)
    g = torch.empty_like(u) if want_grad else None
    Lam = torch.empty((B, n, n), dtype=c128, device=dev) if want_Lambda else None
    op = QAL_OP_FIDELITY_GRAD if want_grad else QAL_OP_FIDELITY
    wsb = workspace_bytes(op, n, B, n_slices, J, ctrl_mode)
    if ws is None or ws.numel() < wsb:
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    L0s = 0 if L0.shape[0] == 1 else n * n
    Lcs = 0
    if Lcomm is not None:
        Lcomm = _dev(Lcomm, c128, "Lcomm")
        Lcs = 0 if Lcomm.shape[0] == 1 else n_comm(J) * n * n
    rc = load().qal_fidelity_grad(d, B, n_slices, float(T), magnus_order, ctrl_mode, J, _ptr(u), _ptr(L0), L0s,
                                  _ptr(Lc), _ptr(Lcomm), Lcs, _ptr(V), _ptr(F), _ptr(g), _ptr(Lam),
                                  _ptr(status), _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "qal_fidelity_grad")
    return F, g, Lam


class GradientSession:
    """qal_propagator_forward / qal_propagator_vjp pair sharing one workspace (same slice range)."""

    def __init__(self, L0, Lc, u, T, n_slices, *, k0=0, magnus_order=4, ctrl_mode=QAL_CTRL_PWC, Lcomm=None,
                 stream=None):
        self.L0 = _dev(L0, torch.complex128, "L0")
        self.Lc = _dev(Lc, torch.complex128, "Lc")
        self.u = _dev(u, torch.float64, "u")
        self.Lcomm = _dev(Lcomm, torch.complex128, "Lcomm") if Lcomm is not None else None
        self.T, self.N, self.k0 = float(T), n_slices, k0
        self.B, self.count = u.shape[0], u.shape[1]
        self.J, self.n = Lc.shape[0], L0.shape[-1]
        self.order, self.mode, self.stream = magnus_order, ctrl_mode, stream
        self.L0s = 0 if self.L0.shape[0] == 1 else self.n * self.n
        self.Lcs = 0 if self.Lcomm is None or self.Lcomm.shape[0] == 1 else n_comm(self.J) * self.n * self.n
        wsb = workspace_bytes(QAL_OP_VJP, self.n, self.B, self.count, self.J, ctrl_mode)
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=u.device)
        self.status = torch.zeros(self.B, dtype=torch.int32, device=u.device)

    def _args(self):
        return (int(round(self.n ** 0.5)), self.B, self.N, self.T, self.k0, self.count, self.order, self.mode, self.J,
                _ptr(self.u), _ptr(self.L0), self.L0s, _ptr(self.Lc), _ptr(self.Lcomm), self.Lcs)

    def forward(self, P_init=None):
        Lam = torch.empty((self.B, self.n, self.n), dtype=torch.complex128, device=self.u.device)
        if P_init is not None:
            P_init = _dev(P_init, torch.complex128, "P_init")
        rc = load().qal_propagator_forward(*self._args(), _ptr(P_init), _ptr(Lam), _ptr(self.status), _ptr(self.ws),
                                           self.ws.numel(), _stream(self.stream))
        _check(rc, "qal_propagator_forward")
        return Lam

    def vjp(self, C):
        C = _dev(C, torch.complex128, "C")
        g = torch.empty_like(self.u)
        rc = load().qal_propagator_vjp(*self._args(), _ptr(C), _ptr(g), _ptr(self.status), _ptr(self.ws),
                                       self.ws.numel(), _stream(self.stream))
        _check(rc, "qal_propagator_vjp")
        return g


def qal_fidelity_cotangent(V, stream=None):
    """C = S_V^dag / d^2 [n][n] (dF = Re Tr(C dLambda))."""
    V = _dev(V, torch.complex128, "V")
    d = V.shape[0]
    C = torch.empty((d * d, d * d), dtype=torch.complex128, device=V.device)
    _check(load().qal_fidelity_cotangent(d, _ptr(V), _ptr(C), _stream(stream)), "qal_fidelity_cotangent")
    return C


def qal_logical_loss(Lam, Pproj, G, want_cotangent=True, stream=None):
    """Eqs. 16-17: (loss [B], cotangent C [B][n][n] or None)."""
    Lam = _dev(Lam, torch.complex128, "Lambda")
    Pproj = _dev(Pproj, torch.complex128, "P")
    G = _dev(G, torch.complex128, "G")
    loss = torch.empty(Lam.shape[0], dtype=torch.float64, device=Lam.device)
    C = torch.empty_like(Lam) if want_cotangent else None
    rc = load().qal_logical_loss(8, Lam.shape[0], _ptr(Lam), _ptr(Pproj), _ptr(G), _ptr(loss), _ptr(C),
                                 _stream(stream))
    _check(rc, "qal_logical_loss")
    return loss, C


def qal_adam_step(theta, grad, m, v, t, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
    """Adam on device tensors (in place on theta, m, v)."""
    for name, x in (("theta", theta), ("grad", grad), ("m", m), ("v", v)):
        _dev(x, torch.float64, name)
    rc = load().qal_adam_step(theta.numel(), _ptr(theta), _ptr(grad), _ptr(m), _ptr(v), t, lr, beta1, beta2, eps,
                              _stream(stream))
    _check(rc, "qal_adam_step")


def qal_sample_controls_sines(prm, u_max, n_slices, T, k0=0, count=None, stream=None):
    """a1 (NODES, A11): controls at the GL nodes of slices k0..k0+count-1 -> [count][2][J] f64."""
    prm = _dev(prm, torch.float64, "prm")
    J, nterm = prm.shape[0], prm.shape[1]
    count = n_slices - k0 if count is None else count
    out = torch.empty((count, 2, J), dtype=torch.float64, device=prm.device)
    rc = load().qal_sample_controls_sines(J, nterm, _ptr(prm), float(u_max), n_slices, float(T), k0, count,
                                          _ptr(out), _stream(stream))
    _check(rc, "qal_sample_controls_sines")
    return out


def qal_profile_begin(dev_counters=None):
    """Open a stage-profiling window (events around every library kernel)."""
    _check(load().qal_profile_begin(_ptr(dev_counters)), "qal_profile_begin")


def qal_profile_end():
    """Close the window: {stage: (device ms summed, launches)} (synchronises the events)."""
    n = len(STAGES)
    ms = (ctypes.c_double * n)()
    la = (ctypes.c_int * n)()
    _check(load().qal_profile_end(ms, la), "qal_profile_end")
    return {STAGES[i]: (ms[i], la[i]) for i in range(n)}


def qal_fp64_peak_probe(kind: int, blocks: int, iters: int, sink, stream=None) -> float:
    """Launch the FP64 probe (K0); returns the flop count of the launch."""
    fl = ctypes.c_double(0.0)
    rc = load().qal_fp64_peak_probe(kind, blocks, iters, ctypes.byref(fl), _ptr(sink), _stream(stream))
    _check(rc, "qal_fp64_peak_probe")
    return fl.value


# --------------------------------------------------------------------------- coherence-block path
QAL_BLK_MAX_GROUPS = 16
QAL_BLK_MAX_ROWS = 96
QAL_ERR_STRUCTURE = -8
QAL_ERR_NONFINITE = -4


class BlockPlan(ctypes.Structure):
    """Mirror of qal_block_plan (include/qal.h)."""
    _fields_ = [("n", ctypes.c_int), ("d", ctypes.c_int), ("mirror", ctypes.c_int), ("ngroups", ctypes.c_int),
                ("nrows", ctypes.c_int), ("packed", ctypes.c_int), ("n_components", ctypes.c_int),
                ("width", ctypes.c_int * QAL_BLK_MAX_GROUPS), ("used", ctypes.c_int * QAL_BLK_MAX_GROUPS),
                ("row0", ctypes.c_int * QAL_BLK_MAX_GROUPS),
                ("off", ctypes.c_int * QAL_BLK_MAX_GROUPS), ("flops", ctypes.c_double * QAL_BLK_MAX_GROUPS),
                ("perm", ctypes.c_int * QAL_BLK_MAX_ROWS), ("weight", ctypes.c_int * QAL_BLK_MAX_ROWS),
                ("inv", ctypes.c_int * 64), ("comp", ctypes.c_int * 64),
                ("real", ctypes.c_int * QAL_BLK_MAX_GROUPS), ("rtype", ctypes.c_int * QAL_BLK_MAX_ROWS),
                ("ncode", ctypes.c_int * 64), ("cplx_mults", ctypes.c_int), ("launch_sets", ctypes.c_int)]

    def groups(self):
        return [(self.width[g], self.row0[g], self.off[g]) for g in range(self.ngroups)]

    def flops_per_product(self) -> float:
        return float(sum(self.flops[g] for g in range(self.ngroups)))


def qal_block_plan_build(mats, mirror=True) -> BlockPlan:
    """Structure detection on the union sparsity of `mats` ([m][n][n] complex128, any device; copied to
    host memory because the library's plan builder is host code)."""
    host = mats.detach().to("cpu", torch.complex128).contiguous().reshape(-1, mats.shape[-2], mats.shape[-1])
    plan = BlockPlan()
    rc = load().qal_block_plan_build(host.shape[-1], host.shape[0], ctypes.c_void_p(host.data_ptr()),
                                     1 if mirror else 0, ctypes.byref(plan))
    _check(rc, "qal_block_plan_build")
    return plan


def qal_block_pack(plan: BlockPlan, nat, check=True, stream=None):
    """natural [..., n, n] -> packed [..., plan.packed]; returns (packed, flag) with flag a device int
    tensor (QAL_ERR_STRUCTURE if an off-block entry is non-zero) or None."""
    nat = _dev(nat, torch.complex128, "nat")
    lead = nat.shape[:-2]
    cnt = max(1, int(torch.tensor(lead).prod().item()) if len(lead) else 1)
    out = torch.empty(tuple(lead) + (plan.packed,), dtype=torch.complex128, device=nat.device)
    flag = torch.zeros(1, dtype=torch.int32, device=nat.device) if check else None
    _check(load().qal_block_pack(ctypes.byref(plan), cnt, _ptr(nat), _ptr(out), _ptr(flag), _stream(stream)),
           "qal_block_pack")
    return out, flag


def qal_block_check(plan: BlockPlan, nat, status, broadcast=False, stream=None):
    """Per-pulse structure check (after the step's block calls): status[e] = QAL_ERR_STRUCTURE for every
    matrix nat[e] coupling two blocks (broadcast: every status entry if any matrix fails)."""
    nat = _dev(nat, torch.complex128, "nat")
    cnt = nat.reshape(-1, plan.n, plan.n).shape[0]
    _check(load().qal_block_check(ctypes.byref(plan), cnt, _ptr(nat), 1 if broadcast else 0, _ptr(status),
                                  status.numel(), _stream(stream)), "qal_block_check")
    return status


def qal_block_unpack(plan: BlockPlan, packed, stream=None):
    packed = _dev(packed, torch.complex128, "packed")
    lead = packed.shape[:-1]
    cnt = max(1, int(torch.tensor(lead).prod().item()) if len(lead) else 1)
    out = torch.empty(tuple(lead) + (plan.n, plan.n), dtype=torch.complex128, device=packed.device)
    _check(load().qal_block_unpack(ctypes.byref(plan), cnt, _ptr(packed), _ptr(out), _stream(stream)),
           "qal_block_unpack")
    return out


def qal_block_expm_slices(plan: BlockPlan, L0p, Lcp, u, T, n_slices, *, k0=0, count=None, chunk=None,
                          magnus_order=4, ctrl_mode=QAL_CTRL_PWC, Lcommp=None, status=None, stream=None):
    """Chunk products [B][count/chunk][packed] of the slices k0..k0+count-1 (packed operands)."""
    c128 = torch.complex128
    L0p = _dev(L0p, c128, "L0p")
    Lcp = _dev(Lcp, c128, "Lcp")
    u = _dev(u, torch.float64, "u")
    B, J = u.shape[0], Lcp.shape[0]
    count = n_slices - k0 if count is None else count
    chunk = count if chunk is None else chunk
    out = torch.empty((B, count // chunk, plan.packed), dtype=c128, device=u.device)
    L0s = 0 if L0p.shape[0] == 1 else plan.packed
    Lcs = 0
    if Lcommp is not None:
        Lcommp = _dev(Lcommp, c128, "Lcommp")
        Lcs = 0 if Lcommp.shape[0] == 1 else n_comm(J) * plan.packed
    rc = load().qal_block_expm_slices(ctypes.byref(plan), B, n_slices, float(T), k0, count, magnus_order, ctrl_mode,
                                      J, _ptr(u), _ptr(L0p), L0s, _ptr(Lcp), _ptr(Lcommp), Lcs, chunk, _ptr(out),
                                      _ptr(status), _stream(stream))
    _check(rc, "qal_block_expm_slices")
    return out


def qal_block_ordered_product(plan: BlockPlan, U, stream=None):
    U = _dev(U, torch.complex128, "U")
    B, cnt = U.shape[0], U.shape[1]
    out = torch.empty((B, plan.packed), dtype=torch.complex128, device=U.device)
    wsb = load().qal_block_workspace_bytes(ctypes.byref(plan), QAL_OP_ORDERED_PRODUCT, B, cnt)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=U.device)
    _check(load().qal_block_ordered_product(ctypes.byref(plan), B, cnt, _ptr(U), _ptr(out), _ptr(ws), wsb,
                                            _stream(stream)), "qal_block_ordered_product")
    return out


def qal_block_fidelity(plan: BlockPlan, Lam, V, stream=None):
    Lam = _dev(Lam, torch.complex128, "Lambda")
    V = _dev(V, torch.complex128, "V")
    F = torch.empty(Lam.shape[0], dtype=torch.float64, device=Lam.device)
    _check(load().qal_block_fidelity(ctypes.byref(plan), Lam.shape[0], _ptr(Lam), _ptr(V), _ptr(F), _stream(stream)),
           "qal_block_fidelity")
    return F


def block_workspace_bytes(plan: BlockPlan, op: int, batch: int, n_slices: int) -> int:
    return load().qal_block_workspace_bytes(ctypes.byref(plan), op, batch, n_slices)


def qal_block_fidelity_grad(plan: BlockPlan, L0p, Lcp, u, T, n_slices, V, *, magnus_order=4,
                            ctrl_mode=QAL_CTRL_PWC, Lcommp=None, want_grad=True, want_Lambda=False, status=None,
                            ws=None, stream=None):
    """The hot path on packed operands: (F [B], grad (layout of u) or None, packed Lambda or None)."""
    c128 = torch.complex128
    L0p = _dev(L0p, c128, "L0p")
    Lcp = _dev(Lcp, c128, "Lcp")
    u = _dev(u, torch.float64, "u")
    V = _dev(V, c128, "V")
    B, J = u.shape[0], Lcp.shape[0]
    dev = u.device
    F = torch.empty(B, dtype=torch.float64, device=dev)
    g = torch.empty_like(u) if want_grad else None
    Lam = torch.empty((B, plan.packed), dtype=c128, device=dev) if want_Lambda else None
    op = QAL_OP_FIDELITY_GRAD if want_grad else QAL_OP_FIDELITY
    wsb = block_workspace_bytes(plan, op, B, n_slices)
    if ws is None or ws.numel() < wsb:
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    L0s = 0 if L0p.shape[0] == 1 else plan.packed
    Lcs = 0
    if Lcommp is not None:
        Lcommp = _dev(Lcommp, c128, "Lcommp")
        Lcs = 0 if Lcommp.shape[0] == 1 else n_comm(J) * plan.packed
    rc = load().qal_block_fidelity_grad(ctypes.byref(plan), B, n_slices, float(T), magnus_order, ctrl_mode, J,
                                        _ptr(u), _ptr(L0p), L0s, _ptr(Lcp), _ptr(Lcommp), Lcs, _ptr(V), _ptr(F),
                                        _ptr(g), _ptr(Lam), _ptr(status), _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "qal_block_fidelity_grad")
    return F, g, Lam


def qal_block_propagator_vjp(plan: BlockPlan, L0p, Lcp, u, T, n_slices, Cp, *, k0=0, count=None, magnus_order=4,
                             ctrl_mode=QAL_CTRL_PWC, Lcommp=None, want_Lambda=False, status=None, ws=None,
                             stream=None):
    """dL/du for dL = Re Tr(C dLambda) over slices k0..k0+count-1 (packed, Hermiticity-preserving C [B][packed]);
    returns (grad (layout of u), packed Lambda or None)."""
    c128 = torch.complex128
    L0p = _dev(L0p, c128, "L0p")
    Lcp = _dev(Lcp, c128, "Lcp")
    u = _dev(u, torch.float64, "u")
    Cp = _dev(Cp, c128, "Cp")
    B, J = u.shape[0], Lcp.shape[0]
    count = u.shape[1] if count is None else count
    g = torch.empty_like(u)
    Lam = torch.empty((B, plan.packed), dtype=c128, device=u.device) if want_Lambda else None
    wsb = block_workspace_bytes(plan, QAL_OP_VJP, B, count)
    if ws is None or ws.numel() < wsb:
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=u.device)
    L0s = 0 if L0p.shape[0] == 1 else plan.packed
    Lcs = 0
    if Lcommp is not None:
        Lcommp = _dev(Lcommp, c128, "Lcommp")
        Lcs = 0 if Lcommp.shape[0] == 1 else n_comm(J) * plan.packed
    rc = load().qal_block_propagator_vjp(ctypes.byref(plan), B, n_slices, float(T), k0, count, magnus_order,
                                         ctrl_mode, J, _ptr(u), _ptr(L0p), L0s, _ptr(Lcp), _ptr(Lcommp), Lcs,
                                         _ptr(Cp), _ptr(g), _ptr(Lam), _ptr(status), _ptr(ws), ws.numel(),
                                         _stream(stream))
    _check(rc, "qal_block_propagator_vjp")
    return g, Lam


class BlockGradientSession:
    """qal_block_propagator_forward / _backward around one workspace: forward() stores the U_k, P_k and
    scheme codes of slices k0..k0+count-1 and returns the packed Lambda [B][packed]; vjp(Cp) runs only the
    reverse pass for the packed cotangent Cp [B][packed] (the GradientSession of the block path)."""

    def __init__(self, plan: BlockPlan, L0p, Lcp, u, T, n_slices, *, k0=0, count=None, magnus_order=4,
                 ctrl_mode=QAL_CTRL_PWC, Lcommp=None, status=None, stream=None):
        c128 = torch.complex128
        self.plan = plan
        self.L0p = _dev(L0p, c128, "L0p")
        self.Lcp = _dev(Lcp, c128, "Lcp")
        self.u = _dev(u, torch.float64, "u")
        self.B, self.J = self.u.shape[0], self.Lcp.shape[0]
        self.count = self.u.shape[1] if count is None else count
        self.args = (float(T), k0, self.count, magnus_order, ctrl_mode)
        self.n_slices = n_slices
        self.L0s = 0 if self.L0p.shape[0] == 1 else plan.packed
        self.Lcommp = None if Lcommp is None else _dev(Lcommp, c128, "Lcommp")
        self.Lcs = 0 if self.Lcommp is None or self.Lcommp.shape[0] == 1 else n_comm(self.J) * plan.packed
        self.status = status
        self.stream = stream
        wsb = block_workspace_bytes(plan, QAL_OP_VJP, self.B, self.count)
        self.ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=self.u.device)

    def _common(self):
        T, k0, count, order, mode = self.args
        return (ctypes.byref(self.plan), self.B, self.n_slices, T, k0, count, order, mode, self.J, _ptr(self.u),
                _ptr(self.L0p), self.L0s, _ptr(self.Lcp), _ptr(self.Lcommp), self.Lcs)

    def forward(self):
        Lam = torch.empty((self.B, self.plan.packed), dtype=torch.complex128, device=self.u.device)
        rc = load().qal_block_propagator_forward(*self._common(), _ptr(Lam), _ptr(self.status), _ptr(self.ws),
                                                 self.ws.numel(), _stream(self.stream))
        _check(rc, "qal_block_propagator_forward")
        return Lam

    def vjp(self, Cp):
        Cp = _dev(Cp, torch.complex128, "Cp")
        g = torch.empty_like(self.u)
        rc = load().qal_block_propagator_backward(*self._common(), _ptr(Cp), _ptr(g), _ptr(self.status),
                                                  _ptr(self.ws), self.ws.numel(), _stream(self.stream))
        _check(rc, "qal_block_propagator_backward")
        return g


def qal_block_ordered_scan(plan: BlockPlan, U, want_prefix=True, want_suffix=True, stream=None):
    U = _dev(U, torch.complex128, "U")
    B, cnt = U.shape[0], U.shape[1]
    pre = torch.empty_like(U) if want_prefix else None
    suf = torch.empty_like(U) if want_suffix else None
    ws = torch.empty(4 * B * cnt * plan.packed * 16, dtype=torch.uint8, device=U.device)
    _check(load().qal_block_ordered_scan(ctypes.byref(plan), B, cnt, _ptr(U), _ptr(pre), _ptr(suf), _ptr(ws),
                                         ws.numel(), _stream(stream)), "qal_block_ordered_scan")
    return pre, suf


def qal_block_batched_matmul(plan: BlockPlan, A, B, stream=None):
    """C[i] = A[i] B[i] on packed matrices [count][packed]; a [packed] (or [1][packed]) operand broadcasts."""
    A = _dev(A, torch.complex128, "A").reshape(-1, plan.packed)
    B = _dev(B, torch.complex128, "B").reshape(-1, plan.packed)
    count = max(A.shape[0], B.shape[0])
    C = torch.empty((count, plan.packed), dtype=torch.complex128, device=A.device)
    sa = 0 if A.shape[0] == 1 else plan.packed
    sb = 0 if B.shape[0] == 1 else plan.packed
    _check(load().qal_block_batched_matmul(ctypes.byref(plan), count, _ptr(A), sa, _ptr(B), sb, _ptr(C),
                                           _stream(stream)), "qal_block_batched_matmul")
    return C


def qal_block_fidelity_cotangent(plan: BlockPlan, V, stream=None):
    V = _dev(V, torch.complex128, "V")
    C = torch.empty(plan.packed, dtype=torch.complex128, device=V.device)
    _check(load().qal_block_fidelity_cotangent(ctypes.byref(plan), _ptr(V), _ptr(C), _stream(stream)),
           "qal_block_fidelity_cotangent")
    return C


# --------------------------------------------------------------------------- coherence blocks, n = 4096
QAL_BB_MAX_BLOCKS = 48
QAL_BB_MAX_ROWS = 8192


class BigBlockPlan(ctypes.Structure):
    """Mirror of qal_bigblock_plan (include/qal.h)."""
    _fields_ = [("n", ctypes.c_int), ("d", ctypes.c_int), ("mirror", ctypes.c_int), ("nb", ctypes.c_int),
                ("n_components", ctypes.c_int), ("size", ctypes.c_int * QAL_BB_MAX_BLOCKS),
                ("nt", ctypes.c_int * QAL_BB_MAX_BLOCKS), ("row0", ctypes.c_int * QAL_BB_MAX_BLOCKS),
                ("weight", ctypes.c_int * QAL_BB_MAX_BLOCKS), ("flops", ctypes.c_double * QAL_BB_MAX_BLOCKS),
                ("flops_per_product", ctypes.c_double), ("nrows", ctypes.c_int), ("ntiles", ctypes.c_int),
                ("total_doubles", ctypes.c_longlong), ("perm", ctypes.c_int * QAL_BB_MAX_ROWS),
                ("inv", ctypes.c_int * 4096), ("comp", ctypes.c_int * 4096),
                ("real", ctypes.c_int * QAL_BB_MAX_BLOCKS), ("rtype", ctypes.c_int * QAL_BB_MAX_ROWS),
                ("ncode", ctypes.c_int * 4096)]

    def sizes(self):
        return [self.size[b] for b in range(self.nb)]


def qal_bigblock_plan_build(mats, mirror=True, stream=None) -> BigBlockPlan:
    """Structure of n = 4096 operators (device tensor [m][4096][4096]; pattern computed on the device)."""
    mats = _dev(mats, torch.complex128, "mats")
    plan = BigBlockPlan()
    ws = torch.empty(load().qal_bigblock_plan_workspace_bytes(), dtype=torch.uint8, device=mats.device)
    rc = load().qal_bigblock_plan_build(mats.shape[0], _ptr(mats), 1 if mirror else 0, ctypes.byref(plan),
                                        _ptr(ws), ws.numel(), _stream(stream))
    _check(rc, "qal_bigblock_plan_build")
    return plan


def qal_bigblock_expm_slices(plan: BigBlockPlan, L0, Lc, u, T, n_slices, *, count=None, chunk=None, status=None,
                             check=True, ws=None, stream=None):
    """Chunk products [count/chunk][4096][4096] (natural) of one pulse's PWC slices (u [count][J])."""
    c128 = torch.complex128
    L0 = _dev(L0, c128, "L0")
    Lc = _dev(Lc, c128, "Lc")
    u = _dev(u, torch.float64, "u")
    count = u.shape[0] if count is None else count
    chunk = count if chunk is None else chunk
    out = torch.empty((count // chunk, 4096, 4096), dtype=c128, device=u.device)
    wsb = load().qal_bigblock_workspace_bytes(ctypes.byref(plan))
    if ws is None or ws.numel() < wsb:
        ws = torch.empty(wsb, dtype=torch.uint8, device=u.device)
    flag = torch.zeros(1, dtype=torch.int32, device=u.device) if check else None
    rc = load().qal_bigblock_expm_slices(ctypes.byref(plan), n_slices, float(T), count, Lc.shape[0], _ptr(u),
                                         _ptr(L0), _ptr(Lc), chunk, _ptr(out), _ptr(status), _ptr(flag), _ptr(ws),
                                         ws.numel(), _stream(stream))
    _check(rc, "qal_bigblock_expm_slices")
    return out, flag
