"""The C-ABI boundary without a GPU: libqal.so loads, exports every symbol that
include/qal.h declares, and validates arguments synchronously (error codes come
back before any launch, so these calls need no device)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qal.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2511_13330_b200 import _build
    _build.build()
    from paper_2511_13330_b200 import qal
    return qal.load()


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qal_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_four_north_star_calls():
    syms = declared_symbols()
    for name in ("qal_build_liouvillian", "qal_magnus_expm_slices", "qal_ordered_product", "qal_fidelity_grad"):
        assert name in syms


def test_every_declared_symbol_is_exported(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_every_symbol():
    from paper_2511_13330_b200 import qal
    assert set(declared_symbols()) == set(qal._EXPORTS)


def test_abi_version_and_status_strings(lib):
    assert lib.qal_abi_version() == 2
    assert isinstance(lib.qal_last_cuda_error(), bytes)
    assert lib.qal_status_string(0) == b"ok"
    assert b"NULL" in lib.qal_status_string(-1)
    assert lib.qal_status_string(-99) == b"unknown status"


NULL = None


def call_magnus(lib, **kw):
    a = dict(n=64, batch=1, n_slices=8, T=1.0, k0=0, count=8, order=4, mode=0, J=2, u=1, L0=1, L0s=0, Lc=1,
             Lcomm=NULL, Lcs=0, U=1, chunk=1, P=NULL, status=NULL)
    a.update(kw)
    p = lambda v: None if v is None else ctypes.c_void_p(v)  # noqa: E731 -- fake non-null pointers
    return lib.qal_magnus_expm_slices(a["n"], a["batch"], a["n_slices"], a["T"], a["k0"], a["count"], a["order"],
                                      a["mode"], a["J"], p(a["u"]), p(a["L0"]), a["L0s"], p(a["Lc"]),
                                      p(a["Lcomm"]), a["Lcs"], p(a["U"]), a["chunk"], p(a["P"]), p(a["status"]),
                                      None, 0, None)


@pytest.mark.parametrize("kw,code", [
    (dict(n=16), -5),                 # only n = 64 (d = 8)
    (dict(batch=0), -3),              # empty batch
    (dict(count=0), -3),              # empty slice range
    (dict(T=float("nan")), -4),       # non-finite horizon
    (dict(T=-1.0), -4),
    (dict(order=3), -5),
    (dict(mode=2), -5),
    (dict(J=0), -5),
    (dict(J=9), -5),
    (dict(u=NULL), -1),
    (dict(L0s=7), -2),
    (dict(k0=4, count=8), -2),        # range past the grid
    (dict(U=NULL, P=NULL), -1),       # no output requested
    (dict(U=NULL, P=1, chunk=3), -2),  # chunk does not divide count
    (dict(mode=1, order=4, Lcomm=NULL), -1),  # NODES order 4 needs the commutator basis
])
def test_magnus_validation(lib, kw, code):
    assert call_magnus(lib, **kw) == code


def test_ordered_product_validation(lib):
    p = ctypes.c_void_p(1)
    assert lib.qal_ordered_product(32, 1, 4, p, p, None, 0, None) == -5
    assert lib.qal_ordered_product(64, 1, 0, p, p, None, 0, None) == -3
    assert lib.qal_ordered_product(64, 1, 4, None, p, None, 0, None) == -1
    assert lib.qal_ordered_product(64, 1, 5, p, p, None, 0, None) == -6   # count > 2 needs workspace


def test_fidelity_grad_validation(lib):
    p = ctypes.c_void_p(1)
    args = [8, 1, 16, 1.0, 4, 0, 2, p, p, 0, p, None, 0, p, p, p, None, None, None, 0, None]
    assert lib.qal_fidelity_grad(*args) == -6          # no workspace
    a2 = list(args)
    a2[0] = 4
    assert lib.qal_fidelity_grad(*a2) == -5            # d = 8 only
    a3 = list(args)
    a3[13] = None
    assert lib.qal_fidelity_grad(*a3) == -1            # V missing
    assert lib.qal_fidelity(8, 0, p, p, p, None) == -3
    assert lib.qal_fidelity_ws(64, 1, p, p, p, None, 0, None) == -6          # d = 64 needs the slab workspace
    assert lib.qal_fidelity_ws(64, 1, p, None, p, p, 1 << 20, None) == -1
    assert lib.qal_fidelity_ws(16, 1, p, p, p, None, 0, None) == -5
    assert lib.qal_build_liouvillian(2, 1, p, 1, p, 0, None, 0, p, p, None, None) == -5
    assert lib.qal_build_liouvillian(8, 1, p, 0, None, 0, None, 1, p, None, p, None) == -2


def test_workspace_sizes(lib):
    MB = 64 * 64 * 16
    assert lib.qal_workspace_bytes(1, 64, 1, 2, 0, 0) == 0
    assert lib.qal_workspace_bytes(1, 64, 2, 7, 0, 0) == 2 * (4 + 2) * MB
    g = lib.qal_workspace_bytes(3, 64, 3, 16, 2, 0)
    assert g >= 3 * 3 * 16 * MB + 3 * MB
    assert lib.qal_workspace_bytes(3, 32, 3, 16, 2, 0) == 0
    # qal_fidelity_ws: 512 partial sums per pulse at n = 4096, nothing at n = 64 (no library-held scratch)
    assert lib.qal_workspace_bytes(6, 4096, 3, 1, 0, 0) == 3 * 512 * 8
    assert lib.qal_workspace_bytes(6, 64, 3, 1, 0, 0) == 0


def test_default_chunk_divides_and_is_power_of_two(lib):
    for b, n in [(1, 256), (4096, 1024), (1, 1 << 20), (3, 96), (1, 7)]:
        c = lib.qal_default_chunk(b, n)
        assert c >= 1 and n % c == 0 and (c & (c - 1)) == 0 and c <= 64


def test_library_has_no_runtime_knobs_or_device_globals():
    """reentrant, no global mutable state, the library never allocates in the hot-path calls:
    no getenv, no __device__ scratch arrays, no cudaMalloc in the CUDA sources."""
    csrc = os.path.join(ROOT, "paper_2511_13330_b200", "csrc")
    for f in sorted(os.listdir(csrc)):
        if not f.endswith((".cu", ".cuh", ".h")):
            continue
        text = re.sub(r"//.*", "", open(os.path.join(csrc, f)).read())
        assert "getenv" not in text, f
        assert not re.search(r"cudaMalloc", text), f
        assert not re.search(r"^\s*__device__\s+(?!__forceinline__|inline|static\s+__forceinline__)[\w:<>]+\s+\w+\s*\[", text, re.M), f


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The product package never imports the oracle and has no CPU compute path."""
    pkg = os.path.join(ROOT, "paper_2511_13330_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, re.M), f
                assert "qalref" not in text and "libqalref" not in text, f


# ------------------------------------------------------------------ coherence-block entry points
@pytest.fixture(scope="module")
def plan(lib):
    """A real plan from the configs[0] basis (host call: no device work)."""
    import numpy as np
    import torch

    import oracle
    from paper_2511_13330_b200 import inputs as qi, qal
    oracle.build()
    p = qi.cfg0(N=4, T=1.0)
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    return qal.qal_block_plan_build(torch.from_numpy(np.concatenate([L0[None], Lc])), mirror=True)


def test_block_plan_rejects_bad_input(lib):
    from paper_2511_13330_b200 import qal
    pl = qal.BlockPlan()
    buf = (ctypes.c_double * (2 * 16 * 16))()
    assert lib.qal_block_plan_build(16, 1, buf, 1, ctypes.byref(pl)) == -5       # n = 64 only
    assert lib.qal_block_plan_build(64, 0, buf, 1, ctypes.byref(pl)) == -3
    assert lib.qal_block_plan_build(64, 1, None, 1, ctypes.byref(pl)) == -1
    nan = (ctypes.c_double * (2 * 64 * 64))()
    nan[0] = float("nan")
    assert lib.qal_block_plan_build(64, 1, nan, 1, ctypes.byref(pl)) == -4


def test_block_calls_validate_before_launch(lib, plan):
    p = ctypes.c_void_p(1)
    bp = ctypes.byref(plan)
    P = plan.packed
    # expm slices: empty batch, bad order, chunk not dividing, missing output, bad stride
    assert lib.qal_block_expm_slices(bp, 0, 8, 1.0, 0, 8, 4, 0, 2, p, p, 0, p, None, 0, 1, p, None, None) == -3
    assert lib.qal_block_expm_slices(bp, 1, 8, 1.0, 0, 8, 3, 0, 2, p, p, 0, p, None, 0, 1, p, None, None) == -5
    assert lib.qal_block_expm_slices(bp, 1, 8, 1.0, 0, 8, 4, 0, 2, p, p, 0, p, None, 0, 3, p, None, None) == -2
    assert lib.qal_block_expm_slices(bp, 1, 8, 1.0, 0, 8, 4, 0, 2, p, p, 0, p, None, 0, 1, None, None, None) == -1
    assert lib.qal_block_expm_slices(bp, 1, 8, 1.0, 0, 8, 4, 0, 2, p, p, P + 1, p, None, 0, 1, p, None, None) == -2
    # fidelity-gradient: workspace, V
    args = [bp, 1, 16, 1.0, 4, 0, 2, p, p, 0, p, None, 0, p, p, p, None, None, None, 0, None]
    assert lib.qal_block_fidelity_grad(*args) == -6
    a2 = list(args)
    a2[13] = None
    assert lib.qal_block_fidelity_grad(*a2) == -1
    # a corrupted plan is refused
    bad = type(plan).from_buffer_copy(plan)
    bad.width[0] = 40
    assert lib.qal_block_pack(ctypes.byref(bad), 1, p, p, None, None) == -2
    assert lib.qal_block_pack(bp, 0, p, p, None, None) == -3
    assert lib.qal_block_ordered_product(bp, 1, 5, p, p, None, 0, None) == -6
    assert lib.qal_block_batched_matmul(bp, 2, p, 7, p, 0, p, None) == -2
    assert lib.qal_block_fidelity_cotangent(bp, None, p, None) == -1
    # stored forward / reverse pass of the block path: workspace, output, slice range
    fw = [bp, 1, 16, 1.0, 0, 16, 4, 0, 2, p, p, 0, p, None, 0, p, None, None, 0, None]
    assert lib.qal_block_propagator_forward(*fw) == -6                       # no workspace
    f2 = list(fw)
    f2[15] = None
    assert lib.qal_block_propagator_forward(*f2) == -1                       # Lambda required
    f3 = list(fw)
    f3[4], f3[5] = 8, 16
    assert lib.qal_block_propagator_forward(*f3) == -2                       # range past the grid
    bw = [bp, 1, 16, 1.0, 0, 16, 4, 0, 2, p, p, 0, p, None, 0, p, p, None, None, 0, None]
    assert lib.qal_block_propagator_backward(*bw) == -6
    b2 = list(bw)
    b2[15] = None
    assert lib.qal_block_propagator_backward(*b2) == -1                      # cotangent required
    # per-pulse structure check: empty, NULL status, per-matrix mode needs one status per matrix
    assert lib.qal_block_check(bp, 0, p, 0, p, 1, None) == -3
    assert lib.qal_block_check(bp, 2, p, 0, None, 2, None) == -1
    assert lib.qal_block_check(bp, 2, p, 0, p, 3, None) == -2
    # the launch-layout option of the plan is validated (no run-time environment knobs)
    bad = type(plan).from_buffer_copy(plan)
    bad.launch_sets = 7
    assert lib.qal_block_pack(ctypes.byref(bad), 1, p, p, None, None) == -5


def test_block_workspace_sizes(lib, plan):
    bp = ctypes.byref(plan)
    M = plan.packed * 16
    assert lib.qal_block_workspace_bytes(bp, 1, 1, 2) == 0
    assert lib.qal_block_workspace_bytes(bp, 1, 2, 7) == 2 * (4 + 2) * M
    assert lib.qal_block_workspace_bytes(bp, 3, 3, 16) >= 3 * 3 * 16 * M
    assert lib.qal_block_workspace_bytes(bp, 5, 3, 16) == lib.qal_block_workspace_bytes(bp, 3, 3, 16)


def test_bigblock_calls_validate(lib):
    from paper_2511_13330_b200 import qal
    p = ctypes.c_void_p(1)
    pl = qal.BigBlockPlan()
    wsb = lib.qal_bigblock_plan_workspace_bytes()
    assert wsb == 4096 * 64 * 8                                                   # the 2 MB bitmask
    assert lib.qal_bigblock_plan_build(0, p, 1, ctypes.byref(pl), p, wsb, None) == -3
    assert lib.qal_bigblock_plan_build(1, None, 1, ctypes.byref(pl), p, wsb, None) == -1
    assert lib.qal_bigblock_plan_build(1, p, 1, ctypes.byref(pl), None, 0, None) == -6   # caller workspace
    assert lib.qal_bigblock_plan_build(1, p, 1, ctypes.byref(pl), p, wsb - 1, None) == -6
    assert lib.qal_bigblock_workspace_bytes(ctypes.byref(pl)) == 0               # empty plan
    assert lib.qal_bigblock_expm_slices(ctypes.byref(pl), 8, 1.0, 8, 2, p, p, p, 8, p, None, None, p, 1, None) == -5
