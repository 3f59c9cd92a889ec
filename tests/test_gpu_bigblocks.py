"""Coherence blocks on the n = 4096 path (configs[4] six spins; the 3-dot Hubbard model, NEXT f3).

The oracle cannot form 4096^2 propagators in test time; the block path is checked against the DENSE
n = 4096 path (itself pinned to the oracle in tests/test_gpu_dense.py) on the same slices, element by
element, plus the block structure against the coherence order computed from the spin basis alone
(A5, A7), the device structure check, and the dense CPTP invariants at full pulse length."""
from collections import Counter

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
    p = qi.cfg4(batch=1)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    plan = qal.qal_bigblock_plan_build(torch.cat([L0, Lc]), mirror=True)
    return p, L0, Lc, plan


def test_six_spin_blocks_are_the_coherence_sectors(cfg4):
    p, L0, Lc, plan = cfg4
    up = [6 - bin(i).count("1") for i in range(64)]
    q = np.array([up[R % 64] - up[R // 64] for R in range(4096)])
    comp = np.array(list(plan.comp))
    # same partition as the coherence order
    for a in range(0, 4096, 37):
        assert np.all((comp == comp[a]) == (q == q[a]))
    # best-fit packing: {924} -> 960, {792} -> 832, {495, 12, 1} -> 512, {220} -> 256, {66} -> 128
    assert sorted(plan.sizes(), reverse=True) == [924, 792, 508, 220, 66]
    assert plan.n_components == 13
    dense = 8.0 * 4096 ** 3
    assert plan.flops_per_product / dense < 0.025


@pytest.mark.parametrize("count,chunk", [(3, 3), (4, 2)])
def test_bigblock_chunks_match_the_dense_path(cfg4, qal, torch_cuda, count, chunk):
    torch = torch_cuda
    p, L0, Lc, plan = cfg4
    u = to(torch, p.u[0, :count])
    P, flag = qal.qal_bigblock_expm_slices(plan, L0, Lc, u, p.T, p.N, chunk=chunk)
    assert flag.item() == 0
    _, D = qal.qal_magnus_expm_slices(L0, Lc, u.unsqueeze(0), p.T, p.N, count=count, chunk=chunk)
    for c in range(count // chunk):
        assert relfro(P[c].cpu().numpy(), D[0, c].cpu().numpy()) <= 1e-12


def test_bigblock_squarings_per_block(cfg4, qal, torch_cuda):
    """Long slices (large ||Omega||): every block picks its own s; still equal to the dense path."""
    torch = torch_cuda
    p, L0, Lc, plan = cfg4
    T, N = 400.0, 4
    u = to(torch, p.u[0, :2])
    P, _ = qal.qal_bigblock_expm_slices(plan, L0, Lc, u, T, N, chunk=2)
    _, D = qal.qal_magnus_expm_slices(L0, Lc, u.unsqueeze(0), T, N, count=2, chunk=2)
    assert relfro(P[0].cpu().numpy(), D[0, 0].cpu().numpy()) <= 1e-11


def test_bigblock_full_pulse_fidelity_matches_dense(cfg4, qal, torch_cuda):
    """configs[4] pulse 0 at full length (512 slices): fidelity and Lambda equal to the dense path."""
    torch = torch_cuda
    p, L0, Lc, plan = cfg4
    u = to(torch, p.u[0])
    P, _ = qal.qal_bigblock_expm_slices(plan, L0, Lc, u, p.T, p.N)
    Fb = qal.qal_fidelity(P, to(torch, p.V)).item()
    Fd, _, Ld = qal.qal_fidelity_grad(L0, Lc, u.unsqueeze(0).contiguous(), p.T, p.N, to(torch, p.V),
                                      want_grad=False, want_Lambda=True)
    assert abs(Fb - Fd.item()) <= 1e-10 * abs(Fd.item())
    assert relfro(P[0].cpu().numpy(), Ld[0].cpu().numpy()) <= 1e-10


def test_hubbard_structure_and_slice(torch_cuda, qal):
    """NEXT f3: the 3-dot Hubbard Liouvillian is block diagonal too (particle number and S_z); the
    block path reproduces the dense slice."""
    torch = torch_cuda
    p = qi.hubbard3(N=2, T=100.0 * 2 / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    plan = qal.qal_bigblock_plan_build(torch.cat([L0, Lc]), mirror=True)
    assert plan.nb >= 2 and plan.flops_per_product < 0.5 * 8.0 * 4096 ** 3
    u = to(torch, p.u[0])
    P, flag = qal.qal_bigblock_expm_slices(plan, L0, Lc, u, p.T, p.N)
    assert flag.item() == 0
    _, D = qal.qal_magnus_expm_slices(L0, Lc, u.unsqueeze(0), p.T, p.N, chunk=p.N)
    assert relfro(P[0].cpu().numpy(), D[0, 0].cpu().numpy()) <= 1e-11


# ---- direct oracle checks of the n = 4096 block path (no dense GPU path in between) ------------------

def test_bigblock_dissipative_slices_vs_oracle_rk4_on_rho(torch_cuda, qal, oracle):
    """configs[4] pulse 0, two dissipative slices on the coherence-block path, applied to random density
    matrices vs the oracle's RK4 of Eq. 6 on rho (256 sub-steps per slice, RK4 error ~1e-13):
    the packed blocks, the Hermitian mirror and the real basis of the q = 0 block all enter Lambda."""
    torch = torch_cuda
    N = 2
    p = qi.cfg4(batch=1, N=N, T=100.0 * N / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    plan = qal.qal_bigblock_plan_build(torch.cat([L0, Lc]), mirror=True)
    P, flag = qal.qal_bigblock_expm_slices(plan, L0, Lc, to(torch, p.u[0]), p.T, p.N)
    assert flag.item() == 0
    Lam = P[0]
    rng = np.random.default_rng(19)
    for _ in range(2):
        a = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
        rho0 = a @ a.conj().T
        rho0 /= np.trace(rho0)
        ref = oracle.evolve_rho(p.H0[0], p.Hc, p.C, p.u[0], p.T, p.N, 256, rho0)
        v = to(torch, rho0.reshape(-1, order="F").copy())
        got = (Lam @ v).cpu().numpy().reshape(64, 64, order="F")
        assert relfro(got, ref) <= 1e-10


def test_bigblock_hubbard_dissipative_slice_vs_oracle_rk4_on_rho(torch_cuda, qal, oracle):
    """NEXT f3 on the block path: one 3-dot Hubbard slice (||Omega||_1 ~ 25: per-block squarings) applied
    to a logical-subspace density matrix vs the oracle's RK4 of Eq. 6 with 8192 sub-steps."""
    torch = torch_cuda
    p = qi.hubbard3(N=1, T=100.0 / 512)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    plan = qal.qal_bigblock_plan_build(torch.cat([L0, Lc]), mirror=True)
    P, flag = qal.qal_bigblock_expm_slices(plan, L0, Lc, to(torch, p.u[0]), p.T, p.N)
    assert flag.item() == 0
    phis = qi.hubbard_logical_states()
    rho0 = 0.7 * np.outer(phis[0], phis[0].conj()) + 0.3 * np.outer(phis[1], phis[1].conj())
    rho0 += 0.2 * (np.outer(phis[0], phis[1].conj()) + np.outer(phis[1], phis[0].conj()))
    ref = oracle.evolve_rho(p.H0[0], p.Hc, p.C, p.u[0], p.T, 1, 8192, rho0)
    v = to(torch, rho0.reshape(-1, order="F").copy())
    got = (P[0] @ v).cpu().numpy().reshape(64, 64, order="F")
    assert relfro(got, ref) <= 1e-10
