"""Structure detection of the coherence-block path (host code in libqal.so; no GPU needed).

Pinned against the physics, not against the library: total S_z conservation (Eq. 6) makes
the Liouvillian block diagonal by coherence order q = m(i) - m(j) of vec(rho)[i + d j] = rho[i][j]
(column stacking, A5), where m counts the up spins of basis state i (A7: bit = 0 is up).  The sectors
are computed here from that definition alone and must equal the plan's components; Hermiticity
preservation pairs q with -q (P-5).
"""
from collections import Counter

import numpy as np
import pytest
import torch

from paper_2511_13330_b200 import inputs as qi


@pytest.fixture(scope="module")
def qal():
    from paper_2511_13330_b200 import _build, qal as q
    _build.build()
    q.load()
    return q


def coherence_order(d=8, nspin=3):
    up = [nspin - bin(i).count("1") for i in range(d)]
    return np.array([up[R % d] - up[R // d] for R in range(d * d)])


@pytest.fixture(scope="module")
def basis(oracle):
    p = qi.cfg2(batch=2, N=4)
    mats = []
    for b in range(2):
        L0, Lc = oracle.build_liouvillian(p.H0[b], p.Hc, p.C)
        mats.append(L0[None])
    mats.append(Lc)
    return torch.from_numpy(np.concatenate(mats))


def plan_components(plan):
    return np.array(list(plan.comp)[:64])


def test_components_are_the_coherence_order_sectors(qal, basis):
    plan = qal.qal_block_plan_build(basis, mirror=False)
    q = coherence_order()
    comp = plan_components(plan)
    # same partition: two indices share a component iff they share q
    assert all((comp[a] == comp[b]) == (q[a] == q[b]) for a in range(64) for b in range(64))
    assert sorted(Counter(q).values(), reverse=True) == [20, 15, 15, 6, 6, 1, 1]
    assert plan.n_components == 7


def test_mirror_keeps_one_of_each_pair(qal, basis):
    plan = qal.qal_block_plan_build(basis, mirror=True)
    q = coherence_order()
    rows = [plan.perm[r] for r in range(plan.nrows) if plan.perm[r] >= 0]
    kept = sorted(set(q[rows]))
    assert len(rows) == 20 + 15 + 6 + 1
    assert len(kept) == 4 and all(-k not in kept or k == 0 for k in kept)   # one of q, -q
    for r in range(plan.nrows):
        R = plan.perm[r]
        if R < 0:
            assert plan.weight[r] == 0
        else:
            assert plan.weight[r] == (1 if q[R] == 0 else 2)


def test_packing_layout_is_consistent(qal, basis):
    for mirror in (True, False):
        plan = qal.qal_block_plan_build(basis, mirror=mirror)
        row = off = 0
        for g in range(plan.ngroups):
            w = plan.width[g]
            assert w in (8, 16, 24) and plan.row0[g] == row and plan.off[g] == off
            row += w
            off += w * w
        assert row == plan.nrows and off == plan.packed
        stored = []
        for r in range(plan.nrows):
            R = plan.perm[r]
            if R < 0 or plan.rtype[r] == 3:
                continue
            stored.append(R)
            if plan.rtype[r] == 2:                     # real pair: a row covers R and its mirror
                stored.append((R // 8) + 8 * (R % 8))
        assert len(stored) == len(set(stored))
        for R in range(64):
            r = plan.inv[R]
            assert r == -1 or plan.perm[r] == R
        if not mirror:
            assert sorted(stored) == list(range(64))


def test_small_components_join_the_narrowest_block(qal, basis):
    """Packing rule (DESIGN 5c): the 1 x 1 q = 3 component joins the 6-block (width 8), not the 15-block,
    so the 15-block's (m, s) choice does not pay for the q = 3 norm.  d = 8 with the mirror:
    {20} real in 24, {15} in 16, {6, 1} in 8."""
    plan = qal.qal_block_plan_build(basis, mirror=True)
    got = sorted((plan.width[g], plan.used[g], plan.real[g]) for g in range(plan.ngroups))
    assert got == [(8, 7, 0), (16, 15, 0), (24, 20, 1)]


def test_flops_are_the_block_cubes(qal, basis):
    plan = qal.qal_block_plan_build(basis, mirror=True)
    mults = plan.cplx_mults
    assert mults in (3, 4)
    # the self-mirrored q = 0 block (20) is real (1 real product), the others complex
    assert plan.flops_per_product() == 2 * 20 ** 3 + 2 * mults * (15 ** 3 + 6 ** 3 + 1)
    dense = 2 * 4 * 64 ** 3
    assert plan.flops_per_product() / dense < 0.05


def test_dense_coupling_gives_one_component_and_is_rejected(qal):
    M = torch.ones((1, 64, 64), dtype=torch.complex128)
    with pytest.raises(qal.QalError):
        qal.qal_block_plan_build(M, mirror=True)     # one 64-wide component > 24: unsupported


def hermitian_basis(plan, g):
    """T (natural x packed rows of group g) from the plan: e_R, (e_R + e_sR)/sqrt2, i(e_R - e_sR)/sqrt2."""
    w, r0 = plan.width[g], plan.row0[g]
    T = np.zeros((64, w), dtype=complex)
    for r in range(w):
        R = plan.perm[r0 + r]
        if R < 0:
            continue
        sR = (R // 8) + 8 * (R % 8)
        t = plan.rtype[r0 + r]
        if t in (0, 1):
            T[R, r] = 1.0
        elif t == 2:
            T[R, r] = T[sR, r] = 2 ** -0.5
        else:
            T[R, r], T[sR, r] = 1j * 2 ** -0.5, -1j * 2 ** -0.5
    return T


def test_real_basis_makes_hermiticity_preserving_maps_real(qal, basis, oracle):
    """A29: in the Hermitian basis of the self-mirrored block, T is an isometry and every
    Hermiticity-preserving generator (L0, L_j, and a propagator) is real."""
    plan = qal.qal_block_plan_build(basis, mirror=True)
    reals = [g for g in range(plan.ngroups) if plan.real[g]]
    assert len(reals) == 1 and plan.used[reals[0]] == 20
    g = reals[0]
    T = hermitian_basis(plan, g)[:, :plan.used[g]]
    assert np.allclose(T.conj().T @ T, np.eye(plan.used[g]), atol=1e-15)
    p = qi.cfg0(N=4, T=2.0)
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Lam = oracle.propagate(L0, Lc, p.u[0], p.T, p.N)
    for M in (L0, Lc[0], Lc[1], Lam):
        Mp = T.conj().T @ M @ T
        assert np.max(np.abs(Mp.imag)) <= 1e-14 * max(1.0, np.max(np.abs(Mp)))
