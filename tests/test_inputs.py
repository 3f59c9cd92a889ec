"""Pins for the seeded input generator (no method arithmetic lives there)."""
import math
import os

import numpy as np

from paper_2511_13330_b200 import inputs as qi

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vector():
    lines = [l for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if not l.startswith("#")]
    seed = int(lines[0].split()[1])
    want = [int(x) for x in lines[1:6]]
    got = [int(x) for x in qi.splitmix64(seed, 5)]
    assert got == want
    # counter form: an offset window equals the tail of the full stream
    assert list(qi.splitmix64(seed, 3, offset=2)) == list(qi.splitmix64(seed, 5)[2:])


def test_uniform_normal_moments():
    u = qi.uniform(0, "t", 0, 200_000)
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.005
    z = qi.normal(0, "t", 1, 200_000)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1.0) < 0.01
    # distinct purposes / indices give distinct streams; same key is deterministic
    assert not np.array_equal(qi.uniform(0, "a", 0, 8), qi.uniform(0, "b", 0, 8))
    assert not np.array_equal(qi.uniform(0, "a", 0, 8), qi.uniform(0, "a", 1, 8))
    assert np.array_equal(qi.uniform(5, "a", 3, 8), qi.uniform(5, "a", 3, 8))


def test_spin_operators_closed_forms():
    # sigma- lowers up -> down (A7)
    assert np.allclose(qi.SMINUS @ np.array([1, 0]), [0, 1])
    # (sigma_i . sigma_j)/4 on 3 spins: triplet +1/4 (x6 with the spectator), singlet -3/4 (x2)
    ev = np.sort(np.linalg.eigvalsh(qi.exchange_op(0, 1, 3)))
    assert np.allclose(ev, [-0.75, -0.75] + [0.25] * 6, atol=1e-14)
    # exchange conserves total S^2 and S_z
    S = [sum(qi.site_op(P, i, 3) for i in range(3)) / 2 for P in (qi.SX, qi.SY, qi.SZ)]
    S2 = sum(s @ s for s in S)
    for Hj in (qi.exchange_op(0, 1, 3), qi.exchange_op(1, 2, 3)):
        assert np.abs(Hj @ S2 - S2 @ Hj).max() < 1e-14
        assert np.abs(Hj @ S[2] - S[2] @ Hj).max() < 1e-14
    # Zeeman: eigenvalues are (+-b1 +- b2 +- b3)/2, diagonal in the product basis with
    # spin 1 most significant: basis index 0 = |up up up>, index 1 flips spin 3.
    b = np.array([0.3, 0.5, 0.7])
    H0 = qi.zeeman_h0(b)
    assert np.allclose(np.diag(np.diag(H0)), H0)
    assert math.isclose(H0[0, 0].real, b.sum() / 2)
    assert math.isclose(H0[1, 1].real, (b[0] + b[1] - b[2]) / 2)
    assert math.isclose(H0[4, 4].real, (-b[0] + b[1] + b[2]) / 2)


def test_collapse_operators_rates():
    C = qi.collapse_ops(3, t1=100.0, t2=10.0)
    assert C.shape == (6, 8, 8)
    # Tr(c^dag c): sigma-_i/sqrt(T1) -> 4/T1 (|up><up| on spin i, x4 spectators)
    for i in range(3):
        assert math.isclose(np.trace(C[i].conj().T @ C[i]).real, 4 / 100.0)
    # sigma_z sqrt(1/(2T2)) -> 8/(2 T2)
    for i in range(3, 6):
        assert math.isclose(np.trace(C[i].conj().T @ C[i]).real, 8 / 20.0)


def test_haar_unitary():
    V = qi.haar_unitary(8, 0)
    assert np.abs(V.conj().T @ V - np.eye(8)).max() < 1e-14
    assert np.array_equal(V, qi.haar_unitary(8, 0))
    assert not np.allclose(V, qi.haar_unitary(8, 1))
    V64 = qi.haar_unitary(64, 4)
    assert np.abs(V64.conj().T @ V64 - np.eye(64)).max() < 1e-13


def test_configs_shapes():
    p0 = qi.cfg0()
    assert p0.u.shape == (1, 256, 2) and p0.u.min() >= 0 and p0.u.max() < qi.U_MAX
    assert p0.H0.shape == (1, 8, 8) and p0.C.shape == (6, 8, 8) and p0.Hc.shape == (2, 8, 8)
    p2 = qi.cfg2(batch=4, N=16)
    assert p2.u.shape == (4, 16, 2) and p2.H0.shape == (4, 8, 8)
    # pulse p of a sub-batch is pulse first_pulse + p of the full stream
    p2b = qi.cfg2(batch=2, N=16, first_pulse=2)
    assert np.array_equal(p2b.u, p2.u[2:]) and np.array_equal(p2b.H0, p2.H0[2:])
    p3 = qi.cfg3(N=1024)
    assert p3.sines.shape == (2, 16, 3) and p3.ctrl_mode == qi.CTRL_NODES
    p4 = qi.cfg4(batch=2, N=4)
    assert p4.H0.shape == (1, 64, 64) and p4.C.shape == (12, 64, 64) and p4.Hc.shape == (5, 64, 64)
