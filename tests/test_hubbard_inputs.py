"""NEXT f3: the Fock-space operators of Eq. 1 -- pinned by the SPEC's worked examples
 and the canonical anticommutation relations."""
import itertools

import numpy as np

from paper_2511_13330_b200 import inputs as qi


def test_basis_order_and_single_dot():
    c_up = qi.fock_creation(0, 0, 1)
    assert c_up[1, 0] == 1.0 and np.count_nonzero(c_up[:, 1]) == 0      # c^dag_up |> = |u>; c^dag_up |u> = 0
    assert np.allclose(np.diag(qi.fock_number(0, 1)).real, [0, 1, 1, 2])
    H0, Hc = qi.hubbard_terms(1, 4.0, [0.5], 0.0)
    assert Hc.shape[0] == 0
    assert np.allclose(np.diag(H0).real, [0, 0.5, 0.5, 5.0])
    # index of |u u d> (N = 3) = 1*16 + 1*4 + 2 = 22
    phi0 = qi.hubbard_logical_states()[0]
    assert abs(phi0[22] - 2 ** -0.5) < 1e-15 and abs(phi0[2 * 16 + 1 * 4 + 1] + 2 ** -0.5) < 1e-15


def test_canonical_anticommutation_two_dots():
    ops = [qi.fock_creation(i, s, 2) for i in range(2) for s in range(2)]
    I = np.eye(16)
    for (a, A), (b, B) in itertools.product(enumerate(ops), repeat=2):
        assert np.allclose(A.conj().T @ B + B @ A.conj().T, I * (a == b), atol=1e-12)
        assert np.allclose(A @ B + B @ A, 0.0, atol=1e-12)


def test_hubbard_hermitian_and_particle_number_conserved():
    H0, Hc = qi.hubbard_terms(3, 2.0, [0.1, -0.2, 0.3], 0.7)
    Ntot = sum(qi.fock_number(i, 3) for i in range(3))
    for H in [H0, *Hc]:
        assert np.allclose(H, H.conj().T, atol=1e-12)
        assert np.allclose(H @ Ntot - Ntot @ H, 0.0, atol=1e-10)
    # single-particle hopping block: <u,-|H_0|-,u> = +-1 (Jordan-Wigner sign)
    H0, Hc = qi.hubbard_terms(2, 0.0, [0.0, 0.0], 0.0)
    assert abs(abs(Hc[0][1 * 4 + 0, 0 * 4 + 1]) - 1.0) < 1e-15


def test_hubbard3_problem_shapes():
    p = qi.hubbard3(N=8)
    assert p.H0.shape == (1, 64, 64) and p.Hc.shape == (2, 64, 64) and p.C.shape == (2, 64, 64)
    phis = qi.hubbard_logical_states()
    assert np.allclose(phis.conj() @ phis.T, np.eye(2), atol=1e-15)
