"""NEXT f1 on the GPU: forward/VJP split with arbitrary cotangents and prefix seeds, the
Eqs. 16-17 logical loss and Adam vs the oracle, and the calibration loop end to end."""
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


def test_logical_loss_matches_oracle(torch_cuda, qal, oracle):
    torch = torch_cuda
    rng = np.random.default_rng(4)
    Lam = (rng.standard_normal((3, 64, 64)) + 1j * rng.standard_normal((3, 64, 64))) / 8
    P = qi.projection_matrix()
    G = qi.LOGICAL_GATES["X"]
    loss, C = qal.qal_logical_loss(to(torch, Lam), to(torch, P), to(torch, G))
    for b in range(3):
        lr, Cr = oracle.logical_loss(Lam[b], P, G)
        assert abs(loss[b].item() - lr) <= 1e-13 * lr
        assert relfro(C[b].cpu().numpy(), Cr) <= 1e-13


@pytest.mark.parametrize("mode", [0, 1])
def test_vjp_with_random_cotangent_matches_oracle(torch_cuda, qal, oracle, mode):
    torch = torch_cuda
    if mode == 0:
        p = qi.cfg0(N=24, T=100.0 * 24 / 256)
        u = p.u
    else:
        p = qi.cfg3()
        u = oracle.sines_nodes(p.sines, p.u_max, 24, 300.0)[None]
        p.T, p.N = 300.0, 24
    L0, Lc, Lcomm = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C),
                                              want_comm=(mode == 1))
    rng = np.random.default_rng(6)
    C = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
    sess = qal.GradientSession(L0, Lc, to(torch, u), p.T, p.N, ctrl_mode=mode, Lcomm=Lcomm)
    Lam = sess.forward()
    g = sess.vjp(to(torch, C[None]))
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    gr, Lr = oracle.vjp(rL0, rLc, u[0], p.T, p.N, C, mode=mode)
    assert relfro(Lam[0].cpu().numpy(), Lr) <= 1e-10
    assert relfro(g[0].cpu().numpy(), gr) <= 1e-8


def test_forward_with_prefix_seed(torch_cuda, qal, oracle):
    """P_init multiplies on the right: Lambda = U_{k0+count-1} ... U_{k0} P_init (time sharding)."""
    torch = torch_cuda
    p = qi.cfg0(N=32, T=100.0 * 32 / 256)
    L0, Lc, _ = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C))
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    first = oracle.propagate(rL0, rLc, p.u[0], p.T, p.N, k0=0, k1=16)
    full = oracle.propagate(rL0, rLc, p.u[0], p.T, p.N)
    sess = qal.GradientSession(L0, Lc, to(torch, p.u[:, 16:]), p.T, p.N, k0=16)
    Lam = sess.forward(P_init=to(torch, first[None]))
    assert relfro(Lam[0].cpu().numpy(), full) <= 1e-10


def test_adam_matches_oracle(torch_cuda, qal, oracle):
    torch = torch_cuda
    rng = np.random.default_rng(1)
    th, m, v = rng.standard_normal(1000), np.zeros(1000), np.zeros(1000)
    tth, tm, tv = to(torch, th), to(torch, m), to(torch, v)
    for t in range(1, 6):
        g = rng.standard_normal(1000)
        oracle.adam_step(th, g, m, v, t, lr=0.03)
        qal.qal_adam_step(tth, to(torch, g), tm, tv, t, lr=0.03)
    assert np.max(np.abs(tth.cpu().numpy() - th)) <= 1e-14


def test_calibration_loop_recovers_a_reachable_target(torch_cuda, qal):
    """Inverse problem (S:385 adapted): the target Pi* comes from a known schedule u*; Adam from a
    perturbed start drives the Eq. 16-17 loss down by orders of magnitude."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg0(N=16, T=60.0)
    P = to(torch, qi.projection_matrix())
    H0, Hc, C = to(torch, p.H0), to(torch, p.Hc), to(torch, p.C)
    ustar = to(torch, p.u)
    L0, Lc, _ = qal.qal_build_liouvillian(H0, Hc, C)
    Lam_star = qal.GradientSession(L0, Lc, ustar, p.T, p.N).forward()
    Pd = P.conj().T
    G = (Pd @ Lam_star[0] @ P).contiguous()                    # reachable logical target
    rng = np.random.default_rng(0)
    u0 = ustar + to(torch, 0.05 * rng.standard_normal(p.u.shape))
    out = driver.calibrate(H0, Hc, C, u0, p.T, P, G, iters=300, lr=5e-3)
    hist = out["loss_history"][:, 0].cpu().numpy()
    assert np.all(np.isfinite(hist)) and np.all(hist >= 0)
    assert np.all(np.diff(np.minimum.accumulate(hist)) <= 0)   # best-so-far non-increasing
    assert out["best_loss"][0].item() <= hist[0] * 1e-3


def test_calibration_loop_on_the_block_path_matches_dense(torch_cuda, qal):
    """NEXT f1 on the coherence-block path: the same Adam trajectory as the dense path (the loss and
    its gradient are identical up to rounding), and the loss falls by orders of magnitude."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg0(N=16, T=60.0)
    P = to(torch, qi.projection_matrix())
    H0, Hc, C = to(torch, p.H0), to(torch, p.Hc), to(torch, p.C)
    ustar = to(torch, p.u)
    L0, Lc, _ = qal.qal_build_liouvillian(H0, Hc, C)
    Lam_star = qal.GradientSession(L0, Lc, ustar, p.T, p.N).forward()
    G = (P.conj().T @ Lam_star[0] @ P).contiguous()
    assert float(G.imag.abs().max()) <= 1e-12                  # real for an HP map and Hermitian projectors
    G = G.real.to(torch.complex128).contiguous()
    rng = np.random.default_rng(0)
    u0 = ustar + to(torch, 0.05 * rng.standard_normal(p.u.shape))
    d = driver.calibrate(H0, Hc, C, u0, p.T, P, G, iters=60, lr=5e-3)
    b = driver.calibrate(H0, Hc, C, u0, p.T, P, G, iters=60, lr=5e-3, structure="blocks")
    hd, hb = d["loss_history"][:, 0].cpu().numpy(), b["loss_history"][:, 0].cpu().numpy()
    assert np.max(np.abs(hd - hb) / np.maximum(hd, 1e-300)) <= 1e-8
    assert hb[-1] <= hb[0] * 1e-1
