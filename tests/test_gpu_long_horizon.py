"""NEXT f2 on the GPU: the time-sharded / segmented long-horizon gradient."""
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


def test_fidelity_cotangent_matches_oracle(torch_cuda, qal, oracle):
    V = qi.haar_unitary(8, 5)
    assert relfro(qal.qal_fidelity_cotangent(to(torch_cuda, V)).cpu().numpy(), oracle.fidelity_cotangent(V)) <= 1e-15


def test_segmented_nodes_gradient_matches_oracle(torch_cuda, qal, oracle):
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg3()
    N, T = 512, 500.0
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)
    L0, Lc, Lcomm = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C), want_comm=True)
    V = to(torch, p.V)
    Lam, g = driver.time_sharded_gradient(L0, Lc, Lcomm, to(torch, u[None]), T, N, 0, ctrl_mode=1,
                                          cotangent=lambda Lm: qal.qal_fidelity_cotangent(V), sub=32)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    Fr, gr, Lr = oracle.gradient(rL0, rLc, u, T, N, p.V, mode=1)
    assert relfro(Lam.cpu().numpy(), Lr) <= 1e-10
    assert relfro(g[0].cpu().numpy(), gr) <= 1e-8


def test_cfg3_full_horizon_gradient_directional_derivative(torch_cuda, qal):
    """configs[3] at full size (2^20 NODES slices, segments of 2^16): sum_k grad . delta equals the
    central difference of the forward fidelity along delta (a property at any size)."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg3()
    N, T = p.N, p.T
    L0, Lc, Lcomm = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C), want_comm=True)
    u = qal.qal_sample_controls_sines(to(torch, p.sines), p.u_max, N, T).unsqueeze(0).contiguous()
    V = to(torch, p.V)
    Lam, g = driver.time_sharded_gradient(L0, Lc, Lcomm, u, T, N, 0, ctrl_mode=1,
                                          cotangent=lambda Lm: qal.qal_fidelity_cotangent(V))
    rng = np.random.default_rng(0)
    delta = torch.zeros_like(u)
    for k0 in (123, 400_000, N - 300):                    # three windows of 200 slices
        delta[0, k0:k0 + 200] = to(torch, rng.choice([-1.0, 1.0], size=(200, 2, 2)))

    def F(uu):
        Lm = driver.time_shard_propagator(L0, Lc, Lcomm, uu, T, N, 0, ctrl_mode=1)
        return qal.qal_fidelity(Lm.unsqueeze(0), V).item()

    eps = 1e-5
    fd = (F(u + eps * delta) - F(u - eps * delta)) / (2 * eps)
    an = float((g * delta).sum().item())
    assert abs(fd - an) <= 1e-5 * abs(an)
    assert torch.isfinite(g).all()
