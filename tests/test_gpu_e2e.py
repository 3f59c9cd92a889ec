"""The end-to-end call PulseBatch.step_host (pinned host inputs -> host results, copies on two streams
overlapped with the compute): results equal step() on device-resident inputs, and consecutive steps with
different inputs do not see each other's buffers (the cross-step ordering of the copy pipeline)."""
import numpy as np
import pytest

from paper_2511_13330_b200 import inputs as qi

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("structure", ["blocks", "dense"])
def test_step_host_equals_device_step(torch_cuda, qal, structure):
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    B, N = 40, 64
    probs = [qi.cfg2(batch=B, N=N, T=200.0 * N / 1024, first_pulse=f) for f in (0, 1000, 2000)]
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    p0 = probs[0]
    # three sub-batches (16, 16, 8): the pipeline's per-sub-batch events
    eng = driver.PulseBatch(dev(p0.H0), dev(p0.Hc), dev(p0.C), dev(p0.u), dev(p0.V), p0.T, sub_batch=16,
                            structure=structure)
    assert len(eng.subs()) == 3
    # device-resident reference results, one per input set
    ref = []
    for p in probs:
        eng.H0.copy_(dev(p.H0))
        eng.u.copy_(dev(p.u))
        F, g = eng.step()
        torch.cuda.synchronize()
        ref.append((F.cpu().clone(), g.cpu().clone()))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hin = [(pin(p.H0), pin(p.u)) for p in probs]
    outs = [(torch.empty(B, dtype=torch.float64).pin_memory(),
             torch.empty((B, N, p0.u.shape[2]), dtype=torch.float64).pin_memory()) for _ in probs]
    # back-to-back steps with different inputs, no host sync in between: each must see its own inputs
    for rep in range(2):
        for (hH0, hu), (hF, hg) in zip(hin, outs):
            hF.fill_(np.nan)
            hg.fill_(np.nan)
            eng.step_host(hH0, hu, hF, hg)
        eng.synchronize_host()
        for (hF, hg), (F, g) in zip(outs, ref):
            assert torch.equal(hF, F)
            assert torch.equal(hg, g)
    assert bool((eng.status == 0).all())
