"""Full-size parity at BASELINE.json sizes, in the launch configuration bench.py times:
sampled outputs the oracle computes one by one, and properties that hold at any size."""
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
def cfg2_full(torch_cuda, qal):
    """configs[2] at full size through driver.PulseBatch with bench.py's sub-batch (296)."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg2()
    eng = driver.PulseBatch(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C), to(torch, p.u), to(torch, p.V),
                            p.T, sub_batch=296)
    F, g = eng.step()
    torch.cuda.synchronize()
    return p, F.cpu().numpy(), g.cpu().numpy(), eng.status.cpu().numpy()


# 16 sampled pulses of configs[2] (a seeded 16-pulse subset including pulses 0 and 4095):
# both ends, the sub-batch boundaries of the dense (296) and block (1776) launches, the rank boundaries of
# the 4096/G split at G = 2, 4, 8 (bench.py), and seeded draws
CFG2_PULSES = sorted({0, 1, 295, 296, 511, 512, 1023, 1775, 1776, 2047, 2048, 3583, 3584, 4095}
                     | set(int(x) for x in np.random.default_rng(2024).choice(4096, 2, replace=False)))


@pytest.fixture(scope="module")
def cfg2_oracle(oracle):
    """O1-O7 of the oracle on each sampled pulse, computed once for the dense and block tests."""
    p = qi.cfg2()
    cache = {}

    def get(pulse):
        if pulse not in cache:
            L0, Lc = oracle.build_liouvillian(p.H0[pulse], p.Hc, p.C)
            Fr, gr, _ = oracle.gradient(L0, Lc, p.u[pulse], p.T, p.N, p.V)
            cache[pulse] = (Fr, gr)
        return cache[pulse]
    return get


def test_cfg2_sample_has_16_pulses_with_both_ends():
    assert len(CFG2_PULSES) == 16 and CFG2_PULSES[0] == 0 and CFG2_PULSES[-1] == 4095


@pytest.mark.parametrize("pulse", CFG2_PULSES)
def test_cfg2_full_size_sampled_pulses(cfg2_full, cfg2_oracle, pulse):
    p, F, g, status = cfg2_full
    assert status[pulse] == 0
    Fr, gr = cfg2_oracle(pulse)
    assert abs(F[pulse] - Fr) / abs(Fr) <= 1e-10
    assert relfro(g[pulse], gr) <= 1e-8


def test_cfg2_full_size_properties(cfg2_full):
    _, F, g, status = cfg2_full
    assert np.all(status == 0)
    assert np.all(np.isfinite(F)) and np.all(np.isfinite(g))
    assert np.all((F > 0.0) & (F < 1.0))          # process fidelity of a CPTP map lies in [0, 1]


@pytest.fixture(scope="module")
def cfg3_full(torch_cuda, qal):
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg3()
    L0, Lc, Lcomm = qal.qal_build_liouvillian(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C), want_comm=True)
    u = qal.qal_sample_controls_sines(to(torch, p.sines), p.u_max, p.N, p.T)
    return p, L0, Lc, Lcomm, u


def test_cfg3_full_horizon_properties_and_bit_identity_across_G(cfg3_full, qal, torch_cuda):
    """N = 2^20: trace / Hermiticity preservation (P-4, P-5), exact coherence-order zeros (P-13),
    and the time-sharded product for G = 2, 4, 8 bit-identical to G = 1 (A16)."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p, L0, Lc, Lcomm, u = cfg3_full
    N = p.N
    lam = {}
    for G in (1, 2, 4, 8):
        parts = []
        for r in range(G):
            k0, k1 = driver.shard_range(N, G, r)
            parts.append(driver.local_partial(L0, Lc, Lcomm, u[k0:k1].unsqueeze(0).contiguous(), p.T, N, k0,
                                              ctrl_mode=1))
        lam[G] = driver.ordered_combine(torch.stack(parts)).cpu().numpy()
    for G in (2, 4, 8):
        assert np.array_equal(lam[G], lam[1]), G
    Lam = lam[1]
    vecI = np.eye(8).reshape(-1, order="F")
    assert np.max(np.abs(vecI @ Lam - vecI)) <= 1e-10
    idx = np.arange(64)
    sw = (idx // 8) + 8 * (idx % 8)
    assert np.max(np.abs(Lam - Lam[sw][:, sw].conj())) <= 1e-10
    m = np.array([bin(i).count("1") for i in range(8)])   # number of down spins
    q = np.array([m[a // 8] - m[a % 8] for a in range(64)])  # coherence order of vec index a = i + 8 j
    off = q[:, None] != q[None, :]
    assert np.all(Lam[off] == 0.0)


def _cfg3_golden():
    """tests/golden/cfg3_*: Lambda and F of the full configs[3] horizon written by tools/golden_cfg3.py,
    which calls only the oracle (sequential left fold of Eq. 15 from Lambda = I, Magnus-4, NODES)."""
    import hashlib
    import json
    import os
    gd = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(gd, "cfg3_meta.json")) as f:
        meta = json.load(f)
    Lam = np.load(os.path.join(gd, "cfg3_lambda.npy"))
    assert hashlib.sha256(Lam.tobytes()).hexdigest() == meta["sha256_lambda"]
    p = qi.cfg3()
    assert meta["N"] == p.N and abs(meta["T_ns"] - p.T) == 0.0
    # the seeded inputs this build generates are the ones the golden was computed from
    assert hashlib.sha256(np.ascontiguousarray(p.sines).tobytes()).hexdigest() == meta["sha256_sines"]
    assert hashlib.sha256(np.ascontiguousarray(p.V).tobytes()).hexdigest() == meta["sha256_V"]
    return Lam, meta["F"]


@pytest.mark.parametrize("structure", ["dense", "blocks"])
def test_cfg3_full_horizon_vs_oracle_golden(cfg3_full, qal, torch_cuda, structure):
    """N = 2^20 end to end (bench.py --config cfg3 at G = 1: chunk fold + balanced tree) against the
    oracle's sequential fold over the whole horizon: relative Frobenius error of Lambda and relative
    error of F within BJ's 1e-10 (SURVEY 7 predicted a fold-vs-tree drift of ~7.5e-12)."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p, L0, Lc, Lcomm, u = cfg3_full
    Lr, Fr = _cfg3_golden()
    V = to(torch, p.V)
    if structure == "dense":
        Lam = driver.time_shard_propagator(L0, Lc, Lcomm, u.unsqueeze(0).contiguous(), p.T, p.N, 0, ctrl_mode=1)
        F = qal.qal_fidelity(Lam.unsqueeze(0), V).item()
        Lg = Lam.cpu().numpy()
    else:
        plan = qal.qal_block_plan_build(torch.cat([L0, Lc, Lcomm.reshape(-1, 64, 64)]), mirror=True)
        mats = [qal.qal_block_pack(plan, m, check=True)[0] for m in (L0, Lc, Lcomm)]
        Lp = driver.time_shard_propagator(*mats, u.unsqueeze(0).contiguous(), p.T, p.N, 0, ctrl_mode=1, plan=plan)
        F = qal.qal_block_fidelity(plan, Lp.unsqueeze(0), V).item()
        Lg = qal.qal_block_unpack(plan, Lp.unsqueeze(0))[0].cpu().numpy()
    eL, eF = relfro(Lg, Lr), abs(F - Fr) / abs(Fr)
    print(f"cfg3 golden ({structure}): |dLambda|/|Lambda| = {eL:.3e}, |dF|/|F| = {eF:.3e}")
    assert eL <= 1e-10 and eF <= 1e-10


@pytest.mark.parametrize("chunk_index", [0, 7777, 16383])
def test_cfg3_full_horizon_sampled_chunks(cfg3_full, qal, oracle, chunk_index):
    """The chunk partials bench.py folds (chunk 64 of the 2^20-slice grid) vs the oracle."""
    p, L0, Lc, Lcomm, u = cfg3_full
    from paper_2511_13330_b200 import driver
    chunk = driver.time_shard_chunk(p.N)
    k0 = chunk_index * chunk
    _, P = qal.qal_magnus_expm_slices(L0, Lc, u[k0:k0 + chunk].unsqueeze(0).contiguous(), p.T, p.N, k0=k0,
                                      count=chunk, ctrl_mode=1, Lcomm=Lcomm, chunk=chunk)
    rL0, rLc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    uref = oracle.sines_nodes(p.sines, p.u_max, p.N, p.T, k0, k0 + chunk)
    ref = oracle_range(oracle, rL0, rLc, uref, p.T, p.N, k0, chunk)
    assert relfro(P[0, 0].cpu().numpy(), ref) <= 1e-10


def oracle_range(oracle, L0, Lc, u_rows, T, N, k0, count):
    """oracle.propagate indexes u by absolute slice; hand it a table whose row k0+i is u_rows[i]."""
    full = np.zeros((k0 + count,) + u_rows.shape[1:])
    full[k0:] = u_rows
    return oracle.propagate(L0, Lc, full, T, N, mode=1, k0=k0, k1=k0 + count)


# ---- coherence-block path (bench.py's default structure) at the same full sizes -----------------------

@pytest.fixture(scope="module")
def cfg2_full_blocks(torch_cuda, qal):
    """configs[2] at full size through driver.PulseBatch(structure="blocks") with bench.py's automatic
    sub-batch -- the exact launch configuration of the headline bench line."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p = qi.cfg2()
    eng = driver.PulseBatch(to(torch, p.H0), to(torch, p.Hc), to(torch, p.C), to(torch, p.u), to(torch, p.V),
                            p.T, structure="blocks")
    F, g = eng.step()
    torch.cuda.synchronize()
    ok = eng.structure_ok()
    out = (p, F.cpu().numpy(), g.cpu().numpy(), eng.status.cpu().numpy(), ok, eng.sub)
    del eng
    torch.cuda.empty_cache()
    return out


@pytest.mark.parametrize("pulse", CFG2_PULSES)
def test_cfg2_blocks_full_size_sampled_pulses(cfg2_full_blocks, cfg2_oracle, pulse):
    p, F, g, status, ok, sub = cfg2_full_blocks
    assert ok
    assert status[pulse] == 0
    Fr, gr = cfg2_oracle(pulse)
    assert abs(F[pulse] - Fr) / abs(Fr) <= 1e-10
    assert relfro(g[pulse], gr) <= 1e-8


def test_cfg2_blocks_full_size_properties_and_dense_agreement(cfg2_full_blocks, cfg2_full):
    """Every one of the 4096 pulses: finite, F in (0, 1), and the same F / gradient as the dense path
    (two independent kernel families; the block path drops only exact zeros, A26)."""
    _, F, g, status, ok, _ = cfg2_full_blocks
    _, Fd, gd, _ = cfg2_full
    assert ok and np.all(status == 0)
    assert np.all(np.isfinite(F)) and np.all(np.isfinite(g))
    assert np.all((F > 0.0) & (F < 1.0))
    assert np.max(np.abs(F - Fd) / np.abs(Fd)) <= 1e-11
    rel = np.linalg.norm((g - gd).reshape(len(g), -1), axis=1) / np.linalg.norm(gd.reshape(len(gd), -1), axis=1)
    assert np.max(rel) <= 1e-9


def test_cfg3_blocks_full_horizon_bit_identity_and_dense_agreement(cfg3_full, qal, torch_cuda):
    """N = 2^20 on the packed block path (bench.py --config cfg3): the time-sharded product is
    bit-identical across G = 1, 2, 4, 8 (A16) and its unpacked Lambda equals the dense one."""
    torch = torch_cuda
    from paper_2511_13330_b200 import driver
    p, L0, Lc, Lcomm, u = cfg3_full
    plan = qal.qal_block_plan_build(torch.cat([L0, Lc, Lcomm.reshape(-1, 64, 64)]), mirror=True)
    L0p, Lcp, Lcommp = (qal.qal_block_pack(plan, m, check=True)[0] for m in (L0, Lc, Lcomm))
    N = p.N
    lam = {}
    for G in (1, 2, 4, 8):
        parts = []
        for r in range(G):
            k0, k1 = driver.shard_range(N, G, r)
            parts.append(driver.local_partial(L0p, Lcp, Lcommp, u[k0:k1].unsqueeze(0).contiguous(), p.T, N, k0,
                                              ctrl_mode=1, plan=plan))
        lam[G] = driver.ordered_combine(torch.stack(parts), plan=plan)
    for G in (2, 4, 8):
        assert torch.equal(lam[G], lam[1]), G
    Lam_b = qal.qal_block_unpack(plan, lam[1].unsqueeze(0))[0].cpu().numpy()
    Lam_d = driver.ordered_combine(torch.stack([driver.local_partial(L0, Lc, Lcomm, u.unsqueeze(0).contiguous(),
                                                                     p.T, N, 0, ctrl_mode=1)])).cpu().numpy()
    assert relfro(Lam_b, Lam_d) <= 1e-10
