"""Multi-GPU host logic on CPU with torch.distributed (gloo, world size 2):
batch partitioning (cfg2) and the time-sharded all-gather + ordered combine (cfg3),
checked against the oracle's sequential fold with a non-commuting fixture."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_13330_b200 import driver


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions_exactly():
    for total, world in [(4096, 1), (4096, 2), (4096, 8), (1 << 20, 8)]:
        spans = [driver.shard_range(total, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == total
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        driver.shard_range(10, 3, 0)


@pytest.mark.parametrize("N", [256, 1024, 1 << 20, 96, 8])
def test_time_shard_chunk_aligns_with_every_rank_range(N):
    c = driver.time_shard_chunk(N)
    assert N % c == 0 and (c & (c - 1)) == 0 and c <= 64
    for G in (1, 2, 4, 8):
        if N % G == 0 and N // G >= 1:
            # every rank range is a whole number of chunks, so the chunk partials -- and for
            # power-of-two ranges the tree over them -- do not depend on G (A16)
            assert (N // G) % c == 0 or N // G < c


def _worker(rank, world, port, N, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    rng = np.random.default_rng(seed)
    n = 16
    Us = (rng.standard_normal((N, n, n)) + 1j * rng.standard_normal((N, n, n))) / np.sqrt(n)  # non-commuting
    lo, hi = driver.shard_range(N, world, rank)
    Q = oracle.ordered_product(Us[lo:hi])                       # this rank's partial (later on the left)
    parts = driver.gather_partials(torch.from_numpy(Q))
    assert parts.shape == (world, n, n)
    Lam = driver.ordered_combine(parts, product=lambda P: torch.from_numpy(oracle.ordered_product(P.numpy())))
    ref = oracle.ordered_product(Us)
    wrong = oracle.ordered_product(Us[::-1].copy())
    err = float(np.linalg.norm(Lam.numpy() - ref) / np.linalg.norm(ref))
    err_wrong = float(np.linalg.norm(Lam.numpy() - wrong) / np.linalg.norm(ref))
    q.put((rank, err, err_wrong, parts[rank].numpy().tobytes() == Q.tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_time_sharded_gather_and_ordered_combine_gloo(world, oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 8, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, err_wrong, own in res:
        assert err <= 1e-13, (rank, err)
        assert err_wrong > 1e-3           # the fixture really detects a wrong order
        assert own                        # gathered slot r is rank r's partial


def _batch_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_13330_b200 import inputs as qi
    B = 4
    p = qi.cfg2(batch=B, N=16, first_pulse=rank * B)
    ref = qi.cfg2(batch=B * world, N=16)
    ok = np.array_equal(p.u, ref.u[rank * B:(rank + 1) * B]) and np.array_equal(p.H0, ref.H0[rank * B:(rank + 1) * B])
    t = torch.tensor([float(ok)])
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    q.put(t.item())
    dist.destroy_process_group()


def test_batch_shards_are_disjoint_slices_of_one_global_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [1.0, 1.0]


@pytest.mark.parametrize("mode", [0, 1])
def test_segment_seed_algebra_reproduces_the_full_horizon_gradient(oracle, mode):
    """NEXT f2: per-segment VJPs with the seeds of driver.segment_seeds (local prefixes, earlier
    segments folded into the suffix seed) equal the oracle's gradient over the whole horizon."""
    from paper_2511_13330_b200 import inputs as qi
    N, S = 12, 3
    if mode == 0:
        p = qi.cfg0(N=N, T=100.0 * N / 256)
        u = p.u[0]
    else:
        p = qi.cfg3()
        u = oracle.sines_nodes(p.sines, p.u_max, N, 60.0)
        p.T = 60.0
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    h = p.T / N
    C = oracle.fidelity_cotangent(p.V)
    g_full, Lam = oracle.vjp(L0, Lc, u, p.T, N, C, mode=mode)
    seg = N // S
    Qs = [oracle.propagate(L0, Lc, u[s * seg:(s + 1) * seg], h * seg, seg, mode=mode) for s in range(S)]
    seeds = driver.segment_seeds(Qs, C, lambda xs: oracle.ordered_product(np.stack(list(xs))))
    g_seg = np.concatenate([oracle.vjp(L0, Lc, u[s * seg:(s + 1) * seg], h * seg, seg, seeds[s], mode=mode)[0]
                            for s in range(S)])
    assert np.allclose(g_seg, g_full, rtol=0, atol=1e-12 * np.abs(g_full).max())
    F = oracle.fidelity(Lam, p.V)
    assert abs(np.trace(C @ Lam).real - F) <= 1e-15           # the cotangent of the fidelity


def _worker_packed(rank, world, port, N, seed, q):
    """Block path (cfg3 with a plan): every rank all-gathers its PACKED partial (the concatenated
    super-block matrices, 1-D); the ordered combine acts block by block."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    widths = [24, 16, 8]
    offs = np.cumsum([0] + [w * w for w in widths])
    rng = np.random.default_rng(seed)
    blocks = [(rng.standard_normal((N, w, w)) + 1j * rng.standard_normal((N, w, w))) / np.sqrt(w) for w in widths]
    lo, hi = driver.shard_range(N, world, rank)
    Q = np.concatenate([oracle.ordered_product(b[lo:hi]).reshape(-1) for b in blocks])   # packed partial
    parts = driver.gather_partials(torch.from_numpy(Q))
    assert parts.shape == (world, offs[-1])

    def blockwise(P):
        P = P.numpy()
        return torch.from_numpy(np.concatenate([
            oracle.ordered_product(P[:, offs[g]:offs[g + 1]].reshape(world, w, w).copy()).reshape(-1)
            for g, w in enumerate(widths)]))

    Lam = driver.ordered_combine(parts, product=blockwise).numpy()
    errs = []
    for g, w in enumerate(widths):
        ref = oracle.ordered_product(blocks[g])
        got = Lam[offs[g]:offs[g + 1]].reshape(w, w)
        errs.append(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
    q.put((rank, max(errs)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_time_sharded_packed_partials_gloo(world):
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_packed, args=(r, world, port, 16, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for _, err in res:
        assert err <= 1e-12


# ---- result gather (cfg2 / cfg4) and the time-sharded gradient's rank seeds (NEXT f2) ----

def _run_world(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B_total, N, J = 12, 5, 2
    lo, hi = driver.shard_range(B_total, world, rank)
    F = torch.arange(lo, hi, dtype=torch.float64) * 0.5
    g = torch.arange(lo * N * J, hi * N * J, dtype=torch.float64).reshape(hi - lo, N, J)
    Fa, ga = driver.gather_results(F, g)
    ok = (torch.equal(Fa, torch.arange(B_total, dtype=torch.float64) * 0.5)
          and torch.equal(ga, torch.arange(B_total * N * J, dtype=torch.float64).reshape(B_total, N, J)))
    Fo, go = driver.gather_results(F)                    # F only (configs[4])
    ok = ok and go is None and torch.equal(Fo, Fa)
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


def test_result_gather_puts_every_rank_shard_in_global_pulse_order():
    assert _run_world(_gather_worker, 2) == [(0, True), (1, True)]


def _seed_worker(rank, world, port, q):
    """rank_seed with the oracle as the product: Re Tr(seed_r E) must equal the directional derivative of
    L(Q_r) = Re Tr(C Q_{G-1} ... Q_0) along E (central difference, exact up to rounding: L is linear)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    oracle.build()
    n = 12
    rng = np.random.default_rng(100 + rank)
    Q = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    ranks = driver.gather_partials(torch.from_numpy(Q))              # [G][n][n], rank order
    crng = np.random.default_rng(7)                                   # the same C on every rank
    C = crng.standard_normal((n, n)) + 1j * crng.standard_normal((n, n))
    combine = lambda P: torch.from_numpy(oracle.ordered_product(np.ascontiguousarray(P.numpy())))  # noqa: E731
    mm = lambda X, Y: torch.from_numpy(oracle.matmul(X.numpy(), Y.numpy()))                          # noqa: E731
    seed = driver.rank_seed(ranks, torch.from_numpy(C), rank, combine, mm).numpy()
    E = np.random.default_rng(200 + rank).standard_normal((n, n)) + 0j

    def loss(Qr):
        parts = ranks.numpy().copy()
        parts[rank] = Qr
        return np.trace(C @ oracle.ordered_product(parts)).real
    eps = 1e-3
    fd = (loss(Q + eps * E) - loss(Q - eps * E)) / (2 * eps)
    an = np.trace(seed @ E).real
    # and a wrong order (seed C B_r A_r) must not pass
    q.put((rank, abs(fd - an) <= 1e-10 * max(1.0, abs(fd)), float(abs(fd))))
    dist.destroy_process_group()


def test_rank_seed_of_the_time_sharded_gradient_gloo():
    res = _run_world(_seed_worker, 2)
    assert [r[:2] for r in res] == [(0, True), (1, True)], res
    assert all(r[2] > 1e-3 for r in res)          # non-trivial derivative


def _seed_worker_vjp(rank, world, port, q):
    """The seeds drive the per-rank VJP: with the oracle's per-direction vjp on each rank's slices and
    C_r = rank_seed(...), the gathered gradient equals the oracle's whole-horizon vjp (the rank > 0 branches
    of driver.time_sharded_gradient, with the oracle as the product)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2511_13330_b200 import inputs as qi
    oracle.build()
    p = qi.cfg0(N=8, T=100.0 * 8 / 256)
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    lo, hi = driver.shard_range(p.N, world, rank)
    # this rank's partial Q_r = U_{hi-1} .. U_lo (oracle.propagate indexes u by absolute slice)
    Q = oracle.propagate(L0, Lc, p.u[0], p.T, p.N, k0=lo, k1=hi)
    ranks = driver.gather_partials(torch.from_numpy(Q))
    crng = np.random.default_rng(9)
    C = (crng.standard_normal((64, 64)) + 1j * crng.standard_normal((64, 64))) / 64
    combine = lambda P: torch.from_numpy(oracle.ordered_product(np.ascontiguousarray(P.numpy())))  # noqa: E731
    mm = lambda X, Y: torch.from_numpy(oracle.matmul(X.numpy(), Y.numpy()))                          # noqa: E731
    Cr = driver.rank_seed(ranks, torch.from_numpy(C), rank, combine, mm).numpy()
    # the rank's VJP on its own slices: a problem whose horizon is [lo, hi)
    h = p.T / p.N
    g_loc, _ = oracle.vjp(L0, Lc, p.u[0, lo:hi], h * (hi - lo), hi - lo, Cr)
    g_all = torch.empty((p.N, p.u.shape[2]), dtype=torch.float64)
    dist.all_gather_into_tensor(g_all.reshape(-1), torch.from_numpy(np.ascontiguousarray(g_loc)).reshape(-1))
    g_ref, _ = oracle.vjp(L0, Lc, p.u[0], p.T, p.N, C)
    err = float(np.linalg.norm(g_all.numpy() - g_ref) / np.linalg.norm(g_ref))
    q.put((rank, err))
    dist.destroy_process_group()


def test_time_sharded_vjp_with_rank_seeds_matches_the_whole_horizon_gloo():
    res = _run_world(_seed_worker_vjp, 2)
    for rank, err in res:
        assert err <= 1e-12, (rank, err)


def _bench_stub(*extra):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--stub", "--steps", "2",
                          "--warmup", "3", "--pulses", "64", "--slices", "8", *extra], capture_output=True, text=True,
                         timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout          # rank 0 alone prints one JSON line
    return json.loads(lines[0])


def test_bench_spawns_its_ranks_and_gathers_the_split_batch():
    """bench.py --gpus 2 with no torchrun environment starts 2 ranks itself (torch.distributed.run,
    127.0.0.1), splits the 64-pulse batch 32/32, gathers F and grad every step (gloo here, NCCL on GPUs)
    in global pulse order, and reports the max-over-ranks time once."""
    line = _bench_stub()
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["pulses_per_rank"] == 32
    assert line["gathered_ok"] is True and line["value"] > 0
    weak = _bench_stub("--weak")
    assert weak["scaling"] == "weak" and weak["pulses_per_rank"] == 64 and weak["gathered_ok"] is None
