#!/usr/bin/env python
"""bench.py -- Magnus slices/s of the Qalibrate hot path on B200 (BASELINE.json metric).

Default workload (one "step" = every SURVEY 8(a) row once over one batch):
  configs[2]: 4096 pulses x 1024 PWC slices (T = 200 ns, d = 8, n = 64, complex128), quasistatic
  Zeeman offsets per pulse; a2 Liouvillian build, a3-a5 Magnus-4 expm + ordered product, a6 fidelity,
  a7 gradient w.r.t. all 2 x 1024 controls of every pulse.  As BASELINE configs[2] says, the fixed
  4096-pulse batch is sharded by pulse over the N GPUs (4096/N per rank, strong scaling) and every
  step ends with the all-gather of F[4096] and grad[4096][1024][2] (NCCL) inside the
  timed region.  value = 4096 x 1024 slices per step / the max over ranks of the step time.
  (--weak: 4096 pulses PER GPU, no gather -- an extra measurement, not the headline.)

Launch: python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config ...]
  N > 1 without a torchrun environment: bench.py starts the N ranks itself
  (python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ...).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Magnus slices/s (c128 64×64 expm+product) and % FP64 roofline at 1/2/4/8 GPU"
UNIT = "slices/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pulses", type=int, default=4096,
                    help="configs[2] batch: pulses of the whole job, split over the ranks (--weak: per rank)")
    ap.add_argument("--weak", action="store_true", help="weak scaling: --pulses per rank, no result gather")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)   # launch-path test (gloo, CPU)
    ap.add_argument("--slices", type=int, default=1024)
    ap.add_argument("--sub-batch", type=int, default=None,
                    help="pulses per library call (default: dense 296, blocks sized to ~80 GB of workspace)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-slices", type=int, default=1024)
    ap.add_argument("--cpu-sample-pulses", type=int, default=3,
                    help="pulses in the cpu_baseline sample of our arm (~5 s of oracle work each)")
    ap.add_argument("--cfg4-slices", type=int, default=None,
                    help="slices per step of the cfg4 / hubbard3 sample (default: dense 8, blocks 64)")
    ap.add_argument("--structure", default="blocks", choices=["blocks", "dense"],
                    help="cfg2 path: coherence-block (default, SURVEY 8(f) row 4) or dense 64x64")
    ap.add_argument("--no-dense-ref", action="store_true",
                    help="skip the dense-path reference measurement that accompanies the block path")
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg3grad", "cfg4", "hubbard3"],
                    help="cfg2: batch fwd+grad (default, pulse-sharded); cfg3: 2^20-slice horizon, time-sharded")
    ap.add_argument("--cfg4-full", action="store_true",
                    help="configs[4] at full size: all 32 pulses x 512 slices per step, split over the ranks")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args):
    """--gpus N > 1 without a torchrun environment: start the N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and return their exit status (rank 0 prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Dist:
    """The process group of the run (NCCL on GPUs, gloo for the CPU launch-path test), barriers and the
    max-over-ranks step time."""

    def __init__(self, backend):
        import torch.distributed as dist
        self.dist = dist
        self.world, self.rank, self.local = dist_env()
        if self.world > 1:
            dist.init_process_group(backend, init_method="env://")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x, device):
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=device)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.item()

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle (CPU) leg
def oracle_sample(prob, n_sample, pulses=1, threads=None):
    """The oracle as it stands (O1-O7: forward + per-direction gradient) on the first n_sample
    slices of pulses 0..pulses-1 (each with its own drift) with the workload's slice width, on
    `threads` OpenMP threads (default: every host core -- torchrun's OMP_NUM_THREADS=1 does not
    apply to this leg); returns (slices/s, seconds, threads)."""
    import oracle
    threads = threads or os.cpu_count() or 1
    oracle.set_threads(threads)
    h = prob.T / prob.N
    t0 = time.perf_counter()
    for p in range(pulses):
        L0, Lc = oracle.build_liouvillian(prob.H0[p], prob.Hc, prob.C)
        oracle.gradient(L0, Lc, prob.u[p, :n_sample], h * n_sample, n_sample, prob.V)
    dt = time.perf_counter() - t0
    return pulses * n_sample / dt, dt, threads


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(args, prob):
    """The oracle as it stands on the host cores of this box: all cores (OpenMP over the gradient
    directions) on a few pulses, and one thread (the sequential definition) on a shorter sample."""
    import oracle
    oracle.build()
    npl = max(1, min(args.cpu_sample_pulses, prob.u.shape[0]))
    v, dt, threads = oracle_sample(prob, args.cpu_sample_slices, npl)
    out = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
           "sample": f"oracle forward + gradient on slices 0..{args.cpu_sample_slices - 1} of pulses 0..{npl - 1} "
                     f"of this workload ({dt:.1f} s), OpenMP over gradient directions",
           "cpu_model": cpu_model(), "host_cores": os.cpu_count()}
    ns1 = max(1, args.cpu_sample_slices // 8)
    v1, dt1, _ = oracle_sample(prob, ns1, 1, threads=1)
    out["single_thread"] = {"value": v1, "unit": UNIT, "cores": 1,
                            "sample": f"oracle forward + gradient on slices 0..{ns1 - 1} of pulse 0 ({dt1:.1f} s), "
                                      "one thread (the sequential definition)"}
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from paper_2511_13330_b200 import inputs as qi
    oracle.build()
    prob = qi.cfg2(batch=1, N=args.slices, T=200.0 * args.slices / 1024)
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt, threads = oracle_sample(prob, args.cpu_sample_slices)
        if i >= args.warmup:
            vals.append((v, dt))
    value = statistics.median(v for v, _ in vals)
    sample = (f"oracle (O1-O7, sequential C, OpenMP over gradient directions) on slices 0..{args.cpu_sample_slices - 1}"
              f" of pulse 0 of configs[2] (h = 200/1024 ns), forward + gradient, per step; host CPU {cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(d for _, d in vals),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "configs[2] bounded sample (oracle)", "slices_per_step": args.cpu_sample_slices},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our leg
def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def roofline_of(stages, prods, steps, peak_tf, units_per_launch):
    """Roofline of the dominant kernel (largest device time in the profiling window), the per-stage
    split and the algorithmic flops per step.  Block stages count flops (8 s^3 per block product),
    dense stages count 64x64 products (qal.FLOP_STAGES, driver.stage_flops).  Every stage's flops are
    those of the launches its time covers: the fused block forward counts its fold products apart
    (blk_fold, no launches of its own; they belong to blk_expm_fold's time), and the split forward's
    concurrent prefix + suffix chains are one timing record (blk_prefix_chain) with both chains' flops."""
    from paper_2511_13330_b200 import driver, qal
    fl = {s: driver.stage_flops(prods[i], s) for i, s in enumerate(qal.STAGES)}
    fl["blk_expm_fold"] += fl.pop("blk_fold")
    stages = {s: v for s, v in stages.items() if s != "blk_fold"}
    dom = max(stages, key=lambda s: stages[s][0])
    dom_ms, dom_launch = stages[dom]
    dom_flops_per_launch = fl[dom] / max(dom_launch, 1)
    achieved = dom_flops_per_launch / (dom_ms / max(dom_launch, 1) * 1e-3) / 1e12
    tr = load_traffic().get(qal.KERNELS[dom])
    traffic = (tr["dram_bytes_per_unit"] * units_per_launch) if (tr and units_per_launch) else None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf, "traffic": traffic, "kernel": qal.KERNELS[dom],
                "peak_source": "measured FP64 DMMA.8x8x4 peak (K0 probe, this run, this GPU); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "flops_per_launch": dom_flops_per_launch, "ms_per_launch": dom_ms / max(dom_launch, 1)}
    step_flops = sum(driver.stage_flops(prods[i], s) for i, s in enumerate(qal.STAGES)) / steps
    split = {s: {"ms_per_step": v[0] / steps, "launches_per_step": v[1] / steps,
                 "flops_per_step": fl[s] / steps,
                 "tflops": (fl[s] / (v[0] * 1e-3) / 1e12) if v[0] > 0 else None}
             for s, v in stages.items() if v[1] > 0}
    return roofline, split, step_flops


def fig2_split(qal, stages, prods, steps):
    """The Fig. 2 analog (matrix exponentials vs the ordered multiplication): algorithmic
    flops and device time per step of the slice expansions (Eq. 14: the persistent expm kernel) and of the
    products (Eq. 15: the prefix fold and the suffix chain, two concurrent chains timed as one launch).
    (Paths with the fused chunk forward apportion that kernel's time by its two flop counts.)"""
    ix = qal.STAGES.index
    f_exp, f_fold = prods[ix("blk_expm_fold")], prods[ix("blk_fold")]
    f_chains = prods[ix("blk_prefix_chain")] + prods[ix("blk_suffix_chain")]
    t_fwd = stages["blk_expm_fold"][0]
    # the fused kernel's time apportioned by its two flop counts (expansions vs the fold products), the
    # chain kernels (split prefix + suffix, per-group suffix) wholly products
    t_exp = t_fwd * f_exp / max(f_exp + f_fold, 1)
    t_mul = t_fwd - t_exp + stages["blk_prefix_chain"][0] + stages["blk_suffix_chain"][0]
    note = ("expansions: the expm work of the forward kernels; products: the fused fold (time apportioned by "
            "flops), the prefix and suffix chains")
    return {"expansion": {"flops_per_step": f_exp / steps, "ms_per_step": t_exp / steps},
            "multiplication": {"flops_per_step": (f_fold + f_chains) / steps, "ms_per_step": t_mul / steps},
            "note": note + "; the gradient stage (dual expansion + products) is reported apart in stage_split"}


def dense_reference(args, driver, qal, torch, H0, Hc, C, u, V, T, B, N, world, peak_tf, barrier):
    """The dense 64x64 path on the same pulses (1 warm-up + 1 timed step): slices/s and the roofline of
    its dominant kernel, reported beside the block path so both numbers come from one run."""
    eng = driver.PulseBatch(H0, Hc, C, u, V, T, sub_batch=296, structure="dense")
    eng.step()
    torch.cuda.synchronize()
    counters = torch.zeros(len(qal.STAGES), dtype=torch.int64, device=u.device)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    qal.qal_profile_begin(counters)
    ev0.record()
    F, g = eng.step()
    ev1.record()
    torch.cuda.synchronize()
    stages = qal.qal_profile_end()
    ms = ev0.elapsed_time(ev1)
    roof, split, flops = roofline_of(stages, counters.cpu().tolist(), 1, peak_tf, eng.sub * N)
    out = {"value": world * B * N / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
           "pct_fp64_roofline": flops / (ms * 1e-3) / 1e12 / peak_tf, "roofline": roof,
           "steps": 1, "warmup": 1, "note": "dense 64x64 superoperators (every SURVEY 8(a) row), same pulses"}
    del eng
    torch.cuda.empty_cache()
    return out


class StubBatch:
    """Launch-path test only (--stub, gloo on CPU): the PulseBatch interface with a trivial step whose
    result identifies the global pulse, F[b] = first + b, grad[b][k][j] = (first + b) + k / N."""

    def __init__(self, B, N, J, first):
        import torch
        self.B, self.N, self.J, self.first = B, N, J, first
        self.F = torch.empty(B, dtype=torch.float64)
        self.grad = torch.empty((B, N, J), dtype=torch.float64)
        self.launches = 0
        self.sub = B

    def step(self):
        import torch
        idx = torch.arange(self.first, self.first + self.B, dtype=torch.float64)
        self.F.copy_(idx)
        self.grad.copy_(idx[:, None, None] + torch.arange(self.N, dtype=torch.float64)[None, :, None] / self.N)
        return self.F, self.grad


def run_ours(args):
    """configs[2]: the fixed batch sharded by pulse over the ranks (strong scaling), one step = the whole
    hot path on the rank's pulses + the C2 all-gather of F and grad."""
    import numpy as np
    import torch

    stub = args.stub
    D = Dist("gloo" if stub else "nccl")
    world, rank, local = D.world, D.rank, D.local
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}")
    from paper_2511_13330_b200 import driver
    B_total, N = args.pulses, args.slices
    T = 200.0 * N / 1024
    if args.weak:
        B, first = B_total, rank * B_total                          # every rank its own 4096 pulses
    else:
        first, hi = driver.shard_range(B_total, world, rank)       # rank owns pulses [first, hi)
        B = hi - first
    if stub:
        dev = torch.device("cpu")
        eng = StubBatch(B, N, 2, first)
        peak_tf = None
    else:
        from paper_2511_13330_b200 import _build, inputs as qi, qal
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        _build.build()
        qal.load()
        prob = qi.cfg2(batch=B, N=N, T=T, first_pulse=first)      # the global pulses [first, first + B)
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        H0, Hc, C, u, V = to(prob.H0), to(prob.Hc), to(prob.C), to(prob.u), to(prob.V)
        sub = args.sub_batch if args.sub_batch else (296 if args.structure == "dense" else None)
        eng = driver.PulseBatch(H0, Hc, C, u, V, T, sub_batch=sub, structure=args.structure)
        sink = torch.zeros(1, dtype=torch.float64, device=dev)
        peak_tf = driver.fp64_peak(sink, blocks=2 * torch.cuda.get_device_properties(dev).multi_processor_count)
    gather = not args.weak

    def step():
        F, g = eng.step()
        if gather:
            F, g = driver.gather_results(F, g)                   # C2: whole batch on every rank
        return F, g

    def sync():
        if not stub:
            torch.cuda.synchronize()

    class Timer:
        def __init__(self):
            if stub:
                self.t0 = self.t1 = 0.0
            else:
                self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def start(self):
            if stub:
                self.t0 = time.perf_counter()
            else:
                self.e0.record()

        def stop(self):
            if stub:
                self.t1 = time.perf_counter()
            else:
                self.e1.record()

        def ms(self):
            return (self.t1 - self.t0) * 1e3 if stub else self.e0.elapsed_time(self.e1)

    for _ in range(args.warmup):
        Fg, gg = step()
    sync()

    # ---------------- timed region: device-resident inputs; every step ends with the result gather
    counters = None
    clocks = None
    if not stub:
        from paper_2511_13330_b200 import qal
        counters = torch.zeros(len(qal.STAGES), dtype=torch.int64, device=dev)
        clocks = ClockSampler(local)
        clocks.start()
    D.barrier()
    sync()
    tm = Timer()
    if not stub:
        qal.qal_profile_begin(counters)
    tm.start()
    launches = 0
    for _ in range(args.steps):
        Fg, gg = step()
        launches += eng.launches
    tm.stop()
    sync()
    stages = qal.qal_profile_end() if not stub else None
    D.barrier()
    clk = clocks.stop() if clocks else None
    ms_max = D.max(tm.ms(), dev)
    slices_total = (world * B if args.weak else B_total) * N * args.steps
    value = slices_total / (ms_max * 1e-3)
    gathered_ok = None
    if gather:
        Fh = Fg.cpu()
        gathered_ok = bool(Fg.shape[0] == B_total and gg.shape[0] == B_total)
        if stub:
            gathered_ok = gathered_ok and bool(torch.equal(Fh, torch.arange(B_total, dtype=torch.float64)))
    if stub:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                              "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                              "scaling": "weak" if args.weak else "strong", "pulses_per_rank": B,
                              "gathered_ok": gathered_ok, "stub": True}), flush=True)
        D.close()
        return 0

    # ---------------- e2e: host (pinned) inputs -> device -> host results, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hu = torch.from_numpy(prob.u).pin_memory()
        hH0 = torch.from_numpy(prob.H0).pin_memory()
        nres = B_total if gather else B
        hF = torch.empty(nres, dtype=torch.float64).pin_memory()
        hg = torch.empty((nres,) + tuple(prob.u.shape[1:]), dtype=torch.float64).pin_memory()
        pipelined = world == 1 or not gather
        if pipelined:
            for _ in range(args.warmup):   # untimed, like the device-resident warm-up (copy streams, events)
                eng.step_host(hH0, hu, hF, hg)
            eng.synchronize_host()
        D.barrier()
        sync()
        tm.start()
        for _ in range(args.steps):
            if pipelined:   # the public end-to-end call: copies on two streams, overlapped with the compute
                eng.step_host(hH0, hu, hF, hg)
            else:           # ranks > 1: the gathered results are copied out after the exchange
                eng.u.copy_(hu, non_blocking=True)
                eng.H0.copy_(hH0, non_blocking=True)
                F2, g2 = step()
                hF.copy_(F2, non_blocking=True)
                hg.copy_(g2, non_blocking=True)
        if pipelined:
            eng.host_fence()   # the timed region ends after the last step's results are in host memory
        tm.stop()
        sync()
        t2 = D.max(tm.ms(), dev)
        e2e = {"value": slices_total / (t2 * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(hu.numel() * 8 + hH0.numel() * 16),
               "d2h_bytes_per_step": int(hF.numel() * 8 + hg.numel() * 8),
               "copies": ("PulseBatch.step_host: per-sub-batch H2D / D2H on two copy streams overlapped with the "
                          "compute (step s + 1's inputs stream in under step s)" if pipelined else
                          "serial H2D before / D2H after each step")}

    # ---------------- roofline of the dominant kernel (largest device time in the window)
    prods = counters.cpu().tolist()
    roofline, split, step_flops = roofline_of(stages, prods, args.steps, peak_tf, eng.sub * N)
    fig2 = fig2_split(qal, stages, prods, args.steps) if args.structure == "blocks" else None
    structure_ok = eng.structure_ok()
    status_ok = bool((eng.status == 0).all().item())

    # ---------------- the dense 64x64 path on the same workload (context for the block path)
    dense_ref = None
    if args.structure == "blocks" and not args.no_dense_ref:
        dense_ref = dense_reference(args, driver, qal, torch, H0, Hc, C, u, V, T, B, N, world, peak_tf, D.barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, prob)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": f"configs[2]: {B_total if not args.weak else world * B} pulses x {N} PWC "
                                       f"slices, T={T:g} ns, d=8 (64x64 c128 superoperators), forward + fidelity "
                                       "+ gradient" + ("" if args.weak else ", all-gather of F and grad per step"),
                           "structure": (f"coherence blocks (detected {eng.plan.n_components} components; "
                                         f"stored widths {[eng.plan.width[g] for g in range(eng.plan.ngroups)]}, "
                                         "Hermitian mirror), identical 64x64 results"
                                         if args.structure == "blocks" else "dense 64x64"),
                           "pulses_per_gpu": B, "slices": N, "sub_batch": eng.sub,
                           "l2": f"inputs larger than L2 (gradient workspace {eng.ws_bytes / 2**30:.1f} GiB)",
                           "parallelism": f"batch-sharded x{world}" + (" (weak)" if args.weak else "")},
                "pulses_per_s": slices_total / N / (ms_max * 1e-3),
                "pct_fp64_roofline": step_flops / (ms_max / args.steps * 1e-3) / 1e12 / peak_tf,
                "fp64_peak_tflops": peak_tf, "roofline": roofline, "stage_split": split, "fig2_split": fig2,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
                "structure_check": "ok" if structure_ok else "FAILED", "status_ok": status_ok,
                "result_gather": ("all_gather_into_tensor (NCCL) of F and grad, every step" if world > 1 and gather
                                  else ("single rank: results already whole" if gather else "none (weak)")),
                "dense_path": dense_ref, "gpu": torch.cuda.get_device_name(dev)}
        print(json.dumps(line), flush=True)
    D.close()
    return 0


def run_cfg3grad(args):
    """NEXT f2: fidelity gradient over the configs[3] horizon (2^20 NODES slices), time-sharded over
    the ranks and segmented (2^16 slices) on each: slices/s of the whole forward + gradient."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_13330_b200 import _build, driver, inputs as qi, qal

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _build.build()
    qal.load()
    prob = qi.cfg3()
    N, T = prob.N, prob.T
    k0, k1 = driver.shard_range(N, world, rank)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    H0, Hc, C, V, prm = to(prob.H0), to(prob.Hc), to(prob.C), to(prob.V), to(prob.sines)
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    peak_tf = driver.fp64_peak(sink, blocks=2 * torch.cuda.get_device_properties(dev).multi_processor_count)

    plan = None
    if args.structure == "blocks":
        L0, Lc, Lcomm = qal.qal_build_liouvillian(H0, Hc, C, want_comm=True)
        plan = qal.qal_block_plan_build(torch.cat([L0, Lc, Lcomm.reshape(-1, 64, 64)]), mirror=True)

    def step():
        u = qal.qal_sample_controls_sines(prm, prob.u_max, N, T, k0, k1 - k0).unsqueeze(0).contiguous()
        L0, Lc, Lcomm = qal.qal_build_liouvillian(H0, Hc, C, want_comm=True)
        if plan is not None:
            mats = [qal.qal_block_pack(plan, m, check=True)[0] for m in (L0, Lc, Lcomm)]
            return driver.time_sharded_gradient(*mats, u, T, N, k0, ctrl_mode=qal.QAL_CTRL_NODES, plan=plan,
                                                group_subsegments=8192,
                                                cotangent=lambda Lm: qal.qal_block_fidelity_cotangent(plan, V))
        return driver.time_sharded_gradient(L0, Lc, Lcomm, u, T, N, k0, ctrl_mode=qal.QAL_CTRL_NODES,
                                            cotangent=lambda Lm: qal.qal_fidelity_cotangent(V))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    counters = torch.zeros(len(qal.STAGES), dtype=torch.int64, device=dev)
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    qal.qal_profile_begin(counters)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    stages = qal.qal_profile_end()
    clk = clocks.stop()
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    prods = counters.cpu().tolist()
    if rank == 0:
        flops = sum(driver.stage_flops(x, st) for x, st in zip(prods, qal.STAGES)) / args.steps
        roofline, split, _ = roofline_of(stages, prods, args.steps, peak_tf, None)
        line = {"metric": METRIC, "value": N * args.steps / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": "configs[3] gradient (NEXT f2): 2^20 NODES slices, fidelity gradient w.r.t. "
                                       "all 2 x 2 x 2^20 node values, time-sharded; 64-slice sub-segments, log-depth prefix/suffix "
                                       "scans, one batched VJP",
                           "structure": "coherence blocks (packed)" if plan is not None else "dense 64x64"},
                "pct_fp64_roofline": flops / (ms / args.steps * 1e-3) / 1e12 / peak_tf,
                "roofline": roofline, "stage_split": split,
                "stage_ms_per_step": {k: v[0] / args.steps for k, v in stages.items() if v[1]},
                "fp64_peak_tflops": peak_tf, "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_cfg3(args):
    """configs[3]: one pulse, N = 2^20 NODES slices over 10 us, time-sharded over the ranks
    (strong scaling): a1 device sampler -> a2 basis (+ commutators) -> a3-a5 local chunk fold +
    tree -> all-gather of the G partials -> ordered combine -> a6 fidelity."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_13330_b200 import _build, driver, inputs as qi, qal

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _build.build()
    qal.load()
    prob = qi.cfg3()
    N, T = prob.N, prob.T
    k0, k1 = driver.shard_range(N, world, rank)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    H0, Hc, C, V, prm = to(prob.H0), to(prob.Hc), to(prob.C), to(prob.V), to(prob.sines)
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    peak_tf = driver.fp64_peak(sink, blocks=2 * torch.cuda.get_device_properties(dev).multi_processor_count)

    state = {}
    plan = None
    if args.structure == "blocks":
        L0, Lc, Lcomm = qal.qal_build_liouvillian(H0, Hc, C, want_comm=True)
        plan = qal.qal_block_plan_build(torch.cat([L0, Lc, Lcomm.reshape(-1, 64, 64)]), mirror=True)
        state["flag"] = torch.zeros(1, dtype=torch.int32, device=dev)

    def step():
        u = qal.qal_sample_controls_sines(prm, prob.u_max, N, T, k0, k1 - k0)
        L0, Lc, Lcomm = qal.qal_build_liouvillian(H0, Hc, C, want_comm=True)
        if plan is not None:
            mats = [qal.qal_block_pack(plan, m, check=True)[0] for m in (L0, Lc, Lcomm)]
            Lam = driver.time_shard_propagator(*mats, u.unsqueeze(0), T, N, k0, ctrl_mode=qal.QAL_CTRL_NODES,
                                               plan=plan)
            state["F"] = qal.qal_block_fidelity(plan, Lam.unsqueeze(0), V)
        else:
            Lam = driver.time_shard_propagator(L0, Lc, Lcomm, u.unsqueeze(0), T, N, k0,
                                               ctrl_mode=qal.QAL_CTRL_NODES)
            state["F"] = qal.qal_fidelity(Lam.unsqueeze(0), V)
        state["Lam"] = Lam

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    counters = torch.zeros(len(qal.STAGES), dtype=torch.int64, device=dev)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    qal.qal_profile_begin(counters)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    stages = qal.qal_profile_end()
    barrier()
    clk = clocks.stop()
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = t.item()
    prods = counters.cpu().tolist()
    value = N * args.steps / (ms_max * 1e-3)
    roofline, split, step_flops = roofline_of(stages, prods, args.steps, peak_tf, None)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "configs[3]: 1 pulse, N=2^20 Magnus-4 NODES slices over 10 us, "
                                       "time-sharded, all-gather of G partials + ordered combine",
                           "slices": N, "chunk": driver.time_shard_chunk(N), "parallelism": f"time-sharded x{world}",
                           "structure": ("coherence blocks (Hermitian mirror), packed partials"
                                         if plan is not None else "dense 64x64"),
                           "l2": "chunk partials larger than L2 (dense 1 GiB, blocks 235 MB)"},
                "pct_fp64_roofline": step_flops / (ms_max / args.steps * 1e-3) / 1e12 / peak_tf,
                "fp64_peak_tflops": peak_tf, "roofline": roofline, "stage_split": split,
                "F": state["F"].item(), "clocks": clk, "gpu": torch.cuda.get_device_name(dev)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_cfg4(args):
    """configs[4]: d = 64 (n = 4096), PWC, 32 pulses sharded by pulse over the ranks (rank r owns pulses
    [r 32/G, (r+1) 32/G)); a step = for every owned pulse the expm + fold of its first S slices and the
    fidelity, then the all-gather of F[32].  --cfg4-full: S = 512, the whole config;
    otherwise S = --cfg4-slices (a bounded sample of every pulse, F of the truncated pulse)."""
    import numpy as np
    import torch

    from paper_2511_13330_b200 import _build, driver, inputs as qi, qal

    D = Dist("nccl")
    world, rank, local = D.world, D.rank, D.local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _build.build()
    qal.load()
    prob = qi.hubbard3() if args.config == "hubbard3" else qi.cfg4()
    P_total = prob.u.shape[0]
    S = prob.N if args.cfg4_full else (args.cfg4_slices or (64 if args.structure == "blocks" else 8))
    if args.structure == "dense" and not args.cfg4_full:
        P_total = min(P_total, max(world, 4))                   # dense sample: a few pulses only
    p0, p1 = driver.shard_range(P_total, world, rank)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    L0, Lc, _ = qal.qal_build_liouvillian(to(prob.H0), to(prob.Hc), to(prob.C))
    u_all = to(prob.u[p0:p1, :S])
    V = to(prob.V)
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    peak_tf = driver.fp64_peak(sink, blocks=2 * torch.cuda.get_device_properties(dev).multi_processor_count)
    n = 4096
    ws = torch.empty(qal.workspace_bytes(qal.QAL_OP_EXPM_SLICES, n, 1, S), dtype=torch.uint8, device=dev)
    P = torch.empty((1, 1, n, n), dtype=torch.complex128, device=dev)
    F = torch.empty(p1 - p0, dtype=torch.float64, device=dev)
    fws = torch.empty(qal.workspace_bytes(qal.QAL_OP_FIDELITY_REDUCE, n, 1, 1), dtype=torch.uint8, device=dev)
    lib = qal.load()
    st = lambda: qal._stream(None)  # noqa: E731

    plan = None
    if args.structure == "blocks":
        plan = qal.qal_bigblock_plan_build(torch.cat([L0[:1], Lc]), mirror=True)
        ws = torch.empty(lib.qal_bigblock_workspace_bytes(ctypes.byref(plan)), dtype=torch.uint8, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)

    def step():
        for i in range(p1 - p0):
            u = u_all[i]
            if plan is not None:
                rc = lib.qal_bigblock_expm_slices(ctypes.byref(plan), prob.N, prob.T, S, prob.J, qal._ptr(u),
                                                  qal._ptr(L0), qal._ptr(Lc), S, qal._ptr(P), None, qal._ptr(flag),
                                                  qal._ptr(ws), ws.numel(), st())
                qal._check(rc, "qal_bigblock_expm_slices")
            else:
                rc = lib.qal_magnus_expm_slices(n, 1, prob.N, prob.T, 0, S, 4, 0, prob.J, qal._ptr(u), qal._ptr(L0),
                                                0, qal._ptr(Lc), None, 0, None, S, qal._ptr(P), None, qal._ptr(ws),
                                                ws.numel(), st())
                qal._check(rc, "qal_magnus_expm_slices")
            qal._check(lib.qal_fidelity_ws(64, 1, qal._ptr(P), qal._ptr(V), ctypes.c_void_p(F.data_ptr() + 8 * i),
                                           qal._ptr(fws), fws.numel(), st()), "qal_fidelity_ws")
        return driver.gather_results(F)[0]                      # F[32] on every rank

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    counters = torch.zeros(len(qal.STAGES), dtype=torch.int64, device=dev)
    clocks = ClockSampler(local)
    clocks.start()
    D.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    qal.qal_profile_begin(counters)
    ev0.record()
    for _ in range(args.steps):
        Fall = step()
    ev1.record()
    torch.cuda.synchronize()
    stages = qal.qal_profile_end()
    clk = clocks.stop()
    ms_max = D.max(ev0.elapsed_time(ev1), dev)
    gstage = "blk_gemm" if plan is not None else "dense_gemm"
    g_ms, g_l = stages[gstage]
    gcount = counters.cpu().tolist()[qal.STAGES.index(gstage)]
    gflops = driver.stage_flops(gcount, gstage) if plan is not None else gcount * driver.complex_product_flops(n)
    nprod = gcount if plan is None else gflops / plan.flops_per_product   # 4096^2 (block) products executed
    if rank == 0:
        ach = gflops / (g_ms * 1e-3) / 1e12
        full = S == prob.N and P_total == prob.u.shape[0]
        line = {"metric": METRIC, "value": P_total * S * args.steps / (ms_max * 1e-3), "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": (f"{prob.name}{' (full size)' if full else ' sample'}: {P_total} pulses x "
                                        f"first {S} of {prob.N} PWC slices, d=64 (4096x4096 c128), expm + fold + "
                                        "fidelity, pulses sharded over the ranks, all-gather of F"),
                           "slices_per_step": P_total * S, "pulses": P_total, "pulses_per_gpu": p1 - p0},
                "roofline": {"bound": "tensor", "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s",
                             "frac": ach / peak_tf, "traffic": None,
                             "kernel": "k_bb_gemm" if plan is not None else "k_dense_gemm",
                             "ms_per_launch": g_ms / max(g_l, 1)},
                "structure": (f"coherence blocks {plan.sizes()} (mirror), {plan.flops_per_product / (8.0 * n ** 3):.4f}"
                              " of the dense flops" if plan is not None else "dense 4096x4096"),
                "fp64_peak_tflops": peak_tf, "stage_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()
                                                                   if v[1]},
                "products_per_slice": nprod / (P_total // world * S * args.steps),
                "F": Fall.cpu().tolist(), "clocks": clk, "gpu": torch.cuda.get_device_name(dev)}
        print(json.dumps(line), flush=True)
    D.close()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)            # the oracle on the host cores; rank 0 only under torchrun
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)              # one process per GPU, started here
    world = dist_env()[0]
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}")
    if args.config in ("cfg4", "hubbard3"):
        return run_cfg4(args)
    if args.config == "cfg3":
        return run_cfg3(args)
    if args.config == "cfg3grad":
        return run_cfg3grad(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
