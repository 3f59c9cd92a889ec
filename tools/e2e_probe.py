"""Probe of the end-to-end copy schedules on the bench workload (configs[2], one GPU): device-resident
steps, serial copies around each step, PulseBatch.step_host (pipelined), and copies on one side stream
without per-sub-batch overlap.  Prints ms per step of each (CUDA events on the compute stream).
usage: python tools/e2e_probe.py [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_13330_b200 import _build, driver, inputs as qi, qal  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
_build.build()
qal.load()
p = qi.cfg2()
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
eng = driver.PulseBatch(dev(p.H0), dev(p.Hc), dev(p.C), dev(p.u), dev(p.V), p.T, structure="blocks")
hu = torch.from_numpy(p.u).pin_memory()
hH0 = torch.from_numpy(p.H0).pin_memory()
hF = torch.empty(eng.B, dtype=torch.float64).pin_memory()
hg = torch.empty(tuple(p.u.shape), dtype=torch.float64).pin_memory()


def timed(fn, label):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    eng.host_fence()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label:28s} {e0.elapsed_time(e1) / steps:8.2f} ms/step", flush=True)


def serial():
    eng.u.copy_(hu, non_blocking=True)
    eng.H0.copy_(hH0, non_blocking=True)
    F, g = eng.step()
    hF.copy_(F, non_blocking=True)
    hg.copy_(g, non_blocking=True)


def h2d_only():
    eng.u.copy_(hu, non_blocking=True)
    eng.H0.copy_(hH0, non_blocking=True)
    eng.step()


def d2h_only():
    F, g = eng.step()
    hF.copy_(F, non_blocking=True)
    hg.copy_(g, non_blocking=True)


timed(eng.step, "device-resident")
timed(serial, "serial copies")
timed(h2d_only, "serial H2D only")
timed(d2h_only, "serial D2H only")
timed(lambda: eng.step_host(hH0, hu, hF, hg), "step_host (pipelined)")
timed(eng.step, "device-resident again")
t = torch.empty(tuple(p.u.shape), dtype=torch.float64, device="cuda")
for label, fn in (("H2D 67 MB alone", lambda: t.copy_(hu, non_blocking=True)),
                  ("D2H 67 MB alone", lambda: hg.copy_(t, non_blocking=True))):
    timed(fn, label)
