#!/usr/bin/env python
"""Race / bounds stress in place of compute-sanitizer (closed on this GPU pool): runs the every-kernel
workload of tools/sanitize_run.py with the default libqal.so and with experiment builds
  jitter  (-DQAL_RACE_JITTER: random per-warp delays before every image access / product / TMEM access)
  checked (-DQAL_CHECKED: device asserts on shared-memory regions and item indices)
and requires every output of every run to equal the default build's BIT FOR BIT (all reductions in the
library have a fixed order, so any hazard that the delays expose changes the result).
usage (GPU box): python tools/stress_check.py OUTDIR [--runs 3]   (outputs in /tmp, logs + report in OUTDIR)"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(lib, out, log):
    env = dict(os.environ)
    if lib:
        env["QAL_LIB"] = lib
    with open(log, "w") as f:
        rc = subprocess.call([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "--save", out],
                             stdout=f, stderr=subprocess.STDOUT, env=env, cwd=ROOT)
    return rc


def main():
    outdir = sys.argv[1]
    runs = int(sys.argv[sys.argv.index("--runs") + 1]) if "--runs" in sys.argv else 3
    os.makedirs(outdir, exist_ok=True)
    var = os.path.join(ROOT, "paper_2511_13330_b200", "variants")
    tmp = "/tmp/qal_stress"
    os.makedirs(tmp, exist_ok=True)
    ref = os.path.join(tmp, "default.npz")
    assert run(None, ref, os.path.join(outdir, "default.log")) == 0
    R = np.load(ref)
    report = []
    ok = True
    for name in ["jitter", "checked"]:
        lib = os.path.join(var, f"libqal_{name}.so")
        for i in range(runs if name == "jitter" else 1):
            out = os.path.join(tmp, f"{name}_{i}.npz")
            rc = run(lib, out, os.path.join(outdir, f"{name}_{i}.log"))
            if rc != 0:
                report.append(f"{name} run {i}: exit {rc}")
                ok = False
                continue
            X = np.load(out)
            diff = [k for k in R.files if not np.array_equal(R[k], X[k], equal_nan=True)]
            report.append(f"{name} run {i}: {len(R.files)} outputs, {len(diff)} differ {diff}")
            ok = ok and not diff
    report.append("STRESS OK" if ok else "STRESS FAILED")
    print("\n".join(report))
    with open(os.path.join(outdir, "report.txt"), "w") as f:
        f.write("\n".join(report) + "\n")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
