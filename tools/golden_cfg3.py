#!/usr/bin/env python
"""Write the configs[3] golden (tests/golden/cfg3_*): the full-horizon propagator of BASELINE
configs[3] computed by the ORACLE ONLY (oracle.sines_nodes -> oracle.propagate in NODES mode,
Magnus-4, sequential left fold from Lambda = I, O3-O6), and its fidelity.

Citations: Eq. 13-15 (the product of Eq. 15 by its definition, a sequential fold),
A11 (sinusoid controls at the Gauss-Legendre nodes), A8 (fidelity).  Nothing here touches the
CUDA path.  Run time: ~20-40 min on 8 host cores (2^20 slices, ~13 64x64 products each).

usage: python tools/golden_cfg3.py [--N 1048576] [--out tests/golden]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2511_13330_b200 import inputs as qi  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1 << 20)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    args = ap.parse_args()
    p = qi.cfg3()
    N, T = args.N, p.T * args.N / p.N
    oracle.build()
    L0, Lc = oracle.build_liouvillian(p.H0[0], p.Hc, p.C)
    u = oracle.sines_nodes(p.sines, p.u_max, N, T)                     # [N][2][J] at the GL nodes
    t0 = time.perf_counter()
    Lam = oracle.propagate(L0, Lc, u, T, N, mode=1, order=4)
    dt = time.perf_counter() - t0
    F = oracle.fidelity(Lam, p.V)
    tag = "cfg3" if N == p.N else f"cfg3_N{N}"
    np.save(os.path.join(args.out, f"{tag}_lambda.npy"), Lam)
    vecI = np.eye(8).reshape(-1, order="F")
    meta = {"what": "configs[3] full-horizon propagator by the oracle (sequential left fold, Magnus-4, NODES)",
            "written_by": "tools/golden_cfg3.py (calls only oracle/ and the seeded input generator)",
            "cite": "P:125-141 (Eqs. 13-15), A8, A11",
            "N": N, "T_ns": T, "seed": 3, "order": 4,
            "F": F, "sha256_u_nodes": sha(u), "sha256_sines": sha(p.sines), "sha256_V": sha(p.V),
            "sha256_lambda": sha(Lam),
            "trace_preservation_err": float(np.max(np.abs(vecI @ Lam - vecI))),
            "oracle_seconds": dt, "omp_threads": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))}
    with open(os.path.join(args.out, f"{tag}_meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
