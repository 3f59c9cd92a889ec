#!/usr/bin/env python
"""Per-kernel summary of an `ncu --set full` report: time, DMMA pipe, issue, occupancy, shared
wavefronts, DRAM bytes and the warp-stall split.  usage: python tools/ncu_summary.py rep.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

M = {
    "time_ms": "gpu__time_duration.sum",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_inst_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "inst": "smsp__inst_executed.sum",
}
STALLS = ["barrier", "long_scoreboard", "math_pipe_throttle", "mio_throttle", "no_instruction", "selected",
          "short_scoreboard", "wait", "lg_throttle", "dispatch_stall", "branch_resolving", "tex_throttle",
          "membar", "sleeping", "drain", "misc", "not_selected"]


def main():
    rep = sys.argv[1]
    names = list(M.values()) + [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(names)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d["Kernel Name"].split("(")[0]}
        for key, m in M.items():
            try:
                k[key] = float(d.get(m, "nan").replace(",", ""))
            except ValueError:
                k[key] = d.get(m)
        st = {}
        for s in STALLS:
            v = d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
            try:
                st[s] = float(v)
            except (TypeError, ValueError):
                pass
        tot = sum(st.values()) or 1.0
        k["stall_shares_pct"] = {s: round(100 * v / tot, 1) for s, v in sorted(st.items(), key=lambda kv: -kv[1])
                                 if 100 * v / tot >= 1.0}
        res.append(k)
    for k in res:
        print(f"{k['kernel'][:48]:48s} {k['time_ms']:8.3f} ms  dmma {k['dmma_pipe_pct']:5.1f}%  issue "
              f"{k['issue_active_pct']:5.1f}%  warps {k['warps_active_pct']:5.1f}%  smem {k['smem_wavefronts_pct']:5.1f}%"
              f"  regs {k['registers']:.0f}  grid {k['grid']:.0f}x{k['block']:.0f}  {k['stall_shares_pct']}")
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
