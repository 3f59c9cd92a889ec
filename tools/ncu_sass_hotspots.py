#!/usr/bin/env python
"""Summarise `ncu -i rep --page source --csv --print-source sass` output: per kernel, warp-stall samples
by SASS opcode (with the dominant stall reasons) and the hottest instructions.

usage: python tools/ncu_sass_hotspots.py sass.csv [--kernel REGEX] [--top 40]
"""
import argparse
import collections
import csv
import re
import sys


def kernels(path):
    cur, rows, hdr = None, [], None
    with open(path, newline="") as f:
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "Kernel Name":
                if cur is not None:
                    yield cur, hdr, rows
                cur, rows, hdr = row[1], [], None
                continue
            if row[0] == "Address":
                hdr = row
                continue
            if hdr is not None:
                rows.append(row)
    if cur is not None:
        yield cur, hdr, rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--kernel", default=".")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    for name, hdr, rows in kernels(a.csv):
        if not re.search(a.kernel, name):
            continue
        ix = {h: i for i, h in enumerate(hdr)}
        stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tot = 0
        by_op = collections.defaultdict(lambda: collections.Counter())
        n_exec = collections.Counter()
        hot = []
        for r in rows:
            src = r[ix["Source"]].strip()
            op = src.split()[0] if src else "?"
            if op.startswith("@"):
                op = src.split()[1]
            op = op.split(".")[0]
            s = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
            ex = int(float(r[ix["Instructions Executed"]] or 0))
            tot += s
            n_exec[op] += ex
            c = by_op[op]
            c["samples"] += s
            for st in stalls:
                v = r[ix[st]]
                if v and v != "0":
                    c[st] += int(float(v))
            hot.append((s, r[ix["Address"]], src, {st: r[ix[st]] for st in stalls if r[ix[st]] not in ("", "0")}))
        print(f"== {name}\n   samples {tot}, instructions executed {sum(n_exec.values())}")
        for op, c in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:25]:
            top = ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(5) if k != "samples")
            print(f"   {op:12s} {c['samples']:8d} ({100 * c['samples'] / max(tot, 1):5.1f}%)  exec {n_exec[op]:10d}  {top}")
        print("   hottest instructions:")
        for s, addr, src, st in sorted(hot, key=lambda x: -x[0])[:a.top]:
            print(f"   {s:7d} {addr[-5:]} {src[:60]:60s} {st}")


if __name__ == "__main__":
    sys.exit(main())
