#!/bin/bash
# configs[2] block-engine sub-batch sweep (bench line without CPU baseline / dense reference / e2e)
mkdir -p gpurun_out/sb
for sb in "$@"; do
  timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-dense-ref --no-e2e --sub-batch $sb \
    > gpurun_out/sb/sb$sb.json 2> gpurun_out/sb/sb$sb.err
  python - gpurun_out/sb/sb$sb.json $sb <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("sub", sys.argv[2], round(d["value"] / 1e6, 3), "M", round(d["ms_per_step"], 2), "ms",
          {k: round(v["ms_per_step"], 2) for k, v in d["stage_split"].items()})
except Exception as e:
    print("sub", sys.argv[2], "FAILED", e)
PY
done
