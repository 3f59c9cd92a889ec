#!/bin/bash
# GPU-box A/B turn: default bench (no CPU baseline / dense reference / e2e) then the block GPU tests.
# usage: bash tools/gpu/quick.sh TAG [pytest -k expr]
tag=${1:-q}; kexpr=${2:-}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-dense-ref --no-e2e > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc $?"
python - gpurun_out/${tag}_bench.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(round(d["value"] / 1e6, 3), "M", round(d["ms_per_step"], 2), "ms",
          {k: round(v["ms_per_step"], 2) for k, v in d["stage_split"].items()}, round(d["roofline"]["frac"], 3))
except Exception as e:
    print("FAILED", e)
PY
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1
fi
echo "pytest rc $?"; tail -2 gpurun_out/${tag}_pytest.log
