#!/bin/bash
# Builder bench lines of the other configs on the GPU box: configs[3] forward and gradient, the 512-pulse
# rank share of configs[2] at G = 8 (one GPU), configs[4] and the Hubbard sample.
# usage: bash tools/gpu/configs.sh TAG
tag=${1:-c}
mkdir -p gpurun_out
run() {  # name args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err
  echo "$name rc $?"
}
run cfg3 --config cfg3 --steps 3 --warmup 3
run cfg3grad --config cfg3grad --steps 3 --warmup 3
run cfg2_512 --pulses 512 --steps 5 --warmup 3 --no-cpu-baseline --no-dense-ref --no-e2e
run cfg4 --config cfg4 --steps 2 --warmup 1
run hubbard3 --config hubbard3 --steps 2 --warmup 1
python - gpurun_out/${tag}_*.json <<'PY'
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 1), d["unit"], "ms", round(d["ms_per_step"], 2), "frac", round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(f, "FAILED", e)
PY
