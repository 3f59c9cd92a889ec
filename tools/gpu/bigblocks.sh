#!/bin/bash
# n = 4096 coherence-block path on the GPU box: bench lines (Hubbard, configs[4]) and the bigblock GPU tests.
# usage: bash tools/gpu/bigblocks.sh TAG
tag=${1:-bb}
mkdir -p gpurun_out
timeout 600 python bench.py --config hubbard3 --steps 2 --warmup 1 > gpurun_out/${tag}_hubbard3.json 2> gpurun_out/${tag}_hubbard3.err
echo "hubbard rc $?"; tail -c 300 gpurun_out/${tag}_hubbard3.err
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 1 > gpurun_out/${tag}_cfg4.json 2> gpurun_out/${tag}_cfg4.err
echo "cfg4 rc $?"
python - gpurun_out/${tag}_hubbard3.json gpurun_out/${tag}_cfg4.json <<'PY'
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 1), d["unit"], "frac", round(d["roofline"]["frac"], 3), d.get("structure", "")[:160])
    except Exception as e:
        print(f, "FAILED", e)
PY
timeout 1200 python -m pytest tests/test_gpu_bigblocks.py -x -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/${tag}_pytest.log
