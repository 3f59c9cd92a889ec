#!/bin/bash
# Hubbard / configs[4] bench lines for the in-tree build and experiment builds (variants/libqal_<v>.so)
# usage: bash tools/gpu/bb_variants.sh v1 v2 ...
mkdir -p gpurun_out/bbv
one() {  # name lib
  for cfg in hubbard3 cfg4; do
    QAL_LIB=$2 timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 > gpurun_out/bbv/$1_$cfg.json 2> gpurun_out/bbv/$1_$cfg.err
    python - gpurun_out/bbv/$1_$cfg.json $1 $cfg <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], sys.argv[3], round(d["value"], 1), d["unit"], "frac", round(d["roofline"]["frac"], 3),
          "gemm ms", round(d.get("stage_ms_per_step", {}).get("blk_gemm", 0), 2))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
}
one default paper_2511_13330_b200/libqal.so
for v in "$@"; do one $v paper_2511_13330_b200/variants/libqal_$v.so; done
