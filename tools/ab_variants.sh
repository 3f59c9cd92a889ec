#!/bin/bash
# A/B of experiment builds (paper_2511_13330_b200/variants/libqal_<v>.so) against the in-tree library on
# the default bench: bash tools/ab_variants.sh OUTDIR v1 v2 ...   (run on the GPU box)
out=$1; shift
mkdir -p $out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-dense-ref --no-e2e > $out/default.json 2>&1
for v in "$@"; do
  QAL_LIB=paper_2511_13330_b200/variants/libqal_$v.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    --no-dense-ref --no-e2e > $out/$v.json 2>&1
done
for f in $out/*.json; do
  python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"] / 1e6, 3), "M", round(d["ms_per_step"], 2), "ms",
          {k: round(v["ms_per_step"], 2) for k, v in d["stage_split"].items()}, round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
