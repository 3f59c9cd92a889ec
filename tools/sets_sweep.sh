#!/bin/bash
# A/B of the block launch sets (QAL_BLK_SETS_FWD / _GRAD) on the default cfg2 bench.
mkdir -p gpurun_out/sets
run() {  # name fwd grad
  QAL_BLK_SETS_FWD="$2" QAL_BLK_SETS_GRAD="$3" timeout 300 python bench.py --steps 4 --warmup 3 --no-dense-ref \
    > gpurun_out/sets/$1.json 2> gpurun_out/sets/$1.err
  python -c "
import json;d=json.loads(open('gpurun_out/sets/$1.json').read().strip().splitlines()[-1])
print('$1', '$2', '$3', round(d['value']/1e6,3), round(d['roofline']['frac'],3), d['stage_split'])" || tail -3 gpurun_out/sets/$1.err
}
run fused "" ""
run A "5:1,2:2" "5:1,2:2"
run B "1:4,2:2,4:4" "1:4,2:2,4:4"
run C "5:1,2:4" "5:1,2:4"
run E "1:4,6:2" "1:4,6:2"
run fused2 "" ""
