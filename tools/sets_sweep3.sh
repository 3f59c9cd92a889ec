#!/bin/bash
# slot counts of the group-specialised launches (role-compiled kernels, swizzled images)
mkdir -p gpurun_out/sets3
run() {  # name fwd grad
  QAL_BLK_SETS_FWD="$2" QAL_BLK_SETS_GRAD="$3" timeout 300 python bench.py --steps 4 --warmup 3 --no-dense-ref \
    --no-cpu-baseline --no-e2e > gpurun_out/sets3/$1.json 2> gpurun_out/sets3/$1.err
  python -c "
import json;d=json.loads(open('gpurun_out/sets3/$1.json').read().strip().splitlines()[-1]); s=d['stage_split']
print('$1 fwd=$2 grad=$3', round(d['value']/1e6,3), round(s['blk_expm_fold']['ms_per_step'],1), round(s['blk_grad_slices']['ms_per_step'],1))" 2>/dev/null || (echo "$1 FAILED"; tail -2 gpurun_out/sets3/$1.err)
}
run d "" ""
run f1 "1:2,2:2,4:4" ""
run f2 "1:4,2:4,4:4" ""
run f3 "1:4,2:2,4:2" ""
run f4 "1:1,2:1,4:1" ""
run g1 "" "1:2,2:2,4:4"
run g2 "" "1:4,2:1,4:4"
run g3 "" "1:4,2:4,4:4"
run g4 "" "1:4,2:2,4:2"
run d2 "" ""
