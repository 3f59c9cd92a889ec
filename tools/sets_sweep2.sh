#!/bin/bash
# per-set timing of the gradient / forward kernels (single sets: timing only, results incomplete)
mkdir -p gpurun_out/sets2
run() {  # name fwd grad [split]
  QAL_BLK_SPLIT="$4" QAL_BLK_SETS_FWD="$2" QAL_BLK_SETS_GRAD="$3" timeout 300 python bench.py --steps 3 --warmup 3 --no-dense-ref \
    > gpurun_out/sets2/$1.json 2> gpurun_out/sets2/$1.err
  python -c "
import json;d=json.loads(open('gpurun_out/sets2/$1.json').read().strip().splitlines()[-1]); s=d['stage_split']
print('$1 fwd=$2 grad=$3 split=$4', round(s['blk_expm_fold']['ms_per_step'],1), round(s['blk_grad_slices']['ms_per_step'],1))" 2>/dev/null || (echo "$1 FAILED"; tail -2 gpurun_out/sets2/$1.err)
}
run s1 "1:1" "1:1"
run s2 "1:2" "1:2"
run s3 "1:4" "1:4"
run s4 "2:1" "2:1"
run s5 "2:2" "2:2"
run s6 "2:4" "2:4"
run s7 "4:1" "4:1"
run s8 "4:2" "4:2"
run s9 "4:4" "4:4"
run s10 "2:2" "2:2" 1
run s11 "2:4" "2:4" 1
run s12 "5:1" "5:1"
run s13 "5:2" "5:2"
run s14 "6:1" "6:1"
run s15 "6:2" "6:2" 1
