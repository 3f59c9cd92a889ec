#!/bin/bash
# role-specialised kernels: register caps (libs) x forward sets
mkdir -p gpurun_out/reg
run() {  # name lib fwdsets
  QAL_LIB="$2" QAL_BLK_SETS_FWD="$3" timeout 300 python bench.py --steps 4 --warmup 3 --no-dense-ref \
    > gpurun_out/reg/$1.json 2> gpurun_out/reg/$1.err
  python -c "
import json;d=json.loads(open('gpurun_out/reg/$1.json').read().strip().splitlines()[-1]); s=d['stage_split']
print('$1', '$2', '$3', round(d['value']/1e6,3), round(d['roofline']['frac'],3), {k:round(v['ms_per_step'],1) for k,v in s.items() if k.startswith('blk')})" 2>/dev/null || (echo "$1 FAILED"; tail -3 gpurun_out/reg/$1.err)
}
run d0 "" ""
run d1 "" "1:4,2:2,4:4"
run a0 tools/bin/libqal_regA.so ""
run a1 tools/bin/libqal_regA.so "1:4,2:2,4:4"
run b0 tools/bin/libqal_regB.so ""
run b1 tools/bin/libqal_regB.so "1:4,2:2,4:4"
