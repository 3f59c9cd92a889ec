#!/bin/bash
# A/B of two libqal builds on the default cfg2 bench: tools/ab.sh name_a lib_a name_b lib_b [bench args]
mkdir -p gpurun_out/ab
na=$1; la=$2; nb=$3; lb=$4; shift 4
for i in 1 2; do
  for pair in "$na:$la" "$nb:$lb"; do
    n=${pair%%:*}; l=${pair#*:}
    QAL_LIB="$l" timeout 300 python bench.py --steps 4 --warmup 3 --no-dense-ref "$@" > gpurun_out/ab/$n.json 2> gpurun_out/ab/$n.err
    python -c "
import json;d=json.loads(open('gpurun_out/ab/$n.json').read().strip().splitlines()[-1]); s=d.get('stage_split',{})
print('$n', round(d['value']/1e6,3), round(d['roofline']['frac'],3), {k:round(v['ms_per_step'],1) for k,v in s.items() if k.startswith('blk')})" 2>/dev/null || (echo "$n FAILED"; tail -3 gpurun_out/ab/$n.err)
  done
done
