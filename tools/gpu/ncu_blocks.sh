#!/bin/bash
# ncu evidence for the block path (run through gpurun, one GPU):
#  1. launch list of the default bench command (per-launch device times; cold-cache, serialised)
#  2. `--set full` of the block kernels of one fwd+grad call (1200 pulses x 128 slices: the fused forward
#     layout, a full gradient grid), with source correlation, exported for tools/ncu_summary.py
# usage: bash tools/gpu/ncu_blocks.sh TAG [pulses] [slices]
tag=${1:-ncu}; B=${2:-1200}; N=${3:-128}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-dense-ref \
  --no-cpu-baseline > gpurun_out/${tag}_launches.log 2>&1
echo "launch list rc $?"
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"k_blk_(grad_slices|expm_fold|suffix_chain|prefix_chain)" \
  -c 12 -f -o gpurun_out/${tag}_full python tools/blk_profile.py $B $N > gpurun_out/${tag}_full.log 2>&1
echo "full rc $?"
tail -3 gpurun_out/${tag}_full.log
