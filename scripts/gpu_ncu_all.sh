#!/bin/bash
# one `ncu --set full` capture of each config's dominant kernel (round summary)
mkdir -p gpurun_out
for spec in "cfg0 k_rowres 0" "cfg1 k_spant 2" "cfg2 k_spant 2" "cfg3 k_dense 2" "cfg4 k_fused 2" "cfg4b k_rowres 0"; do
  set -- $spec
  CMD="python bench.py --config $1 --iterations 3 --steps 1 --warmup 1 --no-cpu-baseline"
  $CMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
      -o gpurun_out/full_$1 $CMD > /dev/null 2>&1
  ls gpurun_out/full_$1.ncu-rep
done
