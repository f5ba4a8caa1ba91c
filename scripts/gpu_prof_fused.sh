#!/bin/bash
set -x
mkdir -p gpurun_out
CMD="python bench.py --config cfg4 --iterations 2 --steps 1 --warmup 1 --no-cpu-baseline"
export FDG_FUSED=1 FDG_FUSED_V=${FDG_FUSED_V:-0}
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
