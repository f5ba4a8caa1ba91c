#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config cfg4 --iterations 4 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_cfg4_fused $CMD > /dev/null 2>&1
ls gpurun_out/prof_cfg4_fused*
