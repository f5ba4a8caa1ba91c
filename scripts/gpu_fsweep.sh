#!/bin/bash
# A/B of prebuilt fused-kernel libraries: gpurun_out/libs/*.so swapped in turn
mkdir -p gpurun_out
for L in scripts/libs/*.so; do
  cp $L paper_1304_7211_b200/libfdgpu.so
  n=$(basename $L .so)
  FDG_FUSED=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fs_$n.json 2> gpurun_out/fs_$n.err
done
