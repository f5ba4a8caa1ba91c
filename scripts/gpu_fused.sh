#!/bin/bash
# fused-engine parity + variant sweep on the GPU box (cfg4 bench)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -15 > gpurun_out/fused_tests.log
for v in ${VARIANTS:-0 1 2 3}; do
  FDG_FUSED=1 FDG_FUSED_V=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fused_v$v.json 2> gpurun_out/fused_v$v.err
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fused_off.json 2> gpurun_out/fused_off.err
