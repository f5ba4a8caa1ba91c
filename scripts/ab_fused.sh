#!/bin/bash
# A/B of fused-kernel variants (FDG_FUSED_V) on config 4: device loop Mpx*it/s and us per launch
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2 3}; do
  for rep in 1 2; do
    FDG_FUSED_V=$v timeout 300 python bench.py --config cfg4 --iterations ${ITERS:-30} --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ab_v$v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_v$v.json'));print('v$v', round(d['value']), round(d['roofline']['kernel_ms']*1e3,1), 'us', d['clocks']['sm_mhz'])"
  done
done
