#!/bin/bash
# fused kernel: work-balanced segments (default) vs the plain band grid (FDG_FUSED_LIN=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_rl.py -x -q > gpurun_out/pt_fused.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pt_fused.log)"
for L in 1 0 1 0; do
  FDG_FUSED_LIN=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bl.json'));print('lin $L', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms']*1e3,1),'us')"
done
