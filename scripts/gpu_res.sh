#!/bin/bash
# resident spans RL (k_spansres) variants on cfg1: parity tests + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rl.py -x -q > gpurun_out/pytest_rl.log 2>&1; echo "pytest rl: $(tail -1 gpurun_out/pytest_rl.log)"
for v in 0 1 2; do
  FDG_RES_VAR=$v timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_res$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_res$v.json'));print('var $v', round(d['value']), d['config']['engine'], round(d['roofline']['kernel_ms'],3), 'ms/launch')"
done
