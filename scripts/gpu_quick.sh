#!/bin/bash
# quick check: GPU suite + bench lines for the configs given as arguments
mkdir -p gpurun_out
[ "$NOTEST" = 1 ] || { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.log)"; }
for c in "$@"; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['value']), round(d['roofline']['kernel_ms']*1e3,2), 'us/launch', 'e2e', round(d['e2e']['value']))" 2>&1 | tail -1; done
