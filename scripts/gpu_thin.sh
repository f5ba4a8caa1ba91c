#!/bin/bash
# thinned cfg3: GPU suite, thin bench (flat work list vs per-tile), optional full parity (PARITY=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.log)"
for t in active50 active25; do
  timeout 400 python bench.py --thin $t --steps 3 --warmup 1 > gpurun_out/bench_cfg3_$t.json 2> gpurun_out/bench_cfg3_$t.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg3_$t.json'));print('flat $t', round(d['value']), round(d['unthinned_value']), round(d.get('speedup_vs_unthinned'),3), round(d['roofline']['achieved'],1))"
  FDG_THIN_TILE=1 timeout 400 python bench.py --thin $t --steps 3 --warmup 1 > gpurun_out/bench_cfg3_${t}_tile.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_cfg3_${t}_tile.json'));print('tile $t', round(d['value']), round(d.get('speedup_vs_unthinned'),3))"
done
if [ "$PARITY" = 1 ]; then timeout 900 python scripts/full_parity.py cfg3 > gpurun_out/parity3.log 2>&1; tail -3 gpurun_out/parity3.log | cut -c1-400; cp profiles/r01_full_parity.json gpurun_out/; fi
