#!/bin/bash
# dense engine (cfg3): GPU suite, bench (plain + thinned), ncu; PARITY=1 adds the full-size oracle check
mkdir -p gpurun_out
[ "$NOTEST" = 1 ] || timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; cut -c1-200 gpurun_out/bench_cfg3.json
for t in active50 active25; do timeout 400 python bench.py --thin $t --steps 3 --warmup 1 > gpurun_out/bench_cfg3_$t.json 2> gpurun_out/bench_cfg3_$t.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg3_$t.json'));print('$t', round(d['value']), d.get('speedup_vs_unthinned'), d['roofline']['achieved'])"; done
CMD="python bench.py --config cfg3 --iterations 2 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_dense -s 2 -c 1 -o gpurun_out/prof_cfg3_dense $CMD > /dev/null 2>&1
if [ "$PARITY" = 1 ]; then timeout 900 python scripts/full_parity.py cfg3 > gpurun_out/parity3.log 2>&1; tail -4 gpurun_out/parity3.log; cp profiles/r01_full_parity.json gpurun_out/; fi
