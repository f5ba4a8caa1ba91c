#!/bin/bash
# Round-end measurements (session 2): default bench line (cfg4, CPU baseline),
# every config, the reference arm, smoke, launch list of the default config.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"; cut -c1-300 gpurun_out/bench_default.json
for c in cfg0 cfg1 cfg2 cfg3 cfg4b; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['value']), d['config']['engine'], 'e2e', round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']))"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; cut -c1-300 gpurun_out/bench_reference.json
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
CMD="python bench.py --config cfg4 --iterations 4 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $CMD > /dev/null 2>&1; echo "ncu rc=$?"
