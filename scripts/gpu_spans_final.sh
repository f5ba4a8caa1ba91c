#!/bin/bash
# spans engine (tile kernel for small images): GPU suite, full-size parity cfg1/cfg2, bench lines, probe, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 600 python scripts/full_parity.py cfg1 cfg2 > gpurun_out/parity12.log 2>&1; tail -3 gpurun_out/parity12.log; cp profiles/r01_full_parity.json gpurun_out/
for c in cfg1 cfg2; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; cut -c1-200 gpurun_out/bench_$c.json; done
for sz in "2048 2048" "4096 4096" "8192 8192"; do timeout 120 python scripts/spans_probe.py disc10 $sz 20; done
for sz in "1024 1024" "2048 2048" "4096 4096"; do timeout 120 python scripts/spans_probe.py oblique21 $sz 20; done
for c in cfg1 cfg2; do
CMD="python bench.py --config $c --iterations 3 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spant -s 2 -c 1 -o gpurun_out/prof_${c}_spant $CMD > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
