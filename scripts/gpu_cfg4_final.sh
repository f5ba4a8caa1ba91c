#!/bin/bash
# cfg4 after the work-balanced fused kernel: full-size parity, default bench line, launch list, ncu of k_fused
mkdir -p gpurun_out
timeout 900 python scripts/full_parity.py cfg4 > gpurun_out/parity4.log 2>&1; tail -1 gpurun_out/parity4.log | cut -c1-400; cp profiles/r01_full_parity.json gpurun_out/
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cut -c1-200 gpurun_out/bench_default.json
CMD="python bench.py --config cfg4 --iterations 4 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $CMD > /dev/null 2>&1
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_cfg4_fused_lin $CMD > /dev/null 2>&1
ls gpurun_out/prof_cfg4_fused_lin*
