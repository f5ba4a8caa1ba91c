#!/bin/bash
# Round-2 evidence on one B200: bench lines of every config (with the CPU
# baselines), thinned cfg3, the ncu launch list of the default bench command,
# DRAM traffic of each dominant kernel.  Results under gpurun_out/r02_*.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/r02_smi.txt 2>&1
for c in cfg4 cfg0 cfg1 cfg2 cfg3 cfg4b; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
  echo "$c rc=$? $(cut -c1-160 gpurun_out/r02_bench_$c.json)"
done
for t in active50 active25; do
  timeout 600 python bench.py --config cfg3 --thin $t --steps 3 --warmup 1 > gpurun_out/r02_bench_cfg3_$t.json 2> gpurun_out/r02_bench_cfg3_$t.err
  echo "cfg3-$t rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_cfg4.json 2> gpurun_out/r02_bench_reference_cfg4.err
echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu_launches.log 2>&1
echo "launch list rc=$?"
for spec in "cfg0 k_rowres 0" "cfg1 k_spant 2" "cfg2 k_spant 2" "cfg3 k_dense 2" "cfg4 k_fused 2" "cfg4b k_rowres 0"; do
  set -- $spec
  CMD="python bench.py --config $1 --iterations 3 --steps 1 --warmup 1 --no-cpu-baseline"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:$2 -s $3 -c 1 --csv $CMD > gpurun_out/r02_traffic_$1.csv 2>/dev/null
  echo "traffic $1 $(grep -c dram gpurun_out/r02_traffic_$1.csv)"
done
