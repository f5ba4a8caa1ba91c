#!/bin/bash
# DRAM bytes per launch of each config's dominant kernel (-> profiles/traffic.json).
# Row-resident configs: the first launch (the device loop's warm-up step); the
# pass engines: the third launch (inside the warm-up step).
mkdir -p gpurun_out
for spec in "cfg0 k_rowres 0" "cfg1 k_spant 2" "cfg2 k_spant 2" "cfg3 k_dense 2" "cfg4 k_fused 2" "cfg4b k_rowres 0"; do
  set -- $spec
  CMD="python bench.py --config $1 --iterations 3 --steps 1 --warmup 1 --no-cpu-baseline"
  $CMD > /dev/null 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:$2 -s $3 -c 1 --csv $CMD > gpurun_out/traffic_$1.csv 2>/dev/null
  echo "$1 $(grep -c dram gpurun_out/traffic_$1.csv)"
done
