# one GPU iteration: tests, benches, launch list + full ncu capture of the top kernel
# usage: bash scripts/gpu_iter.sh <tag> <kernel-regex> [configs...]
set -x
TAG=$1; KRE=$2; shift 2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
for c in "$@"; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 $( [ $c != cfg4 ] && echo --no-cpu-baseline ) > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; tail -1 gpurun_out/bench_${TAG}_$c.json | cut -c1-300; done
CMD="python bench.py --config cfg4 --iterations 2 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > /dev/null 2>&1
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$KRE -s 4 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
