timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_rl.py -m gpu -q -x 2>&1 | tail -2
for c in cfg1 cfg2; do
for v in "0 0" "64 0" "128 0" "64 24" "64 32" "64 48" "128 32" "128 64"; do
  set -- $v
  export FDG_SPANS_NT=$1 FDG_SPANS_BAND=$2
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "import json,sys; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$c nt=$1 band=$2', round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],4))"
done; done
