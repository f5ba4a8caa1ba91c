timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in cfg1 cfg2; do
for v in spans taps; do
  if [ $v = taps ]; then export FDG_NO_SPANS=1; else unset FDG_NO_SPANS; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b_$c_$v.json 2>gpurun_out/b_$c_$v.err; python -c "import json,sys; d=json.loads(open('gpurun_out/b_$c_$v.json').read().strip().splitlines()[-1]); print('$c $v', round(d['value']), round(d['roofline']['frac'],3), d['config']['engine'], round(d['roofline']['kernel_ms'],4))"
done; done
