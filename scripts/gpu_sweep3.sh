timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_rl.py -m gpu -q -x 2>&1 | tail -1
for c in cfg4 cfg4b; do
for v in "rect" "0" "1" "2" "3" "4"; do
  if [ $v = rect ]; then export FDG_FORCE_RECT=1; else unset FDG_FORCE_RECT; export FDG_BOX_VARIANT=$v; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c var=$v', round(d['value']), round(d['roofline']['frac'],3), d['config']['engine'])"
done; done
