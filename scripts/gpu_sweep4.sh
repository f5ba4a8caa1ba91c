timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_rl.py -m gpu -q -x 2>&1 | tail -1
export FDG_FORCE_RECT=1
for c in cfg4 cfg4b; do
for r in 1 2 4; do
  FDG_RECT_R=$r timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c R=$r', round(d['value']), round(d['roofline']['frac'],3), d['config']['engine'])"
done; done
FDG_RECT_R=2 timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_rl.py -m gpu -q -x 2>&1 | tail -1
