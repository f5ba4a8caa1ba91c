timeout 600 python -m pytest tests/test_gpu_conv.py -m gpu -q -x 2>&1 | tail -1
for c in cfg4 cfg4b; do
for v in "rect 0" "0 0" "0 16" "0 32" "0 64" "1 0" "1 32" "2 32" "3 32"; do
  set -- $v
  if [ $1 = rect ]; then export FDG_FORCE_RECT=1; else unset FDG_FORCE_RECT; export FDG_BOX_VARIANT=$1; export FDG_BOX_PD=$2; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c var=$1 pd=$2', round(d['value']), round(d['roofline']['frac'],3), d['config']['engine'])"
done; done
