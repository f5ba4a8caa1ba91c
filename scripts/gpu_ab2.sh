for c in cfg4 cfg4b; do
for v in rect 0 1000 100000; do
  if [ $v = rect ]; then export FDG_FORCE_RECT=1; else unset FDG_FORCE_RECT; export FDG_WAIT_HINT=$v; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $v', round(d['value']), round(d['roofline']['frac'],3), d['config']['engine'])"
done; done
