set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in cfg4 cfg4b cfg0; do
for v in 0 1; do
  if [ $v = 1 ]; then export FDG_FORCE_RECT=1; else unset FDG_FORCE_RECT; fi
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c force_rect=$v', round(d['value']), round(d['roofline']['frac'],3), d['config']['engine'])"
done; done
unset FDG_FORCE_RECT
CMD="python bench.py --config cfg4 --iterations 2 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_box -s 4 -c 2 -o gpurun_out/prof_v3 $CMD > /dev/null 2>&1
ls gpurun_out
