set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for pd in 0 16 32 64; do FDG_BOX_PD=$pd timeout 300 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('PD', $pd, 'cfg4', round(d['value']), round(d['roofline']['frac'],3))"; done
for pd in 0 32; do FDG_BOX_PD=$pd timeout 300 python bench.py --config cfg4b --steps 3 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('PD', $pd, 'cfg4b', round(d['value']), round(d['roofline']['frac'],3))"; done
