b() { python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], 'sure', d['stages']['sure']['ms'], 'iso sure', d['wavelet_isolated']['sure']['ms'], 'dwt+sure', d['wavelet_isolated']['dwt+sure']['ms'])"; }
b; b
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
