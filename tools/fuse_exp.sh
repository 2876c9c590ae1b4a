# fused coarse DWT/IDWT levels vs the per-level launches (HYDE_DWT_NOFUSE=1)
b() { python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], {k: d['stages'][k]['ms'] for k in ('dwt','sure','idwt')}, 'iso', d['wavelet_isolated']['dwt']['ms'], d['wavelet_isolated']['idwt']['ms'], 'forpdn', d['forpdn']['ms'], 'wsrrr', d['wsrrr']['ms'], 'launches', d['gpu_launches'])"; }
echo "== fused"; b
echo "== per-level"; HYDE_DWT_NOFUSE=1 b
echo "== fused"; b
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
