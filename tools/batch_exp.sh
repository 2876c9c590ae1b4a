# batched mode: eigensolver groups (HYDE_BATCH_SPLIT = cubes in the first K2 launch; 0 = one launch)
for v in 0 36 18 0 36 18 27; do
  echo "== HYDE_BATCH_SPLIT=$v"; HYDE_BATCH_SPLIT=$v python bench.py --config batched --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items() if v['ms']})"
done
HYDE_BATCH_SPLIT=36 timeout 900 python -m pytest tests -m gpu -q -x -k "batch" 2>&1 | tail -2
