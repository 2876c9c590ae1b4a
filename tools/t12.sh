for i in 1 2; do python bench.py --config batched --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items() if v['ms']})"; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/run_gram.py large
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qscale|fix|finalize|gram_tc" --csv python tools/run_batched.py 1 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for x in r[1:]:
  d=dict(zip(h,x)); print(d['Kernel Name'][:40], d['Grid Size'], d['Metric Value'])"
