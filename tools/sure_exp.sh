timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_e2e.py -q -x 2>&1 | tail -2
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/t9_bench.json 2> gpurun_out/t9_bench.err
for g in 2 4; do echo "== HYDE_SURE_G=$g"; HYDE_SURE_G=$g python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages']['sure'])"; done
HYDE_SURE_PROF=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/sure_prof.py --count 4
python tools/sure_prof.py --count 4
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
