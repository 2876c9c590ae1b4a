python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/lz_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_stages.py -x -q > gpurun_out/lz_pytest.log 2>&1
python bench.py --steps 10 --no-cpu-baseline --iso-steps 0 > gpurun_out/lz_bench.json 2> gpurun_out/lz_bench.err
HYDE_EIG_LANCZOS=0 python bench.py --steps 10 --no-cpu-baseline --iso-steps 0 > gpurun_out/lz_bench_off.json 2>> gpurun_out/lz_bench.err
