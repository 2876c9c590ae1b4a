for t in 1e-14 1e-12 1e-10; do
  HYDE_EIG_LZTOL=$t python tools/lz_phases.py large > gpurun_out/lz2_large_$t.log 2>&1
  HYDE_EIG_LZTOL=$t python tools/lz_phases.py batched > gpurun_out/lz2_batched_$t.log 2>&1
done
HYDE_EIG_BATCHED_LANCZOS=1 python bench.py --config batched --no-cpu-baseline --steps 10 > gpurun_out/lz2_bl.json 2>/dev/null
python bench.py --config batched --no-cpu-baseline --steps 10 > gpurun_out/lz2_bh.json 2>/dev/null
python bench.py --steps 10 --iso-steps 0 --no-cpu-baseline > gpurun_out/lz2_large.json 2>/dev/null
timeout 600 python -m pytest tests/test_gpu_e2e.py -x -q > gpurun_out/lz2_pytest.log 2>&1
