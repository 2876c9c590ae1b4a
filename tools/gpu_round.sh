set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_v4_smoke.log 2>&1
python bench.py > gpurun_out/r02_v4_bench.json 2> gpurun_out/r02_v4_bench.err
python bench.py --config batched --no-cpu-baseline > gpurun_out/r02_v4_batched.json 2> gpurun_out/r02_v4_batched.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_v4_launches.csv python tools/run_hyres.py large 2 > gpurun_out/ncu.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_v4_pytest_gpu.log 2>&1
