timeout 600 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_stages.py -x -q > gpurun_out/bt_pytest.log 2>&1
python bench.py --config batched --no-cpu-baseline --steps 10 > gpurun_out/bt.json 2>gpurun_out/bt.err
python bench.py --steps 10 --iso-steps 0 --no-cpu-baseline > gpurun_out/bt_large.json 2>>gpurun_out/bt.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bt_launches.csv python tools/run_batched.py 1 > /dev/null 2>&1
