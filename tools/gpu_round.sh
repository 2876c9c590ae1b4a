set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_v16_smoke.log 2>&1
python bench.py > gpurun_out/r02_v16_bench.json 2> gpurun_out/r02_v16_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_v16_reference.json 2> gpurun_out/r02_v16_reference.err
python bench.py --config batched --no-cpu-baseline > gpurun_out/r02_v16_batched.json 2> gpurun_out/r02_v16_batched.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_v16_torchrun1.json 2> gpurun_out/r02_v16_torchrun1.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_v16_launches.csv python tools/run_hyres.py large 2 > gpurun_out/ncu.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_v16_pytest_gpu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k2_cluster|gram_tc_kernel|project_kernel|recon_kernel|sure_kernel" -c 6 -o gpurun_out/r02_v16_full python tools/run_hyres.py large 1 > gpurun_out/r02_v16_ncufull.log 2>&1
