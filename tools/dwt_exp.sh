timeout 600 python -m pytest tests/test_gpu_stages.py -q -x -k "dwt or idwt or wavelet" 2>&1 | tail -2
python tools/iso_wavelet.py > gpurun_out/t8_iso.json 2>&1
python tools/iso_wavelet.py > gpurun_out/t8_iso2.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum --clock-control none -k regex:dwt_inv --launch-skip 4 --launch-count 1 --csv python tools/iso_wavelet.py --steps 1 2>/dev/null | grep -v "^==" | tail -3
