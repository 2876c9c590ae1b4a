timeout 600 python -m pytest tests/test_gpu_hyminor.py tests/test_gpu_frows_large.py -x -q > gpurun_out/l1_pytest.log 2>&1
for v in new old; do
if [ $v = old ]; then export HYDE_L1_THREAD_PER_PIXEL=1; fi
python - <<'PY' >> gpurun_out/l1_sweep2.log 2>&1
import os, sys, torch
sys.path.insert(0, '.')
from harness import synth
import paper_2204_06979_b200 as hy
s = synth.make_cube("large", 0)
x = torch.from_numpy(s.noisy).cuda()
m = hy.hyres(x); out = torch.empty_like(m)
hy.l1_spectral(m, out); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): _, its = hy.l1_spectral(m, out, return_iters=True)
e1.record(); torch.cuda.synchronize()
print("old" if os.environ.get("HYDE_L1_THREAD_PER_PIXEL") else "new", "l1 ms", e0.elapsed_time(e1) / 5, "mean iters", float(its.float().mean()), "checksum", float(out.double().sum()))
PY
done
