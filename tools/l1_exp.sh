# F3 first-iteration experiments: HYDE_L1_SMEM = 0 (y scratch in X) / 32 / 64 (y in shared memory, CTA of 32 / 64 pixels)
cat > /tmp/l1t.py <<'PY'
import os, sys, torch, numpy as np
sys.path.insert(0, '.')
from harness import synth
import paper_2204_06979_b200 as hy
mode = os.environ.get('HYDE_L1_SMEM', '0')
x = torch.from_numpy(synth.make_cube('large', 0).noisy).cuda()
m = hy.hyres(x)
out = torch.empty_like(m)
for _ in range(3):
    _, its = hy.l1_spectral(m, out, return_iters=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    hy.l1_spectral(m, out)
e1.record(); torch.cuda.synchronize()
print(f"mode {mode}: l1 stage {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per call, mean iters {its.float().mean().item():.3f}")
np.save(f'/tmp/l1_{mode}.npy', out.cpu().numpy())
PY
for v in 0 32 64 0 32 64; do HYDE_L1_SMEM=$v python /tmp/l1t.py; done
python -c "
import numpy as np
a=np.load('/tmp/l1_0.npy')
for v in ('32','64'):
    b=np.load(f'/tmp/l1_{v}.npy'); print(v, 'bitwise equal to X-scratch:', (a==b).all())
"
HYDE_L1_SMEM=32 timeout 600 python -m pytest tests/test_gpu_hyminor.py -q -x 2>&1 | tail -2
for v in 0 32; do HYDE_L1_SMEM=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:l1spec_first --csv python tools/run_l1.py large 1 2>/dev/null | grep -v "^==" | tail -3; done
