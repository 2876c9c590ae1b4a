# K1: atomic pair sum (default) vs the reduce kernel (HYDE_GRAM_REDUCE=1): timing and bitwise G
for v in "" "HYDE_GRAM_REDUCE=1" "" "HYDE_GRAM_REDUCE=1"; do
  echo "== $v"; env $v python tools/run_gram.py large
done
for v in 0 1; do
  if [ $v = 1 ]; then export HYDE_GRAM_REDUCE=1; else unset HYDE_GRAM_REDUCE; fi
  python - <<PY
import os, sys, torch, numpy as np
sys.path.insert(0, '.')
from harness import synth
import paper_2204_06979_b200 as hy
for name in ('large', 'small', 'medium', 'wide', 'tiny'):
    cube = torch.from_numpy(synth.make_cube(name, 0).noisy).cuda()
    g = hy.stages.gram(cube).cpu().numpy()
    np.save(f'/tmp/g_{name}_$v.npy', g)
PY
done
unset HYDE_GRAM_REDUCE
python -c "
import numpy as np
for n in ('large','small','medium','wide','tiny'):
    a=np.load(f'/tmp/g_{n}_0.npy'); b=np.load(f'/tmp/g_{n}_1.npy'); print(n, 'atomic == reduce bitwise:', (a==b).all())
"
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_sharded.py tests/test_gpu_e2e.py -q -x 2>&1 | tail -2
python bench.py --steps 10 --no-cpu-baseline > gpurun_out/t7_bench.json 2> gpurun_out/t7_bench.err
python bench.py --config batched --steps 10 --no-cpu-baseline > gpurun_out/t7_batched.json 2> gpurun_out/t7_batched.err
