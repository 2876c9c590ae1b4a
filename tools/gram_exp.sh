# K1 experiments: 8 = CTA-scope forwarder arrive, 16 = merged T_a* MMAs (A = P, B = [P; QS])
for v in "HYDE_GRAM_EXP=8" "HYDE_GRAM_EXP=24" "HYDE_GRAM_EXP=8" "HYDE_GRAM_EXP=24" "HYDE_GRAM_EXP=28"; do
  echo "== $v"; env $v python tools/run_gram.py large
done
for v in 8 24; do HYDE_GRAM_EXP=$v python - <<'PY'
import os, sys, torch, numpy as np
sys.path.insert(0, '.')
from harness import synth
import paper_2204_06979_b200 as hy
v = os.environ['HYDE_GRAM_EXP']
for name in ('large', 'small', 'medium', 'wide', 'tiny'):
    cube = torch.from_numpy(synth.make_cube(name, 0).noisy).cuda()
    g = hy.stages.gram(cube).cpu().numpy()
    np.save(f'/tmp/g_{name}_{v}.npy', g)
PY
done
python -c "
import numpy as np
for n in ('large','small','medium','wide','tiny'):
    a=np.load(f'/tmp/g_{n}_8.npy'); b=np.load(f'/tmp/g_{n}_24.npy'); print(n, a.shape, 'merged == unmerged bitwise:', (a==b).all(), np.abs(a-b).max())
"
