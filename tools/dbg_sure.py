import sys, os; sys.path.insert(0,'/root/repo')
import numpy as np, torch
from harness import synth
from oracle import hyres_ref as O
import paper_2204_06979_b200 as hy
name = sys.argv[1] if len(sys.argv) > 1 else 'medium'
s = synth.make_cube(name, 0)
ref = O.hyres(s.noisy, keep_images=True)
b, r, c = s.noisy.shape
lv = ref.levels
imgs = np.stack([e.astype(np.float32) for e in ref.eigen_images])
co = hy.stages.dwt_fwd(torch.from_numpy(imgs).cuda(), lv, 16)
cpu = co.cpu().numpy()
try:
    ks, ts, ep = hy.stages.sure(co, r, c, lv)
    print('ok', ks.cpu().numpy())
except Exception as e:
    print('ERR', e)
tmpl = O.dwt2(np.zeros((r, c)), lv, 16)
subs = O.flatten_coeffs(tmpl); offs = np.cumsum([0] + [x.size for x in subs])
for i in range(cpu.shape[0]):
    for j in range(len(subs)):
        sr = O.sure_threshold(cpu[i, offs[j]:offs[j+1]].astype(np.float64))
        print(i, j, offs[j+1]-offs[j], 'k*', sr.k, 't*', sr.t, 'margin', sr.margin)
