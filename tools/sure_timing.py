"""Time the SURE stage on 1024x1024 L5 coefficient rows of several kinds."""
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_06979_b200 as hy
r, c, lv = 1024, 1024, 5
nc = hy.stages.coeff_count(r, c, lv)
rng = np.random.default_rng(0)
rows = []
for i in range(8):
    a = rng.standard_normal(nc)
    if i == 0:
        a[rng.random(nc) < 0.05] *= 20
    rows.append(a)
co = torch.from_numpy(np.stack(rows).astype(np.float32)).cuda()
for it in range(4):
    g = co.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); hy.stages.sure(g, r, c, lv); e1.record(); torch.cuda.synchronize()
    print('sure ms', e0.elapsed_time(e1), flush=True)
