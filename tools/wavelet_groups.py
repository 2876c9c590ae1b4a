"""Per-image DWT / SURE / IDWT time of hyde_wavelet_shrink vs the number of
images per call (does L2 residency of a group's coefficients change SURE?)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from harness import synth
import paper_2204_06979_b200 as hy
cfg = synth.CONFIGS["large"]
b = 224
torch.manual_seed(0)
E = torch.randn(b, 1024, 1024, device="cuda") * 3.0
out = torch.empty_like(E)
dev = 0
for g in (8, 16, 32, 64, 224):
    x = E[:g]
    o = out[:g]
    for _ in range(2):
        hy.stages.wavelet_shrink(x, 5, out=o, stats=False)
    torch.cuda.synchronize()
    hy.profile_enable(dev, True)
    reps = max(1, 224 // g)
    for r in range(reps):
        hy.stages.wavelet_shrink(E[(r * g) % b:(r * g) % b + g], 5, out=out[(r * g) % b:(r * g) % b + g], stats=False)
    torch.cuda.synchronize()
    st = hy.profile_read(dev)
    hy.profile_enable(dev, False)
    n = reps * g
    print(json.dumps({"group": g, "images": n, **{k: round(st[k][0] / n * 1e3, 2) for k in ("dwt", "sure", "idwt")}, "unit": "us per image"}))
