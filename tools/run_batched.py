"""Run hyde_hyres_batched on the `batched` config (64 x 256x256x191) a few times (profiling driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from harness import synth
import paper_2204_06979_b200 as hy
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 64
x = torch.stack([torch.from_numpy(synth.make_cube("batched", s).noisy) for s in range(nb)]).cuda()
for _ in range(reps):
    out = hy.hyres_batched(x)
torch.cuda.synchronize()
print("ok", tuple(out.shape))
