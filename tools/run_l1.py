"""Run the HyMiNoR l1 stage on the large cube's HyRes output (profiling driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from harness import synth
import paper_2204_06979_b200 as hy
s = synth.make_cube(sys.argv[1] if len(sys.argv) > 1 else "large", 0)
x = torch.from_numpy(s.noisy).cuda()
m = hy.hyres(x)
out = torch.empty_like(m)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    hy.l1_spectral(m, out)
torch.cuda.synchronize()
print("ok")
