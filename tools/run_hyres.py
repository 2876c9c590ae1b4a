"""Run hyres on one synthetic config a few times (profiling / debug driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from harness import synth
import paper_2204_06979_b200 as hy
name = sys.argv[1] if len(sys.argv) > 1 else "large"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = synth.make_cube(name, 0)
cube = torch.from_numpy(s.noisy).cuda()
out = torch.empty_like(cube)
for _ in range(reps):
    _, info = hy.hyres(cube, out, return_info=True)
torch.cuda.synchronize()
print(info, flush=True)
