"""Run the K1 Gram stage a few times on the `large` cube (profiling driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from harness import synth
import paper_2204_06979_b200 as hy
name = sys.argv[1] if len(sys.argv) > 1 else "large"
s = synth.make_cube(name, 0)
cube = torch.from_numpy(s.noisy).cuda()
for _ in range(3):
    g = hy.stages.gram(cube)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g = hy.stages.gram(cube)
e1.record(); torch.cuda.synchronize()
print(f"gram {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per call")
