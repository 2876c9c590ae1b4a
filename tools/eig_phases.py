"""Print the per-phase SM-cycle split of the K2 (noise + eigen) kernel for a config."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from harness import synth
import paper_2204_06979_b200 as hy
from oracle import hyres_ref as O
name = sys.argv[1] if len(sys.argv) > 1 else "large"
s = synth.make_cube(name, 0)
b, r, c = s.noisy.shape
g = torch.from_numpy(O.gram(s.noisy)).cuda()
for rep in range(3):
    sig, lam, V = hy.stages.eig(g, r * c, 16, all_lam=False)
torch.cuda.synchronize()
clk = (ctypes.c_longlong * 8)()
hy._lib.lib().hyde_debug_eig_clocks(clk)
names = ["sweep", "tridiag", "eigenvalues", "inv_iter", "backtransform"]
tot = clk[5] - clk[0]
print(name, "B=%d total %d cycles (%.1f us at 1.9 GHz)" % (b, tot, tot / 1.9e3))
for i, nm in enumerate(names):
    d = clk[i + 1] - clk[i]
    print("  %-14s %9d cycles %6.1f%%" % (nm, d, 100.0 * d / tot))
