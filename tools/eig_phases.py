"""Print the per-phase SM-cycle split of the K2 (noise + eigen) kernels for a config."""
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for rep in range(10):
    sig, lam, V = hy.stages.eig(g, r * c, 16, all_lam=False)
e1.record(); torch.cuda.synchronize()
clk = (ctypes.c_longlong * 16)()
hy._lib.lib().hyde_debug_eig_clocks(clk)
print(name, "B=%d: K2 (chol+invdiag+tridiag+16 eigpairs) %.1f us per call (CUDA events)" % (b, e0.elapsed_time(e1) / 10 * 1e3))
for nm, a, bb in [("cholesky", 0, 1), ("tridiag", 2, 3), ("eigpair: bisection", 4, 5), ("eigpair: inv_iter", 5, 6), ("eigpair: backtransform", 6, 7)]:
    print("  %-24s %9d cycles (%.1f us)" % (nm, clk[bb] - clk[a], (clk[bb] - clk[a]) / 1.9e3))
for nm, i in [("chol panel block", 8), ("chol panel rows", 9), ("chol trailing", 10), ("tridiag column", 11), ("tridiag symv", 12), ("tridiag update", 13)]:
    print("  %-24s %9d cycles" % (nm, clk[i]))
