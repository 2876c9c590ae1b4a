"""Per-phase SM-cycle split of the K2 cluster kernel (CTA 0 of the cluster)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from harness import synth
import paper_2204_06979_b200 as hy
from oracle import hyres_ref as O
name = sys.argv[1] if len(sys.argv) > 1 else "large"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = synth.make_cube(name, 0)
b, r, c = s.noisy.shape
g = torch.from_numpy(O.gram(s.noisy)).cuda()
for rep in range(3):
    sig, lam, V = hy.stages.eig(g, r * c, k, all_lam=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for rep in range(10):
    sig, lam, V = hy.stages.eig(g, r * c, k, all_lam=False)
e1.record(); torch.cuda.synchronize()
clk = (ctypes.c_longlong * 40)()
hy._lib.lib().hyde_debug_eig_clocks(clk)
print(name, "B=%d K=%d: K2 %.1f us per call (CUDA events)" % (b, k, e0.elapsed_time(e1) / 10 * 1e3))
for nm, a, bb in [("sweep (sigma)", 0, 1), ("whiten+tridiag", 1, 2), ("eigenpairs", 2, 3), ("vectors", 3, 4)]:
    print("  %-24s %9d cycles (%.1f us)" % (nm, clk[bb] - clk[a], (clk[bb] - clk[a]) / 1.965e3))
for nm, i in [("sweep gather", 5), ("sweep cl_sync", 6), ("sweep Pinv", 7), ("sweep Z", 8), ("sweep wi loads", 15), ("sweep upd+send next", 18), ("sweep update rest", 9),
              ("tri symv+send", 10), ("tri Q update", 11), ("tri wait", 12), ("tri update", 13), ("tri reflector", 14), ("bisection", 16), ("inverse iteration", 17)]:
    print("  %-24s %9d cycles" % (nm, clk[i]))
