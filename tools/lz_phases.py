"""Phase-2L (Lanczos) cycle split of the K2 cluster kernel inside hyres (CTA 0)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from harness import synth
import paper_2204_06979_b200 as hy
name = sys.argv[1] if len(sys.argv) > 1 else "large"
s = synth.make_cube(name, 0)
cube = torch.from_numpy(s.noisy).cuda()
out = torch.empty_like(cube)
for _ in range(3):
    _, info = hy.hyres(cube, out, return_info=True)
torch.cuda.synchronize()
z = (ctypes.c_longlong * 40)()
hy._lib.lib().hyde_debug_eig_clocks(z)   # reset the accumulators: one more call
lib = hy._lib.lib()
_, info = hy.hyres(cube, out, return_info=True)
torch.cuda.synchronize()
clk = (ctypes.c_longlong * 40)()
hy._lib.lib().hyde_debug_eig_clocks(clk)
print(name, info)
print("  sweep %.1f us, after sweep -> end %.1f us" % ((clk[1] - clk[0]) / 1.965e3, (clk[4] - clk[1]) / 1.965e3))
for nm, i in [("matvec+send", 20), ("wait", 21), ("cgs2", 22), ("ritz checks", 23)]:
    print("  %-12s %9d cycles (%.1f us)" % (nm, clk[i], clk[i] / 1.965e3))
print("  steps %d converged %d" % (clk[24], clk[25]))
print("  cgs: dots %d, sync %d, update %d, sync %d cycles" % (clk[29], clk[30], clk[31], clk[32] if len(clk) > 32 else -1))
print("  ritz bounds/scale %d, bisect %d, twisted %d cycles (accumulated over calls)" % (clk[28], clk[26], clk[27]))
