import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from harness import synth
from oracle import hyres_ref as O
import paper_2204_06979_b200 as hy
s = synth.low_rank_cube(64, 64, 32, rank=4, seed=11)
b, r, c = s.clean.shape; n = r * c
g = O.gram(s.clean)
sig_ref, _ = O.estimate_noise(s.clean)
lam_ref, v_ref, _ = O.whiten_eig(g, sig_ref, n)
sig, lam, V = hy.stages.eig(torch.from_numpy(g).cuda(), n, 8)
sig, lam, V = sig.cpu().numpy(), lam.cpu().numpy(), V.cpu().numpy()
print("sigma rel err", np.max(np.abs(sig / sig_ref - 1)))
print("lam ref", lam_ref[:8]); print("lam got", lam[:8])
for j in range(6): print(j, np.max(np.abs(V[:, j] - v_ref[:, j])))
for name in ["tiny", "small"]:
    s = synth.make_cube(name, 0); b, r, c = s.noisy.shape; n = r * c
    g = O.gram(s.noisy); sig_ref, _ = O.estimate_noise(s.noisy); lam_ref, v_ref, _ = O.whiten_eig(g, sig_ref, n)
    sig, lam, V = hy.stages.eig(torch.from_numpy(g).cuda(), n, 8)
    sig, lam, V = sig.cpu().numpy(), lam.cpu().numpy(), V.cpu().numpy()
    print(name, "sigma", np.max(np.abs(sig / sig_ref - 1)), "lam", np.max(np.abs(lam - lam_ref)) / lam_ref[0],
          [float(np.max(np.abs(V[:, j] - v_ref[:, j]))) for j in range(4)])
