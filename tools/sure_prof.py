"""K5 phase profile (needs a HYDE_SURE_PROF=1 build): SM cycles per phase summed
over CTAs for one hyde_wavelet_shrink over all B eigen-images of a config.
python tools/sure_prof.py [--config large]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import synth  # noqa: E402
import paper_2204_06979_b200 as hy  # noqa: E402
from paper_2204_06979_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--count", type=int, default=0)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
b, n = cfg.bands, cfg.rows * cfg.cols
cube = torch.from_numpy(np.ascontiguousarray(synth.make_cube(cfg, 0).noisy)).cuda()
G = hy.stages.gram(cube)
sigma, _, _ = hy.stages.eig(G, n, 1, all_lam=False)
_, V = torch.linalg.eigh(G / (sigma[:, None] * sigma[None, :]) / n)
W = (V.flip(1) / sigma[:, None]).to(torch.float32)
cnt = a.count or b
E = (W[:, :cnt].t() @ cube.view(b, n)).view(cnt, cfg.rows, cfg.cols).contiguous()
lv = hy.stages.auto_levels(cfg.rows, cfg.cols)
buf = (ctypes.c_ulonglong * 48)()
hy.stages.wavelet_shrink(E, lv, stats=False)
_lib.lib().hyde_debug_sure_prof(buf)
hy.stages.wavelet_shrink(E, lv, stats=False)
ok = _lib.lib().hyde_debug_sure_prof(buf)
v = list(buf)
print("profiling build:", bool(ok), "images", cnt)
for c, name in ((0, "n > 8192"), (1, "n <= 8192")):
    ctas = max(v[c * 8 + 3], 1)
    tot = sum(v[c * 8 + p] for p in range(3))
    print(f"{name:10s} CTAs {v[c*8+3]:6d}  window {v[c*8]/ctas:10.0f}  compaction {v[c*8+1]/ctas:10.0f}  "
          f"sort+eval {v[c*8+2]/ctas:10.0f} cycles/CTA; hist streaming {v[c*8+4]/ctas:10.0f}, passes {v[c*8+5]/ctas:.2f}, wait after hist {v[c*8+6]/ctas:.0f}, wait at ub exchange {v[c*8+7]/ctas:.0f}   (share of all CTA-cycles {tot / max(1, sum(v[0:3]) + sum(v[8:11])):.2f})")
print(f"window keys (long subbands): max {v[16]}, mean {v[17] / max(v[18], 1):.0f} over {v[18]} items; "
      f"longest sort+eval {v[19]} cycles (long), {v[20]} (short)")
print(f"CTA start spread {(v[22] - v[21]) / 1e3:.1f} us, first start -> last leader end {(v[23] - v[21]) / 1e3:.1f} us, "
      f"longest leader CTA lifetime {v[24]} cycles")
print("longest CTA per phase (cycles): long subbands window/compaction/sort", v[32:35], " short", v[40:43])
