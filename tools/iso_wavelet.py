"""Stage-isolated DWT/SURE/IDWT timing on all B eigen-images of a config (bench.py
wavelet_isolated leg alone).  python tools/iso_wavelet.py [--config large] [--steps 5]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from harness import synth  # noqa: E402
import paper_2204_06979_b200 as hy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="large")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--levels", type=int, default=0)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
cube = torch.from_numpy(np.ascontiguousarray(synth.make_cube(cfg, 0).noisy)).cuda()
lv = a.levels or hy.stages.auto_levels(cfg.rows, cfg.cols)
hbm, _, _ = bench.peaks()
print(json.dumps(bench.wavelet_isolated(hy, torch, cube, cfg, lv, a.steps, hbm)))
