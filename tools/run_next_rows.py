"""Run the F1-F4 NEXT rows once each on the `large` cube (profiling driver for ncu):
python tools/run_next_rows.py [hysime|forpdn|wsrrr|hyminor|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import synth  # noqa: E402
import paper_2204_06979_b200 as hy  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
cube = torch.from_numpy(np.ascontiguousarray(synth.make_cube("large", 0).noisy)).cuda()
if what in ("hysime", "all"):
    print("hysime k", hy.hysime(cube)["k"])
if what in ("forpdn", "all"):
    print("forpdn lambda", hy.forpdn(cube, return_lambda=True)[1])
if what in ("wsrrr", "all"):
    print("wsrrr", hy.wsrrr(cube)["objective"])
if what in ("hyminor", "all"):
    h = hy.hyres(cube)
    print("l1 stage", float(hy.l1_spectral(h).abs().mean()))
torch.cuda.synchronize()
