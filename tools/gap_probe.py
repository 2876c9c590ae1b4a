"""Where does ms/step go beyond the sum of stage times?  Times the hyres loop with
profiling off/on and the host-side duration of each call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from harness import synth
import paper_2204_06979_b200 as hy
name = sys.argv[1] if len(sys.argv) > 1 else "large"
s = synth.make_cube(name, 0)
cube = torch.from_numpy(s.noisy).cuda(); out = torch.empty_like(cube)
for _ in range(5): hy.hyres(cube, out)
torch.cuda.synchronize()
def loop(k, prof):
    hy.profile_enable(0, prof)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); hs = []
    for _ in range(k):
        t = time.perf_counter(); hy.hyres(cube, out); hs.append(time.perf_counter() - t)
    e1.record(); torch.cuda.synchronize()
    st = hy.profile_read(0) if prof else None
    hy.profile_enable(0, False)
    return e0.elapsed_time(e1) / k, np.median(hs) * 1e3, st
for prof in (False, True, False):
    ms, host, st = loop(20, prof)
    print(f"prof={prof}: {ms:.3f} ms/step (events), host per call {host:.3f} ms")
    if st: print("   stage sum %.3f ms" % (sum(v[0] for v in st.values()) / 20), {k: round(v[0] / 20, 3) for k, v in st.items()})
# pure GPU time: capture-free estimate = enqueue everything without sync? measure host cost of the pieces
import ctypes
t = time.perf_counter()
for _ in range(20): hy._lib.lib().hyde_launch_count(hy.handle(0))
print("ctypes call overhead %.1f us" % ((time.perf_counter() - t) / 20 * 1e6))
