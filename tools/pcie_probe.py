import torch, time
n = 940 * 1024 * 1024 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
b = n * 4 / 1e9
th = t(lambda: d.copy_(h, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
tb = t(both)
print(f"H2D {b/th:.1f} GB/s  D2H {b/td:.1f} GB/s  both concurrent {2*b/tb:.1f} GB/s total ({tb*1e3:.1f} ms for {b:.2f} GB each way)")
print(torch.cuda.get_device_name(), torch.cuda.get_device_properties(0))
