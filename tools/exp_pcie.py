# Pinned host <-> device copy bandwidth of the e2e path: 3.2 GB each way, alone and together.
import time
import torch
n = 400 * 1_000_000
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    th = t(lambda: d1.copy_(h1, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    tb = t(both)
    GB = n * 8 / 1e9
    print(f"H2D {GB/th:.1f} GB/s ({th*1e3:.1f} ms)  D2H {GB/td:.1f} GB/s ({td*1e3:.1f} ms)  both {tb*1e3:.1f} ms")
