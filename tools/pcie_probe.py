"""Host<->device copy bandwidth from pinned memory (0.8 GB, the e2e vector size)."""
import torch
n = 100_000_000
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(2):
    d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
def t(fn):
    torch.cuda.synchronize(); e[0].record(); fn(); e[1].record(); torch.cuda.synchronize()
    return e[0].elapsed_time(e[1])
b = 8 * n / 1e9
ms = t(lambda: d.copy_(h, non_blocking=True)); print(f"H2D {b / ms * 1e3:.1f} GB/s")
ms = t(lambda: h.copy_(d, non_blocking=True)); print(f"D2H {b / ms * 1e3:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    s1.synchronize(); s2.synchronize()
ms = t(both); print(f"H2D || D2H {2 * b / ms * 1e3:.1f} GB/s aggregate")
def two_h2d():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    s1.synchronize(); s2.synchronize()
ms = t(two_h2d); print(f"2x H2D concurrent {2 * b / ms * 1e3:.1f} GB/s aggregate")
