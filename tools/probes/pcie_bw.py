"""PCIe ceiling for the e2e path: pinned H2D / D2H of the config-2 lower-triangle bytes (69 MB),
one contiguous copy vs the driver's 32 column-block 2-D copies, one and two streams."""
import torch, time
n = 4096
nbytes = sum((n - j0) * min(128, n - j0) for j0 in range(0, n, 128)) * 8
h = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
H = torch.empty((n, n), dtype=torch.float64).pin_memory()
D = torch.empty((n, n), dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: d.copy_(h, non_blocking=True)); print(f"H2D contiguous {nbytes/1e6:.1f} MB: {ms:.3f} ms {nbytes/ms/1e6:.1f} GB/s")
ms = t(lambda: h.copy_(d, non_blocking=True)); print(f"D2H contiguous: {ms:.3f} ms {nbytes/ms/1e6:.1f} GB/s")
ms = t(lambda: D.copy_(H, non_blocking=True)); print(f"H2D full 134 MB: {ms:.3f} ms {n*n*8/ms/1e6:.1f} GB/s")
