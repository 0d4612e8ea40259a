"""e2e (host-buffer C-ABI call) timing of config 2, as bench.py measures it."""
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200.inputs import skew_lower
N = 4096
x = skew_lower(N, 0)
x_pin = torch.empty((N, N), dtype=torch.float64).pin_memory()
x_pin.copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
L_pin = torch.zeros((N, N), dtype=torch.float64).pin_memory()
tau_pin = torch.empty(N - 1, dtype=torch.float64).pin_memory(); piv_pin = torch.empty(N, dtype=torch.int64).pin_memory()
xh = x_pin.numpy().T; out = (L_pin.numpy().T, tau_pin.numpy(), piv_pin.numpy())
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for it in range(8):
    flush.zero_(); torch.cuda.synchronize()
    e0.record(); pk.ltlt_blk_piv_host(xh, 128, "var1", out=out, sync=False); e1.record(); torch.cuda.synchronize()
    if it >= 2: ts.append(e0.elapsed_time(e1))
print(f"e2e {np.mean(ts):.3f} ms  pivots-ok={bool((piv_pin.numpy() >= 0).all())}")
