"""dev probe: write-only HBM bandwidth on this GPU (fill / memset of the obs-sized buffer)."""
import torch
n = 65536 * 8268
x = torch.empty(n, dtype=torch.float32, device="cuda")
for name, fn in [("fill_", lambda: x.fill_(1.0)), ("zero_", lambda: x.zero_()), ("copy", None)]:
    if fn is None:
        y = torch.empty_like(x)
        fn = lambda: y.copy_(x)
        nbytes = 2 * x.numel() * 4
    else:
        nbytes = x.numel() * 4
    for _ in range(5): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(50): fn()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 50
    print(f"{name}: {ms:.4f} ms  {nbytes / ms / 1e6:.1f} GB/s")
