"""Raw pinned-memory copy bandwidth on this box (H2D, D2H, both at once) for the e2e budget."""
import torch, time
n = 256 * 1024 * 1024  # 1 GiB of float32
h = torch.empty(n, pin_memory=True); h2 = torch.empty(n, pin_memory=True)
d = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(lambda: d.copy_(h, non_blocking=True)); print("H2D GB/s", 4 * n / ms / 1e6)
ms = t(lambda: h2.copy_(d2, non_blocking=True)); print("D2H GB/s", 4 * n / ms / 1e6)
ms = t(both); print("both GB/s each", 4 * n / ms / 1e6)
