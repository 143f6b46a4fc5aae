"""GPU probe (not collected): pinned host <-> device copy bandwidth, each direction alone and
both at once (the e2e pipeline's floor)."""
import torch
n = 1_250_000_000 // 4
h_in = torch.empty(n, pin_memory=True); h_out = torch.empty(n, pin_memory=True)
d_in = torch.empty(n, device="cuda"); d_out = torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
def h2d():
    d_in.copy_(h_in, non_blocking=True)
def d2h():
    h_out.copy_(d_out, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn); print(name, f"{ms:.2f} ms", f"{1.25/ (ms*1e-3):.1f} GB/s per direction")
