"""Host<->device copy bandwidth from pinned memory on this box (the e2e
path's H2D of 2-bit reads and D2H of hit records), alone and with both
directions at once."""
import torch

def bw(n, direction, reps=20):
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        e1.record(s)
    e1.synchronize()
    return n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9

for n in (16 << 20, 25 << 20, 256 << 20):
    print(f"{n >> 20} MiB: H2D {bw(n, 'h2d'):.1f} GB/s, D2H {bw(n, 'd2h'):.1f} GB/s")
