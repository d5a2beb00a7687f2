"""PCIe bandwidth of this box with pinned host memory: H2D alone, D2H alone, and both
directions at once on two streams (the bound for la_host_step's e2e number)."""
import torch

n = 1 << 30  # 1 GiB per transfer
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
t_both = timed(both)
print(f"H2D {n / t_h2d / 1e9:.1f} GB/s, D2H {n / t_d2h / 1e9:.1f} GB/s, concurrent {n / t_both / 1e9:.1f} GB/s each direction")
