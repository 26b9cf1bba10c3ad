"""Host<->device copy bandwidth on the GPU box: H2D alone, D2H alone, both directions at once
(pinned buffers, 4 GiB, CUDA events).  Bounds the e2e (host-buffer) solve throughput."""
import torch

n = 4 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


for s in (s1, s2):
    s.wait_stream(torch.cuda.current_stream())
timed(h2d)
t = timed(h2d)
print(f"H2D {n / t / 1e9:.1f} GB/s")
t = timed(d2h)
print(f"D2H {n / t / 1e9:.1f} GB/s")
t = timed(lambda: (h2d(), d2h()))
print(f"H2D+D2H concurrent: {2 * n / t / 1e9:.1f} GB/s total ({t * 1e3:.1f} ms for 2 x {n >> 30} GiB)")
