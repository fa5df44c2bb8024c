"""Host<->device copy ceilings for the e2e path: pinned H2D, D2H, and both at once."""
import time
import torch

n = 134 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


t = timeit(h2d); print(f"H2D  {n / t / 1e9:6.1f} GB/s")
t = timeit(d2h); print(f"D2H  {n / t / 1e9:6.1f} GB/s")
t = timeit(both); print(f"both {2 * n / t / 1e9:6.1f} GB/s total ({t * 1e3:.2f} ms for {n >> 20} MiB each way)")


def both_chunked(mb):
    c = mb << 20
    for o in range(0, n, c):
        with torch.cuda.stream(s1):
            d_in[o:o + c].copy_(h_in[o:o + c], non_blocking=True)
        with torch.cuda.stream(s2):
            h_out[o:o + c].copy_(d_out[o:o + c], non_blocking=True)


for mb in (4, 16, 64):
    t = timeit(lambda: both_chunked(mb))
    print(f"both, {mb:2d} MiB chunks: {2 * n / t / 1e9:6.1f} GB/s total")
