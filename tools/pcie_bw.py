"""Pinned host <-> device copy bandwidth, one direction at a time and both
concurrently (the e2e decode's transfer ceiling)."""
import time

import torch

n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return n * reps / (time.perf_counter() - t0) / 1e9


print(f"H2D {bw(lambda: d_a.copy_(h_in, non_blocking=True)):.1f} GB/s")
print(f"D2H {bw(lambda: h_out.copy_(d_b, non_blocking=True)):.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


print(f"H2D + D2H concurrently, per direction {bw(both):.1f} GB/s")
