"""Diagnostics: H2D / D2H bandwidth of 537 MB page-locked transfers split
over k concurrent streams (k copy engines), alone and both directions."""
import time
import torch

n = 537 * 1024 * 1024 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(h2d, d2h, k, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        part = (n + k - 1) // k
        for j in range(k):
            sl = slice(j * part, min(n, (j + 1) * part))
            if h2d:
                with torch.cuda.stream(streams[j]):
                    d1[sl].copy_(h1[sl], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[4 + j if k <= 4 else j]):
                    h2[sl].copy_(d2[sl], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for k in (1, 2, 4):
    for lab, a, b in (("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)):
        ms = run(a, b, k)
        print(f"k={k} {lab}: {ms:.2f} ms ({(a + b) * n * 8 / ms / 1e6:.1f} GB/s total)")
