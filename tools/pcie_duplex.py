"""Diagnostics: H2D and D2H bandwidth alone and concurrently (page-locked, 537 MB each;
`python tools/pcie_duplex.py MB` for another size)."""
import sys, torch, time
n = (int(sys.argv[1]) if len(sys.argv) > 1 else 537) * 1024 * 1024 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, k=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
for lab, a, b in (("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)):
    ms = run(a, b); print(f"{lab}: {ms:.2f} ms  ({(a + b) * n * 8 / ms / 1e6:.1f} GB/s total)")
