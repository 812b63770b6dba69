"""Host staging throughput of the numpy e2e path: pageable numpy (config 5
size, 34 GB, F-ordered) -> page-locked block by the StagedHost thread pool,
for several pool sizes; and the plain pinned H2D / D2H rates of this box."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_10440_b200 import _device as D

m, n = 256 ** 3, int(sys.argv[1]) if len(sys.argv) > 1 else 256
Z = np.asfortranarray(torch.randn((n, m), dtype=torch.float64).numpy().T)  # pageable
print(f"os.cpu_count() = {os.cpu_count()}, Z {Z.nbytes / 1e9:.1f} GB", flush=True)
bounds = np.arange(0, n + 1, 8)
for threads in (8, 16, 32):
    D._STAGE_THREADS = threads
    D._pools.clear()
    for rep in range(2):
        t0 = time.perf_counter()
        st = D.StagedHost(Z, bounds)
        st.finish()
        dt = time.perf_counter() - t0
    print(f"staging {threads} threads: {dt:.3f} s = {Z.nbytes / dt / 1e9:.1f} GB/s", flush=True)
    del st
P = torch.empty((n, m), dtype=torch.float64).pin_memory()
G = torch.empty((n, m), dtype=torch.float64, device="cuda")
for name, f in (("H2D", lambda: G.copy_(P, non_blocking=True)), ("D2H", lambda: P.copy_(G, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter(); f(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name} pinned: {dt:.3f} s = {P.numel() * 8 / dt / 1e9:.1f} GB/s", flush=True)
