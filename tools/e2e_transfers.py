"""Diagnostics: host<->device transfer costs of the e2e path (config 2 sizes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems
(ip, ix, dv), Z = problems.config2(device=False)
m, n = Z.shape
op = aqr.CsrSpdOperator(ip, ix, dv)
Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t(); Zh.copy_(torch.from_numpy(Z))
def t(f, k=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
Zd = Zh.to("cuda")
Qh = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
print("H2D pinned ms", t(lambda: Zh.to("cuda", non_blocking=True)))
print("D2H pinned ms", t(lambda: Qh.copy_(Zd, non_blocking=True)))
print("pin alloc+D2H ms", t(lambda: torch.empty((n, m), dtype=torch.float64, pin_memory=True).t().copy_(Zd)))
print("factorize dev ms", t(lambda: aqr.mgs_ha(Zd, op, "row")))
print("factorize pinned ms", t(lambda: aqr.mgs_ha(Zh, op, "row")))
print("factorize numpy ms", t(lambda: aqr.mgs_ha(Z, op, "row"), 2))
