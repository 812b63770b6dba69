"""Diagnostics: plain SpMV / SpMM timing on config 2 (device-resident)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems
(ip, ix, dv), Z = problems.config2(device=False)
op = aqr.CsrSpdOperator(ip, ix, dv)
x = torch.randn(op.dim, dtype=torch.float64, device="cuda")
X = torch.randn((8, op.dim), dtype=torch.float64, device="cuda").t()
def bench(f, k=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3
print("spmv us", bench(lambda: op.apply(x)))
print("spmm k=8 us", bench(lambda: op.apply_block(X), 10))
y = torch.empty_like(x)
print("copy 8MB us", bench(lambda: y.copy_(x)))
print("empty launch-ish (fill 8MB) us", bench(lambda: y.fill_(1.0)))
