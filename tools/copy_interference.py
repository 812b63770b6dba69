"""Diagnostics: device-resident factorization (and its trailing kernels) with
concurrent PCIe copies on other streams."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems, _lib
L = _lib.lib()
(ip, ix, dv), Z = problems.config2(device=False)
op = aqr.CsrSpdOperator(ip, ix, dv)
Zd = torch.from_numpy(Z.T).cuda().t()
n = 64 * 1024 * 1024 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
aqr.mgs_ha(Zd, op, "row"); torch.cuda.synchronize()
def fact(h2d, d2h, k=3):
    for _ in range(60):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c1, c2 = torch.cuda.Event(), torch.cuda.Event()
    c1.record(s1); c2.record(s2)
    L.aqr_trailing_timer_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): aqr.mgs_ha(Zd, op, "row")
    e1.record(); e1.synchronize()
    busy = (not c1.query()) or (not c2.query())
    nl, ms, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.aqr_kernel_timer_read(0, ctypes.byref(nl), ctypes.byref(ms), ctypes.byref(by))
    L.aqr_trailing_timer_enable(0)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k, ms.value / k, busy
for lab, a, b in (("alone", 0, 0), ("with H2D", 1, 0), ("with D2H", 0, 1), ("with both", 1, 1)):
    t, tr, busy = fact(a, b)
    print(f"{lab}: factorization {t:.3f} ms, trailing {tr:.3f} ms, copies still running at end: {busy}")
