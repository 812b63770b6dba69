"""Diagnostics: the host-input pipeline (aqr_gs_factor_pinned) on config 2."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems, _lib
L = _lib.lib()
(ip, ix, dv), Z = problems.config2(device=False)
m, n = Z.shape
op = aqr.CsrSpdOperator(ip, ix, dv)
Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t(); Zh.copy_(torch.from_numpy(Z))
meth = sys.argv[1] if len(sys.argv) > 1 else "mgs-ha-row"
for c in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,16,8,4").split(",")]:
    os.environ["AQR_CHUNK_COLS"] = str(c)
    r = aqr.factorize(Zh, op, meth); r = aqr.factorize(Zh, op, meth); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); r = aqr.factorize(Zh, op, meth); ts.append(time.perf_counter() - t0)
    L.aqr_trailing_timer_enable(1)
    r = aqr.factorize(Zh, op, meth); torch.cuda.synchronize()
    ms = np.zeros(4096); by = np.zeros(4096)
    k = L.aqr_kernel_timer_list(0, ms.ctypes.data, by.ctypes.data, 4096)
    L.aqr_trailing_timer_enable(0)
    print(f"chunk {c} {meth}: median {1e3*np.median(ts):.2f} ms min {1e3*min(ts):.2f}; trailing launches {k} "
          f"sum {ms[:k].sum():.2f} ms", flush=True)
    if os.environ.get("AQR_LIST"):
        for j in range(k):
            print(f"  launch {j:4d} {1e3 * ms[j]:8.1f} us {by[j] / 1e6:8.1f} MB")
