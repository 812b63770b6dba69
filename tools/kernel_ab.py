"""A/B of kernel variants (AQR_TRAIL_VARIANT) on config 2: per-kernel CUDA-event times."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems, _lib
L = _lib.lib()
(ip, ix, dv), Z = problems.config2(device=False)
op = aqr.CsrSpdOperator(ip, ix, dv)
Zd = torch.from_numpy(Z.T).cuda().t()
meth = sys.argv[1] if len(sys.argv) > 1 else "mgs-ha-row"
for _ in range(3):
    aqr.factorize(Zd, op, meth)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(); K = 5
for _ in range(K):
    aqr.factorize(Zd, op, meth)
ev1.record(); torch.cuda.synchronize()
step = ev0.elapsed_time(ev1) / K
L.aqr_trailing_timer_enable(1)
for _ in range(K):
    aqr.factorize(Zd, op, meth)
torch.cuda.synchronize()
out = {"variant": os.environ.get("AQR_TRAIL_VARIANT", "0"), "method": meth, "step_ms": step}
for slot, name in ((0, "trailing"), (1, "spmv_step"), (2, "col_update"), (3, "spmv_trail")):
    n, ms, b = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.aqr_kernel_timer_read(slot, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(b))
    if n.value:
        out[name] = {"ms_per_fact": ms.value / K, "us_per_launch": 1e3 * ms.value / n.value,
                     "GBps": b.value / (ms.value / 1e3) / 1e9}
L.aqr_trailing_timer_enable(0)
print(json.dumps(out))
if os.environ.get("AQR_LIST"):
    import numpy as np
    L.aqr_trailing_timer_enable(1)
    aqr.factorize(Zd, op, meth)
    torch.cuda.synchronize()
    ms = np.zeros(512); by = np.zeros(512)
    k = L.aqr_kernel_timer_list(0, ms.ctypes.data, by.ctypes.data, 512)
    for j in range(k):
        print(f"launch {j:3d} us {1e3*ms[j]:8.1f} MB {by[j]/1e6:8.1f} GB/s {by[j]/(ms[j]/1e3)/1e9:7.0f} ideal_us {by[j]/6554.9e9*1e6:7.1f}")
    L.aqr_trailing_timer_enable(0)
