"""Diagnostics: gaps between the fused SpMV-step and trailing kernels of one
factorization (needs a -DAQR_TRACE build: AQR_LIB_PATH=build_ab/libaqr_trace.so)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
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
n0 = L.aqr_trace_read(None, 0) if False else None
buf = np.zeros(3 * 16384, dtype=np.uint64)
k0 = L.aqr_trace_read(buf.ctypes.data, 16384)
aqr.factorize(Zd, op, meth)
torch.cuda.synchronize()
k = L.aqr_trace_read(buf.ctypes.data, 16384)
t = buf[: 3 * k].reshape(k, 3)[k0:].astype(np.int64)
pre, start, end = t[:, 0], t[:, 1], t[:, 2]
dur = (end - start) / 1e3
gap = (start[1:] - end[:-1]) / 1e3
early = (start[1:] - pre[1:]) / 1e3
print(f"{meth}: {len(t)} launches, span {(end[-1] - start[0]) / 1e3:.1f} us, busy {dur.sum():.1f} us, "
      f"gaps {gap.sum():.1f} us (mean {gap.mean():.2f}, median {np.median(gap):.2f}, max {gap.max():.2f})")
print("  mean wait after early start:", round(float(early.mean()), 2), "us")
print("  mean duration by kind (even = norm step, odd = trailing):",
      round(float(dur[0::2].mean()), 2), round(float(dur[1::2].mean()), 2))
print("  gap after norm step / after trailing:", round(float(gap[0::2].mean()), 2), round(float(gap[1::2].mean()), 2))
