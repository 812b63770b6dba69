"""Diagnostics: kernel durations and gaps of one device-resident factorization,
alone and with a concurrent H2D copy stream (needs a -DAQR_TRACE build:
AQR_LIB_PATH=build_ab/libaqr_trace.so).  argv: method, copy MB, copy count."""
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
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cnt = int(sys.argv[3]) if len(sys.argv) > 3 else 60
nel = mb * 1024 * 1024 // 8
h1 = torch.empty(nel, dtype=torch.float64).pin_memory()
d1 = torch.empty(nel, dtype=torch.float64, device="cuda")
s1 = torch.cuda.Stream()
for _ in range(3):
    aqr.factorize(Zd, op, meth)
torch.cuda.synchronize()
buf = np.zeros(3 * 16384, dtype=np.uint64)
for lab in ("alone", f"with H2D {cnt} x {mb} MB", "alone"):
    if lab != "alone":
        with torch.cuda.stream(s1):
            for _ in range(cnt):
                d1.copy_(h1, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(s1)
    k0 = L.aqr_trace_read(buf.ctypes.data, 16384)
    if os.environ.get("TIMER"):
        L.aqr_trailing_timer_enable(1)
    aqr.factorize(Zd, op, meth)
    busy = not ev.query()
    torch.cuda.synchronize()
    L.aqr_trailing_timer_enable(0)
    k = L.aqr_trace_read(buf.ctypes.data, 16384)
    t = buf[: 3 * k].reshape(k, 3)[k0:].astype(np.int64)
    pre, start, end = t[:, 0], t[:, 1], t[:, 2]
    dur = (end - start) / 1e3
    gap = (start[1:] - end[:-1]) / 1e3
    print(f"{lab}: {len(t)} launches, span {(end[-1] - start[0]) / 1e3:.1f} us, busy {dur.sum():.1f} us, "
          f"gaps {gap.sum():.1f} us (median {np.median(gap):.2f}, max {gap.max():.2f}); "
          f"mean dur even/odd {dur[0::2].mean():.2f} / {dur[1::2].mean():.2f} us; copies busy after: {busy}")
    torch.cuda.synchronize()
