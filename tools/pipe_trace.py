"""Diagnostics: kernel timeline of the host-input pipeline (needs a -DAQR_TRACE
build: AQR_LIB_PATH=build_ab/libaqr_trace.so)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems, _lib
L = _lib.lib()
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2   # python tools/pipe_trace.py [method] [2|5]
GAP = 20000 if cfg == 2 else 500000                    # idle gaps reported (ns)
if cfg == 5:
    csr, Zd = problems.config5()
    m, n = Zd.shape
    op = aqr.CsrSpdOperator(*csr)
    Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t(); Zh.copy_(Zd)
    del csr, Zd
    torch.cuda.empty_cache()
else:
    (ip, ix, dv), Z = problems.config2(device=False)
    m, n = Z.shape
    op = aqr.CsrSpdOperator(ip, ix, dv)
    Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t(); Zh.copy_(torch.from_numpy(Z))
meth = sys.argv[1] if len(sys.argv) > 1 else "mgs-ha-row"
if len(sys.argv) > 3 and sys.argv[3] == "numpy":  # pageable numpy input (the bench's e2e form)
    Zh = np.asfortranarray(np.array(Zh.numpy(), order="F", copy=True))
    print("input: pageable numpy", flush=True)
for _ in range(2 if cfg == 5 else 3):
    r = aqr.factorize(Zh, op, meth)
    del r
buf = np.zeros(3 * 16384, dtype=np.uint64)
k0 = L.aqr_trace_read(buf.ctypes.data, 16384)
t0 = time.perf_counter()
r = aqr.factorize(Zh, op, meth)
t1 = time.perf_counter()
k = L.aqr_trace_read(buf.ctypes.data, 16384)
t = buf[: 3 * k].reshape(k, 3)[k0:].astype(np.int64)
start, end = t[:, 1], t[:, 2]
base = start[0]
print(f"{meth}: wall {1e3 * (t1 - t0):.2f} ms, {len(t)} traced launches, first start -> last end "
      f"{(end[-1] - base) / 1e6:.2f} ms, busy {(end - start).sum() / 1e6:.2f} ms")
# idle gaps > 20 us (config 5: 0.5 ms) between traced kernels (waiting for H2D chunks, untraced kernels)
gaps = [(i, (start[i] - end[i - 1]) / 1e3, (start[i] - base) / 1e6) for i in range(1, len(t)) if start[i] - end[i - 1] > GAP]
for i, g, at in gaps:
    print(f"  idle {g:8.1f} us before launch {i} at {at:.2f} ms")
dur = (end - start) / 1e3
print(f"  launches by duration: >200us {int((dur > 200).sum())}, median {np.median(dur):.1f} us; "
      f"last kernel end {(end[-1] - base) / 1e6:.2f} ms after first start")
# where the busy time goes: first / second half of the span
half = base + (end[-1] - base) // 2
print(f"  busy in first half {dur[start < half].sum() / 1e3:.2f} ms, second half {dur[start >= half].sum() / 1e3:.2f} ms")
# busy time per 100 ms of the span (config 5)
if cfg == 5:
    span = (end[-1] - base) / 1e6
    for w0 in range(0, int(span) + 1, 100):
        lo, hi = base + w0 * 1e6, base + (w0 + 100) * 1e6
        b = (np.minimum(end, hi) - np.maximum(start, lo)).clip(min=0).sum() / 1e6
        print(f"  {w0:5d}-{w0 + 100:5d} ms: traced kernels busy {b:6.1f} ms, launches started {int(((start >= lo) & (start < hi)).sum())}")
for i in range(len(t) if cfg == 2 else 0):
    if dur[i] > 60 or (i > 0 and start[i] - end[i - 1] > 20000):
        print(f"  launch {i:3d} start {(start[i] - base) / 1e6:6.2f} ms dur {dur[i]:7.1f} us"
              f" gap-before {(start[i] - end[i - 1]) / 1e3 if i else 0:7.1f} us")
