"""Config 5 HP end to end vs device-resident: where the time goes.

    python tools/e2e_cfg5.py [method] [chunk_cols...]

Times (wall clock, after a warm call): device-resident Z; page-locked torch
Z in / host Q out (aqr_gs_factor_pinned, no host staging); pageable numpy
Z in / numpy out (the bench's e2e form).  With the library's kernel timer
on, the per-slot kernel times of the pinned call show how much device work
the chunked pipeline adds (catch-ups, chunked block applies)."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems, _lib

L = _lib.lib()
meth = sys.argv[1] if len(sys.argv) > 1 else "mgs-hp-row"
chunks = [int(c) for c in sys.argv[2:]] or [0]
csr, Zd = problems.config5()
op = aqr.CsrSpdOperator(*csr)
del csr
m, n = Zd.shape


def wall(f, reps=1):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
        del r
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def slots():
    out = {}
    for slot, name in ((0, "trailing"), (2, "col_update"), (3, "x_catchup"), (4, "block_apply"), (5, "chunk_catchup")):
        k, ms, b = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        L.aqr_kernel_timer_read(slot, ctypes.byref(k), ctypes.byref(ms), ctypes.byref(b))
        if k.value:
            out[name] = round(ms.value, 1)
    return out


res = {"device_ms": wall(lambda: aqr.factorize(Zd, op, meth))}
Zp = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
Zp.copy_(Zd)
Zh = np.asfortranarray(Zp.numpy())  # numpy view of PAGE-LOCKED memory
Zpg = np.asfortranarray(Zd.t().cpu().numpy().T)  # pageable numpy (the bench's e2e form)
del Zd
torch.cuda.empty_cache()
for c in chunks:
    if c:
        os.environ["AQR_CHUNK_COLS"] = str(c)
    res[f"pinned_ms_chunk{c}"] = wall(lambda: aqr.factorize(Zp, op, meth))
    L.aqr_trailing_timer_enable(1)
    aqr.factorize(Zp, op, meth)
    torch.cuda.synchronize()
    L.aqr_trailing_timer_enable(0)
    res[f"pinned_slots_chunk{c}"] = slots()
    res[f"numpy_pinned_src_ms_chunk{c}"] = wall(lambda: aqr.factorize(Zh, op, meth))
    res[f"numpy_pageable_ms_chunk{c}"] = wall(lambda: aqr.factorize(Zpg, op, meth), 2)
print(json.dumps(res))
