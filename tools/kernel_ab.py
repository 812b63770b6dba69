"""A/B of schedule knobs: per-slot kernel times of one factorization.

    AQR_LIB_PATH=paper_1703_10440_b200/libaqr_b200_exp.so AQR_TRAIL_WIN=4 \
        python tools/kernel_ab.py [method] [config 2|3|5] [reps]

AQR_BANDED=0 builds the operator without the banded view (plain CSR kernels).

Prints one JSON line: the step time (CUDA events, K factorizations back to
back) and, from a second pass with the library's kernel timer on, per slot
(0 trailing pass, 1 fused SpMV step, 2 column update + norm, 3 HP X
catch-up) the time per factorization, per launch and the algorithmic GB/s.
"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems, _lib
L = _lib.lib()
meth = sys.argv[1] if len(sys.argv) > 1 else "mgs-ha-row"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
K = int(sys.argv[3]) if len(sys.argv) > 3 else (5 if cfg == 2 else 2)
banded = None if os.environ.get("AQR_BANDED", "1") != "0" else False  # 0: plain CSR kernels
if cfg == 5:
    csr, Zd = problems.config5()
    op = aqr.CsrSpdOperator(*csr, banded=banded)
    del csr
else:
    (ip, ix, dv), Z = problems.config3(device=False) if cfg == 3 else problems.config2(device=False)
    op = aqr.CsrSpdOperator(ip, ix, dv, banded=banded)
    Zd = torch.from_numpy(Z.T).cuda().t()
for _ in range(2 if cfg == 5 else 3):
    r = aqr.factorize(Zd, op, meth)
    del r
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(K):
    r = aqr.factorize(Zd, op, meth)
    del r
ev1.record(); torch.cuda.synchronize()
step = ev0.elapsed_time(ev1) / K
L.aqr_trailing_timer_enable(1)
for _ in range(K):
    r = aqr.factorize(Zd, op, meth)
    del r
torch.cuda.synchronize()
knobs = {k: v for k, v in os.environ.items() if k.startswith("AQR_")}
out = {"knobs": knobs, "method": meth, "config": cfg, "band": op.band_offsets is not None, "step_ms": step}
for slot, name in ((0, "trailing"), (1, "spmv_step"), (2, "col_update"), (3, "x_catchup"), (4, "block_apply")):
    n, ms, b = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.aqr_kernel_timer_read(slot, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(b))
    if n.value:
        out[name] = {"ms_per_fact": ms.value / K, "us_per_launch": 1e3 * ms.value / n.value,
                     "GBps": b.value / (ms.value / 1e3) / 1e9}
L.aqr_trailing_timer_enable(0)
print(json.dumps(out))
