"""The bench's e2e form (pageable numpy Z in, numpy Q / R out) called K
times in a row on config 5; prints every call's wall time.

    python tools/e2e_repeat.py [method] [K]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems

meth = sys.argv[1] if len(sys.argv) > 1 else "mgs-hp-row"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
csr, Zd = problems.config5()
op = aqr.CsrSpdOperator(*csr)
del csr
Zh = np.asfortranarray(Zd.t().cpu().numpy().T)
del Zd
torch.cuda.empty_cache()
from paper_1703_10440_b200 import _device as D

# AQR_STAGE_THREADS=a,b,...: repeat the series with these host staging pool sizes
for threads in [int(x) for x in os.environ.get("AQR_STAGE_THREADS", "0").split(",")]:
    if threads:
        D._STAGE_THREADS = threads
        D._pools.clear()
    times = []
    for k in range(K + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = aqr.factorize(Zh, op, meth)
        times.append(time.perf_counter() - t0)
        del r
    print(f"staging threads {D._STAGE_THREADS}:", " ".join(f"{1e3 * t:.0f}" for t in times), "ms (first = warm-up)",
          flush=True)
