"""Config 5's rows with n' columns through the host-input pipeline (numpy Z
in), for ncu captures of the chunk catch-up kernel:

    AQR_CHUNK_COLS=16 python tools/cfg5_pipe_narrow.py 64 mgs-hp-row
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
method = sys.argv[2] if len(sys.argv) > 2 else "mgs-hp-row"
csr, Zd = problems.config5(n=n)
op = aqr.CsrSpdOperator(*csr)
Zh = np.asfortranarray(Zd.cpu().numpy())
del Zd
torch.cuda.empty_cache()
t0 = time.perf_counter()
r = aqr.factorize(Zh, op, method)
print(f"{method} host-input m={Zh.shape[0]} n={n}: {1e3 * (time.perf_counter() - t0):.1f} ms")
