"""Diagnostics: host enqueue time vs device time of one factorization (AQR_DEBUG_TIMING)."""
import os, sys, time
os.environ["AQR_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems
(ip, ix, dv), Z = problems.config2(device=False)
op = aqr.CsrSpdOperator(ip, ix, dv)
Zd = torch.from_numpy(Z.T).cuda().t()
meth = sys.argv[1] if len(sys.argv) > 1 else "mgs-ha-row"
for _ in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    aqr.factorize(Zd, op, meth)
    torch.cuda.synchronize(); print("wall ms", (time.perf_counter() - t0) * 1e3, file=sys.stderr)
