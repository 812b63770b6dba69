"""Diagnostics: one config-2 factorization through the host-input pipeline
(page-locked Z) -- the command profiled with ncu -k regex:catchup to see
where a catch-up step's time goes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems
(ip, ix, dv), Z = problems.config2(device=False)
m, n = Z.shape
op = aqr.CsrSpdOperator(ip, ix, dv)
Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
Zh.copy_(torch.from_numpy(Z))
r = aqr.factorize(Zh, op, sys.argv[1] if len(sys.argv) > 1 else "mgs-ha-row")
torch.cuda.synchronize()
print("ok", float(r.R[0, 0]))
