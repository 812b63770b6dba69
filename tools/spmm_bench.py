"""Diagnostics: the HP block apply X = A Z for config 5 (27-point CSR, Z 16.8M x 256),
or config 2 (5-point, Z 1M x 64) with argv[1] == "2"."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems
cfg2 = len(sys.argv) > 1 and sys.argv[1] == "2"
if cfg2:
    (ip, ix, dv), Zn = problems.config2(device=False)
    Z = torch.from_numpy(Zn.T).cuda().t()
else:
    (ip, ix, dv), Z = problems.config5()
op = aqr.CsrSpdOperator(ip, ix, dv)
Zs = Z[:, :32].contiguous().t().contiguous().t() if (len(sys.argv) > 1 and not cfg2) else Z
Y = op.apply_block(Zs); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); Y = op.apply_block(Zs); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
m, k = Zs.shape
nnz = int(ip[-1])
byts = 12 * nnz + 4 * (m + 1) + 16 * m * k
print(f"SpMM m={m} k={k} nnz={nnz}: {ms:.1f} ms, {byts / ms / 1e6:.0f} GB/s algorithmic")
