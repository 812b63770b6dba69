"""Diagnostics: the bitwise dense block apply (config 4: A 32768^2, X 32768 x 256)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems
A, Z = problems.config4()
op = aqr.DenseSpdOperator(A)
Y = op.apply_block(Z); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    Y2 = op.apply_block(Z)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
m, k = Z.shape
print(f"variant {os.environ.get('AQR_GEMM_VARIANT', '0')}: {ms:.2f} ms, {2 * m * m * k / ms / 1e9:.2f} TFLOP/s, "
      f"checksum {float(Y2.double().sum()):.17g}")
