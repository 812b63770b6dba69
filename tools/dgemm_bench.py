"""Config 4's HP block apply (A 32768^2 fp64, Z 32768 x 256): the FP64
tensor-core product (aqr_block_apply) against the sequential-order kernel
(aqr_op_apply), CUDA events, TFLOP/s and the max deviation between them."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import _device as D, _lib, problems

A, Z = problems.config4()
m, k = Z.shape
d = aqr.DenseSpdOperator(A)._native()  # the operator's own device copy / descriptor
L = _lib.lib()
out = {}
for fn in ("aqr_block_apply", "aqr_op_apply"):
    Y = torch.empty((k, m), dtype=torch.float64, device="cuda").t()
    call = lambda: _lib.check(getattr(L, fn)(ctypes.byref(d), k, Z.data_ptr(), Z.stride(1), Y.data_ptr(), m,
                                             D.stream_ptr()), fn)
    call(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5 if fn == "aqr_block_apply" else 2
    e0.record()
    for _ in range(reps):
        call()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[fn] = Y
    print(f"{fn}: {ms:.2f} ms, {2 * m * m * k / ms / 1e9:.2f} TFLOP/s", flush=True)
dev = (out["aqr_block_apply"] - out["aqr_op_apply"]).abs().max().item()
scale = out["aqr_op_apply"].abs().max().item()
print(f"max |fast - sequential| = {dev:.3e} (max |Y| = {scale:.3e}, rel {dev / scale:.3e})")
