"""Diagnostics: where the numpy-in / numpy-out call spends its time (config 2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems, _device as D
(ip, ix, dv), Z = problems.config2(device=False)
m, n = Z.shape
print("Z F-contiguous", Z.flags.f_contiguous, "C", Z.flags.c_contiguous)
op = aqr.CsrSpdOperator(ip, ix, dv)
def t(label, f, k=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): r = f()
    torch.cuda.synchronize(); print(label, round((time.perf_counter() - t0) / k * 1e3, 2), "ms"); return r
Zd = t("to_device_f", lambda: D.to_device_f(Z)[0])
t("pageable H2D torch.from_numpy(Z.T).cuda()", lambda: torch.from_numpy(Z.T).cuda())
t("Q.cpu()", lambda: Zd.cpu())
t("Q.cpu().numpy() + asfortranarray", lambda: np.asfortranarray(Zd.cpu().numpy()))
t("np.empty + touch", lambda: np.empty((m, n), order="F").fill(0.0))
t("np.empty_like fresh + copy", lambda: np.copy(Z, order="F"))
buf = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
t("pinned D2H", lambda: buf.copy_(Zd, non_blocking=True))
t("pinned->numpy copy (np.copyto fresh)", lambda: np.array(buf.numpy(), order="F", copy=True))
cr = torch.cuda.cudart()
def reg():
    A = np.empty((m, n), order="F")
    rc = cr.cudaHostRegister(A.ctypes.data, A.nbytes, 0)
    T = torch.from_numpy(A.T).t()
    T.copy_(Zd, non_blocking=True); torch.cuda.synchronize()
    cr.cudaHostUnregister(A.ctypes.data)
    return A
t("fresh numpy + cudaHostRegister + DMA + unregister", reg)
def reg_in():
    rc = cr.cudaHostRegister(Z.ctypes.data, Z.nbytes, 0)
    T = torch.from_numpy(Z.T).to("cuda", non_blocking=True); torch.cuda.synchronize()
    cr.cudaHostUnregister(Z.ctypes.data)
    return T
t("register input + DMA H2D + unregister", reg_in)
t("factorize numpy", lambda: aqr.mgs_ha(Z, op, "row"), 2)
