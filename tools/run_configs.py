"""Run BASELINE.json configs 2-5 at full size on one B200: time + accuracy.

    python tools_configs.py [2 3 4 5]

Prints one JSON line per (config, method): device time per factorization
(CUDA events, after one warm-up), columns/s, the step-level algorithmic HBM
bytes of this build's schedule (bench.step_bytes) and achieved GB/s, SURVEY
8d's eager-model bytes for comparison, loss of A-orthogonality and
||Z - QR|| / ||Z||.  Config 5 (Z = 34 GB) and config 4 (A = 8.6 GB) are
generated on the GPU (problems.config4 / config5).
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import problems


def timed(fn, reps=1):
    out = fn()
    out = fn()  # steady state: the previous result is alive during the next call
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


from bench import banded_bytes, step_bytes, survey_bytes  # noqa: E402  (this build's schedule model)


def report(cfg, method, op, Z, bytes_A, reps=1, metrics=True):
    ms, r = timed(lambda: aqr.factorize(Z, op, method), reps)
    m, n = Z.shape
    bb = banded_bytes(op, m)  # stencil operators: the banded view's bytes per apply
    b = step_bytes(method.split("-")[1], m, n, bb[0] if bb else bytes_A)
    e = survey_bytes(method.split("-")[1], m, n, bytes_A)
    line = {"config": cfg, "method": method, "m": m, "n": n, "operator": bb[1] if bb else "as given",
            "ms": ms, "cols_per_s": n / (ms / 1e3),
            "alg_GB": b / 1e9, "GBps": b / (ms / 1e3) / 1e9, "survey_8d_GB": e / 1e9,
            "survey_8d_equiv_GBps": e / (ms / 1e3) / 1e9}
    if metrics:
        line["loss_A_orth"] = aqr.loss_of_A_orthogonality(r.Q, op)
        line["residual_rel"] = aqr.residual_rel(Z, r.Q, r.R)
    print(json.dumps(line), flush=True)
    del r
    torch.cuda.empty_cache()


def main():
    which = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]
    if 2 in which:
        (ip, ix, dv), Z = problems.config2(device=True)
        op = aqr.CsrSpdOperator(ip, ix, dv)
        for meth in ("mgs-ha-row", "mgs-hp-row", "mgs-naive-row", "cgs-ha-row"):
            report(2, meth, op, Z, 12 * int(ip[-1]) + 4 * (Z.shape[0] + 1), reps=3)
        del op, Z
    if 3 in which:
        (ip, ix, dv), Z = problems.config3(device=True)
        op = aqr.CsrSpdOperator(ip, ix, dv)
        for meth in ("mgs-ha-row", "mgs-hp-row"):
            report(3, meth, op, Z, 12 * int(ip[-1]) + 4 * (Z.shape[0] + 1), reps=2)
        del op, Z
    if 4 in which:
        t0 = time.time()
        A, Z = problems.config4()
        torch.cuda.synchronize()
        print(json.dumps({"config": 4, "generated_s": time.time() - t0}), flush=True)
        op = aqr.DenseSpdOperator(A)
        for meth in ("mgs-ha-row", "mgs-hp-row"):
            report(4, meth, op, Z, 8 * Z.shape[0] ** 2)
        del op, A, Z
    if 5 in which:
        torch.cuda.empty_cache()
        t0 = time.time()
        (ip, ix, dv), Z = problems.config5()
        op = aqr.CsrSpdOperator(ip, ix, dv)
        del ip, ix, dv
        torch.cuda.synchronize()
        print(json.dumps({"config": 5, "generated_s": time.time() - t0,
                          "mem_GB": torch.cuda.memory_allocated() / 1e9}), flush=True)
        for meth in ("mgs-hp-row", "mgs-ha-row"):
            report(5, meth, op, Z, 12 * op.nnz + 4 * (Z.shape[0] + 1), metrics=False)


if __name__ == "__main__":
    main()
