"""Config 5's operator and rows with only the first n' columns of Z, for ncu.

    python tools/cfg5_narrow.py [n'] [method] [reps]

A full config-5 trailing launch moves up to 68 GB (Z and X = A Z, 34 GB
each); ncu's kernel replay saves and restores the memory a kernel writes
for every one of its ~40 passes, so full captures are taken on this
narrow run instead: the same m = 256^3, the same 27-point CSR, the same
kernel instantiations and grid -- only the number of trailing columns per
launch differs (t = n'-1-i instead of 255-i).  Launch order of one
mgs-hp-row call: block apply (csr_row_kernel / csr_spmm2_kernel), then per
step i the column update + norm and the trailing pass.
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1703_10440_b200 as aqr
    from paper_1703_10440_b200 import problems

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    method = sys.argv[2] if len(sys.argv) > 2 else "mgs-hp-row"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    csr, Z = problems.config5(n=n)
    op = aqr.CsrSpdOperator(*csr)
    torch.cuda.synchronize()
    for _ in range(reps):
        t0 = time.perf_counter()
        r = aqr.factorize(Z, op, method)
        torch.cuda.synchronize()
        print(f"{method} m={Z.shape[0]} n={n}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
        del r


if __name__ == "__main__":
    main()
