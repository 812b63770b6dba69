"""Small-shape sweep of every launch path, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_small.py

Runs the fused step kernels (HA / HP / naive, MGS / CGS, row / col, dense and
CSR operators, short and long rows), the host-input pipeline (catch-up
cooperative kernel), the world-1 peer-memory path, the kernel namespace and
the Cholesky QR on tiny inputs, each once.  Exits non-zero on a wrong result
(vs the C oracle) so a sanitizer run also checks it ran the paths.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np


def main():
    import torch

    import paper_1703_10440_b200 as aqr
    from oracle import oracle as O
    from paper_1703_10440_b200 import backend, problems

    rng = np.random.default_rng(7)
    m = 300
    G = rng.standard_normal((m, m))
    A = np.asfortranarray(G @ G.T + m * np.eye(m))
    Z = np.asfortranarray(rng.standard_normal((m, 6)))
    ip, ix, dv = problems.laplacian5(24, 20, 1e-2)
    Zc = np.asfortranarray(rng.standard_normal((480, 6)))
    s27 = problems.stencil27_device(8, 1e-2, "cuda")
    s27h = (s27[0].cpu().numpy(), s27[1].cpu().numpy().astype(np.int64), s27[2].cpu().numpy())
    Z27 = np.asfortranarray(rng.standard_normal((512, 5)))
    ops = [("dense", aqr.DenseSpdOperator(A), ("dense", A), Z),
           ("csr5", aqr.CsrSpdOperator(ip, ix, dv), ("csr", ip, ix, dv), Zc),
           ("csr27", aqr.CsrSpdOperator(*s27h), ("csr",) + s27h, Z27)]
    worst = 0.0
    for name, op, spec, Zx in ops:
        for meth in ("mgs-ha-row", "mgs-hp-row", "mgs-naive-row", "cgs-ha-row", "mgs-hp-col", "cgs-naive-col"):
            Zd = torch.from_numpy(Zx.T.copy()).cuda().t()
            for Zin in (Zd, Zx):  # device-resident, then the host-input pipeline
                r = aqr.factorize(Zin, op, meth)
                Q = r.Q.cpu().numpy() if hasattr(r.Q, "cpu") else r.Q
                o = O.gs_factor(Zx, spec, meth)
                worst = max(worst, float(np.abs(Q - o.Q).max() / np.abs(o.Q).max()))
        r = aqr.cholesky_qr(Zx, op)
        worst = max(worst, float(np.abs(r.Q - O.cholesky_qr(Zx, spec).Q).max()))
    K = backend.kernels()
    x = rng.standard_normal(1000)
    K.seq_dot(x, x)
    # world-1 peer-memory path (gloo bootstrap)
    import socket

    import torch.distributed as dist

    from paper_1703_10440_b200 import distributed as DD

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    dop = DD.DistCsrSpdOperator(ip, ix, dv, DD.row_partition(480, 1), 0)
    for meth in ("mgs-ha-row", "mgs-hp-row"):
        r = DD.dist_factorize(torch.from_numpy(Zc.T.copy()).cuda().t(), dop, meth, backend="p2p")
        o = O.gs_factor(Zc, ("csr", ip, ix, dv), meth)
        worst = max(worst, float(np.abs(r.Q.cpu().numpy() - o.Q).max()))
    dist.destroy_process_group()
    torch.cuda.synchronize()
    print("worst relative Q difference vs oracle:", worst)
    if not worst < 1e-10:
        sys.exit(1)


if __name__ == "__main__":
    main()
