"""One rank of the multi-process peer-memory test (tests/test_gpu_multirank.py).

Launched N times by the test with RANK / WORLD_SIZE / MASTER_ADDR /
MASTER_PORT / AQR_MP_OUT in the environment.  Every rank uses cuda:0 (one
leased GPU: same-device CUDA IPC between processes) and a gloo process group
(only the bootstrap -- IPC handles, halo plan -- and the result gather use
it; the factorization itself has no collective call).  Writes its results
to AQR_MP_OUT/rank<r>.npz for the parent to check against the oracle.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def cases():
    from paper_1703_10440_b200 import problems

    g = 40  # 2-D 5-point Laplacian, g x g; rows split by whole grid rows
    ip, ix, dv = problems.laplacian5(g, g, 1e-2)
    yield "lap", (ip, ix, dv), g, np.asfortranarray(problems.rng(21, 1).standard_normal((g * g, 8)))
    s = 12  # 27-point stencil on s^3, split by whole planes (rows of 8-27 entries)
    ip, ix, dv = problems.stencil27_device(s, 1e-2, "cuda")
    csr = (ip.cpu().numpy(), ix.cpu().numpy().astype(np.int64), dv.cpu().numpy())
    yield "st27", csr, s * s, np.asfortranarray(problems.rng(21, 2).standard_normal((s ** 3, 6)))


def main():
    import torch
    import torch.distributed as dist

    from paper_1703_10440_b200 import BreakdownError
    from paper_1703_10440_b200 import distributed as DD
    from paper_1703_10440_b200 import p2p

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for name, (ip, ix, dv), align, Z in cases():
        m = Z.shape[0]
        part = DD.row_partition(m, world, align=align)
        r0, r1 = part[rank]
        op = DD.DistCsrSpdOperator(ip[r0:r1 + 1] - ip[r0], ix[ip[r0]:ip[r1]], dv[ip[r0]:ip[r1]], part, rank)
        Zl = torch.from_numpy(np.ascontiguousarray(Z[r0:r1].T)).cuda().t()
        out[f"{name}|rows"] = np.array([r0, r1])
        for meth in ("mgs-ha-row", "mgs-hp-row", "cgs-ha-row", "cgs-hp-row"):
            res = DD.dist_factorize(Zl, op, meth, backend="p2p")
            again = DD.dist_factorize(Zl, op, meth, backend="p2p")  # flags advance between calls
            out[f"{name}|{meth}|Q"] = res.Q.cpu().numpy()
            out[f"{name}|{meth}|R"] = res.R.cpu().numpy()
            out[f"{name}|{meth}|rerun_equal"] = np.array(
                [bool(torch.equal(res.Q, again.Q) and torch.equal(res.R, again.R))])
            out[f"{name}|{meth}|mv"] = np.array([res.cost.mv_count])
            out[f"{name}|{meth}|flag"] = np.array(res.flagged_columns, dtype=np.int64)
        # breakdown: a zero column 3 -> every rank raises at column 3
        Zb = Zl.clone()
        Zb[:, 3] = 0.0
        for meth in ("mgs-ha-row", "mgs-hp-row"):
            try:
                DD.dist_factorize(Zb, op, meth, backend="p2p")
                out[f"{name}|{meth}|breakdown"] = np.array([-1.0, 0.0])
            except BreakdownError as e:
                out[f"{name}|{meth}|breakdown"] = np.array([e.column, e.value])
        # and the group keeps working afterwards
        res = DD.dist_factorize(Zl, op, "mgs-ha-row", backend="p2p")
        out[f"{name}|after_breakdown_equal"] = np.array(
            [bool(np.array_equal(res.R.cpu().numpy(), out[f"{name}|mgs-ha-row|R"]))])
        last_op, last_Z = op, Zl
    # bounded waits: rank 0 calls alone (the others skip the call) and must
    # get PeerExchangeTimeout instead of spinning forever
    dist.barrier()
    if rank == 0:
        try:
            p2p.p2p_factorize(last_Z, last_op, DD.MethodId.parse("mgs-ha-row"), timeout_s=2.0)
            out["timeout_raised"] = np.array([0])
        except p2p.PeerExchangeTimeout:
            out["timeout_raised"] = np.array([1])
    torch.cuda.synchronize()
    dist.barrier()
    np.savez(os.path.join(os.environ["AQR_MP_OUT"], f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
