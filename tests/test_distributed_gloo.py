"""Multi-rank path on CPU: world_size 2 over gloo (127.0.0.1).

Exercises the product driver paper_1703_10440_b200.distributed: the row
partition, the collective halo plan, the halo exchange (bitwise equal to the
global SpMV), the dense all-gather, the per-step all-reduces and the R
assembly.  Per-rank arithmetic runs in the numpy step engine of
tests/dist_cpu_engine.py; results are compared with the oracle.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, method, outdir):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import dist_cpu_engine as E
        from paper_1703_10440_b200 import distributed as DD

        g = np.load(os.path.join(HERE, "golden", "small.npz"))
        Z = g[f"{case}|Z"]
        m, n = Z.shape
        if f"{case}|A" in g:
            A = g[f"{case}|A"]
            part = DD.row_partition(m, world)
            r0, r1 = part[rank]
            op = DD.DistDenseSpdOperator(np.asfortranarray(A[r0:r1]), part, rank,
                                         local_apply=E.local_dense_apply)
        else:
            ip, ix, dv = g[f"{case}|indptr"], g[f"{case}|indices"], g[f"{case}|data"]
            part = DD.row_partition(m, world, align=16 if case == "csr16" else 9)
            r0, r1 = part[rank]
            op = DD.DistCsrSpdOperator(ip[r0:r1 + 1] - ip[r0], ix[ip[r0]:ip[r1]], dv[ip[r0]:ip[r1]],
                                       part, rank, local_apply=E.local_csr_apply)
            # the halo exchange reproduces the global product bitwise
            from oracle import oracle as O

            x = np.random.default_rng(0).standard_normal(m)
            y = op.apply(torch.from_numpy(np.ascontiguousarray(x[r0:r1])))
            ref = O.csr_matvec(ip, ix, dv, x)[r0:r1]
            assert np.array_equal(y.numpy(), ref)
            op.mv_count = 0
            # the peer-memory halo tables name the owner and its local row of every halo column
            gl = ix[ip[r0]:ip[r1]]
            loc = op.indices_local
            halo = loc >= (r1 - r0)
            h = loc[halo] - (r1 - r0)
            owner_start = np.array([part[p][0] for p in op.halo_rank[h]])
            assert np.array_equal(owner_start + op.halo_row[h], gl[halo])
            assert np.all(op.halo_rank != rank) and len(op.halo_rank) == op.n_ext - (r1 - r0)
        fam, var, _ = method.split("-")
        eng = E.CpuStepEngine(r1 - r0, n, fam, var)
        res = DD.dist_factorize(torch.from_numpy(np.asfortranarray(Z[r0:r1])), op, method, engine=eng)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), Q=res.Q.numpy(), R=res.R.numpy(),
                 mv=np.array([res.cost.mv_count]), flagged=np.array(res.flagged_columns, dtype=np.int64),
                 r0=np.array([r0]), r1=np.array([r1]))
    finally:
        dist.destroy_process_group()


def _run(case, method, world, tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, method, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    return outs


def _oracle_op(g, case):
    if f"{case}|A" in g:
        return ("dense", g[f"{case}|A"])
    return ("csr", g[f"{case}|indptr"], g[f"{case}|indices"], g[f"{case}|data"])


@pytest.mark.parametrize("case,method", [
    ("csr16", "mgs-ha-row"), ("csr16", "mgs-hp-row"), ("csr16", "mgs-naive-row"),
    ("dense3", "mgs-ha-row"), ("dense3", "mgs-hp-row"), ("csr9x7", "cgs-ha-row"),
])
def test_world2_matches_oracle(golden, tmp_path, case, method):
    import parity
    from oracle import oracle as O

    outs = _run(case, method, 2, tmp_path)
    Z = golden[f"{case}|Z"]
    n = Z.shape[1]
    spec = _oracle_op(golden, case)
    ref = O.gs_factor(Z, spec, method)
    Q = np.concatenate([o["Q"] for o in outs], axis=0)
    assert [int(o["r0"][0]) for o in outs] == [0, int(outs[0]["r1"][0])]
    # R is replicated: identical on every rank
    assert np.array_equal(outs[0]["R"], outs[1]["R"])
    tq, tr = parity.tolerance(Z, spec, method)
    eq, er = parity.factor_errors(Q, outs[0]["R"], ref.Q, ref.R)
    assert eq <= tq and er <= tr, (eq, tq, er, tr)
    expected_mv = 2 * n if "naive" in method else n
    assert all(int(o["mv"][0]) == expected_mv for o in outs)
    assert outs[0]["flagged"].tolist() == ref.flagged_columns


def test_world1_is_bitwise_oracle(golden, tmp_path):
    # one rank: the driver + numpy engine reproduce the reference exactly
    from oracle import oracle as O

    outs = _run("csr16", "mgs-ha-row", 1, tmp_path)
    ref = O.gs_factor(golden["csr16|Z"], _oracle_op(golden, "csr16"), "mgs-ha-row")
    assert np.array_equal(outs[0]["Q"], ref.Q)
    assert np.array_equal(outs[0]["R"], ref.R)


def test_row_partition():
    from paper_1703_10440_b200.distributed import row_partition

    assert row_partition(10, 2) == [(0, 5), (5, 10)]
    p = row_partition(1024 * 1024, 8, align=1024)
    assert p[0] == (0, 131072) and p[-1][1] == 1024 * 1024
    assert all(b[0] % 1024 == 0 for b in p)
    p = row_partition(100, 3, align=16)
    assert p[-1][1] == 100 and all(r1 > r0 for r0, r1 in p)
