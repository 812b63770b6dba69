"""The multi-GPU driver on one B200 (NCCL, world_size 1).

With a single rank every all-reduce is the identity and the halo is empty,
so paper_1703_10440_b200.distributed (CUDA step engine, step entry points of
libaqr_b200.so) must reproduce the single-GPU drop-in bitwise: same
kernels, same canonical reduction trees.  Both the generic (small m) and the
TMA-pipelined (m >= 2048*148) trailing kernels are covered.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1():
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist


@pytest.mark.parametrize("backend", [None, "nccl"])
@pytest.mark.parametrize("grid,n", [(16, 8), (640, 6)])
@pytest.mark.parametrize("method", ["mgs-ha-row", "mgs-hp-row", "mgs-naive-row", "cgs-hp-row", "cgs-ha-row"])
def test_world1_bitwise_equals_single_gpu(nccl1, grid, n, method, backend):
    import torch

    import paper_1703_10440_b200 as aqr
    from paper_1703_10440_b200 import distributed as DD
    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.laplacian5(grid, grid, 1e-2)
    m = grid * grid
    Z = np.asfortranarray(np.random.default_rng(grid + n).standard_normal((m, n)))
    Zd = torch.from_numpy(Z.T).cuda().t()
    ref = aqr.factorize(Zd, aqr.CsrSpdOperator(ip, ix, dv), method)
    op = DD.DistCsrSpdOperator(ip, ix, dv, DD.row_partition(m, 1), 0)
    for _ in range(2):  # the peer-memory path's flags advance between calls
        res = DD.dist_factorize(Zd, op, method, backend=backend)
        assert torch.equal(res.R, ref.R), method
        assert torch.equal(res.Q, ref.Q), method
        assert res.cost.mv_count == ref.cost.mv_count
        assert res.flagged_columns == ref.flagged_columns


def test_world1_peer_memory_breakdown(nccl1):
    """Peer-memory path: breakdown column / value as the single-GPU call,
    and the group keeps working afterwards."""
    import torch

    import paper_1703_10440_b200 as aqr
    from paper_1703_10440_b200 import distributed as DD
    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.laplacian5(20, 20, 1e-2)
    m, n = 400, 7
    Z = np.asfortranarray(np.random.default_rng(3).standard_normal((m, n)))
    Z[:, 4] = 0.0
    Zd = torch.from_numpy(Z.T).cuda().t()
    op = DD.DistCsrSpdOperator(ip, ix, dv, DD.row_partition(m, 1), 0)
    for method in ("mgs-ha-row", "mgs-hp-row"):
        with pytest.raises(aqr.BreakdownError) as ref:
            aqr.factorize(Zd, aqr.CsrSpdOperator(ip, ix, dv), method)
        with pytest.raises(aqr.BreakdownError) as got:
            DD.dist_factorize(Zd, op, method, backend="p2p")
        assert (got.value.column, got.value.value) == (ref.value.column, ref.value.value) == (4, 0.0)
    Z[:, 4] = 1.0
    Zd = torch.from_numpy(Z.T).cuda().t()
    res = DD.dist_factorize(Zd, op, "mgs-ha-row", backend="p2p")
    ref = aqr.factorize(Zd, aqr.CsrSpdOperator(ip, ix, dv), "mgs-ha-row")
    assert torch.equal(res.Q, ref.Q) and torch.equal(res.R, ref.R)


def test_world1_dense_bitwise(nccl1, golden):
    import torch

    import paper_1703_10440_b200 as aqr
    from paper_1703_10440_b200 import distributed as DD

    A, Z = golden["dense3|A"], golden["dense3|Z"]
    m = A.shape[0]
    Zd = torch.from_numpy(np.ascontiguousarray(Z.T)).cuda().t()
    for method in ("mgs-ha-row", "mgs-hp-row"):
        ref = aqr.factorize(Zd, aqr.DenseSpdOperator(A), method)
        op = DD.DistDenseSpdOperator(np.asfortranarray(A), DD.row_partition(m, 1), 0)
        res = DD.dist_factorize(Zd, op, method)
        assert torch.equal(res.R, ref.R) and torch.equal(res.Q, ref.Q), method
