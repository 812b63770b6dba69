"""The HP block apply of a dense operator on the FP64 tensor cores
(aqr_block_apply -> dense_dmma_kernel: DMMA m8n8k4 with TMA-fed, 128-byte
swizzled tiles).

The reference's apply_block_dense (/root/reference/pkg/src/aqr/_kernels_impl.py:
35-47) sums each entry sequentially; the tensor-core product sums the same
terms with fused multiply-adds in k-blocks, so it is held to the sequential
product (the bitwise kernel, aqr_op_apply) within a rounding-level bound:
|Y - Y_seq| <= 4 K u (|A| |X|) elementwise, u = 2^-53 (the classical dot
product error bound of both orders, summed).  Operators below 4096^2
entries keep the sequential product (bitwise); the tile edges (m, K, k not
multiples of 128 / 16 / 64) are covered by forcing the tensor-core kernel on
small shapes in the experiments build.  Also: a rectangular operator and
the fallback for operands TMA cannot map (odd leading dimension).  The HP
factorizations that use it are gated against the oracle in
test_gpu_parity.py (config 1) and test_gpu_fullsize.py (config 4 family).
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _apply(fn_name, A, X, ncols=0, lda=None):
    import torch

    from paper_1703_10440_b200 import _device as D
    from paper_1703_10440_b200 import _lib

    m = A.shape[0]
    K = A.shape[1]
    lda = lda or m
    Ad = torch.zeros((K, lda), dtype=torch.float64, device="cuda")
    Ad[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T))
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()  # column-major K x k
    k = X.shape[1]
    Yd = torch.full((k, m), np.nan, dtype=torch.float64, device="cuda")
    d = _lib.AqrOp()
    d.kind = _lib.AQR_OP_DENSE
    d.m = m
    d.A = Ad.data_ptr()
    d.lda = lda
    d.ncols = ncols
    _lib.check(getattr(_lib.lib(), fn_name)(ctypes.byref(d), k, Xd.data_ptr(), K, Yd.data_ptr(), m,
                                            D.stream_ptr()), fn_name)
    torch.cuda.synchronize()
    return Yd.cpu().numpy().T


def _check_rounding_bound(m, K, k):
    rng = np.random.default_rng(m * 7 + k)
    A = rng.standard_normal((m, K))  # not symmetric: the kernel reads A as stored
    X = rng.standard_normal((K, k))
    ncols = K if K != m else 0
    fast = _apply("aqr_block_apply", A, X, ncols)
    seq = _apply("aqr_op_apply", A, X, ncols)
    assert np.isfinite(fast).all()
    bound = 4 * K * U * (np.abs(A) @ np.abs(X))
    assert (np.abs(fast - seq) <= bound).all()
    assert np.abs(fast - A @ X).max() <= 4 * K * U * (np.abs(A) @ np.abs(X)).max()
    return fast, seq


@pytest.mark.parametrize("m,K,k", [(4096, 4096, 256), (4100, 4100, 65), (8192, 2048, 33)])
def test_block_apply_within_rounding_of_sequential(m, K, k):
    fast, seq = _check_rounding_bound(m, K, k)
    assert not np.array_equal(fast, seq)  # the tensor-core path ran (operators >= 4096^2 entries)


SMALL = r"""
import sys
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
import test_gpu_dgemm as T
for shape in [(1000, 1000, 50), (300, 300, 7), (130, 128, 65), (16, 16, 2), (1000, 600, 65), (2, 2, 1)]:
    T._check_rounding_bound(*shape)
print("ok")
"""


def test_block_apply_tile_edges_forced_small():
    """Tile edges (m, K, k not multiples of 128 / 16 / 64) on the tensor-core
    kernel, forced below its size threshold (experiments build, AQR_DGEMM=2)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    repo = os.path.dirname(here)
    env = dict(os.environ, AQR_LIB_PATH=os.path.join(repo, "paper_1703_10440_b200", "libaqr_b200_exp.so"),
               AQR_DGEMM="2")
    out = subprocess.run([sys.executable, "-c", SMALL.format(repo=repo, tests=here)], env=env, check=True,
                         capture_output=True, text=True, timeout=600)
    assert out.stdout.strip().endswith("ok")


def test_small_operator_keeps_sequential_bits():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((1000, 1000))
    X = rng.standard_normal((1000, 50))
    assert np.array_equal(_apply("aqr_block_apply", A, X), _apply("aqr_op_apply", A, X))


def test_block_apply_odd_lda_falls_back_bitwise():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((4097, 4097))
    X = rng.standard_normal((4097, 9))
    fast = _apply("aqr_block_apply", A, X, lda=4099)  # lda * 8 not a multiple of 16: no tensor map
    seq = _apply("aqr_op_apply", A, X, lda=4099)
    assert np.array_equal(fast, seq)


def test_dense_hp_factorization_against_oracle():
    import paper_1703_10440_b200 as aqr
    from oracle import oracle as O

    import parity

    rng = np.random.default_rng(11)
    m, n = 4096, 24  # 4096^2 entries: the tensor-core block apply
    G = rng.standard_normal((m, m))
    A = np.asfortranarray(G @ G.T / m + np.eye(m))
    Z = np.asfortranarray(rng.standard_normal((m, n)))
    op = aqr.DenseSpdOperator(A)
    cal = parity.calibrated(Z, ("dense", A), ["mgs-hp-row", "cgs-hp-row", "mgs-hp-col"])
    for meth, (o, tq, tr) in cal.items():
        r = aqr.factorize(Z, op, meth)
        eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
        assert eq <= tq and er <= tr, (meth, eq, tq, er, tr)
        loss_g, loss_o = aqr.loss_of_A_orthogonality(r.Q, op), aqr.loss_of_A_orthogonality(o.Q, op)
        assert loss_g <= 1.05 * loss_o, (meth, loss_g, loss_o)
    # numpy in (host pipeline, block apply chunk by chunk) == device in (one call)
    import torch

    a = aqr.factorize(Z, op, "mgs-hp-row")
    b = aqr.factorize(torch.from_numpy(Z).cuda(), op, "mgs-hp-row")
    assert np.array_equal(a.Q, b.Q.cpu().numpy()) and np.array_equal(a.R, b.R.cpu().numpy())
