"""The kernel namespace (backend.kernels(), row a10) and the weighted
Cholesky QR (row f3) on the B200, against the C oracle's restatement of the
reference kernels (/root/reference/pkg/src/aqr/_kernels_impl.py:17-164) and
the reference's own cholqr fixtures (tests/golden/small.npz).

Every kernel except ``seq_dot`` keeps the reference's operation order, so
those checks are BITWISE; ``seq_dot`` is a tree reduction and is held to the
sequential sum within 1e-12 relative (as test_backends.py:139-145 holds the
reference's to math.fsum).
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_1703_10440_b200 import backend

    return backend.kernels()


@pytest.fixture(scope="module")
def aqr():
    import paper_1703_10440_b200 as P

    return P


def test_backend_selection():
    from paper_1703_10440_b200 import backend

    assert backend.current_backend() == "b200"
    assert backend.set_backend("auto") == "b200"
    with pytest.raises(ValueError):
        backend.set_backend("numba")  # one backend only: no multi-backend dispatch
    with backend.use_backend("b200"):
        assert backend.current_backend() == "b200"


@pytest.mark.parametrize("m", [1, 7, 1000, 300_001])
def test_seq_dot(K, m):
    rng = np.random.default_rng(m)
    x, y = rng.standard_normal(m), rng.standard_normal(m)
    got, ref = K.seq_dot(x, y), O.seq_dot(x, y)
    assert got == pytest.approx(ref, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("m", [1, 1000, 65_537])
def test_sub_scaled_div_scalar_bitwise(K, m):
    rng = np.random.default_rng(m + 1)
    z, q = rng.standard_normal(m), rng.standard_normal(m)
    a, r = float(rng.standard_normal()), float(rng.uniform(0.5, 2.0))
    z1 = z.copy()
    K.sub_scaled(z1, a, q)
    assert np.array_equal(z1, z - a * q)  # numpy: separately rounded a*q, then z - that
    out = np.empty(m)
    K.div_scalar(z, r, out)
    assert np.array_equal(out, z / r)


@pytest.mark.parametrize("m,ncols", [(5, 5), (130, 130), (1000, 1000), (640, 333)])
def test_matvec_bitwise(K, m, ncols):
    rng = np.random.default_rng(m + ncols)
    A = np.asfortranarray(rng.standard_normal((m, ncols)))
    x = rng.standard_normal(ncols)
    y = np.empty(m)
    K.matvec(A, x, y)
    assert np.array_equal(y, O.matvec(A, x))


@pytest.mark.parametrize("m,k", [(40, 1), (300, 7), (1000, 64)])
def test_apply_block_dense_bitwise(K, m, k):
    rng = np.random.default_rng(m * k)
    A = np.asfortranarray(rng.standard_normal((m, m)))
    X = np.asfortranarray(rng.standard_normal((m, k)))
    Y = np.empty((m, k), order="F")
    K.apply_block_dense(A, X, Y)
    assert np.array_equal(Y, O.apply_block_dense(A, X))


def test_csr_matvec_bitwise(K, golden):
    from paper_1703_10440_b200 import problems

    for ip, ix, dv in [(golden["csr9x7|indptr"], golden["csr9x7|indices"], golden["csr9x7|data"]),
                       problems.laplacian5(300, 200, 1e-2),
                       problems.diffusion7(20, 1e-3, problems.rng(3, 0))]:
        m = ip.shape[0] - 1
        x = np.random.default_rng(m).standard_normal(m)
        y = np.empty(m)
        K.csr_matvec(ip, ix, dv, x, y)
        assert np.array_equal(y, O.csr_matvec(ip, ix, dv, x))


@pytest.mark.parametrize("m,p,n", [(1, 1, 1), (50, 7, 9), (1000, 64, 33), (100_003, 40, 40)])
def test_gemm_tn_nn_bitwise(K, m, p, n):
    rng = np.random.default_rng(m + p + n)
    A = np.asfortranarray(rng.standard_normal((m, p)))
    B = np.asfortranarray(rng.standard_normal((m, n)))
    C = np.empty((p, n), order="F")
    K.gemm_tn(A, B, C)
    assert np.array_equal(C, O.gemm_tn(A, B))
    Bn = np.asfortranarray(rng.standard_normal((p, n)))
    Cn = np.empty((m, n), order="F")
    K.gemm_nn(A, Bn, Cn)
    assert np.array_equal(Cn, O.gemm_nn(A, Bn))


def test_cholesky_and_tri_solve_kernels_bitwise(K):
    rng = np.random.default_rng(77)
    for n in (1, 5, 64, 300):
        B = rng.standard_normal((n + 3, n))
        G = np.asfortranarray(B.T @ B + 1e-3 * np.eye(n))
        R = np.zeros((n, n), order="F")
        bad = K.cholesky_upper_kernel(G, R)
        bad_o, R_o = O.cholesky_upper_kernel(G)
        assert bad == bad_o == -1
        assert np.array_equal(R, R_o)
        Z = np.asfortranarray(rng.standard_normal((777, n)))
        X = np.empty_like(Z, order="F")
        K.tri_solve_right_kernel(Z, R, X)
        assert np.array_equal(X, O.tri_solve_right_kernel(Z, R_o))
    G = np.array([[1.0, 2.0], [2.0, 4.0]], order="F")  # singular: pivot 1 fails
    R = np.zeros((2, 2), order="F")
    assert K.cholesky_upper_kernel(G, R) == O.cholesky_upper_kernel(G)[0] == 1


def test_kernels_in_place_on_device_tensors(K):
    import torch

    rng = np.random.default_rng(3)
    z, q = rng.standard_normal(4097), rng.standard_normal(4097)
    zd, qd = torch.from_numpy(z.copy()).cuda(), torch.from_numpy(q).cuda()
    K.sub_scaled(zd, 0.375, qd)
    assert np.array_equal(zd.cpu().numpy(), z - 0.375 * q)
    A = rng.standard_normal((200, 30))
    Ad = torch.from_numpy(A.T.copy()).cuda().t()  # column-major device matrix
    Cd = torch.empty((30, 30), dtype=torch.float64, device="cuda").t()
    K.gemm_tn(Ad, Ad, Cd)
    assert np.array_equal(Cd.cpu().numpy(), O.gemm_tn(A, A))


# ---- weighted Cholesky QR (gram_schmidt.py:209-218) ---------------------------

@pytest.mark.parametrize("key", ["hand", "dense0", "dense1", "dense2", "dense3", "dense7"])
def test_cholqr_golden_bitwise(aqr, golden, key):
    Z, A = golden[f"{key}|Z"], golden[f"{key}|A"]
    op = aqr.DenseSpdOperator(A)
    r = aqr.cholesky_qr(Z, op)
    assert np.array_equal(r.Q, golden[f"{key}|cholqr|Q"]), key
    assert np.array_equal(r.R, golden[f"{key}|cholqr|R"]), key
    assert r.cost.mv_count == int(golden[f"{key}|cholqr|mv"][0]) == op.mv_count
    assert r.cost.flops == int(golden[f"{key}|cholqr|mv"][1])
    assert r.flagged_columns == []
    f = aqr.factorize(Z, aqr.DenseSpdOperator(A), "cholqr")
    assert np.array_equal(f.Q, r.Q) and np.array_equal(f.R, r.R)


def test_cholqr_csr_bitwise_vs_oracle(aqr):
    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.laplacian5(128, 128, 1e-2)
    Z = np.asfortranarray(problems.rng(6, 1).standard_normal((128 * 128, 24)))
    r = aqr.cholesky_qr(Z, aqr.CsrSpdOperator(ip, ix, dv))
    o = O.cholesky_qr(Z, ("csr", ip, ix, dv))
    assert np.array_equal(r.Q, o.Q) and np.array_equal(r.R, o.R)


def test_cholqr_not_positive_definite(aqr):
    Z = np.array([[1.0, 2.0], [0.0, 0.0], [0.0, 0.0]])
    with pytest.raises(aqr.NotPositiveDefiniteError) as info:
        aqr.cholesky_qr(Z, aqr.identity_operator(3))
    assert info.value.pivot == 1


def test_linalg_helpers(aqr):
    import torch

    rng = np.random.default_rng(11)
    A = rng.standard_normal((50, 6))
    assert np.array_equal(aqr.matmul_tn(A, A).cpu().numpy(), O.gemm_tn(A, A))
    B = rng.standard_normal((6, 4))
    assert np.array_equal(aqr.matmul(A, B).cpu().numpy(), O.gemm_nn(A, B))
    with pytest.raises(aqr.SingularMatrixError):
        aqr.tri_solve_right(A, np.diag([1.0, 1.0, 0.0, 1.0, 1.0, 1.0]))
    with pytest.raises(aqr.DimensionError):
        aqr.matmul(A, A)
    # two_norm: the largest singular value
    s = np.linalg.svd(A, compute_uv=False)[0]
    assert aqr.two_norm(A) == pytest.approx(s, rel=1e-13)
    assert aqr.two_norm(torch.from_numpy(A.T.copy()).cuda()) == pytest.approx(s, rel=1e-13)
