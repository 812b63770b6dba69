"""Dense helpers of the reference's linalg module on the device, in its order.

Drop-in for the pieces of /root/reference/pkg/src/aqr/linalg.py that the
weighted Cholesky QR and the accuracy metrics use: ``matmul`` (35-42),
``matmul_tn`` (45-52), ``cholesky_upper`` (191-208) and ``tri_solve_right``
(211-222).  Each runs one sm_100a kernel of libaqr_b200.so that keeps the
reference's per-entry operation order (sequential sums over the ascending
index, separately rounded multiply and add, IEEE division and sqrt), so the
results are bitwise the reference's for bitwise-equal inputs.

Arguments are numpy arrays or torch tensors; results are column-major CUDA
tensors (callers convert back).
"""

from . import _device as D
from . import _lib
from .exceptions import DimensionError, NotPositiveDefiniteError, SingularMatrixError
from .operators import as_matrix


def _dev(a):
    return D.to_device_f(as_matrix(a))


def matmul(A, B):
    """C = A @ B, entry (i, j) accumulated over ascending l (gemm_nn)."""
    (Ad, lda), (Bd, ldb) = _dev(A), _dev(B)
    m, kk = (int(s) for s in Ad.shape)
    if kk != int(Bd.shape[0]):
        raise DimensionError(f"matmul of shapes {tuple(Ad.shape)} and {tuple(Bd.shape)}")
    n = int(Bd.shape[1])
    C = D.empty_f(m, n)
    _lib.check(_lib.lib().aqr_gemm_nn(m, kk, n, Ad.data_ptr(), lda, Bd.data_ptr(), ldb, C.data_ptr(),
                                      max(m, 1), D.stream_ptr()), "aqr_gemm_nn")
    return C


def matmul_tn(A, B):
    """C = A.T @ B, entry (i, j) a sequential sum over ascending rows (gemm_tn)."""
    (Ad, lda), (Bd, ldb) = _dev(A), _dev(B)
    m, p = (int(s) for s in Ad.shape)
    if m != int(Bd.shape[0]):
        raise DimensionError(f"matmul_tn of shapes {tuple(Ad.shape)} and {tuple(Bd.shape)}")
    n = int(Bd.shape[1])
    C = D.empty_f(p, n)
    _lib.check(_lib.lib().aqr_gemm_tn(m, p, n, Ad.data_ptr(), lda, Bd.data_ptr(), ldb, C.data_ptr(),
                                      max(p, 1), D.stream_ptr()), "aqr_gemm_tn")
    return C


def cholesky_upper(G):
    """Upper Cholesky factor of (G + G.T)/2; NotPositiveDefiniteError at the first bad pivot."""
    t = D.torch()
    Gd, ldg = _dev(G)
    n = int(Gd.shape[0])
    if int(Gd.shape[1]) != n:
        raise DimensionError(f"cholesky_upper needs a square matrix, got {tuple(Gd.shape)}")
    Gs = 0.5 * (Gd + Gd.transpose(0, 1))  # elementwise, as numpy's 0.5 * (G + G.T)
    Gs = Gs.t().contiguous().t()
    R = D.empty_f(n, n)
    fail = t.empty(1, dtype=t.int32, device=R.device)
    _lib.check(_lib.lib().aqr_cholesky_upper(n, Gs.data_ptr(), n, R.data_ptr(), n, fail.data_ptr(),
                                             D.stream_ptr()), "aqr_cholesky_upper")
    bad = int(fail.item())
    if bad >= 0:
        raise NotPositiveDefiniteError(bad)
    return R


def tri_solve_right(Z, R):
    """Solve X @ R = Z for X (R upper triangular, diagonal nonzero and finite)."""
    t = D.torch()
    (Zd, ldz), (Rd, ldr) = _dev(Z), _dev(R)
    m, n = (int(s) for s in Zd.shape)
    if tuple(Rd.shape) != (n, n):
        raise DimensionError(f"R must be {n}x{n}, got {tuple(Rd.shape)}")
    diag = t.diagonal(Rd)
    if bool((diag == 0.0).any()) or not bool(t.isfinite(diag).all()):
        raise SingularMatrixError("triangular factor has a zero or non-finite diagonal entry")
    X = D.empty_f(m, n)
    _lib.check(_lib.lib().aqr_tri_solve_right(m, n, Zd.data_ptr(), ldz, Rd.data_ptr(), ldr, X.data_ptr(),
                                              max(m, 1), D.stream_ptr()), "aqr_tri_solve_right")
    return X
