"""ctypes front-end of the CPU oracle (oracle/aqr_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.

``gs_factor`` mirrors ``aqr.gram_schmidt._gs_factor``
(/root/reference/pkg/src/aqr/gram_schmidt.py:126-179) and is bitwise
identical to it (pinned in tests/test_oracle_golden.py).
"""

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libaqr_oracle.so")
_lib = None
_lock = threading.Lock()

FAMILIES = {"mgs": 0, "cgs": 1}
VARIANTS = {"naive": 0, "ha": 1, "hp": 2}
ORIENTATIONS = {"col": 0, "row": 1}

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.POINTER(ctypes.c_int64)
_i32 = ctypes.POINTER(ctypes.c_int32)


def build():
    """Compile the oracle library with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build()
            L = ctypes.CDLL(_LIB_PATH)
            L.aqro_seq_dot.restype = ctypes.c_double
            L.aqro_seq_dot.argtypes = [ctypes.c_int64, _d, _d]
            L.aqro_gs_factor.restype = ctypes.c_int64
            L.aqro_gs_factor.argtypes = [
                ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                _d, ctypes.c_int, _d, _i64, _i64, _d, _d, _d, _i32, _i64, _d,
            ]
            L.aqro_cholesky_upper_kernel.restype = ctypes.c_int64
            L.aqro_cholesky_upper_kernel.argtypes = [ctypes.c_int64, _d, _d]
            L.aqro_tri_solve_right_kernel.restype = None
            L.aqro_tri_solve_right_kernel.argtypes = [ctypes.c_int64, ctypes.c_int64, _d, _d, _d]
            L.aqro_apply_block_dense.restype = None
            L.aqro_apply_block_dense.argtypes = [ctypes.c_int64, ctypes.c_int64, _d, _d, _d]
            L.aqro_cholesky_qr.restype = ctypes.c_int64
            L.aqro_cholesky_qr.argtypes = [ctypes.c_int64, ctypes.c_int64, _d, ctypes.c_int, _d, _i64, _i64, _d,
                                           _d, _d, _i64]
            L.aqro_last_phase_times.restype = None
            L.aqro_last_phase_times.argtypes = [_d]
            L.aqro_set_dot_mode.restype = None
            L.aqro_set_dot_mode.argtypes = [ctypes.c_int]
            L.aqro_householder_qr.restype = ctypes.c_int
            L.aqro_householder_qr.argtypes = [ctypes.c_int64, ctypes.c_int64, _d, _d]
            L.aqro_gemm_nn.restype = None
            L.aqro_gemm_nn.argtypes = [ctypes.c_int64] * 3 + [_d, _d, _d]
            L.aqro_gemm_tn.restype = None
            L.aqro_gemm_tn.argtypes = [ctypes.c_int64] * 3 + [_d, _d, _d]
            L.aqro_csr_matvec.restype = None
            L.aqro_csr_matvec.argtypes = [ctypes.c_int64, _i64, _i64, _d, _d, _d]
            L.aqro_matvec.restype = None
            L.aqro_matvec.argtypes = [ctypes.c_int64, ctypes.c_int64, _d, _d, _d]
            _lib = L
    return _lib


def _p(a, typ=_d):
    return a.ctypes.data_as(typ)


class OracleBreakdown(Exception):
    def __init__(self, column, value):
        super().__init__(f"breakdown at column {column} (z'Az = {value!r})")
        self.column = column
        self.value = value


class OracleResult:
    def __init__(self, Q, R, flagged, mv_count):
        self.Q, self.R, self.flagged_columns, self.mv_count = Q, R, flagged, mv_count


class pairwise_dots:
    """Context manager: run the oracle with pairwise instead of sequential dots.

    Used only to calibrate parity tolerances: the
    spread between the two orders is the rounding noise any reordered
    (e.g. GPU tree) reduction is entitled to.  The mode is per thread (the
    calling thread's oracle calls only).
    """

    def __enter__(self):
        lib().aqro_set_dot_mode(1)
        return self

    def __exit__(self, *exc):
        lib().aqro_set_dot_mode(0)


def seq_dot(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return lib().aqro_seq_dot(x.shape[0], _p(x), _p(y))


def gs_factor(Z, op, method):
    """Run the oracle factorization.

    ``op`` is ``("dense", A)`` or ``("csr", indptr, indices, data)``;
    ``method`` an id like ``"mgs-ha-row"``.  Raises OracleBreakdown.
    """
    family, variant, orientation = method.split("-")
    Z = np.asfortranarray(Z, dtype=np.float64)
    m, n = Z.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    flagged = np.zeros(n, dtype=np.int32)
    mv = ctypes.c_int64(0)
    fail = ctypes.c_double(0.0)
    null_d = ctypes.cast(None, _d)
    null_i = ctypes.cast(None, _i64)
    if op[0] == "dense":
        A = np.asfortranarray(op[1], dtype=np.float64)
        keep = (A,)
        args = (0, _p(A), null_i, null_i, null_d)
    else:
        indptr = np.ascontiguousarray(op[1], dtype=np.int64)
        indices = np.ascontiguousarray(op[2], dtype=np.int64)
        data = np.ascontiguousarray(op[3], dtype=np.float64)
        keep = (indptr, indices, data)
        args = (1, null_d, _p(indptr, _i64), _p(indices, _i64), _p(data))
    rc = lib().aqro_gs_factor(
        FAMILIES[family], VARIANTS[variant], ORIENTATIONS[orientation], m, n, _p(Z),
        *args, _p(Q), _p(R), _p(flagged, _i32), ctypes.byref(mv), ctypes.byref(fail),
    )
    del keep
    if rc == -2:
        raise ValueError(f"oracle: bad shape {Z.shape}")
    if rc == -3:
        raise MemoryError("oracle: allocation failed")
    if rc >= 0:
        raise OracleBreakdown(int(rc), fail.value)
    return OracleResult(Q, R, [int(j) for j in np.flatnonzero(flagged)], int(mv.value))


def last_phase_times():
    """(block apply, all normalize, all project) seconds of this thread's last gs_factor."""
    out = np.zeros(3)
    lib().aqro_last_phase_times(_p(out))
    return tuple(float(v) for v in out)


def extrapolate_seconds(phases, n_run, n_full):
    """Full-width time from a column-truncated run (n_run columns -> n_full).

    The block apply and the normalize steps scale with the column count, the
    projections with the number of (i, j) pairs, n (n - 1) / 2; at fixed m
    every call of one phase costs the same (gram_schmidt.py:136, 147-176)."""
    apply_s, norm_s, proj_s = phases
    lin = n_full / n_run
    pairs = (n_full * (n_full - 1)) / max(n_run * (n_run - 1), 1)
    return (apply_s + norm_s) * lin + proj_s * pairs


class OracleNotPositiveDefinite(Exception):
    def __init__(self, pivot):
        super().__init__(f"matrix not positive definite at pivot {pivot}")
        self.pivot = pivot


def _op_args(op):
    null_d = ctypes.cast(None, _d)
    null_i = ctypes.cast(None, _i64)
    if op[0] == "dense":
        A = np.asfortranarray(op[1], dtype=np.float64)
        return (A,), (0, _p(A), null_i, null_i, null_d)
    indptr = np.ascontiguousarray(op[1], dtype=np.int64)
    indices = np.ascontiguousarray(op[2], dtype=np.int64)
    data = np.ascontiguousarray(op[3], dtype=np.float64)
    return (indptr, indices, data), (1, null_d, _p(indptr, _i64), _p(indices, _i64), _p(data))


def cholesky_qr(Z, op):
    """Weighted Cholesky QR (gram_schmidt.py:209-218); raises OracleNotPositiveDefinite."""
    Z = np.asfortranarray(Z, dtype=np.float64)
    m, n = Z.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    mv = ctypes.c_int64(0)
    keep, args = _op_args(op)
    rc = lib().aqro_cholesky_qr(m, n, _p(Z), *args, _p(Q), _p(R), ctypes.byref(mv))
    del keep
    if rc == -2:
        raise ValueError(f"oracle: bad shape {Z.shape}")
    if rc == -3:
        raise MemoryError("oracle: allocation failed")
    if rc == -4:
        raise ZeroDivisionError("oracle: singular triangular factor")
    if rc >= 0:
        raise OracleNotPositiveDefinite(int(rc))
    return OracleResult(Q, R, [], int(mv.value))


def csr_matvec(indptr, indices, data, x):
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    data = np.ascontiguousarray(data, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(indptr.shape[0] - 1)
    lib().aqro_csr_matvec(y.shape[0], _p(indptr, _i64), _p(indices, _i64), _p(data), _p(x), _p(y))
    return y


def matvec(A, x):
    A = np.asfortranarray(A, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.shape[0])
    lib().aqro_matvec(A.shape[0], A.shape[1], _p(A), _p(x), _p(y))
    return y


def gemm_nn(A, B):
    """Sequential C = A @ B (_kernels_impl.py:59-69)."""
    A = np.asfortranarray(A, dtype=np.float64)
    B = np.asfortranarray(B, dtype=np.float64)
    C = np.empty((A.shape[0], B.shape[1]), order="F")
    lib().aqro_gemm_nn(A.shape[0], A.shape[1], B.shape[1], _p(A), _p(B), _p(C))
    return C


def gemm_tn(A, B):
    """Sequential C = A.T @ B (_kernels_impl.py:72-82)."""
    A = np.asfortranarray(A, dtype=np.float64)
    B = np.asfortranarray(B, dtype=np.float64)
    C = np.empty((A.shape[1], B.shape[1]), order="F")
    lib().aqro_gemm_tn(A.shape[0], A.shape[1], B.shape[1], _p(A), _p(B), _p(C))
    return C


def apply_block_dense(A, X):
    """Y = A X, column c exactly like matvec (_kernels_impl.py:35-47)."""
    A = np.asfortranarray(A, dtype=np.float64)
    X = np.asfortranarray(X, dtype=np.float64)
    Y = np.empty((A.shape[0], X.shape[1]), order="F")
    lib().aqro_apply_block_dense(A.shape[0], X.shape[1], _p(A), _p(X), _p(Y))
    return Y


def cholesky_upper_kernel(G):
    """(pivot or -1, R): _kernels_impl.py:134-152 on G's upper triangle."""
    G = np.asfortranarray(G, dtype=np.float64)
    R = np.zeros_like(G, order="F")
    bad = lib().aqro_cholesky_upper_kernel(G.shape[0], _p(G), _p(R))
    return int(bad), R


def tri_solve_right_kernel(Z, R):
    """X with X R = Z (_kernels_impl.py:155-164)."""
    Z = np.asfortranarray(Z, dtype=np.float64)
    R = np.asfortranarray(R, dtype=np.float64)
    X = np.empty_like(Z, order="F")
    lib().aqro_tri_solve_right_kernel(Z.shape[0], Z.shape[1], _p(Z), _p(R), _p(X))
    return X


def householder_q(G):
    """Thin, sign-fixed Q of a column-major Gaussian block (deterministic)."""
    G = np.asfortranarray(G, dtype=np.float64)
    m, k = G.shape
    Q = np.empty((m, k), order="F")
    bad = lib().aqro_householder_qr(m, k, _p(G), _p(Q))
    return Q, bool(bad)
