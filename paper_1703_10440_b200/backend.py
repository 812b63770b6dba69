"""Kernel namespace (drop-in for /root/reference/pkg/src/aqr/backend.py).

The reference resolves ``kernels()`` to one of two interchangeable CPU
backends (backend.py:17-68) holding the loop-level kernels of
_kernels_impl.py.  Here there is exactly one backend, ``"b200"``: the same
kernel names and calling conventions (caller-owned float64 buffers, in-place
outputs, ``None`` returned except by ``seq_dot`` and
``cholesky_upper_kernel``), each one sm_100a kernel of libaqr_b200.so.  No
CPU fallback and no second backend exist (``set_backend`` accepts only
``"b200"`` / ``"auto"``).

Arguments may be numpy arrays (copied to the device, outputs written back
in place) or CUDA tensors (used in place; vectors contiguous, matrices
column-major).  Every kernel keeps the reference's operation order and is
bitwise equal to it, except ``seq_dot``: a deterministic tree reduction
(the order every factorization kernel uses), equal to the sequential sum
up to rounding.
"""

import ctypes
from contextlib import contextmanager

import numpy as np

from . import _device as D
from . import _lib

ENV_VAR = "AQR_BACKEND"
_NAMES = ("b200",)


def _resolve(name):
    name = (name or "auto").strip().lower()
    if name == "auto":
        return "b200"
    if name not in _NAMES:
        raise ValueError(f"unknown backend {name!r} (choose one of: auto, b200)")
    return name


_current = "b200"  # AQR_BACKEND names the reference's CPU backends; there is one here


def current_backend():
    """Name of the active backend (always ``"b200"``)."""
    return _current


def set_backend(name):
    """Validate and select ``name``; returns the previous backend name."""
    global _current
    previous = _current
    _current = _resolve(name)
    return previous


@contextmanager
def use_backend(name):
    """Context manager form of ``set_backend``."""
    previous = set_backend(name)
    try:
        yield
    finally:
        set_backend(previous)


class _Buf:
    """Device view of an argument; ``done()`` writes an output back to numpy."""

    def __init__(self, a, matrix):
        t = D.torch()
        self.host = None
        if D.is_torch(a) and a.is_cuda:
            if a.dtype != t.float64:
                raise TypeError("kernel buffers are float64")
            if matrix:
                ld = D.leading_dim(a)
                if ld is None:
                    raise ValueError("device matrices must be column-major")
                self.T, self.ld = a, ld
            else:
                if not a.is_contiguous():
                    raise ValueError("device vectors must be contiguous")
                self.T, self.ld = a, max(int(a.shape[0]), 1)
            return
        arr = a.numpy() if D.is_torch(a) else a
        self.host = arr
        if matrix:
            self.T, self.ld = D.to_device_f(np.asarray(arr, dtype=np.float64))
        else:
            self.T = t.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(D.device())
            self.ld = max(int(self.T.shape[0]), 1)

    @property
    def ptr(self):
        return self.T.data_ptr()

    def done(self):
        if self.host is not None:
            self.host[...] = self.T.cpu().numpy()


def _chk(st, what):
    _lib.check(st, what)


def _scalar_dev(v):
    t = D.torch()
    return t.tensor([float(v)], dtype=t.float64, device=D.device())


class _B200Kernels:
    """The kernel namespace (_kernels_impl.py:17-164) on the device."""

    @staticmethod
    def seq_dot(x, y):
        t = D.torch()
        bx, by = _Buf(x, False), _Buf(y, False)
        out = t.empty(1, dtype=t.float64, device=D.device())
        _chk(_lib.lib().aqr_dot(int(bx.T.shape[0]), bx.ptr, by.ptr, out.data_ptr(), D.stream_ptr()), "aqr_dot")
        return float(out.item())

    @staticmethod
    def matvec(A, x, y):
        bA, bx, by = _Buf(A, True), _Buf(x, False), _Buf(y, False)
        m, ncols = (int(s) for s in bA.T.shape)
        op = _lib.AqrOp()
        op.kind, op.m, op.ncols, op.A, op.lda = _lib.AQR_OP_DENSE, m, ncols, bA.ptr, bA.ld
        _chk(_lib.lib().aqr_op_apply(ctypes.byref(op), 1, bx.ptr, max(ncols, 1), by.ptr, max(m, 1),
                                     D.stream_ptr()), "aqr_op_apply")
        by.done()

    @staticmethod
    def apply_block_dense(A, X, Y):
        bA, bX, bY = _Buf(A, True), _Buf(X, True), _Buf(Y, True)
        m, k = int(bA.T.shape[0]), int(bX.T.shape[1])
        _chk(_lib.lib().aqr_apply_block_dense(m, k, bA.ptr, bA.ld, bX.ptr, bX.ld, bY.ptr, bY.ld, D.stream_ptr()),
             "aqr_apply_block_dense")
        bY.done()

    @staticmethod
    def csr_matvec(indptr, indices, data, x, y):
        t = D.torch()
        dev = D.device()
        ip = t.as_tensor(np.asarray(indptr.cpu() if D.is_torch(indptr) else indptr), dtype=t.int32).to(dev)
        ix = t.as_tensor(np.asarray(indices.cpu() if D.is_torch(indices) else indices), dtype=t.int32).to(dev)
        bd, bx, by = _Buf(data, False), _Buf(x, False), _Buf(y, False)
        m = int(ip.shape[0]) - 1
        _chk(_lib.lib().aqr_csr_matvec(m, ip.data_ptr(), ix.data_ptr(), bd.ptr, bx.ptr, by.ptr, D.stream_ptr()),
             "aqr_csr_matvec")
        by.done()

    @staticmethod
    def gemm_nn(A, B, C):
        bA, bB, bC = _Buf(A, True), _Buf(B, True), _Buf(C, True)
        m, kk = (int(s) for s in bA.T.shape)
        n = int(bB.T.shape[1])
        _chk(_lib.lib().aqr_gemm_nn(m, kk, n, bA.ptr, bA.ld, bB.ptr, bB.ld, bC.ptr, bC.ld, D.stream_ptr()),
             "aqr_gemm_nn")
        bC.done()

    @staticmethod
    def gemm_tn(A, B, C):
        bA, bB, bC = _Buf(A, True), _Buf(B, True), _Buf(C, True)
        m, p = (int(s) for s in bA.T.shape)
        n = int(bB.T.shape[1])
        _chk(_lib.lib().aqr_gemm_tn(m, p, n, bA.ptr, bA.ld, bB.ptr, bB.ld, bC.ptr, bC.ld, D.stream_ptr()),
             "aqr_gemm_tn")
        bC.done()

    @staticmethod
    def sub_scaled(z, a, q):
        bz, bq = _Buf(z, False), _Buf(q, False)
        av = _scalar_dev(a)
        _chk(_lib.lib().aqr_sub_scaled(int(bz.T.shape[0]), bz.ptr, av.data_ptr(), bq.ptr, D.stream_ptr()),
             "aqr_sub_scaled")
        bz.done()

    @staticmethod
    def div_scalar(x, r, out):
        bx, bo = _Buf(x, False), _Buf(out, False)
        rv = _scalar_dev(r)
        _chk(_lib.lib().aqr_div_scalar(int(bx.T.shape[0]), bx.ptr, rv.data_ptr(), bo.ptr, D.stream_ptr()),
             "aqr_div_scalar")
        bo.done()

    @staticmethod
    def cholesky_upper_kernel(G, R):
        """Left-looking upper Cholesky of G into R (G's upper triangle used as
        given, like the reference kernel; linalg.cholesky_upper symmetrizes
        first).  Returns the failing pivot index, -1 on success."""
        t = D.torch()
        bG, bR = _Buf(G, True), _Buf(R, True)
        n = int(bG.T.shape[0])
        fail = t.empty(1, dtype=t.int32, device=D.device())
        _chk(_lib.lib().aqr_cholesky_upper(n, bG.ptr, bG.ld, bR.ptr, bR.ld, fail.data_ptr(), D.stream_ptr()),
             "aqr_cholesky_upper")
        bR.done()
        return int(fail.item())

    @staticmethod
    def tri_solve_right_kernel(Z, R, X):
        bZ, bR, bX = _Buf(Z, True), _Buf(R, True), _Buf(X, True)
        m, n = (int(s) for s in bZ.T.shape)
        _chk(_lib.lib().aqr_tri_solve_right(m, n, bZ.ptr, bZ.ld, bR.ptr, bR.ld, bX.ptr, bX.ld, D.stream_ptr()),
             "aqr_tri_solve_right")
        bX.done()


_KERNELS = _B200Kernels()


def kernels():
    """Kernel namespace of the active backend (backend.py:66-68)."""
    return _KERNELS
