"""Instrumented SPD operators, device resident (drop-in for aqr.operators).

Mirrors /root/reference/pkg/src/aqr/operators.py: the same classes, argument
conventions, validation errors and ``mv_count`` cost unit (one increment per
applied column, operators.py:50-66).  The matrix lives in B200 HBM: dense A
column-major fp64, CSR with int32 indptr/indices (guarded nnz < 2^31) and
fp64 values, uploaded once on first use.  Products run in the sm_100a kernels
of libaqr_b200.so and accumulate in the reference's order, so ``apply`` and
``apply_block`` are bitwise equal to the reference's matvec / csr_matvec.

``apply``/``apply_block`` accept numpy arrays (and lists), host torch
tensors and CUDA torch tensors, and return the same kind.  The operator
counter is a plain attribute: confine an operator to one thread per
factorization (operators.py:8-9).
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .exceptions import DimensionError


@dataclass
class CostReport:
    """Cost of one factorization: measured MV count plus a model flop count (operators.py:20-25)."""

    mv_count: int
    flops: int


def as_matrix(a):
    """Coerce to the library's matrix carrier: float64, Fortran-ordered, 2-D (operators.py:28-33).

    Torch tensors are accepted as they are (2-D check only); they are moved
    to the device in column-major layout when a kernel needs them.
    """
    if D.is_torch(a):
        if a.dim() != 2:
            raise DimensionError(f"expected a 2-D matrix, got ndim={a.dim()}")
        return a
    m = np.asfortranarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise DimensionError(f"expected a 2-D matrix, got ndim={m.ndim}")
    return m


def _shape(a):
    return tuple(int(s) for s in a.shape)


def _in_vector(x, dim):
    """Device vector for ``x`` plus a function that converts results back."""
    t = D.torch() if D.is_torch(x) else None
    if t is not None:
        v = x
        if v.dim() != 1 or v.shape[0] != dim:
            raise DimensionError(f"expected a vector of length {dim}, got shape {tuple(v.shape)}")
        dev = D.device()
        on_dev = v.is_cuda
        v = v.to(dev, t.float64).contiguous()
        back = (lambda y: y) if on_dev else (lambda y: y.cpu())
        return v, back
    v = np.ascontiguousarray(x, dtype=np.float64)
    if v.ndim != 1 or v.shape[0] != dim:
        raise DimensionError(f"expected a vector of length {dim}, got shape {np.shape(x)}")
    dev = D.device()
    return D.torch().from_numpy(v).to(dev), (lambda y: y.cpu().numpy())


def _in_block(X, dim):
    X = as_matrix(X)
    if _shape(X)[0] != dim:
        raise DimensionError(f"block has {_shape(X)[0]} rows, operator dimension is {dim}")
    on_dev = D.is_torch(X) and X.is_cuda
    Xd, ld = D.to_device_f(X)
    if on_dev:
        back = lambda Y: Y
    elif D.is_torch(X):
        back = lambda Y: Y.cpu()
    else:
        back = lambda Y: np.asfortranarray(Y.cpu().numpy())
    return Xd, ld, back


class SpdOperator:
    """Base class (operators.py:43-73).

    Subclasses either provide a native device realization (``_native``) or
    implement the reference's host plug-in ``_apply_into(x, y)`` on numpy
    vectors; the latter runs on the host inside the user's operator.
    """

    def __init__(self, dim):
        self.dim = int(dim)
        self.mv_count = 0

    # ---- public API (operators.py:50-66) ----
    def apply(self, x):
        """Return A @ x and increment the counter by one."""
        xd, back = _in_vector(x, self.dim)
        y = D.torch().empty(self.dim, dtype=xd.dtype, device=xd.device)
        self._apply_dev(1, xd.data_ptr(), self.dim, y.data_ptr(), self.dim)
        self.mv_count += 1
        return back(y)

    def apply_block(self, X):
        """Apply to every column (bitwise equal to single applies), counter +k."""
        Xd, ldx, back = _in_block(X, self.dim)
        k = _shape(Xd)[1]
        Y = D.empty_f(self.dim, k)
        if k:
            self._apply_dev(k, Xd.data_ptr(), ldx, Y.data_ptr(), self.dim)
        self.mv_count += k
        return back(Y)

    # ---- device realization ----
    def _native(self):
        """aqr_op descriptor for a built-in realization, else None."""
        return None

    def _apply_dev(self, k, X, ldx, Y, ldy):
        desc = self._native()
        if desc is not None:
            _lib.check(_lib.lib().aqr_op_apply(ctypes.byref(desc), k, X, ldx, Y, ldy, D.stream_ptr()),
                       "aqr_op_apply")
            return
        # host plug-in: column loop of _apply_into (operators.py:68-70)
        for c in range(k):
            xv = D.wrap(X + 8 * c * ldx, self.dim, 1, ldx).cpu().numpy().copy()
            yv = np.empty(self.dim)
            self._apply_into(xv, yv)
            D.wrap(Y + 8 * c * ldy, self.dim, 1, ldy).copy_(D.torch().from_numpy(yv))

    def _apply_into(self, x, y):
        raise NotImplementedError


class DenseSpdOperator(SpdOperator):
    """Dense realization: A m x m, column-major fp64 in HBM (operators.py:76-93)."""

    def __init__(self, matrix):
        A = as_matrix(matrix)
        if _shape(A)[0] != _shape(A)[1]:
            raise DimensionError(f"operator matrix must be square, got {_shape(A)}")
        super().__init__(_shape(A)[0])
        self.matrix = A
        self._dev = None
        self._desc = None

    def _device_matrix(self):
        if self._dev is None:
            self._dev, self._lda = D.to_device_f(self.matrix)
        return self._dev

    def _native(self):
        if self._desc is None:
            A = self._device_matrix()
            d = _lib.AqrOp()
            d.kind = _lib.AQR_OP_DENSE
            d.m = self.dim
            d.A = A.data_ptr()
            d.lda = self._lda
            self._desc = d
        return self._desc

    def to_dense(self):
        return self.matrix


class CsrSpdOperator(SpdOperator):
    """Compressed sparse row realization (operators.py:96-129).

    ``indptr``/``indices``/``data`` may be numpy arrays (validated exactly as
    the reference does, int64 host copies kept) or CUDA tensors (validated on
    the device, used for inputs generated on the GPU).  ``max_row_nnz``: the
    longest row, measured here when not given; it only selects the SpMV
    kernel's row batch (results are identical for every value).
    """

    def __init__(self, indptr, indices, data, dim=None, max_row_nnz=None, banded=None):
        self._band = None
        self.banded = banded  # None: use the banded view when the operator qualifies; False: never
        if D.is_torch(indptr):
            self._init_device(indptr, indices, data, dim)
        else:
            indptr = np.ascontiguousarray(indptr, dtype=np.int64)
            indices = np.ascontiguousarray(indices, dtype=np.int64)
            data = np.ascontiguousarray(data, dtype=np.float64)
            m = indptr.shape[0] - 1
            if dim is not None and dim != m:
                raise DimensionError(f"indptr implies dimension {m}, got dim={dim}")
            if indptr[0] != 0 or indptr[-1] != data.shape[0] or indices.shape[0] != data.shape[0]:
                raise DimensionError("inconsistent CSR arrays")
            if np.any(np.diff(indptr) < 0):
                raise DimensionError("indptr must be non-decreasing")
            if data.shape[0] and (indices.min() < 0 or indices.max() >= m):
                raise DimensionError("column index out of range")
            super().__init__(m)
            self.indptr, self.indices, self.data = indptr, indices, data
            self._dev = None
        if max_row_nnz is None:
            if D.is_torch(self.indptr):
                d = self.indptr[1:] - self.indptr[:-1]
                max_row_nnz = int(d.max()) if d.numel() else 0
            else:
                max_row_nnz = int(np.diff(self.indptr).max()) if self.dim else 0
        self.max_row_nnz = int(max_row_nnz)
        self._desc = None

    def _init_device(self, indptr, indices, data, dim):
        t = D.torch()
        m = int(indptr.shape[0]) - 1
        if dim is not None and dim != m:
            raise DimensionError(f"indptr implies dimension {m}, got dim={dim}")
        nnz = int(data.shape[0])
        if int(indptr[0]) != 0 or int(indptr[-1]) != nnz or int(indices.shape[0]) != nnz:
            raise DimensionError("inconsistent CSR arrays")
        if bool((indptr[1:] < indptr[:-1]).any()):
            raise DimensionError("indptr must be non-decreasing")
        if nnz and (int(indices.min()) < 0 or int(indices.max()) >= m):
            raise DimensionError("column index out of range")
        super().__init__(m)
        self._check_int32(m, nnz)
        self._dev = _pack_csr(indptr, indices, data)
        self.indptr, self.indices, self.data = indptr, indices, data

    @staticmethod
    def _check_int32(m, nnz):
        if nnz >= 2**31 or m >= 2**31:
            raise ValueError("nnz and dim must be < 2**31 for the int32 device CSR layout")

    @property
    def nnz(self):
        return int(self.data.shape[0])

    def _device_arrays(self):
        if self._dev is None:
            self._check_int32(self.dim, self.nnz)
            self._dev = _pack_csr(self.indptr, self.indices, self.data)
        return self._dev

    def _native(self):
        if self._desc is None:
            ip, ix, dv, _ = self._device_arrays()
            d = _lib.AqrOp()
            d.kind = _lib.AQR_OP_CSR
            d.max_row_nnz = min(self.max_row_nnz, 2**31 - 1)
            d.m = self.dim
            d.indptr, d.indices, d.data = ip.data_ptr(), ix.data_ptr(), dv.data_ptr()
            d.nnz = self.nnz
            if self.banded is None or self.banded:
                # stencil operators: offsets + row masks instead of per-entry
                # indices (aqr_csr_band_create; nd == 0 when it does not qualify)
                band = _lib.AqrBand()
                _lib.check(_lib.lib().aqr_csr_band_create(ctypes.byref(d), ctypes.byref(band), D.stream_ptr()),
                           "aqr_csr_band_create")
                if band.nd > 0:
                    self._band = band
                    d.band = ctypes.pointer(band)
            self._desc = d
        return self._desc

    @property
    def band_offsets(self):
        """Column offsets of the banded view (None when the CSR kernels run)."""
        self._native()
        return None if self._band is None else [int(self._band.off[i]) for i in range(self._band.nd)]

    def __del__(self):
        band, self._band = getattr(self, "_band", None), None
        if band is not None and band.nd > 0:
            try:
                _lib.lib().aqr_csr_band_destroy(ctypes.byref(band))
            except Exception:  # interpreter shutdown
                pass

    def to_dense(self):
        indptr = np.asarray(self.indptr.cpu() if D.is_torch(self.indptr) else self.indptr)
        indices = np.asarray(self.indices.cpu() if D.is_torch(self.indices) else self.indices)
        data = np.asarray(self.data.cpu() if D.is_torch(self.data) else self.data)
        A = np.zeros((self.dim, self.dim), order="F")
        rows = np.repeat(np.arange(self.dim), np.diff(indptr))
        np.add.at(A, (rows, indices), data)
        return A


def _pack_csr(indptr, indices, data):
    """Device copies (int32 indptr, int32 indices, fp64 data) in ONE allocation.

    values first, then indices, then row pointers: one contiguous range the
    factorization can mark L2-persisting (aqr_gs_factor, l2_window_begin).
    """
    t = D.torch()
    dev = D.device()
    nnz, m1 = int(data.shape[0]), int(indptr.shape[0])
    off_i = 8 * nnz
    off_p = off_i + 4 * nnz + (4 * nnz) % 8
    buf = t.empty(off_p + 4 * m1 + 16, dtype=t.uint8, device=dev)
    dv = buf[:off_i].view(t.float64)
    ix = buf[off_i:off_i + 4 * nnz].view(t.int32)
    ip = buf[off_p:off_p + 4 * m1].view(t.int32)
    as_t = (lambda a, dt: a.to(dev, dt)) if D.is_torch(data) else \
        (lambda a, dt: t.from_numpy(np.ascontiguousarray(a)).to(dev, dt))
    dv.copy_(as_t(data, t.float64))
    ix.copy_(as_t(indices, t.int32))
    ip.copy_(as_t(indptr, t.int32))
    return ip, ix, dv, buf


def csr_from_coo(dim, rows, cols, values):
    """Build a CSR operator from coordinate triplets; duplicates are summed (operators.py:132-151)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, values = rows[order], cols[order], values[order]
    if rows.shape[0]:
        dup = np.zeros(rows.shape[0], dtype=bool)
        dup[1:] = (rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])
        if dup.any():
            keep = ~dup
            group = np.cumsum(keep) - 1
            summed = np.zeros(int(keep.sum()))
            np.add.at(summed, group, values)
            rows, cols, values = rows[keep], cols[keep], summed
    indptr = np.zeros(dim + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    indptr = np.cumsum(indptr)
    return CsrSpdOperator(indptr, cols, values)


def identity_operator(m):
    """Dense identity operator (applies still count as MVs)."""
    return DenseSpdOperator(np.eye(m))


def diagonal_operator(d):
    """Dense operator with the given diagonal."""
    d = np.asarray(d, dtype=np.float64)
    return DenseSpdOperator(np.diag(d))


def as_operator(obj):
    """Accept an existing operator or a square dense array."""
    if isinstance(obj, SpdOperator):
        return obj
    return DenseSpdOperator(obj)
