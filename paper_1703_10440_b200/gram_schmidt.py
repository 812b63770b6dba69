"""Thin QR in an SPD-weighted inner product on B200 (drop-in for aqr.gram_schmidt).

Same entry points, argument conventions, results and errors as
/root/reference/pkg/src/aqr/gram_schmidt.py: ``mgs_naive``, ``mgs_ha``,
``mgs_hp`` (182-194), ``cgs`` (197-206), ``cholesky_qr`` (209-218),
``factorize`` (227-233), ``MethodId`` (40-76), ``QrResult`` (92-104).

All arithmetic runs in libaqr_b200.so: one C call (``aqr_gs_factor``) runs
the whole factorization on the current CUDA stream, calling the operator
either natively (Dense/CsrSpdOperator) or through a callback into the
operator's public ``apply`` / ``apply_block`` (any other SpdOperator, or an
instance whose methods were replaced), so the MV granularity the reference
exposes (one ``apply_block`` for HP, one ``apply`` per column for HA, two for
naive) is preserved.

Inputs: numpy arrays return numpy results; torch tensors return torch
tensors on the input's device kind (CUDA tensors stay device resident).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .exceptions import BreakdownError, DimensionError
from .operators import CostReport, SpdOperator, as_matrix

UNIT_ROUNDOFF = 2.0 ** -53

FAMILIES = ("mgs", "cgs", "cholqr")
VARIANTS = ("naive", "ha", "hp")
ORIENTATIONS = ("col", "row")


@dataclass(frozen=True)
class MethodId:
    """Identifier of a factorization method (gram_schmidt.py:40-76)."""

    family: str
    variant: str | None = None
    orientation: str | None = None

    def __post_init__(self):
        if self.family == "cholqr":
            if self.variant is not None or self.orientation is not None:
                raise ValueError("cholqr takes no variant or orientation")
        elif self.family in ("mgs", "cgs"):
            if self.variant not in VARIANTS or self.orientation not in ORIENTATIONS:
                raise ValueError(f"bad method spec {self}")
        else:
            raise ValueError(f"unknown family {self.family!r}")

    @classmethod
    def parse(cls, text):
        """Parse ids like ``mgs-ha-col``, ``cgs-naive-row`` or ``cholqr``."""
        text = text.strip().lower()
        if text == "cholqr":
            return cls("cholqr")
        parts = text.split("-")
        if len(parts) != 3:
            raise ValueError(f"bad method id {text!r} (expected family-variant-orientation)")
        return cls(parts[0], parts[1], parts[2])

    def __str__(self):
        if self.family == "cholqr":
            return "cholqr"
        return f"{self.family}-{self.variant}-{self.orientation}"


CHOLQR = MethodId("cholqr")
ALL_GS_METHODS = tuple(
    MethodId(f, v, o) for f in ("mgs", "cgs") for v in VARIANTS for o in ORIENTATIONS
)
SWEEP_METHODS = tuple(
    [MethodId("mgs", v, "col") for v in VARIANTS]
    + [MethodId("cgs", v, "col") for v in VARIANTS]
    + [CHOLQR]
)


@dataclass
class QrResult:
    """Factors plus cost instrumentation (gram_schmidt.py:92-104)."""

    Q: object
    R: object
    cost: CostReport
    flagged_columns: list = field(default_factory=list)


def _model_flops(family, variant, m, n):
    # gram_schmidt.py:107-113
    if family == "cholqr":
        return 2 * m * n * n + m * n * n + n * n * n // 3
    if variant == "hp":
        return 3 * m * n * n
    return 2 * m * n * n


def _check_inputs(Z, op):
    Z = as_matrix(Z)
    m, n = (int(s) for s in Z.shape)
    if n < 1 or m < n:
        raise DimensionError(f"need m >= n >= 1, got {tuple(Z.shape)}")
    if op.dim != m:
        raise DimensionError(f"operator dimension {op.dim} does not match Z with {m} rows")
    return Z, m, n


def _result_converter(Z):
    if D.is_torch(Z):
        if Z.is_cuda:
            return lambda T: T
        if Z.is_pinned():
            def to_pinned(T):
                out = D.torch().empty((T.shape[1], T.shape[0]), dtype=T.dtype, pin_memory=True).t()
                out.copy_(T, non_blocking=True)
                D.torch().cuda.current_stream().synchronize()
                return out
            return to_pinned
        return lambda T: T.cpu()
    return lambda T: np.asfortranarray(T.cpu().numpy())


def _uses_native(op):
    cls = type(op)
    return (
        "apply" not in vars(op)
        and "apply_block" not in vars(op)
        and cls.apply is SpdOperator.apply
        and cls.apply_block is SpdOperator.apply_block
        and cls._apply_dev is SpdOperator._apply_dev
        and op._native() is not None
    )


class _Callback:
    """aqr_op of kind CALLBACK that routes every MV through op.apply / op.apply_block."""

    def __init__(self, op):
        self.op = op
        self.error = None
        m = op.dim

        def call(ctx, k, X, ldx, Y, ldy, stream):
            try:
                if k == 1:
                    # op.apply(Zw[:, j].copy()), gram_schmidt.py:151/163
                    y = op.apply(D.wrap(X, m, 1, ldx).clone())
                else:
                    y = op.apply_block(D.wrap(X, m, k, ldx))  # gram_schmidt.py:136
                D.wrap(Y, m, k, ldy).copy_(D.torch().as_tensor(y, device=D.device()))
                return 0
            except BaseException as e:  # re-raised by _gs_factor
                self.error = e
                return 1

        self._fn = _lib.APPLY_FN(call)
        self.desc = _lib.AqrOp()
        self.desc.kind = _lib.AQR_OP_CALLBACK
        self.desc.m = m
        self.desc.apply = self._fn
        self.desc.apply_block = self._fn


def _expected_mv(variant, n, fail_col):
    if variant == "hp":
        return n
    if fail_col is None:
        return 2 * n if variant == "naive" else n
    return 2 * fail_col + 1 if variant == "naive" else fail_col + 1


def _chunk_cols():
    import os

    return int(os.environ.get("AQR_CHUNK_COLS", "0"))  # 0: the library's schedule (aqr_pipe_chunks)


def _gs_factor(Z, op, family, variant, orientation):
    """The factorization driver (gram_schmidt.py:126-179) on the device."""
    Z, m, n = _check_inputs(Z, op)
    L = _lib.lib()
    t = D.torch()
    back = _result_converter(Z)
    mv_before = op.mv_count

    host_in = not (D.is_torch(Z) and Z.is_cuda)
    if host_in:  # Z stays on the host; aqr_gs_factor_pinned streams it in
        # 0: the library's schedule (n/8-column chunks).  HP: n/32-column
        # chunks -- the steps start after the first few columns arrived, and
        # the library merges the chunks already on the device into one
        # catch-up (config 5 HP numpy end to end 1551 ms at n/16, 1532 ms at
        # n/32; 1639 ms without merging)
        chunk = _chunk_cols() or (max(1, -(-n // 32)) if variant == "hp" else 0)
        bounds = np.zeros(n + 1, dtype=np.int64)
        nch = int(L.aqr_pipe_chunks(n, chunk, bounds.ctypes.data, n + 1))
        staged = D.StagedHost(Z, bounds[: nch + 1])  # page-locked copy, filled while the device starts
        Zh, ldzh = staged.T, staged.ld
        Q = D.empty_f(m, n)
        Zd, ldz = Q, m
    else:
        Zd, ldz = D.to_device_f(Z)
        Q = D.empty_f(m, n)
    R = D.empty_f(n, n)
    fam, var, ori = _lib.FAMILY_CODE[family], _lib.VARIANT_CODE[variant], _lib.ORIENTATION_CODE[orientation]
    wsb = int(L.aqr_workspace_bytes(fam, var, ori, m, n))
    if host_in:  # the pipeline's step vectors and catch-up partials follow
        wsb += int(L.aqr_pipe_workspace_bytes(fam, var, ori, m, n))
    ws = t.empty(wsb, dtype=t.uint8, device=Q.device)
    flags = np.zeros(n, dtype=np.int32)

    native = _uses_native(op)
    cb = None if native else _Callback(op)
    desc = op._native() if native else cb.desc

    a = _lib.AqrFactorArgs()
    a.family, a.variant, a.orientation = fam, var, ori
    a.m, a.n = m, n
    a.Z, a.ldz = Zd.data_ptr(), ldz
    a.Q, a.ldq = Q.data_ptr(), m
    a.R, a.ldr = R.data_ptr(), n
    a.op = ctypes.pointer(desc)
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    a.flagged_host = flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    if host_in:
        # host input (numpy or CPU tensor): Z streams in by column chunks and
        # Q columns stream back into page-locked host memory, both overlapped
        # with the steps (aqr_gs_factor_pinned); numpy callers get F-ordered
        # views of the page-locked block (it returns to torch's host cache
        # when they drop it)
        Qh = t.empty((n, m), dtype=t.float64, pin_memory=True).t()
        Rh = t.empty((n, n), dtype=t.float64, pin_memory=True).t()
        status = L.aqr_gs_factor_pinned(ctypes.byref(a), Zh.data_ptr(), ldzh, Qh.data_ptr(), m, Rh.data_ptr(), n,
                                        chunk, staged.ready, D.stream_ptr())
        staged.finish()
        if D.is_torch(Z):
            back = lambda T: Qh if T is Q else Rh  # noqa: E731
        else:
            back = lambda T: (Qh if T is Q else Rh).numpy()  # noqa: E731
    else:
        status = L.aqr_gs_factor(ctypes.byref(a), D.stream_ptr())
    if cb is not None and cb.error is not None:
        raise cb.error
    fail_col = int(a.fail_col) if status == _lib.AQR_EBREAKDOWN else None
    expected = _expected_mv(variant, n, fail_col)
    if native:
        op.mv_count += expected
    # a user operator counted its own calls: exactly the reference's, also
    # after a breakdown (the library stops calling it at the failing column)
    if status == _lib.AQR_EBREAKDOWN:
        raise BreakdownError(fail_col, float(a.fail_val))
    if status == _lib.AQR_EDIM:
        raise DimensionError(L.aqr_last_error().decode())
    _lib.check(status, "aqr_gs_factor")
    del Zd, ws
    if host_in:
        del Zh
    cost = CostReport(op.mv_count - mv_before, _model_flops(family, variant, m, n))
    return QrResult(back(Q), back(R), cost, [int(j) for j in np.flatnonzero(flags)])


def mgs_naive(Z, op, orientation="col"):
    """Modified Gram-Schmidt, two operator applications per column (2n MV)."""
    return _gs_factor(Z, op, "mgs", "naive", _check_orientation(orientation))


def mgs_ha(Z, op, orientation="col"):
    """Modified Gram-Schmidt, high-accuracy n-MV variant (sequential applies)."""
    return _gs_factor(Z, op, "mgs", "ha", _check_orientation(orientation))


def mgs_hp(Z, op, orientation="col"):
    """Modified Gram-Schmidt, high-performance n-MV variant (one block apply)."""
    return _gs_factor(Z, op, "mgs", "hp", _check_orientation(orientation))


def cgs(Z, op, variant="naive", orientation="col"):
    """Classical Gram-Schmidt in the weighted inner product (gram_schmidt.py:197-206)."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    return _gs_factor(Z, op, "cgs", variant, _check_orientation(orientation))


def cholesky_qr(Z, op):
    """Weighted Cholesky QR: R from chol(Z.T A Z), Q = Z R^{-1} (n MV) (gram_schmidt.py:209-218).

    X = A Z in the block-apply kernel, the Gram product Z^T X, the n x n
    left-looking Cholesky and the triangular solve in the repo's kernels in
    the reference's operation order (linalg.py), so Q and R are bitwise the
    reference's.
    """
    from . import linalg

    Z, m, n = _check_inputs(Z, op)
    t = D.torch()
    back = _result_converter(Z)
    mv_before = op.mv_count
    Zd, _ = D.to_device_f(Z)
    X = t.as_tensor(op.apply_block(Zd), device=Zd.device)
    G = linalg.matmul_tn(Zd, X)
    del X
    R = linalg.cholesky_upper(G)
    Q = linalg.tri_solve_right(Zd, R)
    cost = CostReport(op.mv_count - mv_before, _model_flops("cholqr", None, m, n))
    return QrResult(back(Q), back(R), cost)


def _check_orientation(orientation):
    if orientation not in ORIENTATIONS:
        raise ValueError(f"unknown orientation {orientation!r}")
    return orientation


def factorize(Z, op, method):
    """Run the factorization named by ``method`` (a MethodId or id string)."""
    if not isinstance(method, MethodId):
        method = MethodId.parse(method)
    if method.family == "cholqr":
        return cholesky_qr(Z, op)
    return _gs_factor(Z, op, method.family, method.variant, method.orientation)
