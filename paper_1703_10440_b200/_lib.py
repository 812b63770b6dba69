"""Loader and ctypes signatures of libaqr_b200.so (the C ABI in include/aqr_b200.h).

The extension is built in-tree (``python -m paper_1703_10440_b200._build`` or
``__graft_entry__.build()``) so the .so travels with the repository snapshot.
There is no fallback: if the library or a CUDA device is missing, every
compute entry point raises :class:`ExtensionUnavailable`.
"""

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# AQR_LIB_PATH: an alternative build of the same library (tools/ A/B experiments)
LIB_PATH = os.environ.get("AQR_LIB_PATH") or os.path.join(_HERE, "libaqr_b200.so")
ABI_VERSION = 3

AQR_OK, AQR_EDIM, AQR_EBREAKDOWN, AQR_ECUDA, AQR_EARG, AQR_ENOMEM, AQR_ECALLBACK, AQR_ETIMEOUT = range(8)
AQR_MGS, AQR_CGS = 0, 1
AQR_NAIVE, AQR_HA, AQR_HP = 0, 1, 2
AQR_COL, AQR_ROW = 0, 1
AQR_OP_DENSE, AQR_OP_CSR, AQR_OP_CALLBACK = 0, 1, 2

FAMILY_CODE = {"mgs": AQR_MGS, "cgs": AQR_CGS}
VARIANT_CODE = {"naive": AQR_NAIVE, "ha": AQR_HA, "hp": AQR_HP}
ORIENTATION_CODE = {"col": AQR_COL, "row": AQR_ROW}


class ExtensionUnavailable(RuntimeError):
    """libaqr_b200.so or a CUDA device is missing: the product path refuses to run."""


c_i32, c_i64, c_u64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p

APPLY_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp)


BAND_MAX = 32


class AqrBand(ctypes.Structure):
    _fields_ = [
        ("nd", c_i32), ("constant", c_i32),
        ("off", c_i64 * BAND_MAX), ("val", c_dbl * BAND_MAX),
        ("mask", c_vp), ("dvals", c_vp),
    ]


class AqrOp(ctypes.Structure):
    _fields_ = [
        ("kind", c_i32), ("max_row_nnz", c_i32), ("m", c_i64),
        ("A", c_vp), ("lda", c_i64),
        ("indptr", c_vp), ("indices", c_vp), ("data", c_vp), ("nnz", c_i64),
        ("apply", APPLY_FN), ("apply_block", APPLY_FN), ("ctx", c_vp),
        ("ncols", c_i64),
        ("band", ctypes.POINTER(AqrBand)),
    ]


class AqrFactorArgs(ctypes.Structure):
    _fields_ = [
        ("family", c_i32), ("variant", c_i32), ("orientation", c_i32), ("reserved", c_i32),
        ("m", c_i64), ("n", c_i64),
        ("Z", c_vp), ("ldz", c_i64), ("Q", c_vp), ("ldq", c_i64), ("R", c_vp), ("ldr", c_i64),
        ("op", ctypes.POINTER(AqrOp)),
        ("workspace", c_vp), ("workspace_bytes", c_u64),
        ("fail_col", c_i64), ("fail_val", c_dbl), ("mv_count", c_i64),
        ("flagged_host", ctypes.POINTER(c_i32)),
    ]


MAX_RANKS = 8


class AqrP2PGroup(ctypes.Structure):
    _fields_ = [
        ("nranks", c_i32), ("rank", c_i32),
        ("xbuf", c_vp * MAX_RANKS), ("W", c_vp * MAX_RANKS), ("ldw", c_i64 * MAX_RANKS),
        ("n_halo", c_i64), ("halo_rank", c_vp), ("halo_row", c_vp),
        ("seq0", c_u64), ("timeout_ns", c_u64),
    ]


# name -> (restype, argtypes); every symbol declared in include/aqr_b200.h
SIGNATURES = {
    "aqr_workspace_bytes": (c_u64, [c_i32, c_i32, c_i32, c_i64, c_i64]),
    "aqr_pipe_workspace_bytes": (c_u64, [c_i32, c_i32, c_i32, c_i64, c_i64]),
    "aqr_gs_factor": (c_i32, [ctypes.POINTER(AqrFactorArgs), c_vp]),
    "aqr_p2p_exchange_bytes": (c_u64, [c_i64]),
    "aqr_p2p_alloc": (c_i32, [c_u64, ctypes.POINTER(c_vp)]),
    "aqr_p2p_free": (c_i32, [c_vp]),
    "aqr_ipc_handle": (c_i32, [c_vp, ctypes.c_char_p]),
    "aqr_ipc_open": (c_i32, [ctypes.c_char_p, ctypes.POINTER(c_vp)]),
    "aqr_ipc_close": (c_i32, [c_vp]),
    "aqr_p2p_gs_factor": (c_i32, [ctypes.POINTER(AqrFactorArgs), ctypes.POINTER(AqrP2PGroup), c_vp]),
    "aqr_p2p_gs_factor_lockstep": (c_i32, [c_i32, ctypes.POINTER(ctypes.POINTER(AqrFactorArgs)),
                                           ctypes.POINTER(ctypes.POINTER(AqrP2PGroup)), c_vp]),
    "aqr_trace_read": (c_i64, [c_vp, c_i64]),
    "aqr_gs_factor_d2h": (c_i32, [ctypes.POINTER(AqrFactorArgs), c_vp, c_i64, c_vp, c_i64, c_vp]),
    "aqr_gs_factor_pinned": (c_i32, [ctypes.POINTER(AqrFactorArgs), c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                     c_i64, c_vp, c_vp]),
    "aqr_pipe_chunks": (c_i64, [c_i64, c_i64, c_vp, c_i64]),
    "aqr_gs_factor_host": (c_i32, [c_i32, c_i32, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_i32,
                                   c_vp, c_vp, c_vp, c_vp, c_i64, ctypes.POINTER(c_i64),
                                   ctypes.POINTER(c_dbl), c_vp, ctypes.POINTER(c_i64)]),
    "aqr_csr_band_create": (c_i32, [ctypes.POINTER(AqrOp), ctypes.POINTER(AqrBand), c_vp]),
    "aqr_csr_band_destroy": (None, [ctypes.POINTER(AqrBand)]),
    "aqr_op_apply": (c_i32, [ctypes.POINTER(AqrOp), c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "aqr_block_apply": (c_i32, [ctypes.POINTER(AqrOp), c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "aqr_dot": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "aqr_sub_scaled": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "aqr_div_scalar": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "aqr_matvec": (c_i32, [c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "aqr_apply_block_dense": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "aqr_csr_matvec": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "aqr_gemm_tn": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "aqr_gemm_nn": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "aqr_cholesky_upper": (c_i32, [c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "aqr_tri_solve_right": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "aqr_tile_rows": (c_i64, [c_i64]),
    "aqr_num_tiles": (c_i64, [c_i64]),
    "aqr_step_col_update_norm": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "aqr_step_norm_reduce": (c_i32, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "aqr_step_norm_finish": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "aqr_step_normalize": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "aqr_step_trailing": (c_i32, [c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp,
                                  c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_vp, c_vp]),
    "aqr_step_rrow_reduce": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "aqr_step_finalize_r": (c_i32, [c_i64, c_vp, c_vp, c_i64, c_vp]),
    "aqr_status_bytes": (c_u64, [c_i64]),
    "aqr_status_init": (c_i32, [c_vp, c_i64, c_vp]),
    "aqr_launch_count": (c_u64, []),
    "aqr_trailing_timer_enable": (c_i32, [c_i32]),
    "aqr_trailing_timer_read": (c_i32, [ctypes.POINTER(c_i64), ctypes.POINTER(c_dbl),
                                        ctypes.POINTER(c_dbl)]),
    "aqr_kernel_timer_read": (c_i32, [c_i32, ctypes.POINTER(c_i64), ctypes.POINTER(c_dbl),
                                      ctypes.POINTER(c_dbl)]),
    "aqr_kernel_timer_list": (c_i64, [c_i32, c_vp, c_vp, c_i64]),
    "aqr_last_error": (ctypes.c_char_p, []),
    "aqr_abi_version": (c_i32, []),
}

_lib = None
_lock = threading.Lock()


def load(require_device=False):
    """Load the in-tree library (no device needed to load it)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ExtensionUnavailable(
                    f"{LIB_PATH} is missing; build it with `python -m paper_1703_10440_b200._build`")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            if L.aqr_abi_version() != ABI_VERSION:
                raise ExtensionUnavailable("libaqr_b200.so ABI version mismatch; rebuild it")
            _lib = L
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise ExtensionUnavailable("no CUDA device: the aqr B200 path has no CPU fallback")
    return _lib


def lib():
    """The library, with a CUDA device guaranteed (compute entry points)."""
    return load(require_device=True)


def check(status, what="aqr"):
    if status == AQR_OK:
        return
    msg = _lib.aqr_last_error().decode(errors="replace") if _lib is not None else ""
    raise RuntimeError(f"{what} failed with status {status}: {msg}")
