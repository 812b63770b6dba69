"""CPU-only checks: the drop-in API surface, host-side validation, the C-ABI
library exports, and the problem generators.  No kernel is launched."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1703_10440_b200 as aqr
from paper_1703_10440_b200 import _lib, problems

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_public_names_match_reference_hot_path():
    # names the drop-in keeps (aqr/__init__.py:14-80)
    for name in ["mgs_naive", "mgs_ha", "mgs_hp", "cgs", "cholesky_qr", "factorize", "MethodId",
                 "QrResult", "CostReport", "SpdOperator", "DenseSpdOperator", "CsrSpdOperator",
                 "BreakdownError", "DimensionError", "NotPositiveDefiniteError", "ALL_GS_METHODS",
                 "SWEEP_METHODS", "CHOLQR", "UNIT_ROUNDOFF", "as_matrix", "as_operator",
                 "csr_from_coo", "identity_operator", "diagonal_operator",
                 "loss_of_A_orthogonality", "representation_error", "delta_bounds"]:
        assert hasattr(aqr, name), name
    assert aqr.UNIT_ROUNDOFF == 2.0 ** -53
    assert len(aqr.ALL_GS_METHODS) == 12 and len(aqr.SWEEP_METHODS) == 7


def test_method_id_grammar():
    # test_gram_schmidt.py:254-266
    for text in [str(m) for m in aqr.ALL_GS_METHODS] + ["cholqr"]:
        assert str(aqr.MethodId.parse(text)) == text
    for bad in ("mgs-ha", "qr", "mgs-fast-col", "cholqr-col", "cgs-ha-diag"):
        with pytest.raises(ValueError):
            aqr.MethodId.parse(bad)
    with pytest.raises(ValueError):
        aqr.MethodId("cholqr", "ha", "col")


def test_orientation_and_variant_errors():
    op = aqr.identity_operator(3)
    with pytest.raises(ValueError):
        aqr.mgs_ha(np.ones((3, 2)), op, "diag")
    with pytest.raises(ValueError):
        aqr.cgs(np.ones((3, 2)), op, "fast")


def test_dimension_errors_before_any_work():
    # gram_schmidt.py:116-123: raised before the device is touched
    op = aqr.identity_operator(3)
    with pytest.raises(aqr.DimensionError):
        aqr.mgs_naive(np.ones((2, 3)), op)  # m < n
    with pytest.raises(aqr.DimensionError):
        aqr.mgs_naive(np.ones((4, 2)), op)  # operator mismatch
    with pytest.raises(aqr.DimensionError):
        aqr.mgs_hp(np.ones((3, 0)), op)  # n < 1
    with pytest.raises(aqr.DimensionError):
        aqr.factorize(np.ones(3), op, "mgs-ha-row")  # not 2-D


def test_operator_validation():
    # test_operators.py:93-105
    with pytest.raises(aqr.DimensionError):
        aqr.CsrSpdOperator(np.array([0, 1]), np.array([5]), np.array([1.0]))
    with pytest.raises(aqr.DimensionError):
        aqr.CsrSpdOperator(np.array([0, 2]), np.array([0]), np.array([1.0]))
    with pytest.raises(aqr.DimensionError):
        aqr.CsrSpdOperator(np.array([0, 2, 1]), np.array([0, 1]), np.array([1.0, 2.0]))
    with pytest.raises(aqr.DimensionError):
        aqr.DenseSpdOperator(np.ones((2, 3)))
    op = aqr.csr_from_coo(2, [0, 0, 1], [1, 1, 0], [2.0, 3.0, 4.0])
    A = op.to_dense()
    assert A[0, 1] == 5.0 and A[1, 0] == 4.0 and op.nnz == 2


def test_compute_without_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(aqr.ExtensionUnavailable):
        aqr.mgs_ha(np.eye(3, 2), aqr.identity_operator(3))
    with pytest.raises(aqr.ExtensionUnavailable):
        aqr.identity_operator(3).apply([1.0, 2.0, 3.0])


def _header_functions():
    text = open(os.path.join(REPO, "include", "aqr_b200.h")).read()
    return sorted(set(re.findall(r"AQR_API\s+[\w\s\*]+?\b(aqr_\w+)\s*\(", text)))


def test_c_abi_library_exports_every_header_symbol():
    L = _lib.load(require_device=False)
    names = _header_functions()
    assert len(names) >= 20
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    for name in names:
        assert getattr(L, name) is not None
    assert L.aqr_abi_version() == _lib.ABI_VERSION
    # host-only queries (no device needed)
    assert L.aqr_tile_rows(1000) == 256 and L.aqr_num_tiles(1000) == 4
    assert L.aqr_tile_rows(1 << 20) == 2048 and L.aqr_num_tiles(1 << 20) == 512
    ws = L.aqr_workspace_bytes(_lib.AQR_MGS, _lib.AQR_HP, _lib.AQR_ROW, 1000, 50)
    assert ws >= 8 * 1000 * 50 + 8 * 2 * 1000
    assert L.aqr_status_bytes(50) == 16 + 4 * 50


def _pipe_chunks(n, chunk, sched=None):
    code = (
        "import numpy as np, sys\n"
        "from paper_1703_10440_b200 import _lib\n"
        "L = _lib.load(require_device=False)\n"
        f"b = np.zeros({n} + 1, dtype=np.int64)\n"
        f"k = L.aqr_pipe_chunks({n}, {chunk}, b.ctypes.data, {n} + 1)\n"
        "print(' '.join(str(int(v)) for v in b[: k + 1]))\n"
    )
    import subprocess
    import sys

    env = dict(os.environ)
    env.pop("AQR_PIPE_SCHED", None)
    env.pop("AQR_LIB_PATH", None)
    if sched is not None:  # the alternative schedules exist in the experiments build only
        env["AQR_PIPE_SCHED"] = str(sched)
        env["AQR_LIB_PATH"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "paper_1703_10440_b200", "libaqr_b200_exp.so")
    out = subprocess.run([sys.executable, "-c", code], env=env, check=True, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    return [int(v) for v in out.stdout.split()]


@pytest.mark.parametrize("n", [1, 2, 7, 9, 64, 100, 256])
def test_pipeline_chunk_schedule(n):
    """aqr_pipe_chunks (host logic, no device): boundaries 0 .. n strictly
    increasing; chunk_cols > 0 gives uniform chunks; the default schedule is
    ceil(n/8)-column chunks; the tapered schedule halves towards the end and
    the ramped one also starts with ceil(n/8)/4 columns."""
    w = max(1, (n + 7) // 8)
    for sched in (None, 1, 2):
        b = _pipe_chunks(n, 0, sched)
        assert b[0] == 0 and b[-1] == n and all(x < y for x, y in zip(b, b[1:])), (sched, b)
        widths = [y - x for x, y in zip(b, b[1:])]
        assert max(widths) <= w, (sched, b)
        if sched is None:
            assert widths == [w] * (n // w) + ([n % w] if n % w else []), b
        if sched == 1 and n > w:
            assert widths[-1] == 1 and widths[: (n - w) // w] == [w] * ((n - w) // w), b
        if sched == 2 and w >= 4 and n > 2 * w:
            assert widths[0] == w // 4, b
    b = _pipe_chunks(n, 3, 1)  # explicit chunk width: uniform whatever the schedule
    assert b == list(range(0, n, 3)) + [n], b


def test_ctypes_struct_layout_matches_header():
    # aqr_op / aqr_factor_args as declared in include/aqr_b200.h (LP64)
    assert ctypes.sizeof(_lib.AqrOp) == 4 + 4 + 8 + 8 + 8 + 8 * 3 + 8 + 8 * 3 + 8 + 8
    assert _lib.AqrOp.band.offset == ctypes.sizeof(_lib.AqrOp) - 8
    # aqr_band: nd, constant, off[32], val[32], mask, dvals
    assert ctypes.sizeof(_lib.AqrBand) == 4 + 4 + 8 * 32 + 8 * 32 + 8 + 8
    assert _lib.AqrFactorArgs.flagged_host.offset == 4 * 4 + 8 * 2 + 8 * 6 + 8 + 8 + 8 + 8 + 8 + 8
    # aqr_p2p_group: 2 x int32, 3 arrays of AQR_MAX_RANKS (8) pointers / int64, n_halo, 2 pointers,
    # seq0, timeout_ns
    assert ctypes.sizeof(_lib.AqrP2PGroup) == 8 + 3 * 8 * 8 + 8 + 16 + 8 + 8
    assert _lib.AqrP2PGroup.seq0.offset == 8 + 3 * 64 + 8 + 16
    assert _lib.AqrP2PGroup.timeout_ns.offset == 8 + 3 * 64 + 8 + 16 + 8


def test_generators_match_reference_laplacian(golden):
    ip, ix, dv = problems.laplacian5(9, 7, 0.0)
    assert np.array_equal(ip, golden["csr9x7|indptr"])
    assert np.array_equal(ix, golden["csr9x7|indices"])
    assert np.array_equal(dv, golden["csr9x7|data"])


def test_config2_shape_and_nnz():
    ip, ix, dv = problems.laplacian5(1024, 1024, 1e-2)
    assert ip[-1] == 5_238_784 == dv.shape[0]
    assert np.all(dv[ip[:-1] + (ix[ip[:-1]] < np.arange(1024 * 1024)).astype(int)] != 0)


def test_diffusion7_symmetric_and_diagonally_dominant():
    import scipy.sparse as sp

    ip, ix, dv = problems.diffusion7(12, 1e-3, problems.rng(3, 0))
    A = sp.csr_matrix((dv, ix, ip))
    assert abs(A - A.T).max() == 0.0
    d = A.diagonal()
    off = np.asarray(abs(A).sum(axis=1)).ravel() - d
    assert np.all(d > off)
    assert ip[-1] == 7 * 12 ** 3 - 6 * 12 ** 2


def test_stage_pool_size_follows_input_width():
    """Host staging threads: throttled for wide (compute-bound) inputs, the
    full pool for narrow ones and plain copies; AQR_STAGE_THREADS overrides."""
    from paper_1703_10440_b200 import _device as D

    cores = os.cpu_count() or 4
    old = D._STAGE_THREADS
    try:
        D._STAGE_THREADS = 0
        assert D._stage_pool(256)._max_workers == max(2, min(4, cores))
        assert D._stage_pool(64)._max_workers == max(2, min(8, cores))
        assert D._stage_pool()._max_workers == max(2, min(8, cores))
        assert D._stage_pool(256) is D._stage_pool(1024)  # one pool per size
        D._STAGE_THREADS = 3
        assert D._stage_pool(256)._max_workers == 3 and D._stage_pool(8)._max_workers == 3
    finally:
        D._STAGE_THREADS = old
