"""Parity of the B200 path against the reference (golden fixtures) and the
C oracle, through the drop-in API (which calls libaqr_b200.so's C ABI).

Tolerances.  The GPU differs from the reference only
in the ORDER of the dot-product reductions (tree instead of sequential); all
elementwise updates and operator products are bitwise reference-exact.  The
tolerance for each case is therefore TOL_FACTOR times the spread between the
oracle with sequential dots and the oracle with pairwise dots on the same
inputs (tests/parity.py), floored at a few ulps:

  * Q: max |dQ_ij| / max(|Q_ij|, 1e-3 max_i |Q_ij|)   (column-norm floor)
  * R: max |dR| / max |R|
"""

import numpy as np
import pytest

from oracle import oracle as O

import parity

pytestmark = pytest.mark.gpu

GS_METHODS = [f"{f}-{v}-{o}" for f in ("mgs", "cgs") for v in ("naive", "ha", "hp")
              for o in ("col", "row")]
MGS_METHODS = [m for m in GS_METHODS if m.startswith("mgs")]


@pytest.fixture(scope="module")
def aqr():
    import paper_1703_10440_b200 as P

    return P


def _op(aqr, golden, key):
    if f"{key}|A" in golden:
        return aqr.DenseSpdOperator(golden[f"{key}|A"]), ("dense", golden[f"{key}|A"])
    spec = ("csr", golden[f"{key}|indptr"], golden[f"{key}|indices"], golden[f"{key}|data"])
    return aqr.CsrSpdOperator(*spec[1:]), spec


def test_hand_instance_exact(aqr):
    # test_gram_schmidt.py:66-77 / test_acceptance.py:130-140: exact in binary64
    Z = np.array([[1.0, 1.0], [0.0, 1.0]])
    for meth in GS_METHODS + ["cholqr"]:
        r = aqr.factorize(Z, aqr.diagonal_operator([1.0, 4.0]), meth)
        assert np.array_equal(r.Q, [[1.0, 0.0], [0.0, 0.5]]), meth
        assert np.array_equal(r.R, [[1.0, 1.0], [0.0, 2.0]]), meth


@pytest.mark.parametrize("key", ["dense1", "dense2", "dense3", "dense7", "ident", "illcond",
                                 "csr9x7", "csr16"])
def test_golden_parity(aqr, golden, key):
    Z = golden[f"{key}|Z"]
    op, spec = _op(aqr, golden, key)
    for meth in GS_METHODS:
        if f"{key}|{meth}|Q" not in golden:
            continue
        Qref, Rref = golden[f"{key}|{meth}|Q"], golden[f"{key}|{meth}|R"]
        before = op.mv_count
        r = aqr.factorize(Z, op, meth)
        assert op.mv_count - before == r.cost.mv_count == int(golden[f"{key}|{meth}|mv"][0])
        assert r.cost.flops == int(golden[f"{key}|{meth}|mv"][1])
        tq, tr = parity.tolerance(Z, spec, meth)
        eq, er = parity.factor_errors(r.Q, r.R, Qref, Rref)
        assert eq <= tq and er <= tr, (key, meth, eq, tq, er, tr)
        assert r.flagged_columns == golden[f"{key}|{meth}|flag"].tolist()


@pytest.mark.parametrize("key", ["dense3", "dense7", "csr16", "illcond"])
def test_col_row_bitwise_on_gpu(aqr, golden, key):
    # gram_schmidt.py:19-21; test_gram_schmidt.py:119-130: same reduction tree
    Z = golden[f"{key}|Z"]
    op, _ = _op(aqr, golden, key)
    for fam in ("mgs", "cgs"):
        for var in ("naive", "ha", "hp"):
            a = aqr.factorize(Z, op, f"{fam}-{var}-col")
            b = aqr.factorize(Z, op, f"{fam}-{var}-row")
            assert np.array_equal(a.Q, b.Q) and np.array_equal(a.R, b.R), (fam, var)


def test_rerun_bitwise_deterministic(aqr, golden):
    Z = golden["dense7|Z"]
    op, _ = _op(aqr, golden, "dense7")
    for meth in MGS_METHODS:
        a = aqr.factorize(Z, op, meth)
        b = aqr.factorize(Z, op, meth)
        assert np.array_equal(a.Q, b.Q) and np.array_equal(a.R, b.R)


def test_identity_reduces_to_textbook_mgs(aqr, golden):
    # test_gram_schmidt.py:133-150: HP within 1e-14 ||Z|| of textbook MGS
    Z = golden["ident|Z"]
    Qr, Rr = golden["ident|mgs-ha-col|Q"], golden["ident|mgs-ha-col|R"]  # == textbook MGS
    op = aqr.identity_operator(25)
    scale = np.linalg.norm(Z)
    for meth in MGS_METHODS:
        r = aqr.factorize(Z, op, meth)
        assert np.max(np.abs(r.Q - Qr)) <= 1e-14 * scale, meth
        assert np.max(np.abs(r.R - Rr)) <= 1e-14 * scale, meth


def test_mv_counts_and_flops(aqr, golden):
    Z = golden["dense3|Z"]
    op, _ = _op(aqr, golden, "dense3")
    m, n = Z.shape
    for meth in GS_METHODS + ["cholqr"]:
        before = op.mv_count
        r = aqr.factorize(Z, op, meth)
        expected = 2 * n if "naive" in meth else n
        assert op.mv_count - before == expected == r.cost.mv_count, meth


def test_hp_uses_one_block_call(aqr, golden):
    # test_gram_schmidt.py:97-116: the operator sees the reference's granularity
    Z = golden["dense1|Z"]
    op, _ = _op(aqr, golden, "dense1")
    n = Z.shape[1]
    calls = []
    original_block, original_apply = op.apply_block, op.apply

    def spy_block(X):
        calls.append(("block", X.shape[1]))
        return original_block(X)

    def spy_apply(x):
        calls.append(("single", 1))
        return original_apply(x)

    op.apply_block, op.apply = spy_block, spy_apply
    ref_hp = None
    for orientation in ("row", "col"):  # host-input pipeline and column orientation keep one block call
        calls.clear()
        aqr.mgs_hp(Z, op, orientation)
        assert calls == [("block", n)], orientation
    calls.clear()
    r = aqr.mgs_hp(Z, op)
    assert calls == [("block", n)]
    calls.clear()
    aqr.mgs_ha(Z, op)
    assert calls == [("single", 1)] * n
    calls.clear()
    aqr.mgs_naive(Z, op, "row")
    assert calls == [("single", 1)] * (2 * n)
    # the callback route runs the same kernels: bitwise equal to the native route
    del op.apply_block, op.apply
    ref_hp = aqr.mgs_hp(Z, op)
    assert np.array_equal(r.Q, ref_hp.Q) and np.array_equal(r.R, ref_hp.R)


def test_custom_host_operator_plugin(aqr, golden):
    # a user SpdOperator implementing only the reference's _apply_into hook
    A = golden["dense2|A"]

    class HostOp(aqr.SpdOperator):
        def __init__(self):
            super().__init__(A.shape[0])

        def _apply_into(self, x, y):
            y[:] = O.matvec(A, x)

    Z = golden["dense2|Z"]
    a = aqr.mgs_ha(Z, HostOp(), "row")
    b = aqr.mgs_ha(Z, aqr.DenseSpdOperator(A), "row")
    assert np.array_equal(a.Q, b.Q) and np.array_equal(a.R, b.R)


def test_breakdown_kat(aqr, golden_cases):
    # test_gram_schmidt.py:193-200
    Z = np.array([[1.0, 2.0], [0.0, 0.0], [0.0, 0.0]])
    for meth, (col, val) in golden_cases["breakdown_rank_deficient"].items():
        op = aqr.identity_operator(3)
        with pytest.raises(aqr.BreakdownError) as info:
            aqr.factorize(Z, op, meth)
        assert info.value.column == col, meth
        assert info.value.value == val, meth
        variant = meth.split("-")[1]
        assert op.mv_count == {"hp": 2, "ha": col + 1, "naive": 2 * col + 1}[variant], meth


def test_flag_kat(aqr, golden_cases):
    # test_gram_schmidt.py:269-281
    for meth, ref in golden_cases["flag_tiny_norm"].items():
        r = aqr.factorize(np.array([[1.0], [1e-16]]), aqr.diagonal_operator([1e-30, 1.0]), meth)
        assert r.flagged_columns == [0]
        assert r.R[0, 0] == ref["R00"] > 0
        assert r.Q.ravel().tolist() == ref["Q"]


def test_triangular_positive_diagonal(aqr, golden):
    Z = golden["dense3|Z"]
    op, _ = _op(aqr, golden, "dense3")
    n = Z.shape[1]
    for meth in GS_METHODS + ["cholqr"]:
        R = aqr.factorize(Z, op, meth).R
        assert np.array_equal(np.tril(R, -1), np.zeros((n, n))), meth
        assert np.all(np.diag(R) > 0), meth


def test_input_not_mutated_and_torch_roundtrip(aqr, golden):
    import torch

    Z = golden["dense3|Z"].copy(order="F")
    Z0 = Z.copy()
    op, _ = _op(aqr, golden, "dense3")
    r = aqr.mgs_hp(Z, op, "row")
    assert np.array_equal(Z, Z0)
    Zt = torch.from_numpy(Z).cuda()
    rt = aqr.mgs_hp(Zt, op, "row")
    assert rt.Q.is_cuda and rt.R.is_cuda
    assert np.array_equal(rt.Q.cpu().numpy(), r.Q) and np.array_equal(rt.R.cpu().numpy(), r.R)
    assert torch.equal(Zt.cpu(), torch.from_numpy(Z0))


def test_cfg1_parity_against_oracle(aqr, golden_cases):
    """Config 1 (BASELINE.json configs[0]): every MGS variant x orientation."""
    import cfg1

    A, Z = cfg1.make()
    op = aqr.DenseSpdOperator(A)
    ref = golden_cases["cfg1"]["methods"]
    for meth in MGS_METHODS:
        r = aqr.factorize(Z, op, meth)
        o = O.gs_factor(Z, ("dense", A), meth)
        tq, tr = parity.tolerance(Z, ("dense", A), meth)
        eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
        assert eq <= tq and er <= tr, (meth, eq, tq, er, tr)
        loss = aqr.loss_of_A_orthogonality(r.Q, op)
        rep_rel = aqr.residual_rel(Z, r.Q, r.R)
        # no worse than the reference's own values on the same inputs
        # (margin: the metric's own fp64 evaluation noise, 1.05x)
        assert loss <= 1.05 * ref[meth]["loss_A_orth"], (meth, loss, ref[meth]["loss_A_orth"])
        assert rep_rel <= 1.05 * ref[meth]["rep_rel_Z"] + 1e-17, (meth, rep_rel)
        assert r.flagged_columns == ref[meth]["flagged"]


def test_operator_products_bitwise(aqr, golden):
    # the products are reference-exact: dense (matvec order) and CSR (stored order)
    import torch

    A = golden["dense7|A"]
    op = aqr.DenseSpdOperator(A)
    X = golden["dense7|Z"]
    for c in range(4):
        assert np.array_equal(op.apply(X[:, c]), O.matvec(A, X[:, c]))
    Y = op.apply_block(X)
    for c in range(X.shape[1]):
        assert np.array_equal(Y[:, c], O.matvec(A, X[:, c]))
    ip, ix, dv = golden["csr16|indptr"], golden["csr16|indices"], golden["csr16|data"]
    Zc = golden["csr16|Z"]
    for hint in (0, 1, 4, 5, 6, 8, 64):  # the row-batch hint never changes results
        cop = aqr.CsrSpdOperator(ip, ix, dv, max_row_nnz=hint)
        Y = cop.apply_block(Zc)
        for c in range(Zc.shape[1]):
            ref = O.csr_matvec(ip, ix, dv, Zc[:, c])
            assert np.array_equal(cop.apply(Zc[:, c]), ref), hint
            assert np.array_equal(Y[:, c], ref), hint
    assert torch.equal(cop.apply(torch.from_numpy(Zc[:, 0]).cuda()).cpu(),
                       torch.from_numpy(O.csr_matvec(ip, ix, dv, Zc[:, 0])))


def test_operator_counts_and_errors(aqr):
    op = aqr.identity_operator(3)
    assert np.array_equal(op.apply([1.0, 2.0, 3.0]), [1.0, 2.0, 3.0])
    op.apply_block(np.ones((3, 2), order="F"))
    assert op.mv_count == 3
    with pytest.raises(aqr.DimensionError):
        op.apply([1.0, 2.0])
    with pytest.raises(aqr.DimensionError):
        op.apply_block(np.ones((2, 2)))


@pytest.mark.parametrize("meth,chunk", [("mgs-ha-row", 0), ("mgs-ha-row", 1), ("mgs-ha-row", 3),
                                        ("mgs-hp-row", 0), ("mgs-hp-row", 4), ("mgs-naive-row", 3),
                                        ("cgs-ha-row", 3), ("cgs-hp-row", 0), ("mgs-naive-col", 0)])
def test_pinned_host_input_streams_q_bitwise(aqr, meth, chunk, monkeypatch):
    """Page-locked host Z: Z streams in by column chunks (each chunk replays
    the steps already done) and Q streams back while later steps run
    (aqr_gs_factor_pinned); results equal the device-resident call bitwise."""
    import torch

    monkeypatch.setenv("AQR_CHUNK_COLS", str(chunk))

    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.laplacian5(640, 480, 1e-2)  # m = 307200: the RPT = 8 tiles
    m, n = 640 * 480, 10
    op = aqr.CsrSpdOperator(ip, ix, dv)
    Z = problems.rng(9, 0).standard_normal((n, m)).T
    Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
    Zh.copy_(torch.from_numpy(Z))
    rd = aqr.factorize(Zh.cuda(), op, meth)
    rh = aqr.factorize(Zh, op, meth)
    assert not rh.Q.is_cuda and rh.Q.is_pinned() and not rh.R.is_cuda
    assert torch.equal(rh.Q, rd.Q.cpu()) and torch.equal(rh.R, rd.R.cpu())
    assert rh.cost.mv_count == rd.cost.mv_count


@pytest.mark.parametrize("sched,catchup", [("0", "1"), ("1", "1"), ("2", "1"), ("0", "2"), ("1", "0")])
def test_pipeline_chunk_schedules_bitwise(aqr, sched, catchup, monkeypatch):
    """Every chunk schedule of the host-input pipeline (aqr_pipe_chunks:
    uniform, tapered, ramped + tapered) and every catch-up form (one
    cooperative launch with one grid barrier per step and per-CTA totals;
    with two barriers around a totals phase; per-step launches) -- chunks of
    1 .. n/8 columns, balanced (tile, column) unit ranges -- gives the
    device-resident bits, for numpy (staged) and page-locked inputs."""
    import torch

    from paper_1703_10440_b200 import problems

    monkeypatch.setenv("AQR_PIPE_SCHED", sched)
    monkeypatch.setenv("AQR_CATCHUP", catchup)
    ip, ix, dv = problems.laplacian5(640, 480, 1e-2)
    m, n = 640 * 480, 21
    op = aqr.CsrSpdOperator(ip, ix, dv)
    Z = np.asfortranarray(problems.rng(9, 7).standard_normal((m, n)))
    Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
    Zh.copy_(torch.from_numpy(Z))
    for meth in ("mgs-ha-row", "mgs-hp-row", "cgs-ha-row", "cgs-hp-row", "mgs-naive-row"):
        rd = aqr.factorize(Zh.cuda(), op, meth)
        for Zin in (Zh, Z):
            rh = aqr.factorize(Zin, op, meth)
            Qh = rh.Q if isinstance(rh.Q, np.ndarray) else rh.Q.numpy()
            Rh = rh.R if isinstance(rh.R, np.ndarray) else rh.R.numpy()
            assert np.array_equal(Qh, rd.Q.cpu().numpy()) and np.array_equal(Rh, rd.R.cpu().numpy()), (meth, sched)


def test_host_c_entry_matches_device_path(aqr):
    """aqr_gs_factor_host (numpy buffers, int64 CSR)."""
    import ctypes

    from paper_1703_10440_b200 import _lib, problems

    ip, ix, dv = problems.laplacian5(96, 80, 1e-2)
    m, n = 96 * 80, 9
    Z = np.asfortranarray(problems.rng(9, 1).standard_normal((m, n)))
    op = aqr.CsrSpdOperator(ip, ix, dv)
    L = _lib.lib()
    ip64, ix64 = np.ascontiguousarray(ip, dtype=np.int64), np.ascontiguousarray(ix, dtype=np.int64)
    dv64 = np.ascontiguousarray(dv, dtype=np.float64)
    d, i64 = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
    for fam, var, ori, meth in ((0, 1, 1, "mgs-ha-row"), (0, 2, 1, "mgs-hp-row"), (1, 0, 0, "cgs-naive-col")):
        Q = np.empty((m, n), order="F")
        R = np.empty((n, n), order="F")
        flags = np.zeros(n, dtype=np.int32)
        fail, fval, mv = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int64()
        st = L.aqr_gs_factor_host(fam, var, ori, m, n, Z.ctypes.data_as(d), Q.ctypes.data_as(d),
                                  R.ctypes.data_as(d), 1, None, ip64.ctypes.data_as(i64),
                                  ix64.ctypes.data_as(i64), dv64.ctypes.data_as(d), int(ix64.size),
                                  ctypes.byref(fail), ctypes.byref(fval),
                                  flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(mv))
        assert st == 0, L.aqr_last_error()
        r = aqr.factorize(Z, op, meth)
        assert np.array_equal(Q, r.Q) and np.array_equal(R, r.R), meth
        assert mv.value == r.cost.mv_count


def test_large_numpy_input_staged_h2d_bitwise(aqr):
    """numpy in / numpy out above the staging threshold (threaded page-locked
    H2D staging, streamed D2H): same bits as the device-resident call."""
    import torch

    from paper_1703_10440_b200 import _device, problems

    ip, ix, dv = problems.laplacian5(1024, 1024, 1e-2)
    m, n = 1024 * 1024, 9
    assert 8 * m * n >= _device._STAGE_MIN_BYTES
    op = aqr.CsrSpdOperator(ip, ix, dv)
    Z = np.asfortranarray(problems.rng(9, 2).standard_normal((m, n)))
    Z0 = Z.copy(order="F")
    r = aqr.mgs_ha(Z, op, "row")
    rd = aqr.mgs_ha(torch.from_numpy(Z.T).cuda().t(), op, "row")
    assert isinstance(r.Q, np.ndarray) and r.Q.flags.f_contiguous and r.Q.shape == (m, n)
    assert np.array_equal(r.Q, rd.Q.cpu().numpy()) and np.array_equal(r.R, rd.R.cpu().numpy())
    assert np.array_equal(Z, Z0)


@pytest.mark.parametrize("chunk", [0, 1, 2])
def test_pipeline_breakdown_and_edges(aqr, chunk, monkeypatch):
    """Host-input pipeline edge cases: a breakdown in a late chunk (same
    column, value and mv_count as the device call), n = 1, m = n, and a
    callback operator."""
    import torch

    from paper_1703_10440_b200 import problems

    monkeypatch.setenv("AQR_CHUNK_COLS", str(chunk))
    ip, ix, dv = problems.laplacian5(40, 30, 1e-2)
    m, n = 1200, 9
    op = aqr.CsrSpdOperator(ip, ix, dv)
    Z = np.asfortranarray(problems.rng(9, 4).standard_normal((m, n)))
    Z[:, 6] = 0.0  # breakdown at column 6 (t = 0 exactly)
    for meth in ("mgs-ha-row", "mgs-hp-row", "mgs-naive-row"):
        got = []
        for Zin in (Z, torch.from_numpy(Z.T).cuda().t()):
            o = aqr.CsrSpdOperator(ip, ix, dv)
            with pytest.raises(aqr.BreakdownError) as info:
                aqr.factorize(Zin, o, meth)
            got.append((info.value.column, info.value.value, o.mv_count))
        assert got[0] == got[1], (meth, got)
        assert got[0][0] == 6, (meth, got)
    # n = 1 and m = n
    for Zs in (Z[:, :1], np.asfortranarray(problems.rng(9, 5).standard_normal((8, 8)))):
        A = np.eye(Zs.shape[0]) * 2.0 + 0.1
        dop = aqr.DenseSpdOperator(A)
        for meth in ("mgs-ha-row", "mgs-hp-row", "cgs-naive-row"):
            a = aqr.factorize(np.asfortranarray(Zs), dop, meth)
            b = aqr.factorize(torch.from_numpy(np.ascontiguousarray(Zs.T)).cuda().t(), dop, meth)
            assert np.array_equal(a.Q, b.Q.cpu().numpy()) and np.array_equal(a.R, b.R.cpu().numpy()), meth

    # callback route (user SpdOperator) through the pipeline
    class HostOp(aqr.SpdOperator):
        def __init__(self):
            super().__init__(m)

        def _apply_into(self, x, y):
            y[:] = O.csr_matvec(ip, ix, dv, x)

    Zc = np.asfortranarray(problems.rng(9, 6).standard_normal((m, n)))
    for meth in ("mgs-ha-row", "mgs-hp-row"):
        a = aqr.factorize(Zc, HostOp(), meth)
        b = aqr.factorize(Zc, op, meth)
        assert np.array_equal(a.Q, b.Q) and np.array_equal(a.R, b.R), meth
