"""The banded view of stencil CSR operators (csrc/aqr_band.cuh,
aqr_csr_band_create): analysis, and bitwise equality of every product and
factorization with the plain CSR kernels (which are bitwise the reference's
csr_matvec, /root/reference/pkg/src/aqr/_kernels_impl.py:50-56) and parity
with the C oracle.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aqr():
    import paper_1703_10440_b200 as P

    return P


def _lap5(nx, ny):
    from paper_1703_10440_b200 import problems

    return problems.laplacian5(nx, ny, 1e-2)


def _diff7(n):
    from paper_1703_10440_b200 import problems

    return problems.diffusion7(n, 1e-3, np.random.default_rng(7))


def _st27(n):
    import torch

    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.stencil27_device(n, 1e-2, "cuda")
    torch.cuda.synchronize()
    return ip.cpu().numpy(), ix.cpu().numpy().astype(np.int64), dv.cpu().numpy()


CASES = {
    "lap5": (lambda: _lap5(37, 29), [-37, -1, 0, 1, 37], True),
    "diff7": (lambda: _diff7(11), [-121, -11, -1, 0, 1, 11, 121], False),
    "st27": (lambda: _st27(9), sorted((dz * 9 + dy) * 9 + dx for dz in (-1, 0, 1) for dy in (-1, 0, 1)
                                      for dx in (-1, 0, 1)), True),
    # three staged segments (the grid planes are further apart than a row block)
    "st27b": (lambda: _st27(21), sorted((dz * 21 + dy) * 21 + dx for dz in (-1, 0, 1) for dy in (-1, 0, 1)
                                        for dx in (-1, 0, 1)), True),
}


@pytest.mark.parametrize("name", list(CASES))
def test_analysis(aqr, name):
    make, offs, constant = CASES[name]
    op = aqr.CsrSpdOperator(*make())
    assert op.band_offsets == offs
    assert bool(op._band.constant) == constant
    assert aqr.CsrSpdOperator(*make(), banded=False).band_offsets is None


def test_analysis_rejects(aqr):
    rng = np.random.default_rng(3)
    m = 500
    # random sparsity: far more than 32 distinct offsets
    dense = rng.standard_normal((m, m)) * (rng.random((m, m)) < 0.02)
    dense = dense + dense.T + 50 * np.eye(m)
    ip, ix, dv = _dense_to_csr(dense)
    assert aqr.CsrSpdOperator(ip, ix, dv).band_offsets is None
    # a stencil whose rows are stored with descending columns: stored order != offset order
    ip, ix, dv = _lap5(8, 8)
    ix2, dv2 = ix.copy(), dv.copy()
    for r in range(len(ip) - 1):
        ix2[ip[r]:ip[r + 1]] = ix[ip[r]:ip[r + 1]][::-1]
        dv2[ip[r]:ip[r + 1]] = dv[ip[r]:ip[r + 1]][::-1]
    assert aqr.CsrSpdOperator(ip, ix2, dv2).band_offsets is None
    # sparsely populated diagonals (a diagonal matrix plus one far entry pair per 40 rows)
    m = 4000
    rows = list(range(m)) + [r for r in range(0, m - 100, 40) for _ in (0,)] + [r + 100 for r in range(0, m - 100, 40)]
    cols = list(range(m)) + [r + 100 for r in range(0, m - 100, 40)] + [r for r in range(0, m - 100, 40)]
    vals = [4.0] * m + [-1.0] * (len(rows) - m)
    order = np.lexsort((cols, rows))
    rows, cols, vals = np.array(rows)[order], np.array(cols)[order], np.array(vals)[order]
    ip = np.zeros(m + 1, dtype=np.int64)
    np.add.at(ip, rows + 1, 1)
    ip = np.cumsum(ip)
    assert aqr.CsrSpdOperator(ip, cols, vals).band_offsets is None


def _dense_to_csr(A):
    m = A.shape[0]
    ip = np.zeros(m + 1, dtype=np.int64)
    ix, dv = [], []
    for r in range(m):
        c = np.nonzero(A[r])[0]
        ix.append(c)
        dv.append(A[r, c])
        ip[r + 1] = ip[r] + len(c)
    return ip, np.concatenate(ix).astype(np.int64), np.concatenate(dv)


@pytest.mark.parametrize("name", list(CASES))
def test_products_bitwise(aqr, name):
    make, _, _ = CASES[name]
    csr = make()
    band, plain = aqr.CsrSpdOperator(*csr), aqr.CsrSpdOperator(*csr, banded=False)
    m = band.dim
    rng = np.random.default_rng(11)
    x = rng.standard_normal(m)
    yb, yp = band.apply(x), plain.apply(x)
    assert np.array_equal(yb, yp)
    assert np.array_equal(yb, O.csr_matvec(csr[0], csr[1], csr[2], x))
    for k in (2, 8, 13):
        X = np.asfortranarray(rng.standard_normal((m, k)))
        assert np.array_equal(band.apply_block(X), plain.apply_block(X))
    # an unknown row length (hint 0) takes the long-row route whatever the view's width
    hint0 = aqr.CsrSpdOperator(*csr, max_row_nnz=0)
    X = np.asfortranarray(rng.standard_normal((m, 5)))
    assert np.array_equal(hint0.apply_block(X), plain.apply_block(X))
    assert np.array_equal(hint0.apply(x), yp)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("method", ["mgs-naive-row", "mgs-ha-row", "mgs-hp-row", "mgs-ha-col", "cgs-ha-row",
                                    "cgs-hp-row"])
def test_factorization_bitwise(aqr, name, method):
    make, _, _ = CASES[name]
    csr = make()
    band, plain = aqr.CsrSpdOperator(*csr), aqr.CsrSpdOperator(*csr, banded=False)
    m = band.dim
    Z = np.asfortranarray(np.random.default_rng(5).standard_normal((m, 12)))
    rb, rp = aqr.factorize(Z, band, method), aqr.factorize(Z, plain, method)
    assert np.array_equal(rb.Q, rp.Q) and np.array_equal(rb.R, rp.R)
    assert rb.cost.mv_count == rp.cost.mv_count
    assert list(rb.flagged_columns) == list(rp.flagged_columns)


@pytest.mark.parametrize("name", ["lap5", "st27", "st27b"])
def test_vs_oracle(aqr, name):
    import parity

    make, _, _ = CASES[name]
    csr = make()
    spec = ("csr",) + tuple(csr)
    op = aqr.CsrSpdOperator(*csr)
    assert op.band_offsets is not None
    Z = np.asfortranarray(np.random.default_rng(6).standard_normal((op.dim, 10)))
    for method in ("mgs-ha-row", "mgs-hp-row"):
        r = aqr.factorize(Z, op, method)
        o = O.gs_factor(Z, spec, method)
        tq, tr = parity.tolerance(Z, spec, method)
        eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
        assert eq <= tq and er <= tr, (method, eq, tq, er, tr)
        assert r.cost.mv_count == o.mv_count


def test_large_rows_and_tail(aqr):
    """More rows than one pass of the norm grid (444 CTAs x 256), m not a multiple of 256."""
    csr = _lap5(613, 401)  # 245,813 rows
    band, plain = aqr.CsrSpdOperator(*csr), aqr.CsrSpdOperator(*csr, banded=False)
    Z = np.asfortranarray(np.random.default_rng(8).standard_normal((band.dim, 6)))
    for method in ("mgs-ha-row", "mgs-hp-row"):
        rb, rp = aqr.factorize(Z, band, method), aqr.factorize(Z, plain, method)
        assert np.array_equal(rb.Q, rp.Q) and np.array_equal(rb.R, rp.R)


def test_breakdown_same(aqr):
    """An indefinite stencil (negative shift) breaks down at the same column with the same value."""
    from paper_1703_10440_b200 import problems

    csr = problems.laplacian5(16, 16, -5.0)
    Z = np.asfortranarray(np.random.default_rng(9).standard_normal((256, 8)))
    errs = []
    for banded in (None, False):
        with pytest.raises(aqr.BreakdownError) as ei:
            aqr.mgs_ha(Z, aqr.CsrSpdOperator(*csr, banded=banded), "row")
        errs.append((ei.value.column, ei.value.value))
    assert errs[0] == errs[1]


@pytest.mark.parametrize("name", ["lap5", "diff7", "st27", "st27b"])
def test_padded_leading_dimensions_and_canaries(aqr, name):
    """C ABI products with ldx, ldy > m: results unchanged, the padding rows of Y untouched
    (compute-sanitizer is not available on the GPU pool; this is the bounds check)."""
    import ctypes

    import torch

    from paper_1703_10440_b200 import _device as D
    from paper_1703_10440_b200 import _lib

    make, _, _ = CASES[name]
    csr = make()
    band, plain = aqr.CsrSpdOperator(*csr), aqr.CsrSpdOperator(*csr, banded=False)
    m = band.dim
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(21)
    for k, pad in ((1, 0), (1, 5), (3, 7), (8, 16), (11, 3)):
        ld = m + pad
        X = torch.randn((k, ld), generator=g, device="cuda", dtype=torch.float64)  # column j = row j
        X[:, m:] = float("nan")  # padding rows of X must never be read into a result
        out = []
        for op in (band, plain):
            Y = torch.full((k, ld + 4), -7.5, device="cuda", dtype=torch.float64)
            _lib.check(L.aqr_op_apply(ctypes.byref(op._native()), k, X.data_ptr(), ld, Y.data_ptr(), ld + 4,
                                      D.stream_ptr()), "aqr_op_apply")
            torch.cuda.synchronize()
            assert bool((Y[:, m:] == -7.5).all()), (name, k, pad)
            assert bool(torch.isfinite(Y[:, :m]).all()), (name, k, pad)
            out.append(Y[:, :m].clone())
        assert torch.equal(out[0], out[1]), (name, k, pad)
