"""Accuracy properties and operator KATs the reference's own tests pin,
restated on the B200 path:

* Proposition-1 witness (test_gram_schmidt.py:237-251);
* well-scaled inputs are not flagged (test_gram_schmidt.py:270-272);
* CSR vs dense apply and the Laplacian interior-row KAT
  (test_operators.py:66-80);
* the accuracy envelopes of the acceptance suite, criteria 6, 7 (bound part)
  and 8 (test_acceptance.py:180-237), on a small sweep of our own instances;
* ragged CSR rows (longer than any row batch, empty-ish rows) and ragged m on
  the large-tile path, against the oracle.
"""

import numpy as np
import pytest

from oracle import oracle as O

import parity

pytestmark = pytest.mark.gpu

U = 2.0 ** -53
METHODS_COL_ROW = ["mgs-naive-col", "mgs-ha-col", "mgs-hp-col", "mgs-naive-row", "mgs-ha-row", "mgs-hp-row"]


@pytest.fixture(scope="module")
def aqr():
    import paper_1703_10440_b200 as P

    return P


def _haar(rng, n):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))


def _instance(seed, m, n, kappa_a, kappa_z):
    """A = V diag(l) V^T (log-spaced spectrum in [1, kappa_a]); Z = A^(-1/2) Y
    with kappa(Y) = kappa_z, so kappa(A^(1/2) Z) = kappa_z."""
    rng = np.random.default_rng(np.random.SeedSequence([1703, 10440, 90, seed]))
    V = _haar(rng, m)
    lam = 10.0 ** np.linspace(0.0, np.log10(kappa_a), m)
    A = (V * lam) @ V.T
    A = np.asfortranarray(0.5 * (A + A.T))
    Uy = _haar(rng, m)[:, :n]
    W = _haar(rng, n)
    Y = (Uy * 10.0 ** -np.linspace(0.0, np.log10(kappa_z), n)) @ W.T
    Z = np.asfortranarray((V * lam ** -0.5) @ (V.T @ Y))
    return A, Z


def test_proposition_witness(aqr):
    """Every computed r_ij equals an inner product between a reconstructed
    member of range(Z) and a fresh member of range(AZ), rel 1e-12."""
    A, Z = _instance(1, 20, 6, 1e2, 1e2)
    op = aqr.DenseSpdOperator(A)
    r = aqr.mgs_ha(Z, op)
    Q, R = r.Q, r.R
    for j in range(6):
        for i in range(j):
            zj = Z[:, j].copy()
            for k in range(i):
                zj -= R[k, j] * Q[:, k]
            witness = float(np.dot(A @ Q[:, i], zj))
            assert R[i, j] == pytest.approx(witness, rel=1e-12, abs=1e-12)


def test_well_scaled_not_flagged(aqr):
    A, Z = _instance(2, 16, 5, 10.0, 10.0)
    op = aqr.DenseSpdOperator(A)
    for meth in METHODS_COL_ROW:
        assert aqr.factorize(Z, op, meth).flagged_columns == [], meth


def test_csr_matches_dense_and_laplacian_kat(aqr):
    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.laplacian5(3, 3, 0.0)
    op = aqr.CsrSpdOperator(ip, ix, dv)
    dense = aqr.DenseSpdOperator(op.to_dense())
    x = np.random.default_rng(5).standard_normal(9)
    got, ref = op.apply(x), dense.apply(x)
    scale = np.abs(dense.matrix).max() * np.abs(x).max()
    assert np.max(np.abs(got - ref)) <= 1e-13 * scale
    y = op.apply(np.ones(9))
    assert y[4] == 0.0  # interior point: 4 - 4 neighbours
    assert np.all(y[[0, 2, 6, 8]] == 2.0)  # corners keep two boundary links


def test_accuracy_envelopes(aqr):
    """Criteria 6 (loss <= 10 m^1.5 delta1, MGS variants), 7 (HA loss <=
    10 m^1.5 delta2) and 8 (normalized representation error <= 100 n^1.5 u)
    over a kappa(A) x kappa(A^1/2 Z) grid; breakdowns are recorded, not
    errors (the reference's sweep does the same)."""
    m, n = 160, 12
    worst6 = worst7 = worst8 = 0.0
    rows = 0
    for s, (ka, kz) in enumerate([(1e2, 1e2), (1e4, 1e2), (1e2, 1e6), (1e6, 1e4), (1e8, 1e3), (1e10, 1e2)]):
        A, Z = _instance(10 + s, m, n, ka, kz)
        op = aqr.DenseSpdOperator(A)
        d1, d2 = aqr.delta_bounds(ka, kz)
        for meth in METHODS_COL_ROW:
            try:
                r = aqr.factorize(Z, op, meth)
            except aqr.BreakdownError:
                continue
            rows += 1
            loss = aqr.loss_of_A_orthogonality(r.Q, op)
            rep = aqr.representation_error(Z, r.Q, r.R)[1]
            worst8 = max(worst8, rep / (100 * n ** 1.5 * U))
            if d1 < 1e-2:
                worst6 = max(worst6, loss / (10 * m ** 1.5 * d1))
            if "-ha-" in meth and d2 < 1e-2:
                worst7 = max(worst7, loss / (10 * m ** 1.5 * d2))
    assert rows >= 30
    assert worst6 <= 1.0, worst6
    assert worst7 <= 1.0, worst7
    assert worst8 <= 1.0, worst8


def _ragged_spd_csr(m, seed):
    """Symmetric diagonally dominant CSR with row lengths from 1 to ~40."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    linked = np.array([i for i in range(m) if i % 7])  # rows i % 7 == 0 keep only the diagonal
    for i in linked:
        k = int(rng.integers(0, 20))
        nb = rng.choice(linked, size=k, replace=False)
        for j in nb:
            if j != i:
                rows += [i, j]
                cols += [j, i]
    vals = -rng.uniform(0.1, 1.0, len(rows))
    Aoff = {}
    for i, j, v in zip(rows, cols, vals):
        key = (min(i, j), max(i, j))
        Aoff.setdefault(key, v)
    ent = {}
    for (i, j), v in Aoff.items():
        ent[(i, j)] = v
        ent[(j, i)] = v
    diag = np.ones(m)
    for (i, j), v in ent.items():
        diag[i] += abs(v)
    for i in range(m):
        ent[(i, i)] = diag[i]
    keys = sorted(ent)
    indptr = np.zeros(m + 1, dtype=np.int64)
    for i, _ in keys:
        indptr[i + 1] += 1
    indptr = np.cumsum(indptr)
    indices = np.array([j for _, j in keys], dtype=np.int64)
    data = np.array([ent[k] for k in keys])
    return indptr, indices, data


def test_ragged_csr_rows_against_oracle(aqr):
    ip, ix, dv = _ragged_spd_csr(3000, 7)
    lens = np.diff(ip)
    assert lens.min() == 1 and lens.max() > 16
    m, n = 3000, 10
    Z = np.asfortranarray(np.random.default_rng(8).standard_normal((m, n)))
    for hint in (None, 0, 5):
        op = aqr.CsrSpdOperator(ip, ix, dv, max_row_nnz=hint)
        for meth in ("mgs-ha-row", "mgs-hp-row", "mgs-naive-row", "mgs-ha-col"):
            r = aqr.factorize(Z, op, meth)
            o = O.gs_factor(Z, ("csr", ip, ix, dv), meth)
            tq, tr = parity.tolerance(Z, ("csr", ip, ix, dv), meth)
            eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
            assert eq <= tq and er <= tr, (hint, meth, eq, tq, er, tr)


def test_ragged_m_large_tiles_against_oracle(aqr):
    """m just above the 2048-row-tile threshold and not a multiple of it."""
    from paper_1703_10440_b200 import problems

    nx, ny = 777, 391  # m = 303,807 = 148 * 2048 + 703
    ip, ix, dv = problems.laplacian5(nx, ny, 1e-2)
    m, n = nx * ny, 6
    Z = np.asfortranarray(problems.rng(9, 3).standard_normal((n, m)).T)
    op = aqr.CsrSpdOperator(ip, ix, dv)
    for meth in ("mgs-ha-row", "mgs-hp-row"):
        r = aqr.factorize(Z, op, meth)
        o = O.gs_factor(Z, ("csr", ip, ix, dv), meth)
        tq, tr = parity.tolerance(Z, ("csr", ip, ix, dv), meth)
        eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
        assert eq <= tq and er <= tr, (meth, eq, tq, er, tr)


def test_long_row_block_apply_bitwise(aqr):
    """SpMM for rows longer than every row batch (csr_spmm2_kernel): each
    output column bitwise the reference's csr_matvec (_kernels_impl.py:50-56)."""
    ip, ix, dv = _ragged_spd_csr(2000, 11)
    X = np.asfortranarray(np.random.default_rng(12).standard_normal((2000, 13)))
    for hint in (None, 0):
        op = aqr.CsrSpdOperator(ip, ix, dv, max_row_nnz=hint)
        Y = op.apply_block(X)
        for c in range(X.shape[1]):
            assert np.array_equal(Y[:, c], O.csr_matvec(ip, ix, dv, X[:, c])), (hint, c)


EDGE_METHODS = [f"{f}-{v}-{o}" for f in ("mgs", "cgs") for v in ("naive", "ha", "hp") for o in ("col", "row")]


def _tridiag_csr(m):
    """1-D Laplacian + I (diag 3, off -1), sorted columns."""
    rows, cols, vals = [], [], []
    for i in range(m):
        for j, v in ((i - 1, -1.0), (i, 3.0), (i + 1, -1.0)):
            if 0 <= j < m:
                rows.append(i), cols.append(j), vals.append(v)
    from paper_1703_10440_b200 import csr_from_coo

    op = csr_from_coo(m, np.array(rows), np.array(cols), np.array(vals))
    return op.indptr, op.indices, op.data


@pytest.mark.parametrize("m,n", [(1, 1), (2, 1), (2, 2), (7, 7), (255, 3), (256, 1), (257, 5),
                                 (300, 300), (1025, 17), (2049, 2)])
def test_edge_shapes_all_methods_against_oracle(aqr, m, n):
    """Single columns, square Z, m at and around the 256-row block and the
    tile sizes, for all 12 methods with a dense and a CSR operator."""
    rng = np.random.default_rng(np.random.SeedSequence([1703, 10440, 91, m, n]))
    B = rng.standard_normal((m, m))
    A = np.asfortranarray(B @ B.T / m + np.eye(m))
    Z = np.asfortranarray(rng.standard_normal((m, n)))
    ip, ix, dv = _tridiag_csr(m)
    import torch

    Zd = torch.from_numpy(np.ascontiguousarray(Z.T)).cuda().t()
    for spec, op in ((("dense", A), aqr.DenseSpdOperator(A)), (("csr", ip, ix, dv), aqr.CsrSpdOperator(ip, ix, dv))):
        for meth in EDGE_METHODS:
            r = aqr.factorize(Z, op, meth)
            o = O.gs_factor(Z, spec, meth)
            tq, tr = parity.tolerance(Z, spec, meth)
            eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
            assert eq <= tq and er <= tr, (spec[0], meth, eq, tq, er, tr)
            assert np.array_equal(np.tril(r.R, -1), np.zeros((n, n)))
            assert r.flagged_columns == o.flagged_columns, (spec[0], meth)
            rd = aqr.factorize(Zd, op, meth)  # device input: bitwise the host-input pipeline
            assert np.array_equal(rd.Q.cpu().numpy(), r.Q) and np.array_equal(rd.R.cpu().numpy(), r.R)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_input_breaks_down_like_the_oracle(aqr, bad):
    """A non-finite entry in column 4 makes z'Az non-finite there: the same
    BreakdownError column as the oracle (gram_schmidt.py:153-154), with a
    non-finite value, for all 12 methods, host and device input."""
    import math

    import torch

    m, n = 600, 7
    rng = np.random.default_rng(np.random.SeedSequence([1703, 10440, 92]))
    B = rng.standard_normal((m, m))
    A = np.asfortranarray(B @ B.T / m + np.eye(m))
    Z = np.asfortranarray(rng.standard_normal((m, n)))
    Z[123, 4] = bad
    for meth in EDGE_METHODS:
        with pytest.raises(O.OracleBreakdown) as oinfo:
            O.gs_factor(Z, ("dense", A), meth)
        for Zin in (Z, torch.from_numpy(np.ascontiguousarray(Z.T)).cuda().t()):
            with pytest.raises(aqr.BreakdownError) as info:
                aqr.factorize(Zin, aqr.DenseSpdOperator(A), meth)
            assert info.value.column == oinfo.value.column == 4, meth
            assert not math.isfinite(info.value.value), meth
