"""BASELINE.json configs at full size on the B200.

Configs 2, 3, 4 and the config-5 operator family are in
test_gpu_fullsize.py.  The rest checks size-independent properties -- R
upper triangular with positive diagonal, col == row bitwise, rerun bitwise
-- and reduced grids of the same operator families.
"""

import numpy as np
import pytest

from oracle import oracle as O

import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aqr():
    import paper_1703_10440_b200 as P

    return P


@pytest.fixture(scope="module")
def cfg2(aqr):
    import torch

    from paper_1703_10440_b200 import problems

    (ip, ix, dv), Z = problems.config2(device=False)
    op = aqr.CsrSpdOperator(ip, ix, dv)
    Zd = torch.from_numpy(Z.T).cuda().t()
    return ip, ix, dv, Z, op, Zd


def test_config2_properties_and_invariants(aqr, cfg2):
    import torch

    ip, ix, dv, Z, op, Zd = cfg2
    a = aqr.factorize(Zd, op, "mgs-ha-row")
    b = aqr.factorize(Zd, op, "mgs-ha-row")
    assert torch.equal(a.Q, b.Q) and torch.equal(a.R, b.R)  # rerun bitwise
    R = a.R.cpu().numpy()
    assert np.array_equal(np.tril(R, -1), np.zeros_like(R)) and np.all(np.diag(R) > 0)
    loss = aqr.loss_of_A_orthogonality(a.Q, op)
    res = aqr.residual_rel(Zd, a.Q, a.R)
    # kappa(A) ~ 800, Z Gaussian: loss ~ u kappa(A) kappa(A^1/2 Z), residual ~ u
    assert loss < 1e-12, loss
    assert res < 1e-15, res
    # col == row bitwise at full m (first 6 columns: the column form is
    # latency-bound, n(n-1)/2 dependent reductions)
    Z6 = Zd[:, :6]
    c = aqr.factorize(Z6, op, "mgs-hp-col")
    r = aqr.factorize(Z6, op, "mgs-hp-row")
    assert torch.equal(c.Q, r.Q) and torch.equal(c.R, r.R)


def test_config3_reduced_grid_parity(aqr):
    """Same operator family on a 24^3 grid, against the oracle."""
    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.diffusion7(24, 1e-3, problems.rng(3, 0))
    m, n = 24 ** 3, 24
    scale = 10.0 ** (-6.0 * np.arange(n) / (n - 1))
    Z = np.asfortranarray(problems.rng(3, 1).standard_normal((n, m)).T * scale)
    op = aqr.CsrSpdOperator(ip, ix, dv)
    for meth in ("mgs-ha-row", "mgs-hp-row", "mgs-naive-row", "cgs-ha-row"):
        r = aqr.factorize(Z, op, meth)
        o = O.gs_factor(Z, ("csr", ip, ix, dv), meth)
        tq, tr = parity.tolerance(Z, ("csr", ip, ix, dv), meth)
        eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
        assert eq <= tq and er <= tr, (meth, eq, tq, er, tr)


def test_dense_gemv_path_parity(aqr):
    """Config-4 operator family (A = B^T B / m + 0.1 I) at m = 4096, n = 48."""
    rng = np.random.default_rng(4)
    m, n = 4096, 48
    B = rng.standard_normal((m, m))
    A = np.asfortranarray(B.T @ B / m + 0.1 * np.eye(m))
    A = np.asfortranarray(0.5 * (A + A.T))
    Z = np.asfortranarray(rng.standard_normal((m, n)))
    op = aqr.DenseSpdOperator(A)
    for meth in ("mgs-ha-row", "mgs-hp-row"):
        r = aqr.factorize(Z, op, meth)
        o = O.gs_factor(Z, ("dense", A), meth)
        tq, tr = parity.tolerance(Z, ("dense", A), meth)
        eq, er = parity.factor_errors(r.Q, r.R, o.Q, o.R)
        assert eq <= tq and er <= tr, (meth, eq, tq, er, tr)


def test_many_columns_invariants(aqr):
    """n = 700 > every per-kernel column batch (TMA staging 256, group sizes):
    col == row bitwise, triangular R, A-orthogonality."""
    import torch

    from paper_1703_10440_b200 import problems

    ip, ix, dv = problems.laplacian5(120, 100, 1e-1)
    m, n = 12000, 700
    op = aqr.CsrSpdOperator(ip, ix, dv)
    Zd = torch.from_numpy(problems.rng(9, 8).standard_normal((n, m))).cuda().t()
    r = aqr.factorize(Zd, op, "mgs-hp-row")
    c = aqr.factorize(Zd, op, "mgs-hp-col")
    assert torch.equal(r.Q, c.Q) and torch.equal(r.R, c.R)
    R = r.R.cpu().numpy()
    assert np.array_equal(np.tril(R, -1), np.zeros_like(R)) and np.all(np.diag(R) > 0)
    assert aqr.loss_of_A_orthogonality(r.Q, op) < 1e-12
    h = aqr.factorize(Zd, op, "mgs-ha-row")
    assert aqr.residual_rel(Zd, h.Q, h.R) < 1e-14
