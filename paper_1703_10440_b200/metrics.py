"""Accuracy metrics on the device.

Same definitions and operation order as /root/reference/pkg/src/aqr/
metrics.py:35-53:

* ``loss_of_A_orthogonality(Q, op)`` = || sym(Q^T A Q) - I ||_2 with A Q
  formed by ``op.apply_block`` (so, like the reference, it adds n to
  ``op.mv_count``, metrics.py:40) and Q^T (A Q) by ``linalg.matmul_tn``;
* ``representation_error(Z, Q, R)`` = (||Z - QR||_2, that over
  ||Z||_2 + ||Q||_2 ||R||_2), Q R by ``linalg.matmul``;
* ``residual_rel(Z, Q, R)`` = ||Z - QR||_2 / ||Z||_2 (the north-star form).

The products run in the repo's kernels in the reference's per-entry order
(sequential sums, separately rounded), so for bitwise-equal Q, R the
matrices whose norms are taken are bitwise the reference's.  The reference
then takes eigen/singular values by sequential Jacobi sweeps (linalg.py:
89-188, impractical at m in the millions); here the n x n symmetric eigen
problem runs in cuSOLVER (``torch.linalg.eigvalsh``) and the spectral norm
of a tall m x n matrix is sqrt(lambda_max(M^T M)) with the Gram product in
the same sequential kernel -- both accurate to a few units of roundoff
relative to the value, which the tests pin against the reference's own
numbers (tests/test_gpu_accuracy.py, cases.json).
"""

import numpy as np

from . import _device as D
from . import linalg
from .exceptions import DimensionError
from .operators import as_matrix


def _dev(a):
    T, _ = D.to_device_f(as_matrix(a))
    return T


def two_norm(M):
    """Spectral norm (largest singular value) of a device matrix via its Gram matrix."""
    t = D.torch()
    M = _dev(M)
    if M.shape[0] < M.shape[1]:
        M = M.t()
    if M.shape[0] == 0 or M.shape[1] == 0:
        return 0.0
    G = linalg.matmul_tn(M, M)
    w = t.linalg.eigvalsh(0.5 * (G + G.transpose(0, 1)))
    return float(t.sqrt(t.clamp(w[-1], min=0.0)))


def loss_of_A_orthogonality(Q, op):
    """Spectral norm of Q^T A Q - I (symmetrized before the eigensolve)."""
    t = D.torch()
    Qd = _dev(Q)
    if Qd.shape[0] != op.dim:
        raise DimensionError(f"Q has {Qd.shape[0]} rows, operator dimension is {op.dim}")
    AQ = t.as_tensor(op.apply_block(Qd), device=Qd.device)
    S = linalg.matmul_tn(Qd, AQ)
    del AQ
    M = 0.5 * (S + S.transpose(0, 1)) - t.eye(S.shape[0], dtype=S.dtype, device=S.device)
    w = t.linalg.eigvalsh(M)
    return float(w.abs().max())


def _residual(Z, Q, R):
    Zd, Qd, Rd = _dev(Z), _dev(Q), _dev(R)
    if Qd.shape != Zd.shape or tuple(Rd.shape) != (Zd.shape[1], Zd.shape[1]):
        raise DimensionError("shapes of Z, Q, R do not conform")
    E = linalg.matmul(Qd, Rd)
    E = Zd - E  # Z - Q R, elementwise as numpy
    return Zd, Qd, Rd, E


def representation_error(Z, Q, R):
    """Returns (||Z - Q R||_2, same normalized by ||Z|| + ||Q|| ||R||)."""
    Zd, Qd, Rd, E = _residual(Z, Q, R)
    absolute = two_norm(E)
    del E
    scale = two_norm(Zd) + two_norm(Qd) * two_norm(Rd)
    return absolute, absolute / scale


def residual_rel(Z, Q, R):
    """||Z - Q R||_2 / ||Z||_2."""
    Zd, _, _, E = _residual(Z, Q, R)
    absolute = two_norm(E)
    del E
    return absolute / two_norm(Zd)


def delta_bounds(kappa_A, kappa_AhalfZ):
    """(delta1, delta2) = (u kA kAZ, u (kA + kAZ)) for u = 2^-53 (metrics.py:73-80)."""
    if kappa_A < 1.0 or kappa_AhalfZ < 1.0:
        raise ValueError("condition numbers are >= 1 by definition")
    u = 2.0 ** -53
    return u * kappa_A * kappa_AhalfZ, u * (kappa_A + kappa_AhalfZ)


def relative_factor_error(Q, R, Qref, Rref, floor=1e-3):
    """Max elementwise relative differences of (Q, R) against references.

    Q entries use a column-norm floor, |dQ_ij| / max(|Qref_ij|, floor *
    max_i |Qref_ij|); R uses max|dR| / max|Rref| per
    row-scaled entry.  Returns (q_err, r_err) as floats.
    """
    Q, R, Qref, Rref = (np.asarray(a.cpu() if D.is_torch(a) else a) for a in (Q, R, Qref, Rref))
    colmax = np.abs(Qref).max(axis=0, keepdims=True)
    qden = np.maximum(np.abs(Qref), floor * colmax)
    q_err = float(np.max(np.abs(Q - Qref) / np.where(qden > 0, qden, 1.0)))
    r_err = float(np.max(np.abs(R - Rref)) / max(np.max(np.abs(Rref)), np.finfo(float).tiny))
    return q_err, r_err
