"""Config-1 input generator (BASELINE.json configs[0]), test infrastructure.

Dense m=1000, n=50: A = U diag(lambda) U^T with U Haar-orthogonal (sign-fixed
QR of a seeded Gaussian) and lambda log-spaced over [1, 1e4], exactly the
recipe of aqr.testbed.build_spd (/root/reference/pkg/src/aqr/testbed.py:77-88);
Z = V diag(sigma) W^T with V (m x n) and W (n x n) orthonormal from seeded
Gaussians and sigma log-spaced over [1, 1e-4] (kappa(Z) = 1e4).

The QR and the products run through the oracle's sequential C kernels
(Householder QR + gemm_nn, oracle/aqr_oracle.c) instead of LAPACK/BLAS, so
the bytes are identical on every host: tests/golden/cfg1.json pins their
SHA-256 together with the reference's own outputs on them.

Seeds: np.random.SeedSequence([1703, 10440, 1, s]), s=0 for A, s=1 for Z
(SURVEY.md section 8d).
"""

import functools
import hashlib

import numpy as np

from oracle import oracle as O

M, N = 1000, 50
KAPPA_A = 1e4
KAPPA_Z = 1e4


def _rng(stream):
    return np.random.default_rng(np.random.SeedSequence([1703, 10440, 1, stream]))


def _haar(rng, m, k):
    while True:
        G = np.asfortranarray(rng.standard_normal((m, k)))
        Q, singular = O.householder_q(G)
        if not singular:
            return Q


@functools.lru_cache(maxsize=None)
def make(m=M, n=N):
    rng = _rng(0)
    V = _haar(rng, m, m)
    alpha = np.log10(KAPPA_A) / (m - 1)
    d = 10.0 ** (alpha * np.arange(m))
    A = O.gemm_nn(np.asfortranarray(V * d), np.asfortranarray(V.T))
    A = np.asfortranarray(0.5 * (A + A.T))
    rz = _rng(1)
    U = _haar(rz, m, n)
    W = _haar(rz, n, n)
    sigma = 10.0 ** (-np.log10(KAPPA_Z) * np.arange(n) / (n - 1))
    Z = O.gemm_nn(np.asfortranarray(U * sigma), np.asfortranarray(W.T))
    A.setflags(write=False)
    Z.setflags(write=False)
    return A, Z


def sha(a):
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()
