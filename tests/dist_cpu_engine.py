"""numpy step engine and local operator products for the gloo tests.

TEST INFRASTRUCTURE: lets paper_1703_10440_b200.distributed.dist_factorize
(the product driver: partitioning, halo exchange, all-reduce points, R
assembly) run on CPU ranks.  The per-rank arithmetic follows the reference's
elementwise order (gram_schmidt.py:139-165) with sequential local dots
(oracle seq_dot), so a world_size-1 run is bitwise the oracle and a
world_size-2 run differs only by the cross-rank summation of the dots.
"""

import numpy as np
import torch

from oracle import oracle as O

U = 2.0 ** -53


def local_csr_apply(op, ext, k):
    """Local product of a DistCsrSpdOperator block on [own | halo] values."""
    ext = ext.numpy()
    out = np.empty((op.dim, k), order="F")
    for c in range(k):
        out[:, c] = O.csr_matvec(op.indptr, op.indices_local, op.data, np.ascontiguousarray(ext[:, c]))
    return torch.from_numpy(out)


def local_dense_apply(op, full, k):
    full = full.numpy()
    out = np.empty((op.dim, k), order="F")
    A = np.asfortranarray(op.A_rows)
    for c in range(k):
        out[:, c] = O.matvec(A, np.ascontiguousarray(full[:, c]))
    return torch.from_numpy(out)


class CpuStepEngine:
    def __init__(self, m, n, family, variant):
        self.m, self.n, self.family, self.variant = m, n, family, variant
        self.W = np.zeros((m, n), order="F")
        self.X = np.zeros((m, n), order="F") if variant == "hp" else None
        self.Z0 = None
        self.x = np.zeros(m)
        self.p = np.zeros(m)
        self.pring = np.zeros((2, m))
        self.Rt = np.zeros((n, n))
        self.flags = np.zeros(n, dtype=np.int32)
        self.fail, self.fail_val = -1, 0.0
        self.tot = torch.zeros(3, dtype=torch.float64)

    def load(self, Z):
        self.W[:] = Z.numpy() if hasattr(Z, "numpy") else Z
        if self.family == "cgs":
            self.Z0 = self.W.copy(order="F")

    def z(self, i):
        return torch.from_numpy(np.ascontiguousarray(self.W[:, i]))

    def q(self, i):
        return self.z(i)

    def w_block(self):
        return torch.from_numpy(self.W)

    def set_X(self, X):
        self.X[:] = X.numpy()

    def set_x(self, x):
        self.x[:] = x.numpy()

    def set_p(self, p):
        self.p[:] = p.numpy()

    def col_update(self, i):
        if i == 0 or self.fail >= 0:
            return
        r = self.Rt[i - 1, i]
        self.W[:, i] -= r * self.W[:, i - 1]
        if self.variant == "hp":
            self.X[:, i] -= r * self.pring[(i - 1) & 1]

    def _xcol(self, i):
        return self.X[:, i] if self.variant == "hp" else self.x

    def norm_partials(self, i):
        z, x = np.ascontiguousarray(self.W[:, i]), np.ascontiguousarray(self._xcol(i))
        self.tot[:] = torch.tensor([O.seq_dot(z, x), O.seq_dot(z, z), O.seq_dot(x, x)], dtype=torch.float64)
        return self.tot

    def norm_finish(self, i, tot):
        t, zz, xx = (float(v) for v in tot)
        if self.fail >= 0:
            return
        if not (t > 0.0) or not np.isfinite(t):
            self.fail, self.fail_val = i, t
            return
        if t < 100.0 * U * np.sqrt(zz) * np.sqrt(xx):
            self.flags[i] = 1
        self.Rt[i, i] = np.sqrt(t)

    def normalize_q(self, i):
        self.W[:, i] = self.W[:, i] / self.Rt[i, i]

    def trailing(self, i):
        n = self.n
        if self.fail < 0:
            rii = self.Rt[i, i]
            if self.variant == "naive":
                p = self.p.copy()
            else:
                p = self._xcol(i) / rii
                self.W[:, i] = self.W[:, i] / rii
            if self.variant == "hp":
                self.pring[i & 1] = p
            for j in range(i + 1, n):
                if i > 0:
                    r = self.Rt[i - 1, j]
                    self.W[:, j] -= r * self.W[:, i - 1]
                    if self.variant == "hp":
                        self.X[:, j] -= r * self.pring[(i - 1) & 1]
                src = self.Z0[:, j] if self.family == "cgs" else self.W[:, j]
                self.Rt[i, j] = O.seq_dot(p, np.ascontiguousarray(src))
        view = torch.from_numpy(self.Rt[i, i + 1:])
        return view

    def finish(self):
        R = np.triu(self.Rt)
        return (torch.from_numpy(self.W), torch.from_numpy(np.asfortranarray(R)), self.fail,
                self.fail_val, [int(j) for j in np.flatnonzero(self.flags)])
