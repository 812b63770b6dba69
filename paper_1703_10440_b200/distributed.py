"""Row-partitioned multi-GPU A-orthogonal MGS.

One process per GPU (``torch.distributed``: NCCL over NVLink / NVSwitch on
the GPU box, gloo for the CPU tests).  The rows of Z, Q, A Z and of the
operator are block-partitioned across ranks; the n x n factor R is
replicated.  The reference is single-process (gram_schmidt.py:126-179); the
distributed schedule is its row-oriented loop (lines 172-176) with every
reduction split into a local part and one all-reduce:

  step i  1. deferred projection of column i (local rows)
          2. x_i = A z_i  (HA/naive): ``DistCsrSpdOperator.apply`` = halo
             exchange (point-to-point send/recv of exactly the boundary rows
             each neighbour's stencil touches) + local SpMV over [own | halo]
             values in the reference's in-row order, so the product is
             bitwise the global one; ``DistDenseSpdOperator`` all-gathers z_i
          3. local (z.x, z.z, x.x) -> all_reduce(SUM) -> r_ii, breakdown/flag
          4. naive: q_i = z_i / r_ii, p_i = A q_i (second distributed apply)
          5. fused trailing pass -> local R[i, i+1:] -> all_reduce(SUM)

Two all-reduces per step (3 doubles and n-1-i doubles): latency-bound
messages.  The per-rank compute goes through a *step engine*: the product
engine (``CudaStepEngine``) calls the step entry points of libaqr_b200.so
(include/aqr_b200.h, ``aqr_step_*``); the CPU tests plug in a numpy engine
(tests/dist_cpu_engine.py) to exercise this driver, the partitioning and the
halo exchange under gloo with world_size 2.  With one rank the CUDA engine
is bitwise identical to the single-GPU ``factorize``.
"""

import bisect
import ctypes

import numpy as np

from . import _device as D
from . import _lib
from .exceptions import BreakdownError, DimensionError
from .gram_schmidt import MethodId, QrResult, _model_flops
from .operators import CostReport, SpdOperator


def _dist():
    import torch.distributed as dist

    return dist


def row_partition(m, world, align=1):
    """Contiguous row blocks [(r0, r1)] for ranks 0..world-1.

    Boundaries are multiples of ``align`` (e.g. one grid plane for a stencil
    operator) as far as possible; the last block takes the remainder.
    """
    if world < 1 or m < world:
        raise DimensionError(f"cannot split {m} rows over {world} ranks")
    units = (m + align - 1) // align
    bounds = [min(m, (units * r // world) * align) for r in range(world + 1)]
    bounds[-1] = m
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _halo_need(indices, r0, r1, owner):
    """{owner rank: ascending global columns outside [r0, r1) that the block reads}."""
    ext = np.unique(indices[(indices < r0) | (indices >= r1)])
    need = {}
    for c in ext.tolist():
        need.setdefault(owner(c), []).append(c)
    return need


class DistCsrSpdOperator(SpdOperator):
    """The local row block of a row-partitioned CSR operator.

    ``indptr`` (local, starting at 0), ``indices`` (GLOBAL column indices)
    and ``data`` describe rows [r0, r1) of the global m x m matrix; every
    rank passes its own block and the shared ``partition``.  Construction is
    collective (the halo plan is exchanged once).  ``apply`` / ``apply_block``
    take and return LOCAL vectors / blocks (``dim`` = local rows) and are
    collective too.  ``local_apply(op_arrays, X_ext, k)`` overrides the local
    product (tests on CPU); by default the sm_100a CSR kernel runs it.
    """

    def __init__(self, indptr, indices, data, partition, rank, group=None, local_apply=None,
                 device=None, needs=None):
        self.partition = [tuple(p) for p in partition]
        self.rank = rank
        self.group = group
        r0, r1 = self.partition[rank]
        m_loc = r1 - r0
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        indices = np.ascontiguousarray(indices, dtype=np.int64)
        data = np.ascontiguousarray(data, dtype=np.float64)
        if indptr.shape[0] != m_loc + 1 or indptr[0] != 0 or indptr[-1] != data.shape[0]:
            raise DimensionError("local CSR block does not match the partition")
        super().__init__(m_loc)
        self.global_dim = self.partition[-1][1]
        self.row_offset = r0
        self.local_apply = local_apply
        self.device = device
        starts = [p[0] for p in self.partition]

        def owner(c):
            return bisect.bisect_right(starts, c) - 1

        need = _halo_need(indices, r0, r1, owner)
        world = len(self.partition)
        if needs is None:
            # every rank learns who needs which of its rows (one collective, once)
            gathered = [None] * world
            _dist().all_gather_object(gathered, need, group=group)
        else:  # every rank's halo plan given (single-process emulation, blocks_of)
            gathered = list(needs)
        self.send = {}  # peer -> local row offsets to send
        for peer in range(world):
            if peer == rank:
                continue
            rows = gathered[peer].get(rank, [])
            if rows:
                self.send[peer] = np.asarray(rows, dtype=np.int64) - r0
        self.recv = {p: len(c) for p, c in sorted(need.items())}  # peer -> count
        # halo slots: peers ascending, columns ascending within a peer
        slot = {}
        pos = m_loc
        for p in sorted(need):
            for c in need[p]:
                slot[c] = pos
                pos += 1
        self.n_ext = pos
        # halo slot h (column m_loc + h) = local row halo_row[h] of rank halo_rank[h]
        self.halo_rank = np.fromiter((p for p in sorted(need) for _ in need[p]), dtype=np.int32,
                                     count=pos - m_loc)
        self.halo_row = np.fromiter((c - self.partition[p][0] for p in sorted(need) for c in need[p]),
                                    dtype=np.int32, count=pos - m_loc)
        local = indices - r0
        outside = (indices < r0) | (indices >= r1)
        if outside.any():
            local[outside] = np.fromiter((slot[c] for c in indices[outside].tolist()),
                                         dtype=np.int64, count=int(outside.sum()))
        if data.shape[0] >= 2**31 or self.n_ext >= 2**31:
            raise ValueError("local block too large for the int32 device CSR layout")
        self.indptr, self.indices_local, self.data = indptr, local, data
        self._dev = None
        self._desc = None

    @classmethod
    def blocks_of(cls, indptr, indices, data, partition):
        """Every rank's block of a global CSR matrix, built in one process
        without a process group (the single-device lock-step emulation,
        p2p.p2p_factorize_lockstep)."""
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        starts = [p[0] for p in partition]

        def owner(c):
            return bisect.bisect_right(starts, c) - 1

        needs = [_halo_need(indices[indptr[r0]:indptr[r1]], r0, r1, owner) for r0, r1 in partition]
        return [cls(indptr[r0:r1 + 1] - indptr[r0], indices[indptr[r0]:indptr[r1]], data[indptr[r0]:indptr[r1]],
                    partition, rank, needs=needs) for rank, (r0, r1) in enumerate(partition)]

    @property
    def nnz(self):
        return int(self.data.shape[0])

    # -- halo exchange -------------------------------------------------------
    def _exchange(self, X):
        """Return [X; halo rows] for a local block X (m_loc x k, column-major)."""
        t = D.torch()
        dist = _dist()
        k = X.shape[1]
        ext = t.empty((k, self.n_ext), dtype=X.dtype, device=X.device).t()
        ext[: self.dim].copy_(X)
        ops, recv_bufs = [], []
        for peer, rows in sorted(self.send.items()):
            idx = t.as_tensor(rows, device=X.device)
            buf = X.index_select(0, idx).t().contiguous()
            ops.append(dist.P2POp(dist.isend, buf, peer, group=self.group))
            recv_bufs.append(buf)  # keep alive
        halos = []
        for peer, cnt in sorted(self.recv.items()):
            buf = t.empty((k, cnt), dtype=X.dtype, device=X.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer, group=self.group))
            halos.append(buf)
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        pos = self.dim
        for buf in halos:
            ext[pos: pos + buf.shape[1]].copy_(buf.t())
            pos += buf.shape[1]
        return ext

    def _native(self):
        if self.local_apply is not None:
            return None
        if self._desc is None:
            t = D.torch()
            dev = self.device or D.device()
            self._dev = (t.from_numpy(self.indptr.astype(np.int32)).to(dev),
                         t.from_numpy(self.indices_local.astype(np.int32)).to(dev),
                         t.from_numpy(self.data).to(dev))
            d = _lib.AqrOp()
            d.kind = _lib.AQR_OP_CSR
            d.m = self.dim
            d.indptr, d.indices, d.data = (a.data_ptr() for a in self._dev)
            d.nnz = self.nnz
            d.max_row_nnz = int(np.diff(self.indptr).max()) if self.dim else 0
            self._desc = d
        return self._desc

    def _local_product(self, ext, k):
        t = D.torch()
        if self.local_apply is not None:
            return self.local_apply(self, ext, k)
        Y = D.empty_f(self.dim, k, ext.device)
        _lib.check(_lib.lib().aqr_op_apply(ctypes.byref(self._native()), k, ext.data_ptr(),
                                           self.n_ext, Y.data_ptr(), self.dim, D.stream_ptr()),
                   "aqr_op_apply")
        del t
        return Y

    def apply(self, x):
        X = x.reshape(-1, 1)
        if X.shape[0] != self.dim:
            raise DimensionError(f"expected a local vector of length {self.dim}")
        y = self._local_product(self._exchange(X), 1)
        self.mv_count += 1
        return y.reshape(-1)

    def apply_block(self, X):
        if X.shape[0] != self.dim:
            raise DimensionError(f"block has {X.shape[0]} rows, local dimension is {self.dim}")
        Y = self._local_product(self._exchange(X), X.shape[1])
        self.mv_count += X.shape[1]
        return Y


class DistDenseSpdOperator(SpdOperator):
    """Local row panel (m_loc x m, column-major) of a row-partitioned dense A.

    ``apply`` all-gathers the vector (every rank needs all of it) and runs the
    local rectangular GEMV in the reference's column order (bitwise the
    global product for these rows).
    """

    def __init__(self, A_rows, partition, rank, group=None, local_apply=None):
        self.partition = [tuple(p) for p in partition]
        self.rank = rank
        self.group = group
        r0, r1 = self.partition[rank]
        self.global_dim = self.partition[-1][1]
        if tuple(A_rows.shape) != (r1 - r0, self.global_dim):
            raise DimensionError("row panel does not match the partition")
        super().__init__(r1 - r0)
        self.row_offset = r0
        self.local_apply = local_apply
        self.A_rows = A_rows
        self._desc = None

    def _gather(self, X):
        t = D.torch()
        dist = _dist()
        k = X.shape[1]
        width = max(r1 - r0 for r0, r1 in self.partition)
        pad = t.zeros((k, width), dtype=X.dtype, device=X.device)
        pad[:, : self.dim].copy_(X.t())
        parts = [t.empty_like(pad) for _ in self.partition]
        dist.all_gather(parts, pad, group=self.group)
        full = t.empty((k, self.global_dim), dtype=X.dtype, device=X.device).t()
        for (r0, r1), part in zip(self.partition, parts):
            full[r0:r1].copy_(part[:, : r1 - r0].t())
        return full

    def _native(self):
        if self.local_apply is not None:
            return None
        if self._desc is None:
            A, lda = D.to_device_f(self.A_rows)
            self._A = A
            d = _lib.AqrOp()
            d.kind = _lib.AQR_OP_DENSE
            d.m = self.dim
            d.A = A.data_ptr()
            d.lda = lda
            d.ncols = self.global_dim
            self._desc = d
        return self._desc

    def _local_product(self, full, k):
        if self.local_apply is not None:
            return self.local_apply(self, full, k)
        Y = D.empty_f(self.dim, k, full.device)
        # k > 1: the HP block apply (FP64 tensor cores); k = 1: the bitwise GEMV
        fn = "aqr_block_apply" if k > 1 else "aqr_op_apply"
        _lib.check(getattr(_lib.lib(), fn)(ctypes.byref(self._native()), k, full.data_ptr(),
                                           self.global_dim, Y.data_ptr(), self.dim,
                                           D.stream_ptr()), fn)
        return Y

    def apply(self, x):
        y = self._local_product(self._gather(x.reshape(-1, 1)), 1)
        self.mv_count += 1
        return y.reshape(-1)

    def apply_block(self, X):
        Y = self._local_product(self._gather(X), X.shape[1])
        self.mv_count += X.shape[1]
        return Y


class CudaStepEngine:
    """Per-rank state and kernels of one distributed factorization (libaqr_b200.so step API)."""

    def __init__(self, m, n, family, variant, device):
        t = D.torch()
        self.L = _lib.lib()
        self.m, self.n, self.family, self.variant = m, n, family, variant
        self.dev = device
        f64 = dict(dtype=t.float64, device=device)
        self.W = D.empty_f(m, n, device)
        self.X = D.empty_f(m, n, device) if variant == "hp" else None
        self.Z0 = D.empty_f(m, n, device) if family == "cgs" else None
        self.xvec = t.empty(m, **f64)
        self.pvec = t.empty(m, **f64)
        self.pring = t.empty((2, m), **f64)
        self.Rt = t.zeros((n, n), **f64)
        nt = max(int(self.L.aqr_num_tiles(m)), 1)
        self.partial = t.empty(n * nt, **f64)
        self.npart = t.empty(3 * max((m + 255) // 256, 1), **f64)
        self.tot = t.empty(3, **f64)
        self.status = t.empty(int(self.L.aqr_status_bytes(n)) // 4 + 1, dtype=t.int32, device=device)
        self._chk(self.L.aqr_status_init(self.status.data_ptr(), n, D.stream_ptr()), "status_init")

    def _chk(self, st, what):
        _lib.check(st, what)

    def _col(self, B, j):
        return B.data_ptr() + 8 * j * self.m

    def _rt(self, i, j):
        return self.Rt.data_ptr() + 8 * (i * self.n + j)

    def load(self, Z):
        self.W.copy_(Z)
        if self.Z0 is not None:
            self.Z0.copy_(Z)

    def z(self, i):
        return self.W[:, i]

    def w_block(self):
        return self.W

    def set_X(self, X):
        self.X.copy_(X)

    def set_x(self, x):
        self.xvec.copy_(x)

    def set_p(self, p):
        self.pvec.copy_(p)

    def col_update(self, i):
        if i == 0:
            return
        hp = self.variant == "hp"
        self._chk(self.L.aqr_step_col_update_norm(
            self.m, self._col(self.W, i), self._col(self.W, i - 1),
            self._col(self.X, i) if hp else None,
            self.pring[(i - 1) & 1].data_ptr() if hp else None,
            self._rt(i - 1, i), None, None, self.status.data_ptr(), D.stream_ptr()), "col_update")

    def norm_partials(self, i):
        hp = self.variant == "hp"
        self._chk(self.L.aqr_step_col_update_norm(
            self.m, self._col(self.W, i), None, self._col(self.X, i) if hp else None, None, None,
            None if hp else self.xvec.data_ptr(), self.npart.data_ptr(), self.status.data_ptr(),
            D.stream_ptr()), "norm_partials")
        self._chk(self.L.aqr_step_norm_reduce(self.m, _lib.VARIANT_CODE[self.variant], self.npart.data_ptr(),
                                              self.tot.data_ptr(),
                                              self.status.data_ptr(), D.stream_ptr()), "norm_reduce")
        return self.tot

    def norm_finish(self, i, tot):
        self._chk(self.L.aqr_step_norm_finish(i, tot.data_ptr(), self._rt(i, i), self.status.data_ptr(),
                                              D.stream_ptr()), "norm_finish")

    def normalize_q(self, i):
        self._chk(self.L.aqr_step_normalize(self.m, self._col(self.W, i), self._rt(i, i),
                                            self._col(self.W, i), None, None, self.status.data_ptr(),
                                            D.stream_ptr()), "normalize")

    def q(self, i):
        return self.W[:, i]

    def trailing(self, i):
        n, m = self.n, self.m
        hp, naive = self.variant == "hp", self.variant == "naive"
        upd = i > 0
        self._chk(self.L.aqr_step_trailing(
            m, i, i + 1, n, self.W.data_ptr(), m,
            self.X.data_ptr() if hp else None, m,
            self.Z0.data_ptr() if self.Z0 is not None else None, m,
            self._col(self.W, i - 1) if upd else None,
            self.pring[(i - 1) & 1].data_ptr() if (hp and upd) else None,
            self._rt(i - 1, 0) if upd else None,
            self.pvec.data_ptr() if naive else (self._col(self.X, i) if hp else self.xvec.data_ptr()),
            None if naive else self._rt(i, i),
            self.pring[i & 1].data_ptr() if hp else None,
            self._col(self.W, i), None if naive else self._col(self.W, i),
            self.partial.data_ptr(), self.status.data_ptr(), D.stream_ptr()), "trailing")
        cnt = n - 1 - i
        if cnt > 0:
            self._chk(self.L.aqr_step_rrow_reduce(m, cnt, self.partial.data_ptr(), self._rt(i, i + 1),
                                                  self.status.data_ptr(), D.stream_ptr()), "rrow_reduce")
        return self.Rt[i, i + 1:]

    def finish(self):
        n = self.n
        R = D.empty_f(n, n, self.dev)
        self._chk(self.L.aqr_step_finalize_r(n, self.Rt.data_ptr(), R.data_ptr(), n, D.stream_ptr()),
                  "finalize_r")
        st = self.status.cpu().numpy()
        fail = int(st[0])
        fail_val = float(st[2:4].view(np.float64)[0])
        flags = st[4:4 + n]
        return self.W, R, fail, fail_val, [int(j) for j in np.flatnonzero(flags)]


def dist_factorize(Z_local, op, method="mgs-ha-row", group=None, engine=None, backend=None):
    """Row-partitioned factorization; every rank passes its row block.

    ``op`` is a DistCsrSpdOperator / DistDenseSpdOperator (collective
    applies).  Returns QrResult(Q_local, R (replicated), cost, flagged).
    Only the row-oriented schedule exists here; it is bitwise the single-GPU
    result when world_size == 1.  HA / HP with a DistCsrSpdOperator run on
    the peer-memory path (``p2p.py``: halo reads and both all-reduces fused
    into the step kernels); ``backend="nccl"`` (or naive, or a dense
    operator) runs the step-API engine below with NCCL all-reduces.
    """
    dist = _dist()
    if not isinstance(method, MethodId):
        method = MethodId.parse(method)
    if method.family == "cholqr":
        raise ValueError("the distributed driver runs the Gram-Schmidt methods")
    # col and row orientation give bitwise-identical factors: both run the
    # row-oriented step schedule here (as on one GPU)
    family, variant = method.family, method.variant
    m_loc, n = (int(s) for s in Z_local.shape)
    if n < 1 or op.dim != m_loc:
        raise DimensionError("local block does not match the operator")
    if op.global_dim < n:
        raise DimensionError(f"need m >= n >= 1, got m={op.global_dim}, n={n}")
    from . import p2p

    if backend not in (None, "p2p", "nccl"):
        raise ValueError("backend must be 'p2p' or 'nccl'")
    if engine is None and backend != "nccl" and p2p.supported(op, method):
        # exchanges fused into the step kernels over peer memory (csrc/aqr_p2p.cuh)
        return p2p.p2p_factorize(Z_local, op, method, group=group)
    if backend == "p2p":
        raise ValueError("the peer-memory path runs HA / HP row factorizations with a DistCsrSpdOperator")
    eng = engine or CudaStepEngine(m_loc, n, family, variant, Z_local.device)
    mv_before = op.mv_count
    eng.load(Z_local)
    if variant == "hp":
        eng.set_X(op.apply_block(eng.w_block()))  # gram_schmidt.py:136
    for i in range(n):
        eng.col_update(i)
        if variant != "hp":
            eng.set_x(op.apply(eng.z(i).contiguous()))  # line 151
        tot = eng.norm_partials(i)
        dist.all_reduce(tot, group=group)
        eng.norm_finish(i, tot)
        if variant == "naive":
            eng.normalize_q(i)
            eng.set_p(op.apply(eng.q(i).contiguous()))  # line 163
        rrow = eng.trailing(i)
        if rrow.numel():
            dist.all_reduce(rrow, group=group)
    Q, R, fail, fail_val, flagged = eng.finish()
    if fail >= 0:
        raise BreakdownError(fail, fail_val)
    cost = CostReport(op.mv_count - mv_before, _model_flops(family, variant, op.global_dim, n))
    return QrResult(Q, R, cost, flagged)
