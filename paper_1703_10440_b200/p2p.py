"""Peer-memory multi-GPU path (csrc/aqr_p2p.cuh, ``aqr_p2p_gs_factor``).

One process per GPU of one node.  ``PeerGroup`` (collective construction)
allocates this rank's working matrix W (the local rows of Q) and exchange
buffer with ``aqr_p2p_alloc``, exchanges their CUDA IPC handles with one
``all_gather_object`` and maps every other rank's buffers.  The factorization
then runs with no collective call at all: the SpMV step reads its halo rows
from the owning rank's W over NVLink, and the two per-step all-reduces are
stores into every rank's exchange buffer plus release/acquire flags, summed
in rank order (bitwise the same on every rank; with one rank bitwise the
single-GPU ``factorize``).  ``distributed.dist_factorize`` routes HA / HP
row-oriented factorizations with a ``DistCsrSpdOperator`` here.
"""

import ctypes

import numpy as np

from . import _device as D
from . import _lib
from .exceptions import BreakdownError, DimensionError
from .gram_schmidt import QrResult, _model_flops
from .operators import CostReport


class PeerExchangeTimeout(RuntimeError):
    """A peer's exchange flag did not arrive within the group's timeout.

    Every rank that sees it drops its peer group; the next call re-creates it
    collectively (new buffers, flags from zero)."""


def _dist():
    import torch.distributed as dist

    return dist


class PeerGroup:
    """This rank's W (m_loc x n) and exchange buffer, plus every peer's mapping."""

    def __init__(self, m_loc, n, group=None, timeout_s=60.0):
        dist = _dist()
        self.L = L = _lib.lib()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > _lib.MAX_RANKS:
            raise ValueError(f"the peer-memory path supports up to {_lib.MAX_RANKS} ranks")
        self.m_loc, self.n = int(m_loc), int(n)
        self._own = []
        self.W = self._alloc(8 * max(self.m_loc, 1) * self.n)
        self.xb = self._alloc(int(L.aqr_p2p_exchange_bytes(self.n)))
        hw, hx = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
        _lib.check(L.aqr_ipc_handle(self.W, hw), "aqr_ipc_handle")
        _lib.check(L.aqr_ipc_handle(self.xb, hx), "aqr_ipc_handle")
        infos = [None] * self.world
        dist.all_gather_object(infos, (hw.raw, hx.raw, self.m_loc, self.n), group=group)
        if any(info[3] != self.n for info in infos):
            raise DimensionError("every rank must factorize the same number of columns")
        self._mapped = []
        self.desc = _lib.AqrP2PGroup()
        self.desc.nranks, self.desc.rank = self.world, self.rank
        for r, (h_w, h_x, m_r, _) in enumerate(infos):
            if r == self.rank:
                w, x = self.W, self.xb
            else:
                w, x = self._open(h_w), self._open(h_x)
            self.desc.W[r], self.desc.xbuf[r], self.desc.ldw[r] = w, x, max(int(m_r), 1)
        self.desc.timeout_ns = int(timeout_s * 1e9)
        self.next_seq = 1

    def _alloc(self, nbytes):
        p = ctypes.c_void_p()
        _lib.check(self.L.aqr_p2p_alloc(nbytes, ctypes.byref(p)), "aqr_p2p_alloc")
        self._own.append(p.value)
        return p.value

    def _open(self, handle):
        p = ctypes.c_void_p()
        _lib.check(self.L.aqr_ipc_open(handle, ctypes.byref(p)), "aqr_ipc_open")
        self._mapped.append(p.value)
        return p.value

    def W_tensor(self):
        return D.wrap(self.W, self.m_loc, self.n, max(self.m_loc, 1))

    def close(self):
        for p in self._mapped:
            self.L.aqr_ipc_close(p)
        for p in self._own:
            self.L.aqr_p2p_free(p)
        self._mapped, self._own = [], []

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


def supported(op, method):
    from .distributed import DistCsrSpdOperator

    return (isinstance(op, DistCsrSpdOperator) and op.local_apply is None
            and method.variant in ("ha", "hp") and method.family in ("mgs", "cgs"))


def p2p_factorize(Z_local, op, method, group=None, timeout_s=60.0):
    """Row-partitioned factorization over peer memory (every rank calls it).

    A rank that waits longer than ``timeout_s`` for a peer's exchange flag
    raises PeerExchangeTimeout (the kernels give up instead of spinning
    forever)."""
    t = D.torch()
    L = _lib.lib()
    m_loc, n = (int(s) for s in Z_local.shape)
    if n < 1 or op.dim != m_loc:
        raise DimensionError("local block does not match the operator")
    if op.global_dim < n:
        raise DimensionError(f"need m >= n >= 1, got m={op.global_dim}, n={n}")
    key = (m_loc, n, id(group))
    pg = getattr(op, "_peer_groups", {}).get(key)
    if pg is None:
        pg = PeerGroup(m_loc, n, group, timeout_s)
        op._peer_groups = {**getattr(op, "_peer_groups", {}), key: pg}
    if not hasattr(op, "_halo_dev"):
        op._halo_dev = (t.from_numpy(op.halo_rank).to(D.device()), t.from_numpy(op.halo_row).to(D.device()))
    pg.desc.timeout_ns = int(timeout_s * 1e9)
    hr, hw = op._halo_dev
    pg.desc.n_halo = int(hr.numel())
    pg.desc.halo_rank = hr.data_ptr() if hr.numel() else None
    pg.desc.halo_row = hw.data_ptr() if hw.numel() else None
    pg.desc.seq0 = pg.next_seq
    pg.next_seq += n + 2

    Zd, ldz = D.to_device_f(Z_local)
    W = pg.W_tensor()
    R = D.empty_f(n, n)
    fam, var = _lib.FAMILY_CODE[method.family], _lib.VARIANT_CODE[method.variant]
    ws = t.empty(int(L.aqr_workspace_bytes(fam, var, _lib.ORIENTATION_CODE["row"], m_loc, n)),
                 dtype=t.uint8, device=W.device)
    flags = np.zeros(n, dtype=np.int32)
    a = _lib.AqrFactorArgs()
    a.family, a.variant, a.orientation = fam, var, _lib.ORIENTATION_CODE["row"]
    a.m, a.n = m_loc, n
    a.Z, a.ldz = Zd.data_ptr(), ldz
    a.Q, a.ldq = pg.W, max(m_loc, 1)
    a.R, a.ldr = R.data_ptr(), n
    a.op = ctypes.pointer(op._native())
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    a.flagged_host = flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    mv_before = op.mv_count
    status = L.aqr_p2p_gs_factor(ctypes.byref(a), ctypes.byref(pg.desc), D.stream_ptr())
    if status == _lib.AQR_ETIMEOUT:
        op._peer_groups = {k: v for k, v in op._peer_groups.items() if v is not pg}
        pg.close()
        raise PeerExchangeTimeout(L.aqr_last_error().decode())
    if status == _lib.AQR_EBREAKDOWN:
        f = int(a.fail_col)
        op.mv_count += n if method.variant == "hp" else f + 1
        raise BreakdownError(f, float(a.fail_val))
    _lib.check(status, "aqr_p2p_gs_factor")
    op.mv_count += n
    Q = W.clone()  # W is this group's working matrix, reused by the next call
    cost = CostReport(op.mv_count - mv_before, _model_flops(method.family, method.variant, op.global_dim, n))
    return QrResult(Q, R, cost, [int(j) for j in np.flatnonzero(flags)])


class _EmulatedGroup:
    """Rank ``rank`` of a single-device emulated group: plain device pointers
    to every rank's W / exchange buffer (no IPC)."""

    def __init__(self, L, rank, ws, xbs, m_locs, n, timeout_s):
        self.W, self.xb = ws[rank], xbs[rank]
        self.m_loc, self.n = m_locs[rank], n
        self.desc = _lib.AqrP2PGroup()
        self.desc.nranks, self.desc.rank = len(ws), rank
        for r in range(len(ws)):
            self.desc.W[r], self.desc.xbuf[r], self.desc.ldw[r] = ws[r], xbs[r], max(int(m_locs[r]), 1)
        self.desc.timeout_ns = int(timeout_s * 1e9)

    def W_tensor(self):
        return D.wrap(self.W, self.m_loc, self.n, max(self.m_loc, 1))


def p2p_factorize_lockstep(Z_blocks, ops, method, seq0=1, timeout_s=60.0, solo=None):
    """Run an N-rank peer-memory factorization on ONE device (tests).

    ``Z_blocks[r]`` / ``ops[r]`` are rank r's row block and local operator
    (``DistCsrSpdOperator.blocks_of``).  The library interleaves the ranks'
    launches phase by phase on the current stream
    (``aqr_p2p_gs_factor_lockstep``), so every flag a kernel waits for is
    already raised when it starts -- the multi-rank kernels, flags, halo
    reads and rank-ordered sums run without kernels that wait on one another
    sharing the GPU.  Returns one QrResult per rank (Q = the rank's rows).

    ``solo=r`` launches rank r alone (the others never start): its waits
    must end in PeerExchangeTimeout after ``timeout_s`` (bounded-wait test;
    one kernel waits, nothing else needs to run beside it)."""
    from .gram_schmidt import MethodId

    t = D.torch()
    L = _lib.lib()
    if not isinstance(method, MethodId):
        method = MethodId.parse(method)
    N = len(ops)
    n = int(Z_blocks[0].shape[1])
    m_locs = [int(Zb.shape[0]) for Zb in Z_blocks]
    own = []

    def alloc(nbytes):
        p = ctypes.c_void_p()
        _lib.check(L.aqr_p2p_alloc(nbytes, ctypes.byref(p)), "aqr_p2p_alloc")
        own.append(p.value)
        return p.value

    try:
        ws = [alloc(8 * max(m, 1) * n) for m in m_locs]
        xbs = [alloc(int(L.aqr_p2p_exchange_bytes(n))) for _ in range(N)]
        groups, argv, keep = [], [], []
        fam, var = _lib.FAMILY_CODE[method.family], _lib.VARIANT_CODE[method.variant]
        for r in range(N):
            g = _EmulatedGroup(L, r, ws, xbs, m_locs, n, timeout_s)
            op = ops[r]
            hr = t.from_numpy(op.halo_rank).to(D.device())
            hw = t.from_numpy(op.halo_row).to(D.device())
            g.desc.n_halo = int(hr.numel())
            g.desc.halo_rank = hr.data_ptr() if hr.numel() else None
            g.desc.halo_row = hw.data_ptr() if hw.numel() else None
            g.desc.seq0 = seq0
            Zd, ldz = D.to_device_f(Z_blocks[r])
            R = D.empty_f(n, n)
            wsb = t.empty(int(L.aqr_workspace_bytes(fam, var, _lib.ORIENTATION_CODE["row"], m_locs[r], n)),
                          dtype=t.uint8, device=R.device)
            flags = np.zeros(n, dtype=np.int32)
            a = _lib.AqrFactorArgs()
            a.family, a.variant, a.orientation = fam, var, _lib.ORIENTATION_CODE["row"]
            a.m, a.n = m_locs[r], n
            a.Z, a.ldz = Zd.data_ptr(), ldz
            a.Q, a.ldq = g.W, max(m_locs[r], 1)
            a.R, a.ldr = R.data_ptr(), n
            a.op = ctypes.pointer(op._native())
            a.workspace, a.workspace_bytes = wsb.data_ptr(), wsb.numel()
            a.flagged_host = flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            groups.append(g)
            argv.append(a)
            keep.append((hr, hw, Zd, R, wsb, flags))
        arr_a = (ctypes.POINTER(_lib.AqrFactorArgs) * N)(*[ctypes.pointer(a) for a in argv])
        arr_g = (ctypes.POINTER(_lib.AqrP2PGroup) * N)(*[ctypes.pointer(g.desc) for g in groups])
        if solo is not None:
            status = L.aqr_p2p_gs_factor(ctypes.pointer(argv[solo]), ctypes.pointer(groups[solo].desc),
                                         D.stream_ptr())
        else:
            status = L.aqr_p2p_gs_factor_lockstep(N, arr_a, arr_g, D.stream_ptr())
        if status == _lib.AQR_ETIMEOUT:
            raise PeerExchangeTimeout(L.aqr_last_error().decode())
        if solo is not None:
            raise RuntimeError(f"a solo rank finished with status {status}")
        if status == _lib.AQR_EBREAKDOWN:
            cols = {(int(a.fail_col), float(a.fail_val)) for a in argv}
            if len(cols) != 1:
                raise RuntimeError(f"ranks disagree on the breakdown: {sorted(cols)}")
            f = int(argv[0].fail_col)
            for r in range(N):
                ops[r].mv_count += n if method.variant == "hp" else f + 1
            raise BreakdownError(f, float(argv[0].fail_val))
        _lib.check(status, "aqr_p2p_gs_factor_lockstep")
        out = []
        for r in range(N):
            ops[r].mv_count += n
            Q = groups[r].W_tensor().clone()
            cost = CostReport(n, _model_flops(method.family, method.variant, ops[r].global_dim, n))
            out.append(QrResult(Q, keep[r][3], cost, [int(j) for j in np.flatnonzero(keep[r][5])]))
        D.torch().cuda.current_stream().synchronize()
        return out
    finally:
        D.torch().cuda.synchronize()
        for p in own:
            L.aqr_p2p_free(p)
