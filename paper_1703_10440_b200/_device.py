"""Device-memory plumbing (torch is used for allocation and streams only).

Column-major (Fortran) m x n device matrices are torch tensors of shape
(m, n) with strides (1, ld): column j starts at data_ptr() + 8 * j * ld.
"""

import os

import numpy as np

from ._lib import ExtensionUnavailable

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def is_torch(x):
    try:
        import torch as t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, t.Tensor)


def device():
    t = torch()
    if not t.cuda.is_available():
        raise ExtensionUnavailable("no CUDA device: the aqr B200 path has no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def stream_ptr():
    return torch().cuda.current_stream().cuda_stream


def empty_f(m, n, dev=None):
    """Uninitialized column-major (m, n) fp64 device matrix (ld = m)."""
    t = torch()
    return t.empty((n, m), dtype=t.float64, device=dev or device()).t()


def leading_dim(T):
    """ld of a column-major 2-D tensor view, or None if not column-major."""
    if T.dim() != 2:
        return None
    m, n = T.shape
    s0, s1 = T.stride()
    if (s0 == 1 or m <= 1) and (s1 >= max(m, 1) or n <= 1):
        return max(s1, m, 1)
    return None


def to_device_f(a, dev=None):
    """(device column-major fp64 tensor, ld) for a numpy array or tensor.

    Never modifies ``a``; copies only when ``a`` is not already a column-major
    fp64 tensor on the device.
    """
    t = torch()
    dev = dev or device()
    if is_torch(a):
        T = a
        if T.dtype != t.float64:
            T = T.to(t.float64)
        if T.device != dev:
            T = T.to(dev, non_blocking=T.is_pinned())
        ld = leading_dim(T)
        if ld is None:
            T = T.t().contiguous().t()
            ld = leading_dim(T)
        return T, ld
    A = np.asfortranarray(a, dtype=np.float64)
    if A.ndim == 2 and A.nbytes >= _STAGE_MIN_BYTES:
        return _h2d_staged(A, dev), max(A.shape[0], 1)
    T = t.from_numpy(A.T.copy(order="C") if not A.flags.f_contiguous else A.T).to(dev).t()
    return T, max(A.shape[0], 1)


# Large numpy inputs: a pageable host->device copy runs at ~11 GB/s through
# the driver's staging buffers.  Instead, host threads copy column chunks into
# a page-locked staging block (numpy releases the GIL) and each chunk's DMA is
# queued on the current stream as soon as its copy is done (~55 GB/s).  The
# staging block comes from torch's page-locked cache, which keeps it alive
# until the queued copies complete.
_STAGE_MIN_BYTES = 64 << 20
# host threads copying pageable input into the page-locked staging block.
# Alone, 16 threads stage at 83-91 GB/s (tools/stage_bench.py), but inside the
# factorization call the copies compete with the H2D / D2H DMA for host
# memory bandwidth.  Wide problems are compute-bound (device time ~ n x the
# transfer time / 170): there the staging only has to keep loosely ahead, and
# with 16 threads the first chunks reach the device every 43 ms instead of
# every 20 ms (tools/pipe_trace.py mgs-hp-row 5 numpy) -- the device idles
# through the first half second.  Config 5 HP (n = 256), numpy in / numpy out
# on a 16-core host (tools/e2e_repeat.py, AQR_STAGE_THREADS sweep): 1.70-1.78 s
# with 16 threads, 1.65-1.71 (8), 1.58-1.67 (6), 1.55-1.64 (4), 1.63 (3),
# 1.83 (2).  Narrow problems are transfer-bound and want the full staging
# rate: config 2 / 3 HA (n = 64 / 128) 21.5 / 85.9 ms with 8 threads,
# 22.9 / 86.0 (16), 25.1-25.7 / 104 (4).  AQR_STAGE_THREADS overrides both.
_STAGE_THREADS = int(os.environ.get("AQR_STAGE_THREADS", "0"))
_pools = {}


def _stage_pool(n_cols=0):
    """The host staging pool for an input of ``n_cols`` columns."""
    from concurrent.futures import ThreadPoolExecutor

    cores = os.cpu_count() or 4
    size = _STAGE_THREADS or (max(2, min(4, cores)) if n_cols >= 192 else max(2, min(8, cores)))
    if size not in _pools:
        _pools[size] = ThreadPoolExecutor(size, thread_name_prefix="aqr-h2d")
    return _pools[size]


class StagedHost:
    """Page-locked column-major copy of a host matrix, filled concurrently.

    ``a`` (numpy array or CPU tensor, m x n) is copied column by column on
    the host thread pool, chunk after chunk (chunk c = columns
    ``bounds[c] .. bounds[c + 1] - 1``, the pipeline's schedule);
    ``ready`` (a page-locked uint32) counts the chunks that are complete, in
    order, so the device can start copying chunk c once ready >= c + 1
    (aqr_gs_factor_pinned) while later chunks are still being written.  A
    tensor that already is page-locked, fp64 and column-major is used as it
    is (``ready`` is None).
    """

    def __init__(self, a, bounds):
        import threading

        t = torch()
        if is_torch(a) and a.is_pinned() and a.dtype == t.float64 and leading_dim(a) is not None:
            self.T, self.ld, self.ready, self._futs = a, leading_dim(a), None, []
            return
        m, n = a.shape
        _pool = _stage_pool(n)
        self.stage = t.empty((n, m), dtype=t.float64, pin_memory=True)
        self.T, self.ld = self.stage.t(), max(m, 1)
        self.flag = t.zeros(1, dtype=t.int32, pin_memory=True)
        self.ready = self.flag.data_ptr()
        flag = self.flag.numpy()
        if is_torch(a):
            src, dst = a.t(), self.stage
            copy = lambda j: dst[j].copy_(src[j])  # noqa: E731
        else:
            src, dst = np.asarray(a, dtype=np.float64).T, self.stage.numpy()
            copy = lambda j: np.copyto(dst[j], src[j])  # noqa: E731
        bounds = [int(b) for b in bounds]
        nch = len(bounds) - 1
        left = [bounds[c + 1] - bounds[c] for c in range(nch)]
        state = {"next": 0, "error": None}
        lock = threading.Lock()

        def task(c, j):
            try:
                copy(j)
            except BaseException as exc:  # never leave the device waiting
                state["error"] = exc
            with lock:
                left[c] -= 1
                while state["next"] < nch and left[state["next"]] == 0:
                    state["next"] += 1
                if state["error"] is not None:
                    state["next"] = nch
                flag[0] = state["next"]

        self._state = state
        self._futs = [_pool.submit(task, c, j) for c in range(nch) for j in range(bounds[c], bounds[c + 1])]

    def finish(self):
        """Wait for the copy tasks; re-raise a copy error."""
        for f in self._futs:
            f.result()
        if self._futs and self._state["error"] is not None:
            raise self._state["error"]


def _h2d_staged(A, dev):
    t = torch()
    m, n = A.shape
    _pool = _stage_pool()  # a plain copy: nothing to overlap with, the full staging rate
    out = t.empty((n, m), dtype=t.float64, device=dev)  # row j = column j (column-major (m, n))
    stage = t.empty((n, m), dtype=t.float64, pin_memory=True)
    src, dst = A.T, stage.numpy()  # (n, m) C-ordered views
    nchunks = min(n, 4 * _pool._max_workers)
    bounds = [(k * n) // nchunks for k in range(nchunks + 1)]
    futs = [_pool.submit(np.copyto, dst[b0:b1], src[b0:b1]) for b0, b1 in zip(bounds[:-1], bounds[1:]) if b1 > b0]
    k = 0
    for b0, b1 in zip(bounds[:-1], bounds[1:]):
        if b1 <= b0:
            continue
        futs[k].result()
        k += 1
        out[b0:b1].copy_(stage[b0:b1], non_blocking=True)
    return out.t()


class CudaArray:
    """Zero-copy wrapper of a raw device pointer (``__cuda_array_interface__``)."""

    def __init__(self, ptr, shape, strides_bytes, readonly=False):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape),
            "typestr": "<f8",
            "data": (int(ptr), readonly),
            "version": 3,
            "strides": tuple(int(s) for s in strides_bytes),
            "stream": None,
        }


def wrap(ptr, m, k, ld):
    """Torch view of a raw column-major device block (m x k, leading dim ld)."""
    t = torch()
    if k == 1:
        arr = CudaArray(ptr, (m,), (8,))
    else:
        arr = CudaArray(ptr, (m, k), (8, 8 * ld))
    return t.as_tensor(arr, device=device())
