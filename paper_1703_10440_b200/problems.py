"""Seeded synthetic inputs for BASELINE.json configs 2-5.

No dataset is named by the reference; these generators stand in with the
shapes, stencils and value distributions BASELINE.json specifies.  Seeds
follow the reference's PCG64/SeedSequence convention (testbed.py:29-31):
SeedSequence([1703, 10440, config, stream]), stream 0 for A, 1 for Z.

CSR row order and in-row column order follow laplacian_spd
(testbed.py:128-153): row = (iz * ny + iy) * nx + ix, neighbours sorted by
column index.  Config 1 (dense, the oracle case) lives in tests/cfg1.py.

Every generator returns host numpy arrays (``device=False``) or CUDA
tensors (``device=True``; configs 4-5 are too large for host-side use).
"""

import numpy as np


def rng(config, stream):
    return np.random.default_rng(np.random.SeedSequence([1703, 10440, config, stream]))


def _stencil_csr(shape, offsets, values_fn, diag_fn):
    """CSR of a Dirichlet stencil on a grid (x fastest), columns ascending.

    ``offsets``: list of (dz, dy, dx) neighbour offsets (the centre excluded);
    ``values_fn(k, mask)`` off-diagonal values for offset k at valid points;
    ``diag_fn()`` the diagonal (one value per grid point).
    """
    nz, ny, nx = shape
    m = nx * ny * nz
    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    iz, iy, ix = iz.ravel(), iy.ravel(), ix.ravel()
    row = np.arange(m, dtype=np.int64)
    entries = []  # (col, val, valid) per slot, slot order = ascending column offset
    full = sorted(list(offsets) + [(0, 0, 0)], key=lambda o: (o[0] * ny + o[1]) * nx + o[2])
    for off in full:
        dz, dy, dx = off
        valid = ((iz + dz >= 0) & (iz + dz < nz) & (iy + dy >= 0) & (iy + dy < ny)
                 & (ix + dx >= 0) & (ix + dx < nx))
        col = row + (dz * ny + dy) * nx + dx
        val = diag_fn() if off == (0, 0, 0) else values_fn(offsets.index(off), valid)
        entries.append((col, val, valid))
    cols = np.stack([e[0] for e in entries], axis=1)
    vals = np.stack([np.broadcast_to(e[1], (m,)) for e in entries], axis=1)
    valid = np.stack([e[2] for e in entries], axis=1)
    counts = valid.sum(axis=1)
    indptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, cols[valid].astype(np.int64), vals[valid].astype(np.float64)


def laplacian5(nx, ny, shift):
    """2-D 5-point Laplacian, Dirichlet boundary, + shift*I (diag 4+shift, off -1)."""
    offs = [(0, -1, 0), (0, 0, -1), (0, 0, 1), (0, 1, 0)]
    m = nx * ny
    return _stencil_csr((1, ny, nx), offs, lambda k, v: -1.0, lambda: np.full(m, 4.0 + shift))


def config2(device=False):
    """m = 1024^2 = 1,048,576, n = 64; 5-pt Laplacian + 1e-2 I; Z ~ N(0,1)."""
    indptr, indices, data = laplacian5(1024, 1024, 1e-2)
    m, n = 1024 * 1024, 64
    Z = np.asfortranarray(rng(2, 1).standard_normal((n, m)).T)
    return _out((indptr, indices, data), Z, device)


def diffusion7(n_side, shift, seed_rng):
    """3-D 7-point variable-coefficient diffusion on n^3, Dirichlet.

    Face coefficients c_f = 10^U(-2, 2) on every face of the (n+1) x n x n
    x-face lattice (and likewise y, z), boundary faces included; A_ii =
    sum of the 6 face coefficients + shift, A_ij = -c_f.
    """
    n = n_side
    cx = 10.0 ** seed_rng.uniform(-2, 2, size=(n, n, n + 1))  # [z, y, x-face]
    cy = 10.0 ** seed_rng.uniform(-2, 2, size=(n, n + 1, n))
    cz = 10.0 ** seed_rng.uniform(-2, 2, size=(n + 1, n, n))
    west, east = cx[:, :, :-1].ravel(), cx[:, :, 1:].ravel()
    south, north = cy[:, :-1, :].ravel(), cy[:, 1:, :].ravel()
    down, up = cz[:-1, :, :].ravel(), cz[1:, :, :].ravel()
    diag = west + east + south + north + down + up + shift
    face = {(-1, 0, 0): down, (0, -1, 0): south, (0, 0, -1): west,
            (0, 0, 1): east, (0, 1, 0): north, (1, 0, 0): up}
    offs = list(face)
    return _stencil_csr((n, n, n), offs, lambda k, v: -face[offs[k]], lambda: diag)


def config3(device=False):
    """m = 128^3 = 2,097,152, n = 128; 7-pt diffusion + 1e-3 I; Z = G diag(10^(-6 j/127))."""
    indptr, indices, data = diffusion7(128, 1e-3, rng(3, 0))
    m, n = 128 ** 3, 128
    scale = 10.0 ** (-6.0 * np.arange(n) / (n - 1))
    Z = np.asfortranarray(rng(3, 1).standard_normal((n, m)).T * scale)
    return _out((indptr, indices, data), Z, device)


def _torch_gen(config, stream, device, sub=None):
    import torch

    key = [1703, 10440, config, stream] + ([] if sub is None else [sub])
    ss = np.random.SeedSequence(key)
    g = torch.Generator(device=device)
    g.manual_seed(int(ss.generate_state(1, dtype=np.uint64)[0] & ((1 << 63) - 1)))
    return g


def config4(device=True, m=32768, n=256, rows=None):
    """Dense m = 32768, n = 256: A = B^T B / m + 0.1 I (B ~ N(0,1)), Z ~ N(0,1), on the GPU.

    ``rows = (r0, r1)`` returns only that row panel of A (all m columns) and
    of Z -- what one rank of the row-partitioned run owns (Z rows exactly
    those of the full Z; A's panel equal to the full A's rows up to the
    rounding of the Gram product)."""
    import torch

    dev = torch.device("cuda")
    r0, r1 = rows if rows is not None else (0, m)
    B = torch.randn((m, m), generator=_torch_gen(4, 0, dev), dtype=torch.float64, device=dev)
    if rows is None:
        A = B.transpose(0, 1) @ B
        del B
        A /= m
        A = 0.5 * (A + A.transpose(0, 1))
        A.diagonal().add_(0.1)
    else:  # the panel of the symmetrised matrix, formed as the full one forms it
        P = B[:, r0:r1].transpose(0, 1) @ B  # rows r0..r1 of B^T B
        PT = (B.transpose(0, 1) @ B[:, r0:r1]).transpose(0, 1)  # rows r0..r1 of (B^T B)^T
        del B
        P /= m
        PT /= m
        A = 0.5 * (P + PT)
        del P, PT
        A[:, r0:r1].diagonal().add_(0.1)
        A = A.t().contiguous().t()  # column-major panel, ld = r1 - r0
    Z = torch.randn((n, m), generator=_torch_gen(4, 1, dev), dtype=torch.float64, device=dev)
    Z = Z[:, r0:r1].contiguous().t() if rows is not None else Z.t()
    return A, Z


def stencil27_device(n_side, shift, device, planes=None):
    """3-D 27-point stencil on n^3 (centre 26 + shift, neighbours -1), CSR on the GPU.

    ``planes = (z0, z1)`` builds only rows z0 n^2 .. z1 n^2 - 1 (whole grid
    planes, what one rank of the row-partitioned run owns) with GLOBAL column
    indices; indptr starts at 0.  Returns (indptr int64, indices int32,
    values fp64)."""
    import torch

    n = n_side
    m = n ** 3
    z0, z1 = planes if planes is not None else (0, n)
    dev = torch.device(device)
    idx = torch.arange(z0 * n * n, z1 * n * n, device=dev, dtype=torch.int64)
    iz, iy, ix = idx // (n * n), (idx // n) % n, idx % n
    cols, vals, valids = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                v = ((iz + dz >= 0) & (iz + dz < n) & (iy + dy >= 0) & (iy + dy < n)
                     & (ix + dx >= 0) & (ix + dx < n))
                valids.append(v)
                cols.append((idx + (dz * n + dy) * n + dx).to(torch.int32))
                vals.append(26.0 + shift if (dz, dy, dx) == (0, 0, 0) else -1.0)
    del iz, iy, ix
    valid = torch.stack(valids, dim=1)
    del valids
    counts = valid.sum(dim=1)
    indptr = torch.zeros(idx.numel() + 1, dtype=torch.int64, device=dev)
    indptr[1:] = torch.cumsum(counts, 0)
    col = torch.stack(cols, dim=1)[valid]
    del cols
    val = torch.tensor(vals, dtype=torch.float64, device=dev).expand(idx.numel(), 27)[valid]
    assert m < 2 ** 31
    return indptr, col, val


CONFIG5_ZCHUNK = 16  # columns of Z drawn per seeded generator (config5_Z)


def config5_Z(m, n, rows=None):
    """Config-5 Z ~ N(0,1), m x n column-major on the GPU, drawn in blocks of
    CONFIG5_ZCHUNK columns, block b from SeedSequence([1703, 10440, 5, 1, b]),
    so any row range (one rank's rows) is reproducible without the whole
    34 GB matrix on one device."""
    import torch

    dev = torch.device("cuda")
    r0, r1 = rows if rows is not None else (0, m)
    Zt = torch.empty((n, r1 - r0), dtype=torch.float64, device=dev)
    for b, c0 in enumerate(range(0, n, CONFIG5_ZCHUNK)):
        c1 = min(n, c0 + CONFIG5_ZCHUNK)
        if rows is None:
            torch.randn((c1 - c0, m), generator=_torch_gen(5, 1, dev, b), dtype=torch.float64,
                        device=dev, out=Zt[c0:c1])
        else:
            blk = torch.randn((c1 - c0, m), generator=_torch_gen(5, 1, dev, b), dtype=torch.float64, device=dev)
            Zt[c0:c1].copy_(blk[:, r0:r1])
            del blk
    return Zt.t()


def config5(device=True, n_side=256, n=256, planes=None):
    """m = 256^3 = 16,777,216, n = 256; 27-pt + 1e-2 I; Z ~ N(0,1) (34.4 GB) on the GPU.

    ``planes = (z0, z1)``: only those grid planes' rows (row-partitioned runs)."""
    import torch

    dev = torch.device("cuda")
    indptr, indices, data = stencil27_device(n_side, 1e-2, dev, planes)
    m = n_side ** 3
    z0, z1 = planes if planes is not None else (0, n_side)
    Z = config5_Z(m, n, rows=(z0 * n_side * n_side, z1 * n_side * n_side) if planes is not None else None)
    return (indptr, indices, data), Z


def _out(csr, Z, device):
    if not device:
        return csr, Z
    import torch

    indptr, indices, data = (torch.from_numpy(a).cuda() for a in csr)
    return (indptr, indices, data), torch.from_numpy(Z.T).cuda().t()


# ---- the reference's testbed generators used by the bench / factor CLI ----

def make_rng(seed):
    """The reference's deterministic generator (testbed.py:29-31)."""
    return np.random.default_rng(np.random.SeedSequence(seed))


def haar_orthogonal(rng, k):
    """Haar orthogonal k x k: QR of a Gaussian, column signs fixed (linalg.py:59-75)."""
    from .exceptions import DimensionError

    if k < 1:
        raise DimensionError("k must be >= 1")
    while True:
        G = rng.standard_normal((k, k))
        Q, R = np.linalg.qr(G)
        d = np.diag(R)
        if np.all(d != 0.0):
            break
    return np.asfortranarray(Q * np.where(d < 0.0, -1.0, 1.0))


def build_spd(m, kappa, rng):
    """(eigenvalues, DenseSpdOperator) with eigenvalues 10^(alpha (i-1)) (testbed.py:77-88).

    A = (V diag(d)) V^T is formed by the bitwise sequential dense block apply
    on the device (the reference's per-entry sequential matmul), then
    symmetrized."""
    from .exceptions import DimensionError
    from .operators import DenseSpdOperator

    if m < 2:
        raise DimensionError("m must be >= 2")
    if kappa < 1.0:
        raise ValueError("kappa must be >= 1")
    V = haar_orthogonal(rng, m)
    d = 10.0 ** (np.log10(kappa) / (m - 1) * np.arange(m))
    A = np.asarray(DenseSpdOperator(np.asfortranarray(V * d)).apply_block(np.asfortranarray(V.T)))
    return d, DenseSpdOperator(np.asfortranarray(0.5 * (A + A.T)))


def laplacian_spd(nx, ny):
    """5-point Laplacian on an nx-by-ny grid, Dirichlet boundary, CSR (testbed.py:128-153)."""
    from .exceptions import DimensionError
    from .operators import CsrSpdOperator

    if nx < 2 or ny < 2:
        raise DimensionError("grid must be at least 2x2")
    return CsrSpdOperator(*laplacian5(nx, ny, 0.0))
