// aqr_kernels.cuh -- sm_100a device kernels of the A-orthogonal MGS hot path.
//
// Layout: column-major fp64 matrices with explicit leading dimension; CSR
// with int32 indptr/indices and fp64 values.  Reductions are atomic-free
// and depend only on (m, launch geometry fixed by m): rows are cut into
// tiles of tile_rows(m) rows, each tile partial is a fixed function of the
// tile's rows (per-thread ascending order, warp xor-butterfly 16..1, warps
// summed in ascending order) and tile partials are summed in a fixed order
// by *_reduce kernels.  Column grouping (blockIdx.y) never changes a tile
// partial, so the column-oriented schedule (one trailing column per launch)
// and the row-oriented schedule (all trailing columns per launch) produce
// bitwise-identical R and Q, the property the reference guarantees for its
// sequential loops (gram_schmidt.py:19-21).
//
// Elementwise updates follow the reference exactly: z -= a*q is a rounded
// multiply then a rounded subtract (__dmul_rn/__dsub_rn, no FMA contraction;
// _kernels_impl.py:85-88), x / r is an IEEE division (:91-93).  Operator
// products accumulate in the reference's order with separate rounding
// (_kernels_impl.py:24-56) and are therefore bitwise equal to it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace aqr {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

// Rows per thread of the reduction tile.  Depends on m only (never on the
// step, the variant or the orientation).
__host__ __device__ inline int rows_per_thread(int64_t m) {
    return m >= (int64_t)2048 * 148 ? 8 : 1;
}
__host__ __device__ inline int64_t tile_rows(int64_t m) { return (int64_t)kBlock * rows_per_thread(m); }
__host__ __device__ inline int64_t num_tiles(int64_t m) {
    const int64_t t = tile_rows(m);
    return (m + t - 1) / t;
}

__device__ __forceinline__ bool failed(const int32_t *status) {
    return status != nullptr && *(volatile const int32_t *)status >= 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Fixed-order block sum; every thread returns the same value.
__device__ __forceinline__ double block_sum(double v, double *smem /* kWarps */) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double s = smem[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) s = __dadd_rn(s, smem[w]);
    __syncthreads();
    return s;
}

// ---------------------------------------------------------------------------
// Fused trailing pass (one MGS step, row-oriented look-ahead schedule)
// ---------------------------------------------------------------------------
struct TrailArgs {
    int64_t m;
    int32_t ntiles;
    int32_t cpg;  // columns per blockIdx.y group
    int32_t jbeg, jend;
    double *W;
    int64_t ldw;
    double *X;  // HP carried A z (nullptr otherwise)
    int64_t ldx;
    const double *Z0;  // CGS original columns (nullptr for MGS)
    int64_t ldz0;
    const double *qprev;  // q_{i-1}; nullptr at i == 0 (no deferred update)
    const double *pprev;  // p_{i-1} (HP)
    const double *rprev;  // r_{i-1, j} = rprev[j] (row i-1 of row-major Rt)
    const double *psrc;   // p_i = psrc / *rii  (or psrc itself when rii == nullptr)
    const double *rii;
    double *pout;         // store p_i (blockIdx.y == 0)
    const double *zsrc;   // z_i
    double *qout;         // store q_i = z_i / *rii (blockIdx.y == 0)
    double *partial;      // [(j - jbeg) * ntiles + tile]
    const int32_t *status;
};

template <int RPT, int CU, bool HP, bool CGS>
__global__ void __launch_bounds__(kBlock) trailing_kernel(TrailArgs a) {
    if (failed(a.status)) return;
    extern __shared__ double wsum[];  // [kWarps][cpg]
    const int tile = blockIdx.x;
    const int64_t row0 = (int64_t)tile * (kBlock * RPT) + threadIdx.x;
    const int cbeg = a.jbeg + blockIdx.y * a.cpg;
    const int cend = min(a.jend, cbeg + a.cpg);
    const bool upd = a.qprev != nullptr;
    const double rii = a.rii ? *a.rii : 1.0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    double q[RPT], p[RPT], pp[RPT];
    bool ok[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t r = row0 + (int64_t)u * kBlock;
        ok[u] = r < a.m;
        const double ps = ok[u] ? a.psrc[r] : 0.0;
        p[u] = a.rii ? ps / rii : ps;
        q[u] = (ok[u] && upd) ? a.qprev[r] : 0.0;
        pp[u] = (HP && ok[u] && upd) ? a.pprev[r] : 0.0;
        if (blockIdx.y == 0 && ok[u]) {
            if (a.qout) a.qout[r] = a.zsrc[r] / rii;
            if (a.pout) a.pout[r] = p[u];
        }
    }

    for (int j0 = cbeg; j0 < cend; j0 += CU) {
        double z[CU][RPT], x[CU][RPT], rj[CU];
#pragma unroll
        for (int c = 0; c < CU; ++c) {
            const int j = j0 + c;
            const bool cj = j < cend;
            rj[c] = (cj && upd) ? a.rprev[j] : 0.0;
            const double *zc = a.W + (int64_t)j * a.ldw;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int64_t r = row0 + (int64_t)u * kBlock;
                z[c][u] = (cj && ok[u]) ? zc[r] : 0.0;
                if (HP) x[c][u] = (cj && ok[u] && upd) ? a.X[(int64_t)j * a.ldx + r] : 0.0;
            }
        }
        double acc[CU];
#pragma unroll
        for (int c = 0; c < CU; ++c) {
            const int j = j0 + c;
            const bool cj = j < cend;
            acc[c] = 0.0;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int64_t r = row0 + (int64_t)u * kBlock;
                if (upd) {
                    z[c][u] = __dsub_rn(z[c][u], __dmul_rn(rj[c], q[u]));
                    if (cj && ok[u]) a.W[(int64_t)j * a.ldw + r] = z[c][u];
                    if (HP) {
                        x[c][u] = __dsub_rn(x[c][u], __dmul_rn(rj[c], pp[u]));
                        if (cj && ok[u]) a.X[(int64_t)j * a.ldx + r] = x[c][u];
                    }
                }
                double d = z[c][u];
                if (CGS) d = (cj && ok[u]) ? a.Z0[(int64_t)j * a.ldz0 + r] : 0.0;
                acc[c] = fma(p[u], d, acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < CU; ++c) {
            const double s = warp_sum(acc[c]);
            if (lane == 0 && j0 + c < cend) wsum[warp * a.cpg + (j0 + c - cbeg)] = s;
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cend - cbeg; c += kBlock) {
        double s = wsum[c];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) s = __dadd_rn(s, wsum[w * a.cpg + c]);
        a.partial[(int64_t)(cbeg - a.jbeg + c) * a.ntiles + tile] = s;
    }
}

// out[c] = sum over tiles of partial[c * ntiles + tile], fixed order.
__global__ void __launch_bounds__(kBlock)
    rrow_reduce_kernel(const double *partial, int32_t ntiles, double *out, const int32_t *status) {
    if (failed(status)) return;
    __shared__ double sm[kWarps];
    const double *p = partial + (int64_t)blockIdx.x * ntiles;
    double s = 0.0;
    for (int t = threadIdx.x; t < ntiles; t += kBlock) s = __dadd_rn(s, p[t]);
    s = block_sum(s, sm);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ---------------------------------------------------------------------------
// Column update (deferred step i-1 projection of column i) + norm partials
// ---------------------------------------------------------------------------
struct ColArgs {
    int64_t m;
    int32_t ntiles;
    double *z;
    const double *qprev;
    double *x;  // HP: carried column, updated in place (nullptr otherwise)
    const double *pprev;
    const double *r;      // r_{i-1,i} (nullptr: no update)
    const double *xnorm;  // x used for the norm partials (== x for HP)
    double *npart;        // [3 * ntiles] or nullptr
    const int32_t *status;
};

template <int RPT>
__global__ void __launch_bounds__(kBlock) col_update_norm_kernel(ColArgs a) {
    if (failed(a.status)) return;
    __shared__ double sm[kWarps];
    const int64_t row0 = (int64_t)blockIdx.x * (kBlock * RPT) + threadIdx.x;
    const bool upd = a.r != nullptr;
    const double rj = upd ? *a.r : 0.0;
    double t = 0.0, zz = 0.0, xx = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t r = row0 + (int64_t)u * kBlock;
        if (r >= a.m) continue;
        double z = a.z[r];
        if (upd) {
            z = __dsub_rn(z, __dmul_rn(rj, a.qprev[r]));
            a.z[r] = z;
        }
        double xv = 0.0;
        if (a.x) {
            xv = a.x[r];
            if (upd) {
                xv = __dsub_rn(xv, __dmul_rn(rj, a.pprev[r]));
                a.x[r] = xv;
            }
        } else if (a.xnorm) {
            xv = a.xnorm[r];
        }
        t = fma(z, xv, t);
        zz = fma(z, z, zz);
        xx = fma(xv, xv, xx);
    }
    if (a.npart == nullptr) return;  // uniform across the block
    t = block_sum(t, sm);
    zz = block_sum(zz, sm);
    xx = block_sum(xx, sm);
    if (threadIdx.x == 0) {
        a.npart[blockIdx.x] = t;
        a.npart[a.ntiles + blockIdx.x] = zz;
        a.npart[2 * a.ntiles + blockIdx.x] = xx;
    }
}

// Status block: int32 fail column at [0], double fail value at byte 8,
// int32 flags[n] at byte 16.
__device__ __forceinline__ void norm_finish_dev(int64_t i, double t, double zz, double xx,
                                                double *rii, int32_t *status) {
    if (!(t > 0.0) || !isfinite(t)) {
        if (status[0] < 0) {
            status[0] = (int32_t)i;
            *reinterpret_cast<double *>(status + 2) = t;
        }
        return;
    }
    const double unit_roundoff = 1.1102230246251565e-16;  // 2**-53, gram_schmidt.py:33
    const double nz = sqrt(zz), nx = sqrt(xx);
    if (t < 100.0 * unit_roundoff * nz * nx) status[4 + i] = 1;  // gram_schmidt.py:155-158
    *rii = sqrt(t);
}

// 3 fixed-order sums of the norm partials; optionally finish in place.
__global__ void __launch_bounds__(kBlock)
    norm_reduce_kernel(const double *npart, int32_t ntiles, double *tot, int64_t i, double *rii,
                       int32_t *status) {
    if (failed(status)) return;
    __shared__ double sm[kWarps];
    double v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double s = 0.0;
        for (int t = threadIdx.x; t < ntiles; t += kBlock) s = __dadd_rn(s, npart[k * ntiles + t]);
        v[k] = block_sum(s, sm);
    }
    if (threadIdx.x == 0) {
        if (tot) {
            tot[0] = v[0];
            tot[1] = v[1];
            tot[2] = v[2];
        }
        if (rii) norm_finish_dev(i, v[0], v[1], v[2], rii, status);
    }
}

__global__ void norm_finish_kernel(int64_t i, const double *tot, double *rii, int32_t *status) {
    if (failed(status)) return;
    norm_finish_dev(i, tot[0], tot[1], tot[2], rii, status);
}

// q = z / rii ; p = x / rii  (normalize(j), gram_schmidt.py:159-165)
__global__ void __launch_bounds__(kBlock)
    normalize_kernel(int64_t m, const double *z, const double *rii, double *q, const double *x,
                     double *p, const int32_t *status) {
    if (failed(status)) return;
    const double r = *rii;
    for (int64_t i = blockIdx.x * (int64_t)kBlock + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * kBlock) {
        q[i] = z[i] / r;
        if (p) p[i] = x[i] / r;
    }
}

__global__ void finalize_r_kernel(int64_t n, const double *Rt, double *R, int64_t ldr) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * n) return;
    const int64_t i = idx % n, j = idx / n;  // R column-major: (i, j)
    R[i + j * ldr] = i <= j ? Rt[i * n + j] : 0.0;
}

__global__ void status_init_kernel(int32_t *status, int64_t n) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx == 0) {
        status[0] = -1;
        status[1] = 0;
        *reinterpret_cast<double *>(status + 2) = 0.0;
    }
    if (idx < n) status[4 + idx] = 0;
}

// ---------------------------------------------------------------------------
// Reference kernel namespace (backend.kernels()): dot, sub_scaled, div_scalar
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock)
    dot_partial_kernel(int64_t m, int rpt, const double *x, const double *y, double *part) {
    __shared__ double sm[kWarps];
    const int64_t row0 = (int64_t)blockIdx.x * (kBlock * rpt) + threadIdx.x;
    double s = 0.0;
    for (int u = 0; u < rpt; ++u) {
        const int64_t r = row0 + (int64_t)u * kBlock;
        if (r < m) s = fma(x[r], y[r], s);
    }
    s = block_sum(s, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sub_scaled_kernel(int64_t m, double *z, const double *a, const double *q) {
    const double s = *a;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        z[i] = __dsub_rn(z[i], __dmul_rn(s, q[i]));
}

__global__ void div_scalar_kernel(int64_t m, const double *x, const double *r, double *out) {
    const double s = *r;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = x[i] / s;
}

// ---------------------------------------------------------------------------
// Operators: CSR SpMV / SpMM, dense GEMV / GEMM -- reference-exact order
// ---------------------------------------------------------------------------

// L lanes per row.  Products are formed in parallel, then summed strictly in
// stored order (shuffle chain), bitwise equal to csr_matvec
// (_kernels_impl.py:50-56).  k columns handled in one pass (SpMM, the HP
// block apply) with the row's entries kept in registers.
template <int L>
__global__ void __launch_bounds__(kBlock)
    csr_spmm_kernel(int64_t m, int64_t k, const int32_t *__restrict__ indptr,
                    const int32_t *__restrict__ indices, const double *__restrict__ data,
                    const double *__restrict__ X, int64_t ldx, double *__restrict__ Y,
                    int64_t ldy) {
    const int64_t gid = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    const int64_t row = gid / L;
    if (row >= m) return;  // whole groups exit together
    const int lane = threadIdx.x & (L - 1);
    const unsigned mask =
        L == 32 ? 0xffffffffu : (((1u << L) - 1u) << ((threadIdx.x & 31) & ~(L - 1)));
    const int s = __ldg(indptr + row), e = __ldg(indptr + row + 1);
    if (L == 1) {
        for (int64_t c = 0; c < k; ++c) {
            const double *x = X + c * ldx;
            double acc = 0.0;
            for (int q = s; q < e; ++q) acc = __dadd_rn(acc, __dmul_rn(__ldg(data + q), __ldg(x + __ldg(indices + q))));
            Y[row + c * ldy] = acc;
        }
        return;
    }
    if (e - s <= L) {
        const int q = s + lane;
        const bool has = q < e;
        const double v = has ? __ldg(data + q) : 0.0;
        const int col = has ? __ldg(indices + q) : 0;
        const int cnt = e - s;
        for (int64_t c = 0; c < k; ++c) {
            const double prod = has ? __dmul_rn(v, __ldg(X + c * ldx + col)) : 0.0;
            double acc = 0.0;
            for (int u = 0; u < cnt; ++u) acc = __dadd_rn(acc, __shfl_sync(mask, prod, u, L));
            if (lane == 0) Y[row + c * ldy] = acc;
        }
    } else {
        for (int64_t c = 0; c < k; ++c) {
            const double *x = X + c * ldx;
            double acc = 0.0;
            for (int base = s; base < e; base += L) {
                const int q = base + lane;
                const double prod = q < e ? __dmul_rn(__ldg(data + q), __ldg(x + __ldg(indices + q))) : 0.0;
                const int cnt = min(L, e - base);
                for (int u = 0; u < cnt; ++u) acc = __dadd_rn(acc, __shfl_sync(mask, prod, u, L));
            }
            if (lane == 0) Y[row + c * ldy] = acc;
        }
    }
}

// Dense y = A x, one thread per row, ascending j, separately rounded
// (bitwise equal to matvec, _kernels_impl.py:24-32).  Loads of A are
// coalesced across the warp (column-major); 16 in flight per thread.
constexpr int kGemvBlock = 128;
__global__ void __launch_bounds__(kGemvBlock)
    dense_gemv_kernel(int64_t m, const double *__restrict__ A, int64_t lda,
                      const double *__restrict__ X, int64_t ldx, double *__restrict__ Y,
                      int64_t ldy) {
    const int64_t row = blockIdx.x * (int64_t)kGemvBlock + threadIdx.x;
    const double *x = X + blockIdx.y * ldx;
    if (row >= m) return;
    const double *a = A + row;
    double acc = 0.0;
    int64_t j = 0;
    constexpr int U = 16;
    for (; j + U <= m; j += U) {
        double av[U];
#pragma unroll
        for (int u = 0; u < U; ++u) av[u] = __ldg(a + (j + u) * lda);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(av[u], __ldg(x + j + u)));
    }
    for (; j < m; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(a + j * lda), __ldg(x + j)));
    Y[row + blockIdx.y * ldy] = acc;
}

// Dense Y = A X (k columns), shared-memory tiled, every output accumulated
// over ascending j with separate rounding: bitwise equal to k matvecs
// (apply_block_dense, _kernels_impl.py:35-47).
constexpr int kGemmBM = 64, kGemmBN = 64, kGemmBK = 16;
__global__ void __launch_bounds__(256)
    dense_gemm_kernel(int64_t m, int64_t k, const double *__restrict__ A, int64_t lda,
                      const double *__restrict__ X, int64_t ldx, double *__restrict__ Y,
                      int64_t ldy) {
    __shared__ double As[kGemmBK][kGemmBM + 1];
    __shared__ double Xs[kGemmBK][kGemmBN + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4x4 each
    const int64_t i0 = (int64_t)blockIdx.x * kGemmBM, c0 = (int64_t)blockIdx.y * kGemmBN;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int64_t j0 = 0; j0 < m; j0 += kGemmBK) {
        for (int e = threadIdx.x; e < kGemmBM * kGemmBK; e += 256) {
            const int ii = e % kGemmBM, jj = e / kGemmBM;
            const int64_t gi = i0 + ii, gj = j0 + jj;
            As[jj][ii] = (gi < m && gj < m) ? A[gi + gj * lda] : 0.0;
        }
        for (int e = threadIdx.x; e < kGemmBN * kGemmBK; e += 256) {
            const int jj = e % kGemmBK, cc = e / kGemmBK;
            const int64_t gj = j0 + jj, gc = c0 + cc;
            Xs[jj][cc] = (gj < m && gc < k) ? X[gj + gc * ldx] : 0.0;
        }
        __syncthreads();
        const int kmax = (m - j0) < kGemmBK ? (int)(m - j0) : kGemmBK;
        for (int jj = 0; jj < kmax; ++jj) {
            double av[4], xv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[jj][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) xv[b] = Xs[jj][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(av[a], xv[b]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gi = i0 + ty + 16 * a, gc = c0 + tx + 16 * b;
            if (gi < m && gc < k) Y[gi + gc * ldy] = acc[a][b];
        }
}

}  // namespace aqr
