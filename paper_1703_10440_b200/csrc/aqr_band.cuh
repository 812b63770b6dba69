// Banded (diagonal-offset) view of a CSR operator and the kernels that run on
// it.  A stencil operator's rows all carry the same few column offsets
// (col - row); stored as CSR, every entry costs 12 bytes of HBM traffic and a
// dependent index -> gather round trip per row.  The view keeps, per row, a
// bit mask of the offsets present (4 bytes) and either one value per diagonal
// (constant-coefficient stencils) or the values diagonal-major (nd x m), so a
// thread forms all of a row's gather addresses from its row number alone.
//
// Arithmetic: a row's sum runs over the offsets in ascending order -- the
// stored order of a CSR row with ascending column indices, which the
// analysis requires -- with the reference's separately rounded multiply and
// add (csr_matvec, _kernels_impl.py:50-56): bitwise equal to the CSR kernels
// (tests/test_gpu_band.py), and the fused step keeps the canonical norm grid.
#pragma once

#include "aqr_kernels.cuh"

namespace aqr {

constexpr int kBandMax = 32;  // == AQR_BAND_MAX (include/aqr_b200.h)

// Build knobs (A/B): diagonals per batch of gathers in the step kernel, and
// owned rows per iteration for <= 5 / 6-9 offsets (longer rows: 1).
#ifndef AQR_BAND_DB
#define AQR_BAND_DB 9
#endif
#ifndef AQR_BAND_U5
#define AQR_BAND_U5 2
#endif
#ifndef AQR_BAND_U9
#define AQR_BAND_U9 1
#endif
#ifndef AQR_BAND_PF
#define AQR_BAND_PF 1  // 1 / 2: prefetch the next row's operands into L1 / L2 (6-9 offsets); 0: off
#endif

struct BandDesc {
    int32_t nd;
    int32_t constant;
    int64_t off[kBandMax];  // ascending; off[d] = 0 for d >= nd (never selected: mask bit clear)
    double val[kBandMax];   // constant diagonals
    const uint32_t *mask;   // [m]
    const double *dvals;    // [nd][m] when !constant
};

__device__ __forceinline__ void band_prefetch(const double *p) {
#if AQR_BAND_PF == 1
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
}

struct BandArgs {
    CsrArgs c;  // indptr / indices / data unused
    BandDesc b;
};

// ---- analysis ----------------------------------------------------------------
// Pass 1: the set of distinct offsets (open-addressed table of 64 slots,
// kBandMax keys at most) and the ascending-column check.
constexpr int kBandSlots = 64;
constexpr long long kBandEmpty = (long long)0x8000000000000000ull;

struct BandScan {
    long long keys[kBandSlots];
    unsigned long long first[kBandMax];  // pass 2: first value seen per diagonal (bits)
    int32_t nkeys;
    int32_t bad;       // > kBandMax offsets, or a row with non-ascending columns
    int32_t varying;   // pass 2: a diagonal carries more than one value
};

constexpr unsigned long long kBandNoValue = 0x7ff8badc0ffee000ull;  // a NaN payload no operator carries

__global__ void band_scan_init_kernel(BandScan *sc) {
    const int t = threadIdx.x;
    if (t < kBandSlots) sc->keys[t] = kBandEmpty;
    if (t < kBandMax) sc->first[t] = kBandNoValue;
    if (t == 0) sc->nkeys = 0, sc->bad = 0, sc->varying = 0;
}

__global__ void __launch_bounds__(kBlock) band_collect_kernel(int64_t m, const int32_t *indptr, const int32_t *indices,
                                                              BandScan *sc) {
    const int64_t row = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (row >= m) return;
    if (*(volatile int32_t *)&sc->bad) return;
    const int s = __ldg(indptr + row), e = __ldg(indptr + row + 1);
    long long prev = -1;
    for (int q = s; q < e; ++q) {
        const long long c = __ldg(indices + q);
        if (c <= prev) {
            sc->bad = 1;
            return;
        }
        prev = c;
        const long long off = c - row;
        unsigned h = (unsigned)((unsigned long long)off * 0x9e3779b97f4a7c15ull >> 58);  // 6 bits
        bool done = false;
        for (int probe = 0; probe < kBandSlots && !done; ++probe, h = (h + 1) & (kBandSlots - 1)) {
            long long key = *(volatile long long *)&sc->keys[h];
            if (key == kBandEmpty) {
                key = (long long)atomicCAS((unsigned long long *)&sc->keys[h], (unsigned long long)kBandEmpty,
                                           (unsigned long long)off);
                if (key == kBandEmpty) {
                    if (atomicAdd(&sc->nkeys, 1) >= kBandMax) sc->bad = 1;
                    done = true;
                }
            }
            if (key == off) done = true;
        }
        if (!done) {
            sc->bad = 1;
            return;
        }
    }
}

// Pass 2: the row masks, and whether every diagonal carries one value.
__global__ void __launch_bounds__(kBlock) band_mask_kernel(int64_t m, const int32_t *indptr, const int32_t *indices,
                                                           const double *data, BandDesc b, uint32_t *mask,
                                                           BandScan *sc) {
    const int64_t row = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (row >= m) return;
    const int s = __ldg(indptr + row), e = __ldg(indptr + row + 1);
    uint32_t mk = 0;
    int d = 0;
    for (int q = s; q < e; ++q) {
        const long long off = (long long)__ldg(indices + q) - row;
        while (d < b.nd && b.off[d] < off) ++d;  // both ascending
        if (d >= b.nd || b.off[d] != off) {       // cannot happen after pass 1
            sc->bad = 1;
            return;
        }
        mk |= 1u << d;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(__ldg(data + q));
        unsigned long long f = *(volatile unsigned long long *)&sc->first[d];
        if (f == kBandNoValue) {
            f = atomicCAS(&sc->first[d], kBandNoValue, bits);
            if (f == kBandNoValue) f = bits;
        }
        if (f != bits || bits == kBandNoValue) sc->varying = 1;
    }
    mask[row] = mk;
}

// Varying coefficients: the values diagonal-major (absent entries 0.0, never read).
__global__ void __launch_bounds__(kBlock) band_vals_kernel(int64_t m, const int32_t *indptr, const int32_t *indices,
                                                           const double *data, BandDesc b, double *dvals) {
    const int64_t row = blockIdx.x * (int64_t)kBlock + threadIdx.x;
    if (row >= m) return;
    const int s = __ldg(indptr + row), e = __ldg(indptr + row + 1);
    int d = 0;
    for (int q = s; q < e; ++q) {
        const long long off = (long long)__ldg(indices + q) - row;
        while (d < b.nd - 1 && b.off[d] < off) ++d;
        dvals[(int64_t)d * m + row] = __ldg(data + q);
    }
}

// ---- fused HA / naive step and plain y = A x (k = 1) ----------------------------
// The canonical norm grid of csr_step_kernel: CTA b owns the 256-row blocks
// b, b+G, ..., one row per thread, the norm chains in ascending block order.
// U owned rows per iteration: their mask loads, then all gathers (addresses
// from the row number), then the sums in offset order.
// FULL: every row of the warp carries all ND offsets (interior rows of the
// grid): no predicates.
template <int ND, bool CONST, int U, bool FULL, bool UPD>
__device__ __forceinline__ void band_step_rows(const BandArgs &A, const int64_t (&row)[U], const uint32_t (&mk)[U],
                                               double rj, double &t, double &zz, double &xx) {
    constexpr bool upd = UPD;
    const CsrArgs &a = A.c;
    constexpr int DB = ND <= AQR_BAND_DB ? ND : AQR_BAND_DB;  // diagonals per batch of gathers
    double y[U], zc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        y[u] = 0.0;
        zc[u] = (FULL || row[u] < a.m) ? a.X[row[u]] : 0.0;
        if (upd) zc[u] = __dsub_rn(zc[u], __dmul_rn(rj, (FULL || row[u] < a.m) ? a.qprev[row[u]] : 0.0));
    }
#pragma unroll
    for (int d0 = 0; d0 < ND; d0 += DB) {
        double xv[U][DB];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int h = 0; h < DB; ++h) {
                const bool has = d0 + h < ND && (FULL || (mk[u] >> (d0 + h) & 1u));
                xv[u][h] = has ? __ldg(a.X + row[u] + A.b.off[(d0 + h) % ND]) : 0.0;
            }
        if (upd) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                double qv[DB];
#pragma unroll
                for (int h = 0; h < DB; ++h) {
                    const bool has = d0 + h < ND && (FULL || (mk[u] >> (d0 + h) & 1u));
                    qv[h] = has ? __ldg(a.qprev + row[u] + A.b.off[(d0 + h) % ND]) : 0.0;
                }
#pragma unroll
                for (int h = 0; h < DB; ++h) xv[u][h] = __dsub_rn(xv[u][h], __dmul_rn(rj, qv[h]));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int h = 0; h < DB; ++h)
                if (d0 + h < ND && (FULL || (mk[u] >> (d0 + h) & 1u))) {
                    const int d = (d0 + h) % ND;
                    const double v = CONST ? A.b.val[d] : __ldg(A.b.dvals + (int64_t)d * a.m + row[u]);
                    y[u] = __dadd_rn(y[u], __dmul_rn(v, xv[u][h]));
                }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (!FULL && row[u] >= a.m) continue;
        a.Y[row[u]] = y[u];
        if (a.znew) a.znew[row[u]] = zc[u];
        t = fma(zc[u], y[u], t);
        zz = fma(zc[u], zc[u], zz);
        xx = fma(y[u], y[u], xx);
    }
}

template <int ND, bool CONST, int U, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) band_step_kernel(BandArgs A) {
    const CsrArgs &a = A.c;
    trace_mark(a.trace, 0);
    const int64_t G = gridDim.x, cta = blockIdx.x;
    const int64_t stride = G * kBlock;
    int64_t row[U];
    uint32_t mk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // the operator is read-only: masks before the dependency wait
        row[u] = (cta + u * G) * kBlock + threadIdx.x;
        mk[u] = row[u] < a.m ? __ldg(A.b.mask + row[u]) : 0u;
    }
    pdl_wait();
    trace_mark(a.trace, 1);
    if (failed(a.out.status)) return;
    const bool upd = a.r != nullptr;
    const double rj = a.rin.partial ? rrow_first(a.rin, cta == 0) : (upd ? *a.r : 0.0);
    const int64_t nblk = (a.m + kBlock - 1) / kBlock;
    const uint32_t full = A.b.nd >= 32 ? 0xffffffffu : (1u << A.b.nd) - 1u;
    double t = 0.0, zz = 0.0, xx = 0.0;
    for (int64_t blk = cta; blk < nblk; blk += (int64_t)U * G) {
        int64_t nrow[U];
        uint32_t nmk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            nrow[u] = row[u] + U * stride;
            nmk[u] = nrow[u] < a.m ? __ldg(A.b.mask + nrow[u]) : 0u;
        }
#if AQR_BAND_PF
        // one row per iteration (6-9 offsets): the next owned row's operands on
        // their way into the cache while this row's gathers are in flight (rows
        // whose whole offset range lies inside the vector; the others just
        // miss).  Config 3 fused step 57 -> 53 us (L1 and L2 alike); with two
        // rows per iteration (<= 5 offsets) it costs: config 2 19.2 -> 21.2 us.
        if (U == 1 && ND <= 9) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (nrow[u] + A.b.off[0] >= 0 && nrow[u] + A.b.off[(ND - 1) % kBandMax] < a.m &&
                    A.b.off[(ND - 1) % kBandMax] != 0) {
#pragma unroll
                    for (int d = 0; d < ND; ++d) {
                        band_prefetch(a.X + nrow[u] + A.b.off[d]);
                        if (upd) band_prefetch(a.qprev + nrow[u] + A.b.off[d]);
                        if (!CONST) band_prefetch(A.b.dvals + (int64_t)d * a.m + nrow[u]);
                    }
                }
        }
#endif
        // interior warps of short stencils skip the predicates (config 2 fused
        // step 21.0 -> 19.2 us, config 3 65 -> 57 us); with 27 offsets the two
        // unrolled paths spill and the step is slower (98 -> 117 ms on config 5)
        bool fullw = ND <= 9 && A.b.nd == ND;
#pragma unroll
        for (int u = 0; u < U; ++u) fullw &= mk[u] == full;
        if (ND <= 9 && __all_sync(0xffffffffu, fullw)) {
            if (upd) band_step_rows<ND, CONST, U, true, true>(A, row, mk, rj, t, zz, xx);
            else band_step_rows<ND, CONST, U, true, false>(A, row, mk, rj, t, zz, xx);
        } else {
            if (upd) band_step_rows<ND, CONST, U, false, true>(A, row, mk, rj, t, zz, xx);
            else band_step_rows<ND, CONST, U, false, false>(A, row, mk, rj, t, zz, xx);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) row[u] = nrow[u], mk[u] = nmk[u];
    }
    pdl_trigger();
    if (a.out.npart != nullptr) {  // uniform; nullptr: plain y = A x
        norm_cta_partial(a.out, t, zz, xx, cta);
        norm_last_cta(a.out, (unsigned)G);
    }
    rrow_rest(a.rin, cta, G);
    trace_mark(a.trace, 2);
}

// ---- Y = A X, k >= 2 columns (HP block apply) -----------------------------------
// CTA = (256-row block, K columns), launch order as csr_spmm2_kernel
// (super-groups of column blocks so the rows of X a super-group gathers stay
// in L2 while the row front advances); thread = (row, K columns), the
// diagonals in batches of DB (DB x K gathers in flight).
template <int ND, bool CONST, int K, int DB, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) band_spmm_kernel(BandArgs A) {
    const CsrArgs &a = A.c;
    const int64_t ncb = (a.k + K - 1) / K;
    const int64_t nrb = (a.m + kBlock - 1) / kBlock;
    const int64_t sg = (a.sg > 0 && a.sg < ncb) ? a.sg : ncb;
    const int64_t per_sg = sg * nrb;
    const int64_t g = blockIdx.x / per_sg, rest = blockIdx.x - g * per_sg;
    const int64_t w = min(sg, ncb - g * sg);
    const int64_t rb = rest / w, cb = g * sg + rest % w;
    const int64_t row = rb * kBlock + threadIdx.x;
    const int64_t col0 = cb * K;
    if (row >= a.m) return;
    const uint32_t mk = __ldg(A.b.mask + row);
    double acc[K];
#pragma unroll
    for (int kk = 0; kk < K; ++kk) acc[kk] = 0.0;
    const double *xb = a.X + col0 * a.ldx + row;
    int64_t coff[K];  // a clamped column re-reads the block's first column; its sums are not stored
#pragma unroll
    for (int kk = 0; kk < K; ++kk) coff[kk] = (col0 + kk < a.k ? (int64_t)kk : 0) * a.ldx;
#pragma unroll
    for (int d0 = 0; d0 < ND; d0 += DB) {
        double xv[K][DB], v[DB];
#pragma unroll
        for (int h = 0; h < DB; ++h) {
            const int d = d0 + h;
            const bool ok = d < ND && (mk >> d & 1u);
            v[h] = !ok ? 0.0 : (CONST ? A.b.val[d < ND ? d : 0] : __ldg(A.b.dvals + (int64_t)d * a.m + row));
#pragma unroll
            for (int kk = 0; kk < K; ++kk) xv[kk][h] = ok ? __ldg(xb + A.b.off[d < ND ? d : 0] + coff[kk]) : 0.0;
        }
#pragma unroll
        for (int h = 0; h < DB; ++h) {
            const int d = d0 + h;
            if (d < ND && (mk >> d & 1u)) {
#pragma unroll
                for (int kk = 0; kk < K; ++kk) acc[kk] = __dadd_rn(acc[kk], __dmul_rn(v[h], xv[kk][h]));
            }
        }
    }
#pragma unroll
    for (int kk = 0; kk < K; ++kk)
        if (col0 + kk < a.k) a.Y[row + (col0 + kk) * a.ldy] = acc[kk];
}

// ---- staged tiles: Y = A X with long rows (27-point stencils) ----------------------
// With many offsets per row the gather kernel above is bound by instruction
// issue and the L1 data path (27 8-byte gathers per row and column).  A
// block of NB consecutive rows needs, per offset d, the NB consecutive
// elements x[r0 + off_d ..]; offsets closer than NB apart overlap, so the
// union is a few contiguous segments (a 27-point stencil on an n^3 grid
// with NB >= n: three, one per grid plane).  The CTA copies the segments of
// a column into shared memory with asynchronous copies (cp.async, no
// registers), double-buffered so the next column's copies run under the
// current column's arithmetic, and every row reads its operands from there
// (one shared-memory load per operand, its address a per-offset constant
// plus the thread's base).  Same operands, same order, same rounding as the
// gather kernels.
constexpr int kBandSegMax = 8;

struct BandStage {
    int32_t nseg;
    int32_t total;                // doubles of shared memory per buffer
    int64_t lo[kBandSegMax];      // first offset of the segment (relative to r0)
    int32_t len[kBandSegMax];     // elements staged
    int32_t base[kBandSegMax];    // shared-memory index of the segment
    int32_t sbyte[kBandMax];      // shared-memory byte offset of (row r0, offset d)
};

struct BandTileArgs {
    CsrArgs c;
    BandDesc b;
    BandStage st;
};

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issues the copies of one column's segments for the row block at r0.
// Elements outside [0, m) are skipped: no row reads them (its mask bit for
// that offset is clear).
__device__ __forceinline__ void band_stage_async(const BandStage &st, const double *__restrict__ x, int64_t r0,
                                                 int64_t m, double *sm, bool inside) {
    for (int s = 0; s < st.nseg; ++s) {
        const int64_t g0 = r0 + st.lo[s];
        const double *src = x + g0;
        double *dst = sm + st.base[s];
        const int len = st.len[s];
        if (inside) {
#pragma unroll 4
            for (int e = threadIdx.x; e < len; e += kBlock) cp_async8(dst + e, src + e);
        } else {
            for (int e = threadIdx.x; e < len; e += kBlock)
                if (g0 + e >= 0 && g0 + e < m) cp_async8(dst + e, src + e);
        }
    }
}

// CTA = (block of RPT x 256 rows, KC columns), thread = rows tid + 256 i of
// the block.  Launch order as csr_spmm2_kernel (super-groups of a.sg column
// groups).
template <int ND, bool CONST, int RPT, int KC, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) band_spmm_tile_kernel(BandTileArgs A) {
    extern __shared__ double band_sm[];  // two buffers of st.total doubles
    const CsrArgs &a = A.c;
    constexpr int NB = RPT * kBlock;
    const int64_t ncb = (a.k + KC - 1) / KC;
    const int64_t nrb = (a.m + NB - 1) / NB;
    const int64_t sg = (a.sg > 0 && a.sg < ncb) ? a.sg : ncb;
    const int64_t per_sg = sg * nrb;
    const int64_t g = blockIdx.x / per_sg, rest = blockIdx.x - g * per_sg;
    const int64_t w = min(sg, ncb - g * sg);
    const int64_t rb = rest / w, cb = g * sg + rest % w;
    const int64_t r0 = rb * NB;
    uint32_t mk[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int64_t row = r0 + threadIdx.x + i * kBlock;
        mk[i] = row < a.m ? __ldg(A.b.mask + row) : 0u;
    }
    const uint32_t full = A.b.nd >= 32 ? 0xffffffffu : (1u << A.b.nd) - 1u;
    bool interior = A.b.nd == ND;  // the unpredicated path runs all ND offsets
#pragma unroll
    for (int i = 0; i < RPT; ++i) interior &= mk[i] == full;
    interior = __all_sync(0xffffffffu, interior);  // one path per warp
    const int last = A.st.nseg - 1;
    const bool inside = r0 + A.st.lo[0] >= 0 && r0 + A.st.lo[last] + A.st.len[last] <= a.m;
    const int64_t cend = min(a.k, (cb + 1) * KC);
    int64_t col = cb * KC;
    band_stage_async(A.st, a.X + col * a.ldx, r0, a.m, band_sm, inside);
    cp_async_commit();
    for (int c = 0; col < cend; ++col, ++c) {
        double *buf = band_sm + (c & 1) * A.st.total;
        if (col + 1 < cend)
            band_stage_async(A.st, a.X + (col + 1) * a.ldx, r0, a.m, band_sm + ((c & 1) ^ 1) * A.st.total, inside);
        cp_async_commit();
        cp_async_wait<1>();  // this column's copies (all groups but the newest) have landed
        __syncthreads();
        const char *sp0 = reinterpret_cast<const char *>(buf + threadIdx.x);
        double y[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) y[i] = 0.0;
        if (interior) {  // all of this thread's rows carry every offset: no predicates
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                const double *sp = reinterpret_cast<const double *>(sp0 + A.st.sbyte[d]);
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const double v = CONST ? A.b.val[d]
                                           : __ldg(A.b.dvals + (int64_t)d * a.m + r0 + threadIdx.x + i * kBlock);
                    y[i] = __dadd_rn(y[i], __dmul_rn(v, sp[i * kBlock]));
                }
            }
        } else {  // branch-free: the sum is formed and kept only where the entry exists
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                const double *sp = reinterpret_cast<const double *>(sp0 + A.st.sbyte[d]);
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const bool has = mk[i] >> d & 1u;
                    const double v = CONST ? A.b.val[d]
                                           : (has ? __ldg(A.b.dvals + (int64_t)d * a.m + r0 + threadIdx.x + i * kBlock)
                                                  : 0.0);
                    const double yn = __dadd_rn(y[i], __dmul_rn(v, sp[i * kBlock]));
                    y[i] = has ? yn : y[i];
                }
            }
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int64_t row = r0 + threadIdx.x + i * kBlock;
            if (row < a.m) a.Y[row + col * a.ldy] = y[i];
        }
        __syncthreads();  // the buffer is free for the column after next
    }
}

}  // namespace aqr
