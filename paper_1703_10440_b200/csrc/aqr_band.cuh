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

struct BandDesc {
    int32_t nd;
    int32_t constant;
    int64_t off[kBandMax];  // ascending; off[d] = 0 for d >= nd (never selected: mask bit clear)
    double val[kBandMax];   // constant diagonals
    const uint32_t *mask;   // [m]
    const double *dvals;    // [nd][m] when !constant
};

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
template <int ND, bool CONST, int U>
__device__ __forceinline__ void band_step_rows(const BandArgs &A, const int64_t (&row)[U], const uint32_t (&mk)[U],
                                               bool upd, double rj, double &t, double &zz, double &xx) {
    const CsrArgs &a = A.c;
    constexpr int DB = ND <= 9 ? ND : 9;  // diagonals per batch of gathers
    double y[U], zc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        y[u] = 0.0;
        zc[u] = row[u] < a.m ? a.X[row[u]] : 0.0;
        if (upd) zc[u] = __dsub_rn(zc[u], __dmul_rn(rj, row[u] < a.m ? a.qprev[row[u]] : 0.0));
    }
#pragma unroll
    for (int d0 = 0; d0 < ND; d0 += DB) {
        double xv[U][DB];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int h = 0; h < DB; ++h)
                xv[u][h] = (d0 + h < ND && (mk[u] >> (d0 + h) & 1u)) ? __ldg(a.X + row[u] + A.b.off[(d0 + h) % ND]) : 0.0;
        if (upd) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                double qv[DB];
#pragma unroll
                for (int h = 0; h < DB; ++h)
                    qv[h] = (d0 + h < ND && (mk[u] >> (d0 + h) & 1u)) ? __ldg(a.qprev + row[u] + A.b.off[(d0 + h) % ND])
                                                                      : 0.0;
#pragma unroll
                for (int h = 0; h < DB; ++h) xv[u][h] = __dsub_rn(xv[u][h], __dmul_rn(rj, qv[h]));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int h = 0; h < DB; ++h)
                if (d0 + h < ND && (mk[u] >> (d0 + h) & 1u)) {
                    const int d = (d0 + h) % ND;
                    const double v = CONST ? A.b.val[d] : __ldg(A.b.dvals + (int64_t)d * a.m + row[u]);
                    y[u] = __dadd_rn(y[u], __dmul_rn(v, xv[u][h]));
                }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (row[u] >= a.m) continue;
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
    double t = 0.0, zz = 0.0, xx = 0.0;
    for (int64_t blk = cta; blk < nblk; blk += (int64_t)U * G) {
        int64_t nrow[U];
        uint32_t nmk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            nrow[u] = row[u] + U * stride;
            nmk[u] = nrow[u] < a.m ? __ldg(A.b.mask + nrow[u]) : 0u;
        }
        band_step_rows<ND, CONST, U>(A, row, mk, upd, rj, t, zz, xx);
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

}  // namespace aqr
