// aqr_kernels.cuh -- sm_100a device kernels of the A-orthogonal MGS hot path.
//
// Layout: column-major fp64 matrices with explicit leading dimension; CSR
// with int32 indptr/indices and fp64 values.
//
// Determinism.  Every reduction is atomic-free in its arithmetic and depends
// only on m (never on the step, variant, orientation, grid size or column
// grouping):
//   * rows are cut into tiles of tile_rows(m) = 256 * RPT rows; thread k of a
//     tile owns rows k + 256 u (u = 0..RPT-1), accumulates them in ascending u
//     with fma, the warp reduces with an xor butterfly (16, 8, 4, 2, 1) and the
//     8 warps are added in ascending order -> one partial per (tile, column);
//   * the norm partials (z.x, z.z, x.x): per-CTA chains over a fixed grid
//     (norm_tiles), one block tree per CTA;
//   * a column total over tiles is block_totals(): thread k adds the tiles
//     k, k+256, k+512, ... in ascending order, then the warp xor butterfly
//     and the 8 warps in ascending order.
// Every kernel that produces or consumes these partials uses exactly these
// functions, so the row- and column-oriented schedules, the native and the
// callback operator routes and the step API all return bitwise-identical
// factors, the property the reference guarantees for its sequential loops
// (gram_schmidt.py:19-21).  Atomics are used only as completion tickets
// ("last CTA finishes"), never to accumulate values.
//
// Elementwise updates follow the reference exactly: z -= a*q is a rounded
// multiply then a rounded subtract (__dmul_rn/__dsub_rn, no FMA contraction;
// _kernels_impl.py:85-88), x / r is an IEEE division (:91-93).  Operator
// products accumulate in the reference's order with separate rounding
// (_kernels_impl.py:24-56) and are therefore bitwise equal to it.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace aqr {

// Columns of the register-resident-row SpMM in flight per thread (build knob;
// config 2 HP block apply 366 / 352 / 582 us at 2 / 4 / 8 with the gathers of
// a column block issued before its stores; 480 us before that)
#ifndef AQR_SPMM_UNROLL
#define AQR_SPMM_UNROLL 4
#endif
constexpr int kSpmmUnroll = AQR_SPMM_UNROLL;

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

// Rows per thread of the reduction tile: depends on m only (build-time
// AQR_BIG_RPT for the large-m tile, 8 -> 2048-row tiles).
#ifndef AQR_BIG_RPT
#define AQR_BIG_RPT 8
#endif
constexpr int kBigRpt = AQR_BIG_RPT;
constexpr int kBigCu = kBigRpt >= 8 ? 2 : 4;  // columns per iteration of the windowed pass at that tile
__host__ __device__ inline int rows_per_thread(int64_t m) {
    return m >= (int64_t)2048 * 148 ? kBigRpt : 1;
}
__host__ __device__ inline int64_t tile_rows(int64_t m) { return (int64_t)kBlock * rows_per_thread(m); }
__host__ __device__ inline int64_t num_tiles(int64_t m) {
    const int64_t t = tile_rows(m);
    return (m + t - 1) / t;
}
// The norm partials (z.x, z.z, x.x) are formed by a FIXED grid of
// norm_tiles(m, hp) = min(ceil(m/256), G) CTAs, G depending only on the
// variant: CTA b owns the 256-row blocks b, b+G, b+2G, ...; thread k
// accumulates (fma) its row k of each owned block in ascending block order;
// one block tree (warp xor butterfly, warps ascending) per CTA gives partial
// b.  Totals are block_totals over the G partials.  G is one wave of the
// kernel that forms the partials: 3 CTAs/SM for the software-pipelined
// fused SpMV step (HA / naive), 4 CTAs/SM for the HP column update.
#ifndef AQR_SPMV_MINB
#define AQR_SPMV_MINB 3  // resident fused-SpMV CTAs per SM (the HA norm grid is this x 148)
#endif
#ifndef AQR_NORM_GRID_HA
#define AQR_NORM_GRID_HA (148 * 3)
#endif
#ifndef AQR_NORM_GRID_HP
#define AQR_NORM_GRID_HP (148 * 4)
#endif
constexpr int kNormGridHA = AQR_NORM_GRID_HA;
constexpr int kNormGridHP = AQR_NORM_GRID_HP;
constexpr int kNormGridMax = kNormGridHA > kNormGridHP ? kNormGridHA : kNormGridHP;
__host__ __device__ inline int64_t norm_tiles(int64_t m, bool hp) {
    const int64_t b = (m + kBlock - 1) / kBlock;
    const int64_t g = hp ? kNormGridHP : kNormGridHA;
    return b < g ? b : g;
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start (launch, prologue) while
// its predecessor drains; pdl_wait() blocks until the predecessor grid has
// completed and its memory is visible, pdl_trigger() lets the successor
// launch.  Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Diagnostics (compiled in with -DAQR_TRACE): per-launch first-CTA start /
// last-CTA end from %globaltimer, to measure the gaps between kernels.
#ifdef AQR_TRACE
__device__ unsigned long long *g_trace = nullptr;  // [slot][3]: pre-wait start, start, end
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_mark(int32_t slot, int which) {
    if (slot < 0 || g_trace == nullptr || threadIdx.x != 0) return;
    if (which < 2) atomicMin(g_trace + 3 * slot + which, gtimer());
    else atomicMax(g_trace + 3 * slot + 2, gtimer());
}
#else
__device__ __forceinline__ void trace_mark(int32_t, int) {}
#endif

__device__ __forceinline__ bool failed(const int32_t *status) {
    return status != nullptr && *(volatile const int32_t *)status >= 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Warp totals of 8 values per lane (8 columns) at once, by a transposed
// butterfly: round 1 (xor 16) keeps 4 columns per lane, round 2 (xor 8) 2,
// round 3 (xor 4) 1, rounds 4-5 (xor 2, 1) finish.  Every column is summed
// over the same hypercube tree as warp_sum (16, 8, 4, 2, 1 -- IEEE addition
// is commutative), so the totals are bitwise warp_sum's, with 9 shuffles
// instead of 40.  Lane l returns the total of column (l >> 2).
__device__ __forceinline__ double warp_sum8(const double (&v)[8]) {
    const int lane = threadIdx.x & 31;
    const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
    double a4[4], a2[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double keep = b4 ? v[4 + k] : v[k], send = b4 ? v[k] : v[4 + k];
        a4[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double keep = b3 ? a4[2 + k] : a4[k], send = b3 ? a4[k] : a4[2 + k];
        a2[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    }
    const double keep = b2 ? a2[1] : a2[0], send = b2 ? a2[0] : a2[1];
    double c = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
    c = __dadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 2));
    c = __dadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 1));
    return c;
}

// Same for 4 columns (xor 16 keeps 2, xor 8 keeps 1, then 4, 2, 1); lane l
// returns the total of column (l >> 3).
__device__ __forceinline__ double warp_sum4(const double (&v)[4]) {
    const int lane = threadIdx.x & 31;
    const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1;
    double a2[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double keep = b4 ? v[2 + k] : v[k], send = b4 ? v[k] : v[2 + k];
        a2[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
    const double keep = b3 ? a2[1] : a2[0], send = b3 ? a2[0] : a2[1];
    double c = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    c = __dadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 4));
    c = __dadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 2));
    c = __dadd_rn(c, __shfl_xor_sync(0xffffffffu, c, 1));
    return c;
}

template <int NB>
__device__ __forceinline__ double warp_sum_batch(const double (&v)[NB]);
template <>
__device__ __forceinline__ double warp_sum_batch<8>(const double (&v)[8]) { return warp_sum8(v); }
template <>
__device__ __forceinline__ double warp_sum_batch<4>(const double (&v)[4]) { return warp_sum4(v); }

// Fixed-order block sum over kBlock threads; every thread returns the value.
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

// Canonical total of NC partial arrays p + c * stride (c < NC), each of n
// tile partials: thread k (k < 256) adds the tiles k, k+256, k+512, ... in
// ascending order, the warp reduces with the xor butterfly and the 8 warps
// are added in ascending order.  Called by threads 0..255 of the CTA (the
// other threads must not call it); `bar` is the barrier those 256 threads
// share (__syncthreads, or a named barrier in warp-specialized kernels).
// Loads are issued 4 per chain ahead of the adds, so even 8192 tiles cost
// only a few dependent L2 round trips.
// H: tiles per column loaded together per iteration (registers vs round
// trips; the sum order -- ascending t -- does not depend on it).
template <int NC, typename Bar, int H = 4>
__device__ __forceinline__ void block_totals(const double *p, int64_t stride, int32_t n,
                                             double *out /* smem or global, NC */,
                                             double *sm /* NC * kWarps */, Bar bar) {
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    for (int t0 = threadIdx.x; t0 < n; t0 += H * kBlock) {
        double v[NC][H];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int t = t0 + h * kBlock;
                v[c][h] = t < n ? __ldcg(p + c * stride + t) : 0.0;
            }
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int h = 0; h < H; ++h)
                if (t0 + h * kBlock < n) acc[c] = __dadd_rn(acc[c], v[c][h]);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const double w = warp_sum(acc[c]);
        if (lane == 0) sm[c * kWarps + warp] = w;
    }
    bar();
    if (threadIdx.x < NC) {
        double s = sm[threadIdx.x * kWarps];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) s = __dadd_rn(s, sm[threadIdx.x * kWarps + w]);
        out[threadIdx.x] = s;
    }
    bar();
}

struct SyncAll {
    __device__ void operator()() const { __syncthreads(); }
};

// Status block: int32 fail column at [0], double fail value at byte 8,
// int32 flags[n] at byte 16.
__device__ __forceinline__ void norm_finish_dev(int64_t i, double t, double zz, double xx,
                                                double *rii, int32_t *status) {
    if (!(t > 0.0) || !isfinite(t)) {  // gram_schmidt.py:153-154
        if (status[0] < 0) {
            status[0] = (int32_t)i;
            *reinterpret_cast<double *>(status + 2) = t;
        }
        return;
    }
    const double unit_roundoff = 1.1102230246251565e-16;  // 2**-53, gram_schmidt.py:33
    const double nz = sqrt(zz), nx = sqrt(xx);
    if (t < 100.0 * unit_roundoff * nz * nx) status[4 + i] = 1;  // gram_schmidt.py:155-158
    *rii = sqrt(t);                                               // gram_schmidt.py:159
}

// Block-wide "am I the last CTA" ticket (all kBlock threads call it; the
// CTA's partials were written by thread 0, which alone fences before taking
// the ticket -- the other warps retire without waiting for their stores).
// Resets the counter when it fires.
__device__ __forceinline__ bool last_block(unsigned *counter, unsigned expected) {
    __shared__ unsigned ticket;
    if (threadIdx.x == 0) {
        // release: thread 0's partial stores are ordered before the ticket
        // (the other warps' stores are consumed by the next kernel only);
        // cheaper than a full fence.sc, which also waits for those
        unsigned tk;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(tk) : "l"(counter) : "memory");
        ticket = tk;
    }
    __syncthreads();
    const bool last = ticket == expected - 1;
    if (last) {
        __threadfence();
        if (threadIdx.x == 0) *counter = 0u;
    }
    return last;
}

// The three norm partials of a tile -> npart, and the last CTA finishes:
// totals (tot, optional) and the breakdown / flag / r_ii record.
struct NormOut {
    double *npart;  // [3 * ntiles] or nullptr
    int32_t ntiles;
    unsigned *counter;  // nullptr: no finish in-kernel
    double *tot;        // optional totals
    double *rii;        // optional: finish (breakdown check, flag, sqrt)
    int64_t step;
    int32_t *status;
};

// Norm partial of this CTA (all kBlock threads call it once, with their
// accumulated chains): block tree, then partial blockIdx.x of each term.
__device__ __forceinline__ void norm_cta_partial(const NormOut &o, double t, double zz, double xx,
                                                 int64_t cta) {
    __shared__ double sm[3 * kWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    t = warp_sum(t);
    zz = warp_sum(zz);
    xx = warp_sum(xx);
    if (lane == 0) {
        sm[0 * kWarps + warp] = t;
        sm[1 * kWarps + warp] = zz;
        sm[2 * kWarps + warp] = xx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // thread 0 writes all three (see last_block)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double s = sm[c * kWarps];
#pragma unroll
            for (int w = 1; w < kWarps; ++w) s = __dadd_rn(s, sm[c * kWarps + w]);
            o.npart[(int64_t)c * o.ntiles + cta] = s;
        }
    }
}

// After a CTA wrote all its tiles' partials: the last CTA of the grid forms
// the totals (block_totals) and finishes the column (one ticket per CTA).
// Called by all kBlock threads.
__device__ __forceinline__ void norm_last_cta(const NormOut &o, unsigned ctas) {
    if (o.counter == nullptr) return;
    if (!last_block(o.counter, ctas)) return;
    __shared__ double tot[3];
    __shared__ double sm3[3 * kWarps];
    block_totals<3>(o.npart, o.ntiles, o.ntiles, tot, sm3, SyncAll());
    if (threadIdx.x == 0) {
        if (o.tot) {
            o.tot[0] = tot[0];
            o.tot[1] = tot[1];
            o.tot[2] = tot[2];
        }
        if (o.rii) norm_finish_dev(o.step, tot[0], tot[1], tot[2], o.rii, o.status);
    }
}

// Deferred r-row totals.  The trailing pass of step i-1 leaves per-tile
// partials of r_{i-1,j}, j = i .. n-1; instead of a separate reduction
// launch, the next norm kernel (step i) forms them: every CTA reduces column
// i (r_{i-1,i} is needed by all of its rows) and CTA b >= 1 also reduces
// column i+b.  Same block_totals tree as rrow_reduce_kernel: bitwise equal.
struct RrowIn {
    const double *partial;  // [ncols][ntiles]; nullptr: r_{i-1,i} is read from *r
    int32_t ntiles, ncols;
    double *rrow;  // rrow[b] = Rt[i-1][i+b]
};

__device__ __forceinline__ double rrow_first(const RrowIn &in, bool writer) {
    __shared__ double tot1[1];
    __shared__ double sm1[kWarps];
    block_totals<1>(in.partial, in.ntiles, in.ntiles, tot1, sm1, SyncAll());
    const double r = tot1[0];
    if (writer && threadIdx.x == 0) in.rrow[0] = r;
    return r;
}

// CTA `cta` of `G` reduces columns cta, cta + G, ... (column 0 excluded).
__device__ __forceinline__ void rrow_rest(const RrowIn &in, int64_t cta, int64_t G) {
    if (in.partial == nullptr) return;
    __shared__ double sm1[kWarps];
    for (int64_t b = cta; b < in.ncols; b += G)
        if (b >= 1)
            block_totals<1>(in.partial + b * in.ntiles, in.ntiles, in.ntiles, in.rrow + b, sm1, SyncAll());
}

// ---------------------------------------------------------------------------
// Column update (deferred step i-1 projection of column i) + norm partials
// ---------------------------------------------------------------------------
struct ColArgs {
    int64_t m;
    double *z;
    const double *zsrc;  // read z from here instead of z (nullptr: z); results go to z
    const double *qprev;
    double *x;  // HP: carried column, updated in place (nullptr otherwise)
    const double *pprev;
    const double *r;      // r_{i-1,i} (nullptr: no update)
    const double *xnorm;  // x used for the norm partials when x == nullptr
    NormOut out;          // out.npart == nullptr: update only
    RrowIn rin;           // deferred r-row totals (rin.partial == nullptr: none)
    int32_t trace;        // AQR_TRACE builds: launch slot (-1 off)
    // col_lazy_norm_kernel (HP, row form): x_j = X_j - sum_k r_{k,j} p_k
    const double *P;      // p_0 .. p_{j-1}, ld ldp
    int64_t ldp;
    const double *rcol;   // r_{k,j} = rcol[k * rstride], k < j - 1 (final totals)
    int64_t rstride;
    int32_t nprev;        // j
    double *xout;         // x_j goes here (X_j itself is only read)
};

// Column update (+ norm chains when out.npart): launched with exactly
// norm_tiles(m, hp) CTAs (the canonical norm grid of the variant); kColTiles owned blocks are
// processed per iteration with all their loads in flight, rows accumulated
// in ascending block order.
#ifndef AQR_COL_TILES
#define AQR_COL_TILES 4
#endif
constexpr int kColTiles = AQR_COL_TILES;
__global__ void __launch_bounds__(kBlock, 4) col_update_norm_kernel(ColArgs a) {
    trace_mark(a.trace, 0);
    pdl_wait();
    trace_mark(a.trace, 1);
    if (failed(a.out.status)) return;
    const bool upd = a.r != nullptr;
    const int64_t nblk = (a.m + kBlock - 1) / kBlock;
    const int64_t G = gridDim.x;
    double t = 0.0, zz = 0.0, xx = 0.0;
    double z[kColTiles], xv[kColTiles], q[kColTiles], pp[kColTiles];
    auto load = [&](int64_t b0) {  // loads first
#pragma unroll
        for (int g = 0; g < kColTiles; ++g) {
            const int64_t r = (b0 + g * G) * kBlock + threadIdx.x;
            const bool ok = b0 + g * G < nblk && r < a.m;
            z[g] = ok ? (a.zsrc ? a.zsrc[r] : a.z[r]) : 0.0;
            q[g] = (ok && upd) ? a.qprev[r] : 0.0;
            xv[g] = ok ? (a.x ? a.x[r] : (a.xnorm ? a.xnorm[r] : 0.0)) : 0.0;
            pp[g] = (ok && upd && a.x) ? a.pprev[r] : 0.0;
        }
    };
    // the first batch is in flight while the r-row total forms (it does not
    // depend on r_{i-1,i})
    if (blockIdx.x < nblk) load(blockIdx.x);
    const double rj = a.rin.partial ? rrow_first(a.rin, blockIdx.x == 0) : (upd ? *a.r : 0.0);
    for (int64_t b0 = blockIdx.x; b0 < nblk; b0 += G * kColTiles) {
        if (b0 != blockIdx.x) load(b0);
#pragma unroll
        for (int g = 0; g < kColTiles; ++g) {
            const int64_t r = (b0 + g * G) * kBlock + threadIdx.x;
            const bool ok = b0 + g * G < nblk && r < a.m;
            if (upd) {
                z[g] = __dsub_rn(z[g], __dmul_rn(rj, q[g]));
                if (ok) a.z[r] = z[g];
                if (a.x) {
                    xv[g] = __dsub_rn(xv[g], __dmul_rn(rj, pp[g]));
                    if (ok) a.x[r] = xv[g];
                }
            }
            if (ok) {
                t = fma(z[g], xv[g], t);
                zz = fma(z[g], z[g], zz);
                xx = fma(xv[g], xv[g], xx);
            }
        }
    }
    pdl_trigger();
    if (a.out.npart != nullptr) {  // uniform
        norm_cta_partial(a.out, t, zz, xx, blockIdx.x);
        norm_last_cta(a.out, gridDim.x);
    }
    rrow_rest(a.rin, blockIdx.x, gridDim.x);
    trace_mark(a.trace, 2);
}

// HP, row form, with X read-only after the block apply.  project(k, j)
// (gram_schmidt.py:139-145) updates X[:, j] at every step k < j, but
// normalize(j) (:148-149) is the only reader of X[:, j]: here x_j is formed
// when it is needed, X_j - r_{0,j} p_0 - r_{1,j} p_1 - ... - r_{j-1,j} p_{j-1},
// in ascending k with the separately rounded multiply and subtract of the
// reference's sub_scaled -- the very sequence of roundings the eager updates
// would have applied, so the bits are unchanged.  Per step this reads the j
// finished p columns (8 m j bytes) instead of reading and writing the n-1-j
// trailing X columns at every step (16 m (n-1-j)): over the factorization
// the X traffic halves and the whole HP step traffic drops by a quarter.
// Also: the deferred update of z_j (r_{j-1,j} q_{j-1}), the norm partials
// (z.x, z.z, x.x) on the canonical HP norm grid (same per-thread chains as
// col_update_norm_kernel) and x_j -> a.xout for the trailing pass.
constexpr int kLazyBlk = 4;    // owned 256-row blocks per load batch
constexpr int kLazyK = 4;      // p columns per batch of loads
constexpr int kLazyRs = 1024;  // r_{k,j} staged in shared memory per chunk
// The body: x_j formed, z_j's deferred update (rj), x_j -> a.xout, the
// thread's norm chains (t, zz, xx) returned.  All kBlock threads.
__device__ __forceinline__ void col_lazy_body(const ColArgs &a, double rj, bool upd, double &t, double &zz,
                                              double &xx) {
    __shared__ double rs[kLazyRs];
    const int32_t nk = a.nprev;  // lazy terms k = j - nk .. j-1 (X_j holds x_j^(j - nk))
    const int64_t nblk = (a.m + kBlock - 1) / kBlock;
    const int64_t G = gridDim.x;
    auto stage = [&](int kc, int kn) {
        for (int k = threadIdx.x; k < kn; k += kBlock)
            rs[k] = (kc + k == nk - 1 && upd) ? rj : __ldcg(a.rcol + (int64_t)(kc + k) * a.rstride);
    };
    const bool one_chunk = nk <= kLazyRs;
    if (one_chunk) stage(0, nk);
    __syncthreads();
    t = zz = xx = 0.0;
    for (int64_t b0 = blockIdx.x; b0 < nblk; b0 += G * kLazyBlk) {
        int64_t row[kLazyBlk];
        bool ok[kLazyBlk];
        double z[kLazyBlk], x[kLazyBlk], q[kLazyBlk];
#pragma unroll
        for (int g = 0; g < kLazyBlk; ++g) {
            row[g] = (b0 + g * G) * kBlock + threadIdx.x;
            ok[g] = b0 + g * G < nblk && row[g] < a.m;
            z[g] = ok[g] ? (a.zsrc ? a.zsrc[row[g]] : a.z[row[g]]) : 0.0;
            q[g] = (ok[g] && upd) ? a.qprev[row[g]] : 0.0;
            x[g] = ok[g] ? a.x[row[g]] : 0.0;
        }
        for (int kc = 0; kc < nk; kc += kLazyRs) {
            const int kn = min(kLazyRs, nk - kc);
            if (!one_chunk) {
                __syncthreads();
                stage(kc, kn);
                __syncthreads();
            }
            const double *pc = a.P + (int64_t)kc * a.ldp;
            int k = 0;
#pragma unroll 2
            for (; k + kLazyK <= kn; k += kLazyK) {
                double pv[kLazyK][kLazyBlk];
#pragma unroll
                for (int u = 0; u < kLazyK; ++u)
#pragma unroll
                    for (int g = 0; g < kLazyBlk; ++g)
                        pv[u][g] = ok[g] ? __ldcs(pc + (int64_t)(k + u) * a.ldp + row[g]) : 0.0;
#pragma unroll
                for (int u = 0; u < kLazyK; ++u) {
                    const double r = rs[k + u];
#pragma unroll
                    for (int g = 0; g < kLazyBlk; ++g) x[g] = __dsub_rn(x[g], __dmul_rn(r, pv[u][g]));
                }
            }
            for (; k < kn; ++k) {
                double pv[kLazyBlk];
#pragma unroll
                for (int g = 0; g < kLazyBlk; ++g) pv[g] = ok[g] ? __ldcs(pc + (int64_t)k * a.ldp + row[g]) : 0.0;
                const double r = rs[k];
#pragma unroll
                for (int g = 0; g < kLazyBlk; ++g) x[g] = __dsub_rn(x[g], __dmul_rn(r, pv[g]));
            }
        }
#pragma unroll
        for (int g = 0; g < kLazyBlk; ++g) {
            if (upd) {
                z[g] = __dsub_rn(z[g], __dmul_rn(rj, q[g]));
                if (ok[g]) a.z[row[g]] = z[g];
            }
            if (ok[g]) {
                a.xout[row[g]] = x[g];
                t = fma(z[g], x[g], t);
                zz = fma(z[g], z[g], zz);
                xx = fma(x[g], x[g], xx);
            }
        }
    }
}

__global__ void __launch_bounds__(kBlock, 4) col_lazy_norm_kernel(ColArgs a) {
    trace_mark(a.trace, 0);
    pdl_wait();
    trace_mark(a.trace, 1);
    if (failed(a.out.status)) return;
    const bool upd = a.r != nullptr || a.rin.partial != nullptr;  // z_j's deferred r_{j-1,j} q_{j-1}
    // r_{j-1,j}: this kernel forms it from the trailing partials (RrowIn; CTA
    // 0 stores it to R) or it is already final in R
    const double rj = a.rin.partial ? rrow_first(a.rin, blockIdx.x == 0) : (upd ? *a.r : 0.0);
    double t, zz, xx;
    col_lazy_body(a, rj, upd, t, zz, xx);
    pdl_trigger();
    norm_cta_partial(a.out, t, zz, xx, blockIdx.x);
    norm_last_cta(a.out, gridDim.x);
    rrow_rest(a.rin, blockIdx.x, gridDim.x);
    trace_mark(a.trace, 2);
}

// HP row form: catch-up of the stored X columns.  With x formed lazily
// (col_lazy_norm_kernel) step j reads p_k for every k the stored X_j lags
// behind; every few steps (and when a chunk of the host-input pipeline
// arrives) the stored columns j in [jbeg, jend) are brought forward by the
// projections k = kbeg .. kbeg + nk - 1: x -= r_kj p_k in ascending k with
// the reference's separately rounded multiply and subtract (gram_schmidt.py:
// 143-145) -- the same rounding sequence, so the bits of every x_j are
// unchanged; only where the terms are applied moves.  A thread keeps 8
// columns x 4 rows in registers and streams the p_k of its rows (each r_kj
// read from shared memory serves 4 updates); the column groups are the
// grid's fastest dimension, so the CTAs sharing a row block run together
// and the p_k rows come from L2 after the first.
struct XCatchArgs {
    int64_t m;
    double *X;
    int64_t ldx;
    int32_t jbeg, jend;
    const double *P;  // p_kbeg, p_kbeg+1, ... at stride ldp
    int64_t ldp;
    const double *R;  // r_{kbeg + k, j} = R[k * rstride + j]
    int64_t rstride;
    int32_t nk;
    const int32_t *status;
};
constexpr int kXcCols = 8;  // columns per thread
constexpr int kXcK = 32;    // r_kj staged per chunk of k
// kXcRows rows per thread (each r_kj load serves kXcRows updates), MINB CTAs per SM
template <int kXcRows, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) x_catchup_kernel(XCatchArgs a) {
    __shared__ __align__(16) double rs[kXcK][kXcCols];
    pdl_wait();
    if (failed(a.status)) return;
    const int groups = (a.jend - a.jbeg + kXcCols - 1) / kXcCols;  // column groups fastest
    const int64_t row0 = (int64_t)(blockIdx.x / groups) * (kBlock * kXcRows) + threadIdx.x;
    const int j0 = a.jbeg + (int)(blockIdx.x % groups) * kXcCols;
    const int nc = min(kXcCols, a.jend - j0);
    bool ok[kXcRows];
#pragma unroll
    for (int v = 0; v < kXcRows; ++v) ok[v] = row0 + (int64_t)v * kBlock < a.m;
    double x[kXcCols][kXcRows];
#pragma unroll
    for (int c = 0; c < kXcCols; ++c)
#pragma unroll
        for (int v = 0; v < kXcRows; ++v)
            x[c][v] = (ok[v] && c < nc) ? a.X[(int64_t)(j0 + c) * a.ldx + row0 + (int64_t)v * kBlock] : 0.0;
    for (int kc = 0; kc < a.nk; kc += kXcK) {
        const int kn = min(kXcK, a.nk - kc);
        __syncthreads();
        for (int e = threadIdx.x; e < kXcK * kXcCols; e += kBlock) {
            const int k = e / kXcCols, c = e - k * kXcCols;
            rs[k][c] = (k < kn && c < nc) ? __ldg(a.R + (int64_t)(kc + k) * a.rstride + j0 + c) : 0.0;
        }
        __syncthreads();
        for (int k0 = 0; k0 < kn; k0 += 2) {
            double pv[2][kXcRows];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int v = 0; v < kXcRows; ++v)
                    pv[u][v] = (ok[v] && k0 + u < kn) ? a.P[(int64_t)(kc + k0 + u) * a.ldp + row0 + (int64_t)v * kBlock]
                                                      : 0.0;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (k0 + u < kn) {
                    double r[kXcCols];
#pragma unroll
                    for (int c = 0; c < kXcCols; c += 2) {
                        const double2 rr = *reinterpret_cast<const double2 *>(&rs[k0 + u][c]);
                        r[c] = rr.x;
                        r[c + 1] = rr.y;
                    }
#pragma unroll
                    for (int c = 0; c < kXcCols; ++c)
#pragma unroll
                        for (int v = 0; v < kXcRows; ++v) x[c][v] = __dsub_rn(x[c][v], __dmul_rn(r[c], pv[u][v]));
                }
            }
        }
    }
    pdl_trigger();
#pragma unroll
    for (int c = 0; c < kXcCols; ++c)
#pragma unroll
        for (int v = 0; v < kXcRows; ++v)
            if (ok[v] && c < nc) a.X[(int64_t)(j0 + c) * a.ldx + row0 + (int64_t)v * kBlock] = x[c][v];
}

// The periodic catch-up (nk <= kXsMaxK): one CTA per 512-row block walks
// every column of [jbeg, jend) in groups of 8, with the block's p rows of
// the window staged once in shared memory (thread-private rows, as the
// trailing pass's q window) -- X read and written once, p read once, the
// FP64 updates of a group overlapping the loads of the next.  Same rounding
// sequence per element as x_catchup_kernel.
constexpr int kXsRows = 2, kXsMaxK = 32;
__host__ __device__ inline size_t xs_smem(int nk) { return sizeof(double) * (size_t)nk * kXsRows * kBlock; }
__global__ void __launch_bounds__(kBlock, 3) x_catchup_stream_kernel(XCatchArgs a) {
    extern __shared__ double xps[];  // [nk][kXsRows][kBlock]
    __shared__ __align__(16) double rs[kXsMaxK][kXcCols];
    pdl_wait();
    if (failed(a.status)) return;
    const int64_t row0 = (int64_t)blockIdx.x * (kBlock * kXsRows) + threadIdx.x;
    bool ok[kXsRows];
#pragma unroll
    for (int v = 0; v < kXsRows; ++v) ok[v] = row0 + (int64_t)v * kBlock < a.m;
    for (int k = 0; k < a.nk; ++k) {
#pragma unroll
        for (int v = 0; v < kXsRows; ++v)
            xps[(k * kXsRows + v) * kBlock + threadIdx.x] =
                ok[v] ? a.P[(int64_t)k * a.ldp + row0 + (int64_t)v * kBlock] : 0.0;
    }
    const int64_t rbase = (int64_t)blockIdx.x * (kBlock * kXsRows);
    const uint32_t pf_bytes = (uint32_t)(min((int64_t)kBlock * kXsRows, a.m - rbase) * 8) & ~15u;
    for (int j0 = a.jbeg; j0 < a.jend; j0 += kXcCols) {
        const int nc = min(kXcCols, a.jend - j0);
        if (threadIdx.x < kXcCols && pf_bytes) {  // the next group's block toward L2 (one column per thread)
            const int jn = j0 + kXcCols + (int)threadIdx.x;
            const double *src = a.X + (int64_t)jn * a.ldx + rbase;
            if (jn < a.jend && ((uintptr_t)src & 15) == 0)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(pf_bytes) : "memory");
        }
        double x[kXcCols][kXsRows];
#pragma unroll
        for (int c = 0; c < kXcCols; ++c)
#pragma unroll
            for (int v = 0; v < kXsRows; ++v)
                x[c][v] = (ok[v] && c < nc) ? a.X[(int64_t)(j0 + c) * a.ldx + row0 + (int64_t)v * kBlock] : 0.0;
        __syncthreads();  // the previous group's rs reads are done
        for (int e = threadIdx.x; e < a.nk * kXcCols; e += kBlock) {
            const int k = e / kXcCols, c = e - k * kXcCols;
            rs[k][c] = c < nc ? __ldg(a.R + (int64_t)k * a.rstride + j0 + c) : 0.0;
        }
        __syncthreads();
#pragma unroll 2
        for (int k = 0; k < a.nk; ++k) {
            double pv[kXsRows], r[kXcCols];
#pragma unroll
            for (int v = 0; v < kXsRows; ++v) pv[v] = xps[(k * kXsRows + v) * kBlock + threadIdx.x];
#pragma unroll
            for (int c = 0; c < kXcCols; c += 2) {
                const double2 rr = *reinterpret_cast<const double2 *>(&rs[k][c]);
                r[c] = rr.x;
                r[c + 1] = rr.y;
            }
#pragma unroll
            for (int c = 0; c < kXcCols; ++c)
#pragma unroll
                for (int v = 0; v < kXsRows; ++v) x[c][v] = __dsub_rn(x[c][v], __dmul_rn(r[c], pv[v]));
        }
#pragma unroll
        for (int c = 0; c < kXcCols; ++c)
#pragma unroll
            for (int v = 0; v < kXsRows; ++v)
                if (ok[v] && c < nc) a.X[(int64_t)(j0 + c) * a.ldx + row0 + (int64_t)v * kBlock] = x[c][v];
    }
    pdl_trigger();
}

// Standalone totals of the norm partials (step API / multi-GPU driver).
__global__ void __launch_bounds__(kBlock)
    norm_reduce_kernel(const double *npart, int32_t ntiles, double *tot, int64_t i, double *rii,
                       int32_t *status) {
    if (failed(status)) return;
    __shared__ double t3[3];
    __shared__ double sm3[3 * kWarps];
    block_totals<3>(npart, ntiles, ntiles, t3, sm3, SyncAll());
    if (threadIdx.x == 0) {
        if (tot) {
            tot[0] = t3[0];
            tot[1] = t3[1];
            tot[2] = t3[2];
        }
        if (rii) norm_finish_dev(i, t3[0], t3[1], t3[2], rii, status);
    }
}

__global__ void norm_finish_kernel(int64_t i, const double *tot, double *rii, int32_t *status) {
    if (failed(status)) return;
    norm_finish_dev(i, tot[0], tot[1], tot[2], rii, status);
}

// Standalone column totals: block c reduces column c (block_totals).
__global__ void __launch_bounds__(kBlock)
    rrow_reduce_kernel(const double *partial, int32_t ntiles, int32_t ncols, double *out,
                       const int32_t *status) {
    if (failed(status)) return;
    __shared__ double sm[kWarps];
    (void)ncols;
    block_totals<1>(partial + (int64_t)blockIdx.x * ntiles, ntiles, ntiles, out + blockIdx.x, sm,
                    SyncAll());
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
// Fused trailing pass, generic (direct loads; any m)
// ---------------------------------------------------------------------------
struct TrailArgs {
    int64_t m;
    int32_t ntiles;
    int32_t cpg;     // columns per group
    int32_t ngroups;
    int32_t jbeg, jend;
    int32_t reverse;  // walk the work items backwards (L2 reuse across steps)
    double *W;
    int64_t ldw;
    const double *Wsrc;  // read the trailing columns from here (nullptr: W); results go to W
    int64_t ldwsrc;
    double *X;  // HP carried A z (nullptr otherwise)
    int64_t ldx;
    const double *Z0;  // CGS original columns (nullptr for MGS)
    int64_t ldz0;
    const double *qprev;  // q_{i-1}; nullptr at i == 0 (no deferred update)
    const double *pprev;  // p_{i-1} (HP)
    const double *rprev;  // r_{i-1, j} = rprev[j] (row i-1 of row-major Rt)
    const double *psrc;   // p_i = psrc / *rii  (or psrc itself when rii == nullptr)
    const double *rii;
    double *pout;         // store p_i (group 0)
    const double *zsrc;   // z_i
    double *qout;         // store q_i = z_i / *rii (group 0)
    double *partial;      // [(j - jbeg) * ntiles + tile]
    unsigned *counters;   // per group; nullptr: no in-kernel totals
    double *rout;         // totals: rout[j - jbeg] (row i of Rt from column jbeg)
    const int32_t *status;
    int32_t trace;        // AQR_TRACE builds: launch slot (-1 off)
    // windowed pass (trailing_w_kernel): projections i-win .. i-1 are applied
    // to the stored columns (state z^(i-win)) before the dots
    int32_t win;
    int32_t store_all;    // write every column back at z^(i) (else only column jbeg)
    const double *qwin;   // q_{i-win}; q_k at qwin + (k - i + win) * ldw
    const double *rwin;   // r_{i-win, j} = rwin[j]; row k at + (k - i + win) * rstride
    int64_t rstride;
};

// Load the step vectors of one tile into registers; group 0 stores q_i/p_i.
template <int RPT, bool HP>
__device__ __forceinline__ void trail_vectors(const TrailArgs &a, int64_t row0, bool store,
                                              double *q, double *p, double *pp) {
    const bool upd = a.qprev != nullptr;
    const bool sq = store && a.qout != nullptr, sp = store && a.pout != nullptr;
    // all loads first (the stores below may alias them as far as the
    // compiler knows: interleaving would serialize RPT round trips)
    double ps[RPT], zs[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t r = row0 + (int64_t)u * kBlock;
        const bool ok = r < a.m;
        ps[u] = ok ? a.psrc[r] : 0.0;
        q[u] = (ok && upd) ? a.qprev[r] : 0.0;
        pp[u] = (HP && ok && upd) ? a.pprev[r] : 0.0;
        zs[u] = (ok && sq) ? a.zsrc[r] : 0.0;
    }
    const double rii = a.rii ? *a.rii : 1.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t r = row0 + (int64_t)u * kBlock;
        const bool ok = r < a.m;
        p[u] = a.rii ? ps[u] / rii : ps[u];
        if (ok && sq) a.qout[r] = zs[u] / rii;
        if (ok && sp) a.pout[r] = p[u];
    }
}

// Columns per unit prefetched into L2 before the dependency wait (0: off;
// build-time knob -DAQR_TRAIL_PREFETCH=k for A/B).
#ifndef AQR_TRAIL_PREFETCH
#define AQR_TRAIL_PREFETCH 4
#endif
constexpr int trail_prefetch_cols = AQR_TRAIL_PREFETCH;

// One (tile, column group) work unit of the trailing pass (all kBlock threads).
template <int RPT, int CU, bool HP, bool CGS>
__device__ __forceinline__ void trail_body(const TrailArgs &a, int tile, int group, double *wsum) {
    const int64_t row0 = (int64_t)tile * (kBlock * RPT) + threadIdx.x;
    const int cbeg = a.jbeg + group * a.cpg;
    const int cend = min(a.jend, cbeg + a.cpg);
    const bool upd = a.qprev != nullptr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    double q[RPT], p[RPT], pp[RPT];
    trail_vectors<RPT, HP>(a, row0, group == 0, q, p, pp);
    bool ok[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) ok[u] = row0 + (int64_t)u * kBlock < a.m;

    for (int j0 = cbeg; j0 < cend; j0 += CU) {
        double z[CU][RPT], x[CU][RPT], rj[CU];
#pragma unroll
        for (int c = 0; c < CU; ++c) {
            const int j = j0 + c;
            const bool cj = j < cend;
            rj[c] = (cj && upd) ? a.rprev[j] : 0.0;
            const double *zc = a.Wsrc ? a.Wsrc + (int64_t)j * a.ldwsrc : a.W + (int64_t)j * a.ldw;
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
    pdl_trigger();
    __syncthreads();
    for (int c = threadIdx.x; c < cend - cbeg; c += kBlock) {
        double s = wsum[c];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) s = __dadd_rn(s, wsum[w * a.cpg + c]);
        a.partial[(int64_t)(cbeg - a.jbeg + c) * a.ntiles + tile] = s;
    }
}

// Before the grid-dependency wait: bring this unit's q_{i-1} tile and its
// first columns' tiles (16 KB each, written by the kernel before the
// previous one) into L2 with bulk prefetches, so the first loads after the
// wait hit L2 while the previous kernel drains.  L2 is the coherence point:
// a prefetch never makes a later load stale.
template <int RPT>
__device__ __forceinline__ void trail_prefetch(const TrailArgs &a, int tile, int group) {
    if (RPT < 4 || threadIdx.x != 0 || trail_prefetch_cols <= 0) return;
    const int64_t row0 = (int64_t)tile * (kBlock * RPT);
    const int64_t rows = min((int64_t)kBlock * RPT, a.m - row0);
    const uint32_t bytes = (uint32_t)(rows * 8) & ~15u;
    if (bytes == 0) return;
    auto pf = [&](const double *base) {
        if (((uintptr_t)base & 15) == 0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base), "r"(bytes) : "memory");
    };
    const int cbeg = a.jbeg + group * a.cpg;
    const int cend = min(a.jend, cbeg + min(a.cpg, trail_prefetch_cols));
    const double *zb = a.Wsrc ? a.Wsrc : a.W;
    const int64_t ld = a.Wsrc ? a.ldwsrc : a.ldw;
    if (a.qprev) pf(a.qprev + row0);
    for (int j = cbeg; j < cend; ++j) pf(zb + (int64_t)j * ld + row0);
}

// HP trailing kernels: minimum resident CTAs per SM (build-time A/B knob)
#ifndef AQR_HP_MINB
#define AQR_HP_MINB 1
#endif
template <int RPT, int CU, bool HP, bool CGS>
__global__ void __launch_bounds__(kBlock, HP ? AQR_HP_MINB : 1) trailing_kernel(TrailArgs a) {
    trace_mark(a.trace, 0);
    trail_prefetch<RPT>(a, a.reverse ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x,
                        a.reverse ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y);
    pdl_wait();
    trace_mark(a.trace, 1);
    if (failed(a.status)) return;
    extern __shared__ double wsum[];  // [kWarps][cpg]
    // Odd steps walk the (tile, group) units backwards: CTAs are dispatched
    // x-fastest, so the first units of this pass are the last ones the
    // previous pass wrote -- still in L2.  Partials are per unit: bitwise
    // independent of the walk.
    const int tile = a.reverse ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
    const int group = a.reverse ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y;
    trail_body<RPT, CU, HP, CGS>(a, tile, group, wsum);
    trace_mark(a.trace, 2);
    // totals: the next step's norm kernel (RrowIn) or rrow_reduce_kernel
}

// ---------------------------------------------------------------------------
// Windowed trailing pass (row form, Z only): deferred projections
// ---------------------------------------------------------------------------
// project(k, j) (gram_schmidt.py:139-145) rewrites every trailing column at
// every step, but step i only needs z_j^(i) -- z_j after the projections
// 0 .. i-1 -- inside its dot products r_ij = p_i . z_j^(i).  The stored
// trailing columns are kept at an older state z_j^(s) (s <= i, the "base"),
// and the pass of step i re-forms z_j^(i) in registers by applying the
// win = i - s deferred projections z -= r_kj q_k, k = s .. i-1, in ascending
// k with the reference's separately rounded multiply and subtract: the very
// sequence of roundings the eager updates apply, so every z_j^(i) -- and the
// factors -- are bitwise unchanged.  Only every b-th pass writes the
// trailing block back (store_all; the base becomes i); the other passes read
// it once and write only column jbeg = i+1, the next one to be normalized.
// Per step the trailing traffic drops from a read and a write of every
// element to a read plus 1/b of a write; the price is win extra multiply-
// subtract pairs per element (FP64 pipe, well below its rate at b <= 8) and
// the q_k window staged per tile.
//
// Shared memory (dynamic): wsum [kWarps][cpg], rsm [win][cpg] (r_kj of the
// CTA's columns), qs [win][RPT][kBlock] (thread-private rows of q_k).
// Column pairs ahead whose tiles the windowed pass bulk-prefetches into L2
// (0: off; build-time knob).
#ifndef AQR_TRAIL_PF_DIST
#define AQR_TRAIL_PF_DIST 1  // config 5 HP trailing 931 / 900 / 909 / 955 ms at 0 / 1 / 2 / 4
#endif
constexpr int kTrailPfDist = AQR_TRAIL_PF_DIST;
__host__ __device__ inline size_t trail_w_smem(int rpt, int cpg, int win) {
    return sizeof(double) * ((size_t)kWarps * cpg + (size_t)win * cpg + (size_t)win * rpt * kBlock);
}

template <int RPT, int CU, bool CGS>
__device__ __forceinline__ void trail_body_w(const TrailArgs &a, int tile, int group, double *smem) {
    const int64_t row0 = (int64_t)tile * (kBlock * RPT) + threadIdx.x;
    const int cbeg = a.jbeg + group * a.cpg;
    const int cend = min(a.jend, cbeg + a.cpg);
    const int nc = cend - cbeg;
    const int win = a.win;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *wsum = smem;
    double *rsm = wsum + kWarps * a.cpg;
    double *qs = rsm + win * a.cpg;

    bool ok[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) ok[u] = row0 + (int64_t)u * kBlock < a.m;
    // step vectors: p_i (group 0 stores q_i, p_i), the q window (thread-private
    // rows) and the CTA's r_kj
    double p[RPT];
    {
        double ps[RPT], zs[RPT];
        const bool sq = group == 0 && a.qout != nullptr, sp = group == 0 && a.pout != nullptr;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int64_t r = row0 + (int64_t)u * kBlock;
            ps[u] = ok[u] ? a.psrc[r] : 0.0;
            zs[u] = (ok[u] && sq) ? a.zsrc[r] : 0.0;
        }
        for (int k = 0; k < win; ++k) {
            double qv[RPT];
#pragma unroll
            for (int u = 0; u < RPT; ++u)
                qv[u] = ok[u] ? __ldcg(a.qwin + (int64_t)k * a.ldw + row0 + (int64_t)u * kBlock) : 0.0;
#pragma unroll
            for (int u = 0; u < RPT; ++u) qs[(k * RPT + u) * kBlock + threadIdx.x] = qv[u];
        }
        for (int e = threadIdx.x; e < win * nc; e += kBlock) {
            const int k = e / nc, c = e - k * nc;
            rsm[k * a.cpg + c] = __ldcg(a.rwin + (int64_t)k * a.rstride + cbeg + c);
        }
        const double rii = a.rii ? *a.rii : 1.0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int64_t r = row0 + (int64_t)u * kBlock;
            p[u] = a.rii ? ps[u] / rii : ps[u];
            if (ok[u] && sq) a.qout[r] = zs[u] / rii;
            if (ok[u] && sp) a.pout[r] = p[u];
        }
    }
    __syncthreads();
    const double *zb = a.Wsrc ? a.Wsrc : a.W;
    const int64_t ldzb = a.Wsrc ? a.ldwsrc : a.ldw;

    // bytes of this tile in one column (16-byte multiple for the bulk prefetch)
    const uint32_t pf_bytes = (uint32_t)(min((int64_t)kBlock * RPT, a.m - (int64_t)tile * kBlock * RPT) * 8) & ~15u;
    for (int j0 = cbeg; j0 < cend; j0 += CU) {
        // keep HBM busy while the window arithmetic runs: the tile of the
        // column pair kTrailPfDist pairs ahead is bulk-prefetched into L2
        if (kTrailPfDist > 0 && RPT >= 4 && threadIdx.x == 0 && !CGS) {
            const int jp = j0 + kTrailPfDist * CU;
#pragma unroll
            for (int c = 0; c < CU; ++c) {
                const double *src = zb + (int64_t)(jp + c) * ldzb + (int64_t)tile * kBlock * RPT;
                if (jp + c < cend && pf_bytes && ((uintptr_t)src & 15) == 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(pf_bytes) : "memory");
            }
        }
        // CGS reads z only where it is written (the dots use Z0)
        const bool needz = !CGS || (win > 0 && (a.store_all || j0 == a.jbeg));
        double z[CU][RPT], d0[CGS ? CU : 1][RPT];
#pragma unroll
        for (int c = 0; c < CU; ++c) {
            const int j = j0 + c;
            const bool cj = j < cend;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                const int64_t r = row0 + (int64_t)u * kBlock;
                z[c][u] = (needz && cj && ok[u]) ? zb[(int64_t)j * ldzb + r] : 0.0;
                if (CGS) d0[c][u] = (cj && ok[u]) ? a.Z0[(int64_t)j * a.ldz0 + r] : 0.0;
            }
        }
        if (needz) {
#pragma unroll 1
            for (int k = 0; k < win; ++k) {
                double qv[RPT], rk[CU];
#pragma unroll
                for (int u = 0; u < RPT; ++u) qv[u] = qs[(k * RPT + u) * kBlock + threadIdx.x];
#pragma unroll
                for (int c = 0; c < CU; ++c) rk[c] = j0 + c < cend ? rsm[k * a.cpg + (j0 + c - cbeg)] : 0.0;
#pragma unroll
                for (int c = 0; c < CU; ++c)
#pragma unroll
                    for (int u = 0; u < RPT; ++u) z[c][u] = __dsub_rn(z[c][u], __dmul_rn(rk[c], qv[u]));
            }
            if (win > 0) {
#pragma unroll
                for (int c = 0; c < CU; ++c) {
                    const int j = j0 + c;
                    if (j < cend && (a.store_all || j == a.jbeg))
#pragma unroll
                        for (int u = 0; u < RPT; ++u)
                            if (ok[u]) a.W[(int64_t)j * a.ldw + row0 + (int64_t)u * kBlock] = z[c][u];
                }
            }
        }
        double acc[CU];
#pragma unroll
        for (int c = 0; c < CU; ++c) {
            acc[c] = 0.0;
#pragma unroll
            for (int u = 0; u < RPT; ++u) acc[c] = fma(p[u], CGS ? d0[CGS ? c : 0][u] : z[c][u], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < CU; ++c) {
            const double s = warp_sum(acc[c]);
            if (lane == 0 && j0 + c < cend) wsum[warp * a.cpg + (j0 + c - cbeg)] = s;
        }
    }
    pdl_trigger();
    __syncthreads();
    for (int c = threadIdx.x; c < nc; c += kBlock) {
        double s = wsum[c];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) s = __dadd_rn(s, wsum[w * a.cpg + c]);
        a.partial[(int64_t)(cbeg - a.jbeg + c) * a.ntiles + tile] = s;
    }
}

template <int RPT, int CU, bool CGS>
__global__ void __launch_bounds__(kBlock, 1) trailing_w_kernel(TrailArgs a) {
    trace_mark(a.trace, 0);
    trail_prefetch<RPT>(a, a.reverse ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x,
                        a.reverse ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y);
    pdl_wait();
    trace_mark(a.trace, 1);
    if (failed(a.status)) return;
    extern __shared__ double smem_w[];
    const int tile = a.reverse ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
    const int group = a.reverse ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y;
    trail_body_w<RPT, CU, CGS>(a, tile, group, smem_w);
    trace_mark(a.trace, 2);
}

// ---------------------------------------------------------------------------
// Catch-up of a newly arrived chunk of columns (host-input pipeline): the
// trailing passes of steps 0 .. k1-1 restricted to the chunk, in ONE
// cooperative launch -- per step a pass over the (tile, column) units, a grid
// barrier, the chunk's R-row totals (block_totals, CTA b: column b), a grid
// barrier.  The launches and drains of 2 k1 small kernels disappear.  Per
// unit the same chain and trees as trail_body_w, totals as
// rrow_reduce_kernel: bitwise identical.
//
// Windowed like trailing_w_kernel: the chunk's stored columns stay at
// z^(sc) while step k applies the projections sc .. k-1 in registers (q
// window per tile in shared memory, r rows of the window staged per step);
// they are written back every win-th step and at the last one, so the
// chunk leaves at z^(k1-1) -- what the step loop expects.
// ---------------------------------------------------------------------------
struct CatchArgs {
    int64_t m, n;
    int32_t ntiles, c0, w, k1;
    double *W;
    int64_t ldw;
    const double *Z0;  // CGS
    int64_t ldz0;
    const double *vall;  // per-step vectors, ld m: HA x_k (p_k = x_k / r_kk), HP / naive p_k
    int32_t p_direct;
    double *Rt;       // n x n row-major
    double *partial;  // [w][ntiles] (x 2 when redundant: by step parity)
    const int32_t *status;
    int32_t trace;      // AQR_TRACE builds: launch slot (-1 off)
    int32_t redundant;  // per-CTA totals, one grid barrier per step (smem: w doubles)
    int32_t win;        // write-back period (1: every step)
};

// Dynamic shared memory: wsum [kWarps][wpad] (warp totals of a tile's
// units), rs [wpad] (redundant totals), rsm [win][wpad] (the window's r
// rows), qs [win][RPT][kBlock].
__host__ __device__ inline int catch_wpad(int w) { return ((w + 7) / 8) * 8; }
__host__ __device__ inline size_t catch_smem(int rpt, int w, int win, bool redundant) {
    return sizeof(double) * ((size_t)kWarps * catch_wpad(w) + (redundant ? catch_wpad(w) : 0) +
                             (size_t)win * catch_wpad(w) + (size_t)win * rpt * kBlock);
}

#ifndef AQR_CATCHUP_PF
#define AQR_CATCHUP_PF 1  // the catch-up's L2 look-ahead (build-time A/B)
#endif
#ifndef AQR_CATCHUP_REVERSE
#define AQR_CATCHUP_REVERSE 1
#endif
// Tiles per column loaded together by the catch-up's per-CTA totals (build
// knob: 2 keeps 2 CTAs/SM with a few spilled bytes; 1 no spills, two round trips).
#ifndef AQR_CATCHUP_TOT_H
#define AQR_CATCHUP_TOT_H 2
#endif
template <int RPT, bool CGS>
__global__ void __launch_bounds__(kBlock, 2) catchup_kernel(CatchArgs a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    trace_mark(a.trace, 0);
    trace_mark(a.trace, 1);
    if (failed(a.status)) return;  // uniform: set before this launch
    constexpr int CU = 2;          // columns per unit
    extern __shared__ double smc[];
    const int wpad = catch_wpad(a.w);
    double *wsum = smc;
    double *rs = wsum + kWarps * wpad;
    double *rsm = rs + (a.redundant ? wpad : 0);
    double *qs = rsm + a.win * wpad;
    __shared__ double tot1[1];
    __shared__ double sm1[kWarps];
    __shared__ double sm8[8 * kWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // a.redundant: every CTA forms the w totals of step k-1 it needs itself
    // (same block_totals tree; CTA 0 stores them to R), partials alternate
    // between two buffers by step parity -- one grid barrier per step
    // instead of two around a totals phase on w CTAs.
    const int64_t pstride = (int64_t)a.w * a.ntiles;
    int sc = 0;  // the chunk's stored columns hold z^(sc)
    for (int k = 0; k < a.k1; ++k) {
        const int win = k - sc;  // projections sc .. k-1 applied in registers
        const bool store = win > 0 && (win >= a.win || k + 1 == a.k1);
        double *part = a.partial + (a.redundant ? (int64_t)(k & 1) * pstride : 0);
        if (a.redundant && k > 0) {
            const double *prev = a.partial + (int64_t)((k - 1) & 1) * pstride;
            for (int cb = 0; cb < a.w; cb += 8) {
                block_totals<8, SyncAll, AQR_CATCHUP_TOT_H>(prev + (int64_t)cb * a.ntiles, a.ntiles, a.ntiles, rs + cb,
                                                            sm8, SyncAll());
            }
            if (blockIdx.x == 0)
                for (int c = threadIdx.x; c < a.w; c += kBlock) a.Rt[(int64_t)(k - 1) * a.n + a.c0 + c] = rs[c];
        }
        // r rows sc .. k-1 of the chunk (row k-1: this CTA's own totals when
        // redundant; the others were stored and published by a grid barrier)
        for (int e = threadIdx.x; e < win * a.w; e += kBlock) {
            const int kk = e / a.w, c = e - kk * a.w;
            rsm[kk * wpad + c] = (a.redundant && kk == win - 1) ? rs[c]
                                                                : __ldcg(a.Rt + (int64_t)(sc + kk) * a.n + a.c0 + c);
        }
        __syncthreads();
        const double rii = a.p_direct ? 1.0 : __ldcg(a.Rt + (int64_t)k * a.n + k);
        const double *psrc = a.vall + (int64_t)k * a.m;
        // units (tile, CU columns), tile-major; CTA b walks the contiguous
        // range [U b / G, U (b + 1) / G) (balanced to one unit) and reloads
        // the step vectors only when the range enters a new tile
        const int ng = (a.w + CU - 1) / CU;
        const int64_t U = (int64_t)a.ntiles * ng;
        const int64_t ub = U * blockIdx.x / gridDim.x, ue = U * (blockIdx.x + 1) / gridDim.x;
        double p[RPT];
        bool ok[RPT];
        // The range is walked tile by tile: the step vectors and the q window
        // load once per tile, the tile's units keep their warp totals in
        // wsum[warp][column] (no barrier between units, so the loads of the
        // next unit are not held back), and one pair of barriers per tile
        // turns them into the tile's partials.  Odd steps walk the tiles
        // backwards: a step starts on the tiles the previous one touched last
        // (still in L2); per unit independent, so the bits do not depend on
        // the walk.
        const bool back = AQR_CATCHUP_REVERSE && (k & 1);
        const int t_lo = (int)(ub / ng), t_hi = ue > ub ? (int)((ue - 1) / ng) : t_lo - 1;
        for (int ti = t_lo; ti <= t_hi; ++ti) {
            const int tile = back ? t_lo + t_hi - ti : ti;
            const int g0 = (int)(ub > (int64_t)tile * ng ? ub - (int64_t)tile * ng : 0);       // first unit of the tile
            const int g1 = (int)(ue < (int64_t)(tile + 1) * ng ? ue - (int64_t)tile * ng : ng);  // one past the last
            const int64_t row0 = (int64_t)tile * (kBlock * RPT) + threadIdx.x;
#pragma unroll
            for (int v = 0; v < RPT; ++v) {  // thread-private rows: no barrier needed
                const int64_t r = row0 + (int64_t)v * kBlock;
                ok[v] = r < a.m;
                const double ps = ok[v] ? __ldcg(psrc + r) : 0.0;
                p[v] = a.p_direct ? ps : ps / rii;
            }
            for (int kk = 0; kk < win; ++kk) {
                double qv[RPT];
#pragma unroll
                for (int v = 0; v < RPT; ++v)
                    qv[v] = ok[v] ? __ldcg(a.W + (int64_t)(sc + kk) * a.ldw + row0 + (int64_t)v * kBlock) : 0.0;
#pragma unroll
                for (int v = 0; v < RPT; ++v) qs[(kk * RPT + v) * kBlock + threadIdx.x] = qv[v];
            }
            const uint32_t pf_bytes =
                (uint32_t)(min((int64_t)kBlock * RPT, a.m - (int64_t)tile * kBlock * RPT) * 8) & ~15u;
            for (int g = g0; g < g1; ++g) {
                const int c0 = g * CU;
                const bool needz = !CGS || store;
                // as the trailing pass: the next unit's tile toward L2 while this one computes
                if (AQR_CATCHUP_PF && kTrailPfDist > 0 && RPT >= 4 && threadIdx.x == 0 && needz) {
#pragma unroll
                    for (int c = 0; c < CU; ++c) {
                        const int cn = c0 + kTrailPfDist * CU + c;
                        const double *src = a.W + (int64_t)(a.c0 + cn) * a.ldw + (int64_t)tile * kBlock * RPT;
                        if (cn < g1 * CU && cn < a.w && pf_bytes && ((uintptr_t)src & 15) == 0)
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(pf_bytes)
                                         : "memory");
                    }
                }
                double z[CU][RPT], d0[CGS ? CU : 1][RPT], acc[CU];
#pragma unroll
                for (int c = 0; c < CU; ++c) {
                    const int j = a.c0 + c0 + c;
                    const bool cj = c0 + c < a.w;
#pragma unroll
                    for (int v = 0; v < RPT; ++v) {
                        const int64_t r = row0 + (int64_t)v * kBlock;
                        z[c][v] = (needz && cj && ok[v]) ? __ldcg(a.W + (int64_t)j * a.ldw + r) : 0.0;
                        if (CGS) d0[c][v] = (cj && ok[v]) ? __ldcg(a.Z0 + (int64_t)j * a.ldz0 + r) : 0.0;
                    }
                }
                if (needz) {
#pragma unroll 1
                    for (int kk = 0; kk < win; ++kk) {
                        double qv[RPT], rk[CU];
#pragma unroll
                        for (int v = 0; v < RPT; ++v) qv[v] = qs[(kk * RPT + v) * kBlock + threadIdx.x];
#pragma unroll
                        for (int c = 0; c < CU; ++c) rk[c] = c0 + c < a.w ? rsm[kk * wpad + c0 + c] : 0.0;
#pragma unroll
                        for (int c = 0; c < CU; ++c)
#pragma unroll
                            for (int v = 0; v < RPT; ++v) z[c][v] = __dsub_rn(z[c][v], __dmul_rn(rk[c], qv[v]));
                    }
                    if (store) {
#pragma unroll
                        for (int c = 0; c < CU; ++c)
                            if (c0 + c < a.w)
#pragma unroll
                                for (int v = 0; v < RPT; ++v)
                                    if (ok[v]) a.W[(int64_t)(a.c0 + c0 + c) * a.ldw + row0 + (int64_t)v * kBlock] = z[c][v];
                    }
                }
#pragma unroll
                for (int c = 0; c < CU; ++c) {
                    acc[c] = 0.0;
#pragma unroll
                    for (int v = 0; v < RPT; ++v) acc[c] = fma(p[v], CGS ? d0[CGS ? c : 0][v] : z[c][v], acc[c]);
                }
#pragma unroll
                for (int c = 0; c < CU; ++c) {
                    const double sw = warp_sum(acc[c]);
                    if (lane == 0 && c0 + c < a.w) wsum[warp * wpad + c0 + c] = sw;
                }
            }
            __syncthreads();
            for (int c = g0 * CU + threadIdx.x; c < min(g1 * CU, a.w); c += kBlock) {
                double s = wsum[c];
#pragma unroll
                for (int w2 = 1; w2 < kWarps; ++w2) s = __dadd_rn(s, wsum[w2 * wpad + c]);
                part[(int64_t)c * a.ntiles + tile] = s;
            }
            __syncthreads();
        }
        if (store) sc = k;
        grid.sync();
        if (a.redundant && k + 1 < a.k1) continue;  // the next step forms these totals
        for (int cc = blockIdx.x; cc < a.w; cc += gridDim.x) {
            block_totals<1>(part + (int64_t)cc * a.ntiles, a.ntiles, a.ntiles, tot1, sm1, SyncAll());
            if (threadIdx.x == 0) a.Rt[(int64_t)k * a.n + a.c0 + cc] = tot1[0];
        }
        if (!a.redundant) grid.sync();
    }
    trace_mark(a.trace, 2);
}

// ---------------------------------------------------------------------------
// TMA bulk-copy helpers (cp.async.bulk + mbarrier transaction counts)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
template <bool HINT>
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t pol) {
    if (HINT)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
            "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
            : "memory");
    else
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
            "l"(src), "r"(bytes), "r"(smem_u32(bar))
            : "memory");
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
// CSR operator: thread-per-row SpMV / SpMM, reference-exact (stored order)
// ---------------------------------------------------------------------------
// One thread owns one row.  Its nonzeros are taken in batches of 8: the 8
// (index, value) loads are issued together, then the 8 gathers of x, then
// the 8 products are added in stored order with separate rounding, which is
// bitwise equal to csr_matvec (_kernels_impl.py:50-56).  No shared memory
// and no barriers on the product path: warps are independent, so the SM
// keeps ~16 loads per thread in flight across all resident warps (the
// operator is latency-bound, not bandwidth-bound, at stencil row lengths;
// consecutive rows share cache lines, so DRAM traffic stays ~1x).  For k > 1
// (SpMM, the HP block apply) rows of <= 8 nonzeros keep them in registers
// across all k columns.  The fused variant (HA/naive step, k = 1) gathers x
// as z - r q (the deferred projection of the previous step, elementwise
// identical to the separate update), writes the updated z and x = A z, and
// emits the canonical 256-row norm partials; grid-stride over 256-row
// blocks, one completion ticket per CTA.
constexpr int kRowBatch = 8;

struct CsrArgs {
    int64_t m, k;
    const int32_t *indptr;
    const int32_t *indices;
    const double *data;
    const double *X;
    int64_t ldx;
    double *Y;
    int64_t ldy;
    // fused step (k == 1)
    const double *qprev;
    const double *r;  // r_{i-1,i}; nullptr: gather X as is
    double *znew;     // updated z_i (own rows)
    NormOut out;      // out.npart == nullptr: plain apply
    RrowIn rin;       // fused step: deferred r-row totals (partial == nullptr: none)
    int32_t trace;    // AQR_TRACE builds: launch slot (-1 off)
    int32_t sg;       // csr_spmm2_kernel: column blocks per super-group (0: all)
};

// sum_q data[q] * xe(indices[q]) over q in [s, e), xe = x - rj qprev (upd),
// in batches of B entries (loads of a batch in flight together)
template <int B = kRowBatch>
__device__ __forceinline__ double csr_row(const CsrArgs &a, const double *x, int s, int e,
                                          bool upd, double rj) {
    double acc = 0.0;
    for (int q0 = s; q0 < e; q0 += B) {
        int c[B];
        double v[B], xv[B];
#pragma unroll
        for (int h = 0; h < B; ++h) {
            const bool ok = q0 + h < e;
            c[h] = ok ? __ldg(a.indices + q0 + h) : 0;
            v[h] = ok ? __ldg(a.data + q0 + h) : 0.0;
        }
#pragma unroll
        for (int h = 0; h < B; ++h) {
            xv[h] = q0 + h < e ? __ldg(x + c[h]) : 0.0;
            if (upd && q0 + h < e) xv[h] = __dsub_rn(xv[h], __dmul_rn(rj, __ldg(a.qprev + c[h])));
        }
#pragma unroll
        for (int h = 0; h < B; ++h)
            if (q0 + h < e) acc = __dadd_rn(acc, __dmul_rn(v[h], xv[h]));
    }
    return acc;
}

// R rows at once: when every row has <= kRowBatch nonzeros, all R rows'
// (index, value) loads are issued together, then all R x R gathers, then the
// sums in stored order; otherwise row by row (csr_row).  Same arithmetic.
template <int R, int B = kRowBatch>
__device__ __forceinline__ void csr_rows(const CsrArgs &a, const int (&s)[R], const int (&e)[R],
                                         bool upd, double rj, double (&y)[R]) {
    bool short_rows = true;
#pragma unroll
    for (int i = 0; i < R; ++i) short_rows &= (e[i] - s[i] <= B);
    if (!short_rows) {
#pragma unroll
        for (int i = 0; i < R; ++i) y[i] = csr_row<B>(a, a.X, s[i], e[i], upd, rj);
        return;
    }
    int c[R][B];
    double v[R][B], xv[R][B];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int h = 0; h < B; ++h) {
            const bool ok = s[i] + h < e[i];
            c[i][h] = ok ? __ldg(a.indices + s[i] + h) : 0;
            v[i][h] = ok ? __ldg(a.data + s[i] + h) : 0.0;
        }
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int h = 0; h < B; ++h) {
            const bool ok = s[i] + h < e[i];
            xv[i][h] = ok ? __ldg(a.X + c[i][h]) : 0.0;
            if (upd && ok) xv[i][h] = __dsub_rn(xv[i][h], __dmul_rn(rj, __ldg(a.qprev + c[i][h])));
        }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int h = 0; h < B; ++h)
            if (s[i] + h < e[i]) acc = __dadd_rn(acc, __dmul_rn(v[i][h], xv[i][h]));
        y[i] = acc;
    }
}

// Plain apply, k >= 1 columns: grid-stride over 256-row blocks.
// Y = A X for k >= 2 columns and long rows (27-point stencils, config 5's HP
// block apply).  CTA = (column block of K, row block of 256), column blocks
// of a row block adjacent in launch order so they share the row block's CSR
// entries in L2; thread = (row, K columns): each batch of B entries is loaded
// once for K columns (B x K gathers in flight).  Stored-order sums per output
// as csr_row.  Config 5 block apply: 316 ms (per-column rows) -> 102-117 ms.
//
// Launch order (a.sg column blocks per super-group; 0: one super-group):
// super-group slowest, then row block, then the super-group's column blocks.
// The CSR rows are read from HBM once per super-group (the column blocks of
// a row block share them in L2), and the rows of X a super-group gathers
// -- for a 3-D stencil three grid planes of each of its columns around the
// advancing row front -- stay in L2 until every row that needs them has
// run, so X is read about once instead of once per neighbouring plane.
template <int B, int K, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) csr_spmm2_kernel(CsrArgs a) {
    const int64_t ncb = (a.k + K - 1) / K;
    const int64_t nrb = (a.m + kBlock - 1) / kBlock;
    const int64_t sg = (a.sg > 0 && a.sg < ncb) ? a.sg : ncb;  // column blocks per super-group
    const int64_t per_sg = sg * nrb;                           // CTAs per (full) super-group
    const int64_t g = blockIdx.x / per_sg, rest = blockIdx.x - g * per_sg;
    const int64_t w = min(sg, ncb - g * sg);                   // column blocks in this super-group
    const int64_t rb = rest / w, cb = g * sg + rest % w;
    const int64_t row = rb * kBlock + threadIdx.x;
    const int64_t col0 = cb * K;
    if (row >= a.m) return;
    const int s = __ldg(a.indptr + row);
    const int e = __ldg(a.indptr + row + 1);
    double acc[K];
#pragma unroll
    for (int kk = 0; kk < K; ++kk) acc[kk] = 0.0;
    // gather addresses: X + c + (col0 + kk) ldx, formed as one wide
    // multiply-add per gather from the entry's column-block base (a clamped
    // column re-reads the block's first column; its sums are not stored)
    const double *xb = a.X + col0 * a.ldx;
    const uint32_t cstride = (uint32_t)(a.ldx * 8);  // bytes between columns (host checks < 2^32 / K)
    uint32_t coff[K];
#pragma unroll
    for (int kk = 0; kk < K; ++kk) coff[kk] = (col0 + kk < a.k ? (uint32_t)kk : 0u);
    auto gat = [&](int c, int kk) {
        const char *p = reinterpret_cast<const char *>(xb + c);
        return __ldg(reinterpret_cast<const double *>(p + (uint64_t)coff[kk] * cstride));
    };
    int q0 = s;
    for (; q0 + B <= e; q0 += B) {  // full batches: no predicates
        int c[B];
        double v[B];
#pragma unroll
        for (int h = 0; h < B; ++h) {
            c[h] = __ldg(a.indices + q0 + h);
            v[h] = __ldg(a.data + q0 + h);
        }
        double xv[K][B];
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
#pragma unroll
            for (int h = 0; h < B; ++h) xv[kk][h] = gat(c[h], kk);
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
#pragma unroll
            for (int h = 0; h < B; ++h) acc[kk] = __dadd_rn(acc[kk], __dmul_rn(v[h], xv[kk][h]));
    }
    for (; q0 < e; ++q0) {  // the rest, one entry at a time (stored order)
        const int c = __ldg(a.indices + q0);
        const double v = __ldg(a.data + q0);
        double xv[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) xv[kk] = gat(c, kk);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) acc[kk] = __dadd_rn(acc[kk], __dmul_rn(v, xv[kk]));
    }
#pragma unroll
    for (int kk = 0; kk < K; ++kk)
        if (col0 + kk < a.k) a.Y[row + (col0 + kk) * a.ldy] = acc[kk];
}

template <int B>
__global__ void __launch_bounds__(kBlock) csr_row_kernel(CsrArgs a) {
    const int64_t nblocks = (a.m + kBlock - 1) / kBlock;
    for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
        const int64_t row = blk * kBlock + threadIdx.x;
        if (row >= a.m) continue;
        const int s = __ldg(a.indptr + row);
        const int e = __ldg(a.indptr + row + 1);
        if (e - s <= B && a.k > 1) {  // entries stay in registers across columns
            int c[B];
            double val[B];
#pragma unroll
            for (int h = 0; h < B; ++h) {
                const bool ok = s + h < e;
                c[h] = ok ? __ldg(a.indices + s + h) : 0;
                val[h] = ok ? __ldg(a.data + s + h) : 0.0;
            }
            // kSpmmUnroll columns per block: all their gathers are issued
            // before the first store (a store to Y could alias X as far as
            // the compiler knows, which would serialize the columns)
            int64_t col = 0;
            for (; col + kSpmmUnroll <= a.k; col += kSpmmUnroll) {
                double xv[kSpmmUnroll][B];
#pragma unroll
                for (int u = 0; u < kSpmmUnroll; ++u) {
                    const double *x = a.X + (col + u) * a.ldx;
#pragma unroll
                    for (int h = 0; h < B; ++h) xv[u][h] = s + h < e ? __ldg(x + c[h]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kSpmmUnroll; ++u) {
                    double acc = 0.0;
#pragma unroll
                    for (int h = 0; h < B; ++h)
                        if (s + h < e) acc = __dadd_rn(acc, __dmul_rn(val[h], xv[u][h]));
                    a.Y[row + (col + u) * a.ldy] = acc;
                }
            }
            for (; col < a.k; ++col) {
                const double *x = a.X + col * a.ldx;
                double xv[B];
#pragma unroll
                for (int h = 0; h < B; ++h) xv[h] = s + h < e ? __ldg(x + c[h]) : 0.0;
                double acc = 0.0;
#pragma unroll
                for (int h = 0; h < B; ++h)
                    if (s + h < e) acc = __dadd_rn(acc, __dmul_rn(val[h], xv[h]));
                a.Y[row + col * a.ldy] = acc;
            }
        } else {
            for (int64_t col = 0; col < a.k; ++col)
                a.Y[row + col * a.ldy] = csr_row<B>(a, a.X + col * a.ldx, s, e, false, 0.0);
        }
    }
}

// The fused step of virtual CTA `cta` of the canonical norm grid G (called by
// all kBlock threads of a CTA).
template <int B>
__device__ __forceinline__ void csr_step_body(const CsrArgs &a, int64_t cta, int64_t G) {
    const bool upd = a.r != nullptr;
    const int64_t nblk = (a.m + kBlock - 1) / kBlock;
    double t = 0.0, zz = 0.0, xx = 0.0;
    int64_t row = cta * kBlock + threadIdx.x;
    int s = row < a.m ? __ldg(a.indptr + row) : 0;
    int e = row < a.m ? __ldg(a.indptr + row + 1) : 0;
    const double rj = a.rin.partial ? rrow_first(a.rin, cta == 0) : (upd ? *a.r : 0.0);
    for (int64_t blk = cta; blk < nblk; blk += G) {
        const int64_t nrow = row + G * kBlock;  // prefetch the next owned row's pointers
        const int ns = nrow < a.m ? __ldg(a.indptr + nrow) : 0;
        const int ne = nrow < a.m ? __ldg(a.indptr + nrow + 1) : 0;
        if (row < a.m) {
            int sa[1] = {s}, ea[1] = {e};
            double y[1];
            csr_rows<1, B>(a, sa, ea, upd, rj, y);
            double z = a.X[row];
            if (upd) z = __dsub_rn(z, __dmul_rn(rj, a.qprev[row]));
            a.Y[row] = y[0];
            if (a.znew) a.znew[row] = z;
            t = fma(z, y[0], t);
            zz = fma(z, z, zz);
            xx = fma(y[0], y[0], xx);
        }
        row = nrow;
        s = ns;
        e = ne;
    }
    pdl_trigger();
    norm_cta_partial(a.out, t, zz, xx, cta);
    norm_last_cta(a.out, (unsigned)G);
}

// Software-pipelined variant: while the gathers of row r are in flight, the
// (index, value) entries of row r + G*256 and the pointers of the row after
// it are already loading, so each row costs one dependent round trip instead
// of two.  Same rows, order and arithmetic as csr_step_body (bitwise equal).
template <int B>
__device__ __forceinline__ void load_entries(const CsrArgs &a, int s, int e, int (&c)[B], double (&v)[B]) {
#pragma unroll
    for (int h = 0; h < B; ++h) {
        const bool ok = s + h < e;
        c[h] = ok ? __ldg(a.indices + s + h) : 0;
        v[h] = ok ? __ldg(a.data + s + h) : 0.0;
    }
}

// PRE: the first rows' pointers and entries (the operator is read-only for
// the whole factorization) are loaded before the grid-dependency wait, so
// their two dependent round trips overlap the tail of the previous kernel;
// returns false when an earlier step failed.
template <int B, bool PRE = false>
__device__ __forceinline__ bool csr_step_body_pf(const CsrArgs &a, int64_t cta, int64_t G) {
    const bool upd = a.r != nullptr;
    const int64_t nblk = (a.m + kBlock - 1) / kBlock;
    const int64_t stride = G * kBlock;
    double t = 0.0, zz = 0.0, xx = 0.0;
    int64_t row = cta * kBlock + threadIdx.x;
    int s = row < a.m ? __ldg(a.indptr + row) : 0;
    int e = row < a.m ? __ldg(a.indptr + row + 1) : 0;
    int64_t nrow = row + stride;
    int ns = nrow < a.m ? __ldg(a.indptr + nrow) : 0;
    int ne = nrow < a.m ? __ldg(a.indptr + nrow + 1) : 0;
    int c[B];
    double v[B];
    load_entries<B>(a, s, e, c, v);
    if (PRE) {
        pdl_wait();
        if (failed(a.out.status)) return false;
    }
    const double rj = a.rin.partial ? rrow_first(a.rin, cta == 0) : (upd ? *a.r : 0.0);
    for (int64_t blk = cta; blk < nblk; blk += G) {
        // stage 1: pointers two rows ahead; stage 2: entries one row ahead
        const int64_t n2 = nrow + stride;
        const int s2 = n2 < a.m ? __ldg(a.indptr + n2) : 0;
        const int e2 = n2 < a.m ? __ldg(a.indptr + n2 + 1) : 0;
        int nc[B];
        double nv[B];
        load_entries<B>(a, ns, ne, nc, nv);
        if (row < a.m) {
            double y;
            if (e - s <= B) {  // stage 3: gathers and the stored-order sum of this row
                double xv[B];
#pragma unroll
                for (int h = 0; h < B; ++h) {
                    const bool ok = s + h < e;
                    xv[h] = ok ? __ldg(a.X + c[h]) : 0.0;
                    if (upd && ok) xv[h] = __dsub_rn(xv[h], __dmul_rn(rj, __ldg(a.qprev + c[h])));
                }
                y = 0.0;
#pragma unroll
                for (int h = 0; h < B; ++h)
                    if (s + h < e) y = __dadd_rn(y, __dmul_rn(v[h], xv[h]));
            } else {
                y = csr_row<B>(a, a.X, s, e, upd, rj);
            }
            double z = a.X[row];
            if (upd) z = __dsub_rn(z, __dmul_rn(rj, a.qprev[row]));
            a.Y[row] = y;
            if (a.znew) a.znew[row] = z;
            t = fma(z, y, t);
            zz = fma(z, z, zz);
            xx = fma(y, y, xx);
        }
        row = nrow;
        s = ns;
        e = ne;
        nrow = n2;
        ns = s2;
        ne = e2;
#pragma unroll
        for (int h = 0; h < B; ++h) {
            c[h] = nc[h];
            v[h] = nv[h];
        }
    }
    pdl_trigger();
    norm_cta_partial(a.out, t, zz, xx, cta);
    norm_last_cta(a.out, (unsigned)G);
    return true;
}

// Deeper pipeline (default; build knob AQR_SPMV_PF2 = 2: L2, 1: L1, 0: the
// csr_step_body_pf form): pointers three rows ahead, the entries of the row
// after next prefetched into the cache, the next row's entries loaded into
// registers (now a cache hit), and a row's X and q gathers all issued before
// the arithmetic.  Config 2 HA 7.31 -> 7.20 ms, CGS-HA 9.45 -> 9.37-9.44 ms
// (alternating builds, tools/ab_libs.sh); prefetching the next row's gathers
// too was slower (spills).  Same rows, order and arithmetic as
// csr_step_body_pf (bitwise equal).
#ifndef AQR_SPMV_PF2
#define AQR_SPMV_PF2 2
#endif
__device__ __forceinline__ void prefetch_entries(const CsrArgs &a, int s, int e) {
    if (e <= s) return;
    if (AQR_SPMV_PF2 == 1) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.indices + s));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.data + s));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.data + e - 1));
    } else {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.indices + s));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.data + s));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.data + e - 1));
    }
}

template <int B, bool PRE = false>
__device__ __forceinline__ bool csr_step_body_pf2(const CsrArgs &a, int64_t cta, int64_t G) {
    const bool upd = a.r != nullptr;
    const int64_t nblk = (a.m + kBlock - 1) / kBlock;
    const int64_t stride = G * kBlock;
    double t = 0.0, zz = 0.0, xx = 0.0;
    int64_t row = cta * kBlock + threadIdx.x;
    int s = row < a.m ? __ldg(a.indptr + row) : 0;
    int e = row < a.m ? __ldg(a.indptr + row + 1) : 0;
    int64_t nrow = row + stride;
    int ns = nrow < a.m ? __ldg(a.indptr + nrow) : 0;
    int ne = nrow < a.m ? __ldg(a.indptr + nrow + 1) : 0;
    int64_t n2 = nrow + stride;
    int s2 = n2 < a.m ? __ldg(a.indptr + n2) : 0;
    int e2 = n2 < a.m ? __ldg(a.indptr + n2 + 1) : 0;
    int c[B];
    double v[B];
    load_entries<B>(a, s, e, c, v);
    prefetch_entries(a, ns, ne);
    if (PRE) {
        pdl_wait();
        if (failed(a.out.status)) return false;
    }
    const double rj = a.rin.partial ? rrow_first(a.rin, cta == 0) : (upd ? *a.r : 0.0);
    for (int64_t blk = cta; blk < nblk; blk += G) {
        // stage 0: pointers three rows ahead; stage 1: entries two rows ahead
        // toward the cache; stage 2: entries of the next row into registers
        const int64_t n3 = n2 + stride;
        const int s3 = n3 < a.m ? __ldg(a.indptr + n3) : 0;
        const int e3 = n3 < a.m ? __ldg(a.indptr + n3 + 1) : 0;
        prefetch_entries(a, s2, e2);
        int nc[B];
        double nv[B];
        load_entries<B>(a, ns, ne, nc, nv);
        if (row < a.m) {
            double y;
            if (e - s <= B) {
                double xv[B], qv[B];
#pragma unroll
                for (int h = 0; h < B; ++h) {
                    const bool ok = s + h < e;
                    xv[h] = ok ? __ldg(a.X + c[h]) : 0.0;
                    qv[h] = (upd && ok) ? __ldg(a.qprev + c[h]) : 0.0;
                }
#pragma unroll
                for (int h = 0; h < B; ++h)
                    if (upd && s + h < e) xv[h] = __dsub_rn(xv[h], __dmul_rn(rj, qv[h]));
                y = 0.0;
#pragma unroll
                for (int h = 0; h < B; ++h)
                    if (s + h < e) y = __dadd_rn(y, __dmul_rn(v[h], xv[h]));
            } else {
                y = csr_row<B>(a, a.X, s, e, upd, rj);
            }
            double z = a.X[row];
            if (upd) z = __dsub_rn(z, __dmul_rn(rj, a.qprev[row]));
            a.Y[row] = y;
            if (a.znew) a.znew[row] = z;
            t = fma(z, y, t);
            zz = fma(z, z, zz);
            xx = fma(y, y, xx);
        }
        row = nrow;
        s = ns;
        e = ne;
        nrow = n2;
        ns = s2;
        ne = e2;
        n2 = n3;
        s2 = s3;
        e2 = e3;
#pragma unroll
        for (int h = 0; h < B; ++h) {
            c[h] = nc[h];
            v[h] = nv[h];
        }
    }
    pdl_trigger();
    if (a.out.npart != nullptr) {  // uniform; nullptr: plain y = A x (k = 1)
        norm_cta_partial(a.out, t, zz, xx, cta);
        norm_last_cta(a.out, (unsigned)G);
    }
    return true;
}

// AQR_SPMV_PREWAIT=0: wait before any load (A/B; config 2 HA 7.60 vs 7.62 ms).
#ifndef AQR_SPMV_PREWAIT
#define AQR_SPMV_PREWAIT 1
#endif
template <int B, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) csr_step_pf_kernel(CsrArgs a) {
    trace_mark(a.trace, 0);
    if (!AQR_SPMV_PREWAIT) {
        pdl_wait();
        if (failed(a.out.status)) return;
    }
    trace_mark(a.trace, 1);  // with PRE: before the wait
    if (AQR_SPMV_PF2 != 0) {
        if (!csr_step_body_pf2<B, AQR_SPMV_PREWAIT != 0>(a, blockIdx.x, gridDim.x)) return;
    } else {
        if (!csr_step_body_pf<B, AQR_SPMV_PREWAIT != 0>(a, blockIdx.x, gridDim.x)) return;
    }
    rrow_rest(a.rin, blockIdx.x, gridDim.x);
    trace_mark(a.trace, 2);
}

// Fused HA/naive step, launched with exactly norm_tiles(m) CTAs (the
// canonical norm grid): CTA b handles rows of the 256-row blocks b, b+G, ...
// one per thread, accumulating the norm chains in ascending block order; the
// next row's pointers are prefetched; one block tree per CTA at the end.
template <int B, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) csr_step_kernel(CsrArgs a) {
    trace_mark(a.trace, 0);
    pdl_wait();
    trace_mark(a.trace, 1);
    if (failed(a.out.status)) return;
    csr_step_body<B>(a, blockIdx.x, gridDim.x);
    rrow_rest(a.rin, blockIdx.x, gridDim.x);
    trace_mark(a.trace, 2);
}

// ---------------------------------------------------------------------------
// Dense operator: GEMV / GEMM, reference-exact (ascending column index)
// ---------------------------------------------------------------------------
// y = A x, one thread per row, ascending j, separately rounded (bitwise equal
// to matvec, _kernels_impl.py:24-32).  Loads of A are coalesced across the
// warp (column-major); x is staged in shared memory in chunks.
constexpr int kGemvBlock = 64;
constexpr int kGemvU = 16;
// Software-pipelined: the next 16 columns of A are in flight while the
// current 16 are accumulated (32 loads per thread outstanding); x[j] is a
// warp-uniform (broadcast) load.  With one row per thread, m = 32768 gives
// only ~7 warps per SM, so the loads in flight per thread set the bandwidth.
__global__ void __launch_bounds__(kGemvBlock)
    dense_gemv_kernel(int64_t m, int64_t ncols, const double *__restrict__ A, int64_t lda,
                      const double *__restrict__ X, int64_t ldx, double *__restrict__ Y,
                      int64_t ldy) {
    constexpr int U = kGemvU;
    const int64_t row = blockIdx.x * (int64_t)kGemvBlock + threadIdx.x;
    if (row >= m) return;
    const double *x = X + blockIdx.y * ldx;
    const double *arow = A + row;
    double acc = 0.0;
    const int64_t full = ncols / U * U;
    double a0[U], a1[U];
    if (full > 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) a0[u] = __ldg(arow + u * lda);
    }
    for (int64_t j = 0; j < full; j += 2 * U) {
        const bool has1 = j + U < full, has2 = j + 2 * U < full;
        if (has1) {
#pragma unroll
            for (int u = 0; u < U; ++u) a1[u] = __ldg(arow + (j + U + u) * lda);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(a0[u], __ldg(x + j + u)));
        if (!has1) break;
        if (has2) {
#pragma unroll
            for (int u = 0; u < U; ++u) a0[u] = __ldg(arow + (j + 2 * U + u) * lda);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, __dmul_rn(a1[u], __ldg(x + j + U + u)));
    }
    for (int64_t j = full; j < ncols; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(arow + j * lda), __ldg(x + j)));
    Y[row + blockIdx.y * ldy] = acc;
}

// y = A x streamed by TMA (the north star's "x staged in shared memory"):
// a CTA owns kGvRows rows; one producer warp streams kGvCols-column panels
// of A (kGvCols bulk copies of one column segment each, contiguous in the
// column-major layout) plus the matching slice of x into a kGvStages-deep
// shared-memory ring with mbarrier transaction counts; consumer thread r
// accumulates row r over ascending j from shared memory -- the reference's
// order, bitwise matvec.  The bytes in flight no longer depend on registers
// (one row per thread gives only ~7 warps per SM at m = 32768).
// Requires lda, m even (16-byte-aligned segments); else dense_gemv_kernel.
constexpr int kGvRows = 128, kGvCols = 32, kGvStages = 3;
constexpr size_t kGvStageBytes = (size_t)kGvRows * kGvCols * 8 + kGvCols * 8;
constexpr size_t kGvSmem = kGvStages * kGvStageBytes + 2 * kGvStages * 8;
__device__ __forceinline__ void gv_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__global__ void __launch_bounds__(kGvRows + 32, 2)
    dense_gemv_tma_kernel(int64_t m, int64_t ncols, const double *__restrict__ A, int64_t lda,
                          const double *__restrict__ x, double *__restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kGvStages * kGvStageBytes);
    uint64_t *empty = full + kGvStages;
    const int64_t r0 = (int64_t)blockIdx.x * kGvRows;
    const int rows = (m - r0) < kGvRows ? (int)(m - r0) : kGvRows;
    const int64_t ntile = (ncols + kGvCols - 1) / kGvCols;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kGvStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kGvRows / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kGvRows / 32) {  // producer
        if (lane == 0) {
            for (int64_t t = 0; t < ntile; ++t) {
                const int s = (int)(t % kGvStages);
                const uint32_t ph = (uint32_t)((t / kGvStages) & 1);
                const int64_t j0 = t * kGvCols;
                const int cols = (ncols - j0) < kGvCols ? (int)(ncols - j0) : kGvCols;
                mbar_wait(empty + s, ph ^ 1);
                mbar_expect_tx(full + s, (uint32_t)(cols * rows * 8 + ((cols * 8 + 15) & ~15)));
                double *dst = reinterpret_cast<double *>(smem + s * kGvStageBytes);
                for (int c = 0; c < cols; ++c)
                    bulk_g2s<false>(dst + c * kGvRows, A + r0 + (j0 + c) * lda, (uint32_t)(rows * 8),
                                    full + s, 0);
                bulk_g2s<false>(dst + kGvRows * kGvCols, x + j0, (uint32_t)((cols * 8 + 15) & ~15),
                                full + s, 0);
            }
        }
        return;
    }
    double acc = 0.0;
    for (int64_t t = 0; t < ntile; ++t) {
        const int s = (int)(t % kGvStages);
        const uint32_t ph = (uint32_t)((t / kGvStages) & 1);
        const int64_t j0 = t * kGvCols;
        const int cols = (ncols - j0) < kGvCols ? (int)(ncols - j0) : kGvCols;
        mbar_wait(full + s, ph);
        const double *src = reinterpret_cast<const double *>(smem + s * kGvStageBytes);
        const double *xs = src + kGvRows * kGvCols;
        if (cols == kGvCols) {
#pragma unroll
            for (int c = 0; c < kGvCols; ++c)
                acc = __dadd_rn(acc, __dmul_rn(src[c * kGvRows + threadIdx.x], xs[c]));
        } else {
            for (int c = 0; c < cols; ++c)
                acc = __dadd_rn(acc, __dmul_rn(src[c * kGvRows + threadIdx.x], xs[c]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
    if (threadIdx.x < rows) y[r0 + threadIdx.x] = acc;
}

// Y = A X (k columns): 128 x 64 output tiles, 16-deep k slices, every
// output accumulated over ascending j with separate rounding -- bitwise equal
// to k matvecs (apply_block_dense, _kernels_impl.py:35-47).
constexpr int kG2BM = 128, kG2BN = 64, kG2BK = 16;

// Same tiles, operands streamed into a 3-stage shared-memory ring with
// cp.async (no register staging: <= 128 registers, 2 CTAs per SM).
constexpr int kG3Stages = 3;
constexpr size_t kG3StageWords = (size_t)kG2BK * kG2BM + (size_t)kG2BK * kG2BN;
constexpr size_t kG3Smem = kG3Stages * kG3StageWords * sizeof(double);
__device__ __forceinline__ void cp_async8_g2s(double *dst, const double *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__global__ void __launch_bounds__(256, 2)
    dense_gemm3_kernel(int64_t m, int64_t ncols, int64_t k, const double *__restrict__ A, int64_t lda,
                       const double *__restrict__ X, int64_t ldx, double *__restrict__ Y, int64_t ldy) {
    extern __shared__ __align__(16) double g3[];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t i0 = (int64_t)blockIdx.x * kG2BM, c0 = (int64_t)blockIdx.y * kG2BN;
    const int64_t nk = (ncols + kG2BK - 1) / kG2BK;
    auto As = [&](int st) { return g3 + (size_t)st * kG3StageWords; };            // [BK][BM]
    auto Xs = [&](int st) { return g3 + (size_t)st * kG3StageWords + kG2BK * kG2BM; };  // [BK][BN]
    auto issue = [&](int64_t kt) {
        if (kt < nk) {
            const int st = (int)(kt % kG3Stages);
            const int64_t j0 = kt * kG2BK;
            double *as = As(st), *xs = Xs(st);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int ii = tid & 127, jj = (tid >> 7) + 2 * u;
                const int64_t gi = i0 + ii, gj = j0 + jj;
                if (gi < m && gj < ncols) cp_async8_g2s(as + jj * kG2BM + ii, A + gi + gj * lda);
                else as[jj * kG2BM + ii] = 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int jj = tid & 15, cc = (tid >> 4) + 16 * u;
                const int64_t gj = j0 + jj, gc = c0 + cc;
                if (gj < ncols && gc < k) cp_async8_g2s(xs + jj * kG2BN + cc, X + gj + gc * ldx);
                else xs[jj * kG2BN + cc] = 0.0;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
#pragma unroll
    for (int s = 0; s < kG3Stages - 1; ++s) issue(s);
    for (int64_t kt = 0; kt < nk; ++kt) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kG3Stages - 2) : "memory");
        __syncthreads();  // tile kt landed; tile kt-1's stage is free for kt+2
        issue(kt + kG3Stages - 1);
        const int st = (int)(kt % kG3Stages);
        const double *as = As(st), *xs = Xs(st);
        const int kmax = (ncols - kt * kG2BK) < kG2BK ? (int)(ncols - kt * kG2BK) : kG2BK;
        if (kmax == kG2BK) {
#pragma unroll
            for (int jj = 0; jj < kG2BK; ++jj) {
                double av[8], xv[4];
#pragma unroll
                for (int a = 0; a < 8; ++a) av[a] = as[jj * kG2BM + ty + 16 * a];
#pragma unroll
                for (int b = 0; b < 4; ++b) xv[b] = xs[jj * kG2BN + tx + 16 * b];
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(av[a], xv[b]));
            }
        } else {
            for (int jj = 0; jj < kmax; ++jj) {
                double av[8], xv[4];
#pragma unroll
                for (int a = 0; a < 8; ++a) av[a] = as[jj * kG2BM + ty + 16 * a];
#pragma unroll
                for (int b = 0; b < 4; ++b) xv[b] = xs[jj * kG2BN + tx + 16 * b];
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(av[a], xv[b]));
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gi = i0 + ty + 16 * a, gc = c0 + tx + 16 * b;
            if (gi < m && gc < k) Y[gi + gc * ldy] = acc[a][b];
        }
}

}  // namespace aqr
