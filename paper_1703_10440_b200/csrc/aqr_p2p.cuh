// aqr_p2p.cuh -- multi-GPU step kernels with the exchanges fused in, over
// NVLink / NVSwitch peer memory (one process per GPU, CUDA IPC mappings).
//
// The row-partitioned schedule of distributed.py has
// three exchanges per MGS step: the SpMV halo, the all-reduce of the norm
// partials (3 doubles) and the all-reduce of the R row (n-1-i doubles).  Here
// none of them is a separate collective call:
//
//   * halo: the fused SpMV step gathers the boundary rows it needs straight
//     from the owning rank's working matrix (peer loads), applying the
//     deferred projection z - r q on the fly exactly as for its own rows;
//   * all-reduces: the kernel that forms a rank's local totals stores them
//     into EVERY rank's exchange buffer (slot [parity][source rank]) and then
//     releases a flag there; the consumer kernel acquires all flags and adds
//     the slots in rank order 0..N-1, so every rank gets bitwise the same sum
//     and (N = 1) bitwise the single-GPU result.
//
// Ordering argument (why no extra barrier is needed):
//   * a rank reads a peer's columns z_i, q_{i-1} during its SpMV of step i,
//     after acquiring the peer's R-row flag of step i-1, which the peer
//     released after its trailing pass of step i-1 (the last writer of
//     those columns) -- step 0 waits for the start barrier instead;
//   * the peer overwrites column i (with q_i) only in its trailing pass of
//     step i, which needs the norm totals of step i, which include this
//     rank's contribution, released only after all of this rank's gathers;
//   * exchange slots alternate by step parity; a slot is rewritten two steps
//     later, which requires every rank to have consumed it.
// Flags hold monotonically increasing sequence numbers (a per-group counter
// advanced by n + 2 per factorization), so nothing is reset between calls.
#pragma once

#include "aqr_kernels.cuh"

namespace aqr {

constexpr int kMaxRanks = 8;
enum { kFlagNorm = 0, kFlagRrow = 1, kFlagBar = 2, kFlagKinds = 3 };

// Exchange buffer of one rank (doubles, then uint64 flags):
//   rrow  [2][kMaxRanks][n]   R-row local totals, absolute column index
//   norm  [2][kMaxRanks][4]   (z.x, z.z, x.x) local totals
//   flags [kFlagKinds][kMaxRanks]
__host__ __device__ inline int64_t xb_rrow(int64_t n, int par, int src) {
    return ((int64_t)par * kMaxRanks + src) * n;
}
__host__ __device__ inline int64_t xb_norm(int64_t n, int par, int src) {
    return 2 * kMaxRanks * n + ((int64_t)par * kMaxRanks + src) * 4;
}
__host__ __device__ inline int64_t xb_flags(int64_t n) { return 2 * kMaxRanks * n + 2 * kMaxRanks * 4; }
__host__ __device__ inline int64_t xb_words(int64_t n) { return xb_flags(n) + kFlagKinds * kMaxRanks; }

struct P2PArgs {
    int32_t nranks, rank;
    double *xb[kMaxRanks];       // exchange buffers of all ranks (peer mappings; own = local)
    const double *W[kMaxRanks];  // working matrices of all ranks (peer mappings)
    int64_t ldw[kMaxRanks];
    int64_t n;
    uint64_t seq0;  // start barrier = seq0; norm / R row of step i = seq0 + 1 + i
    int64_t m_loc;
    const int32_t *halo_rank;  // extended column m_loc + h lives on rank halo_rank[h] ...
    const int32_t *halo_row;   // ... at its local row halo_row[h]
    int32_t *status;           // this rank's status block (timeout record: [1] = 1)
    uint64_t timeout_ns;       // longest wait for one flag
};

__device__ __forceinline__ uint64_t *xb_flag(double *xb, int64_t n, int kind, int src) {
    return reinterpret_cast<uint64_t *>(xb + xb_flags(n)) + kind * kMaxRanks + src;
}
__device__ __forceinline__ void flag_release(uint64_t *f, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t flag_acquire(const uint64_t *f) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
    return v;
}

// One thread: make this thread's (and, after a CTA barrier, its CTA's) prior
// peer stores visible system-wide, then raise `kind` to v on every rank.
__device__ __forceinline__ void publish(const P2PArgs &p, int kind, uint64_t v) {
    __threadfence_system();
    for (int r = 0; r < p.nranks; ++r) flag_release(xb_flag(p.xb[r], p.n, kind, p.rank), v);
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One thread: wait until every rank raised `kind` to at least v.  Bounded:
// a wait longer than p.timeout_ns (a peer died or was never launched)
// records the timeout in the status block -- [1] = 1 and [0] set, so every
// later kernel of this rank returns at its status check -- and gives up;
// it also gives up as soon as the status block records a failure.  Returns
// false when it gave up.
__device__ __forceinline__ bool wait_all(const P2PArgs &p, int kind, uint64_t v) {
    const uint64_t t0 = global_ns();
    for (int src = 0; src < p.nranks; ++src) {
        const uint64_t *f = xb_flag(p.xb[p.rank], p.n, kind, src);
        while (flag_acquire(f) < v) {
            if (failed(p.status)) return false;
            if (global_ns() - t0 > p.timeout_ns) {
                atomicExch(p.status + 1, 1);
                atomicCAS(p.status, -1, 0x7fffffff);
                __threadfence_system();
                return false;
            }
            __nanosleep(200);
        }
    }
    return true;
}

__device__ __forceinline__ uint64_t seq_step(const P2PArgs &p, int64_t i) { return p.seq0 + 1 + (uint64_t)i; }

// Rank-ordered sum of slot values (deterministic; N = 1 returns the value).
__device__ __forceinline__ double sum_ranks(const P2PArgs &p, int64_t off0, int64_t stride) {
    const double *b = p.xb[p.rank];
    double s = __ldcg(b + off0);
    for (int src = 1; src < p.nranks; ++src) s = __dadd_rn(s, __ldcg(b + off0 + src * stride));
    return s;
}

// Prologue of a step-i norm kernel (all threads): wait for the R row of step
// i-1 (or, at i = 0, the start barrier), return r_{i-1,i}; CTA 0 also stores
// the global row i-1 of R (columns i..n-1) for the trailing pass.
__device__ __forceinline__ double p2p_rrow_in(const P2PArgs &p, int64_t i, double *Rt) {
    __shared__ double r_sh;
    if (threadIdx.x == 0) {
        if (i == 0) {
            wait_all(p, kFlagBar, p.seq0);
            r_sh = 0.0;
        } else {
            wait_all(p, kFlagRrow, seq_step(p, i - 1));
            r_sh = sum_ranks(p, xb_rrow(p.n, (int)((i - 1) & 1), 0) + i, p.n);
        }
    }
    __syncthreads();
    if (i > 0 && blockIdx.x == 0)
        for (int64_t j = i + threadIdx.x; j < p.n; j += kBlock)
            Rt[(i - 1) * p.n + j] = sum_ranks(p, xb_rrow(p.n, (int)((i - 1) & 1), 0) + j, p.n);
    return r_sh;
}

// Epilogue of a step-i norm kernel (all threads, after the CTA's partial was
// written): the last CTA forms the local totals and sends them to every rank.
__device__ __forceinline__ void p2p_norm_out(const P2PArgs &p, const NormOut &o, unsigned ctas, int64_t i) {
    if (!last_block(o.counter, ctas)) return;
    __shared__ double tot[3];
    __shared__ double sm3[3 * kWarps];
    block_totals<3>(o.npart, o.ntiles, o.ntiles, tot, sm3, SyncAll());
    if (threadIdx.x == 0) {
        const int par = (int)(i & 1);
        for (int r = 0; r < p.nranks; ++r) {
            double *dst = p.xb[r] + xb_norm(p.n, par, p.rank);
            dst[0] = tot[0];
            dst[1] = tot[1];
            dst[2] = tot[2];
        }
        publish(p, kFlagNorm, seq_step(p, i));
    }
}

__global__ void p2p_barrier_kernel(P2PArgs p) { publish(p, kFlagBar, p.seq0); }

// x - r q at extended column c: own rows from this rank's columns, halo rows
// from the owning rank's working matrix (peer loads, L2 of the owner).
__device__ __forceinline__ double p2p_xe(const CsrArgs &a, const P2PArgs &p, int64_t i, int c, bool upd,
                                         double rj) {
    double x, qv = 0.0;
    if (c < p.m_loc) {
        x = __ldg(a.X + c);
        if (upd) qv = __ldg(a.qprev + c);
    } else {
        const int64_t hh = c - p.m_loc;
        const int pr = __ldg(p.halo_rank + hh);
        const int64_t rr = __ldg(p.halo_row + hh);
        const double *Wr = p.W[pr];
        x = __ldcg(Wr + i * p.ldw[pr] + rr);
        if (upd) qv = __ldcg(Wr + (i - 1) * p.ldw[pr] + rr);
    }
    return upd ? __dsub_rn(x, __dmul_rn(rj, qv)) : x;
}

// Fused SpMV step over the local rows (HA), halo columns gathered from the
// owning ranks; software-pipelined like csr_step_body_pf (the next row's
// entries load during this row's gathers).  Same per-row arithmetic and norm
// chains as the single-GPU kernels.
template <int B>
__global__ void __launch_bounds__(kBlock, 3) p2p_csr_step_kernel(CsrArgs a, P2PArgs p, int64_t i, double *Rt) {
    const bool upd = i > 0;
    const int64_t nblk = (a.m + kBlock - 1) / kBlock;
    const int64_t G = gridDim.x, stride = G * kBlock;
    double t = 0.0, zz = 0.0, xx = 0.0;
    int64_t row = blockIdx.x * (int64_t)kBlock + threadIdx.x;
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
    load_entries<B>(a, s, e, c, v);  // the operator is read-only: before the wait
    prefetch_entries(a, ns, ne);
    pdl_wait();
    if (failed(a.out.status)) return;
    const double rj = p2p_rrow_in(p, i, Rt);
    for (int64_t blk = blockIdx.x; blk < nblk; blk += G) {
        // as csr_step_body_pf2: pointers three rows ahead, the entries of the
        // row after next toward L2, the next row's entries into registers
        const int64_t n3 = n2 + stride;
        const int s3 = n3 < a.m ? __ldg(a.indptr + n3) : 0;
        const int e3 = n3 < a.m ? __ldg(a.indptr + n3 + 1) : 0;
        prefetch_entries(a, s2, e2);
        int nc[B];
        double nv[B];
        load_entries<B>(a, ns, ne, nc, nv);
        if (row < a.m) {
            double y = 0.0;
            if (e - s <= B) {
                double xv[B];
#pragma unroll
                for (int h = 0; h < B; ++h) xv[h] = s + h < e ? p2p_xe(a, p, i, c[h], upd, rj) : 0.0;
#pragma unroll
                for (int h = 0; h < B; ++h)
                    if (s + h < e) y = __dadd_rn(y, __dmul_rn(v[h], xv[h]));
            } else {
                for (int q = s; q < e; ++q)
                    y = __dadd_rn(y, __dmul_rn(__ldg(a.data + q), p2p_xe(a, p, i, __ldg(a.indices + q), upd, rj)));
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
    norm_cta_partial(a.out, t, zz, xx, blockIdx.x);
    p2p_norm_out(p, a.out, gridDim.x, i);
}

// HP, lazy x (as col_lazy_norm_kernel): r_{i-1,i} and row i-1 of R from the
// exchanged R rows, x_i formed from the stored X_i and the p window, the
// deferred z_i update, the norm partials -> every rank.
__global__ void __launch_bounds__(kBlock, 4) p2p_col_lazy_kernel(ColArgs a, P2PArgs p, int64_t i, double *Rt) {
    pdl_wait();
    if (failed(a.out.status)) return;
    const double rj = p2p_rrow_in(p, i, Rt);
    double t, zz, xx;
    col_lazy_body(a, rj, i > 0, t, zz, xx);
    norm_cta_partial(a.out, t, zz, xx, blockIdx.x);
    p2p_norm_out(p, a.out, gridDim.x, i);
}

// Trailing pass of step i: global norm totals (rank-ordered) -> r_ii, the
// breakdown / flag record (CTA 0), then the pass over the local rows
// (WIN: the windowed Z-only pass, trail_body_w).
template <int RPT, int CU, bool HP, bool CGS, bool WIN>
__global__ void __launch_bounds__(kBlock) p2p_trailing_kernel(TrailArgs a, P2PArgs p, int64_t i, double *rii_out,
                                                              int32_t *status) {
    // as trailing_kernel: odd steps walk the units backwards, and this
    // unit's first tiles are prefetched into L2 before the dependency wait
    const int tile = a.reverse ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
    const int group = a.reverse ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y;
    trail_prefetch<RPT>(a, tile, group);
    pdl_wait();
    if (failed(a.status)) return;
    extern __shared__ double wsum[];
    __shared__ double rii_sh;
    __shared__ int ok_sh;
    if (threadIdx.x == 0) ok_sh = 0;
    if (threadIdx.x == 0 && wait_all(p, kFlagNorm, seq_step(p, i))) {
        const int par = (int)(i & 1);
        const double t = sum_ranks(p, xb_norm(p.n, par, 0) + 0, 4);
        const double zz = sum_ranks(p, xb_norm(p.n, par, 0) + 1, 4);
        const double xx = sum_ranks(p, xb_norm(p.n, par, 0) + 2, 4);
        if (blockIdx.x == 0 && blockIdx.y == 0) norm_finish_dev(i, t, zz, xx, rii_out, status);
        ok_sh = (t > 0.0) && isfinite(t);
        rii_sh = sqrt(t);  // norm_finish_dev's r_ii (gram_schmidt.py:159)
    }
    __syncthreads();
    if (!ok_sh) return;
    TrailArgs b = a;
    b.rii = &rii_sh;
    if (WIN)
        trail_body_w<RPT, CU, CGS>(b, tile, group, wsum);
    else
        trail_body<RPT, CU, HP, CGS>(b, tile, group, wsum);
}

// Local R-row totals of step i (CTA c: column jbeg + c), sent to every rank;
// the last CTA releases the R-row flag.
__global__ void __launch_bounds__(kBlock) p2p_rrow_kernel(const double *partial, int32_t ntiles, int64_t jbeg,
                                                          P2PArgs p, int64_t i, unsigned *counter,
                                                          const int32_t *status) {
    pdl_wait();
    pdl_trigger();  // the next step's SpMV may launch (it waits for this grid)
    if (failed(status)) return;
    __shared__ double tot[1];
    __shared__ double sm[kWarps];
    block_totals<1>(partial + (int64_t)blockIdx.x * ntiles, ntiles, ntiles, tot, sm, SyncAll());
    __shared__ unsigned ticket;
    if (threadIdx.x == 0) {
        const int par = (int)(i & 1);
        for (int r = 0; r < p.nranks; ++r) p.xb[r][xb_rrow(p.n, par, p.rank) + jbeg + blockIdx.x] = tot[0];
        __threadfence_system();
        ticket = atomicAdd(counter, 1u);
        if (ticket == gridDim.x - 1) {
            *counter = 0u;
            publish(p, kFlagRrow, seq_step(p, i));
        }
    }
}

// HP block apply X = A Z with halo columns from the owning ranks (after the
// start barrier).  Per output entry the stored-order sum of csr_row.
__global__ void __launch_bounds__(kBlock) p2p_csr_block_kernel(CsrArgs a, P2PArgs p) {
    if (threadIdx.x == 0) wait_all(p, kFlagBar, p.seq0);
    __syncthreads();
    const int64_t nblocks = (a.m + kBlock - 1) / kBlock;
    for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
        const int64_t row = blk * kBlock + threadIdx.x;
        if (row >= a.m) continue;
        const int s = __ldg(a.indptr + row), e = __ldg(a.indptr + row + 1);
        for (int64_t col = 0; col < a.k; ++col) {
            double y = 0.0;
            for (int q = s; q < e; ++q) {
                const int c = __ldg(a.indices + q);
                double x;
                if (c < p.m_loc) {
                    x = __ldg(a.X + col * a.ldx + c);
                } else {
                    const int64_t hh = c - p.m_loc;
                    const int pr = __ldg(p.halo_rank + hh);
                    x = __ldcg(p.W[pr] + col * p.ldw[pr] + __ldg(p.halo_row + hh));
                }
                y = __dadd_rn(y, __dmul_rn(__ldg(a.data + q), x));
            }
            a.Y[row + col * a.ldy] = y;
        }
    }
}

}  // namespace aqr
