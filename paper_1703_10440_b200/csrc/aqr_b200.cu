// aqr_b200.cu -- C ABI (include/aqr_b200.h) and the native step sequencer of
// the A-orthogonal MGS factorization on B200 (sm_100a).
//
// The sequencer restates gram_schmidt._gs_factor
// (/root/reference/pkg/src/aqr/gram_schmidt.py:126-179) as a one-pass-per-
// step schedule: step i of the row form applies the deferred projection of
// step i-1 to every trailing column and accumulates p_i . z_j in the same
// HBM pass ("fused trailing pass").  With a native CSR operator a
// HA/naive step is two launches: the fused SpMV step (z update + x = A z +
// norm + r_ii) and the fused trailing pass (+ the r row); both finish their
// reductions in the last CTA, so there are no separate reduction launches.
// The column form runs the same kernels one column at a time, so both
// orientations return bitwise-identical Q, R.
#include <cuda.h>  // driver types for cuStreamWaitValue32 (fetched at run time, no link)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/aqr_b200.h"
#include "aqr_dense.cuh"
#include "aqr_dgemm.cuh"
#include "aqr_kernels.cuh"
#include "aqr_band.cuh"
#include "aqr_p2p.cuh"

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

aqr_status set_err(aqr_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

#define AQR_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_err(AQR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define AQR_TRY(expr)                \
    do {                             \
        aqr_status s_ = (expr);      \
        if (s_ != AQR_OK) return s_; \
    } while (0)

aqr_status launched(const char *what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(AQR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return AQR_OK;
}

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int elementwise_grid(int64_t m) {
    int64_t g = (m + aqr::kBlock - 1) / aqr::kBlock;
    return (int)std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 16);
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cached[dev] == 0) {
        int v = 148;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

// Opt a kernel into > 48 KB of dynamic shared memory (once per device and
// kernel: the attribute is sticky, and setting it on every launch costs
// host time on the latency-bound small steps).
template <typename K>
aqr_status ensure_smem(K kernel, size_t bytes) {
    if (bytes == 0) return AQR_OK;  // (static + dynamic > 48 KB needs the opt-in too)
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void *, int>, size_t>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const void *key = reinterpret_cast<const void *>(kernel);
    std::lock_guard<std::mutex> lk(mu);
    for (auto &e : done)
        if (e.first.first == key && e.first.second == dev && e.second >= bytes) return AQR_OK;
    AQR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done.push_back({{key, dev}, bytes});
    return AQR_OK;
}

// ---- kernel timer (bench.py's roofline leg) ---------------------------------
// Slot 0: fused trailing pass; slot 1: fused SpMV step; slot 2: column
// update + norm; slot 3: HP X catch-up; slot 4: block apply (k > 1); slot 5:
// catch-up of a host-pipeline chunk.  When enabled, a CUDA event pair is recorded around every
// launch of those kernels on the launching stream.
struct KernelTimer {
    struct Rec {
        int slot;
        cudaEvent_t e0, e1;
        double bytes;
    };
    std::mutex mu;
    bool enabled = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<Rec> recs;
} g_timer;

cudaEvent_t timer_event() {
    if (g_timer.used == g_timer.pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        g_timer.pool.push_back(e);
    }
    return g_timer.pool[g_timer.used++];
}

// Returns the record index, or -1 when the timer is off.
long timer_begin(int slot, double bytes, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_timer.mu);
    if (!g_timer.enabled) return -1;
    cudaEvent_t e0 = timer_event(), e1 = timer_event();
    if (!e0 || !e1) return -1;
    cudaEventRecord(e0, s);
    g_timer.recs.push_back({slot, e0, e1, bytes});
    return (long)g_timer.recs.size() - 1;
}

void timer_end(long idx, cudaStream_t s) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_timer.mu);
    cudaEventRecord(g_timer.recs[(size_t)idx].e1, s);
}

// Experiment knobs.  The A/B measurements behind the design (tools/ab_*.sh,
// DESIGN.md) select alternative schedules through environment variables --
// but only in the experiments build (-DAQR_EXPERIMENTS,
// libaqr_b200_exp.so, _build.build_experiments()).  The shipped library
// compiles every knob to its default: no environment variable changes what
// it runs.
int knob(const char *name, int dflt) {
#ifdef AQR_EXPERIMENTS
    const char *e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
#else
    (void)name;
    return dflt;
#endif
}
#define AQR_KNOB(fn, name, dflt)                   \
    int fn() {                                     \
        static const int v = knob(name, dflt);     \
        return v;                                  \
    }

// AQR_CARVEOUT = -1 leaves the driver's choice, otherwise the preferred
// shared-memory carveout (percent) of the per-step kernels.
AQR_KNOB(carveout_pct, "AQR_CARVEOUT", -1)
// AQR_PDL=0: no programmatic dependent launch for the per-step kernels.
AQR_KNOB(pdl_mode, "AQR_PDL", 1)
// AQR_LDG_REVERSE=0: the trailing kernel always walks forwards.
AQR_KNOB(ldg_reverse_mode, "AQR_LDG_REVERSE", 1)
// AQR_TRAIL_VARIANT=6: the X-carrying (HP column loop) trailing pass with two
// columns per iteration for MGS (default one).
#ifdef AQR_EXPERIMENTS
AQR_KNOB(trail_variant, "AQR_TRAIL_VARIANT", 0)
// AQR_TRAIL_CU=4: the windowed MGS pass with four columns per iteration
AQR_KNOB(trail_cu, "AQR_TRAIL_CU", 2)
#endif
// AQR_SPMV_VARIANT=3: the unpipelined fused SpMV step.
AQR_KNOB(spmv_variant, "AQR_SPMV_VARIANT", 0)
// AQR_PLAIN_PF=0: plain SpMV on csr_row_kernel.
AQR_KNOB(plain_pf_mode, "AQR_PLAIN_PF", 1)
// AQR_TRAIL_CTAS: CTAs per SM the column grouping aims at.
AQR_KNOB(trail_ctas_knob, "AQR_TRAIL_CTAS", 3)
// AQR_COL_SCHEDULE=1: the column-oriented loop for the col methods.
AQR_KNOB(col_schedule_mode, "AQR_COL_SCHEDULE", 0)
// AQR_DIRECT=0: copy Z into Q first instead of reading Z in place.
AQR_KNOB(direct_mode, "AQR_DIRECT", 1)
// AQR_DEFER=0: a separate r-row reduction launch per step.
AQR_KNOB(defer_mode, "AQR_DEFER", 1)
// AQR_SPMV_REPEAT=k: k idempotent repeats of every fused SpMV step (diagnostics).
AQR_KNOB(spmv_repeat, "AQR_SPMV_REPEAT", 0)
// AQR_TRAIL_WIN=b: the row form's trailing block is written back every b-th
// pass (trailing_w_kernel; 1 = every pass, the eager schedule).
AQR_KNOB(trail_win_knob, "AQR_TRAIL_WIN", 4)
int trail_win() { return std::min(std::max(trail_win_knob(), 1), 8); }
// AQR_X_WIN=b: HP row form, the stored X columns catch up every b steps
// (0 = never: x_j formed from all j finished p columns).
AQR_KNOB(x_win_knob, "AQR_X_WIN", 16)
int64_t x_win() { return x_win_knob() > 0 ? x_win_knob() : (int64_t)1 << 40; }
// AQR_DGEMM=0: the HP block apply of a dense operator in the reference's
// sequential order (dense_gemm3_kernel) instead of the FP64 tensor cores;
// 2: the tensor cores for every size (default: operators >= 4096^2 entries).
AQR_KNOB(dgemm_mode, "AQR_DGEMM", 1)
// AQR_SPMM_SG=s: long-row SpMM (csr_spmm2_kernel) launch order, s column
// blocks of 8 per super-group (0: all column blocks of a row block adjacent).
AQR_KNOB(spmm_sg, "AQR_SPMM_SG", 4)
// AQR_SPLIT_LONG=0: HA steps with long CSR rows gather z and q_{j-1} in the
// fused SpMV step instead of a separate update pass.
AQR_KNOB(split_long_mode, "AQR_SPLIT_LONG", 1)
// AQR_BAND=0: ignore an operator's banded view (plain CSR kernels).
AQR_KNOB(band_mode, "AQR_BAND", 1)
// AQR_BAND_STAGE=0: the block apply of long banded rows gathers from global
// memory instead of staging the operand segments in shared memory.
AQR_KNOB(band_stage_mode, "AQR_BAND_STAGE", 1)
// AQR_PIPE_MERGE=0: the host-input pipeline catches up one chunk at a time.
AQR_KNOB(pipe_merge_mode, "AQR_PIPE_MERGE", 1)
// AQR_XC_STREAM=0: the periodic X catch-up on the column-group grid too.
AQR_KNOB(xc_stream_mode, "AQR_XC_STREAM", 1)
// AQR_XC_ROWS=r: rows per thread of the X catch-up (1, 2 or 4; CTAs/SM 6 / 4 / 2;
// config 5 HP catch-up 187 / 160 / 174 ms, profiles/r02/ab_xc_spmm.jsonl).
AQR_KNOB(xc_rows_knob, "AQR_XC_ROWS", 2)
int xc_rows() { const int r = xc_rows_knob(); return (r == 1 || r == 4) ? r : 2; }
// AQR_DEBUG_TIMING=1: host-side enqueue timings on stderr.
AQR_KNOB(debug_timing, "AQR_DEBUG_TIMING", 0)

template <typename K>
void ensure_carveout(K kernel) {
    const int pct = carveout_pct();
    if (pct < 0) return;
    static std::mutex mu;
    static std::vector<std::pair<const void *, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const void *key = reinterpret_cast<const void *>(kernel);
    std::lock_guard<std::mutex> lk(mu);
    for (auto &e : done)
        if (e.first == key && e.second == dev) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    done.push_back({key, dev});
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args) {
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_mode() != 0 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ---- diagnostics: kernel trace (AQR_TRACE builds) ----------------------------
#ifdef AQR_TRACE
struct Trace {
    unsigned long long *dev = nullptr;
    int32_t next = 0, cap = 0;
} g_tr;
int32_t trace_slot() {
    if (!g_tr.dev) {
        g_tr.cap = 1 << 14;
        cudaMalloc(&g_tr.dev, 3 * sizeof(unsigned long long) * g_tr.cap);
        cudaMemcpyToSymbol(aqr::g_trace, &g_tr.dev, sizeof(g_tr.dev));
        std::vector<unsigned long long> init(3 * g_tr.cap);
        for (int i = 0; i < g_tr.cap; ++i) init[3 * i] = init[3 * i + 1] = ~0ull, init[3 * i + 2] = 0;
        cudaMemcpy(g_tr.dev, init.data(), init.size() * 8, cudaMemcpyHostToDevice);
    }
    return g_tr.next < g_tr.cap ? g_tr.next++ : -1;
}
#else
int32_t trace_slot() { return -1; }
#endif

// ---- operators ---------------------------------------------------------------

aqr::NormOut no_norm() {
    aqr::NormOut o;
    std::memset(&o, 0, sizeof o);
    return o;
}

// ---- banded view of a CSR operator (aqr_band.cuh) ------------------------------
// Offsets per row rounded up to an instantiated width; a mask bit is never
// set for d >= nd, so the wider kernel computes the same sums.
#ifndef AQR_BAND_RPT
#define AQR_BAND_RPT 4  // staged SpMM: 256-row sub-blocks per CTA
#endif
#ifndef AQR_BAND_KC
#define AQR_BAND_KC 8   // staged SpMM: columns per CTA
#endif
#ifndef AQR_BAND_SPMM_MINB
#define AQR_BAND_SPMM_MINB 2
#endif

// Segments of the operand a block of NB rows reads (offsets closer than NB
// apart share one); false when they do not fit the staged kernels.
bool band_stage_plan(const aqr_band *band, int64_t NB, aqr::BandStage *st) {
    std::memset(st, 0, sizeof *st);
    int ns = -1;
    int64_t hi = 0, total = 0;
    for (int d = 0; d < band->nd; ++d) {
        const int64_t off = band->off[d];
        if (ns < 0 || off > hi + 32) {  // a new segment (small gaps are staged through)
            if (ns >= 0) {
                st->len[ns] = (int32_t)(hi - st->lo[ns]);
                total += (st->len[ns] + 1) & ~1;
            }
            if (++ns >= aqr::kBandSegMax) return false;
            st->lo[ns] = off;
            st->base[ns] = (int32_t)total;
        }
        hi = off + NB;
        if (total + (off - st->lo[ns]) + NB > (int64_t)1 << 20) return false;
        st->sbyte[d] = 8 * (st->base[ns] + (int32_t)(off - st->lo[ns]));
    }
    if (ns < 0) return false;
    st->len[ns] = (int32_t)(hi - st->lo[ns]);
    total += (st->len[ns] + 1) & ~1;
    st->nseg = ns + 1;
    st->total = (int32_t)total;
    return 2 * total * 8 <= 200 * 1024;  // two buffers
}

template <int ND, bool CONST>
aqr_status launch_band_tile(const aqr::BandArgs &b, const aqr_band *band, cudaStream_t s) {
    aqr::BandTileArgs t;
    t.c = b.c;
    t.b = b.b;
    constexpr int NB = AQR_BAND_RPT * aqr::kBlock;
    if (!band_stage_plan(band, NB, &t.st)) return AQR_EARG;
    auto kern = aqr::band_spmm_tile_kernel<ND, CONST, AQR_BAND_RPT, AQR_BAND_KC, AQR_BAND_SPMM_MINB>;
    const size_t smem = 2 * (size_t)t.st.total * 8;
    AQR_TRY(ensure_smem(kern, smem));
    const int64_t grid = ((b.c.m + NB - 1) / NB) * ((b.c.k + AQR_BAND_KC - 1) / AQR_BAND_KC);
    kern<<<(unsigned)grid, aqr::kBlock, smem, s>>>(t);
    return AQR_OK;
}

template <int ND, bool CONST>
void launch_band_nd(const aqr::BandArgs &b, bool step, cudaStream_t s) {
    const int64_t m = b.c.m;
    if (step) {  // fused HA / naive step or plain y = A x on the canonical norm grid
        constexpr int U = ND <= 5 ? AQR_BAND_U5 : (ND <= 9 ? AQR_BAND_U9 : 1);
        launch_pdl(aqr::band_step_kernel<ND, CONST, U, AQR_SPMV_MINB>, (unsigned)aqr::norm_tiles(m, false),
                   aqr::kBlock, 0, s, b);
    } else if constexpr (ND >= 9) {  // CTA = (8 columns, 256 rows); rows of <= 8 entries run csr_row_kernel
        const int64_t nb = (m + aqr::kBlock - 1) / aqr::kBlock;
        aqr::band_spmm_kernel<ND, CONST, 8, 4, 2><<<(unsigned)(((b.c.k + 7) / 8) * nb), aqr::kBlock, 0, s>>>(b);
    }
}

template <bool CONST>
void launch_band_c(const aqr::BandArgs &b, const aqr_band *band, bool step, cudaStream_t s) {
    const int nd = b.b.nd;
    // long rows, k > 1: operands staged in shared memory.  (The k = 1 step staged the
    // same way -- cp.async, double-buffered over the CTA's owned row blocks -- measured
    // 104 vs 100 ms per config-5 HA factorization and is not kept.)
    if (!step && nd > 9 && band_stage_mode() != 0) {
        aqr_status st = AQR_EARG;
        if (nd <= 16) st = launch_band_tile<16, CONST>(b, band, s);
        else if (nd <= 27) st = launch_band_tile<27, CONST>(b, band, s);
        else st = launch_band_tile<32, CONST>(b, band, s);
        if (st == AQR_OK) return;
    }
    if (nd <= 5) launch_band_nd<5, CONST>(b, step, s);
    else if (nd <= 7) launch_band_nd<7, CONST>(b, step, s);
    else if (nd <= 9) launch_band_nd<9, CONST>(b, step, s);
    else if (nd <= 16) launch_band_nd<16, CONST>(b, step, s);
    else if (nd <= 27) launch_band_nd<27, CONST>(b, step, s);
    else launch_band_nd<32, CONST>(b, step, s);
}

void launch_band(const aqr::CsrArgs &a, const aqr_band *band, bool step, cudaStream_t s) {
    aqr::BandArgs b;
    b.c = a;
    b.b.nd = band->nd;
    b.b.constant = band->constant;
    for (int d = 0; d < aqr::kBandMax; ++d) {
        b.b.off[d] = d < band->nd ? band->off[d] : 0;
        b.b.val[d] = d < band->nd ? band->val[d] : 0.0;
    }
    b.b.mask = band->mask;
    b.b.dvals = band->dvals;
    if (band->constant) launch_band_c<true>(b, band, step, s);
    else launch_band_c<false>(b, band, step, s);
}

bool band_usable(const aqr_op *op) {
    return op->band != nullptr && op->band->nd > 0 && op->band->nd <= aqr::kBandMax && op->band->mask != nullptr &&
           (op->band->constant || op->band->dvals != nullptr) && band_mode() != 0;
}

aqr_status launch_csr(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                      int64_t ldy, const double *qprev, const double *r, double *znew,
                      const aqr::NormOut &out, cudaStream_t s, const aqr::RrowIn *rin = nullptr) {
    aqr::CsrArgs a;
    std::memset(&a, 0, sizeof a);
    a.trace = out.npart != nullptr ? trace_slot() : -1;
    a.sg = spmm_sg();
    if (rin && out.npart != nullptr) a.rin = *rin;
    a.m = op->m;
    a.k = k;
    a.indptr = op->indptr;
    a.indices = op->indices;
    a.data = op->data;
    a.X = X;
    a.ldx = ldx;
    a.Y = Y;
    a.ldy = ldy;
    a.qprev = qprev;
    a.r = r;
    a.znew = znew;
    a.out = out;
    if (op->m == 0) return AQR_OK;
    // 256-row blocks (== the canonical norm tiles when fused), grid-stride
    // over a persistent grid: one completion ticket per CTA.
    const int64_t nblocks = (op->m + aqr::kBlock - 1) / aqr::kBlock;
    const int64_t grid = std::min<int64_t>(nblocks, (int64_t)sm_count() * 8);
    if (out.npart != nullptr) {
        const int64_t nt = aqr::norm_tiles(op->m, false);
        const long tix = timer_begin(1, (double)op->m * 40.0 + (double)op->nnz * 12.0, s);
        const int sv = spmv_variant();
        const unsigned g1 = (unsigned)nt;  // the canonical norm grid (HA / naive)
        // software-pipelined fused step; row batch B = the longest row when
        // known and <= 8 (all of a row's loads in one batch, no predicated-off
        // slots); longer rows loop.  AQR_SPMV_VARIANT=3: unpipelined, B = 8.
        const int32_t mr = op->max_row_nnz;
        if (band_usable(op))
            launch_band(a, op->band, true, s);
        else if (sv == 3)
            launch_pdl(aqr::csr_step_kernel<8, 3>, g1, aqr::kBlock, 0, s, a);
        else if (mr >= 1 && mr <= 4)
            launch_pdl(aqr::csr_step_pf_kernel<4, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else if (mr == 5)
            launch_pdl(aqr::csr_step_pf_kernel<5, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else if (mr == 6)
            launch_pdl(aqr::csr_step_pf_kernel<6, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else if (mr == 7)
            launch_pdl(aqr::csr_step_pf_kernel<7, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else if (mr == 8)
            launch_pdl(aqr::csr_step_pf_kernel<8, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else  // long or unknown rows: batches of 8 without the row look-ahead
            launch_pdl(aqr::csr_step_kernel<8, 3>, g1, aqr::kBlock, 0, s, a);
        timer_end(tix, s);
        return launched("csr_step_kernel");
    }
    const int32_t mr = op->max_row_nnz;
    const int plain_pf = plain_pf_mode();
    if (band_usable(op) && k == 1) {  // plain y = A x on the banded view
        launch_band(a, op->band, true, s);
        return launched("band_step_kernel");
    }
    // long rows (>= 9 offsets; narrower views have no k > 1 kernel and run the CSR ones)
    if (band_usable(op) && k > 1 && (mr > 8 || mr <= 0) && op->band->nd >= 9) {
        launch_band(a, op->band, false, s);
        return launched("band_spmm_kernel");
    }
    if (k == 1 && mr >= 1 && mr <= 8 && plain_pf != 0 && AQR_SPMV_PF2 != 0) {
        // plain y = A x through the pipelined step kernel (no norms, no
        // update): rows three deep instead of one dependent chain per row
        const unsigned g1 = (unsigned)aqr::norm_tiles(op->m, false);
        if (mr <= 4)
            launch_pdl(aqr::csr_step_pf_kernel<4, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else if (mr == 5)
            launch_pdl(aqr::csr_step_pf_kernel<5, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else if (mr == 6)
            launch_pdl(aqr::csr_step_pf_kernel<6, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else if (mr == 7)
            launch_pdl(aqr::csr_step_pf_kernel<7, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        else
            launch_pdl(aqr::csr_step_pf_kernel<8, AQR_SPMV_MINB>, g1, aqr::kBlock, 0, s, a);
        return launched("csr_step_kernel");
    }
    if (k > 1 && (mr > 8 || mr <= 0) && ldx < ((int64_t)1 << 29)) {  // long (or unknown) rows: CTA = (8 columns, 256 rows)
        const int64_t nb = (op->m + aqr::kBlock - 1) / aqr::kBlock;
        // (batch, columns, CTAs/SM) = (4, 8, 2); (4, 4, 4) / (2, 8, 3) / (8, 4, 3)
        // measured 115.6 / 85.3 / 114.4 vs 87.5 ms on config 5 (profiles/r02/ab_xc_spmm.jsonl)
        aqr::csr_spmm2_kernel<4, 8, 2><<<(unsigned)(((k + 7) / 8) * nb), aqr::kBlock, 0, s>>>(a);
        return launched("csr_spmm2_kernel");
    }
    if (mr >= 1 && mr <= 4)
        aqr::csr_row_kernel<4><<<(unsigned)grid, aqr::kBlock, 0, s>>>(a);
    else if (mr == 5)
        aqr::csr_row_kernel<5><<<(unsigned)grid, aqr::kBlock, 0, s>>>(a);
    else if (mr == 6)
        aqr::csr_row_kernel<6><<<(unsigned)grid, aqr::kBlock, 0, s>>>(a);
    else
        aqr::csr_row_kernel<8><<<(unsigned)grid, aqr::kBlock, 0, s>>>(a);
    return launched("csr_row_kernel");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point table (the
// library does not link libcuda; nullptr when unavailable).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static const EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

// 2D fp64 tensor map of a column-major rows x cols matrix (ld in elements),
// box {box_rows, box_cols}, 128-byte swizzle, out-of-bounds zero fill.
static bool tensor_map_2d(CUtensorMap *map, const double *base, int64_t rows, int64_t cols, int64_t ld,
                          uint32_t box_rows, uint32_t box_cols) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {box_rows, box_cols};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Y = A X on the FP64 tensor cores (dense_dmma_kernel): the HP block apply
// of a dense operator.  Returns false (nothing launched) when the operands
// do not meet TMA's alignment rules.
// The choice must not depend on k or on which columns X starts at: the
// host-input pipeline applies the HP block chunk by chunk (X at column c0 of
// the staged Z) and must produce the bits of the one-call block apply --
// so the criteria are the operands' base alignment and even leading
// dimensions (then every column of X is 16-byte aligned), and k = 1 runs
// on the tensor cores too.
static bool launch_dense_dmma(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y, int64_t ldy,
                              cudaStream_t s) {
    const int64_t m = op->m, K = op->ncols > 0 ? op->ncols : op->m;
    if (m < 1 || K < 1 || k < 1 || m > INT32_MAX || K > INT32_MAX) return false;
    // operators below 4096^2 entries keep the sequential product: there the
    // block apply is a few hundred microseconds at most, and the bits stay
    // the reference's (HP is sensitive to X's rounding on ill-conditioned
    // inputs; the golden cases pin it)
    if (m * K < ((int64_t)1 << 24) && dgemm_mode() != 2) return false;
    if (op->lda % 2 || ldx % 2 || (uintptr_t)op->A % 16 || (uintptr_t)X % 16) return false;
    CUtensorMap ta, tx;
    if (!tensor_map_2d(&ta, op->A, m, K, op->lda, 16, aqr::kDgBK)) return false;
    if (!tensor_map_2d(&tx, X, K, k, ldx, aqr::kDgBK, aqr::kDgBN)) return false;
    if (ensure_smem(aqr::dense_dmma_kernel, aqr::kDgSmem) != AQR_OK) return false;
    const int64_t tiles = ((m + aqr::kDgBM - 1) / aqr::kDgBM) * ((k + aqr::kDgBN - 1) / aqr::kDgBN);
    aqr::dense_dmma_kernel<<<(unsigned)tiles, aqr::kDgThreads, aqr::kDgSmem, s>>>(ta, tx, m, K, k, Y, ldy);
    return true;
}

// HP block apply X = op.apply_block(Zw) (gram_schmidt.py:136) of the
// factorization: dense operators on the FP64 tensor cores (tolerance-gated
// rounding), everything else as op_apply.
aqr_status block_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y, int64_t ldy,
                       cudaStream_t s);

aqr_status dense_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                       int64_t ldy, cudaStream_t s) {
    const int64_t m = op->m;
    const int64_t ncols = op->ncols > 0 ? op->ncols : m;
    if (m == 0) return AQR_OK;
    const bool tma_ok = m % 2 == 0 && ncols % 2 == 0 && op->lda % 2 == 0 &&
                        (uintptr_t)op->A % 16 == 0 && (uintptr_t)X % 16 == 0;
    if (k == 1 && tma_ok) {
        AQR_TRY(ensure_smem(aqr::dense_gemv_tma_kernel, aqr::kGvSmem));
        aqr::dense_gemv_tma_kernel<<<(unsigned)((m + aqr::kGvRows - 1) / aqr::kGvRows), aqr::kGvRows + 32,
                                     aqr::kGvSmem, s>>>(m, ncols, op->A, op->lda, X, Y);
        return launched("dense_gemv_tma_kernel");
    }
    if (k == 1) {
        dim3 grid((unsigned)((m + aqr::kGemvBlock - 1) / aqr::kGemvBlock), 1);
        aqr::dense_gemv_kernel<<<grid, aqr::kGemvBlock, 0, s>>>(m, ncols, op->A, op->lda, X, ldx, Y, ldy);
        return launched("dense_gemv_kernel");
    }
    dim3 grid((unsigned)((m + aqr::kG2BM - 1) / aqr::kG2BM), (unsigned)((k + aqr::kG2BN - 1) / aqr::kG2BN));
    AQR_TRY(ensure_smem(aqr::dense_gemm3_kernel, aqr::kG3Smem));
    aqr::dense_gemm3_kernel<<<grid, 256, aqr::kG3Smem, s>>>(m, ncols, k, op->A, op->lda, X, ldx, Y, ldy);
    return launched("dense_gemm3_kernel");
}

aqr_status op_apply_impl(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                         int64_t ldy, cudaStream_t s);

// Block applies (k > 1) are timed in slot 4: A once + X in + Y out.
aqr_status op_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                    int64_t ldy, cudaStream_t s) {
    if (!op || k <= 1 || op->kind == AQR_OP_CALLBACK) return op_apply_impl(op, k, X, ldx, Y, ldy, s);
    const double abytes = op->kind == AQR_OP_DENSE ? 8.0 * (double)op->m * (double)(op->ncols > 0 ? op->ncols : op->m)
                                                   : 12.0 * (double)op->nnz + 4.0 * (double)(op->m + 1);
    const long tix = timer_begin(4, abytes + 16.0 * (double)op->m * (double)k, s);
    const aqr_status st = op_apply_impl(op, k, X, ldx, Y, ldy, s);
    timer_end(tix, s);
    return st;
}

aqr_status block_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y, int64_t ldy,
                       cudaStream_t s) {
    if (op && op->kind == AQR_OP_DENSE && k >= 1 && op->A && op->lda >= op->m && dgemm_mode() != 0) {
        const double abytes = 8.0 * (double)op->m * (double)(op->ncols > 0 ? op->ncols : op->m);
        const long tix = timer_begin(4, abytes + 16.0 * (double)op->m * (double)k, s);
        const bool ok = launch_dense_dmma(op, k, X, ldx, Y, ldy, s);
        timer_end(tix, s);
        if (ok) return launched("dense_dmma_kernel");
    }
    return op_apply(op, k, X, ldx, Y, ldy, s);
}

aqr_status op_apply_impl(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                         int64_t ldy, cudaStream_t s) {
    if (!op) return set_err(AQR_EARG, "null operator");
    switch (op->kind) {
        case AQR_OP_DENSE:
            if (!op->A || op->lda < op->m) return set_err(AQR_EARG, "dense operator: bad A/lda");
            return dense_apply(op, k, X, ldx, Y, ldy, s);
        case AQR_OP_CSR:
            if (!op->indptr || (op->nnz && (!op->indices || !op->data)))
                return set_err(AQR_EARG, "csr operator: null arrays");
            return launch_csr(op, k, X, ldx, Y, ldy, nullptr, nullptr, nullptr, no_norm(), s);
        case AQR_OP_CALLBACK: {
            aqr_apply_fn fn = (k > 1 && op->apply_block) ? op->apply_block : op->apply;
            if (!fn) return set_err(AQR_EARG, "callback operator without apply");
            if (k > 1 && !op->apply_block) {
                for (int64_t c = 0; c < k; ++c)
                    if (fn(op->ctx, 1, X + c * ldx, ldx, Y + c * ldy, ldy, s) != 0)
                        return set_err(AQR_ECALLBACK, "operator apply callback failed");
                return AQR_OK;
            }
            if (fn(op->ctx, k, X, ldx, Y, ldy, s) != 0)
                return set_err(AQR_ECALLBACK, "operator apply callback failed");
            return AQR_OK;
        }
        default:
            return set_err(AQR_EARG, "unknown operator kind");
    }
}

// ---- step launchers ------------------------------------------------------------

aqr_status launch_col_update_norm(int64_t m, double *z, const double *qprev, double *x,
                                  const double *pprev, const double *r, const double *xnorm,
                                  const aqr::NormOut &out, bool hp_grid, cudaStream_t s,
                                  const aqr::RrowIn *rin = nullptr, const double *zsrc = nullptr) {
    aqr::ColArgs a;
    std::memset(&a.rin, 0, sizeof a.rin);
    a.zsrc = zsrc;
    a.trace = out.npart != nullptr ? trace_slot() : -1;
    if (rin) a.rin = *rin;
    a.m = m;
    a.z = z;
    a.qprev = qprev;
    a.x = x;
    a.pprev = pprev;
    a.r = r;
    a.xnorm = xnorm;
    a.out = out;
    a.out.ntiles = (int32_t)aqr::norm_tiles(m, hp_grid);
    const int64_t nt = aqr::norm_tiles(m, hp_grid);
    if (nt == 0) return AQR_OK;
    const int64_t grid = nt;  // the canonical norm grid (also without norm output)
    ensure_carveout(aqr::col_update_norm_kernel);
    const long tix = timer_begin(2, (double)m * (8.0 + (r ? 16.0 : 0.0) + (x ? (r ? 24.0 : 8.0) : 0.0) +
                                                 (xnorm ? 8.0 : 0.0)), s);
    launch_pdl(aqr::col_update_norm_kernel, (unsigned)grid, aqr::kBlock, 0, s, a);
    timer_end(tix, s);
    return launched("col_update_norm_kernel");
}

// HP row form, step j: x_j = X_j - sum_{k<j} r_{k,j} p_k, the deferred z_j
// update and the norm partials (col_lazy_norm_kernel).
aqr_status launch_col_lazy_norm(int64_t m, int64_t j, int64_t nprev, double *z, const double *zsrc, const double *qprev,
                                const double *Xj, const double *P, int64_t ldp, const double *rcol,
                                int64_t rstride, const double *r, double *xout, const aqr::NormOut &out,
                                const aqr::RrowIn *rin, cudaStream_t s) {
    aqr::ColArgs a;
    std::memset(&a, 0, sizeof a);
    a.trace = trace_slot();
    if (rin) a.rin = *rin;
    a.m = m;
    a.z = z;
    a.zsrc = zsrc;
    a.qprev = qprev;
    a.x = const_cast<double *>(Xj);
    a.r = r;
    a.out = out;
    a.out.ntiles = (int32_t)aqr::norm_tiles(m, true);
    a.P = P;
    a.ldp = ldp;
    a.rcol = rcol;
    a.rstride = rstride;
    a.nprev = (int32_t)nprev;
    a.xout = xout;
    const int64_t nt = aqr::norm_tiles(m, true);
    if (nt == 0) return AQR_OK;
    ensure_carveout(aqr::col_lazy_norm_kernel);
    // bytes: p_{j-nprev}..p_{j-1}, X_j, z_j (+ q_{j-1} and the z_j store), x_j store
    const long tix = timer_begin(2, (double)m * (8.0 * (double)nprev + 8.0 + 8.0 + (j > 0 ? 16.0 : 0.0) + 8.0), s);
    launch_pdl(aqr::col_lazy_norm_kernel, (unsigned)nt, aqr::kBlock, 0, s, a);
    timer_end(tix, s);
    return launched("col_lazy_norm_kernel");
}

// X_j -= sum_k r_kj p_k over k = kbeg .. kbeg+nk-1 for j in [jbeg, jend)
// (x_catchup_kernel); P = p_kbeg (columns at stride ldp), R = row kbeg of Rt.
aqr_status launch_x_catchup(int64_t m, double *X, int64_t ldx, int64_t jbeg, int64_t jend, const double *P,
                            int64_t ldp, const double *R, int64_t rstride, int64_t nk, const int32_t *status,
                            cudaStream_t s) {
    if (jend <= jbeg || nk <= 0 || m <= 0) return AQR_OK;
    aqr::XCatchArgs a;
    a.m = m;
    a.X = X;
    a.ldx = ldx;
    a.jbeg = (int32_t)jbeg;
    a.jend = (int32_t)jend;
    a.P = P;
    a.ldp = ldp;
    a.R = R;
    a.rstride = rstride;
    a.nk = (int32_t)nk;
    a.status = status;
    if (nk <= aqr::kXsMaxK && xc_stream_mode() != 0) {  // one CTA per row block walks all columns
        const long tix = timer_begin(3, (double)m * (16.0 * (double)(jend - jbeg) + 8.0 * (double)nk), s);
        const size_t sm = aqr::xs_smem((int)nk);
        AQR_TRY(ensure_smem(aqr::x_catchup_stream_kernel, sm));
        const int64_t blocks = (m + aqr::kBlock * aqr::kXsRows - 1) / (aqr::kBlock * aqr::kXsRows);
        launch_pdl(aqr::x_catchup_stream_kernel, dim3((unsigned)blocks), aqr::kBlock, sm, s, a);
        timer_end(tix, s);
        return launched("x_catchup_stream_kernel");
    }
    const int64_t groups = (jend - jbeg + aqr::kXcCols - 1) / aqr::kXcCols;
    const int rpt = xc_rows();
    const int64_t rows = (m + aqr::kBlock * rpt - 1) / (aqr::kBlock * rpt);
    const long tix = timer_begin(3, (double)m * (16.0 * (double)(jend - jbeg) + 8.0 * (double)nk), s);
    if (rpt == 4)
        launch_pdl(aqr::x_catchup_kernel<4, 2>, dim3((unsigned)(groups * rows)), aqr::kBlock, 0, s, a);
    else if (rpt == 1)
        launch_pdl(aqr::x_catchup_kernel<1, 6>, dim3((unsigned)(groups * rows)), aqr::kBlock, 0, s, a);
    else
        launch_pdl(aqr::x_catchup_kernel<2, 4>, dim3((unsigned)(groups * rows)), aqr::kBlock, 0, s, a);
    timer_end(tix, s);
    return launched("x_catchup_kernel");
}

// Algorithmic HBM bytes of one trailing launch: every trailing element read
// once (and written once when the deferred update applies), the step's
// vectors once.  Re-reads caused by column grouping are not counted.
// Windowed passes (trailing_w_kernel): every trailing element read once
// (CGS: its Z0 element, and z only where written), written only when the
// pass stores it (store_all, or column jbeg); the q window and the step's
// vectors once per row.
double trailing_bytes(const aqr::TrailArgs &a, bool hp, bool cgs, bool windowed) {
    const double m = (double)a.m, t = (double)std::max(0, a.jend - a.jbeg);
    if (windowed) {
        const double stored = a.win <= 0 ? 0.0 : (a.store_all ? t : std::min(t, 1.0));
        const double cols = cgs ? 8.0 * t + 16.0 * stored : 8.0 * t + 8.0 * stored;
        const double vec = 8.0 /* psrc */ + 8.0 * a.win + (a.qout ? 16.0 : 0.0) + (a.pout ? 8.0 : 0.0);
        return m * (cols + vec);
    }
    const bool upd = a.qprev != nullptr;
    double per_col = 8.0 + (upd ? 8.0 : 0.0) + ((hp && upd) ? 16.0 : 0.0) + (cgs ? 8.0 : 0.0);
    double vec = 8.0 /* psrc */ + (upd ? 8.0 : 0.0) + ((hp && upd) ? 8.0 : 0.0) +
                 (a.qout ? 16.0 : 0.0) + (a.pout ? 8.0 : 0.0);
    return m * (t * per_col + vec);
}

// Generic kernel: column groups so that ~trail_ctas_per_sm() CTAs per SM are in flight.
constexpr int kMaxCpg = 256;
// CTAs per SM the column grouping aims at (AQR_TRAIL_CTAS for A/B).  Columns
// are split into groups only when the tiles alone give fewer CTAs: on config
// 2 (512 tiles) one group per tile -- each CTA walks all t columns and reads
// the step vectors once -- beat two groups by 2.8 % (HA 7.51 -> 7.30 ms) and
// 2 % (HP 12.59 -> 12.34 ms); 2 and 3 give the same grouping there.
int trail_ctas_per_sm() { return std::max(1, trail_ctas_knob()); }

int choose_cpg_generic(int64_t ntiles, int64_t ncols) {
    if (ncols <= 0) return 1;
    const int64_t want_ctas = (int64_t)sm_count() * trail_ctas_per_sm();
    int64_t groups = std::max<int64_t>(1, (want_ctas + ntiles - 1) / ntiles);
    groups = std::min<int64_t>(groups, ncols);
    int64_t cpg = (ncols + groups - 1) / groups;
    cpg = std::min<int64_t>(cpg, kMaxCpg);
    return (int)std::max<int64_t>(cpg, 1);
}

aqr_status launch_rrow_reduce(int64_t m, int64_t ncols, const double *partial, double *out,
                              const int32_t *status, cudaStream_t s);

// deferred != nullptr: the caller's next norm kernel forms the r-row totals
// (RrowIn); *deferred tells whether the generic kernel left them pending.
aqr_status launch_trailing(const aqr::TrailArgs &a0, bool hp, bool cgs, cudaStream_t s,
                           bool *deferred = nullptr) {
    if (deferred) *deferred = false;
    aqr::TrailArgs a = a0;
    a.trace = trace_slot();
    const int64_t ncols = std::max<int64_t>(0, (int64_t)a.jend - a.jbeg);
    if (a.ntiles == 0) return AQR_OK;
    const bool big = aqr::rows_per_thread(a.m) == aqr::kBigRpt;
    // A persistent TMA-bulk (cp.async.bulk + mbarrier, warp-specialized)
    // form of this pass measured slower than this short-lived LDG kernel with
    // deferred totals (HA 9.26 vs 8.84 ms, HP 14.4 vs 14.1 ms on config 2;
    // DESIGN.md section 3) and was removed.
    a.cpg = choose_cpg_generic(a.ntiles, ncols);
    a.ngroups = ncols > 0 ? (int32_t)((ncols + a.cpg - 1) / a.cpg) : 1;
    if (ldg_reverse_mode() == 0) a.reverse = 0;

    if (!hp) {  // the Z-only pass runs windowed (trailing_w_kernel); one eager projection = window 1
        if (a.win == 0 && a.qprev != nullptr) {
            a.win = 1;
            a.qwin = a.qprev;
            a.rwin = a.rprev;
            a.rstride = 0;
            a.store_all = 1;
        }
        a.qprev = nullptr;  // (trail_prefetch: the window's first column instead)
        if (a.win > 0) a.qprev = a.qwin + (int64_t)(a.win - 1) * a.ldw;
    }
    const long tix = timer_begin(0, trailing_bytes(a, hp, cgs, !hp), s);
    dim3 grid((unsigned)a.ntiles, (unsigned)a.ngroups);
    if (!hp) {
        const int rpt = big ? aqr::kBigRpt : 1;
        const size_t smw = aqr::trail_w_smem(rpt, std::max(a.cpg, 1), a.win);
#define LAUNCHW(RPT, CU, CGS)                                                            \
    do {                                                                                 \
        AQR_TRY(ensure_smem(aqr::trailing_w_kernel<RPT, CU, CGS>, smw));                 \
        launch_pdl(aqr::trailing_w_kernel<RPT, CU, CGS>, grid, aqr::kBlock, smw, s, a); \
    } while (0)
#ifdef AQR_EXPERIMENTS
        if (big && !cgs && trail_cu() == 4) { LAUNCHW(aqr::kBigRpt, 4, false); goto done; }
#endif
        if (big) { if (cgs) LAUNCHW(aqr::kBigRpt, 2, true); else LAUNCHW(aqr::kBigRpt, aqr::kBigCu, false); }
        else     { if (cgs) LAUNCHW(1, 4, true); else LAUNCHW(1, 4, false); }
#undef LAUNCHW
        goto done;
    }
    {
    const size_t smem = sizeof(double) * aqr::kWarps * (size_t)std::max(a.cpg, 1);
#define LAUNCH(RPT, CU, HP, CGS)                                                           \
    do {                                                                                   \
        AQR_TRY(ensure_smem(aqr::trailing_kernel<RPT, CU, HP, CGS>, smem));                \
        launch_pdl(aqr::trailing_kernel<RPT, CU, HP, CGS>, grid, aqr::kBlock, smem, s, a); \
    } while (0)
    // Passes that carry X (the HP column loop): MGS one column per iteration
    // (128 registers, 2 CTAs/SM: 2.8 % faster than two at 164 registers /
    // 1 CTA/SM on config 2), CGS two (144 registers either way; 12 % faster).
    if (big) {
#ifdef AQR_EXPERIMENTS
        if (trail_variant() == 6 && !cgs) { LAUNCH(aqr::kBigRpt, 2, true, false); goto done; }  // MGS-HP, two columns
#endif
        if (cgs) LAUNCH(aqr::kBigRpt, 2, true, true); else LAUNCH(aqr::kBigRpt, 1, true, false);
    } else {
        if (cgs) LAUNCH(1, 4, true, true); else LAUNCH(1, 4, true, false);
    }
#undef LAUNCH
    }
done:
    timer_end(tix, s);
    AQR_TRY(launched("trailing_kernel"));
    if (a.counters != nullptr && ncols > 0) {  // totals pending
        if (deferred) {
            *deferred = true;
            return AQR_OK;
        }
        return launch_rrow_reduce(a.m, ncols, a.partial, a.rout, a.status, s);
    }
    return AQR_OK;
}

aqr_status launch_rrow_reduce(int64_t m, int64_t ncols, const double *partial, double *out,
                              const int32_t *status, cudaStream_t s) {
    if (ncols <= 0) return AQR_OK;
    aqr::rrow_reduce_kernel<<<(unsigned)ncols, aqr::kBlock, 0, s>>>(
        partial, (int32_t)aqr::num_tiles(m), (int32_t)ncols, out, status);
    return launched("rrow_reduce_kernel");
}

aqr_status launch_normalize(int64_t m, const double *z, const double *rii, double *q,
                            const double *x, double *p, const int32_t *status, cudaStream_t s) {
    aqr::normalize_kernel<<<elementwise_grid(m), aqr::kBlock, 0, s>>>(m, z, rii, q, x, p, status);
    return launched("normalize_kernel");
}

// ---- side streams for the look-ahead schedule ------------------------------
struct SideCtx {
    int dev;
    cudaStream_t side;
    cudaEvent_t e1, e2;
};
std::mutex g_side_mu;
std::vector<SideCtx> g_side_free;

aqr_status side_acquire(SideCtx &c) {
    int dev = 0;
    AQR_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_side_mu);
        for (size_t k = 0; k < g_side_free.size(); ++k)
            if (g_side_free[k].dev == dev) {
                c = g_side_free[k];
                g_side_free.erase(g_side_free.begin() + (long)k);
                return AQR_OK;
            }
    }
    int lo = 0, hi = 0;
    AQR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    c.dev = dev;
    (void)hi;
    AQR_CUDA(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, lo));  // copy streams
    AQR_CUDA(cudaEventCreateWithFlags(&c.e1, cudaEventDisableTiming));
    AQR_CUDA(cudaEventCreateWithFlags(&c.e2, cudaEventDisableTiming));
    return AQR_OK;
}

void side_release(const SideCtx &c) {
    std::lock_guard<std::mutex> lk(g_side_mu);
    g_side_free.push_back(c);
}


// Column-block copy (rows x cols doubles, leading dimensions in elements):
// one linear cudaMemcpyAsync when both sides are contiguous (the DMA engines'
// fast path), else a pitched copy.
cudaError_t copy_cols(double *dst, int64_t ldd, const double *src, int64_t lds, int64_t rows, int64_t cols,
                      cudaMemcpyKind kind, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    if ((ldd == rows && lds == rows) || cols == 1)
        return cudaMemcpyAsync(dst, src, 8 * (size_t)rows * (size_t)cols, kind, s);
    return cudaMemcpy2DAsync(dst, 8 * (size_t)ldd, src, 8 * (size_t)lds, 8 * (size_t)rows, (size_t)cols, kind, s);
}

// ---- workspace ---------------------------------------------------------------

inline uint64_t al(uint64_t b) { return (b + 255) & ~uint64_t(255); }

struct Layout {
    uint64_t status, counters, rt, partial, npart, xvec, zvec, pvec, pring, P, X, Z0, total;
};

constexpr uint64_t kNone = ~0ull;

Layout layout(int32_t family, int32_t variant, int32_t orientation, int64_t m, int64_t n) {
    Layout L;
    const uint64_t ntiles = std::max<uint64_t>((uint64_t)aqr::num_tiles(m), 1);
    const uint64_t mm = (uint64_t)m, nn = (uint64_t)n;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t o = off;
        off += al(bytes);
        return o;
    };
    L.status = take(16 + 4 * nn);
    L.counters = take(4 * (nn + 8));
    L.rt = take(8 * nn * nn);
    L.partial = take(8 * nn * ntiles);
    L.npart = take(8 * 3 * std::max<uint64_t>((uint64_t)aqr::norm_tiles(m, variant == AQR_HP), 1));
    L.xvec = variant != AQR_HP ? take(8 * 2 * mm) : kNone;  // 2-slot ring (look-ahead)
    L.zvec = variant != AQR_HP ? take(8 * 2 * mm) : kNone;
    L.pvec = (variant == AQR_NAIVE && orientation == AQR_ROW) ? take(8 * mm) : kNone;
    L.pring = (variant == AQR_HP && orientation == AQR_ROW) ? take(8 * 2 * mm) : kNone;
    L.P = orientation == AQR_COL ? take(8 * mm * nn) : kNone;
    L.X = variant == AQR_HP ? take(8 * mm * nn) : kNone;
    L.Z0 = family == AQR_CGS ? take(8 * mm * nn) : kNone;
    L.total = off;
    return L;
}

template <typename T>
T *at(void *base, uint64_t off) {
    return off == kNone ? nullptr : reinterpret_cast<T *>(static_cast<char *>(base) + off);
}

// ---- the sequencer -------------------------------------------------------------

// Streaming of the finished Q columns to host memory (aqr_gs_factor_d2h):
// column i is final once step i's launches are enqueued; an event on the
// compute stream releases its D2H copy on the copy stream, so the transfer
// of Q overlaps the remaining steps.
struct HostOut {
    double *qhost = nullptr;
    int64_t ldqh = 0;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev = nullptr;
};

// AQR_CATCHUP=0: one trailing launch (+ totals) per caught-up step; 2: the
// cooperative launch with two grid barriers per step (A/B; read per call)
int catchup_mode() { return knob("AQR_CATCHUP", 1); }  // read per call

template <int RPT, bool CGS>
aqr_status launch_catchup_t(const aqr::CatchArgs &c, cudaStream_t s) {
    constexpr int kCu = 2;  // columns per unit (catchup_kernel)
    const size_t smem = aqr::catch_smem(RPT, c.w, c.win, c.redundant != 0);
    AQR_TRY(ensure_smem(aqr::catchup_kernel<RPT, CGS>, smem));
    int o = 0;
    AQR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, aqr::catchup_kernel<RPT, CGS>, aqr::kBlock, smem));
    const int64_t units = (int64_t)c.ntiles * ((c.w + kCu - 1) / kCu);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)sm_count() * std::max(1, o)));
    aqr::CatchArgs cc = c;
    void *args[] = {&cc};
    AQR_CUDA(cudaLaunchCooperativeKernel((const void *)aqr::catchup_kernel<RPT, CGS>, grid, aqr::kBlock, args, smem, s));
    return launched("catchup_kernel");
}

aqr_status launch_catchup(const aqr::CatchArgs &c, bool cgs, cudaStream_t s) {
    if (aqr::rows_per_thread(c.m) == aqr::kBigRpt)
        return cgs ? launch_catchup_t<aqr::kBigRpt, true>(c, s) : launch_catchup_t<aqr::kBigRpt, false>(c, s);
    return cgs ? launch_catchup_t<1, true>(c, s) : launch_catchup_t<1, false>(c, s);
}

// Host-input pipeline (aqr_gs_factor_pinned): Z arrives in column chunks on
// an H2D stream.  A chunk joins the live columns when the step loop needs
// it, after a catch-up of the steps already done: the trailing passes
// k = 0 .. i-1 over the chunk's columns (left-looking MGS on the chunk), with
// the same (tile, column) units, deferred updates and reduction trees as the
// main loop -- results are bitwise those of the device-resident call.  The
// step vectors (HA: x_k, HP / naive: p_k) are kept for all k (vall).
struct Pipe {
    std::vector<int64_t> bounds;  // chunk c = columns [bounds[c], bounds[c + 1])
    std::vector<cudaEvent_t> ev;  // H2D of chunk c complete
    double *vall = nullptr;       // m x n
    double *partial2 = nullptr;   // catch-up partials, n x ntiles
    size_t next = 0;
};

struct Run {
    aqr_factor_args *a;
    HostOut *ho = nullptr;
    Pipe *pp = nullptr;
    int64_t live = 0;  // columns [0, live) are resident and caught up
    // Row form, windowed trailing passes: the stored trailing columns hold
    // z_j^(zbase) (projections 0 .. zbase-1 applied); the pass of step i
    // applies zbase .. i-1 in registers (trailing_w_kernel).
    int64_t zbase = 0;
    // HP row form: the stored X columns j >= live-from hold x_j^(xbase)
    // (x_catchup_kernel brings them forward every few steps); step j forms
    // x_j^(j) from them and p_xbase .. p_{j-1} (col_lazy_norm_kernel).
    int64_t xbase = 0;
    // Direct mode (row form, Z distinct from Q): the input Z is read in place
    // until the first write-back pass (column j+1 alone is written by every
    // pass j >= 1; zread: steps 0 and 1 read their own column from Z), so the
    // copy Zw = Z (gram_schmidt.py:131) is never materialized; CGS dots use Z
    // itself as Z0.
    const double *Zin = nullptr;
    int64_t ldzin = 0;
    const double *Z0p = nullptr;
    int64_t ldz0 = 0;
    const double *zread(int64_t j, int64_t step) const {
        return (Zin && step <= 1) ? Zin + j * ldzin : nullptr;
    }
    cudaStream_t s;
    bool hp, cgs, naive, csr_native;
    int64_t m, n;
    double *W;  // == Q
    int64_t ldw;
    int32_t *status;
    unsigned *counters;  // [0]: norm, [1 ..]: trailing column groups
    double *Rt, *partial, *npart, *xvec, *zvec, *pvec, *pring, *P, *X, *Z0;
    int64_t mv = 0;
    bool pending = false;  // row i-1 of R left as trailing partials (RrowIn)
    int32_t pending_cols = 0;

    double *col(double *B, int64_t ld, int64_t j) const { return B + j * ld; }

    // Column j of Q is final: stream it to the host (HostOut).
    aqr_status col_final(int64_t j) {
        if (!ho || !ho->qhost) return AQR_OK;
        AQR_CUDA(cudaEventRecord(ho->ev, s));
        AQR_CUDA(cudaStreamWaitEvent(ho->cs, ho->ev, 0));
        AQR_CUDA(copy_cols(ho->qhost + j * ho->ldqh, ho->ldqh, W + j * ldw, ldw, m, 1, cudaMemcpyDeviceToHost,
                           ho->cs));
        return AQR_OK;
    }

    aqr::RrowIn rrow_in(int64_t j) const {
        aqr::RrowIn in;
        in.partial = partial;
        in.ntiles = (int32_t)aqr::num_tiles(m);
        in.ncols = pending_cols;
        in.rrow = rt(j - 1, j);
        return in;
    }
    double *rt(int64_t i, int64_t j) const { return Rt + i * n + j; }

    // A user operator (callback) sees exactly the reference's calls: the
    // reference raises BreakdownError inside normalize(f) (gram_schmidt.py:
    // 153-154), so no apply follows the one that fed the failing column.  The
    // breakdown record is on the device; before each callback the stream is
    // drained and it is read (the callback costs a host round trip anyway).
    // After a breakdown the callback is skipped; the device kernels already
    // early-exit on the record.
    bool stopped = false;
    aqr_status mv1(const double *x, double *y) {
        if (a->op->kind == AQR_OP_CALLBACK && !stopped) {
            int32_t st0 = -1;
            AQR_CUDA(cudaMemcpyAsync(&st0, status, sizeof st0, cudaMemcpyDeviceToHost, s));
            AQR_CUDA(cudaStreamSynchronize(s));
            stopped = st0 >= 0;
        }
        if (stopped) return AQR_OK;
        AQR_TRY(op_apply(a->op, 1, x, m, y, m, s));
        ++mv;
        return AQR_OK;
    }

    bool long_rows() const { return a->op->max_row_nnz <= 0 || a->op->max_row_nnz > 8; }

    aqr::NormOut norm_out(int64_t j) const {
        aqr::NormOut o;
        o.npart = npart;
        o.ntiles = (int32_t)aqr::norm_tiles(m, hp);
        o.counter = counters;
        o.tot = nullptr;
        o.rii = rt(j, j);
        o.step = j;
        o.status = status;
        return o;
    }

    // Where step j's vector goes: HA x_j (xout), HP / naive p_j (pout_slot).
    double *xout(int64_t j) const { return (pp && !hp && !naive) ? pp->vall + j * m : xvec; }
    // HP (row form): p_j is kept for the lazy x of later steps -- in vall
    // (Pipe) or in X's column j, which col_lazy_norm_kernel read at step j
    // and nothing reads afterwards.
    double *pout_slot(int64_t j) const {
        if (pp) return pp->vall + j * m;
        return hp ? X + j * m : pvec;
    }
    const double *pbase() const { return pp ? pp->vall : X; }

    // Bring the next chunk of Z in at step i (Pipe): wait for its H2D, form
    // its X = A Z (HP) / saved copy (CGS), then run steps 0 .. i-1's trailing
    // passes over it (totals by rrow_reduce into R).
    aqr_status make_live(int64_t i) {
        const size_t c = pp->next++;
        const int64_t c0 = pp->bounds[c];
        // Merge the chunks that have already arrived when the steps get here
        // into one catch-up (i > 0): a wider chunk reloads the step vectors
        // and the q window once per step for more columns.  The host waits
        // for the compute stream to reach this point (one drain per chunk
        // brought in), then takes every further chunk whose H2D is complete.
        size_t c2 = c + 1;
        if (i > 0 && pipe_merge_mode() != 0 && c2 < pp->ev.size()) {
            AQR_CUDA(cudaStreamSynchronize(s));
            while (c2 < pp->ev.size() && pp->bounds[c2 + 1] - c0 <= 512 && cudaEventQuery(pp->ev[c2]) == cudaSuccess)
                ++c2;
            (void)cudaGetLastError();  // (cudaErrorNotReady from the query is not an error)
        }
        pp->next = c2;
        const int64_t c1 = pp->bounds[c2], w = c1 - c0;
        for (size_t e = c; e < c2; ++e) AQR_CUDA(cudaStreamWaitEvent(s, pp->ev[e], 0));
        if (cgs)
            AQR_CUDA(copy_cols(col(Z0, m, c0), m, col(W, ldw, c0), ldw, m, w, cudaMemcpyDeviceToDevice, s));
        if (hp) {  // X = op.apply_block(Zw), chunk by chunk
            AQR_TRY(block_apply(a->op, w, col(W, ldw, c0), ldw, col(X, m, c0), m, s));
            mv += w;
        }
        // steps 0 .. i-1 in one cooperative launch (chunks of <= 512 columns:
        // the kernel keeps a tile's warp totals of every column in shared memory)
        if (i > 0 && catchup_mode() != 0 && w <= 512) {
            aqr::CatchArgs c;
            std::memset(&c, 0, sizeof c);
            c.m = m;
            c.n = n;
            c.ntiles = (int32_t)aqr::num_tiles(m);
            c.c0 = (int32_t)c0;
            c.w = (int32_t)w;
            c.k1 = (int32_t)i;
            c.W = W;
            c.ldw = ldw;
            c.Z0 = Z0;
            c.ldz0 = m;
            c.vall = pp->vall;
            c.p_direct = (hp || naive) ? 1 : 0;  // HP: X is not caught up (lazy x)
            c.Rt = Rt;
            c.partial = pp->partial2;
            c.status = status;
            c.trace = trace_slot();
            // one barrier per step, every CTA forming the previous step's
            // totals itself, while that costs at most 128 loads per thread
            // (partial2 holds two parity buffers of the widest chunk); above
            // (config 5: 16 columns x 8192 tiles) w CTAs form them between two
            // barriers
            c.redundant = (catchup_mode() != 2 && (int64_t)w * c.ntiles <= 128 * aqr::kBlock) ? 1 : 0;
            c.win = trail_win();
            const long tix = timer_begin(5, 0.0, s);  // (time only)
            AQR_TRY(launch_catchup(c, cgs, s));
            timer_end(tix, s);
            live = c1;
            zbase = i - 1;  // the chunk holds z^(i-1): projection i-1 is left to step i
            return x_chunk(i, c0, c1);
        }
        for (int64_t k = 0; k < i; ++k) {
            aqr::TrailArgs t = trail(k, c0, c1);
            t.qprev = k > 0 ? col(W, ldw, k - 1) : nullptr;
            t.psrc = pp->vall + k * m;
            t.rii = (hp || naive) ? nullptr : rt(k, k);
            t.partial = pp->partial2;
            AQR_TRY(launch_trailing(t, false, cgs, s));
        }
        live = c1;
        zbase = i > 0 ? i - 1 : 0;
        return x_chunk(i, c0, c1);
    }

    // HP: a chunk's X = A Z arrives at x^(0); with R rows 0 .. i-1 of its
    // columns final (catch-up) it is brought to x^(i) in one pass.
    aqr_status x_chunk(int64_t i, int64_t c0, int64_t c1) {
        xbase = 0;
        if (!hp || i == 0) return AQR_OK;
        AQR_TRY(launch_x_catchup(m, X, m, c0, c1, pbase(), m, rt(0, 0), n, i, status, s));
        xbase = i;
        return AQR_OK;
    }

    // Column j receives the deferred projection r_{j-1,j} (z_j and, for HP,
    // x_j); x = A z (HA/naive); then t = z.x, |z|, |x| -> R[j,j] and the
    // breakdown / flag record (normalize(j), gram_schmidt.py:148-160).
    // Returns the columns holding the updated z and x.
    aqr_status norm_step(int64_t j, const double *pprev_col, const double *&zcol,
                         const double *&xcol, bool lazy = false) {
        double *z = col(W, ldw, j);
        const double *qprev = j > 0 ? col(W, ldw, j - 1) : nullptr;
        const double *r = j > 0 ? rt(j - 1, j) : nullptr;
        const aqr::RrowIn rin = rrow_in(j);
        const aqr::RrowIn *pin = pending ? &rin : nullptr;
        pending = false;
        const double *zs = zread(j, j);  // column j as read at step j (nullptr: W)
        if (hp && lazy) {  // row form: x_j formed from X_j and p_0 .. p_{j-1}
            double *xo = xvec + (j & 1) * m;
            AQR_TRY(launch_col_lazy_norm(m, j, j - xbase, z, zs, qprev, col(X, m, j), pbase() + xbase * m, m,
                                         rt(xbase, j), n, r, xo, norm_out(j), pin, s));
            // every x_win() steps: the stored columns j+1 .. live-1 catch up
            // to x^(j) (R rows < j are final once this step's kernel ran)
            // (a side-stream form -- the columns needed soon on this stream,
            // the rest overlapping the next trailing passes -- measured no
            // faster: 1235-1618 vs 1240 ms on config 5)
            if (j - xbase >= x_win() && j + 1 < live) {
                AQR_TRY(launch_x_catchup(m, X, m, j + 1, live, pbase() + xbase * m, m, rt(xbase, 0), n, j - xbase,
                                         status, s));
                xbase = j;
            }
            zcol = (zs && !r) ? zs : z;
            xcol = xo;
        } else if (hp) {
            double *x = col(X, m, j);
            AQR_TRY(launch_col_update_norm(m, z, qprev, x, pprev_col, r, nullptr, norm_out(j), true, s, pin, zs));
            zcol = (zs && !r) ? zs : z;  // without an update nothing was written to W
            xcol = x;
        } else if (csr_native && r && long_rows() && split_long_mode() != 0) {
            // long rows (> 8 entries, e.g. the 27-point stencil): the fused
            // form would gather z AND q_{j-1} for every entry; instead the
            // deferred update runs as one streaming pass (z_j -> zvec, with
            // r_{j-1,j} and the rest of row j-1 of R from the partials) and
            // the step kernel gathers the updated z only
            double *xo = xout(j);
            AQR_TRY(launch_col_update_norm(m, zvec, qprev, nullptr, nullptr, r, nullptr, no_norm(), false, s, pin,
                                           zs ? zs : z));
            AQR_TRY(launch_csr(a->op, 1, zvec, m, xo, m, nullptr, nullptr, nullptr, norm_out(j), s, nullptr));
            ++mv;
            zcol = zvec;
            xcol = xo;
        } else if (csr_native) {
            // one fused launch: r_{j-1,j} (and the rest of row j-1 of R),
            // gather (z - r q), x = A z, z_new, norm, r_jj
            double *xo = xout(j);
            const double *zx = zs ? zs : z;
            AQR_TRY(launch_csr(a->op, 1, zx, m, xo, m, qprev, r, zvec, norm_out(j), s, pin));
            const int rep = spmv_repeat();
            for (int k = 0; k < rep; ++k)
                AQR_TRY(launch_csr(a->op, 1, zx, m, xo, m, qprev, r, zvec, norm_out(j), s, pin));
            ++mv;
            zcol = zvec;
            xcol = xo;
        } else {
            double *xo = xout(j);
            if (r)
                AQR_TRY(launch_col_update_norm(m, z, qprev, nullptr, nullptr, r, nullptr, no_norm(), false, s,
                                               nullptr, zs));
            const double *zr = (zs && !r) ? zs : z;  // the current z_j
            AQR_TRY(mv1(zr, xo));  // op.apply(Zw[:, j].copy()), line 151
            AQR_TRY(launch_col_update_norm(m, z, nullptr, nullptr, nullptr, nullptr, xo, norm_out(j), false, s,
                                           nullptr, zr));
            zcol = zr;
            xcol = xo;
        }
        return AQR_OK;
    }

    aqr::TrailArgs trail(int64_t i, int64_t jbeg, int64_t jend) const {
        aqr::TrailArgs t;
        std::memset(&t, 0, sizeof t);
        t.m = m;
        t.ntiles = (int32_t)aqr::num_tiles(m);
        t.jbeg = (int32_t)jbeg;
        t.jend = (int32_t)jend;
        t.W = W;
        t.ldw = ldw;
        t.X = X;
        t.ldx = m;
        t.Z0 = Z0p ? Z0p : Z0;
        t.ldz0 = Z0p ? ldz0 : m;
        t.Wsrc = zread(0, i);  // steps 0 and 1 read the input Z in place
        t.ldwsrc = ldzin;
        t.rprev = i > 0 ? Rt + (i - 1) * n : nullptr;
        t.partial = partial;
        t.counters = counters + 1;
        t.rout = rt(i, jbeg);
        t.status = status;
        return t;
    }

    aqr_status row_form() {
        live = pp ? 0 : n;
        for (int64_t i = 0; i < n; ++i) {
            const auto hs = std::chrono::steady_clock::now();
            while (live <= i) AQR_TRY(make_live(i));
            const double *zcol = nullptr, *xcol = nullptr;
            AQR_TRY(norm_step(i, nullptr, zcol, xcol, true));
            aqr::TrailArgs t = trail(i, i + 1, std::max<int64_t>(i + 1, live));
            // deferred projections zbase .. i-1; the block is written back
            // when the window is full (the last pass has no trailing columns)
            t.win = t.jend > t.jbeg ? (int32_t)(i - zbase) : 0;
            t.store_all = t.win >= trail_win() ? 1 : 0;
            t.qwin = t.win > 0 ? col(W, ldw, zbase) : nullptr;
            t.rwin = t.win > 0 ? rt(zbase, 0) : nullptr;
            t.rstride = n;
            t.Wsrc = (Zin && zbase == 0) ? Zin : nullptr;  // nothing written back yet: read Z in place
            t.reverse = (int32_t)(i & 1);
            if (naive) {
                // q_i first, then p_i = A q_i (lines 161-163)
                AQR_TRY(launch_normalize(m, zcol, rt(i, i), col(W, ldw, i), nullptr, nullptr, status, s));
                AQR_TRY(mv1(col(W, ldw, i), pout_slot(i)));
                t.psrc = pout_slot(i);
                t.rii = nullptr;
            } else {
                t.psrc = xcol;
                t.rii = rt(i, i);
                t.zsrc = zcol;
                t.qout = col(W, ldw, i);
                t.pout = hp ? pout_slot(i) : nullptr;
            }
            {
                const bool dbg = debug_timing() != 0;
                const auto h0 = std::chrono::steady_clock::now();
                const bool can_defer = (hp || csr_native) && i + 1 < n && defer_mode() != 0;
                // HP too runs the Z-only pass: X is never rewritten (lazy x)
                AQR_TRY(launch_trailing(t, false, cgs, s, can_defer ? &pending : nullptr));
                pending_cols = t.jend - t.jbeg;
                if (t.store_all) zbase = i;
                AQR_TRY(col_final(i));
                if (dbg) {
                    const auto h1 = std::chrono::steady_clock::now();
                    std::fprintf(stderr, "  step %ld trailing launch host %.1f us, norm-step host %.1f us\n", (long)i,
                                 std::chrono::duration<double, std::micro>(h1 - h0).count(),
                                 std::chrono::duration<double, std::micro>(h0 - hs).count());
                }
            }
        }
        return AQR_OK;
    }

    aqr_status col_form() {
        for (int64_t j = 0; j < n; ++j) {
            for (int64_t i = 0; i < j; ++i) {  // project(i, j), lines 169-170
                aqr::TrailArgs t = trail(i, j, j + 1);
                t.qprev = i > 0 ? col(W, ldw, i - 1) : nullptr;
                t.pprev = (hp && i > 0) ? col(P, m, i - 1) : nullptr;
                t.psrc = col(P, m, i);
                t.rii = nullptr;
                AQR_TRY(launch_trailing(t, hp, cgs, s));
            }
            const double *pprev = (hp && j > 0) ? col(P, m, j - 1) : nullptr;
            const double *zcol = nullptr, *xcol = nullptr;
            AQR_TRY(norm_step(j, pprev, zcol, xcol));  // normalize(j), line 171
            if (naive) {
                AQR_TRY(launch_normalize(m, zcol, rt(j, j), col(W, ldw, j), nullptr, nullptr, status, s));
                AQR_TRY(mv1(col(W, ldw, j), col(P, m, j)));
            } else {
                AQR_TRY(launch_normalize(m, zcol, rt(j, j), col(W, ldw, j), xcol, col(P, m, j), status, s));
            }
            AQR_TRY(col_final(j));
        }
        return AQR_OK;
    }
};

// Peer-memory trailing pass of step i (windowed Z-only pass for HA and for
// HP with lazy x, as the single-GPU row form).
template <bool CGS>
aqr_status launch_p2p_trailing(const aqr::TrailArgs &a0, const aqr::P2PArgs &P, int64_t i, double *rii,
                               int32_t *status, cudaStream_t s) {
    aqr::TrailArgs a = a0;
    const int64_t ncols = std::max<int64_t>(0, (int64_t)a.jend - a.jbeg);
    a.cpg = choose_cpg_generic(a.ntiles, ncols);
    a.ngroups = ncols > 0 ? (int32_t)((ncols + a.cpg - 1) / a.cpg) : 1;
    dim3 grid((unsigned)a.ntiles, (unsigned)a.ngroups);
    const bool big = aqr::rows_per_thread(a.m) == aqr::kBigRpt;
    const size_t smem = aqr::trail_w_smem(big ? aqr::kBigRpt : 1, std::max(a.cpg, 1), a.win);
    if (a.win > 0) a.qprev = a.qwin + (int64_t)(a.win - 1) * a.ldw;  // trail_prefetch
    const long tix = timer_begin(0, trailing_bytes(a, false, CGS, true), s);
    if (big) {
        AQR_TRY(ensure_smem(aqr::p2p_trailing_kernel<aqr::kBigRpt, aqr::kBigCu, false, CGS, true>, smem));
        launch_pdl(aqr::p2p_trailing_kernel<aqr::kBigRpt, aqr::kBigCu, false, CGS, true>, grid, aqr::kBlock, smem, s, a,
                   P, i, rii, status);
    } else {
        AQR_TRY(ensure_smem(aqr::p2p_trailing_kernel<1, 4, false, CGS, true>, smem));
        launch_pdl(aqr::p2p_trailing_kernel<1, 4, false, CGS, true>, grid, aqr::kBlock, smem, s, a, P, i, rii, status);
    }
    timer_end(tix, s);
    return launched("p2p_trailing_kernel");
}

}  // namespace

extern "C" {

const char *aqr_last_error(void) { return g_err.c_str(); }
uint64_t aqr_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

aqr_status aqr_trailing_timer_enable(int32_t enable) {
    std::lock_guard<std::mutex> lk(g_timer.mu);
    g_timer.enabled = enable != 0;
    if (g_timer.enabled) {
        g_timer.recs.clear();
        g_timer.used = 0;
    }
    return AQR_OK;
}

aqr_status aqr_kernel_timer_read(int32_t slot, int64_t *launches, double *ms, double *bytes) {
    std::lock_guard<std::mutex> lk(g_timer.mu);
    double total = 0.0, b = 0.0;
    int64_t n = 0;
    for (const auto &r : g_timer.recs) {
        if (r.slot != slot) continue;
        AQR_CUDA(cudaEventSynchronize(r.e1));
        float dt = 0.f;
        AQR_CUDA(cudaEventElapsedTime(&dt, r.e0, r.e1));
        total += dt;
        b += r.bytes;
        ++n;
    }
    if (launches) *launches = n;
    if (ms) *ms = total;
    if (bytes) *bytes = b;
    return AQR_OK;
}

int64_t aqr_kernel_timer_list(int32_t slot, double *ms_out, double *bytes_out, int64_t max) {
    std::lock_guard<std::mutex> lk(g_timer.mu);
    int64_t k = 0;
    for (const auto &r : g_timer.recs) {
        if (r.slot != slot) continue;
        if (k < max) {
            if (cudaEventSynchronize(r.e1) != cudaSuccess) return -1;
            float dt = 0.f;
            if (cudaEventElapsedTime(&dt, r.e0, r.e1) != cudaSuccess) return -1;
            if (ms_out) ms_out[k] = dt;
            if (bytes_out) bytes_out[k] = r.bytes;
        }
        ++k;
    }
    return k;
}

aqr_status aqr_trailing_timer_read(int64_t *launches, double *ms, double *bytes) {
    AQR_TRY(aqr_kernel_timer_read(0, launches, ms, bytes));
    std::lock_guard<std::mutex> lk(g_timer.mu);
    g_timer.recs.clear();
    g_timer.used = 0;
    return AQR_OK;
}

int32_t aqr_abi_version(void) { return AQR_ABI_VERSION; }

// Diagnostics: copies the kernel trace (3 x uint64 per launch slot: first
// CTA start before / after the dependency wait, last CTA end; globaltimer ns)
// and returns the number of slots used; -1 when built without AQR_TRACE.
int64_t aqr_trace_read(uint64_t *out, int64_t max_slots) {
#ifdef AQR_TRACE
    const int64_t n = std::min<int64_t>(g_tr.next, max_slots);
    cudaDeviceSynchronize();
    if (n > 0 && g_tr.dev) cudaMemcpy(out, g_tr.dev, 3 * 8 * (size_t)n, cudaMemcpyDeviceToHost);
    return n;
#else
    (void)out;
    (void)max_slots;
    return -1;
#endif
}
int64_t aqr_tile_rows(int64_t m) { return aqr::tile_rows(m); }
int64_t aqr_num_tiles(int64_t m) { return aqr::num_tiles(m); }
uint64_t aqr_status_bytes(int64_t n) { return 16 + 4 * (uint64_t)std::max<int64_t>(n, 0); }

uint64_t aqr_workspace_bytes(int32_t family, int32_t variant, int32_t orientation, int64_t m,
                             int64_t n) {
    return layout(family, variant, orientation, m, n).total;
}

aqr_status aqr_status_init(int32_t *status, int64_t n, void *stream) {
    const int64_t cnt = std::max<int64_t>(n, 1);
    aqr::status_init_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, S(stream)>>>(status, n);
    return launched("status_init_kernel");
}

static aqr_status gs_factor_impl(aqr_factor_args *a, void *stream, HostOut *ho, Pipe *pp = nullptr) {
    if (!a) return set_err(AQR_EARG, "null args");
    a->fail_col = -1;
    a->fail_val = 0.0;
    a->mv_count = 0;
    if (a->family < 0 || a->family > 1 || a->variant < 0 || a->variant > 2 || a->orientation < 0 ||
        a->orientation > 1)
        return set_err(AQR_EARG, "bad family/variant/orientation");
    const int64_t m = a->m, n = a->n;
    if (n < 1 || m < n) return set_err(AQR_EDIM, "need m >= n >= 1");
    if (!a->op || a->op->m != m) return set_err(AQR_EDIM, "operator dimension does not match Z");
    if (n > (int64_t)INT32_MAX / 2 || m > ((int64_t)1 << 40)) return set_err(AQR_EARG, "size out of range");
    if (!a->Z || !a->Q || !a->R || a->ldz < m || a->ldq < m || a->ldr < n)
        return set_err(AQR_EARG, "bad Z/Q/R pointer or leading dimension");
    const Layout L = layout(a->family, a->variant, a->orientation, m, n);
    if (!a->workspace || a->workspace_bytes < L.total)
        return set_err(AQR_ENOMEM, "workspace smaller than aqr_workspace_bytes()");

    Run r;
    r.a = a;
    r.ho = ho;
    // Both orientations give bitwise-identical factors (same per-column
    // sequence of updates, same reduction trees; tested), so the column
    // orientation runs the row-oriented step schedule unless
    // AQR_COL_SCHEDULE=1 asks for the column loop (n(n-1)/2 dependent global
    // reductions: latency-bound, 27 vs 7.6 ms on config 2).
    const bool row_sched = a->orientation == AQR_ROW || col_schedule_mode() == 0;
    r.pp = (pp && row_sched) ? pp : nullptr;
    r.s = S(stream);
    r.hp = a->variant == AQR_HP;
    r.naive = a->variant == AQR_NAIVE;
    r.cgs = a->family == AQR_CGS;
    r.csr_native = a->op->kind == AQR_OP_CSR;
    r.m = m;
    r.n = n;
    r.W = a->Q;
    r.ldw = a->ldq;
    void *ws = a->workspace;
    r.status = at<int32_t>(ws, L.status);
    r.counters = at<unsigned>(ws, L.counters);
    r.Rt = at<double>(ws, L.rt);
    r.partial = at<double>(ws, L.partial);
    r.npart = at<double>(ws, L.npart);
    r.xvec = at<double>(ws, L.xvec);
    r.zvec = at<double>(ws, L.zvec);
    r.pvec = at<double>(ws, L.pvec);
    r.pring = at<double>(ws, L.pring);
    r.P = at<double>(ws, L.P);
    r.X = at<double>(ws, L.X);
    r.Z0 = at<double>(ws, L.Z0);
    if (row_sched && a->orientation == AQR_COL) {  // the row schedule's vectors live in P's storage
        r.pvec = r.P;
        r.pring = r.P;  // n >= 2: 2m <= mn; n = 1 uses slot 0 only
    }
    if (r.hp) r.xvec = r.pring;  // HP row form: the lazy x_j ring (p_j lives in X / vall)
    cudaStream_t s = r.s;

    const bool direct = a->Z != a->Q && row_sched && !r.pp && direct_mode() != 0;
    if (direct) {  // Zw = Z.copy(order="F") (line 131) is read in place instead
        r.Zin = a->Z;
        r.ldzin = a->ldz;
        if (r.cgs) {  // Z0 = Z (line 132): the input itself stays untouched
            r.Z0p = a->Z;
            r.ldz0 = a->ldz;
        }
    } else if (a->Z != a->Q) {  // Zw = Z.copy(order="F"), line 131
        AQR_CUDA(copy_cols(a->Q, a->ldq, a->Z, a->ldz, m, n, cudaMemcpyDeviceToDevice, s));
    }
    AQR_TRY(aqr_status_init(r.status, n, stream));
    AQR_CUDA(cudaMemsetAsync(r.counters, 0, 4 * (size_t)(n + 8), s));
    AQR_CUDA(cudaMemsetAsync(r.Rt, 0, 8 * (size_t)n * n, s));
    if (r.cgs && !r.pp && !direct)  // Z0, line 132 (per chunk when pipelined)
        AQR_CUDA(copy_cols(r.Z0, m, a->Q, a->ldq, m, n, cudaMemcpyDeviceToDevice, s));
    if (r.hp && !r.pp) {  // X = op.apply_block(Zw), line 136 (per chunk when pipelined)
        AQR_TRY(block_apply(a->op, n, direct ? a->Z : a->Q, direct ? a->ldz : a->ldq, r.X, m, s));
        r.mv += n;
    }
    const bool dbg_timing = debug_timing() != 0;
    const auto t_loop = std::chrono::steady_clock::now();
    AQR_TRY(row_sched ? r.row_form() : r.col_form());
    aqr::finalize_r_kernel<<<(unsigned)((n * n + 255) / 256), 256, 0, s>>>(n, r.Rt, a->R, a->ldr);
    AQR_TRY(launched("finalize_r_kernel"));
    std::vector<int32_t> st((16 + 4 * n) / 4);
    AQR_CUDA(cudaMemcpyAsync(st.data(), r.status, 16 + 4 * n, cudaMemcpyDeviceToHost, s));
    const auto t_enq = std::chrono::steady_clock::now();
    AQR_CUDA(cudaStreamSynchronize(s));
    if (dbg_timing) {
        const auto t_end = std::chrono::steady_clock::now();
        std::fprintf(stderr, "aqr_gs_factor: enqueue loop %.1f us, wait %.1f us\n",
                     std::chrono::duration<double, std::micro>(t_enq - t_loop).count(),
                     std::chrono::duration<double, std::micro>(t_end - t_enq).count());
    }
    a->mv_count = r.mv;
    if (a->flagged_host) std::memcpy(a->flagged_host, st.data() + 4, 4 * n);
    if (st[0] >= 0) {
        a->fail_col = st[0];
        std::memcpy(&a->fail_val, st.data() + 2, 8);
        return set_err(AQR_EBREAKDOWN, "breakdown at column " + std::to_string(st[0]));
    }
    return AQR_OK;
}

aqr_status aqr_gs_factor(aqr_factor_args *a, void *stream) { return gs_factor_impl(a, stream, nullptr); }

// Extra workspace of the host-input pipeline (caller-owned, after the
// factorization's own layout): vall (every step vector, m x n) and the
// catch-up partials (two parity buffers of up to n columns, + 8 columns read
// past the end by block_totals<8>).
static void pipe_extra(int64_t m, int64_t n, uint64_t *vall_bytes, uint64_t *partial_bytes) {
    const uint64_t ntiles = (uint64_t)std::max<int64_t>(aqr::num_tiles(m), 1);
    *vall_bytes = al(8 * (uint64_t)m * (uint64_t)n);
    *partial_bytes = al(8 * (2 * (uint64_t)n + 8) * ntiles);
}

uint64_t aqr_pipe_workspace_bytes(int32_t family, int32_t variant, int32_t orientation, int64_t m, int64_t n) {
    (void)family, (void)variant, (void)orientation;
    uint64_t a = 0, b = 0;
    pipe_extra(std::max<int64_t>(m, 0), std::max<int64_t>(n, 0), &a, &b);
    return a + b;
}

// Column chunks of the host-input pipeline: chunk_cols > 0 gives uniform
// chunks; 0 the default schedule, uniform n/8.  AQR_PIPE_SCHED selects the
// measured alternatives (1: n/8 then halving towards the end, 2: also
// ramping up from n/32 at the start): small final chunks still need a
// catch-up over all previous steps each, small first ones start the D2H of
// Q earlier, and neither beat uniform chunks.
int pipe_sched_mode() { return knob("AQR_PIPE_SCHED", 0); }  // read per call

std::vector<int64_t> pipe_bounds(int64_t n, int64_t chunk_cols) {
    std::vector<int64_t> b{0};
    if (n <= 0) return b;
    if (chunk_cols < 0) {  // ramp: w/8, w/4, w/2, then w (w = -chunk_cols)
        const int64_t w = -chunk_cols;
        int64_t c = 0;
        for (int64_t r = std::max<int64_t>(1, w / 8); r < w && c < n; r *= 2) b.push_back(c = std::min(n, c + r));
        while (c < n) b.push_back(c = std::min(n, c + w));
        return b;
    }
    const int sched = chunk_cols > 0 ? 0 : pipe_sched_mode();
    const int64_t w = chunk_cols > 0 ? chunk_cols : std::max<int64_t>(1, (n + 7) / 8);
    int64_t c = 0;
    if (sched == 2)  // ramp: w/4, w/2, then w
        for (int64_t r = std::max<int64_t>(1, w / 4); r < w && c + r < n; r *= 2) b.push_back(c += r);
    while (n - c > (sched >= 1 ? w : 0)) b.push_back(c = std::min(n, c + w));
    while (c < n) b.push_back(c += std::max<int64_t>(1, (n - c) / 2));  // taper: halves, then 1
    return b;
}

// cuStreamWaitValue32 through the runtime's driver entry point table (the
// library does not link libcuda; nullptr when unavailable).
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValue32Fn wait_value32() {
    static const WaitValue32Fn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (WaitValue32Fn) nullptr;
        return (WaitValue32Fn)p;
    }();
    return fn;
}

int64_t aqr_pipe_chunks(int64_t n, int64_t chunk_cols, int64_t *bounds, int64_t max_bounds) {
    const std::vector<int64_t> b = pipe_bounds(n, chunk_cols);
    for (size_t k = 0; k < b.size() && (int64_t)k < max_bounds; ++k) bounds[k] = b[k];
    return (int64_t)b.size() - 1;
}

aqr_status aqr_gs_factor_pinned(aqr_factor_args *a, const double *Z_host, int64_t ldzh, double *Q_host,
                                int64_t ldqh, double *R_host, int64_t ldrh, int64_t chunk_cols,
                                const uint32_t *ready, void *stream) {
    if (!a || !Z_host || !Q_host || !R_host) return set_err(AQR_EARG, "null args / host buffers");
    const int64_t m = a->m, n = a->n;
    if (n < 1 || m < n) return set_err(AQR_EDIM, "need m >= n >= 1");
    if (!a->Q || ldzh < m || ldqh < m || ldrh < n || a->ldq < m) return set_err(AQR_EARG, "bad buffers / leading dimensions");
    cudaStream_t s = S(stream);
    a->Z = a->Q;  // Z is staged into Q (factorized in place)
    a->ldz = a->ldq;
    // Whole H2D first, then the streamed D2H: for the column loop, and for HP
    // with a user operator, whose apply_block must see all n columns in one
    // call (gram_schmidt.py:136; the pipeline applies it chunk by chunk).
    const bool hp_callback = a->variant == AQR_HP && a->op && a->op->kind == AQR_OP_CALLBACK;
    const int64_t nchunks = (int64_t)pipe_bounds(n, chunk_cols).size() - 1;
    // host-side wait for the staging producer (when the stream wait is unavailable)
    auto host_wait = [&](uint32_t v) {
        if (!ready) return;
        while (*(const volatile uint32_t *)ready < v) std::this_thread::yield();
    };
    if ((a->orientation != AQR_ROW && col_schedule_mode() != 0) || hp_callback) {
        host_wait((uint32_t)nchunks);
        AQR_CUDA(copy_cols(a->Q, a->ldq, Z_host, ldzh, m, n, cudaMemcpyHostToDevice, s));
        return aqr_gs_factor_d2h(a, Q_host, ldqh, R_host, ldrh, stream);
    }
    CUdeviceptr ready_dev = 0;
    WaitValue32Fn wfn = ready ? wait_value32() : nullptr;
    if (wfn) {
        void *dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, const_cast<uint32_t *>(ready), 0) == cudaSuccess)
            ready_dev = (CUdeviceptr)dp;
        else
            wfn = nullptr;
    }
    Pipe pp;
    pp.bounds = pipe_bounds(n, chunk_cols);
    const size_t nch = pp.bounds.size() - 1;
    {
        const uint64_t base = layout(a->family, a->variant, a->orientation, m, n).total;
        uint64_t vb = 0, pb = 0;
        pipe_extra(m, n, &vb, &pb);
        if (!a->workspace || a->workspace_bytes < base + vb + pb)
            return set_err(AQR_ENOMEM, "workspace smaller than aqr_workspace_bytes() + aqr_pipe_workspace_bytes()");
        pp.vall = at<double>(a->workspace, base);
        pp.partial2 = at<double>(a->workspace, base + vb);
    }
    SideCtx h2d;
    AQR_TRY(side_acquire(h2d));
    aqr_status st = AQR_OK;
    // the H2D stream starts after everything already queued on `stream`
    if (cudaEventRecord(h2d.e1, s) != cudaSuccess || cudaStreamWaitEvent(h2d.side, h2d.e1, 0) != cudaSuccess)
        st = set_err(AQR_ECUDA, "h2d stream ordering");
    for (size_t c = 0; c < nch && st == AQR_OK; ++c) {
        cudaEvent_t e = nullptr;
        const int64_t c0 = pp.bounds[c], cw = pp.bounds[c + 1] - c0;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            st = set_err(AQR_ECUDA, "event");
            break;
        }
        pp.ev.push_back(e);
        if (ready) {  // chunk c is in host memory once *ready >= c + 1 (staged by the caller)
            if (wfn) {
                if (wfn((CUstream)h2d.side, ready_dev, (cuuint32_t)(c + 1), CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
                    st = set_err(AQR_ECUDA, "cuStreamWaitValue32");
                    break;
                }
            } else {
                host_wait((uint32_t)(c + 1));
            }
        }
        if (copy_cols(a->Q + c0 * a->ldq, a->ldq, Z_host + c0 * ldzh, ldzh, m, cw, cudaMemcpyHostToDevice,
                      h2d.side) != cudaSuccess ||
            cudaEventRecord(e, h2d.side) != cudaSuccess)
            st = set_err(AQR_ECUDA, "H2D Z chunk");
    }
    if (st == AQR_OK) {
        SideCtx d2h;
        st = side_acquire(d2h);
        if (st == AQR_OK) {
            HostOut ho;
            ho.qhost = Q_host;
            ho.ldqh = ldqh;
            ho.cs = d2h.side;
            ho.ev = d2h.e1;
            st = gs_factor_impl(a, stream, &ho, &pp);
            if (st == AQR_OK &&
                cudaMemcpy2DAsync(R_host, 8 * (size_t)ldrh, a->R, 8 * (size_t)a->ldr, 8 * (size_t)n, (size_t)n,
                                  cudaMemcpyDeviceToHost, s) != cudaSuccess)
                st = set_err(AQR_ECUDA, "D2H R");
            if (cudaStreamSynchronize(d2h.side) != cudaSuccess && st == AQR_OK) st = set_err(AQR_ECUDA, "D2H Q");
            side_release(d2h);
        }
    }
    cudaStreamSynchronize(h2d.side);
    side_release(h2d);
    for (cudaEvent_t e : pp.ev) cudaEventDestroy(e);
    if (cudaStreamSynchronize(s) != cudaSuccess && st == AQR_OK) st = set_err(AQR_ECUDA, "stream");
    return st;
}

aqr_status aqr_gs_factor_d2h(aqr_factor_args *a, double *Q_host, int64_t ldqh, double *R_host, int64_t ldrh,
                             void *stream) {
    if (!a || !Q_host || !R_host) return set_err(AQR_EARG, "null args / host buffers");
    if (ldqh < a->m || ldrh < a->n) return set_err(AQR_EARG, "bad host leading dimension");
    SideCtx sc;
    AQR_TRY(side_acquire(sc));
    HostOut ho;
    ho.qhost = Q_host;
    ho.ldqh = ldqh;
    ho.cs = sc.side;
    ho.ev = sc.e1;
    aqr_status st = gs_factor_impl(a, stream, &ho);  // returns after the compute stream drained
    if (st == AQR_OK &&
        cudaMemcpy2DAsync(R_host, 8 * (size_t)ldrh, a->R, 8 * (size_t)a->ldr, 8 * (size_t)a->n, (size_t)a->n,
                          cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess)
        st = set_err(AQR_ECUDA, "D2H R");
    if (cudaStreamSynchronize(sc.side) != cudaSuccess && st == AQR_OK) st = set_err(AQR_ECUDA, "D2H Q");
    if (cudaStreamSynchronize(S(stream)) != cudaSuccess && st == AQR_OK) st = set_err(AQR_ECUDA, "D2H R");
    side_release(sc);
    return st;
}

// ---- multi-GPU over peer memory (aqr_p2p.cuh) -------------------------------

uint64_t aqr_p2p_exchange_bytes(int64_t n) { return 8 * (uint64_t)aqr::xb_words(std::max<int64_t>(n, 1)); }

aqr_status aqr_p2p_alloc(uint64_t bytes, void **out) {
    if (!out) return set_err(AQR_EARG, "null out");
    *out = nullptr;
    AQR_CUDA(cudaMalloc(out, std::max<uint64_t>(bytes, 256)));
    AQR_CUDA(cudaMemset(*out, 0, std::max<uint64_t>(bytes, 256)));
    return AQR_OK;
}

aqr_status aqr_p2p_free(void *ptr) {
    if (ptr) AQR_CUDA(cudaFree(ptr));
    return AQR_OK;
}

aqr_status aqr_ipc_handle(const void *ptr, uint8_t out[64]) {
    cudaIpcMemHandle_t h;
    AQR_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)));
    static_assert(sizeof(h) == 64, "CUDA IPC handle size");
    std::memcpy(out, &h, 64);
    return AQR_OK;
}

aqr_status aqr_ipc_open(const uint8_t handle[64], void **out) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    AQR_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return AQR_OK;
}

aqr_status aqr_ipc_close(void *ptr) {
    if (ptr) AQR_CUDA(cudaIpcCloseMemHandle(ptr));
    return AQR_OK;
}

}  // extern "C"

namespace {

// One rank's peer-memory factorization, split into the phases of the step
// loop so that the single-rank driver (aqr_p2p_gs_factor) runs them in order
// and the lock-step emulation (aqr_p2p_gs_factor_lockstep) interleaves the
// ranks phase by phase on one stream.
struct P2PRun {
    aqr_factor_args *a = nullptr;
    const aqr_p2p_group *g = nullptr;
    cudaStream_t s = nullptr;
    int64_t m = 0, n = 0, ldw = 0, mv = 0;
    bool hp = false, cgs = false;
    int32_t *status = nullptr;
    unsigned *counters = nullptr;
    double *Rt = nullptr, *partial = nullptr, *npart = nullptr, *xvec = nullptr, *zvec = nullptr,
           *pring = nullptr, *X = nullptr, *Z0 = nullptr, *W = nullptr;
    int32_t ntiles = 0;
    aqr::P2PArgs P;
    aqr::CsrArgs c;
    std::vector<int32_t> st;
    // as Run: stored trailing columns at z^(zbase); HP's stored X at x^(xbase)
    int64_t zbase = 0, xbase = 0;

    double *col(double *B, int64_t ld, int64_t j) const { return B + j * ld; }

    aqr_status init(aqr_factor_args *args, const aqr_p2p_group *grp, cudaStream_t stream) {
        a = args;
        g = grp;
        s = stream;
        if (!a || !g) return set_err(AQR_EARG, "null args");
        a->fail_col = -1;
        a->fail_val = 0.0;
        a->mv_count = 0;
        m = a->m;
        n = a->n;
        if (g->nranks < 1 || g->nranks > aqr::kMaxRanks || g->rank < 0 || g->rank >= g->nranks)
            return set_err(AQR_EARG, "bad group");
        if (a->orientation != AQR_ROW || (a->variant != AQR_HA && a->variant != AQR_HP) || a->family < 0 ||
            a->family > 1)
            return set_err(AQR_EARG, "peer-memory path: row orientation, HA or HP");
        if (!a->op || a->op->kind != AQR_OP_CSR || a->op->m != m)
            return set_err(AQR_EARG, "peer-memory path: local CSR operator with m = local rows");
        if (n < 1 || m < 1) return set_err(AQR_EDIM, "empty local block");
        if (a->Q != g->W[g->rank] || a->ldq != g->ldw[g->rank] || a->ldq < m || !a->Z || a->ldz < m || !a->R ||
            a->ldr < n)
            return set_err(AQR_EARG, "Q must be the group's working matrix of this rank");
        if (g->n_halo > 0 && (!g->halo_rank || !g->halo_row)) return set_err(AQR_EARG, "halo tables missing");
        const Layout L = layout(a->family, a->variant, AQR_ROW, m, n);
        if (!a->workspace || a->workspace_bytes < L.total)
            return set_err(AQR_ENOMEM, "workspace smaller than aqr_workspace_bytes()");
        hp = a->variant == AQR_HP;
        cgs = a->family == AQR_CGS;
        void *ws = a->workspace;
        status = at<int32_t>(ws, L.status);
        counters = at<unsigned>(ws, L.counters);
        Rt = at<double>(ws, L.rt);
        partial = at<double>(ws, L.partial);
        npart = at<double>(ws, L.npart);
        xvec = at<double>(ws, L.xvec);
        zvec = at<double>(ws, L.zvec);
        pring = at<double>(ws, L.pring);
        X = at<double>(ws, L.X);
        Z0 = at<double>(ws, L.Z0);
        W = a->Q;
        ldw = a->ldq;
        ntiles = (int32_t)aqr::num_tiles(m);
        std::memset(&P, 0, sizeof P);
        P.nranks = g->nranks;
        P.rank = g->rank;
        for (int r = 0; r < g->nranks; ++r) {
            P.xb[r] = g->xbuf[r];
            P.W[r] = g->W[r];
            P.ldw[r] = g->ldw[r];
        }
        P.n = n;
        P.seq0 = g->seq0;
        P.m_loc = m;
        P.halo_rank = g->halo_rank;
        P.halo_row = g->halo_row;
        P.status = status;
        P.timeout_ns = g->timeout_ns ? g->timeout_ns : 60ull * 1000000000ull;
        const aqr_op *op = a->op;
        std::memset(&c, 0, sizeof c);
        c.m = m;
        c.indptr = op->indptr;
        c.indices = op->indices;
        c.data = op->data;
        c.trace = -1;
        return AQR_OK;
    }

    // Z into W, the status block, the start barrier (this rank's Z is in place).
    aqr_status begin() {
        if (a->Z != a->Q) AQR_CUDA(copy_cols(a->Q, a->ldq, a->Z, a->ldz, m, n, cudaMemcpyDeviceToDevice, s));
        AQR_TRY(aqr_status_init(status, n, s));
        AQR_CUDA(cudaMemsetAsync(counters, 0, 4 * (size_t)(n + 8), s));
        AQR_CUDA(cudaMemsetAsync(Rt, 0, 8 * (size_t)n * n, s));
        if (cgs) AQR_CUDA(copy_cols(Z0, m, a->Q, a->ldq, m, n, cudaMemcpyDeviceToDevice, s));
        aqr::p2p_barrier_kernel<<<1, 1, 0, s>>>(P);
        return launched("p2p_barrier_kernel");
    }

    // HP: X = op.apply_block(Zw) (line 136), halo columns from the owners
    // (waits for every rank's start barrier).
    aqr_status block_apply() {
        if (!hp) return AQR_OK;
        aqr::CsrArgs b = c;
        b.k = n;
        b.X = W;
        b.ldx = ldw;
        b.Y = X;
        b.ldy = m;
        const int64_t nb = (m + aqr::kBlock - 1) / aqr::kBlock;
        aqr::p2p_csr_block_kernel<<<(unsigned)std::min<int64_t>(nb, (int64_t)sm_count() * 8), aqr::kBlock, 0, s>>>(b, P);
        AQR_TRY(launched("p2p_csr_block_kernel"));
        mv += n;
        return AQR_OK;
    }

    // Step i, first launch: r_{i-1,i} from the exchanged R rows, the deferred
    // column update (+ SpMV for HA), the norm partials -> every rank.
    aqr_status norm(int64_t i) {
        aqr::NormOut o;
        std::memset(&o, 0, sizeof o);
        o.npart = npart;
        o.ntiles = (int32_t)aqr::norm_tiles(m, hp);
        o.counter = counters;
        o.step = i;
        o.status = status;
        const unsigned gn = (unsigned)aqr::norm_tiles(m, hp);
        if (hp) {  // lazy x: X_i at x^(xbase), p_k in X's column k (k < i)
            aqr::ColArgs ca;
            std::memset(&ca, 0, sizeof ca);
            ca.m = m;
            ca.z = col(W, ldw, i);
            ca.qprev = i > 0 ? col(W, ldw, i - 1) : nullptr;
            ca.x = col(X, m, i);
            ca.P = col(X, m, xbase);
            ca.ldp = m;
            ca.rcol = Rt + xbase * n + i;
            ca.rstride = n;
            ca.nprev = (int32_t)(i - xbase);
            ca.xout = pring + (i & 1) * m;
            ca.out = o;
            ca.trace = -1;
            launch_pdl(aqr::p2p_col_lazy_kernel, gn, aqr::kBlock, 0, s, ca, P, i, Rt);
            AQR_TRY(launched("p2p_col_lazy_kernel"));
            // every x_win() steps the stored X columns i+1 .. n-1 catch up
            // (local rows; R rows < i are final once this kernel ran)
            if (i - xbase >= x_win() && i + 1 < n) {
                AQR_TRY(launch_x_catchup(m, X, m, i + 1, n, col(X, m, xbase), m, Rt + xbase * n, n, i - xbase,
                                         status, s));
                xbase = i;
            }
            return AQR_OK;
        }
        aqr::CsrArgs ca = c;
        ca.k = 1;
        ca.X = col(W, ldw, i);
        ca.ldx = m;
        ca.qprev = i > 0 ? col(W, ldw, i - 1) : nullptr;
        ca.Y = xvec;
        ca.ldy = m;
        ca.znew = zvec;
        ca.out = o;
        if (a->op->max_row_nnz >= 1 && a->op->max_row_nnz <= 5)
            launch_pdl(aqr::p2p_csr_step_kernel<5>, gn, aqr::kBlock, 0, s, ca, P, i, Rt);
        else
            launch_pdl(aqr::p2p_csr_step_kernel<8>, gn, aqr::kBlock, 0, s, ca, P, i, Rt);
        ++mv;
        return launched("p2p_csr_step_kernel");
    }

    // Step i, second launch: r_ii from every rank's norm totals, the trailing pass.
    aqr_status trail(int64_t i) {
        aqr::TrailArgs t;
        std::memset(&t, 0, sizeof t);
        t.m = m;
        t.ntiles = ntiles;
        t.jbeg = (int32_t)(i + 1);
        t.jend = (int32_t)n;
        t.W = W;
        t.ldw = ldw;
        t.X = X;
        t.ldx = m;
        t.Z0 = Z0;
        t.ldz0 = m;
        // windowed: projections zbase .. i-1 applied in registers, the block
        // written back every trail_win()-th pass (column i+1 by every pass
        // with a window: the next step's SpMV halo reads it on the peers)
        t.win = t.jend > t.jbeg ? (int32_t)(i - zbase) : 0;
        t.store_all = t.win >= trail_win() ? 1 : 0;
        t.qwin = t.win > 0 ? col(W, ldw, zbase) : nullptr;
        t.rwin = t.win > 0 ? Rt + zbase * n : nullptr;
        t.rstride = n;
        t.psrc = hp ? pring + (i & 1) * m : xvec;
        t.zsrc = hp ? col(W, ldw, i) : zvec;
        t.qout = col(W, ldw, i);
        t.pout = hp ? col(X, m, i) : nullptr;  // p_i kept for the lazy x of later steps
        t.partial = partial;
        t.status = status;
        t.trace = -1;
        t.reverse = (int32_t)(i & 1);  // backwards on odd steps (L2 reuse, as the single-GPU pass)
        double *rii = Rt + i * n + i;
        const aqr_status st = cgs ? launch_p2p_trailing<true>(t, P, i, rii, status, s)
                                  : launch_p2p_trailing<false>(t, P, i, rii, status, s);
        if (t.store_all) zbase = i;
        return st;
    }

    // Step i, third launch: this rank's R-row totals -> every rank.
    aqr_status rrow(int64_t i) {
        if (i + 1 >= n) return AQR_OK;
        launch_pdl(aqr::p2p_rrow_kernel, (unsigned)(n - 1 - i), aqr::kBlock, 0, s, (const double *)partial,
                   (int32_t)ntiles, (int64_t)(i + 1), P, (int64_t)i, counters + 1, (const int32_t *)status);
        return launched("p2p_rrow_kernel");
    }

    aqr_status end() {
        aqr::finalize_r_kernel<<<(unsigned)((n * n + 255) / 256), 256, 0, s>>>(n, Rt, a->R, a->ldr);
        AQR_TRY(launched("finalize_r_kernel"));
        st.assign((16 + 4 * n) / 4, 0);
        AQR_CUDA(cudaMemcpyAsync(st.data(), status, 16 + 4 * n, cudaMemcpyDeviceToHost, s));
        return AQR_OK;
    }

    // After the stream drained: the status record -> return code / outputs.
    aqr_status finish() {
        a->mv_count = mv;
        if (st[1] == 1) return set_err(AQR_ETIMEOUT, "peer exchange timed out (a rank is missing or failed)");
        if (a->flagged_host) std::memcpy(a->flagged_host, st.data() + 4, 4 * n);
        if (st[0] >= 0) {
            a->fail_col = st[0];
            std::memcpy(&a->fail_val, st.data() + 2, 8);
            return set_err(AQR_EBREAKDOWN, "breakdown at column " + std::to_string(st[0]));
        }
        return AQR_OK;
    }
};

}  // namespace

extern "C" {

aqr_status aqr_p2p_gs_factor(aqr_factor_args *a, const aqr_p2p_group *g, void *stream) {
    P2PRun r;
    AQR_TRY(r.init(a, g, S(stream)));
    AQR_TRY(r.begin());
    AQR_TRY(r.block_apply());
    for (int64_t i = 0; i < r.n; ++i) {
        AQR_TRY(r.norm(i));
        AQR_TRY(r.trail(i));
        AQR_TRY(r.rrow(i));
    }
    AQR_TRY(r.end());
    AQR_CUDA(cudaStreamSynchronize(r.s));
    return r.finish();
}

aqr_status aqr_p2p_gs_factor_lockstep(int32_t nranks, aqr_factor_args *const *args,
                                      const aqr_p2p_group *const *groups, void *stream) {
    if (nranks < 1 || nranks > aqr::kMaxRanks || !args || !groups) return set_err(AQR_EARG, "bad rank list");
    std::vector<P2PRun> runs((size_t)nranks);
    for (int r = 0; r < nranks; ++r) {
        AQR_TRY(runs[r].init(args[r], groups[r], S(stream)));
        if (groups[r]->rank != r || groups[r]->nranks != nranks || runs[r].n != runs[0].n)
            return set_err(AQR_EARG, "lock-step ranks must be 0..nranks-1 of one group, same n");
    }
    // every phase of every rank is enqueued only after the phases it waits
    // for (stream order), so no kernel ever spins on a flag not yet raised
    for (auto &r : runs) AQR_TRY(r.begin());
    for (auto &r : runs) AQR_TRY(r.block_apply());
    for (int64_t i = 0; i < runs[0].n; ++i) {
        for (auto &r : runs) AQR_TRY(r.norm(i));
        for (auto &r : runs) AQR_TRY(r.trail(i));
        for (auto &r : runs) AQR_TRY(r.rrow(i));
    }
    for (auto &r : runs) AQR_TRY(r.end());
    AQR_CUDA(cudaStreamSynchronize(S(stream)));
    aqr_status first = AQR_OK;
    for (auto &r : runs) {
        const aqr_status st = r.finish();
        if (first == AQR_OK) first = st;
    }
    return first;
}

aqr_status aqr_gs_factor_host(int32_t family, int32_t variant, int32_t orientation, int64_t m,
                              int64_t n, const double *Z_host, double *Q_host, double *R_host,
                              int32_t op_kind, const double *A_host, const int64_t *indptr_host,
                              const int64_t *indices_host, const double *data_host, int64_t nnz,
                              int64_t *fail_col, double *fail_val, int32_t *flagged_host,
                              int64_t *mv_count) {
    if (n < 1 || m < n) return set_err(AQR_EDIM, "need m >= n >= 1");
    if (op_kind == AQR_OP_CSR && (nnz >= ((int64_t)1 << 31) || m >= ((int64_t)1 << 31)))
        return set_err(AQR_EARG, "nnz/m >= 2^31 does not fit the int32 CSR layout");
    cudaStream_t s;
    AQR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    std::vector<void *> bufs;
    auto dalloc = [&](size_t bytes) -> void * {
        void *p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(bytes, 256), s) != cudaSuccess) return nullptr;
        bufs.push_back(p);
        return p;
    };
    auto cleanup = [&]() {
        for (void *p : bufs) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    };
    aqr_op op;
    std::memset(&op, 0, sizeof op);
    op.kind = op_kind;
    op.m = m;
    aqr_status st = AQR_OK;
    double *Q = (double *)dalloc(8 * (size_t)m * n);
    double *R = (double *)dalloc(8 * (size_t)n * n);
    const uint64_t wsb = aqr_workspace_bytes(family, variant, orientation, m, n);
    void *ws = dalloc(wsb);
    std::vector<int32_t> ip32, ix32;
    if (!Q || !R || !ws) st = set_err(AQR_ENOMEM, "device allocation failed");
    if (st == AQR_OK && op_kind == AQR_OP_DENSE) {
        double *A = (double *)dalloc(8 * (size_t)m * m);
        if (!A) st = set_err(AQR_ENOMEM, "device allocation failed");
        else if (cudaMemcpyAsync(A, A_host, 8 * (size_t)m * m, cudaMemcpyHostToDevice, s) != cudaSuccess)
            st = set_err(AQR_ECUDA, "H2D A");
        op.A = A;
        op.lda = m;
    } else if (st == AQR_OK && op_kind == AQR_OP_CSR) {
        ip32.resize(m + 1);
        ix32.resize(nnz);
        int64_t longest = 0;
        for (int64_t i = 0; i <= m; ++i) {
            ip32[i] = (int32_t)indptr_host[i];
            if (i > 0) longest = std::max<int64_t>(longest, indptr_host[i] - indptr_host[i - 1]);
        }
        op.max_row_nnz = (int32_t)std::min<int64_t>(longest, INT32_MAX);
        for (int64_t k = 0; k < nnz; ++k) ix32[k] = (int32_t)indices_host[k];
        int32_t *ip = (int32_t *)dalloc(4 * (size_t)(m + 1));
        int32_t *ix = (int32_t *)dalloc(4 * (size_t)nnz);
        double *dv = (double *)dalloc(8 * (size_t)nnz);
        if (!ip || !ix || !dv) st = set_err(AQR_ENOMEM, "device allocation failed");
        else if (cudaMemcpyAsync(ip, ip32.data(), 4 * (m + 1), cudaMemcpyHostToDevice, s) != cudaSuccess ||
                 cudaMemcpyAsync(ix, ix32.data(), 4 * nnz, cudaMemcpyHostToDevice, s) != cudaSuccess ||
                 cudaMemcpyAsync(dv, data_host, 8 * nnz, cudaMemcpyHostToDevice, s) != cudaSuccess)
            st = set_err(AQR_ECUDA, "H2D CSR");
        op.indptr = ip;
        op.indices = ix;
        op.data = dv;
        op.nnz = nnz;
    } else if (st == AQR_OK) {
        st = set_err(AQR_EARG, "host entry supports dense and CSR operators");
    }
    if (st == AQR_OK && cudaMemcpyAsync(Q, Z_host, 8 * (size_t)m * n, cudaMemcpyHostToDevice, s) != cudaSuccess)
        st = set_err(AQR_ECUDA, "H2D Z");
    aqr_band band;  // stencil operators run on the banded view (nd == 0: plain CSR)
    std::memset(&band, 0, sizeof band);
    if (st == AQR_OK && op_kind == AQR_OP_CSR && aqr_csr_band_create(&op, &band, s) == AQR_OK && band.nd > 0)
        op.band = &band;
    aqr_factor_args a;
    std::memset(&a, 0, sizeof a);
    if (st == AQR_OK) {
        a.family = family;
        a.variant = variant;
        a.orientation = orientation;
        a.m = m;
        a.n = n;
        a.Z = Q;
        a.ldz = m;
        a.Q = Q;
        a.ldq = m;
        a.R = R;
        a.ldr = n;
        a.op = &op;
        a.workspace = ws;
        a.workspace_bytes = wsb;
        a.flagged_host = flagged_host;
        st = aqr_gs_factor_d2h(&a, Q_host, m, R_host, n, s);  // Q streamed as columns finish
        if (fail_col) *fail_col = a.fail_col;
        if (fail_val) *fail_val = a.fail_val;
        if (mv_count) *mv_count = a.mv_count;
    }
    aqr_csr_band_destroy(&band);
    cleanup();
    return st;
}

aqr_status aqr_op_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                        int64_t ldy, void *stream) {
    const int64_t xrows = (op && op->kind == AQR_OP_DENSE && op->ncols > 0) ? op->ncols : (op ? op->m : 0);
    if (!op || k < 0 || (k > 1 && ldx < xrows) || ldy < op->m) return set_err(AQR_EARG, "bad apply arguments");
    if (k == 0) return AQR_OK;
    return op_apply(op, k, X, ldx, Y, ldy, S(stream));
}

aqr_status aqr_block_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y, int64_t ldy,
                           void *stream) {
    const int64_t xrows = (op && op->kind == AQR_OP_DENSE && op->ncols > 0) ? op->ncols : (op ? op->m : 0);
    if (!op || k < 0 || (k > 1 && ldx < xrows) || ldy < op->m) return set_err(AQR_EARG, "bad apply arguments");
    if (k == 0) return AQR_OK;
    return block_apply(op, k, X, ldx, Y, ldy, S(stream));
}

aqr_status aqr_dot(int64_t m, const double *x, const double *y, double *out, void *stream) {
    const int64_t nt = aqr::num_tiles(m);
    if (nt == 0) return set_err(AQR_EARG, "empty vector");
    double *part = nullptr;
    AQR_CUDA(cudaMallocAsync(&part, 8 * nt, S(stream)));
    aqr::dot_partial_kernel<<<(unsigned)nt, aqr::kBlock, 0, S(stream)>>>(m, aqr::rows_per_thread(m), x, y, part);
    aqr_status st = launched("dot_partial_kernel");
    if (st == AQR_OK) st = launch_rrow_reduce(m, 1, part, out, nullptr, S(stream));
    cudaFreeAsync(part, S(stream));
    return st;
}

aqr_status aqr_sub_scaled(int64_t m, double *z, const double *a_dev, const double *q, void *stream) {
    aqr::sub_scaled_kernel<<<elementwise_grid(m), aqr::kBlock, 0, S(stream)>>>(m, z, a_dev, q);
    return launched("sub_scaled_kernel");
}

aqr_status aqr_div_scalar(int64_t m, const double *x, const double *r_dev, double *out, void *stream) {
    aqr::div_scalar_kernel<<<elementwise_grid(m), aqr::kBlock, 0, S(stream)>>>(m, x, r_dev, out);
    return launched("div_scalar_kernel");
}

aqr_status aqr_matvec(int64_t m, const double *A, int64_t lda, const double *x, double *y, void *stream) {
    aqr_op op;
    std::memset(&op, 0, sizeof op);
    op.kind = AQR_OP_DENSE;
    op.m = m;
    op.A = A;
    op.lda = lda;
    return aqr_op_apply(&op, 1, x, m, y, m, stream);
}

aqr_status aqr_apply_block_dense(int64_t m, int64_t k, const double *A, int64_t lda, const double *X,
                                 int64_t ldx, double *Y, int64_t ldy, void *stream) {
    aqr_op op;
    std::memset(&op, 0, sizeof op);
    op.kind = AQR_OP_DENSE;
    op.m = m;
    op.A = A;
    op.lda = lda;
    return aqr_op_apply(&op, k, X, ldx, Y, ldy, stream);
}

aqr_status aqr_csr_matvec(int64_t m, const int32_t *indptr, const int32_t *indices, const double *data,
                          const double *x, double *y, void *stream) {
    aqr_op op;
    std::memset(&op, 0, sizeof op);
    op.kind = AQR_OP_CSR;
    op.m = m;
    op.indptr = indptr;
    op.indices = indices;
    op.data = data;
    return aqr_op_apply(&op, 1, x, m, y, m, stream);
}

// ---- banded view of a CSR operator (aqr_band.cuh) -----------------------------

aqr_status aqr_csr_band_create(const aqr_op *csr, aqr_band *out, void *stream) {
    if (!out) return set_err(AQR_EARG, "null band");
    std::memset(out, 0, sizeof *out);
    if (!csr || csr->kind != AQR_OP_CSR || !csr->indptr || (csr->nnz && (!csr->indices || !csr->data)))
        return set_err(AQR_EARG, "band analysis needs a CSR operator");
    const int64_t m = csr->m, nnz = csr->nnz;
    if (m < 1 || nnz < 1) return AQR_OK;
    cudaStream_t s = S(stream);
    aqr::BandScan *sc = nullptr;
    uint32_t *mask = nullptr;
    double *dvals = nullptr;
    auto fail = [&](aqr_status st, const char *msg) {
        cudaFree(sc);
        cudaFree(mask);
        cudaFree(dvals);
        return msg ? set_err(st, msg) : st;
    };
    if (cudaMalloc(&sc, sizeof(aqr::BandScan)) != cudaSuccess) return fail(AQR_ENOMEM, "band: device allocation failed");
    const unsigned grid = (unsigned)((m + aqr::kBlock - 1) / aqr::kBlock);
    aqr::band_scan_init_kernel<<<1, 64, 0, s>>>(sc);
    aqr::band_collect_kernel<<<grid, aqr::kBlock, 0, s>>>(m, csr->indptr, csr->indices, sc);
    aqr::BandScan h;
    if (cudaMemcpyAsync(&h, sc, sizeof h, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(AQR_ECUDA, "band: offset scan failed");
    std::vector<int64_t> offs;
    for (int i = 0; i < aqr::kBandSlots; ++i)
        if (h.keys[i] != aqr::kBandEmpty) offs.push_back((int64_t)h.keys[i]);
    // not banded: too many offsets, unsorted rows, or diagonals less than half populated
    if (h.bad || offs.empty() || offs.size() > (size_t)aqr::kBandMax || 2 * nnz < (int64_t)offs.size() * m)
        return fail(AQR_OK, nullptr);
    std::sort(offs.begin(), offs.end());
    aqr::BandDesc d;
    std::memset(&d, 0, sizeof d);
    d.nd = (int32_t)offs.size();
    for (int i = 0; i < d.nd; ++i) d.off[i] = offs[(size_t)i];
    if (cudaMalloc(&mask, 4 * (size_t)m) != cudaSuccess) return fail(AQR_ENOMEM, "band: device allocation failed");
    aqr::band_mask_kernel<<<grid, aqr::kBlock, 0, s>>>(m, csr->indptr, csr->indices, csr->data, d, mask, sc);
    if (cudaMemcpyAsync(&h, sc, sizeof h, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(AQR_ECUDA, "band: mask pass failed");
    if (h.bad) return fail(AQR_OK, nullptr);
    if (h.varying) {
        if (cudaMalloc(&dvals, 8 * (size_t)m * (size_t)d.nd) != cudaSuccess)
            return fail(AQR_OK, nullptr);  // no room for the diagonal-major values: stay on CSR
        cudaMemsetAsync(dvals, 0, 8 * (size_t)m * (size_t)d.nd, s);
        aqr::band_vals_kernel<<<grid, aqr::kBlock, 0, s>>>(m, csr->indptr, csr->indices, csr->data, d, dvals);
        if (cudaStreamSynchronize(s) != cudaSuccess) return fail(AQR_ECUDA, "band: value pass failed");
    }
    cudaFree(sc);
    out->nd = d.nd;
    out->constant = h.varying ? 0 : 1;
    for (int i = 0; i < d.nd; ++i) {
        out->off[i] = d.off[i];
        const long long bits = (long long)h.first[i];
        double v;
        std::memcpy(&v, &bits, 8);
        out->val[i] = h.varying ? 0.0 : v;
    }
    out->mask = mask;
    out->dvals = dvals;
    return AQR_OK;
}

void aqr_csr_band_destroy(aqr_band *band) {
    if (!band) return;
    cudaFree(const_cast<uint32_t *>(band->mask));
    cudaFree(const_cast<double *>(band->dvals));
    std::memset(band, 0, sizeof *band);
}

// ---- dense helpers in the reference's order (aqr_dense.cuh) -----------------

aqr_status aqr_gemm_tn(int64_t m, int64_t p, int64_t n, const double *A, int64_t lda, const double *B,
                       int64_t ldb, double *C, int64_t ldc, void *stream) {
    if (m < 0 || p < 0 || n < 0 || (m > 0 && (lda < m || ldb < m)) || ldc < std::max<int64_t>(p, 1))
        return set_err(AQR_EARG, "gemm_tn: bad shape / leading dimension");
    if (p == 0 || n == 0) return AQR_OK;
    dim3 grid((unsigned)((p + aqr::kTnTile - 1) / aqr::kTnTile), (unsigned)((n + aqr::kTnTile - 1) / aqr::kTnTile));
    aqr::gemm_tn_seq_kernel<<<grid, aqr::kBlock, 0, S(stream)>>>(m, p, n, A, lda, B, ldb, C, ldc);
    return launched("gemm_tn_seq_kernel");
}

aqr_status aqr_gemm_nn(int64_t m, int64_t kk, int64_t n, const double *A, int64_t lda, const double *B,
                       int64_t ldb, double *C, int64_t ldc, void *stream) {
    if (m < 0 || kk < 0 || n < 0 || lda < std::max<int64_t>(m, 1) || ldb < std::max<int64_t>(kk, 1) ||
        ldc < std::max<int64_t>(m, 1))
        return set_err(AQR_EARG, "gemm_nn: bad shape / leading dimension");
    if (m == 0 || n == 0) return AQR_OK;
    if (kk == 0) {
        AQR_CUDA(cudaMemset2DAsync(C, 8 * (size_t)ldc, 0, 8 * (size_t)m, (size_t)n, S(stream)));
        return AQR_OK;
    }
    // C(:, j) accumulates exactly like matvec: the rectangular dense apply
    aqr_op op;
    std::memset(&op, 0, sizeof op);
    op.kind = AQR_OP_DENSE;
    op.m = m;
    op.ncols = kk;
    op.A = A;
    op.lda = lda;
    return dense_apply(&op, n, B, ldb, C, ldc, S(stream));
}

aqr_status aqr_cholesky_upper(int64_t n, const double *G, int64_t ldg, double *R, int64_t ldr, int32_t *fail_dev,
                              void *stream) {
    if (n < 1 || ldg < n || ldr < n || !G || !R || !fail_dev) return set_err(AQR_EARG, "cholesky_upper: bad arguments");
    aqr::cholesky_upper_kernel<<<1, aqr::kBlock, 0, S(stream)>>>(n, G, ldg, R, ldr, fail_dev);
    return launched("cholesky_upper_kernel");
}

aqr_status aqr_tri_solve_right(int64_t m, int64_t n, const double *Z, int64_t ldz, const double *R, int64_t ldr,
                               double *X, int64_t ldx, void *stream) {
    if (m < 0 || n < 1 || ldz < std::max<int64_t>(m, 1) || ldx < std::max<int64_t>(m, 1) || ldr < n)
        return set_err(AQR_EARG, "tri_solve_right: bad shape / leading dimension");
    if (m == 0) return AQR_OK;
    const int64_t grid = std::min<int64_t>((m + aqr::kBlock - 1) / aqr::kBlock, (int64_t)sm_count() * 8);
    aqr::tri_solve_right_kernel<<<(unsigned)grid, aqr::kBlock, 0, S(stream)>>>(m, n, Z, ldz, R, ldr, X, ldx);
    return launched("tri_solve_right_kernel");
}

aqr_status aqr_step_col_update_norm(int64_t m, double *z, const double *qprev, double *x,
                                    const double *pprev, const double *r_dev, const double *xnorm,
                                    double *npart, const int32_t *status, void *stream) {
    aqr::NormOut o = no_norm();
    o.npart = npart;
    o.status = const_cast<int32_t *>(status);
    // HP carries x (passed as x); HA / naive pass the product as xnorm
    return launch_col_update_norm(m, z, qprev, x, pprev, r_dev, xnorm, o, x != nullptr, S(stream));
}

aqr_status aqr_step_norm_reduce(int64_t m, int32_t variant, const double *npart, double *tot,
                                const int32_t *status, void *stream) {
    const bool hp = variant == AQR_HP;
    aqr::norm_reduce_kernel<<<1, aqr::kBlock, 0, S(stream)>>>(npart, (int32_t)aqr::norm_tiles(m, hp), tot, 0,
                                                            nullptr, const_cast<int32_t *>(status));
    return launched("norm_reduce_kernel");
}

aqr_status aqr_step_norm_finish(int64_t i, const double *tot, double *rii, int32_t *status, void *stream) {
    aqr::norm_finish_kernel<<<1, 1, 0, S(stream)>>>(i, tot, rii, status);
    return launched("norm_finish_kernel");
}

aqr_status aqr_step_normalize(int64_t m, const double *z, const double *rii, double *q, const double *x,
                              double *p, const int32_t *status, void *stream) {
    return launch_normalize(m, z, rii, q, x, p, status, S(stream));
}

aqr_status aqr_step_trailing(int64_t m, int64_t i, int64_t jbeg, int64_t jend, double *W, int64_t ldw,
                             double *X, int64_t ldx, const double *Z0, int64_t ldz0, const double *qprev,
                             const double *pprev, const double *rprev, const double *psrc,
                             const double *rii, double *pout, const double *zsrc, double *qout,
                             double *partial, const int32_t *status, void *stream) {
    aqr::TrailArgs t;
    std::memset(&t, 0, sizeof t);
    t.m = m;
    t.ntiles = (int32_t)aqr::num_tiles(m);
    t.jbeg = (int32_t)jbeg;
    t.jend = (int32_t)jend;
    t.reverse = (int32_t)(i & 1);
    t.W = W;
    t.ldw = ldw;
    t.X = X;
    t.ldx = ldx;
    t.Z0 = Z0;
    t.ldz0 = ldz0;
    t.qprev = qprev;
    t.pprev = pprev;
    t.rprev = rprev;
    t.psrc = psrc;
    t.rii = rii;
    t.pout = pout;
    t.zsrc = zsrc;
    t.qout = qout;
    t.partial = partial;
    t.status = status;
    if (qprev && !rprev) return set_err(AQR_EARG, "qprev without rprev");
    if (X == nullptr && pprev != nullptr) return set_err(AQR_EARG, "pprev without X");
    return launch_trailing(t, X != nullptr, Z0 != nullptr, S(stream));
}

aqr_status aqr_step_rrow_reduce(int64_t m, int64_t ncols, const double *partial, double *out,
                                const int32_t *status, void *stream) {
    return launch_rrow_reduce(m, ncols, partial, out, status, S(stream));
}

aqr_status aqr_step_finalize_r(int64_t n, const double *Rt, double *R, int64_t ldr, void *stream) {
    aqr::finalize_r_kernel<<<(unsigned)((n * n + 255) / 256), 256, 0, S(stream)>>>(n, Rt, R, ldr);
    return launched("finalize_r_kernel");
}

}  // extern "C"
