/*
 * aqr_b200.h -- C ABI of libaqr_b200.so, the B200 (sm_100a) implementation of
 * the A-orthogonal modified Gram-Schmidt hot path of the reference package
 * `aqr` (arXiv 1703.10440).
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; no torch/C++ types cross this boundary;
 *   - every double* / int32_t* argument is a DEVICE pointer unless the name
 *     ends in _host;
 *   - matrices are column-major (Fortran) with an explicit leading dimension,
 *     the layout aqr.operators.as_matrix produces (operators.py:28-33);
 *   - work is enqueued on the caller's `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream); nothing allocates on the hot path
 *     except the *_host convenience entry, which owns its device buffers;
 *   - every function returns an aqr_status; aqr_last_error() describes the
 *     last failure on the calling thread.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/aqr):
 *   aqr_gs_factor / aqr_gs_factor_host  <- gram_schmidt._gs_factor (126-179),
 *       reached by mgs_naive/mgs_ha/mgs_hp/cgs/factorize (182-206, 227-233)
 *   aqr_op (+ callbacks)                <- operators.SpdOperator.apply /
 *       apply_block plug-in point (operators.py:43-73), DenseSpdOperator
 *       (76-93), CsrSpdOperator (96-129)
 *   aqr_dot / aqr_sub_scaled / aqr_div_scalar / aqr_matvec /
 *   aqr_apply_block_dense / aqr_csr_matvec <- the kernel namespace returned
 *       by backend.kernels() (backend.py:66-68): seq_dot, sub_scaled,
 *       div_scalar, matvec, apply_block_dense, csr_matvec
 *       (_kernels_impl.py:17-56, 85-93)
 *   aqr_block_apply                     <- SpdOperator.apply_block (58-66) as
 *       the HP path calls it (gram_schmidt.py:136): dense operators on the
 *       FP64 tensor cores, otherwise aqr_op_apply
 *   aqr_step_*                          <- the bodies of _gs_factor's
 *       project(i, j) (139-145) and normalize(j) (147-165), restated as the
 *       fused one-pass-per-step schedule used by the multi-GPU driver.
 */
#ifndef AQR_B200_H
#define AQR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AQR_ABI_VERSION 3

#if defined(__GNUC__)
#define AQR_API __attribute__((visibility("default")))
#else
#define AQR_API
#endif

typedef enum {
    AQR_OK = 0,
    AQR_EDIM = 1,       /* DimensionError (gram_schmidt.py:116-123)            */
    AQR_EBREAKDOWN = 2, /* BreakdownError(column, value) (gram_schmidt.py:153) */
    AQR_ECUDA = 3,      /* CUDA runtime / launch failure                       */
    AQR_EARG = 4,       /* bad enum, null pointer, size out of range           */
    AQR_ENOMEM = 5,     /* workspace too small / device allocation failed      */
    AQR_ECALLBACK = 6,  /* a user operator callback returned non-zero          */
    AQR_ETIMEOUT = 7    /* multi-GPU: a peer's exchange flag did not arrive in
                           time (the group must be re-created on every rank) */
} aqr_status;

typedef enum { AQR_MGS = 0, AQR_CGS = 1 } aqr_family;           /* MethodId.family  */
typedef enum { AQR_NAIVE = 0, AQR_HA = 1, AQR_HP = 2 } aqr_variant; /* MethodId.variant */
typedef enum { AQR_COL = 0, AQR_ROW = 1 } aqr_orientation;      /* MethodId.orientation */

typedef enum {
    AQR_OP_DENSE = 0,   /* DenseSpdOperator: A m x m column-major, lda >= m   */
    AQR_OP_CSR = 1,     /* CsrSpdOperator: int32 indptr/indices, fp64 data    */
    AQR_OP_CALLBACK = 2 /* user operator: apply/apply_block callbacks         */
} aqr_op_kind;

/* Y[:, 0:k] = A X[:, 0:k] on `stream`; return 0 on success.  k == 1 is
 * SpdOperator.apply, k > 1 SpdOperator.apply_block. */
typedef int (*aqr_apply_fn)(void *ctx, int64_t k, const double *X, int64_t ldx, double *Y,
                            int64_t ldy, void *stream);

/* Banded view of a CSR operator whose rows carry a fixed set of column
 * offsets (stencils): built once by aqr_csr_band_create, attached to the
 * operator through aqr_op.band.  The SpMV / SpMM kernels then form a row's
 * gather addresses from its row number (4 bytes of mask per row instead of
 * 12 bytes per entry); sums run in stored order, results are bitwise those
 * of the CSR kernels (csr_matvec, _kernels_impl.py:50-56). */
#define AQR_BAND_MAX 32
typedef struct aqr_band {
    int32_t nd;       /* distinct offsets col - row (0: the operator is not banded) */
    int32_t constant; /* 1: every diagonal carries one value (val[d])             */
    int64_t off[AQR_BAND_MAX]; /* ascending                                       */
    double val[AQR_BAND_MAX];
    const uint32_t *mask; /* device, m words: bit d = row has an entry at off[d]  */
    const double *dvals;  /* device, nd x m diagonal-major values (constant == 0) */
} aqr_band;

typedef struct aqr_op {
    int32_t kind; /* aqr_op_kind */
    int32_t max_row_nnz; /* CSR: longest row (0 = unknown); picks the SpMV row batch, results unchanged */
    int64_t m;
    /* AQR_OP_DENSE */
    const double *A;
    int64_t lda;
    /* AQR_OP_CSR (nnz < 2^31) */
    const int32_t *indptr;
    const int32_t *indices;
    const double *data;
    int64_t nnz;
    /* AQR_OP_CALLBACK */
    aqr_apply_fn apply;       /* called with k == 1                      */
    aqr_apply_fn apply_block; /* called with k == n (HP); may equal apply */
    void *ctx;
    /* AQR_OP_DENSE: columns of A (0 = m, square).  A local row panel of a
     * row-partitioned operator is m_local x ncols (multi-GPU driver). */
    int64_t ncols;
    /* AQR_OP_CSR: optional banded view (NULL: plain CSR kernels) */
    const aqr_band *band;
} aqr_op;

/* Analyses a device CSR operator (ascending column indices per row, at most
 * AQR_BAND_MAX distinct offsets, diagonals at least half populated) and
 * allocates the view's device arrays; out->nd == 0 when the operator does
 * not qualify (not an error).  Synchronizes `stream`. */
AQR_API aqr_status aqr_csr_band_create(const aqr_op *csr, aqr_band *out, void *stream);
AQR_API void aqr_csr_band_destroy(aqr_band *band);

/* Everything _gs_factor takes and returns.  Inputs above the marker. */
typedef struct aqr_factor_args {
    int32_t family, variant, orientation;
    int32_t reserved;
    int64_t m, n;
    const double *Z; /* m x n, ldz; may alias Q (then factorized in place) */
    int64_t ldz;
    double *Q; /* m x n output, ldq */
    int64_t ldq;
    double *R; /* n x n output, ldr; strict lower part set to 0.0 */
    int64_t ldr;
    const aqr_op *op;
    void *workspace; /* device, >= aqr_workspace_bytes(...) bytes, 256-B aligned */
    uint64_t workspace_bytes;
    /* ---- outputs (host memory) ---- */
    int64_t fail_col;        /* -1, or the BreakdownError column           */
    double fail_val;         /* the offending z'Az                          */
    int64_t mv_count;        /* operator applications performed (built-in ops) */
    int32_t *flagged_host;   /* optional: n entries, 1 where column flagged */
} aqr_factor_args;

/* ---- whole factorization (the drop-in for _gs_factor) ------------------ */

AQR_API uint64_t aqr_workspace_bytes(int32_t family, int32_t variant, int32_t orientation, int64_t m,
                             int64_t n);

/* Runs the full factorization on `stream`, then synchronizes it to read the
 * breakdown/flag record (one small D2H copy).  AQR_EBREAKDOWN leaves Q/R
 * undefined, as the reference raises without a partial result. */
AQR_API aqr_status aqr_gs_factor(aqr_factor_args *args, void *stream);

/* As aqr_gs_factor, and every column of Q is copied to Q_host (column-major,
 * leading dimension ldqh; page-locked memory for the copies to overlap) as
 * soon as it is final -- column i after step i -- on an internal copy
 * stream, so the device-to-host transfer of Q overlaps the remaining steps;
 * R goes to R_host (ldrh) at the end.  Returns after all copies completed.
 * Used by the Python API for page-locked host inputs and by
 * aqr_gs_factor_host. */
AQR_API aqr_status aqr_gs_factor_d2h(aqr_factor_args *args, double *Q_host, int64_t ldqh, double *R_host,
                                     int64_t ldrh, void *stream);

/* Host Z in, host Q / R out, with both transfers overlapped with the
 * factorization (row orientation): Z is copied in chunks of `chunk_cols`
 * columns (0 = the library's schedule, see aqr_pipe_chunks) on an internal
 * stream; when `ready` (page-locked
 * host memory) is given, chunk c is copied only once *ready >= c + 1, so the
 * caller can still be writing later chunks into Z_host (a GPU-side stream
 * wait; the caller advances *ready in chunk order); the step loop brings a chunk in
 * when it needs it, after replaying the steps already done on it (the same
 * trailing passes and reduction trees: results are bitwise those of
 * aqr_gs_factor), and Q columns stream out as in aqr_gs_factor_d2h.  args->Q
 * is the device working matrix (Z is staged into it; args->Z is ignored);
 * Z_host / Q_host should be page-locked.  The workspace must hold
 * aqr_workspace_bytes(...) + aqr_pipe_workspace_bytes(...) bytes (the
 * pipeline's step vectors and catch-up partials follow the factorization's
 * workspace; nothing is allocated inside).  The column form copies Z in
 * whole, then runs aqr_gs_factor_d2h.  Returns after all copies completed. */
AQR_API aqr_status aqr_gs_factor_pinned(aqr_factor_args *args, const double *Z_host, int64_t ldzh,
                                        double *Q_host, int64_t ldqh, double *R_host, int64_t ldrh,
                                        int64_t chunk_cols, const uint32_t *ready, void *stream);

/* Extra workspace bytes of aqr_gs_factor_pinned beyond aqr_workspace_bytes:
 * every step vector (m x n) and two parity buffers of catch-up partials. */
AQR_API uint64_t aqr_pipe_workspace_bytes(int32_t family, int32_t variant, int32_t orientation, int64_t m,
                                          int64_t n);

/* Column chunks the host-input pipeline uses for n columns (chunk_cols as
 * passed to aqr_gs_factor_pinned; 0 = the library's schedule; w > 0 uniform
 * chunks of w columns; -w a ramp w/8, w/4, w/2, then chunks of w): writes the
 * chunk boundaries (first 0, last n; at most max_bounds entries) and returns
 * the number of chunks.  A caller staging Z for the `ready` counter fills
 * chunk c = columns [bounds[c], bounds[c + 1]) in order. */
AQR_API int64_t aqr_pipe_chunks(int64_t n, int64_t chunk_cols, int64_t *bounds, int64_t max_bounds);

/* Same, with HOST Z/Q/R (column-major, ld = m / m / n) and a host-side
 * operator description (dense A, or CSR with int64 indptr/indices as the
 * reference's CsrSpdOperator holds them, operators.py:100-101).  Owns all
 * device memory; H2D of inputs and D2H of Q/R happen inside the call. */
AQR_API aqr_status aqr_gs_factor_host(int32_t family, int32_t variant, int32_t orientation, int64_t m,
                              int64_t n, const double *Z_host, double *Q_host, double *R_host,
                              int32_t op_kind, const double *A_host, const int64_t *indptr_host,
                              const int64_t *indices_host, const double *data_host, int64_t nnz,
                              int64_t *fail_col, double *fail_val, int32_t *flagged_host,
                              int64_t *mv_count);

/* ---- operator kernels (SpdOperator realizations) ---------------------- */

/* Y = A X for k columns.  Each output entry accumulates strictly in the
 * reference order (dense: ascending column index, _kernels_impl.py:24-47;
 * CSR: stored order, :50-56) with separately rounded multiply and add, so
 * the results are bitwise equal to the reference's matvec / csr_matvec. */
AQR_API aqr_status aqr_op_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                        int64_t ldy, void *stream);

/* Y = A X as the HP type's block apply runs it (X = op.apply_block(Zw),
 * gram_schmidt.py:136): dense operators on the FP64 tensor cores (DMMA,
 * TMA-fed tiles; fused multiply-adds in k-blocks of 4, so the entries differ
 * from aqr_op_apply's at rounding level), CSR and callback operators exactly
 * as aqr_op_apply.  Replaces operators.py:58-66 (apply_block) on the HP path
 * only; aqr_op_apply stays the bitwise kernel-namespace product. */
AQR_API aqr_status aqr_block_apply(const aqr_op *op, int64_t k, const double *X, int64_t ldx, double *Y,
                                   int64_t ldy, void *stream);

/* ---- the reference kernel namespace (backend.kernels()) ---------------- */

/* out[0] = x . y  (deterministic tree reduction; device scalar out)       */
AQR_API aqr_status aqr_dot(int64_t m, const double *x, const double *y, double *out, void *stream);
/* z -= a * q with a read from device memory a_dev[0] (no FMA contraction) */
AQR_API aqr_status aqr_sub_scaled(int64_t m, double *z, const double *a_dev, const double *q,
                          void *stream);
/* out = x / r_dev[0] (IEEE division)                                      */
AQR_API aqr_status aqr_div_scalar(int64_t m, const double *x, const double *r_dev, double *out,
                          void *stream);
AQR_API aqr_status aqr_matvec(int64_t m, const double *A, int64_t lda, const double *x, double *y,
                      void *stream);
AQR_API aqr_status aqr_apply_block_dense(int64_t m, int64_t k, const double *A, int64_t lda,
                                 const double *X, int64_t ldx, double *Y, int64_t ldy,
                                 void *stream);
AQR_API aqr_status aqr_csr_matvec(int64_t m, const int32_t *indptr, const int32_t *indices,
                          const double *data, const double *x, double *y, void *stream);

/* Dense helpers of the reference's kernel namespace, same operation order
 * (_kernels_impl.py:59-82, 134-164), on caller-owned device buffers:
 *   aqr_gemm_tn        C (p x n) = A^T B, A m x p, B m x n; every entry a
 *                      sequential sum over ascending rows (gemm_tn; the
 *                      Gram products of cholesky_qr and of the metrics)
 *   aqr_gemm_nn        C (m x n) = A B, A m x kk; entry (i, j) accumulated
 *                      over ascending l (gemm_nn / linalg.matmul)
 *   aqr_cholesky_upper R = upper Cholesky factor of G (its upper triangle;
 *                      linalg.cholesky_upper passes (G + G^T) / 2), left
 *                      looking (cholesky_upper_kernel); *fail_dev (device
 *                      int32) = -1, or the first failing pivot
 *   aqr_tri_solve_right X with X R = Z (tri_solve_right_kernel); the caller
 *                      checks that diag(R) is nonzero and finite (linalg.py). */
AQR_API aqr_status aqr_gemm_tn(int64_t m, int64_t p, int64_t n, const double *A, int64_t lda, const double *B,
                               int64_t ldb, double *C, int64_t ldc, void *stream);
AQR_API aqr_status aqr_gemm_nn(int64_t m, int64_t kk, int64_t n, const double *A, int64_t lda, const double *B,
                               int64_t ldb, double *C, int64_t ldc, void *stream);
AQR_API aqr_status aqr_cholesky_upper(int64_t n, const double *G, int64_t ldg, double *R, int64_t ldr,
                                      int32_t *fail_dev, void *stream);
AQR_API aqr_status aqr_tri_solve_right(int64_t m, int64_t n, const double *Z, int64_t ldz, const double *R,
                                       int64_t ldr, double *X, int64_t ldx, void *stream);

/* ---- step kernels (one MGS step of the row-oriented fused schedule) ----
 * Used by the multi-GPU driver, which inserts its NCCL all-reduces between
 * *_partials and *_finish.  `ntiles` = aqr_num_tiles(m_local).
 * Rt is the n x n R factor stored ROW-major (Rt[i*n + j] = R[i, j]).      */

AQR_API int64_t aqr_tile_rows(int64_t m);
AQR_API int64_t aqr_num_tiles(int64_t m);

/* z_i -= r * q_{i-1} (and x_i -= r * p_{i-1} when x/pprev given) where
 * r = r_dev[0] (skipped when r_dev == NULL); then, if npart != NULL, the
 * per-CTA partials of (z.x, z.z, x.x) into npart (3 x the variant's norm
 * grid; HP when x is given, HA / naive otherwise). */
AQR_API aqr_status aqr_step_col_update_norm(int64_t m, double *z, const double *qprev, double *x,
                                    const double *pprev, const double *r_dev,
                                    const double *xnorm, double *npart, const int32_t *status,
                                    void *stream);
/* tot[0..2] = fixed-order sums of npart (for the all-reduce).  `variant`
 * (aqr_variant) selects the norm grid the partials were formed on: HP
 * (aqr_step_col_update_norm called with x) or HA / naive (called with xnorm). */
AQR_API aqr_status aqr_step_norm_reduce(int64_t m, int32_t variant, const double *npart, double *tot,
                                const int32_t *status, void *stream);
/* From tot: breakdown check (status), flag, R[i,i] = sqrt(t) into rii. */
AQR_API aqr_status aqr_step_norm_finish(int64_t i, const double *tot, double *rii, int32_t *status,
                                void *stream);
/* q = z / rii ; p = x / rii when x != NULL */
AQR_API aqr_status aqr_step_normalize(int64_t m, const double *z, const double *rii, double *q,
                              const double *x, double *p, const int32_t *status, void *stream);
/* The fused trailing pass of step i over columns [jbeg, jend) of W:
 *   (q_i, p_i written when qout / pout given)
 *   z_j -= r_{i-1,j} q_{i-1};  x_j -= r_{i-1,j} p_{i-1} (HP);
 *   partial[(j - jbeg) * ntiles + tile] = sum over the tile of p_i . z_j
 *   (p_i . z0_j for CGS). */
AQR_API aqr_status aqr_step_trailing(int64_t m, int64_t i, int64_t jbeg, int64_t jend, double *W,
                             int64_t ldw, double *X, int64_t ldx, const double *Z0,
                             int64_t ldz0, const double *qprev, const double *pprev,
                             const double *rprev, const double *psrc, const double *rii,
                             double *pout, const double *zsrc, double *qout, double *partial,
                             const int32_t *status, void *stream);
/* out[c] = fixed-order sum over tiles of partial[c * ntiles + tile], c < ncols */
AQR_API aqr_status aqr_step_rrow_reduce(int64_t m, int64_t ncols, const double *partial, double *out,
                                const int32_t *status, void *stream);
/* R (column-major, ldr) <- upper triangle of row-major Rt, zeros below */
AQR_API aqr_status aqr_step_finalize_r(int64_t n, const double *Rt, double *R, int64_t ldr,
                               void *stream);

/* status block layout used by the step API: int32 [0] fail column (-1),
 * [1] pad, then double fail value at byte 8, then int32 flags[n] at byte 16 */
AQR_API uint64_t aqr_status_bytes(int64_t n);
AQR_API aqr_status aqr_status_init(int32_t *status, int64_t n, void *stream);

/* ---- multi-GPU: exchanges fused into the step kernels over peer memory ---
 * One process per GPU; the rows of Z and of the CSR operator are
 * block-partitioned.  Each rank owns a working matrix W (m_loc x n, the Q
 * output) and an exchange buffer, both allocated with aqr_p2p_alloc and
 * mapped into every other rank with CUDA IPC (aqr_ipc_handle / aqr_ipc_open;
 * the Python group in paper_1703_10440_b200/p2p.py does the collective
 * handle exchange).  The halo of the local CSR block is read straight from
 * the owning rank's W; the two all-reduces of every step are stores into all
 * ranks' exchange buffers plus release/acquire flags, summed in rank order
 * (bitwise equal on every rank; with one rank bitwise the single-GPU
 * aqr_gs_factor).  Row orientation, HA or HP, MGS or CGS, CSR operators. */
#define AQR_MAX_RANKS 8
typedef struct aqr_p2p_group {
    int32_t nranks, rank;
    double *xbuf[AQR_MAX_RANKS];     /* exchange buffers (own pointer + peer mappings) */
    const double *W[AQR_MAX_RANKS];  /* working matrices of every rank (own = args->Q) */
    int64_t ldw[AQR_MAX_RANKS];
    /* local CSR column m_loc + h (the halo) is row halo_row[h] of rank halo_rank[h] */
    int64_t n_halo;
    const int32_t *halo_rank, *halo_row; /* device */
    uint64_t seq0; /* flag epoch: advance by n + 2 per factorization, same on all ranks */
    uint64_t timeout_ns; /* longest wait for one peer flag (0: 60 s), then AQR_ETIMEOUT */
} aqr_p2p_group;

/* Bytes of one rank's exchange buffer for n columns. */
AQR_API uint64_t aqr_p2p_exchange_bytes(int64_t n);
/* cudaMalloc'd, zeroed device memory that can be IPC-mapped. */
AQR_API aqr_status aqr_p2p_alloc(uint64_t bytes, void **out);
AQR_API aqr_status aqr_p2p_free(void *ptr);
/* 64-byte CUDA IPC handle of an aqr_p2p_alloc block; open / close a peer's. */
AQR_API aqr_status aqr_ipc_handle(const void *ptr, uint8_t out[64]);
AQR_API aqr_status aqr_ipc_open(const uint8_t handle[64], void **out);
AQR_API aqr_status aqr_ipc_close(void *ptr);
/* The row-partitioned factorization of this rank's rows.  args: m = local
 * rows, Q = group->W[rank] (ld = ldw[rank]), op = the local CSR block over
 * m_loc + n_halo extended columns; R (replicated) is written on every rank.
 * Collective: every rank calls it with the same n, method and seq0. */
AQR_API aqr_status aqr_p2p_gs_factor(aqr_factor_args *args, const aqr_p2p_group *group, void *stream);

/* Single-device emulation of an N-rank group (tests; one GPU standing in for
 * N): args[r] / groups[r] describe rank r (all W / exchange buffers on the
 * current device, plain pointers instead of IPC mappings).  The ranks'
 * launches are interleaved phase by phase on `stream` -- step i's norm
 * kernels of all ranks, then their trailing passes, then their R-row pushes
 * -- so every flag a kernel waits for was raised by a kernel that precedes
 * it in stream order: the same kernels, flags, halo reads and rank-ordered
 * sums as N processes, without kernels that wait on one another running
 * concurrently on one GPU.  Returns the first non-OK rank status. */
AQR_API aqr_status aqr_p2p_gs_factor_lockstep(int32_t nranks, aqr_factor_args *const *args,
                                              const aqr_p2p_group *const *groups, void *stream);

/* ---- instrumentation (bench.py) ------------------------------------------
 * aqr_launch_count: number of kernels this library has launched so far in
 * the process (monotonic; read before/after a timed region).
 * aqr_trailing_timer_enable(1) makes aqr_gs_factor record a CUDA event pair
 * around every fused trailing launch on the launching stream;
 * aqr_trailing_timer_read returns the number of timed launches, their summed
 * device time in ms and summed algorithmic bytes, then resets the timer
 * (it synchronizes the recorded events). */
AQR_API uint64_t aqr_launch_count(void);
AQR_API aqr_status aqr_trailing_timer_enable(int32_t enable);
AQR_API aqr_status aqr_trailing_timer_read(int64_t *launches, double *ms, double *bytes);
/* Same for any timed kernel slot (0 trailing, 1 fused SpMV step, 2 column
 * update + norm), without resetting; enabling the timer resets it. */
AQR_API aqr_status aqr_kernel_timer_read(int32_t slot, int64_t *launches, double *ms, double *bytes);
/* Per-launch device times (ms) and algorithmic bytes of a slot, in launch
 * order; returns the number of timed launches (-1 on a CUDA error). */
AQR_API int64_t aqr_kernel_timer_list(int32_t slot, double *ms_out, double *bytes_out, int64_t max);
/* Diagnostics: per-launch trace of the fused SpMV step and trailing kernels
 * (3 x uint64 per launch: first-CTA start before / after the dependency wait,
 * last-CTA end, %globaltimer ns) in libraries built with -DAQR_TRACE; returns
 * the number of launches recorded, or -1 in production builds. */
AQR_API int64_t aqr_trace_read(uint64_t *out, int64_t max_slots);

AQR_API const char *aqr_last_error(void);
AQR_API int32_t aqr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AQR_B200_H */
