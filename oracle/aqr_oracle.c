/*
 * aqr_oracle.c -- CPU restatement of the reference's A-orthogonal
 * Gram-Schmidt hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * as the timed CPU baseline.  The product path (paper_1703_10440_b200/)
 * never links, imports or calls it.
 *
 * Every routine follows the reference `aqr` package
 * (/root/reference/pkg/src/aqr/...) operation for operation, including the
 * sequential-accumulation contract of _kernels_impl.py:1-12: every reduction
 * runs strictly left to right, products and sums are separately rounded (the
 * library is compiled with -ffp-contract=off, see Makefile), divisions are
 * true IEEE divisions and sqrt is the correctly rounded libm sqrt.  With that
 * the oracle is bitwise identical to the reference (pinned by
 * tests/test_oracle_golden.py against fixtures produced by the reference
 * itself, tests/golden/make_golden.py).
 *
 * Layout: every matrix is column-major (Fortran) with leading dimension equal
 * to its row count, as aqr.operators.as_matrix produces (operators.py:28-33).
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define UNIT_ROUNDOFF (1.0 / 9007199254740992.0) /* 2**-53, gram_schmidt.py:33 */

/* ---- L0 kernels: _kernels_impl.py ---------------------------------- */

/* Tolerance calibration only: mode 1 swaps the
 * sequential dot for a pairwise one, the perturbation a GPU tree reduction
 * introduces.  Mode 0 (default) is the reference. */
static _Thread_local int g_dot_mode = 0; /* per thread: concurrent calibration runs */
void aqro_set_dot_mode(int mode) { g_dot_mode = mode; }

static double pairwise_dot(int64_t m, const double *x, const double *y) {
    if (m <= 8) {
        double s = 0.0;
        for (int64_t k = 0; k < m; ++k) s += x[k] * y[k];
        return s;
    }
    const int64_t h = m / 2;
    return pairwise_dot(h, x, y) + pairwise_dot(m - h, x + h, y + h);
}

/* _kernels_impl.py:17-21 */
double aqro_seq_dot(int64_t m, const double *x, const double *y) {
    if (g_dot_mode == 1) return pairwise_dot(m, x, y);
    double s = 0.0;
    for (int64_t k = 0; k < m; ++k) s += x[k] * y[k];
    return s;
}

/* _kernels_impl.py:85-88 : z -= a * q */
void aqro_sub_scaled(int64_t m, double *z, double a, const double *q) {
    for (int64_t i = 0; i < m; ++i) z[i] -= a * q[i];
}

/* _kernels_impl.py:91-93 */
void aqro_div_scalar(int64_t m, const double *x, double r, double *out) {
    for (int64_t i = 0; i < m; ++i) out[i] = x[i] / r;
}

/* _kernels_impl.py:24-32 : y = A x, column-axpy order */
void aqro_matvec(int64_t m, int64_t ncol, const double *A, const double *x, double *y) {
    for (int64_t i = 0; i < m; ++i) y[i] = 0.0;
    for (int64_t j = 0; j < ncol; ++j) {
        const double xj = x[j];
        const double *a = A + j * m;
        for (int64_t i = 0; i < m; ++i) y[i] += a[i] * xj;
    }
}

/* _kernels_impl.py:35-47 : column c of Y accumulates exactly like matvec */
void aqro_apply_block_dense(int64_t m, int64_t k, const double *A, const double *X, double *Y) {
    for (int64_t c = 0; c < k; ++c) aqro_matvec(m, m, A, X + c * m, Y + c * m);
}

/* _kernels_impl.py:50-56 (int64 indptr/indices, operators.py:100-101) */
void aqro_csr_matvec(int64_t m, const int64_t *indptr, const int64_t *indices,
                     const double *data, const double *x, double *y) {
    for (int64_t i = 0; i < m; ++i) {
        double s = 0.0;
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) s += data[k] * x[indices[k]];
        y[i] = s;
    }
}

/* _kernels_impl.py:59-69 : C = A @ B, entry (i,j) accumulated over ascending l */
void aqro_gemm_nn(int64_t m, int64_t kk, int64_t n, const double *A, const double *B, double *C) {
    for (int64_t j = 0; j < n; ++j) {
        double *c = C + j * m;
        for (int64_t i = 0; i < m; ++i) c[i] = 0.0;
        for (int64_t l = 0; l < kk; ++l) {
            const double blj = B[l + j * kk];
            const double *a = A + l * m;
            for (int64_t i = 0; i < m; ++i) c[i] += a[i] * blj;
        }
    }
}

/* _kernels_impl.py:72-82 : C = A.T @ B, entry (i,j) accumulated over ascending rows */
void aqro_gemm_tn(int64_t m, int64_t p, int64_t n, const double *A, const double *B, double *C) {
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < p; ++i) C[i + j * p] = aqro_seq_dot(m, A + i * m, B + j * m);
}

/* ---- L1 operator: operators.py:43-129 ------------------------------- */

enum { AQRO_DENSE = 0, AQRO_CSR = 1 };

typedef struct {
    int kind;              /* AQRO_DENSE | AQRO_CSR */
    int64_t m;
    const double *A;       /* dense, m x m column-major */
    const int64_t *indptr; /* CSR */
    const int64_t *indices;
    const double *data;
} aqro_op;

/* SpdOperator.apply -> _apply_into (operators.py:50-56, 86-87, 121-122) */
static void op_apply(const aqro_op *op, const double *x, double *y) {
    if (op->kind == AQRO_DENSE) aqro_matvec(op->m, op->m, op->A, x, y);
    else aqro_csr_matvec(op->m, op->indptr, op->indices, op->data, x, y);
}

/* SpdOperator.apply_block (operators.py:58-70, 89-90): dense goes through
 * apply_block_dense, CSR through the base-class column loop.  Both are
 * bitwise equal to k single applies. */
static void op_apply_block(const aqro_op *op, int64_t k, const double *X, double *Y) {
    if (op->kind == AQRO_DENSE) aqro_apply_block_dense(op->m, k, op->A, X, Y);
    else
        for (int64_t c = 0; c < k; ++c) op_apply(op, X + c * op->m, Y + c * op->m);
}

/* ---- L2 driver: gram_schmidt.py:126-179 ----------------------------- */

enum { AQRO_MGS = 0, AQRO_CGS = 1 };
enum { AQRO_NAIVE = 0, AQRO_HA = 1, AQRO_HP = 2 };
enum { AQRO_COL = 0, AQRO_ROW = 1 };

/* Phase timers of the calling thread's last aqro_gs_factor (seconds):
 * [0] the block apply (HP, gram_schmidt.py:136), [1] all normalize(j) calls
 * (including their operator applies), [2] all project(i, j) calls.  Used
 * only by bench.py to extrapolate a column-truncated CPU run to the full
 * column count (each phase scales with its own call count). */
static _Thread_local double g_phase[3];
void aqro_last_phase_times(double *out) { memcpy(out, g_phase, sizeof g_phase); }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct {
    int family, variant;
    int64_t m, n;
    double *Zw, *Z0, *Q, *R, *P, *X, *xbuf;
    const aqro_op *op;
    int32_t *flagged; /* per column 0/1 */
    int64_t mv;
    int64_t fail_col;
    double fail_val;
} gs_state;

/* project(i, j): gram_schmidt.py:139-145 */
static void project(gs_state *s, int64_t i, int64_t j) {
    const int64_t m = s->m;
    const double *src = (s->family == AQRO_CGS ? s->Z0 : s->Zw) + j * m;
    const double r = aqro_seq_dot(m, s->P + i * m, src);
    s->R[i + j * s->n] = r;
    aqro_sub_scaled(m, s->Zw + j * m, r, s->Q + i * m);
    if (s->variant == AQRO_HP) aqro_sub_scaled(m, s->X + j * m, r, s->P + i * m);
}

/* normalize(j): gram_schmidt.py:147-165.  Returns 0, or 1 on breakdown. */
static int normalize(gs_state *s, int64_t j) {
    const int64_t m = s->m;
    double *z = s->Zw + j * m;
    const double *x;
    if (s->variant == AQRO_HP) {
        x = s->X + j * m;
    } else {
        op_apply(s->op, z, s->xbuf); /* op.apply(Zw[:, j].copy()) */
        s->mv += 1;
        x = s->xbuf;
    }
    const double t = aqro_seq_dot(m, z, x);
    if (!(t > 0.0) || !isfinite(t)) {
        s->fail_col = j;
        s->fail_val = t;
        return 1;
    }
    const double nz = sqrt(aqro_seq_dot(m, z, z));
    const double nx = sqrt(aqro_seq_dot(m, x, x));
    if (t < 100.0 * UNIT_ROUNDOFF * nz * nx) s->flagged[j] = 1;
    const double rjj = sqrt(t);
    s->R[j + j * s->n] = rjj;
    aqro_div_scalar(m, z, rjj, s->Q + j * m);
    if (s->variant == AQRO_NAIVE) {
        op_apply(s->op, s->Q + j * m, s->P + j * m); /* op.apply(Q[:, j].copy()) */
        s->mv += 1;
    } else {
        aqro_div_scalar(m, x, rjj, s->P + j * m);
    }
    return 0;
}

/*
 * Whole factorization, _gs_factor (gram_schmidt.py:126-179).
 *   Z        m x n column-major input (never modified)
 *   Q        m x n output, R n x n output (zero-filled here, strict lower 0.0)
 *   flagged  n int32 (0/1) output
 *   mv_count number of operator applications (CostReport.mv_count)
 *   fail_val breakdown value t on breakdown
 * Returns -1 on success, the breakdown column on BreakdownError, -2 on a
 * DimensionError (m < n, n < 1), -3 on allocation failure.
 */
int64_t aqro_gs_factor(int family, int variant, int orientation, int64_t m, int64_t n,
                       const double *Z, int op_kind, const double *A, const int64_t *indptr,
                       const int64_t *indices, const double *data, double *Q, double *R,
                       int32_t *flagged, int64_t *mv_count, double *fail_val) {
    if (n < 1 || m < n) return -2; /* _check_inputs, gram_schmidt.py:116-123 */
    aqro_op op = {op_kind, m, A, indptr, indices, data};
    gs_state s;
    memset(&s, 0, sizeof s);
    s.family = family;
    s.variant = variant;
    s.m = m;
    s.n = n;
    s.op = &op;
    s.Q = Q;
    s.R = R;
    s.flagged = flagged;
    s.fail_col = -1;
    const size_t mn = (size_t)m * (size_t)n;
    s.Zw = (double *)malloc(mn * sizeof(double));
    s.P = (double *)calloc(mn, sizeof(double));
    s.xbuf = (double *)malloc((size_t)m * sizeof(double));
    if (family == AQRO_CGS) s.Z0 = (double *)malloc(mn * sizeof(double));
    if (variant == AQRO_HP) s.X = (double *)malloc(mn * sizeof(double));
    if (!s.Zw || !s.P || !s.xbuf || (family == AQRO_CGS && !s.Z0) || (variant == AQRO_HP && !s.X)) {
        free(s.Zw); free(s.P); free(s.xbuf); free(s.Z0); free(s.X);
        return -3;
    }
    memcpy(s.Zw, Z, mn * sizeof(double));
    if (s.Z0) memcpy(s.Z0, Z, mn * sizeof(double));
    memset(Q, 0, mn * sizeof(double));
    memset(R, 0, (size_t)n * (size_t)n * sizeof(double));
    memset(flagged, 0, (size_t)n * sizeof(int32_t));
    memset(g_phase, 0, sizeof g_phase);
    double t0 = now_s(), t1;
    if (variant == AQRO_HP) { /* X = op.apply_block(Zw), gram_schmidt.py:136 */
        op_apply_block(&op, n, s.Zw, s.X);
        s.mv += n;
    }
    g_phase[0] = now_s() - t0;
    int bad = 0;
    if (orientation == AQRO_COL) { /* gram_schmidt.py:167-171 */
        for (int64_t j = 0; j < n && !bad; ++j) {
            t0 = now_s();
            for (int64_t i = 0; i < j; ++i) project(&s, i, j);
            t1 = now_s();
            bad = normalize(&s, j);
            g_phase[2] += t1 - t0;
            g_phase[1] += now_s() - t1;
        }
    } else { /* gram_schmidt.py:172-176 */
        for (int64_t i = 0; i < n && !bad; ++i) {
            t0 = now_s();
            bad = normalize(&s, i);
            t1 = now_s();
            g_phase[1] += t1 - t0;
            if (bad) break;
            for (int64_t j = i + 1; j < n; ++j) project(&s, i, j);
            g_phase[2] += now_s() - t1;
        }
    }
    if (mv_count) *mv_count = s.mv;
    if (fail_val) *fail_val = s.fail_val;
    free(s.Zw); free(s.P); free(s.xbuf); free(s.Z0); free(s.X);
    return bad ? s.fail_col : -1;
}

/* ---- weighted Cholesky QR: gram_schmidt.py:209-218 ---------------- */

/* cholesky_upper_kernel (_kernels_impl.py:134-152): left-looking, G's upper
 * triangle as given, R zero-filled first.  Returns -1, or the failing pivot. */
int64_t aqro_cholesky_upper_kernel(int64_t n, const double *G, double *R) {
    memset(R, 0, (size_t)n * n * sizeof(double));
    for (int64_t k = 0; k < n; ++k) {
        double s = 0.0;
        for (int64_t i = 0; i < k; ++i) s += R[i + k * n] * R[i + k * n];
        const double t = G[k + k * n] - s;
        if (!(t > 0.0) || !isfinite(t)) return k;
        const double rkk = sqrt(t);
        R[k + k * n] = rkk;
        for (int64_t j = k + 1; j < n; ++j) {
            s = 0.0;
            for (int64_t i = 0; i < k; ++i) s += R[i + k * n] * R[i + j * n];
            R[k + j * n] = (G[k + j * n] - s) / rkk;
        }
    }
    return -1;
}

/* linalg.cholesky_upper (linalg.py:191-208): the kernel on (G + G^T) / 2 */
static int64_t cholesky_upper(int64_t n, const double *G, double *R) {
    double *Gs = (double *)malloc((size_t)n * n * sizeof(double));
    if (!Gs) return -3;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) Gs[i + j * n] = 0.5 * (G[i + j * n] + G[j + i * n]);
    const int64_t bad = aqro_cholesky_upper_kernel(n, Gs, R);
    free(Gs);
    return bad;
}

/* linalg.tri_solve_right -> tri_solve_right_kernel (_kernels_impl.py:155-164) */
void aqro_tri_solve_right_kernel(int64_t m, int64_t n, const double *Z, const double *R, double *X) {
    for (int64_t k = 0; k < n; ++k) {
        const double rkk = R[k + k * n];
        for (int64_t r = 0; r < m; ++r) {
            double s = 0.0;
            for (int64_t i = 0; i < k; ++i) s += X[r + i * m] * R[i + k * n];
            X[r + k * m] = (Z[r + k * m] - s) / rkk;
        }
    }
}

/* Returns -1 on success, the pivot (>= 0) on NotPositiveDefiniteError, -2 on
 * a DimensionError, -3 on allocation failure, -4 on SingularMatrixError. */
int64_t aqro_cholesky_qr(int64_t m, int64_t n, const double *Z, int op_kind, const double *A,
                         const int64_t *indptr, const int64_t *indices, const double *data, double *Q,
                         double *R, int64_t *mv_count) {
    if (n < 1 || m < n) return -2;
    aqro_op op = {op_kind, m, A, indptr, indices, data};
    double *X = (double *)malloc((size_t)m * n * sizeof(double));
    double *G = (double *)malloc((size_t)n * n * sizeof(double));
    if (!X || !G) {
        free(X); free(G);
        return -3;
    }
    op_apply_block(&op, n, Z, X); /* X = op.apply_block(Z) */
    if (mv_count) *mv_count = n;
    aqro_gemm_tn(m, n, n, Z, X, G); /* G = matmul_tn(Z, X) */
    int64_t bad = cholesky_upper(n, G, R);
    if (bad == -1) {
        for (int64_t k = 0; k < n; ++k)
            if (R[k + k * n] == 0.0 || !isfinite(R[k + k * n])) bad = -4;
        if (bad == -1) aqro_tri_solve_right_kernel(m, n, Z, R, Q);
    }
    free(X); free(G);
    return bad;
}

/* ---- generator helpers (tests only) ---------------------------------- */

/*
 * Householder QR of a column-major m x k matrix G (m >= k), returning the
 * thin Q (m x k) with column signs fixed so that diag(R) > 0, i.e. the
 * convention of linalg.haar_orthogonal (linalg.py:59-75).  Written here so
 * the config-1 generator is bitwise reproducible on any host, independent of
 * the LAPACK build numpy happens to link.  Returns 0, or 1 if diag(R) has an
 * exact zero (the caller redraws, as haar_orthogonal does).
 */
int aqro_householder_qr(int64_t m, int64_t k, const double *G, double *Qout) {
    double *Aw = (double *)malloc((size_t)m * k * sizeof(double));
    double *V = (double *)malloc((size_t)m * k * sizeof(double));
    double *beta = (double *)malloc((size_t)k * sizeof(double));
    double *rdiag = (double *)malloc((size_t)k * sizeof(double));
    memcpy(Aw, G, (size_t)m * k * sizeof(double));
    int singular = 0;
    for (int64_t c = 0; c < k; ++c) {
        double *a = Aw + c * m;
        double *v = V + c * m;
        double sigma = 0.0;
        for (int64_t i = c; i < m; ++i) sigma += a[i] * a[i];
        const double norm = sqrt(sigma);
        const double alpha = a[c] >= 0.0 ? -norm : norm; /* R[c,c] = alpha */
        for (int64_t i = 0; i < m; ++i) v[i] = 0.0;
        for (int64_t i = c; i < m; ++i) v[i] = a[i];
        v[c] -= alpha;
        double vv = 0.0;
        for (int64_t i = c; i < m; ++i) vv += v[i] * v[i];
        beta[c] = vv > 0.0 ? 2.0 / vv : 0.0;
        rdiag[c] = alpha;
        if (alpha == 0.0) singular = 1;
        /* apply H_c = I - beta v v^T to the remaining columns */
        for (int64_t j = c; j < k; ++j) {
            double *aj = Aw + j * m;
            double d = 0.0;
            for (int64_t i = c; i < m; ++i) d += v[i] * aj[i];
            d *= beta[c];
            for (int64_t i = c; i < m; ++i) aj[i] -= d * v[i];
        }
    }
    /* Q = H_0 H_1 ... H_{k-1} [I_k; 0], accumulated backwards */
    for (int64_t j = 0; j < k; ++j) {
        double *q = Qout + j * m;
        for (int64_t i = 0; i < m; ++i) q[i] = 0.0;
        q[j] = 1.0;
    }
    for (int64_t c = k - 1; c >= 0; --c) {
        const double *v = V + c * m;
        for (int64_t j = 0; j < k; ++j) {
            double *q = Qout + j * m;
            double d = 0.0;
            for (int64_t i = c; i < m; ++i) d += v[i] * q[i];
            d *= beta[c];
            for (int64_t i = c; i < m; ++i) q[i] -= d * v[i];
        }
    }
    /* sign fix: make diag(R) positive (flip Q columns where R[c,c] < 0) */
    for (int64_t c = 0; c < k; ++c)
        if (rdiag[c] < 0.0)
            for (int64_t i = 0; i < m; ++i) Qout[i + c * m] = -Qout[i + c * m];
    free(Aw); free(V); free(beta); free(rdiag);
    return singular;
}
