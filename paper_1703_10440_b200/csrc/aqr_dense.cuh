// aqr_dense.cuh -- the reference's dense helper kernels in its own operation
// order (/root/reference/pkg/src/aqr/_kernels_impl.py:59-82, 134-164): the
// Gram product C = A^T B with every entry a sequential sum over ascending
// rows, the left-looking upper Cholesky factorization and the right
// triangular solve.  They carry the weighted Cholesky QR
// (gram_schmidt.py:209-218) and the accuracy metrics (metrics.py:35-53) on
// the device; separately rounded multiply and add everywhere
// (__dmul_rn / __dadd_rn), true IEEE division and sqrt, so the results are
// bitwise the reference's for bitwise-equal inputs.
#pragma once

#include "aqr_kernels.cuh"

namespace aqr {

// ---- C = A^T B, C(i, j) = sum_{r ascending} A(r, i) B(r, j) (gemm_tn) -------
// CTA = 32 x 32 entries of C, 256 threads, 2 x 2 entries per thread (four
// independent sequential chains).  Rows stream through shared memory in
// blocks of kTnRows: column slices of A and B, loaded along r (coalesced).
// No split over rows -- that would reorder the sums -- so the parallelism
// is p n / 4 threads; fine for the n x n Gram products this serves.
constexpr int kTnTile = 32, kTnRows = 64;
__global__ void __launch_bounds__(kBlock)
    gemm_tn_seq_kernel(int64_t m, int64_t p, int64_t n, const double *__restrict__ A, int64_t lda,
                       const double *__restrict__ B, int64_t ldb, double *__restrict__ C, int64_t ldc) {
    __shared__ double As[kTnTile][kTnRows + 1];  // [column][row] (+1: no bank conflicts on the column walk)
    __shared__ double Bs[kTnTile][kTnRows + 1];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t i0 = (int64_t)blockIdx.x * kTnTile, j0 = (int64_t)blockIdx.y * kTnTile;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int64_t r0 = 0; r0 < m; r0 += kTnRows) {
        const int rows = (int)((m - r0) < kTnRows ? (m - r0) : kTnRows);
        // 32 columns x 64 rows per operand: thread -> (row tid & 63, columns (tid >> 6) + 4u)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int rr = tid & 63, cc = (tid >> 6) + 4 * u;
            const int64_t gi = i0 + cc, gj = j0 + cc;
            As[cc][rr] = (rr < rows && gi < p) ? __ldg(A + (r0 + rr) + gi * lda) : 0.0;
            Bs[cc][rr] = (rr < rows && gj < n) ? __ldg(B + (r0 + rr) + gj * ldb) : 0.0;
        }
        __syncthreads();
        for (int rr = 0; rr < rows; ++rr) {
            const double a0 = As[ty][rr], a1 = As[ty + 16][rr];
            const double b0 = Bs[tx][rr], b1 = Bs[tx + 16][rr];
            acc[0][0] = __dadd_rn(acc[0][0], __dmul_rn(a0, b0));
            acc[0][1] = __dadd_rn(acc[0][1], __dmul_rn(a0, b1));
            acc[1][0] = __dadd_rn(acc[1][0], __dmul_rn(a1, b0));
            acc[1][1] = __dadd_rn(acc[1][1], __dmul_rn(a1, b1));
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int64_t gi = i0 + ty + 16 * a, gj = j0 + tx + 16 * b;
            if (gi < p && gj < n) C[gi + gj * ldc] = acc[a][b];
        }
}

// ---- left-looking upper Cholesky (cholesky_upper_kernel) -------------------
// G's upper triangle as given (linalg.cholesky_upper passes (G + G^T) / 2).
// One CTA.  Row k of R: t = G(k,k) - sum_{i<k} R(i,k)^2 (ascending i),
// r_kk = sqrt(t) (fail at the first t that is not > 0 or not finite), then
// R(k,j) = (G(k,j) - sum_{i<k} R(i,k) R(i,j)) / r_kk for j > k, one thread
// per j.  R's strict lower part is set to 0.0.  *fail = -1 or the pivot.
__global__ void __launch_bounds__(kBlock)
    cholesky_upper_kernel(int64_t n, const double *__restrict__ G, int64_t ldg, double *R, int64_t ldr,
                          int32_t *fail) {
    __shared__ double rkk_sh;
    __shared__ int bad_sh;
    const int tid = threadIdx.x;
    for (int64_t e = tid; e < n * n; e += kBlock) {
        const int64_t i = e % n, j = e / n;
        if (i > j) R[i + j * ldr] = 0.0;
    }
    if (tid == 0) bad_sh = -1;
    __syncthreads();
    for (int64_t k = 0; k < n; ++k) {
        if (tid == 0) {
            double s = 0.0;
            for (int64_t i = 0; i < k; ++i) s = __dadd_rn(s, __dmul_rn(R[i + k * ldr], R[i + k * ldr]));
            const double t = __dsub_rn(G[k + k * ldg], s);
            if (!(t > 0.0) || !isfinite(t)) {
                bad_sh = (int)k;
            } else {
                rkk_sh = __dsqrt_rn(t);
                R[k + k * ldr] = rkk_sh;
            }
        }
        __syncthreads();
        if (bad_sh >= 0) break;
        const double rkk = rkk_sh;
        for (int64_t j = k + 1 + tid; j < n; j += kBlock) {
            double s = 0.0;
            for (int64_t i = 0; i < k; ++i) s = __dadd_rn(s, __dmul_rn(R[i + k * ldr], R[i + j * ldr]));
            R[k + j * ldr] = __ddiv_rn(__dsub_rn(G[k + j * ldg], s), rkk);
        }
        __syncthreads();
    }
    if (tid == 0) *fail = bad_sh;
}

// ---- X R = Z for upper triangular R (tri_solve_right_kernel) ---------------
// X(r,k) = (Z(r,k) - sum_{i<k} X(r,i) R(i,k)) / R(k,k), ascending i; one
// thread per row (rows are independent; the order inside a row is the
// reference's).  R's columns are read through the read-only cache.
__global__ void __launch_bounds__(kBlock)
    tri_solve_right_kernel(int64_t m, int64_t n, const double *__restrict__ Z, int64_t ldz,
                           const double *__restrict__ R, int64_t ldr, double *X, int64_t ldx) {
    for (int64_t r = (int64_t)blockIdx.x * kBlock + threadIdx.x; r < m; r += (int64_t)gridDim.x * kBlock) {
        for (int64_t k = 0; k < n; ++k) {
            double s = 0.0;
            for (int64_t i = 0; i < k; ++i) s = __dadd_rn(s, __dmul_rn(X[r + i * ldx], __ldg(R + i + k * ldr)));
            X[r + k * ldx] = __ddiv_rn(__dsub_rn(Z[r + k * ldz], s), __ldg(R + k + k * ldr));
        }
    }
}

}  // namespace aqr
