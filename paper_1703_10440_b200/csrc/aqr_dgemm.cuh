// aqr_dgemm.cuh -- fp64 block apply Y = A X on the FP64 tensor cores (DMMA)
// with TMA-fed shared-memory tiles: the HP type's one operator product
// X = op.apply_block(Zw) (gram_schmidt.py:136) for a dense operator
// (config 4: 32768^2 x 32768 x 256, 550 GFLOP -- the one compute-bound
// phase of the hot path).
//
// The reference's apply_block_dense (_kernels_impl.py:35-47) sums every
// entry sequentially over ascending columns of A; that order is kept by
// dense_gemm3_kernel for the kernel namespace and the Cholesky-QR Gram
// products.  This kernel accumulates with fused multiply-adds in k-blocks
// of 4 (mma.sync.m8n8k4.f64) -- a different rounding of the same sums, so
// the HP factors move at rounding level and are gated by the oracle
// tolerance (tests/test_gpu_dgemm.py, tests/parity.py).
//
// Tiles: CTA 128 (rows of A) x 64 (columns of X), K in steps of 16; eight
// consumer warps as 4 x 2, warp tile 32 x 32 = 4 x 4 DMMA tiles, 32 fp64
// accumulators per thread; a producer warp issues the TMA loads
// (cp.async.bulk.tensor.2d, 128-byte swizzle) into a 4-stage mbarrier ring.
//
// Bank conflicts.  A arrives column-major (16 rows per 128-byte line, one
// line per k); X column-major (16 k per line, one line per column).  With
// the 128-byte swizzle (16-byte chunk index XOR line % 8) a DMMA operand
// fragment -- 8 rows x 4 k, one double per lane -- reads conflict-free
// (two wavefronts) when its 8 rows are {0-3, 8-11} or {4-7, 12-15} of a
// 16-row group: the chunk sets {0,1,4,5} / {2,3,6,7} XOR any 4 consecutive
// line indices cover every chunk exactly twice.  The X fragment (4 k x 8
// columns) spans 8 consecutive lines and is conflict-free as is.
#pragma once

#include <cuda.h>

#include "aqr_kernels.cuh"

namespace aqr {

constexpr int kDgBM = 128, kDgBN = 64, kDgBK = 16, kDgStages = 4;
constexpr int kDgConsumers = 8;                          // 4 (m) x 2 (n) warps
constexpr int kDgThreads = (kDgConsumers + 1) * 32;      // + the TMA producer warp
constexpr uint32_t kDgABytes = kDgBM * kDgBK * 8;        // 16 KB: 8 boxes of 16 rows x 16 k
constexpr uint32_t kDgXBytes = kDgBN * kDgBK * 8;        // 8 KB: one box of 16 k x 64 columns
constexpr uint32_t kDgStageBytes = kDgABytes + kDgXBytes;
constexpr size_t kDgSmem = (size_t)kDgStages * kDgStageBytes + 1024 /* alignment */ + 2 * kDgStages * 8;

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// Byte offset of (line, byte-in-line) inside a 128B-swizzled TMA box (box
// base 1024-byte aligned): the 16-byte chunk index XOR line % 8.
__device__ __forceinline__ uint32_t swz128(uint32_t line, uint32_t byte) {
    return line * 128u + (byte ^ ((line & 7u) << 4));
}

__device__ __forceinline__ double lds64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

// A fragment row i (0..7) of fragment f (0, 1) in a 16-row group.
__device__ __forceinline__ int dg_frag_row(int i, int f) { return (i < 4 ? i : i + 4) + 4 * f; }

// Y (m x k, ld ldy) = A (m x K, column-major, via tmA: box {16 rows, 16 k})
//                   x X (K x k, column-major, via tmX: box {16 k, 64 columns}).
__global__ void __launch_bounds__(kDgThreads, 2)
    dense_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX, int64_t m,
                      int64_t K, int64_t k, double *__restrict__ Y, int64_t ldy) {
    extern __shared__ uint8_t dg_raw[];
    uint8_t *base = (uint8_t *)(((uintptr_t)dg_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(base + kDgStages * kDgStageBytes);
    uint64_t *empty = full + kDgStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // column blocks fastest: the CTAs sharing a row block of A run together
    // and read it from L2 after the first
    const int nblk_n = (int)((k + kDgBN - 1) / kDgBN);
    const int64_t m0 = (int64_t)(blockIdx.x / nblk_n) * kDgBM;
    const int n0 = (int)(blockIdx.x % nblk_n) * kDgBN;
    const int ksteps = (int)((K + kDgBK - 1) / kDgBK);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kDgStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kDgConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kDgConsumers) {  // producer
        if (lane == 0) {
            for (int t = 0; t < ksteps; ++t) {
                const int s = t % kDgStages;
                if (t >= kDgStages) mbar_wait(empty + s, (uint32_t)((t / kDgStages - 1) & 1));
                uint8_t *st = base + (size_t)s * kDgStageBytes;
                mbar_expect_tx(full + s, kDgStageBytes);
                const int k0 = t * kDgBK;
#pragma unroll
                for (int g = 0; g < kDgBM / 16; ++g)
                    tma_load_2d(st + g * (16 * kDgBK * 8), &tmA, (int)(m0 + 16 * g), k0, full + s);
                tma_load_2d(st + kDgABytes, &tmX, k0, n0, full + s);
            }
        }
        return;
    }

    // consumers: warp (wm, wn) owns rows m0 + 32 wm .. +32, columns n0 + 32 wn .. +32
    const int wm = warp & 3, wn = warp >> 2;
    const int fi = lane >> 2, fk = lane & 3;  // fragment row / k of this lane
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    for (int t = 0; t < ksteps; ++t) {
        const int s = t % kDgStages;
        mbar_wait(full + s, (uint32_t)((t / kDgStages) & 1));
        const uint32_t sa = smem_u32(base) + (uint32_t)s * kDgStageBytes;
        const uint32_t sx = sa + kDgABytes;
#pragma unroll
        for (int kq = 0; kq < kDgBK / 4; ++kq) {
            const uint32_t kk = (uint32_t)(4 * kq + fk);
            double af[4], xf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {  // row tile a: 16-row group 2 wm + (a >> 1), fragment a & 1
                const int g = 2 * wm + (a >> 1);
                const uint32_t row = (uint32_t)dg_frag_row(fi, a & 1);
                af[a] = lds64(sa + (uint32_t)g * (16 * kDgBK * 8) + swz128(kk, row * 8u));
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {  // column tile b: columns 32 wn + 8 b + fi
                const uint32_t col = (uint32_t)(32 * wn + 8 * b + fi);
                xf[b] = lds64(sx + swz128(col, kk * 8u));
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b], af[a], xf[b]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }

    // epilogue: lane holds rows (fragment row fi) x columns 2 (lane & 3) + {0, 1}
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int64_t r = m0 + 32 * wm + 16 * (a >> 1) + dg_frag_row(fi, a & 1);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t c = n0 + 32 * wn + 8 * b + 2 * (lane & 3);
            if (r < m) {
                if (c < k) Y[c * ldy + r] = acc[a][b][0];
                if (c + 1 < k) Y[(c + 1) * ldy + r] = acc[a][b][1];
            }
        }
    }
}

}  // namespace aqr
