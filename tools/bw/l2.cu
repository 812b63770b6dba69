// Diagnostics: read-modify-write bandwidth of a W-MB working set swept
// repeatedly (L2-resident when it fits): nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2.cu -o l2
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rmw(double *z, const double *q, size_t n, double r) {
    size_t i = (size_t)blockIdx.x * blockDim.x * 8 + threadIdx.x;
    double v[8], w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { size_t k = i + (size_t)u * blockDim.x; if (k < n) { v[u] = z[k]; w[u] = q[k]; } }
#pragma unroll
    for (int u = 0; u < 8; ++u) { size_t k = i + (size_t)u * blockDim.x; if (k < n) z[k] = __dsub_rn(v[u], __dmul_rn(r, w[u])); }
}
int main() {
    for (size_t mb : {16, 32, 48, 64, 80, 96, 128, 256, 1024}) {
        size_t n = mb * 1024 * 1024 / 8 / 2;  // z and q each mb/2
        double *z, *q;
        cudaMalloc(&z, n * 8); cudaMalloc(&q, n * 8);
        cudaMemset(z, 0, n * 8); cudaMemset(q, 0, n * 8);
        unsigned grid = (unsigned)((n + 2047) / 2048);
        for (int k = 0; k < 3; ++k) rmw<<<grid, 256>>>(z, q, n, 0.5);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int k = 0; k < 50; ++k) rmw<<<grid, 256>>>(z, q, n, 0.5);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("working set %5zu MB: %.1f GB/s (%.2f us per sweep)\n", mb, 3.0 * n * 8 / (ms / 50) / 1e6, ms / 50 * 1e3);
        cudaFree(z); cudaFree(q);
    }
    return 0;
}
