// Diagnostics: achievable HBM bandwidth on this B200 for read+write streams
// with 8 / 16 / 32 byte accesses per thread (the trailing pass is a
// read-modify-write stream).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a bw.cu -o bw
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int U>
__global__ void rmw(T *z, const T *q, size_t n, double r) {
    size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
    T v[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        size_t k = i + (size_t)u * blockDim.x;
        if (k < n) { v[u] = z[k]; w[u] = q[k]; }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        size_t k = i + (size_t)u * blockDim.x;
        if (k < n) {
            double *a = reinterpret_cast<double *>(&v[u]);
            const double *b = reinterpret_cast<const double *>(&w[u]);
            for (int e = 0; e < (int)(sizeof(T) / 8); ++e) a[e] = __dsub_rn(a[e], __dmul_rn(r, b[e]));
            z[k] = v[u];
        }
    }
}

template <typename T, int U>
float run(double *z, double *q, size_t nd, int reps) {
    size_t n = nd * 8 / sizeof(T);
    unsigned grid = (unsigned)((n + 256 * U - 1) / (256 * U));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    rmw<T, U><<<grid, 256>>>((T *)z, (const T *)q, n, 0.5);
    cudaEventRecord(a);
    for (int k = 0; k < reps; ++k) rmw<T, U><<<grid, 256>>>((T *)z, (const T *)q, n, 0.5);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const size_t nd = (size_t)1 << 27;  // 1 GiB per array (z read+write, q read: 3 GiB traffic)
    double *z, *q;
    cudaMalloc(&z, nd * 8);
    cudaMalloc(&q, nd * 8);
    cudaMemset(z, 0, nd * 8);
    cudaMemset(q, 0, nd * 8);
    const double bytes = 3.0 * nd * 8;
    float t;
    t = run<double, 8>(z, q, nd, 10); printf("double  x8 : %.1f GB/s\n", bytes / t / 1e6);
    t = run<double, 16>(z, q, nd, 10); printf("double  x16: %.1f GB/s\n", bytes / t / 1e6);
    t = run<double2, 4>(z, q, nd, 10); printf("double2 x4 : %.1f GB/s\n", bytes / t / 1e6);
    t = run<double2, 8>(z, q, nd, 10); printf("double2 x8 : %.1f GB/s\n", bytes / t / 1e6);
    t = run<double4, 4>(z, q, nd, 10); printf("double4 x4 : %.1f GB/s\n", bytes / t / 1e6);
    // copy only (2 streams): read z, write q
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaMemcpy(q, z, nd * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(a);
    for (int k = 0; k < 10; ++k) cudaMemcpy(q, z, nd * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b);
    printf("cudaMemcpy D2D: %.1f GB/s\n", 2.0 * nd * 8 / (t / 10) / 1e6);
    return 0;
}
