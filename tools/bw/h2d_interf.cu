// Diagnostics: how a concurrent host->device transfer slows a latency-bound
// CSR SpMV (5-point Laplacian, 1024^2 rows) and a streaming read-modify-write
// pass, for different ways of moving the bytes:
//   ce_pinned   cudaMemcpyAsync from cudaHostAlloc memory (copy engine)
//   ce_huge     cudaMemcpyAsync from mmap'd memory with MADV_HUGEPAGE, cudaHostRegister'ed
//   ce_d2d      cudaMemcpyAsync device -> device (copy engine, no PCIe)
//   zc_kernel   a kernel on K CTAs reading the mapped pinned memory (SM loads over PCIe)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a h2d_interf.cu -o h2d_interf
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

__global__ void spmv(int m, const int *ip, const int *ix, const double *v, const double *x, double *y) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = ip[r]; k < ip[r + 1]; ++k) s = fma(v[k], x[ix[k]], s);
        y[r] = s;
    }
}

__global__ void rmw(double *z, const double *q, size_t n, double r) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        z[i] = __dsub_rn(z[i], __dmul_rn(r, q[i]));
}

// zero-copy H2D: K CTAs stream the mapped host buffer into device memory
__global__ void zc_copy(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t n2, int reps) {
    for (int k = 0; k < reps; ++k)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
            dst[i] = src[i];
}

int main() {
    const int g = 1024, m = g * g;
    std::vector<int> ip(m + 1), ix;
    std::vector<double> v;
    ix.reserve(5 * m);
    v.reserve(5 * m);
    for (int r = 0; r < m; ++r) {
        const int iy = r / g, jx = r % g;
        ip[r] = (int)ix.size();
        if (iy > 0) { ix.push_back(r - g); v.push_back(-1); }
        if (jx > 0) { ix.push_back(r - 1); v.push_back(-1); }
        ix.push_back(r); v.push_back(4.01);
        if (jx < g - 1) { ix.push_back(r + 1); v.push_back(-1); }
        if (iy < g - 1) { ix.push_back(r + g); v.push_back(-1); }
    }
    ip[m] = (int)ix.size();
    int *dip, *dix;
    double *dv, *dx, *dy, *dz, *dq;
    const size_t nz = 64ull * m;  // 64 columns, like config 2's Z (537 MB)
    CK(cudaMalloc(&dip, 4 * (m + 1)));
    CK(cudaMalloc(&dix, 4 * ix.size()));
    CK(cudaMalloc(&dv, 8 * v.size()));
    CK(cudaMalloc(&dx, 8 * m));
    CK(cudaMalloc(&dy, 8 * m));
    CK(cudaMalloc(&dz, 8 * nz / 2));
    CK(cudaMalloc(&dq, 8 * nz / 2));
    CK(cudaMemcpy(dip, ip.data(), 4 * (m + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dix, ix.data(), 4 * ix.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dv, v.data(), 8 * v.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dx, 0, 8 * m));
    CK(cudaMemset(dz, 0, 8 * nz / 2));
    CK(cudaMemset(dq, 0, 8 * nz / 2));

    const size_t cb = 256ull << 20;  // transfer buffer 256 MB
    double *hp, *hh, *dsrc, *ddst;
    CK(cudaHostAlloc(&hp, cb, cudaHostAllocMapped));
    std::memset(hp, 0, cb);
    hh = (double *)mmap(nullptr, cb, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(hh, cb, MADV_HUGEPAGE);
    std::memset(hh, 0, cb);
    CK(cudaHostRegister(hh, cb, cudaHostRegisterMapped));
    CK(cudaMalloc(&dsrc, cb));
    CK(cudaMalloc(&ddst, cb));
    CK(cudaMemset(dsrc, 0, cb));
    double *hp_dev = nullptr;
    CK(cudaHostGetDevicePointer((void **)&hp_dev, hp, 0));

    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t sc, sx;
    CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sx, cudaStreamNonBlocking));
    cudaEvent_t a, b, xa, xb;
    cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&xa); cudaEventCreate(&xb);

    auto measure = [&](const char *label, int mode, int zc_ctas) {
        // start the interfering transfer (long enough to cover the timed region)
        cudaEventRecord(xa, sx);
        for (int k = 0; k < (mode == 3 ? 100 : 8); ++k) {
            if (mode == 1) cudaMemcpyAsync(ddst, hp, cb, cudaMemcpyHostToDevice, sx);
            if (mode == 2) cudaMemcpyAsync(ddst, hh, cb, cudaMemcpyHostToDevice, sx);
            if (mode == 3) cudaMemcpyAsync(ddst, dsrc, cb, cudaMemcpyDeviceToDevice, sx);
            if (mode == 5) cudaMemcpyAsync(hp, dsrc, cb, cudaMemcpyDeviceToHost, sx);
        }
        if (mode == 4) zc_copy<<<zc_ctas, 512, 0, sx>>>((const double2 *)hp_dev, (double2 *)ddst, cb / 16, 8);
        cudaEventRecord(xb, sx);
        // timed: 100 SpMVs, then 20 streaming passes
        cudaEventRecord(a, sc);
        for (int k = 0; k < 100; ++k) spmv<<<sms * 3, 256, 0, sc>>>(m, dip, dix, dv, dx, dy);
        cudaEventRecord(b, sc);
        CK(cudaEventSynchronize(b));
        float ms_spmv = 0;
        cudaEventElapsedTime(&ms_spmv, a, b);
        cudaEventRecord(a, sc);
        for (int k = 0; k < 20; ++k) rmw<<<sms * 4, 256, 0, sc>>>(dz, dq, nz / 2, 0.5);
        cudaEventRecord(b, sc);
        CK(cudaEventSynchronize(b));
        float ms_rmw = 0;
        cudaEventElapsedTime(&ms_rmw, a, b);
        const bool busy = cudaEventQuery(xb) == cudaErrorNotReady;
        CK(cudaStreamSynchronize(sx));
        float ms_x = 0;
        cudaEventElapsedTime(&ms_x, xa, xb);
        const double gbs = mode ? (mode == 3 ? 100.0 : 8.0) * cb / (ms_x / 1e3) / 1e9 : 0.0;
        std::printf("%-12s spmv %7.1f us  rmw pass %7.1f us  transfer %6.1f GB/s  (still running after: %s)\n", label,
                    ms_spmv * 10.0, ms_rmw * 50.0, gbs, busy ? "yes" : "NO");
    };
    measure("warmup", 0, 0);
    measure("alone", 0, 0);
    measure("ce_pinned", 1, 0);
    measure("ce_huge", 2, 0);
    measure("ce_d2d", 3, 0);
    measure("ce_d2h", 5, 0);
    for (int k : {4, 8, 16, 32}) {
        char lab[32];
        std::snprintf(lab, sizeof lab, "zc_kernel%d", k);
        measure(lab, 4, k);
    }
    measure("alone", 0, 0);
    return 0;
}
