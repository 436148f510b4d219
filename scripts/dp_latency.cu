// Microbenchmark (dev tool): dependent-chain latency of DADD/DMUL/FFMA/SHFL.f64
// on one warp, and DADD issue throughput per SM with many warps.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dadd(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x, y = a * 1e-30;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __dadd_rn(x, y); x = __dadd_rn(x, y); x = __dadd_rn(x, y); x = __dadd_rn(x, y); }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_dmul(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x, y = 1.0000000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __dmul_rn(x, y); x = __dmul_rn(x, y); x = __dmul_rn(x, y); x = __dmul_rn(x, y); }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_shfl(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __shfl_up_sync(~0u, x, 1); x = __shfl_up_sync(~0u, x, 1); x = __shfl_up_sync(~0u, x, 1); x = __shfl_up_sync(~0u, x, 1); }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_lds(double* out, double a, int n, long long* cyc) {
    __shared__ double sm[64];
    sm[threadIdx.x] = threadIdx.x * 0.0;
    __syncwarp();
    int idx = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { idx = (int)sm[idx]; idx = (int)sm[idx]; idx = (int)sm[idx]; idx = (int)sm[idx]; }
    long long t1 = clock64();
    out[threadIdx.x] = idx;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 1024 * sizeof(double)); cudaMalloc(&cyc, sizeof(long long));
    const int n = 4096;
    const char* names[] = {"DADD", "DMUL", "SHFL.f64(2x SHFL)", "LDS.64->F2I chain"};
    for (int k = 0; k < 4; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            if (k == 0) chain_dadd<<<1, 32>>>(out, 1.0, n, cyc);
            if (k == 1) chain_dmul<<<1, 32>>>(out, 1.0, n, cyc);
            if (k == 2) chain_shfl<<<1, 32>>>(out, 1.0, n, cyc);
            if (k == 3) chain_lds<<<1, 32>>>(out, 1.0, n, cyc);
        }
        cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        printf("%-20s latency %.1f cycles\n", names[k], (double)h / (4.0 * n));
    }
    return 0;
}
