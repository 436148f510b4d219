// TMEM ld/st throughput and latency probe (dev): is TMEM usable as a per-thread
// spill space for the z-queue, and does it share the LSU pipe with SHFL/LDS?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD16(a, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(a))
#define ST16(a, r) asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
    :: "r"(a), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]) : "memory")

// mode 0: ld only, 1: st only, 2: ld+st, 3: ld+st with SHFL traffic, 4: SHFL only, 5: correctness
__global__ void __launch_bounds__(256) probe(int mode, int iters, long long* cyc, unsigned* sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // lanes 32*(warp%4).., columns: warps 0-3 use [0,256), warps 4-7 [256,512)
    const uint32_t ta = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * (warp >> 2));
    uint32_t r[16], acc = 0;
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
    for (int c = 0; c < 256; c += 16) ST16(ta + c, r);
    asm volatile("tcgen05.wait::st.sync.aligned;");
    __syncthreads();
    long long t0 = clock64();
    if (mode == 5) {
        // each thread wrote its own pattern: read back from column 32
        for (int i = 0; i < 16; ++i) r[i] = 0x1000000u + threadIdx.x * 64 + i;
        ST16(ta + 32, r);
        asm volatile("tcgen05.wait::st.sync.aligned;");
        uint32_t q[16];
        LD16(ta + 32, q);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        unsigned bad = 0;
        for (int i = 0; i < 16; ++i) bad += q[i] != 0x1000000u + threadIdx.x * 64 + i;
        sink[blockIdx.x * 256 + threadIdx.x] = bad;
        goto done;
    }
    for (int it = 0; it < iters; ++it) {
        if (mode == 0 || mode == 2 || mode == 3) {
            uint32_t q[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                LD16(ta + ((it * 64 + c * 16) & 255), q);
                asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
                for (int i = 0; i < 16; ++i) acc += q[i];
            }
        }
        if (mode == 1 || mode == 2 || mode == 3) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                r[0] = acc + c;
                ST16(ta + ((it * 64 + c * 16 + 128) & 255), r);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;");
        }
        if (mode == 3 || mode == 4) {
#pragma unroll
            for (int c = 0; c < 64; ++c) acc += __shfl_up_sync(0xffffffffu, acc + c, 1);
        }
    }
done:
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (mode != 5) sink[blockIdx.x * 256 + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}

int main() {
    long long* cyc; unsigned* sink;
    cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 256 * 4);
    const int iters = 2000;
    const char* names[] = {"ld x16 (4/iter)", "st x16 (4/iter)", "ld+st", "ld+st+64 SHFL", "64 SHFL", "check"};
    for (int mode = 0; mode < 6; ++mode) {
        probe<<<148, 256>>>(mode, iters, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
        long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        if (mode == 5) {
            static unsigned hs[148 * 256]; cudaMemcpy(hs, sink, sizeof(hs), cudaMemcpyDeviceToHost);
            unsigned bad = 0; for (int i = 0; i < 148 * 256; ++i) bad += hs[i];
            printf("check: %u mismatches\n", bad);
            continue;
        }
        double c = (double)h[0] / iters;
        // bytes per iteration per SM: 4 x16 ops * 64 B/thread * 256 threads (each direction)
        double bytes = 4.0 * 64 * 256;
        printf("%-18s %8.1f cycles/iter", names[mode], c);
        if (mode <= 2) printf("  -> %.1f B/clk/SM per direction", bytes / c);
        if (mode == 4) printf("  -> %.2f SHFL/clk/SM", 64.0 * 8 / c);
        printf("\n");
    }
    return 0;
}
