// TMEM -> register latency / bandwidth of the softmax's S load in
// attn_ws.cu: each warp reads its 32 lanes x 128 columns (16 KiB) as
// 4 x tcgen05.ld.32x32b.x32 with ONE wait (mode 0), with a wait after each
// load (mode 1), or as 2 x .x64 (mode 2).  4 warps = one softmax group,
// 8 warps = both groups at once (columns 0-127 and 256-383).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld128 tmem_ld128.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

#define LD32(r, o, addr)                                                                         \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11," \
                 "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,"  \
                 "%31}, [%32];"                                                                  \
                 : "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]),               \
                   "=r"(r[o + 4]), "=r"(r[o + 5]), "=r"(r[o + 6]), "=r"(r[o + 7]),               \
                   "=r"(r[o + 8]), "=r"(r[o + 9]), "=r"(r[o + 10]), "=r"(r[o + 11]),             \
                   "=r"(r[o + 12]), "=r"(r[o + 13]), "=r"(r[o + 14]), "=r"(r[o + 15]),           \
                   "=r"(r[o + 16]), "=r"(r[o + 17]), "=r"(r[o + 18]), "=r"(r[o + 19]),           \
                   "=r"(r[o + 20]), "=r"(r[o + 21]), "=r"(r[o + 22]), "=r"(r[o + 23]),           \
                   "=r"(r[o + 24]), "=r"(r[o + 25]), "=r"(r[o + 26]), "=r"(r[o + 27]),           \
                   "=r"(r[o + 28]), "=r"(r[o + 29]), "=r"(r[o + 30]), "=r"(r[o + 31])            \
                 : "r"(addr))

template <int MODE>
__global__ void __launch_bounds__(256, 1) bench(int iters, unsigned long long* cycles, uint32_t* sink) {
    __shared__ uint32_t base;
    const uint32_t warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = base + (((warp & 3) * 32) << 16) + 256 * (warp >> 2);
    uint32_t acc = 0;
    uint32_t r[128];
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            LD32(r, 0, t);
            LD32(r, 32, t + 32);
            LD32(r, 64, t + 64);
            LD32(r, 96, t + 96);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                LD32(r, 32 * c, t + 32 * c);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
        }
#pragma unroll
        for (int j = 0; j < 128; ++j) acc += r[j];
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x % 32 == 0) cycles[blockIdx.x * 8 + warp] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

template <int MODE>
void run(int warps) {
    const int iters = 1000, ctas = 148;
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, sizeof(unsigned long long) * ctas * 8);
    cudaMalloc(&sink, 4);
    bench<MODE><<<ctas, 32 * warps>>>(10, cyc, sink);
    bench<MODE><<<ctas, 32 * warps>>>(iters, cyc, sink);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("error\n");
        return;
    }
    unsigned long long h[148 * 8];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < ctas; ++i) avg += h[i * 8];
    avg /= ctas;
    printf("mode %d warps %d: %.0f clk per 16 KiB row-block load per warp (+128 IADD), %.1f B/clk/SM\n",
           MODE, warps, avg / iters, warps * 16384.0 * iters / avg);
}

int main() {
    for (int w : {4, 8}) run<0>(w);
    for (int w : {4, 8}) run<1>(w);
    return 0;
}
