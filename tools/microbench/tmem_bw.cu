// TMEM read/write bandwidth per SM: W warps (multiple of 4) repeatedly
// tcgen05.ld / tcgen05.st 32x32b.x32 (or 16x256b.x4) over 128 lanes x 128
// columns, timed with clock64 inside one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>  // 0 = ld 32x32b.x32, 1 = st 32x32b.x32, 2 = ld 16x256b.x4 (x2)
__global__ void tmem_bw(int iters, unsigned long long* cycles, uint32_t* sink) {
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
    const uint32_t nw = blockDim.x / 32;
    // warp w: lane quarter w%4, column block (w/4) of the 128-column window
    const uint32_t quarter = warp & 3, cb = warp >> 2, ncb = nw / 4;
    const uint32_t cols = 128 / ncb;
    const uint32_t t = base + ((quarter * 32) << 16) + cb * cols;
    uint32_t acc = 0;
    uint32_t r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = threadIdx.x + j;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (uint32_t c = 0; c < cols; c += 32) {
            if (MODE == 0) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
                    "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31},"
                    " [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                      "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                      "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
                      "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]),
                      "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(t + c));
                asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
                for (int j = 0; j < 32; ++j) acc += r[j];
            } else {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"
                    "%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,"
                    "%30,%31,%32};" ::"r"(t + c),
                    "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                    "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
                    "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
                    "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                    "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]),
                    "r"(r[31])
                    : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;");
            }
        }
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

template <int MODE>
void run(int warps) {
    const int iters = 2000, ctas = 148;
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, sizeof(unsigned long long) * ctas);
    cudaMalloc(&sink, 4);
    tmem_bw<MODE><<<ctas, 32 * warps>>>(10, cyc, sink);
    tmem_bw<MODE><<<ctas, 32 * warps>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return;
    }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < ctas; ++i) avg += h[i];
    avg /= ctas;
    const double bytes = double(iters) * 128 * 128 * 4;  // per CTA per pass: 64 KiB
    printf("%s warps=%2d: %.1f B/clk/SM (%.0f clk per 64 KiB)\n", MODE == 0 ? "ld" : "st", warps,
           bytes / avg, avg / iters);
    cudaFree(cyc);
    cudaFree(sink);
}

int main() {
    for (int w : {4, 8, 16}) run<0>(w);
    for (int w : {4, 8, 16}) run<1>(w);
    return 0;
}
