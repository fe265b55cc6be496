// Does a MUFU.EX2 warp-instruction cost the MUFU pipe less when most lanes
// are inactive?  Throughput of ex2 with a per-lane (divergent) predicate that
// enables 32 / 16 / 4 / 1 / 0 lanes of each warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_mask mufu_mask.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
#define IT 512
__global__ void k(float* out, long long* cyc, int active) {
    float f[CH];
    for (int c = 0; c < CH; ++c) f[c] = threadIdx.x * 1e-3f - c;
    const bool on = (threadIdx.x & 31) < active;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            float r = f[c];
            asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; @p ex2.approx.ftz.f32 %0, %0;}" : "+f"(r) : "r"((unsigned)on));
            f[c] = r;
        }
    }
    long long t1 = clock64();
    float a = 0; for (int c = 0; c < CH; ++c) a += f[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
    for (int act : {32, 16, 8, 4, 1, 0}) {
        k<<<148, 1024>>>(o, c, act); cudaDeviceSynchronize();
        k<<<148, 1024>>>(o, c, act); cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double wi = 32.0 * IT * CH;  // warp-instructions per SM
        printf("active lanes %2d: %.3f warp-instr/clk/SM\n", act, wi / h);
    }
}
