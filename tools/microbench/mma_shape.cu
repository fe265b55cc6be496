// tcgen05.mma cost per instruction vs N (cta_group::1, M = 128), one issuing
// thread, R MMAs into one accumulator back to back, commit, wait; one CTA per
// SM.  Question it answers: is the tensor core's cost in the two-Q-tile kernel
// per instruction (then a transposed P.V with N = 256 -- both Q tiles of the
// CTA in one MMA -- halves the P.V time) or per FLOP?
//   f16 : kind::f16 K16, A K-major SW128, B MN-major SW128 (the kernel's P.V)
//   f16T: kind::f16 K16, A MN-major SW128 (V^T), B K-major SW128 (P^T): the
//         transposed P.V form O^T = V^T P^T
//   i8  : kind::i8 K32, A and B K-major SW128 (the kernel's S)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2409_16997_b200/csrc -o mma_shape mma_shape.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ifa_b200::ptx;

__host__ __device__ constexpr uint32_t idesc_f16x(uint32_t m, uint32_t n, bool a_mn, bool b_mn) {
    return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_i8x(uint32_t m, uint32_t n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}

constexpr int REPS = 96;
// mode 0 f16, 1 f16T, 2 i8; chains = independent accumulators interleaved
template <int mode, int n, int chains>
__global__ void __launch_bounds__(128, 1) bench(long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x00010001u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tbase);
    fence_proxy_async_shared();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tm = tbase;
    const uint32_t a_base = smem_u32(base), b_base = a_base + 32 * 1024;
    long long dt = 0;
    if (warp == 1) {
        const uint32_t bb = smem_u32(&bar);
        uint32_t ph = 0;
        constexpr uint32_t i_f16 = idesc_f16x(128, n, false, true), i_f16t = idesc_f16x(128, n, true, false);
        constexpr uint32_t i_i8 = idesc_i8x(128, n);
        for (int it = 0; it < 3; ++it) {
            const long long t0 = clock64();
            // descriptors as base + compile-time offsets (uniform registers, no
            // per-MMA descriptor arithmetic on the issue path)
            const uint64_t a0 = smem_desc(a_base, 16, 1024, kLayoutSw128);
            const uint64_t b0 = smem_desc(b_base, 128 * 128, 1024, kLayoutSw128);
            const uint64_t a1 = smem_desc(a_base, 128 * 128, 1024, kLayoutSw128);
            const uint64_t b1 = smem_desc(b_base, 16, 1024, kLayoutSw128);
            if (elect_one()) {
                for (int r = 0; r < REPS / 8; ++r) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t d = tm + (chains == 2 ? (kk & 1) * n : 0);
                        if constexpr (mode == 0)
                            mma_f16(d, a0 + ((kk >> 2) * (128 * 128) + (kk & 3) * 32) / 16, b0 + (kk * 16 * 128) / 16, i_f16);
                        else if constexpr (mode == 1)
                            mma_f16(d, a1 + (kk * 16 * 128) / 16, b1 + ((kk >> 2) * (256 * 128) + (kk & 3) * 32) / 16, i_f16t);
                        else
                            mma_i8_ss(d, a0 + ((kk & 3) * 32) / 16, b1 + ((kk & 3) * 32) / 16, i_i8, 1u);
                    }
                }
                mma_commit_u32(bb);
            }
            __syncwarp();
            bar_wait(bb, ph);
            ph ^= 1;
            const long long t1 = clock64();
            if (it == 2) dt = t1 - t0;
        }
        if (lane == 0) out[blockIdx.x] = dt;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

template <int mode, int n, int chains>
void run1(long long* d, const char* name) {
    if constexpr (chains * n <= 512) {
        cudaFuncSetAttribute(bench<mode, n, chains>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
        cudaMemset(d, 0, 148 * 8);
        bench<mode, n, chains><<<148, 128, 170 * 1024>>>(d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double cyc = (double)h / REPS;
        printf("%-44s N%-3d chains %d: %6.1f cyc/MMA, %6.1f cyc per N128-equivalent (%s)\n", name, n, chains, cyc,
               cyc * 128.0 / n, cudaGetErrorString(e));
    }
}
template <int mode>
void run_mode(long long* d, const char* name) {
    run1<mode, 64, 1>(d, name); run1<mode, 64, 2>(d, name);
    run1<mode, 128, 1>(d, name); run1<mode, 128, 2>(d, name);
    run1<mode, 256, 1>(d, name); run1<mode, 256, 2>(d, name);
}
int main() {
    long long* d; cudaMalloc(&d, 148 * 8);
    run_mode<0>(d, "kind::f16 K16 A K-major, B MN-major (P.V)");
    run_mode<1>(d, "kind::f16 K16 A MN-major, B K-major (O^T)");
    run_mode<2>(d, "kind::i8  K32 A, B K-major (S)");
}
