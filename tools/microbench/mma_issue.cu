// How fast can one warp ISSUE tcgen05.mma?  The two-Q-tile kernel's MMA
// warps run the issue code on lane 0 only (`if (lane == 0)`), so every
// descriptor lives in a per-thread register and goes through R2UR before the
// UTCHMMA; here the same 8-MMA P.V sequence (kind::f16, SS, M128 N128 K16)
// is issued (a) lane-0 style, (b) by the whole warp with the descriptors
// computed warp-uniformly and elect.sync around each MMA, and (c) the same
// with the 8 descriptors precomputed before the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2409_16997_b200/csrc -o mma_issue mma_issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ifa_b200::ptx;

__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
constexpr uint32_t kIdesc = (1u << 4) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr int TILES = 32;  // 8 MMAs each

__global__ void __launch_bounds__(640, 1) bench(long long* out, int variant, int busy, uint32_t rt_off) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint64_t cbar[8];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 8; ++i) mbar_init(&cbar[i], 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tbase);
    fence_proxy_async_shared();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tm = tbase;
    const uint32_t p_base = smem_u32(base), v_base = p_base + 32 * 1024;
    const uint32_t bb = smem_u32(&bar);
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (warp != 1 && (warp & 3) == 1 && busy) {  // math-like warps sharing the issuer's SMSP
        float a = lane * 1e-3f, b = 1.0001f, c = 0.5f;
        while (!done) {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                a = __fmaf_rn(a, b, c);
                if (busy == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
            }
        }
        if (a == 1234.5f) out[0] = 1;
    }
    if (warp == 1) {
        long long dt = 0;
        uint32_t ph = 0;
        for (int it = 0; it < 3; ++it) {
            const long long t0 = clock64();
            if (variant == 0) {
                if (lane == 0) {
                    for (int t = 0; t < TILES; ++t) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t ad = smem_desc(p_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                            const uint64_t bd = smem_desc(v_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                            mma_f16_ss(tm + 128, ad, bd, kIdesc, (t == 0 && kk == 0) ? 0u : 1u);
                        }
                    }
                    mma_commit_u32(bb);
                }
                __syncwarp();
            } else if (variant == 1) {
                for (int t = 0; t < TILES; ++t) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint64_t ad = smem_desc(p_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                        const uint64_t bd = smem_desc(v_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                        if (elect_one()) mma_f16_ss(tm + 128, ad, bd, kIdesc, (t == 0 && kk == 0) ? 0u : 1u);
                        __syncwarp();
                    }
                }
                if (elect_one()) mma_commit_u32(bb);
                __syncwarp();
            } else if (variant >= 4) {  // kernel mix per tile: 4 i8 S MMAs + 8 f16 P.V MMAs
                constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
                if (lane == 0) {
                    for (int t = 0; t < TILES; ++t) {
                        const uint32_t so = variant == 6 ? 0 : 256 * (t & 1);  // 5: alternate groups' TMEM
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t ad = smem_desc(p_base + kk * 32, 16, 1024, kLayoutSw128);
                            const uint64_t bd = smem_desc(v_base + kk * 32, 16, 1024, kLayoutSw128);
                            if (variant == 4 || variant == 5)
                                mma_i8_ss(tm + so, ad, bd, kIdescI8, kk ? 1u : 0u);
                            else  // 6: S as f16 (8 K=16 steps would be needed; rate only)
                                mma_f16_ss(tm + so, ad, bd, kIdesc, kk ? 1u : 0u);
                        }
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t ad = smem_desc(p_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                            const uint64_t bd = smem_desc(v_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                            mma_f16_ss(tm + so + 128, ad, bd, kIdesc, 1u);
                        }
                    }
                    mma_commit_u32(bb);
                }
                __syncwarp();
            } else if (variant == 7 || variant == 8) {  // the mix + the kernel's commits per tile
                constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
                if (lane == 0) {
                    for (int t = 0; t < TILES; ++t) {
                        const uint32_t so = 256 * (t & 1);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t ad = smem_desc(p_base + kk * 32, 16, 1024, kLayoutSw128);
                            const uint64_t bd = smem_desc(v_base + kk * 32, 16, 1024, kLayoutSw128);
                            mma_i8_ss(tm + so, ad, bd, kIdescI8, kk ? 1u : 0u);
                        }
                        mma_commit_u32(smem_u32(&cbar[0]));  // s_full
                        if (variant == 8) mma_commit_u32(smem_u32(&cbar[1]));  // k_empty
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t ad = smem_desc(p_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                            const uint64_t bd = smem_desc(v_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                            mma_f16_ss(tm + so + 128, ad, bd, kIdesc, 1u);
                        }
                        mma_commit_u32(smem_u32(&cbar[2]));  // p_empty
                        if (variant == 8) { mma_commit_u32(smem_u32(&cbar[3])); mma_commit_u32(smem_u32(&cbar[4])); }  // v_empty, ...
                    }
                    mma_commit_u32(bb);
                }
                __syncwarp();
            } else if (variant == 3) {  // the kernel's form: runtime slot offsets, lane 0
                if (lane == 0) {
                    for (int t = 0; t < TILES; ++t) {
                        const uint32_t pb = p_base + (t & 1) * rt_off, vb = v_base + (t & 1) * rt_off;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t ad = smem_desc(pb + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                            const uint64_t bd = smem_desc(vb + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                            mma_f16_ss(tm + 128, ad, bd, kIdesc, (t == 0 && kk == 0) ? 0u : 1u);
                        }
                    }
                    mma_commit_u32(bb);
                }
                __syncwarp();
            } else {
                uint64_t ad[8], bd[8];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    ad[kk] = smem_desc(p_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                    bd[kk] = smem_desc(v_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                }
                if (lane == 0) {
                    for (int t = 0; t < TILES; ++t) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_f16_ss(tm + 128, ad[kk], bd[kk], kIdesc, (t == 0 && kk == 0) ? 0u : 1u);
                    }
                    mma_commit_u32(bb);
                }
                __syncwarp();
            }
            bar_wait(bb, ph);
            ph ^= 1;
            if (it == 2) dt = clock64() - t0;
        }
        if (lane == 0) out[blockIdx.x] = dt;
        done = 1;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
    long long* d; cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const char* names[] = {"lane 0 issues, descriptors per MMA", "whole warp + elect.sync per MMA", "lane 0, descriptors precomputed", "lane 0, runtime slot offsets (kernel form)",
                           "mix: 4 i8 S + 8 f16 PV per tile, 1 group", "mix, two groups' TMEM alternating", "4 f16 + 8 f16 per tile (no kind switch)",
                           "mix + 2 commits per tile", "mix + 5 commits per tile (the kernel's)"};
    const char* bn[] = {"quiet SMSP", "+4 FFMA warps on the SMSP", "+4 FFMA+MUFU warps"};
    for (int busy = 0; busy < 2; ++busy)
        for (int v : {5, 7, 8}) {
            bench<<<148, 640, 80 * 1024>>>(d, v, busy, 0);
            cudaError_t e = cudaDeviceSynchronize();
            long long h; cudaMemcpy(&h, d + 1, 8, cudaMemcpyDeviceToHost);
            printf("%-44s %-26s: %.1f cyc per MMA (%s)\n", names[v], bn[busy], (double)h / (TILES * (v >= 4 ? 12 : 8)), cudaGetErrorString(e));
        }
}
