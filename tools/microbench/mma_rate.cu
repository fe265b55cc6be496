// tcgen05.mma issue-to-completion rate with the two-Q-tile kernel's operand
// forms, one CTA per SM, nothing else running:
//   S : kind::i8  M128 N128 K32, A and B K-major SW128 (4 per 128x128x128 tile)
//   PV: kind::f16 M128 N128 K16, A K-major SW128 (P), B MN-major SW128 (V)
//       (8 per tile), and the same with A from TMEM (TS form) for comparison
// Reports cycles per MMA instruction (R MMAs issued back to back, commit,
// wait), 1 or 2 issuing threads (two groups, as in the kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2409_16997_b200/csrc -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ifa_b200::ptx;

__host__ __device__ constexpr uint32_t idesc_f16(uint32_t m, uint32_t n, bool b_mn_major) {
    return (1u << 4) | ((b_mn_major ? 1u : 0u) << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

constexpr int REPS = 96;
__device__ volatile int g_stop;
__global__ void __launch_bounds__(384, 1) bench(long long* out, int mode, int issuers, int noise) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
    __shared__ int done;
    if (threadIdx.x == 0) done = 0;
    if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tbase);
    fence_proxy_async_shared();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tm = tbase;
    const uint32_t a_base = smem_u32(base), b_base = a_base + 32 * 1024;
    constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t kIdescF16 = idesc_f16(128, 128, true);
    long long dt = 0;
    if ((warp == 1 || (issuers == 2 && warp == 2)) && lane == 0) {
        const int g = warp - 1;
        const uint32_t d = tm + 256 * g + (mode == 2 ? 128 : 0);  // modes 0, 1, 2
        const uint32_t bb = smem_u32(&bar[g]);
        uint32_t ph = 0;
        for (int it = 0; it < 3; ++it) {
            const long long t0 = clock64();
            for (int r = 0; r < REPS; ++r) {
                if (mode == 0) {  // S: kind::i8, K-major SW128 both
                    const uint64_t ad = smem_desc(a_base + (r & 3) * 32, 16, 1024, kLayoutSw128);
                    const uint64_t bd = smem_desc(b_base + (r & 3) * 32, 16, 1024, kLayoutSw128);
                    mma_i8_ss(d, ad, bd, kIdescI8, 1u);
                } else if (mode == 1) {  // PV: kind::f16, A K-major SW128, B MN-major SW128
                    const int kk = r & 7;
                    const uint64_t ad = smem_desc(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                    const uint64_t bd = smem_desc(b_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                    mma_f16_ss(d, ad, bd, kIdescF16, 1u);
                } else if (mode == 3 || mode == 4) {  // the kernel's mix: per 12 MMAs 4 S (i8) + 8 PV (f16)
                    const int k12 = r % 12;
                    if (k12 < 4) {
                        const uint64_t ad = smem_desc(a_base + k12 * 32, 16, 1024, kLayoutSw128);
                        const uint64_t bd = smem_desc(b_base + k12 * 32, 16, 1024, kLayoutSw128);
                        mma_i8_ss(tm + 256 * g + (mode == 4 ? 0 : 0), ad, bd, kIdescI8, 1u);
                    } else {
                        const int kk = k12 - 4;
                        const uint64_t ad = smem_desc(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024, kLayoutSw128);
                        const uint64_t bd = smem_desc(b_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                        mma_f16_ss(tm + 256 * g + 128, ad, bd, kIdescF16, 1u);
                    }
                } else if (mode == 5) {  // 12 f16 MMAs, two accumulators (S as f16, K = 16 x 8)
                    const int k12 = r % 12;
                    const uint64_t ad = smem_desc(a_base + ((k12 & 7) >> 2) * (128 * 128) + (k12 & 3) * 32, 16, 1024, kLayoutSw128);
                    const uint64_t bd = smem_desc(b_base + (k12 & 7) * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                    mma_f16_ss(tm + 256 * g + (k12 < 4 ? 0 : 128), ad, bd, kIdescF16, 1u);
                } else {  // PV with A (P) from TMEM
                    const int kk = r & 7;
                    const uint64_t bd = smem_desc(b_base + kk * 16 * 128, 128 * 128, 1024, kLayoutSw128);
                    mma_f16_ts(d, tm + 256 * g + 8 * kk, bd, kIdescF16, 1u);
                }
            }
            mma_commit_u32(bb);
            bar_wait(bb, ph);
            ph ^= 1;
            const long long t1 = clock64();
            if (it == 2) dt = t1 - t0;
        }
        out[blockIdx.x * 2 + g] = dt;
        atomicAdd(&done, 1);
    } else if (warp >= 4 && noise) {
        // interference: noise 1 = st.shared.v4 stream (P stores), 2 = tcgen05.ld
        // 16x256b of TMEM columns 384.. (S / O loads), 3 = both
        const uint32_t region = a_base + 64 * 1024 + ((warp - 4) * 32 + lane) * 16;
        const uint32_t q = warp & 3;
        uint32_t acc = 0;
        while (*(volatile int*)&done < issuers) {
            if (noise & 1) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(region + (i & 1) * 4096), "r"(acc) : "memory");
            }
            if (noise & 2) {
                uint32_t r[16];
                asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                               "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                             : "r"(tm + 384 + ((q * 32) << 16)) : "memory");
                tmem_wait_ld();
                for (int i = 0; i < 16; ++i) acc += r[i];
            }
        }
        if (acc == 0x12345678u) out[0] = acc;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
    long long* d; cudaMalloc(&d, 148 * 2 * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const char* names[] = {"S  kind::i8  SS M128N128K32", "PV kind::f16 SS M128N128K16 (B MN-major)", "PV kind::f16 TS M128N128K16 (A in TMEM)",
                           "mix 4 i8 S + 8 f16 PV (2 accumulators)", "mix (same)", "12 f16 (2 accumulators)"};
    const char* nn[] = {"quiet", "+STS.128 stream", "+LDTM 16x256b stream", "+STS and LDTM"};
    for (int mode : {0, 1, 3, 5})
        for (int iss = 1; iss <= 2; ++iss)
            for (int noise = 0; noise < 1; ++noise) {
                cudaMemset(d, 0, 148 * 2 * 8);
                bench<<<148, 384, 100 * 1024>>>(d, mode, iss, noise);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                printf("%-44s issuers %d %-22s: %.1f cyc/MMA (%s)\n", names[mode], iss, nn[noise], (double)h[0] / REPS, cudaGetErrorString(e));
            }
}
