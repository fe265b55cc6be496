// Read bandwidth that P SMs alone can pull from HBM (the streamed quantizer
// runs on a few SMs next to the attention kernel):
//   mode 0: LDG.128, 1024 threads, U float4 in flight per thread
//   mode 1: cp.async.bulk (TMA bulk copy) into a STAGES x CHUNK shared-memory
//           ring, one thread issuing, every thread consuming (sums)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_bw sm_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(1024, 1) ldg_kernel(const float4* __restrict__ x, int64_t n4,
                                                      float* out) {
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

constexpr int CHUNK = 32768, STAGES = 6;
__global__ void __launch_bounds__(1024, 1) tma_kernel(const char* __restrict__ x, int64_t bytes,
                                                      float* out) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const int64_t nchunks = bytes / CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    float acc = 0.f;
    int64_t my = 0;
    auto issue = [&](int64_t c, int s) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(smem + s * CHUNK)), "l"(x + c * CHUNK), "r"(CHUNK), "r"(bar) : "memory");
    };
    // chunks blockIdx.x, blockIdx.x + gridDim.x, ...
    int64_t first = blockIdx.x;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s)
            if (first + (int64_t)s * gridDim.x < nchunks) issue(first + (int64_t)s * gridDim.x, s);
    for (int64_t c = first, k = 0; c < nchunks; c += gridDim.x, ++k) {
        const int s = (int)(k % STAGES);
        const uint32_t ph = (uint32_t)((k / STAGES) & 1);
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[s]);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0,1,0,P;}" : "=r"(ok) : "r"(bar), "r"(ph));
        const float4* v = reinterpret_cast<const float4*>(smem + s * CHUNK);
        for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) { float4 a = v[i]; acc += a.x + a.y + a.z + a.w; }
        __syncthreads();
        const int64_t nc = c + (int64_t)STAGES * gridDim.x;
        if (threadIdx.x == 0 && nc < nchunks) issue(nc, s);
        ++my;
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const int64_t bytes = (int64_t)2 << 30;  // 2 GiB
    char* x; float* out;
    cudaMalloc(&x, bytes); cudaMalloc(&out, 4);
    cudaMemset(x, 0, bytes);
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CHUNK * STAGES);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int P : {4, 8, 12, 16, 24, 148}) {
        auto t = [&](auto launch) {
            launch(); cudaDeviceSynchronize();
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); return bytes / (ms * 1e-3) / 1e9;
        };
        double g4 = t([&] { ldg_kernel<4><<<P, 1024>>>((const float4*)x, bytes / 16, out); });
        double g8 = t([&] { ldg_kernel<8><<<P, 1024>>>((const float4*)x, bytes / 16, out); });
        double g16 = t([&] { ldg_kernel<16><<<P, 1024>>>((const float4*)x, bytes / 16, out); });
        double gt = t([&] { tma_kernel<<<P, 1024, CHUNK * STAGES>>>(x, bytes, out); });
        printf("P=%3d  LDG u4 %7.0f  u8 %7.0f  u16 %7.0f  TMA %7.0f GB/s   (per SM: %5.0f %5.0f %5.0f %5.0f)\n",
               P, g4, g8, g16, gt, g4 / P, g8 / P, g16 / P, gt / P);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
