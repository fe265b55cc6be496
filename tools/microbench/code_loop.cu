// Clocks per 128-key row of the attn_ws.cu code loop (phase B) with W warps
// per SM: t = u*sq + cr (FFMA2), 2^t (MUFU.EX2 x2), + 1.5*2^23 (FADD2), PRMT
// pack, integer row sum, st.shared.v4 every 4 words.  The floor is the MUFU
// rate: 128 ex2 per row at 16/clk/SM = 8 clk per warp-instruction per SMSP,
// i.e. 1024 clk per row with one warp per SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o code_loop code_loop.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmov.b64 rc, "
        "{%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tadd.rn.f32x2 rd, "
        "ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float ex2(float t) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
    return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

template <int MODE>  // 0: MUFU for every pair; 1: only the MUFUs; 2: no MUFU (FFMA2 stand-in)
__global__ void __launch_bounds__(256, 1) bench(int iters, unsigned long long* cycles, uint32_t* sink,
                                                float sq, float cr) {
    __shared__ __align__(16) uint32_t p[8][32][32];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    float u[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) u[i] = -0.01f * i - 0.0001f * lane;
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 3) {  // attn_ws.cu order: all 128 exp2 first, then pack (lag 8 pairs)
            float2 y[64];
#pragma unroll
            for (int k = 0; k < 64; ++k) {
                const float2 t = ffma2(make_float2(u[2 * k], u[2 * k + 1]), make_float2(sq, sq),
                                       make_float2(cr, cr));
                y[k] = make_float2(ex2(t.x), ex2(t.y));
            }
#pragma unroll
            for (int ch = 0; ch < 16; ++ch) {
                uint32_t wd[4];
                const int dep = 4 * ch + 3 + 8 < 63 ? 4 * ch + 3 + 8 : 63;
                const float mg = __fmaf_rn(0.0f, y[dep].y, 12582912.0f);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 c = fadd2(y[4 * ch + e], make_float2(mg, mg));
                    wd[e] = prmt(__float_as_uint(c.x), __float_as_uint(c.y), 0x5410u);
                }
                acc += wd[0] + wd[1];
                acc += wd[2] + wd[3];
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(static_cast<uint32_t>(
                                 __cvta_generic_to_shared(&p[warp][lane][4 * ((ch & 7) ^ (lane & 7))]))),
                             "r"(wd[0]), "r"(wd[1]), "r"(wd[2]), "r"(wd[3])
                             : "memory");
            }
            cr += 1e-7f;
            continue;
        }
#pragma unroll
        for (int ch = 0; ch < 16; ++ch) {
            uint32_t wd[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 4 * ch + e;
                const float2 t = ffma2(make_float2(u[2 * k], u[2 * k + 1]), make_float2(sq, sq),
                                       make_float2(cr, cr));
                float2 y;
                if (MODE == 2) y = ffma2(t, t, t);
                else y = make_float2(ex2(t.x), ex2(t.y));
                if (MODE == 1) {
                    wd[e] = __float_as_uint(y.x) ^ __float_as_uint(y.y);
                } else {
                    const float2 c = fadd2(y, make_float2(12582912.0f, 12582912.0f));
                    wd[e] = prmt(__float_as_uint(c.x), __float_as_uint(c.y), 0x5410u);
                }
            }
            acc += wd[0] + wd[1];
            acc += wd[2] + wd[3];
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(static_cast<uint32_t>(
                             __cvta_generic_to_shared(&p[warp][lane][4 * ((ch & 7) ^ (lane & 7))]))),
                         "r"(wd[0]), "r"(wd[1]), "r"(wd[2]), "r"(wd[3])
                         : "memory");
        }
        cr += 1e-7f;
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) cycles[blockIdx.x * 8 + warp] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE>
void run(int warps) {
    const int iters = 200, ctas = 148;
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, sizeof(unsigned long long) * ctas * 8);
    cudaMalloc(&sink, 4);
    bench<MODE><<<ctas, 32 * warps>>>(4, cyc, sink, 0.7f, 6.9f);
    bench<MODE><<<ctas, 32 * warps>>>(iters, cyc, sink, 0.7f, 6.9f);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("error\n");
        return;
    }
    unsigned long long h[148 * 8];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < ctas; ++i) avg += h[i * 8];
    printf("mode %d warps/SM %d: %.0f clk per row per warp\n", MODE, warps, avg / ctas / iters);
}

int main() {
    for (int w : {4, 8}) run<0>(w);
    for (int w : {4, 8}) run<1>(w);
    for (int w : {4, 8}) run<2>(w);
    for (int w : {4, 8}) run<3>(w);
    return 0;
}
