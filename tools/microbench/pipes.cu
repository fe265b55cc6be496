// Per-SM throughput of the instructions the softmax inner loop is built
// from (warp-instructions per clock per SM).  One CTA of 1024 threads per
// SM, 8 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 256

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { float2 d; asm volatile("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0,%1}, rd;}" : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y)); return d; }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { float2 d; asm volatile("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mov.b64 rc, {%6,%7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;}" : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y)); return d; }

template <int OP>
__global__ void bench(float* out, long long* cyc, int seed) {
    float f[CHAINS]; int iv[CHAINS]; float2 p[CHAINS];
    for (int c = 0; c < CHAINS; ++c) { f[c] = threadIdx.x * 0.001f + c; iv[c] = threadIdx.x + c * seed; p[c] = make_float2(f[c], f[c] + 1); }
    __syncthreads();
    long long t0 = clock64();
    #pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
        #pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (OP == 0) { float r; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(r) : "r"(iv[c])); iv[c] = __float_as_int(r) ^ c; }
            if (OP == 1) { p[c] = fadd2(p[c], make_float2(1.0f, 2.0f)); }
            if (OP == 2) { p[c] = ffma2(p[c], make_float2(1.0001f, 0.9999f), make_float2(1.0f, 2.0f)); }
            if (OP == 3) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c])); f[c] = r; }
            if (OP == 4) { asm volatile("prmt.b32 %0, %0, %1, 0x0040;" : "+r"(iv[c]) : "r"(iv[(c+1)%CHAINS])); }
            if (OP == 5) { asm volatile("dp4a.u32.u32 %0, %0, 16843009, %0;" : "+r"(iv[c])); }
            if (OP == 6) { asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(f[(c+1)%CHAINS]), "f"(f[(c+2)%CHAINS])); }
            if (OP == 7) { asm volatile("add.s32 %0, %0, 1262485504;" : "+r"(iv[c])); }
            if (OP == 8) { asm volatile("add.rn.f32 %0, %0, 0f3F800000;" : "+f"(f[c])); }
            if (OP == 9) { float r; asm volatile("cvt.rni.f32.f32 %0, %1;" : "=f"(r) : "f"(f[c])); f[c] = r + 0.5f; }
            if (OP == 11) { asm volatile("mad.lo.s32 %0, %0, 1, 1262485504;" : "+r"(iv[c])); }
            if (OP == 12) { float2 q = p[c]; asm volatile("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%0,%1};\n mov.b64 rb, {%2,%3};\n mul.rn.f32x2 rd, ra, rb;\n mov.b64 {%0,%1}, rd;}" : "+f"(q.x), "+f"(q.y) : "f"(1.0001f), "f"(0.9999f)); p[c] = q; }
            if (OP == 13) { float r; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(r) : "r"(iv[c])); float r2; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(f[c])); f[c] = r2; iv[c] = __float_as_int(r) ^ c; }
            if (OP == 14) { unsigned r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[c]), "f"(f[(c+1)%CHAINS])); iv[c] ^= r; f[c] += 1.0f; }
            if (OP == 15) { unsigned h = 0x3c003c00u ^ (iv[c] & 0x00ff00ff); unsigned r; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h)); iv[c] = r; }
            if (OP == 10) { asm volatile("setp.gt.f32 %%p1, %0, 0f3EFFF000; selp.b32 %1, 1, %1, %%p1;" : "+f"(f[c]), "+r"(iv[c])); }
        }
        }
    }
    long long t1 = clock64();
    float acc = 0; for (int c = 0; c < CHAINS; ++c) acc += f[c] + p[c].x + p[c].y + iv[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; long long* cyc; cudaMalloc(&out, sms * 1024 * 4); cudaMalloc(&cyc, sms * 8);
    const char* names[] = {"I2F(cvt.rn.f32.s32)", "FADD2", "FFMA2", "MUFU.EX2", "PRMT", "IDP4A", "FMNMX3", "IADD", "FADD", "FRND", "FSETP+SEL", "IMAD(x*1+c)", "FMUL2", "I2F+MUFU mix", "F2F.F16x2", "EX2.F16x2"};
    auto run = [&](auto kern, int op) {
        kern<<<sms, 1024>>>(out, cyc, 3); cudaDeviceSynchronize();
        kern<<<sms, 1024>>>(out, cyc, 3); cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double warp_instr = 32.0 * ITERS * 4 * CHAINS;  // per SM (32 warps)
        printf("%-22s %8.3f warp-instr/clk/SM  (%6.1f lanes/clk)\n", names[op], warp_instr / c, 32 * warp_instr / c);
    };
    run(bench<0>, 0); run(bench<1>, 1); run(bench<2>, 2); run(bench<3>, 3); run(bench<4>, 4); run(bench<5>, 5);
    run(bench<6>, 6); run(bench<7>, 7); run(bench<8>, 8); run(bench<9>, 9); run(bench<10>, 10);
    run(bench<11>, 11); run(bench<12>, 12); run(bench<13>, 13); run(bench<14>, 14); run(bench<15>, 15);
    return 0;
}
