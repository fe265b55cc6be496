#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int8_t* out, int D) {
  __shared__ alignas(1024) int8_t buf[128*128];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(128*D));
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      :: "r"((uint32_t)__cvta_generic_to_shared(buf)), "l"(&m), "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(0), "r"(0), "r"(0), "r"(0), "r"(4) : "memory");
    uint32_t ok=0; while(!ok){ asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0,1,0,P;}" : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar))); }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128*D; i += blockDim.x) out[i] = buf[i];
}
int main() {
  const int D = 128, N = 512;
  int8_t* g; cudaMalloc(&g, N*D); int8_t h[N*D]; for (int r=0;r<N;++r) for(int c=0;c<D;++c) h[r*D+c]=(int8_t)(r&127);
  cudaMemcpy(g,h,N*D,cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled",&p,cudaEnableDefault,&q);
  PFN enc=(PFN)p; CUtensorMap m;
  // dims: d, e(2, stride D), m(4, stride 8D), t0(4, stride 2D), k'(N/32, stride 32D)
  cuuint64_t dims[5]={D,2,4,4,(cuuint64_t)(N/32)}; cuuint64_t str[4]={(cuuint64_t)D,(cuuint64_t)8*D,(cuuint64_t)2*D,(cuuint64_t)32*D};
  cuuint32_t box[5]={(cuuint32_t)D,2,4,4,4}; cuuint32_t es[5]={1,1,1,1,1};
  CUresult r=enc(&m,CU_TENSOR_MAP_DATA_TYPE_UINT8,5,g,dims,str,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_NONE,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode result %d\n",(int)r);
  if (r) return 1;
  int8_t* o; cudaMalloc(&o,128*D); k<<<1,128>>>(m,o,D); cudaError_t e=cudaDeviceSynchronize(); printf("kernel %s\n", cudaGetErrorString(e));
  int8_t ho[128*D]; cudaMemcpy(ho,o,128*D,cudaMemcpyDeviceToHost);
  // expect smem row p = e + 2m + 8t0 + 32k' holds key 128 + e + 8m + 2t0 + 32k' (k'' start 4 -> key 128)
  int bad=0; for(int p=0;p<128;++p){int e=p&1,mm=(p>>1)&3,t0=(p>>3)&3,kk=p>>5; int key=128+e+8*mm+2*t0+32*kk; if(ho[p*D]!=(int8_t)(key&127)) ++bad;}
  printf("rows wrong: %d\n",bad); return 0;
}
