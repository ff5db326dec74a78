// Probe 2: TMA load with runtime-aligned dynamic smem (debug tool).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__global__ void __launch_bounds__(1024, 1) probe(const __grid_constant__ CUtensorMap tmap, float* out, int align_rt, int c, int cy) {
  extern __shared__ __align__(16) unsigned char raw[];
  unsigned char* sm = align_rt ? raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u) : raw;
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(166464u) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(sm)), "l"(&tmap), "r"(c), "r"(cy), "r"(cy), "r"(b) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(b) : "memory");
  if (threadIdx.x == 0) { out[0] = reinterpret_cast<float*>(sm)[0]; out[1] = float(smem_u32(sm)); out[2] = float(smem_u32(raw)); }
}
int main(int argc, char** argv) {
  const int align_rt = atoi(argv[1]); const int smem = atoi(argv[2]); const int c = atoi(argv[3]);
  const int X = 64, Y = 64, Z = 64;
  float* d; cudaMalloc(&d, 4 * X * Y * Z); cudaMemset(d, 0, 4 * X * Y * Z);
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m; memset(&m, 0, sizeof m);
  cuuint64_t gd[3] = {X, Y, Z}, gs[2] = {X * 4ull, X * Y * 4ull};
  cuuint32_t box[3] = {36, 34, 34}, es[3] = {1, 1, 1};
  ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA);
  float* o; cudaMalloc(&o, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<8, 1024, smem>>>(m, o, align_rt, c, argc > 4 ? atoi(argv[4]) : c);
  cudaError_t e = cudaDeviceSynchronize();
  float h[3] = {0, 0, 0}; cudaMemcpy(h, o, 12, cudaMemcpyDeviceToHost);
  printf("align_rt=%d smem=%d c=%d: %s  v=%f dst=%f raw=%f\n", align_rt, smem, c, cudaGetErrorString(e), h[0], h[1], h[2]);
}
