// Standalone probe of a 3-D TMA tensor load (debug tool, not product code).
// Usage: tma_probe <bx> <by> <bz> <mode>   mode 0: grid_constant map, 1: global map
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

__global__ void probe_gc(const __grid_constant__ CUtensorMap tmap, unsigned bytes, float* out, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    if (!(mode & 4)) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int c0 = (mode & 8) ? 40 : ((mode & 1) ? 0 : -1);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(sm)),
        "l"(&tmap), "r"(c0), "r"(c0), "r"(c0), "r"(b)
        : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(b)
               : "memory");
  if (threadIdx.x == 0) {
    const float* f = reinterpret_cast<const float*>(sm);
    out[0] = f[0];
    out[1] = f[1];
    out[2] = f[bytes / 4 - 1];
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 4 ? atoi(argv[4]) : 0;
  const unsigned bx = argc > 1 ? atoi(argv[1]) : 36, by = argc > 2 ? atoi(argv[2]) : 34,
                 bz = argc > 3 ? atoi(argv[3]) : 34;
  const int X = 64, Y = 64, Z = 64;
  float* d;
  cudaMalloc(&d, sizeof(float) * X * Y * Z);
  float* h = (float*)malloc(sizeof(float) * X * Y * Z);
  for (int i = 0; i < X * Y * Z; ++i) h[i] = float(i);
  cudaMemcpy(d, h, sizeof(float) * X * Y * Z, cudaMemcpyHostToDevice);
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn encode = (EncodeFn)fn;
  CUtensorMap m;
  memset(&m, 0, sizeof m);
  cuuint64_t gd[3] = {X, Y, Z}, gs[2] = {X * 4ull, X * Y * 4ull};
  cuuint32_t box[3] = {bx, by, bz}, es[3] = {1, 1, 1};
  CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, (mode & 32) ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      (mode & 2) ? CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE : CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA);
  printf("encode=%d q=%d\n", int(r), int(q));
  const unsigned bytes = bx * by * bz * 4;
  float* o;
  cudaMalloc(&o, 16);
  cudaFuncSetAttribute(probe_gc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe_gc<<<1, (mode & 16) ? 1024 : 128, bytes + 1024>>>(m, bytes, o, mode);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[3];
  cudaMemcpy(ho, o, 12, cudaMemcpyDeviceToHost);
  printf("mode %d box %u %u %u: %s  f0=%f f1=%f flast=%f\n", mode, bx, by, bz, cudaGetErrorString(e), ho[0], ho[1], ho[2]);
  return 0;
}
