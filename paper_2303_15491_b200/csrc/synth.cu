// Seeded synthetic scalar fields on the device (benchmark / test harness
// utility, not part of the segmentation path). The input definition is
// include/plmss_synth.h: separable Gaussian sums from float32 axis tables
// built on the host, every product and sum rounded separately, so a host
// loop (oracle/, bench.py's reference arm) produces the same bytes. 512
// Gaussians over 2^30 voxels take ~0.1 s here and ~1 min on 8 host cores.
#include <math.h>

#include <vector>

#include "common.cuh"
#include "plmss_synth.h"

namespace plmss_b200 {
namespace {

// One CTA per (y, z) row of the generated layers; thread i takes x = i,
// i + 256, ... The axis tables: ex [ng][X], ey [ng][Y], ez [ng][Z], amp [ng].
constexpr int kSynthThreads = 256;
constexpr int kSynthX = 4;  // x values per thread kept in registers (X <= 1024 in one pass)

__global__ void __launch_bounds__(kSynthThreads) k_synth_gauss(float* __restrict__ f, uint32_t X, uint32_t Y,
                                                               uint32_t z0, const float* __restrict__ ex,
                                                               const float* __restrict__ ey,
                                                               const float* __restrict__ ez,
                                                               const float* __restrict__ amp, int ng, uint32_t Z,
                                                               double noise_amp, uint64_t seed) {
  const uint32_t row = blockIdx.x;  // local row: y + Y * (z - z0)
  const uint32_t y = row % Y, z = z0 + row / Y;
  for (uint32_t xb = 0; xb < X; xb += kSynthThreads * kSynthX) {
    float s[kSynthX];
#pragma unroll
    for (int j = 0; j < kSynthX; ++j) s[j] = 0.f;
    for (int k = 0; k < ng; ++k) {
      const float w = __fmul_rn(__ldg(amp + k), __fmul_rn(__ldg(ey + size_t(k) * Y + y), __ldg(ez + size_t(k) * Z + z)));
      const float* exk = ex + size_t(k) * X;
#pragma unroll
      for (int j = 0; j < kSynthX; ++j) {
        const uint32_t x = xb + threadIdx.x + j * kSynthThreads;
        if (x < X) s[j] = __fadd_rn(s[j], __fmul_rn(__ldg(exk + x), w));
      }
    }
#pragma unroll
    for (int j = 0; j < kSynthX; ++j) {
      const uint32_t x = xb + threadIdx.x + j * kSynthThreads;
      if (x < X) {
        const uint64_t v = uint64_t(x) + uint64_t(X) * (uint64_t(y) + uint64_t(Y) * z);
        const double u = plmss_synth_uniform01(seed, v);
        // (double)s + noise * (2u - 1), no contraction into an FMA
        const double nz = __dmul_rn(noise_amp, __dadd_rn(__dmul_rn(2.0, u), -1.0));
        f[uint64_t(row) * X + x] = float(__dadd_rn(double(s[j]), nz));
      }
    }
  }
}

__global__ void k_synth_uniform(float* __restrict__ f, uint64_t v0, uint64_t n, uint64_t seed) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) f[i] = float(plmss_synth_uniform01(seed, v0 + i));
}

__device__ __forceinline__ unsigned ord(float x) {
  const unsigned b = __float_as_uint(x);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord(unsigned k) {
  return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}

__global__ void k_minmax(const float* __restrict__ f, uint64_t n, unsigned* __restrict__ mm) {
  unsigned lo = 0xffffffffu, hi = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned k = ord(f[i]);
    lo = min(lo, k);
    hi = max(hi, k);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void k_quantise(float* __restrict__ f, uint64_t n, const unsigned* __restrict__ mm, int levels) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo = unord(mm[0]), hi = unord(mm[1]);
  const double t = hi > lo ? __ddiv_rn(__dadd_rn(double(f[i]), -lo), __dadd_rn(hi, -lo)) : 0.0;
  int q = int(floor(__dmul_rn(t, double(levels))));
  q = q < 0 ? 0 : (q >= levels ? levels - 1 : q);
  f[i] = float(q);
}

}  // namespace

// Vertex layers [z0, z0 + nz) of the field (nz == Z, z0 == 0: the whole
// volume, then quantised when levels > 0).
void synth(Ctx& c, const Grid& g, int kind, const double* h_gauss, int n_gauss, double noise_amp, uint64_t seed,
           int levels, float* field, int64_t z0, int64_t nz) {
  if (n_gauss < 0 || n_gauss > 65536) fail(PLMSS_ERR_INVALID_ARGUMENT, "n_gauss out of range");
  if (z0 < 0 || nz < 1 || z0 + nz > g.Z) fail(PLMSS_ERR_INVALID_ARGUMENT, "synth layer range outside the grid");
  if (levels > 0 && (z0 != 0 || nz != g.Z))
    fail(PLMSS_ERR_INVALID_ARGUMENT, "quantised fields are generated whole (the levels span the global range)");
  const uint64_t n = uint64_t(g.X) * uint64_t(g.Y) * uint64_t(nz);
  if (kind == 0) {
    const int ng = n_gauss;
    std::vector<float> tab(size_t(ng) * size_t(g.X + g.Y + g.Z + 1));
    float* ex = tab.data();
    float* ey = ex + size_t(ng) * g.X;
    float* ez = ey + size_t(ng) * g.Y;
    float* am = ez + size_t(ng) * g.Z;
    for (int k = 0; k < ng; ++k) {
      const double* p = h_gauss + 5 * k;
      plmss_synth_axis_table(p[0], p[3], g.X, ex + size_t(k) * g.X);
      plmss_synth_axis_table(p[1], p[3], g.Y, ey + size_t(k) * g.Y);
      plmss_synth_axis_table(p[2], p[3], g.Z, ez + size_t(k) * g.Z);
      am[k] = float(p[4]);
    }
    float* d_tab = nullptr;
    CK(cudaMallocAsync(&d_tab, std::max<size_t>(tab.size(), 1) * sizeof(float), c.stream));
    CK(cudaMemcpyAsync(d_tab, tab.data(), tab.size() * sizeof(float), cudaMemcpyHostToDevice, c.stream));
    const float* dex = d_tab;
    const float* dey = dex + size_t(ng) * g.X;
    const float* dez = dey + size_t(ng) * g.Y;
    const float* dam = dez + size_t(ng) * g.Z;
    const uint64_t rows = uint64_t(g.Y) * uint64_t(nz);
    if (rows >= (uint64_t(1) << 31)) fail(PLMSS_ERR_INVALID_ARGUMENT, "too many rows for the generator");
    k_synth_gauss<<<unsigned(rows), kSynthThreads, 0, c.stream>>>(field, uint32_t(g.X), uint32_t(g.Y), uint32_t(z0),
                                                                   dex, dey, dez, dam, ng, uint32_t(g.Z), noise_amp,
                                                                   seed);
    CK_LAUNCH("k_synth_gauss");
    CK(cudaFreeAsync(d_tab, c.stream));
  } else {
    k_synth_uniform<<<blocks_for(int64_t(n), 256), 256, 0, c.stream>>>(
        field, uint64_t(z0) * uint64_t(g.X) * uint64_t(g.Y), n, seed);
    CK_LAUNCH("k_synth_uniform");
  }
  if (levels > 0) {
    const unsigned nb = blocks_for(int64_t(n), 256);
    unsigned* mm = static_cast<unsigned*>(c.get(S_FLAGS, 64));
    const unsigned init[2] = {0xffffffffu, 0u};
    CK(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, c.stream));
    k_minmax<<<4 * 148, 256, 0, c.stream>>>(field, n, mm);
    CK_LAUNCH("k_minmax");
    k_quantise<<<nb, 256, 0, c.stream>>>(field, n, mm, levels);
    CK_LAUNCH("k_quantise");
  }
  c.sync();
}

}  // namespace plmss_b200
