// Seeded synthetic scalar fields on the device (benchmark / test harness
// utility, not part of the segmentation path). The BASELINE configs'
// distributions (Gaussian sums + uniform noise, white noise, quantised sums)
// are generated here because 512 Gaussians over 2^30 voxels is too slow on
// the host; the bytes are then shared with the CPU oracle.
#include <math.h>

#include <vector>

#include "common.cuh"

namespace plmss_b200 {
namespace {

constexpr int kMaxGauss = 1024;
__constant__ float4 c_gauss[kMaxGauss];  // cx, cy, cz, -1/(2 sigma^2)
__constant__ float c_amp[kMaxGauss];

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// u in [0, 1): 53 high bits of a hash of (seed, v), the reference's
// (rng() >> 11) * 2^-53 mapping (synth.cpp:15-17) over a counter-based hash.
__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t v) {
  return double(splitmix64(seed ^ (v * 0xD1B54A32D192ED03ull)) >> 11) * 0x1.0p-53;
}

__global__ void k_synth(float* __restrict__ f, uint32_t X, uint32_t Y, uint64_t n, int kind, int ng,
                        double noise_amp, uint64_t seed) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= n) return;
  if (kind == 1) {
    f[v] = float(uniform01(seed, v));
    return;
  }
  const float x = float(v % X), y = float((v / X) % Y), z = float(v / (uint64_t(X) * Y));
  float s = 0.f;
  for (int k = 0; k < ng; ++k) {
    const float4 g = c_gauss[k];
    const float dx = x - g.x, dy = y - g.y, dz = z - g.z;
    s += c_amp[k] * expf((dx * dx + dy * dy + dz * dz) * g.w);
  }
  f[v] = float(double(s) + noise_amp * (2.0 * uniform01(seed, v) - 1.0));
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
  const double t = hi > lo ? (double(f[i]) - lo) / (hi - lo) : 0.0;
  int q = int(floor(t * levels));
  q = q < 0 ? 0 : (q >= levels ? levels - 1 : q);
  f[i] = float(q);
}

}  // namespace

void synth(Ctx& c, const Grid& g, int kind, const double* h_gauss, int n_gauss, double noise_amp, uint64_t seed,
           int levels, float* field) {
  if (n_gauss < 0 || n_gauss > kMaxGauss) fail(PLMSS_ERR_INVALID_ARGUMENT, "n_gauss out of range");
  if (kind == 0 && n_gauss > 0) {
    std::vector<float4> gp(n_gauss);
    std::vector<float> amp(n_gauss);
    for (int k = 0; k < n_gauss; ++k) {
      const double* p = h_gauss + 5 * k;
      gp[k] = make_float4(float(p[0]), float(p[1]), float(p[2]), float(-1.0 / (2.0 * p[3] * p[3])));
      amp[k] = float(p[4]);
    }
    CK(cudaMemcpyToSymbolAsync(c_gauss, gp.data(), sizeof(float4) * n_gauss, 0, cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyToSymbolAsync(c_amp, amp.data(), sizeof(float) * n_gauss, 0, cudaMemcpyHostToDevice, c.stream));
  }
  const unsigned nb = blocks_for(g.n, 256);
  k_synth<<<nb, 256, 0, c.stream>>>(field, uint32_t(g.X), uint32_t(g.Y), uint64_t(g.n), kind,
                                    kind == 0 ? n_gauss : 0, noise_amp, seed);
  CK_LAUNCH("k_synth");
  if (levels > 0) {
    unsigned* mm = static_cast<unsigned*>(c.get(S_FLAGS, 64));
    const unsigned init[2] = {0xffffffffu, 0u};
    CK(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, c.stream));
    k_minmax<<<4 * 148, 256, 0, c.stream>>>(field, uint64_t(g.n), mm);
    CK_LAUNCH("k_minmax");
    k_quantise<<<nb, 256, 0, c.stream>>>(field, uint64_t(g.n), mm, levels);
    CK_LAUNCH("k_quantise");
  }
  c.sync();
}

}  // namespace plmss_b200
