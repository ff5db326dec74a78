// Segmentation kernels: steepest-neighbour hops (K1), path compression (K2),
// ordered extrema compaction, and the GPU order field.
//
// Reference semantics:
//  * u is higher than v iff (key(u), u) > (key(v), v) lexicographically — the
//    simulation-of-simplicity order of compute_order (orderfield.cpp:21-26),
//    compared directly on the keys (F5): no global sort is needed.
//  * neighbours = the 14-offset Freudenthal stencil, out-of-volume offsets
//    skipped (complex.cpp:53-64, complex.hpp:84-101).
//  * desc[v] = highest neighbour if higher than v, else v; asc symmetric
//    (segmentation.cpp:60-85); labels = fixpoint of label <- label[label]
//    (segmentation.cpp:87-105), unique and schedule-independent (F6).
#include <math.h>

#include "common.cuh"

namespace plmss_b200 {
namespace {

template <class K>
struct KeyOps;
template <>
struct KeyOps<float> {
  static __device__ __forceinline__ bool finite(float v) { return isfinite(v); }
};
template <>
struct KeyOps<double> {
  static __device__ __forceinline__ bool finite(double v) { return isfinite(v); }
};
template <>
struct KeyOps<int64_t> {
  static __device__ __forceinline__ bool finite(int64_t) { return true; }
};

// (ku, u) > (kv, v). IEEE compare: -0.0 == +0.0 falls through to the id.
template <class K>
__device__ __forceinline__ bool higher(K ku, uint32_t u, K kv, uint32_t v) {
  return ku > kv || (ku == kv && u > v);
}

struct Dims {
  uint32_t X, Y, Z, XY;
  uint32_t n;
};

// K1 (v1): one thread per vertex, neighbour keys through L1/L2.
template <class K>
__global__ void __launch_bounds__(256) k_seed_hops(const K* __restrict__ key, Dims d,
                                                   uint32_t* __restrict__ desc,
                                                   uint32_t* __restrict__ asc,
                                                   uint32_t* __restrict__ bad) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= d.n) return;
  const uint32_t x = v % d.X;
  const uint32_t y = (v / d.X) % d.Y;
  const uint32_t z = v / d.XY;
  const K kv = __ldg(key + v);
  if (bad && !KeyOps<K>::finite(kv)) atomicMin(bad, v);
  K kup = kv, kdn = kv;
  uint32_t up = v, dn = v;
  const bool xm = x > 0, xp = x + 1 < d.X, ym = y > 0, yp = y + 1 < d.Y, zm = z > 0, zp = z + 1 < d.Z;
  auto visit = [&](bool ok, uint32_t u) {
    if (!ok) return;
    const K ku = __ldg(key + u);
    if (higher(ku, u, kup, up)) {
      kup = ku;
      up = u;
    }
    if (higher(kdn, dn, ku, u)) {
      kdn = ku;
      dn = u;
    }
  };
  // 14 offsets: nonzero components share a sign.
  visit(xm && ym && zm, v - d.XY - d.X - 1);
  visit(ym && zm, v - d.XY - d.X);
  visit(xm && zm, v - d.XY - 1);
  visit(zm, v - d.XY);
  visit(xm && ym, v - d.X - 1);
  visit(ym, v - d.X);
  visit(xm, v - 1);
  visit(xp, v + 1);
  visit(yp, v + d.X);
  visit(xp && yp, v + d.X + 1);
  visit(zp, v + d.XY);
  visit(xp && zp, v + d.XY + 1);
  visit(yp && zp, v + d.XY + d.X);
  visit(xp && yp && zp, v + d.XY + d.X + 1);
  if (desc) desc[v] = up;
  if (asc) asc[v] = dn;
}

// K2 (v1): each sweep follows up to kHops links per vertex on the live
// arrays. Every value read lies on the vertex's monotone chain (the same
// argument as the reference's relaxed atomics, segmentation.cpp:14-20), so
// any interleaving converges to the unique fixpoint; a sweep with no change
// proves desc[desc[v]] == desc[v] for all v.
constexpr int kHops = 6;

__global__ void __launch_bounds__(256) k_jump(uint32_t* __restrict__ lab, uint32_t n, int* __restrict__ changed) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  bool ch = false;
  if (v < n) {
    const uint32_t l0 = lab[v];
    uint32_t l = l0;
#pragma unroll
    for (int k = 0; k < kHops; ++k) {
      const uint32_t nx = lab[l];
      if (nx == l) break;
      l = nx;
    }
    if (l != l0) {
      lab[v] = l;
      ch = lab[l] != l;  // not yet at a root: needs another sweep
    }
  }
  if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

// One sweep over an explicit active list; keep[i] = 1 while unsettled.
__global__ void k_sweep_list(uint32_t* __restrict__ desc, uint32_t* __restrict__ asc,
                             const uint32_t* __restrict__ active, int64_t na, uint32_t* __restrict__ keep) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= na) return;
  const uint32_t v = active[i];
  const uint32_t d2 = desc[desc[v]];
  desc[v] = d2;
  bool settled = desc[d2] == d2;
  if (asc) {
    const uint32_t a2 = asc[asc[v]];
    asc[v] = a2;
    settled = settled && asc[a2] == a2;
  }
  keep[i] = settled ? 0u : 1u;
}

// ---------------------------------------------------- ordered compaction --
constexpr int kCThreads = 256;
constexpr int kCRows = 16;
constexpr int kCTile = kCThreads * kCRows;

__global__ void __launch_bounds__(kCThreads) k_count_self(const uint32_t* __restrict__ lab, uint32_t n,
                                                          uint64_t* __restrict__ counts) {
  const uint32_t base = blockIdx.x * kCTile;
  uint32_t c = 0;
#pragma unroll
  for (int r = 0; r < kCRows; ++r) {
    const uint32_t i = base + r * kCThreads + threadIdx.x;
    if (i < n && lab[i] == i) ++c;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t wsum[kCThreads / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kCThreads / 32; ++w) t += wsum[w];
    counts[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kCThreads) k_write_self(const uint32_t* __restrict__ lab, uint32_t n,
                                                          const uint64_t* __restrict__ offsets,
                                                          uint32_t* __restrict__ out,
                                                          uint32_t* __restrict__ rank_map) {
  __shared__ uint32_t wcnt[kCThreads / 32];
  __shared__ uint32_t wpre[kCThreads / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t base = blockIdx.x * kCTile;
  uint64_t running = offsets[blockIdx.x];
  for (int r = 0; r < kCRows; ++r) {
    const uint32_t i = base + r * kCThreads + threadIdx.x;
    const bool hit = i < n && lab[i] == i;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int k = 0; k < kCThreads / 32; ++k) {
        wpre[k] = s;
        s += wcnt[k];
      }
      wpre[kCThreads / 32] = s;
    }
    __syncthreads();
    if (hit) {
      const uint64_t pos = running + wpre[w] + __popc(m & ((1u << lane) - 1));
      if (out) out[pos] = i;
      if (rank_map) rank_map[i] = static_cast<uint32_t>(pos);
    }
    running += wpre[kCThreads / 32];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kCThreads) k_count_flag(const uint32_t* __restrict__ flag, int64_t n,
                                                          uint64_t* __restrict__ counts) {
  const int64_t base = int64_t(blockIdx.x) * kCTile;
  uint32_t c = 0;
  for (int r = 0; r < kCRows; ++r) {
    const int64_t i = base + r * kCThreads + threadIdx.x;
    if (i < n && flag[i]) ++c;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[kCThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kCThreads / 32; ++w) t += ws[w];
    counts[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kCThreads) k_write_flag(const uint32_t* __restrict__ flag,
                                                          const uint32_t* __restrict__ vals, int64_t n,
                                                          const uint64_t* __restrict__ offsets,
                                                          uint32_t* __restrict__ out) {
  __shared__ uint32_t wc[kCThreads / 32];
  __shared__ uint32_t wp[kCThreads / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = int64_t(blockIdx.x) * kCTile;
  uint64_t running = offsets[blockIdx.x];
  for (int r = 0; r < kCRows; ++r) {
    const int64_t i = base + r * kCThreads + threadIdx.x;
    const bool hit = i < n && flag[i];
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wc[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int k = 0; k < kCThreads / 32; ++k) {
        wp[k] = s;
        s += wc[k];
      }
      wp[kCThreads / 32] = s;
    }
    __syncthreads();
    if (hit) out[running + wp[w] + __popc(m & ((1u << lane) - 1))] = vals[i];
    running += wp[kCThreads / 32];
    __syncthreads();
  }
}

// ------------------------------------------------------------ order field --
// Order-preserving u64 image of a finite double with -0.0 canonicalised to
// +0.0 (compute_order compares with ==, orderfield.cpp:24).
__device__ __forceinline__ uint64_t order_key(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t b = __double_as_longlong(x);
  return (b >> 63) ? ~b : (b | (uint64_t(1) << 63));
}

template <class T>
__global__ void k_order_keys(const T* __restrict__ v, int64_t n, uint64_t* __restrict__ keys,
                             uint64_t* __restrict__ ids, unsigned long long* __restrict__ bad) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = static_cast<double>(v[i]);
  if (!isfinite(x)) atomicMin(bad, static_cast<unsigned long long>(i));
  keys[i] = order_key(x);
  ids[i] = static_cast<uint64_t>(i);
}

__global__ void k_scatter_rank(const uint64_t* __restrict__ ids, int64_t n, int64_t* __restrict__ rank) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) rank[ids[i]] = i;
}

Dims to_dims(const Grid& g) {
  Dims d;
  d.X = static_cast<uint32_t>(g.X);
  d.Y = static_cast<uint32_t>(g.Y);
  d.Z = static_cast<uint32_t>(g.Z);
  d.XY = d.X * d.Y;
  d.n = static_cast<uint32_t>(g.n);
  return d;
}

}  // namespace

void seed_hops(Ctx& c, const Grid& g, int key_type, const void* keys, uint32_t* desc, uint32_t* asc,
               uint32_t* bad) {
  const Dims d = to_dims(g);
  const unsigned nb = blocks_for(g.n, 256);
  switch (key_type) {
    case PLMSS_KEY_F32:
      k_seed_hops<float><<<nb, 256, 0, c.stream>>>(static_cast<const float*>(keys), d, desc, asc, bad);
      break;
    case PLMSS_KEY_F64:
      k_seed_hops<double><<<nb, 256, 0, c.stream>>>(static_cast<const double*>(keys), d, desc, asc, bad);
      break;
    case PLMSS_KEY_RANK:
      k_seed_hops<int64_t><<<nb, 256, 0, c.stream>>>(static_cast<const int64_t*>(keys), d, desc, asc, nullptr);
      break;
    default:
      fail(PLMSS_ERR_INVALID_ARGUMENT, "unknown key type");
  }
  CK_LAUNCH("k_seed_hops");
}

// Slab halo layers become terminals: label = self.
__global__ void k_terminal_layer(uint32_t* __restrict__ desc, uint32_t* __restrict__ asc, uint32_t first,
                                 uint32_t count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  desc[first + i] = first + i;
  asc[first + i] = first + i;
}

void terminal_layers(Ctx& c, const Grid& g, bool lo, bool hi, uint32_t* desc, uint32_t* asc) {
  const uint32_t XY = uint32_t(g.X * g.Y);
  if (lo) {
    k_terminal_layer<<<blocks_for(XY, 256), 256, 0, c.stream>>>(desc, asc, 0u, XY);
    CK_LAUNCH("k_terminal_layer");
  }
  if (hi) {
    k_terminal_layer<<<blocks_for(XY, 256), 256, 0, c.stream>>>(desc, asc, uint32_t(g.n) - XY, XY);
    CK_LAUNCH("k_terminal_layer");
  }
}

int compress(Ctx& c, int64_t n, uint32_t* desc, uint32_t* asc) {
  int* flag = static_cast<int*>(c.get(S_FLAGS, 64));
  int sweeps = 0;
  const unsigned nb = blocks_for(n, 256);
  for (;;) {
    CK(cudaMemsetAsync(flag, 0, sizeof(int), c.stream));
    if (desc) k_jump<<<nb, 256, 0, c.stream>>>(desc, static_cast<uint32_t>(n), flag);
    if (asc) k_jump<<<nb, 256, 0, c.stream>>>(asc, static_cast<uint32_t>(n), flag);
    CK_LAUNCH("k_jump");
    ++sweeps;
    CK(cudaMemcpyAsync(c.h_pinned, flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (*reinterpret_cast<int*>(c.h_pinned) == 0) break;
    if (sweeps > 64) fail(PLMSS_ERR_LOGIC, "path compression did not converge");
  }
  return sweeps;
}

int64_t count_extrema(Ctx& c, int64_t n, const uint32_t* labels) {
  const int64_t nb = (n + kCTile - 1) / kCTile;
  uint64_t* counts = c.get_t<uint64_t>(S_TMP1, nb);
  k_count_self<<<(unsigned)nb, kCThreads, 0, c.stream>>>(labels, static_cast<uint32_t>(n), counts);
  CK_LAUNCH("k_count_self");
  return static_cast<int64_t>(exclusive_scan_u64(c, counts, nb, true));
}

void write_extrema(Ctx& c, int64_t n, const uint32_t* labels, uint32_t* out, uint32_t* rank_map) {
  if (!out && !rank_map) return;
  const int64_t nb = (n + kCTile - 1) / kCTile;
  uint64_t* counts = c.get_t<uint64_t>(S_TMP1, nb);
  k_write_self<<<(unsigned)nb, kCThreads, 0, c.stream>>>(labels, static_cast<uint32_t>(n), counts, out, rank_map);
  CK_LAUNCH("k_write_self");
}

int64_t compress_sweep_list(Ctx& c, uint32_t* desc, uint32_t* asc, const uint32_t* active, int64_t na,
                            uint32_t* next) {
  if (na <= 0) return 0;
  uint32_t* keep = c.get_t<uint32_t>(S_TMP0, na);
  k_sweep_list<<<blocks_for(na, 256), 256, 0, c.stream>>>(desc, asc, active, na, keep);
  CK_LAUNCH("k_sweep_list");
  const int64_t nb = (na + kCTile - 1) / kCTile;
  uint64_t* counts = c.get_t<uint64_t>(S_TMP1, nb);
  k_count_flag<<<(unsigned)nb, kCThreads, 0, c.stream>>>(keep, na, counts);
  CK_LAUNCH("k_count_flag");
  const int64_t total = int64_t(exclusive_scan_u64(c, counts, nb, true));
  k_write_flag<<<(unsigned)nb, kCThreads, 0, c.stream>>>(keep, active, na, counts, next);
  CK_LAUNCH("k_write_flag");
  return total;
}

void compute_order(Ctx& c, int key_type, const void* values, int64_t n, int64_t* rank) {
  if (n <= 0) return;
  uint64_t* keys = c.get_t<uint64_t>(S_SORT_A, n);
  uint64_t* ids = c.get_t<uint64_t>(S_SORT_B, n);
  unsigned long long* bad = static_cast<unsigned long long*>(c.get(S_FLAGS, 64));
  CK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), c.stream));
  const unsigned nb = blocks_for(n, 256);
  if (key_type == PLMSS_KEY_F32)
    k_order_keys<float><<<nb, 256, 0, c.stream>>>(static_cast<const float*>(values), n, keys, ids, bad);
  else if (key_type == PLMSS_KEY_F64)
    k_order_keys<double><<<nb, 256, 0, c.stream>>>(static_cast<const double*>(values), n, keys, ids, bad);
  else
    fail(PLMSS_ERR_INVALID_ARGUMENT, "compute_order needs f32 or f64 values");
  CK_LAUNCH("k_order_keys");
  CK(cudaMemcpyAsync(c.h_pinned, bad, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (c.h_pinned[0] != ~uint64_t(0))
    fail(PLMSS_ERR_INVALID_ARGUMENT, "non-finite scalar value at vertex " + std::to_string(c.h_pinned[0]));
  radix_sort_pairs(c, keys, ids, n, 64);
  k_scatter_rank<<<nb, 256, 0, c.stream>>>(ids, n, rank);
  CK_LAUNCH("k_scatter_rank");
}

}  // namespace plmss_b200
