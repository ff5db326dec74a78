// Fused B200 pipeline (the benchmarked path).
//
//  A  k_tile_segment  : 32x16x16-vertex tiles staged in shared memory with a
//                       1-voxel halo. Steepest up/down hops from the 14-point
//                       stencil (SoS on (f, id)), then pointer jumping INSIDE
//                       shared memory until every tile vertex points at a
//                       terminal: a root (extremum) or an exit vertex outside
//                       the tile. Writes the partial labels (global ids) into
//                       desc/asc, appends roots to the extremum lists, exit
//                       targets to the exit list E, and distinct (asc, desc)
//                       partial pairs to a hash set.
//  B  k_exit_jump     : pointer jumping restricted to E (closed under the
//                       partial-label map), to the global fixpoint.
//  C  pairs           : partial pairs -> final pairs -> unique, sorted ->
//                       dense MS ids (hash value slots).
//  D  k_finalize_march: ordered single pass over row-slab tiles in the
//                       reference cell order: final labels = L[L[v]], dense
//                       id lookup, desc/asc/ms writes, 6-tet codes per cube,
//                       decoupled look-back for output offsets, separator
//                       records in reference order.
//
// Correctness: every partial label lies on the vertex's steepest chain and
// the chain's terminal extremum is unique, so any order of
// these resolutions reproduces the reference labels exactly.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "tet_tables.h"

namespace plmss_b200 {

namespace {

constexpr int TX = 32, TY = 16, TZ = 16;
constexpr int HX = TX + 2, HY = TY + 2, HZ = TZ + 2;
constexpr int HN = HX * HY * HZ;  // 11016
constexpr int TN = TX * TY * TZ;  // 8192
constexpr int A_THREADS = 512;
constexpr int A_PER = TN / A_THREADS;  // 16
constexpr uint16_t TERM = 0x8000, EXIT = 0x4000;
constexpr int kASmem = 4 * HN + 2 * 2 * TN + HN;  // f, Pd, Pa, exit flags
constexpr uint64_t kEmpty = ~uint64_t(0);

struct FDims {
  uint32_t X, Y, Z, XY, n;
  uint32_t tx, ty, tz;  // tile counts
};


__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// Insert k into an open-addressing set; returns false on probe overflow.
__device__ __forceinline__ bool set_insert(unsigned long long* __restrict__ t, uint64_t mask, uint64_t k) {
  uint64_t s = mix64(k) & mask;
#pragma unroll 1
  for (int probe = 0; probe < 1024; ++probe) {
    const unsigned long long cur = t[s];
    if (cur == k) return true;
    if (cur == kEmpty) {
      const unsigned long long prev = atomicCAS(t + s, kEmpty, k);
      if (prev == kEmpty || prev == k) return true;
    }
    s = (s + 1) & mask;
  }
  return false;
}

__device__ __forceinline__ uint64_t set_find(const unsigned long long* __restrict__ t, uint64_t mask, uint64_t k) {
  uint64_t s = mix64(k) & mask;
  while (t[s] != k) s = (s + 1) & mask;
  return s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Stencil offset s as 2-bit-per-axis code (x low), selected without local
// memory: a 14-entry x 6-bit table packed into two 64-bit immediates.
__device__ __forceinline__ uint32_t kOffTable(int s) {
  constexpr uint64_t lo = 0x00ull | 0x01ull << 6 | 0x04ull << 12 | 0x05ull << 18 | 0x10ull << 24 | 0x11ull << 30 |
                          0x14ull << 36 | 0x16ull << 42 | 0x19ull << 48 | 0x1aull << 54;
  constexpr uint64_t hi = 0x25ull | 0x26ull << 6 | 0x29ull << 12 | 0x2aull << 18;
  return s < 10 ? uint32_t((lo >> (6 * s)) & 63) : uint32_t((hi >> (6 * (s - 10))) & 63);
}

struct ACounters {
  unsigned long long n_max, n_min, n_exit;
  int overflow;
  uint32_t bad;
};

// ---------------------------------------------------------------- pass A --
__global__ void __launch_bounds__(A_THREADS, 2)
    k_tile_segment(const float* __restrict__ field, FDims d, uint32_t* __restrict__ desc,
                   uint32_t* __restrict__ asc, uint32_t* __restrict__ maxima, uint32_t* __restrict__ minima,
                   uint64_t ext_cap, uint32_t* __restrict__ exits, uint64_t exit_cap,
                   ACounters* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char a_smem[];
  float* f = reinterpret_cast<float*>(a_smem);                   // HN floats
  uint16_t* Pd = reinterpret_cast<uint16_t*>(a_smem + 4 * HN);   // TN
  uint16_t* Pa = Pd + TN;                                        // TN
  uint8_t* xflag = reinterpret_cast<uint8_t*>(Pa + TN);          // HN
  __shared__ uint32_t s_cnt;
  __shared__ unsigned long long s_base;

  const uint32_t bt = blockIdx.x;
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const int gx0 = int(tx * TX), gy0 = int(ty * TY), gz0 = int(tz * TZ);

  // 1. halo'd tile of f (x-rows are contiguous in global memory). Vertices
  //    outside the volume hold NaN: fmaxf/fminf ignore NaN and NaN == x is
  //    false, so a missing neighbour can never be selected.
  for (int i = threadIdx.x; i < HN; i += A_THREADS) {
    const int hx = i % HX, hy = (i / HX) % HY, hz = i / (HX * HY);
    const int gx = gx0 + hx - 1, gy = gy0 + hy - 1, gz = gz0 + hz - 1;
    float val = __int_as_float(0x7fc00000);
    if (gx >= 0 && gx < int(d.X) && gy >= 0 && gy < int(d.Y) && gz >= 0 && gz < int(d.Z))
      val = __ldg(field + (uint32_t(gx) + d.X * (uint32_t(gy) + d.Y * uint32_t(gz))));
    f[i] = val;
    xflag[i] = 0;
  }
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();

  // 2. hops. Stencil s = 0..13 in ascending id-delta order (complex.cpp:78-88);
  //    the vertex itself sits between s = 6 and s = 7. With M = max f over the
  //    neighbours, the steepest-up vertex under (f, id) order is the highest s
  //    with f == M when M > f(v), or when M == f(v) and that s > 6 (a larger
  //    id); otherwise v itself. Steepest-down mirrors it (lowest s, s < 7).
  //    bit codes: 2 bits per axis (0 = -1, 1 = 0, 2 = +1), x low.
  constexpr uint32_t kOff[14] = {0x00, 0x01, 0x04, 0x05, 0x10, 0x11, 0x14,
                                 0x16, 0x19, 0x1a, 0x25, 0x26, 0x29, 0x2a};
#pragma unroll 1
  for (int k = 0; k < A_PER; ++k) {
    const int l = threadIdx.x + k * A_THREADS;
    const int lx = l % TX, ly = (l / TX) % TY, lz = l / (TX * TY);
    const int gx = gx0 + lx, gy = gy0 + ly, gz = gz0 + lz;
    if (gx >= int(d.X) || gy >= int(d.Y) || gz >= int(d.Z)) {
      Pd[l] = TERM | uint16_t(l);
      Pa[l] = TERM | uint16_t(l);
      continue;
    }
    const int h = (lz + 1) * HX * HY + (ly + 1) * HX + (lx + 1);
    const float fv = f[h];
    if (!isfinite(fv)) atomicMin(&ctr->bad, uint32_t(gx) + d.X * (uint32_t(gy) + d.Y * uint32_t(gz)));
    float fn[14];
#pragma unroll
    for (int s = 0; s < 14; ++s) {
      const int dx = int(kOff[s] & 3) - 1, dy = int((kOff[s] >> 2) & 3) - 1, dz = int((kOff[s] >> 4) & 3) - 1;
      fn[s] = f[h + dx + HX * dy + HX * HY * dz];
    }
    float M = fn[0], m = fn[0];
#pragma unroll
    for (int s = 1; s < 14; ++s) {
      M = fmaxf(M, fn[s]);
      m = fminf(m, fn[s]);
    }
    int su = -1, sd = -1;
#pragma unroll
    for (int s = 0; s < 14; ++s) su = fn[s] == M ? s : su;  // highest s attaining M
#pragma unroll
    for (int s = 13; s >= 0; --s) sd = fn[s] == m ? s : sd;  // lowest s attaining m
    if (!(M > fv || (M == fv && su > 6))) su = -1;
    if (!(m < fv || (m == fv && sd < 7))) sd = -1;
    auto enc = [&](int s) -> uint16_t {
      if (s < 0) return TERM | uint16_t(l);
      const uint32_t o = kOffTable(s);
      const int dx = int(o & 3) - 1, dy = int((o >> 2) & 3) - 1, dz = int((o >> 4) & 3) - 1;
      const int mx = lx + dx, my = ly + dy, mz = lz + dz;
      const bool inside = mx >= 0 && mx < TX && my >= 0 && my < TY && mz >= 0 && mz < TZ;
      return inside ? uint16_t(l + dx + TX * dy + TX * TY * dz)
                    : uint16_t(TERM | EXIT | (h + dx + HX * dy + HX * HY * dz));
    };
    const uint16_t pu = enc(su), pd = enc(sd);
    Pd[l] = pu;
    Pa[l] = pd;
    if ((pu & (TERM | EXIT)) == (TERM | EXIT)) xflag[pu & 0x3fff] = 1;
    if ((pd & (TERM | EXIT)) == (TERM | EXIT)) xflag[pd & 0x3fff] = 1;
  }
  __syncthreads();

  // 3. in-tile pointer jumping to terminals
  for (;;) {
    bool changed = false;
#pragma unroll 4
    for (int k = 0; k < A_PER; ++k) {
      const int l = threadIdx.x + k * A_THREADS;
      uint16_t p = Pd[l];
      if (!(p & TERM)) {
        const uint16_t q = Pd[p];
        Pd[l] = q;
        changed |= !(q & TERM);
      }
      p = Pa[l];
      if (!(p & TERM)) {
        const uint16_t q = Pa[p];
        Pa[l] = q;
        changed |= !(q & TERM);
      }
    }
    if (!__syncthreads_or(changed)) break;
  }

  // 4. partial labels, roots, partial pairs
  auto gid_of = [&](uint16_t p) -> uint32_t {
    if (p & EXIT) {
      const int hh = p & 0x3fff;
      const int hx = hh % HX, hy = (hh / HX) % HY, hz = hh / (HX * HY);
      return uint32_t(gx0 + hx - 1) + d.X * (uint32_t(gy0 + hy - 1) + d.Y * uint32_t(gz0 + hz - 1));
    }
    const int ll = p & 0x1fff;
    const int lx = ll % TX, ly = (ll / TX) % TY, lz = ll / (TX * TY);
    return uint32_t(gx0 + lx) + d.X * (uint32_t(gy0 + ly) + d.Y * uint32_t(gz0 + lz));
  };
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int k = 0; k < A_PER; ++k) {
    const int l = threadIdx.x + k * A_THREADS;
    const int lx = l % TX, ly = (l / TX) % TY, lz = l / (TX * TY);
    const int gx = gx0 + lx, gy = gy0 + ly, gz = gz0 + lz;
    const bool valid = gx < int(d.X) && gy < int(d.Y) && gz < int(d.Z);
    uint32_t ld = 0, la = 0;
    bool is_max = false, is_min = false;
    if (valid) {
      const uint32_t gv = uint32_t(gx) + d.X * (uint32_t(gy) + d.Y * uint32_t(gz));
      const uint16_t pd = Pd[l], pa = Pa[l];
      ld = gid_of(pd);
      la = gid_of(pa);
      desc[gv] = ld;
      asc[gv] = la;
      is_max = ld == gv;
      is_min = la == gv;
    }
    // warp-aggregated extremum appends
    unsigned m = __ballot_sync(0xffffffffu, is_max);
    if (m) {
      unsigned long long base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(&ctr->n_max, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      const uint64_t pos = base + __popc(m & ((1u << lane) - 1));
      if (is_max && pos < ext_cap) maxima[pos] = ld;
    }
    m = __ballot_sync(0xffffffffu, is_min);
    if (m) {
      unsigned long long base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(&ctr->n_min, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      const uint64_t pos = base + __popc(m & ((1u << lane) - 1));
      if (is_min && pos < ext_cap) minima[pos] = la;
    }
  }

  // 5. exit targets of this tile -> E
  uint32_t mine = 0;
  for (int i = threadIdx.x; i < HN; i += A_THREADS) mine += xflag[i];
  mine = __reduce_add_sync(0xffffffffu, mine);
  if (lane == 0 && mine) atomicAdd(&s_cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0) s_base = s_cnt ? atomicAdd(&ctr->n_exit, (unsigned long long)s_cnt) : 0;
  __syncthreads();
  if (s_cnt == 0) return;
  __shared__ uint32_t s_pos;
  if (threadIdx.x == 0) s_pos = 0;
  __syncthreads();
  for (int i0 = 0; i0 < HN; i0 += A_THREADS) {
    const int i = i0 + threadIdx.x;
    const bool hit = i < HN && xflag[i];
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    uint32_t wbase = 0;
    if (lane == 0 && m) wbase = atomicAdd(&s_pos, __popc(m));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (hit) {
      const uint64_t pos = s_base + wbase + __popc(m & ((1u << lane) - 1));
      const int hx = i % HX, hy = (i / HX) % HY, hz = i / (HX * HY);
      if (pos < exit_cap)
        exits[pos] = uint32_t(gx0 + hx - 1) + d.X * (uint32_t(gy0 + hy - 1) + d.Y * uint32_t(gz0 + hz - 1));
    }
  }
}

// ---------------------------------------------------------------- pass B --
// Chain following on the live arrays: each exit vertex walks up to kChase
// links (both directions interleaved for memory-level parallelism) and
// stores the furthest vertex reached. Values read from entries other
// threads have already advanced only shorten the walk; every value lies on
// the vertex's chain, so concurrent updates are safe.
constexpr int kChase = 16;

__global__ void __launch_bounds__(256) k_exit_jump(const uint32_t* __restrict__ E, uint64_t ne,
                                                   uint32_t* __restrict__ desc, uint32_t* __restrict__ asc,
                                                   int* __restrict__ changed) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool ch = false;
  if (i < ne) {
    const uint32_t e = E[i];
    const uint32_t d0 = desc[e], a0 = asc[e];
    uint32_t xd = d0, xa = a0;
    bool dd = false, da = false;
#pragma unroll 4
    for (int k = 0; k < kChase && !(dd && da); ++k) {
      const uint32_t nd = dd ? xd : desc[xd];
      const uint32_t na = da ? xa : asc[xa];
      dd = nd == xd;
      da = na == xa;
      xd = nd;
      xa = na;
    }
    if (xd != d0) desc[e] = xd;
    if (xa != a0) asc[e] = xa;
    ch = !(dd && da);
  }
  if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

// ---------------------------------------------------------------- pass C --
constexpr int kCThreads = 256;
constexpr int kCRows = 16;
constexpr int kCTile = kCThreads * kCRows;

__global__ void __launch_bounds__(kCThreads) k_count_occ(const unsigned long long* __restrict__ t, int64_t n,
                                                         uint64_t* __restrict__ counts) {
  const int64_t base = int64_t(blockIdx.x) * kCTile;
  uint32_t c = 0;
  for (int r = 0; r < kCRows; ++r) {
    const int64_t i = base + r * kCThreads + threadIdx.x;
    if (i < n && t[i] != kEmpty) ++c;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[kCThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kCThreads / 32; ++w) s += ws[w];
    counts[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kCThreads) k_write_occ(const unsigned long long* __restrict__ t, int64_t n,
                                                         const uint64_t* __restrict__ off, uint64_t* __restrict__ keys,
                                                         uint64_t* __restrict__ slots) {
  __shared__ uint32_t wc[kCThreads / 32];
  __shared__ uint32_t wp[kCThreads / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = int64_t(blockIdx.x) * kCTile;
  uint64_t running = off[blockIdx.x];
  for (int r = 0; r < kCRows; ++r) {
    const int64_t i = base + r * kCThreads + threadIdx.x;
    const unsigned long long k = i < n ? t[i] : kEmpty;
    const bool hit = k != kEmpty;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wc[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int q = 0; q < kCThreads / 32; ++q) {
        wp[q] = s;
        s += wc[q];
      }
      wp[kCThreads / 32] = s;
    }
    __syncthreads();
    if (hit) {
      const uint64_t pos = running + wp[w] + __popc(m & ((1u << lane) - 1));
      keys[pos] = k;
      if (slots) slots[pos] = uint64_t(i);
    }
    running += wp[kCThreads / 32];
    __syncthreads();
  }
}

// Pass C: final labels in place, desc[v] <- desc[desc[v]] (partial labels
// point at roots or at exit vertices already resolved by pass B, and those
// entries never change value here), and every final (asc, desc) pair into
// the region set with warp-level dedup. 4 vertices per thread per step keep
// enough independent loads in flight.
constexpr int C_VPT = 4;
// Vertices are visited in pass-A tile order (32x16x16 bricks, x-rows of 32
// inside), so the gathers desc[desc[v]] hit the few exit vertices around the
// brick while they are still in L2.
__global__ void __launch_bounds__(256) k_mark_pairs(FDims dm, uint32_t* __restrict__ desc,
                                                    uint32_t* __restrict__ asc,
                                                    unsigned long long* __restrict__ fset, uint64_t fmask,
                                                    int* __restrict__ overflow) {
  const int lane = threadIdx.x & 31;
  const uint64_t total = uint64_t(dm.tx) * dm.ty * dm.tz * TN;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * C_VPT;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x * C_VPT; base < total; base += stride) {
    uint32_t v[C_VPT], pd[C_VPT], pa[C_VPT], fd[C_VPT], fa[C_VPT];
    bool okv[C_VPT];
#pragma unroll
    for (int k = 0; k < C_VPT; ++k) {
      const uint64_t idx = base + uint64_t(k) * blockDim.x + threadIdx.x;
      const uint32_t t = uint32_t(idx / TN), l = uint32_t(idx % TN);
      const uint32_t tx = t % dm.tx, ty = (t / dm.tx) % dm.ty, tz = t / (dm.tx * dm.ty);
      const uint32_t x = tx * TX + (l % TX), y = ty * TY + ((l / TX) % TY), z = tz * TZ + l / (TX * TY);
      okv[k] = idx < total && x < dm.X && y < dm.Y && z < dm.Z;
      v[k] = x + dm.X * (y + dm.Y * z);
      pd[k] = okv[k] ? desc[v[k]] : 0;
      pa[k] = okv[k] ? asc[v[k]] : 0;
    }
#pragma unroll
    for (int k = 0; k < C_VPT; ++k) {
      fd[k] = okv[k] ? desc[pd[k]] : 0;
      fa[k] = okv[k] ? asc[pa[k]] : 0;
    }
#pragma unroll
    for (int k = 0; k < C_VPT; ++k) {
      const bool ok = okv[k];
      if (ok && fd[k] != pd[k]) desc[v[k]] = fd[k];
      if (ok && fa[k] != pa[k]) asc[v[k]] = fa[k];
      const uint64_t key = ok ? ((uint64_t(fa[k]) << 32) | fd[k]) : kEmpty;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (ok && (peers & ((1u << lane) - 1)) == 0)
        if (!set_insert(fset, fmask, key)) *overflow = 1;
    }
  }
}

__global__ void k_set_ids(const uint64_t* __restrict__ sorted_slots, int64_t r, uint32_t* __restrict__ slot_id) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < r) slot_id[sorted_slots[i]] = uint32_t(i);
}

__global__ void k_u64_to_u32(const uint64_t* __restrict__ in, int64_t n, uint32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = uint32_t(in[i]);
}

__global__ void k_u32_to_u64(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out,
                             uint64_t* __restrict__ vals) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    out[i] = in[i];
    vals[i] = 0;
  }
}

// ---------------------------------------------------------------- pass D --
// D1: ms[v] = dense id of the final pair (hash value slot), warp-deduped
// lookups, 4 vertices per thread per step.
__global__ void __launch_bounds__(256) k_assign_ms(uint32_t n, const uint32_t* __restrict__ desc,
                                                   const uint32_t* __restrict__ asc,
                                                   const unsigned long long* __restrict__ fset, uint64_t fmask,
                                                   const uint32_t* __restrict__ slot_id, uint32_t* __restrict__ ms) {
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x * C_VPT;
  for (uint32_t base = blockIdx.x * blockDim.x * C_VPT; base < n; base += stride) {
    uint64_t key[C_VPT];
#pragma unroll
    for (int k = 0; k < C_VPT; ++k) {
      const uint32_t v = base + k * blockDim.x + threadIdx.x;
      key[k] = v < n ? ((uint64_t(__ldg(asc + v)) << 32) | __ldg(desc + v)) : kEmpty;
    }
#pragma unroll
    for (int k = 0; k < C_VPT; ++k) {
      const uint32_t v = base + k * blockDim.x + threadIdx.x;
      const unsigned peers = __match_any_sync(0xffffffffu, key[k]);
      const int leader = __ffs(peers) - 1;
      uint32_t id = 0;
      if (lane == leader && key[k] != kEmpty) id = __ldg(slot_id + set_find(fset, fmask, key[k]));
      id = __shfl_sync(0xffffffffu, id, leader);
      if (v < n) ms[v] = id;
    }
  }
}

// D2: ordered single-pass marching over row slabs in the reference cell
// order (cube-major, x fastest): ms rows of the slab plus the +y row and +z
// layer staged in shared memory, 6 tet codes per cube, block scan, decoupled
// look-back across slabs for the output offset, records in reference order.
constexpr int D_THREADS = 512;
constexpr int D_CUBES = 8192;  // cubes per row-slab tile (target)

__constant__ uint32_t c_rows[PLMSS_TET_ROWS];
__constant__ uint16_t c_cases[32];

struct DDims {
  uint32_t X, Y, Z, XY, n;
  uint32_t ty;      // rows per slab
  uint32_t nyb;     // slabs per z layer
  uint32_t ntiles;  // Z * nyb
};

__device__ __forceinline__ int tet_code(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  const int l1 = b == a ? 0 : 1;
  const int l2 = c == a ? 0 : (c == b ? l1 : 2);
  const int l3 = d == a ? 0 : (d == b ? l1 : (d == c ? l2 : 3));
  return (l1 << 4) | (l2 << 2) | l3;
}

constexpr uint64_t FLAG_A = uint64_t(1) << 62, FLAG_P = uint64_t(2) << 62, VAL_MASK = (uint64_t(1) << 62) - 1;

__device__ __forceinline__ uint32_t pick4(int i, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return i == 0 ? a : (i == 1 ? b : (i == 2 ? c : d));
}

__device__ __forceinline__ int case_count6(uint32_t code6, const uint16_t* cases) {
  return (cases[code6 & 31] & 15) + (cases[(code6 >> 5) & 31] & 15) + (cases[(code6 >> 10) & 31] & 15) +
         (cases[(code6 >> 15) & 31] & 15) + (cases[(code6 >> 20) & 31] & 15) + (cases[(code6 >> 25) & 31] & 15);
}

// Cubes are processed in 32-cube chunks (lane i <-> cube 32*chunk + i), so
// consecutive lanes touch consecutive shared-memory words (no bank
// conflicts) and a warp's records land in one contiguous output range.
constexpr int D_CHUNKS = D_CUBES / 32;

__global__ void __launch_bounds__(D_THREADS, 2)
    k_march(DDims d, const uint32_t* __restrict__ ms, unsigned long long* __restrict__ tile_state,
            unsigned int* __restrict__ ticket, plmss_tri* __restrict__ out, uint64_t out_cap, float inv_cx,
            uint32_t ms_words) {
  extern __shared__ uint32_t dsm[];
  uint32_t* s_ms = dsm;                 // (ty + 1) rows x 2 layers x X
  uint32_t* s_code = dsm + ms_words;    // packed 6 x 5-bit tet codes per cube
  __shared__ uint32_t s_rows[PLMSS_TET_ROWS];
  __shared__ uint16_t s_cases[32];
  __shared__ uint32_t s_chunk[D_CHUNKS];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_excl;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  if (threadIdx.x < PLMSS_TET_ROWS) s_rows[threadIdx.x] = c_rows[threadIdx.x];
  if (threadIdx.x < 32) s_cases[threadIdx.x] = c_cases[threadIdx.x];
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t z = tile / d.nyb, yb = tile % d.nyb;
  const uint32_t y0 = yb * d.ty, y1 = min(d.Y, y0 + d.ty);
  const uint32_t rows = min(d.Y, y1 + 1) - y0;  // rows staged (incl. the +1 halo row)
  const bool has_cubes = z + 1 < d.Z && y0 + 1 < d.Y;
  const uint32_t X = d.X, CX = d.X - 1;

  // Stage the slab: two contiguous runs (layer z rows y0.., layer z+1 rows
  // y0..). With 16-byte alignment they go through the bulk-copy (TMA) engine
  // on an mbarrier; otherwise an unrolled vector-free loop.
  __shared__ __align__(8) uint64_t s_bar;
  if (has_cubes) {
    const uint32_t rx = rows * X;
    const uint32_t* src0 = ms + uint64_t(X) * (y0 + uint64_t(d.Y) * z);
    const uint32_t* src1 = src0 + d.XY;
    const bool bulk = ((reinterpret_cast<uintptr_t>(src0) | reinterpret_cast<uintptr_t>(src1)) & 15) == 0 &&
                      (rx & 3) == 0;
    if (bulk) {
      const uint32_t bar = smem_u32(&s_bar);
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rx * 8) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(s_ms)),
            "l"(src0), "r"(rx * 4), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(s_ms + rx)),
            "l"(src1), "r"(rx * 4), "r"(bar)
            : "memory");
      }
      asm volatile(
          "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(
              bar)
          : "memory");
    } else {
      const uint32_t nload = 2 * rx;
      for (uint32_t i0 = 0; i0 < nload; i0 += 8 * D_THREADS) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t i = i0 + k * D_THREADS + threadIdx.x;
          v[k] = i < nload ? __ldg(i < rx ? src0 + i : src1 + (i - rx)) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t i = i0 + k * D_THREADS + threadIdx.x;
          if (i < nload) s_ms[i] = v[k];
        }
      }
    }
  }
  __syncthreads();

  const uint32_t cy1 = min(y1, d.Y - 1);
  const uint32_t ncubes = has_cubes ? CX * (cy1 - y0) : 0;
  const uint32_t nchunks = (ncubes + 31) / 32;
  const uint32_t LZ = rows * X;
  // phase 2: codes and per-chunk counts
  for (uint32_t ch = w; ch < nchunks; ch += D_THREADS / 32) {
    const uint32_t q = ch * 32 + lane;
    uint32_t code6 = 0;
    int cnt = 0;
    if (q < ncubes) {
      const uint32_t cr = uint32_t((float(q) + 0.5f) * inv_cx), cx = q - cr * CX;
      const uint32_t b = cx + X * cr;
      const uint32_t l0 = s_ms[b], l1 = s_ms[b + 1], l2 = s_ms[b + X], l3 = s_ms[b + X + 1];
      const uint32_t l4 = s_ms[b + LZ], l5 = s_ms[b + LZ + 1], l6 = s_ms[b + LZ + X], l7 = s_ms[b + LZ + X + 1];
      if (!(l0 == l7 && l1 == l7 && l2 == l7 && l3 == l7 && l4 == l7 && l5 == l7 && l6 == l7)) {
        code6 = uint32_t(tet_code(l0, l1, l3, l7)) | uint32_t(tet_code(l0, l1, l5, l7)) << 5 |
                uint32_t(tet_code(l0, l2, l3, l7)) << 10 | uint32_t(tet_code(l0, l2, l6, l7)) << 15 |
                uint32_t(tet_code(l0, l4, l5, l7)) << 20 | uint32_t(tet_code(l0, l4, l6, l7)) << 25;
        cnt = case_count6(code6, s_cases);
      }
      s_code[q] = code6;
    }
    const uint32_t tot = __reduce_add_sync(0xffffffffu, uint32_t(cnt));
    if (lane == 0) s_chunk[ch] = tot;
  }
  __syncthreads();
  // chunk offsets (warp 0) + decoupled look-back across slabs
  if (w == 0) {
    constexpr int PER = D_CHUNKS / 32;
    uint32_t v[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint32_t ch = lane * PER + k;
      v[k] = ch < nchunks ? s_chunk[ch] : 0;
      sum += v[k];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint32_t ch = lane * PER + k;
      if (ch < nchunks) s_chunk[ch] = run;
      run += v[k];
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    // tile 0 always publishes a prefix, so a window reaching it stops there
    if (lane == 0) {
      if (tile == 0) {
        atomicExch(tile_state, FLAG_P | uint64_t(total));
        s_excl = 0;
      } else {
        atomicExch(tile_state + tile, FLAG_A | uint64_t(total));
      }
    }
    if (tile != 0) {
      uint64_t excl = 0;
      int64_t j = int64_t(tile) - 1;
      for (;;) {
        const int64_t jj = j - lane;
        uint64_t st = 0;
        if (jj >= 0) {
          do {
            st = *((volatile unsigned long long*)(tile_state + jj));
          } while ((st >> 62) == 0);
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int stop = pmask ? __ffs(pmask) - 1 : 32;
        uint64_t vv = (lane <= stop && jj >= 0) ? (st & VAL_MASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vv += __shfl_xor_sync(0xffffffffu, vv, o);
        excl += vv;
        if (pmask) break;
        j -= 32;
      }
      if (lane == 0) {
        atomicExch(tile_state + tile, FLAG_P | (excl + total));
        s_excl = excl;
      }
    }
  }
  __syncthreads();
  // phase 3: emission in reference order
  const uint64_t cell_base = 6ull * (uint64_t(CX) * (uint64_t(y0) + uint64_t(d.Y - 1) * z));
  const uint64_t tile_base = s_excl;
  for (uint32_t ch = w; ch < nchunks; ch += D_THREADS / 32) {
    const uint32_t q = ch * 32 + lane;
    const uint32_t code6 = q < ncubes ? s_code[q] : 0;
    const uint32_t cnt = code6 ? uint32_t(case_count6(code6, s_cases)) : 0u;
    if (!__any_sync(0xffffffffu, cnt != 0)) continue;
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (!cnt) continue;
    uint64_t pos = tile_base + s_chunk[ch] + (inc - cnt);
    const uint32_t cr = uint32_t((float(q) + 0.5f) * inv_cx), cx = q - cr * CX;
    const uint32_t b = cx + X * cr;
    const uint32_t l0 = s_ms[b], l1 = s_ms[b + 1], l2 = s_ms[b + X], l3 = s_ms[b + X + 1];
    const uint32_t l4 = s_ms[b + LZ], l5 = s_ms[b + LZ + 1], l6 = s_ms[b + LZ + X], l7 = s_ms[b + LZ + X + 1];
    const uint64_t cube_cell = cell_base + 6ull * q;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const uint32_t vb = t < 2 ? l1 : (t < 4 ? l2 : l4);
      const uint32_t vc = (t == 0 || t == 2) ? l3 : ((t == 1 || t == 4) ? l5 : l6);
      const uint32_t cs = s_cases[(code6 >> (5 * t)) & 31];
      const int n = cs & 15;
      const int first = cs >> 4;
      for (int r = 0; r < n; ++r) {
        const uint32_t row = s_rows[first + r];
        const uint32_t la = pick4((row >> 12) & 3, l0, vb, vc, l7);
        const uint32_t lb = pick4((row >> 14) & 3, l0, vb, vc, l7);
        if (pos < out_cap) {
          const uint64_t cr64 = ((cube_cell + t) << 6) | uint64_t(first + r);
          uint4 rec;
          rec.x = uint32_t(cr64);
          rec.y = uint32_t(cr64 >> 32);
          rec.z = min(la, lb);
          rec.w = max(la, lb);
          *reinterpret_cast<uint4*>(out + pos) = rec;
        }
        ++pos;
      }
    }
  }
}

__global__ void k_read_total(const unsigned long long* __restrict__ tile_state, uint32_t last,
                             unsigned long long* __restrict__ out) {
  *out = tile_state[last] & VAL_MASK;
}

bool g_consts_ready[64] = {};

}  // namespace

// Host driver of the fused pipeline. Returns false when the dims are outside
// the fused path's envelope (then the caller uses the staged kernels).
bool fused_supported(const Grid& g) { return g.X - 1 <= D_CUBES && g.n < (int64_t(1) << 32) - 1; }

FusedOut fused_pipeline(Ctx& c, const Grid& g, const float* field, uint32_t* desc, uint32_t* asc, uint32_t* ms) {
  FusedOut o{};
  for (auto& s : c.stats) s = 0;
  if (c.device >= 0 && c.device < 64 && !g_consts_ready[c.device]) {
    CK(cudaMemcpyToSymbol(c_rows, kTetRowsPacked, sizeof(kTetRowsPacked)));
    CK(cudaMemcpyToSymbol(c_cases, kTetCasePacked, sizeof(kTetCasePacked)));
    CK(cudaFuncSetAttribute(k_march, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_tile_segment, cudaFuncAttributeMaxDynamicSharedMemorySize, kASmem));
    g_consts_ready[c.device] = true;
  }
  FDims d;
  d.X = uint32_t(g.X);
  d.Y = uint32_t(g.Y);
  d.Z = uint32_t(g.Z);
  d.XY = d.X * d.Y;
  d.n = uint32_t(g.n);
  d.tx = uint32_t((g.X + TX - 1) / TX);
  d.ty = uint32_t((g.Y + TY - 1) / TY);
  d.tz = uint32_t((g.Z + TZ - 1) / TZ);
  const uint64_t ntiles = uint64_t(d.tx) * d.ty * d.tz;

  // Device counters: [0, 64) ACounters, int flag at +128, ticket at +160,
  // triangle total at +192 (bytes).
  char* ctr_base = static_cast<char*>(c.get(S_FLAGS, 256));
  ACounters* ctr = reinterpret_cast<ACounters*>(ctr_base);
  int* flag = reinterpret_cast<int*>(ctr_base + 128);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(ctr_base + 160);
  unsigned long long* tot = reinterpret_cast<unsigned long long*>(ctr_base + 192);
  for (int attempt = 0;; ++attempt) {
    const uint64_t ext_cap = c.fused_ext_cap ? c.fused_ext_cap : uint64_t(g.n / 4 + 1024);
    uint32_t* maxima = c.get_t<uint32_t>(S_MAXIMA, ext_cap);
    uint32_t* minima = c.get_t<uint32_t>(S_MINIMA, ext_cap);
    const uint64_t exit_cap = c.fused_exit_cap ? c.fused_exit_cap : uint64_t(g.n / 4 + 1024);
    uint32_t* E = c.get_t<uint32_t>(S_TMP0, exit_cap);
    CK(cudaMemsetAsync(ctr, 0, sizeof(ACounters), c.stream));
    CK(cudaMemsetAsync(&ctr->bad, 0xff, 4, c.stream));
    c.mark(0);
    k_tile_segment<<<unsigned(ntiles), A_THREADS, kASmem, c.stream>>>(field, d, desc, asc, maxima, minima, ext_cap, E,
                                                                  exit_cap, ctr);
    CK_LAUNCH("k_tile_segment");
    c.mark(1);
    ACounters h;
    CK(cudaMemcpyAsync(c.h_pinned, ctr, sizeof(ACounters), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    memcpy(&h, c.h_pinned, sizeof h);
    if (h.bad != 0xffffffffu)
      fail(PLMSS_ERR_INVALID_ARGUMENT, "non-finite scalar value at vertex " + std::to_string(h.bad));
    bool retry = false;
    if (h.n_exit > exit_cap) {
      c.fused_exit_cap = h.n_exit + h.n_exit / 4 + 1024;
      retry = true;
    }
    if (h.n_max > ext_cap || h.n_min > ext_cap) {
      c.fused_ext_cap = std::max(h.n_max, h.n_min) + 1024;
      retry = true;
    }
    if (retry) {
      if (attempt > 6) fail(PLMSS_ERR_LOGIC, "fused pipeline capacity retries exhausted");
      continue;
    }
    c.stats[0] = int64_t(h.n_exit);
    c.stats[1] = attempt;
    o.n_max = int64_t(h.n_max);
    o.n_min = int64_t(h.n_min);
    // ---- B: exit graph to the fixpoint
    o.sweeps = 0;
    if (h.n_exit) {
      for (;;) {
        CK(cudaMemsetAsync(flag, 0, 4, c.stream));
        k_exit_jump<<<blocks_for(h.n_exit, 256), 256, 0, c.stream>>>(E, h.n_exit, desc, asc, flag);
        CK_LAUNCH("k_exit_jump");
        ++o.sweeps;
        CK(cudaMemcpyAsync(c.h_pinned, flag, 4, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (*reinterpret_cast<int*>(c.h_pinned) == 0) break;
        if (o.sweeps > 64) fail(PLMSS_ERR_LOGIC, "exit graph did not converge");
      }
    }
    c.mark(2);
    // ---- extrema lists sorted ascending
    for (int dir = 0; dir < 2; ++dir) {
      uint32_t* list = dir ? minima : maxima;
      const int64_t k = dir ? o.n_min : o.n_max;
      if (k > 1) {
        uint64_t* kk = c.get_t<uint64_t>(S_SORT_A, k);
        uint64_t* vv = c.get_t<uint64_t>(S_SORT_B, k);
        k_u32_to_u64<<<blocks_for(k, 256), 256, 0, c.stream>>>(list, k, kk, vv);
        CK_LAUNCH("k_u32_to_u64");
        int bits = 0;
        while ((uint64_t(1) << bits) < uint64_t(g.n)) ++bits;
        radix_sort_pairs(c, kk, vv, k, bits);
        k_u64_to_u32<<<blocks_for(k, 256), 256, 0, c.stream>>>(kk, k, list);
        CK_LAUNCH("k_u64_to_u32");
      }
    }
    c.mark(3);
    // ---- C: final pairs of all vertices -> unique, sorted -> dense ids
    uint64_t fcap = 1024;
    {
      const uint64_t want = c.fused_pair_hint ? c.fused_pair_hint * 2 : uint64_t(1) << 20;
      while (fcap < want) fcap <<= 1;
    }
    unsigned long long* fset = nullptr;
    for (int tries = 0;; ++tries) {
      fset = c.get_t<unsigned long long>(S_HASH_V, fcap);
      CK(cudaMemsetAsync(fset, 0xff, fcap * 8, c.stream));
      CK(cudaMemsetAsync(flag, 0, 4, c.stream));
      k_mark_pairs<<<unsigned(std::min<int64_t>((g.n + 1023) / 1024, int64_t(c.sm_count) * 16)), 256, 0,
                     c.stream>>>(d, desc, asc, fset, fcap - 1, flag);
      CK_LAUNCH("k_mark_pairs");
      CK(cudaMemcpyAsync(c.h_pinned, flag, 4, cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      if (*reinterpret_cast<int*>(c.h_pinned) == 0) break;
      if (fcap >= 4 * uint64_t(g.n) || tries > 8) fail(PLMSS_ERR_LOGIC, "region set overflow");
      fcap <<= 2;
    }
    const int64_t fb = int64_t((fcap + kCTile - 1) / kCTile);
    uint64_t* fcounts = c.get_t<uint64_t>(S_TMP2, fb);
    k_count_occ<<<unsigned(fb), kCThreads, 0, c.stream>>>(fset, fcap, fcounts);
    CK_LAUNCH("k_count_occ");
    const int64_t R = int64_t(exclusive_scan_u64(c, fcounts, fb, true));
    c.fused_pair_hint = uint64_t(R);
    uint64_t* keys = c.get_t<uint64_t>(S_KEYS, R);
    uint64_t* slots = c.get_t<uint64_t>(S_SORT_B, R);
    k_write_occ<<<unsigned(fb), kCThreads, 0, c.stream>>>(fset, fcap, fcounts, keys, slots);
    CK_LAUNCH("k_write_occ");
    int kb = 32;
    while ((uint64_t(1) << (kb - 32)) < uint64_t(g.n)) ++kb;
    radix_sort_pairs(c, keys, slots, R, kb);
    uint32_t* slot_id = c.get_t<uint32_t>(S_BITMAP, fcap);
    k_set_ids<<<blocks_for(R, 256), 256, 0, c.stream>>>(slots, R, slot_id);
    CK_LAUNCH("k_set_ids");
    o.n_regions = R;
    c.stats[2] = int64_t(fcap);
    // ---- D1: dense MS ids per vertex
    k_assign_ms<<<unsigned(std::min<int64_t>((g.n + 1023) / 1024, int64_t(c.sm_count) * 16)), 256, 0, c.stream>>>(
        d.n, desc, asc, fset, fcap - 1, slot_id, ms);
    CK_LAUNCH("k_assign_ms");
    c.mark(4);
    // ---- D2: ordered marching
    DDims dd;
    dd.X = d.X;
    dd.Y = d.Y;
    dd.Z = d.Z;
    dd.XY = d.XY;
    dd.n = d.n;
    dd.ty = std::max<uint32_t>(1, uint32_t(D_CUBES / std::max<int64_t>(1, g.X - 1)));
    dd.ty = std::min<uint32_t>(dd.ty, d.Y);
    dd.nyb = (d.Y + dd.ty - 1) / dd.ty;
    dd.ntiles = dd.nyb * d.Z;
    const uint32_t ms_words = (dd.ty + 1) * 2 * d.X;
    const size_t smem = size_t(ms_words + D_CUBES) * sizeof(uint32_t);
    if (smem > 200 * 1024) fail(PLMSS_ERR_LOGIC, "row slab exceeds shared memory");
    auto* tstate = c.get_t<unsigned long long>(S_SCAN_C, dd.ntiles + 1);
    for (int pass = 0;; ++pass) {
      const uint64_t cap = c.fused_tri_cap ? c.fused_tri_cap : uint64_t(g.n / 2 + 1024);
      plmss_tri* tris = c.get_t<plmss_tri>(S_TRIS, cap);
      CK(cudaMemsetAsync(tstate, 0, (dd.ntiles + 1) * 8, c.stream));
      CK(cudaMemsetAsync(ticket, 0, 4, c.stream));
      k_march<<<dd.ntiles, D_THREADS, smem, c.stream>>>(dd, ms, tstate, ticket, tris, cap,
                                                        1.0f / float(std::max<int64_t>(1, g.X - 1)), ms_words);
      CK_LAUNCH("k_march");
      k_read_total<<<1, 1, 0, c.stream>>>(tstate, dd.ntiles - 1, tot);
      CK_LAUNCH("k_read_total");
      CK(cudaMemcpyAsync(c.h_pinned, tot, 8, cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      const uint64_t T = c.h_pinned[0];
      if (T > cap) {
        c.fused_tri_cap = T + T / 20 + 1024;
        if (pass > 2) fail(PLMSS_ERR_LOGIC, "separator capacity retries exhausted");
        ++c.stats[3];
        continue;  // re-run D2 only
      }
      o.n_tris = int64_t(T);
      o.tris = tris;
      break;
    }
    c.mark(5);
    o.maxima = maxima;
    o.minima = minima;
    o.keys = keys;
    return o;
  }
}

}  // namespace plmss_b200
