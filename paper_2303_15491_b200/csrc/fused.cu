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

#include <cuda.h>

#include "common.cuh"
#include "tet_tables.h"

namespace plmss_b200 {

namespace {

constexpr int TX = 32, TY = 32, TZ = 32;
// Halo brick in shared memory: x from gx0-4 (the TMA start coordinate in x
// must be 16-byte aligned on this platform, tools/tma_probe2.cu) to gx0+35,
// y and z from g0-1 to g0+32.
constexpr int HX = TX + 8, HY = TY + 2, HZ = TZ + 2;
constexpr int HXO = 4;            // x offset of the brick inside the halo box
constexpr int HN = HX * HY * HZ;  // 46240
constexpr int TN = TX * TY * TZ;  // 32768
constexpr int A_THREADS = 1024;
constexpr int kASmem = 4 * HN + TN + 1024;  // f (later the two u16 pointer arrays), hop codes, alignment slack
static_assert(2 * 2 * TN <= 4 * HN, "pointer arrays must fit in the f region");
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
// One CTA (1024 threads, one per (x, y) column of 32 vertices) per 32^3
// brick. The halo'd brick of f (36 x 34 x 34, x padded to a 16-byte multiple)
// arrives by one TMA tensor copy whose out-of-volume elements are NaN
// (fmaxf/fminf ignore NaN and NaN == x is false, so a missing neighbour is
// never selected). Phase 1 stores each vertex's steepest up/down stencil code
// (4 bits each) — f is then dead and its shared memory becomes the two u16
// pointer arrays of phase 2, where a vertex points at its in-brick hop target
// or at itself when it is a root or its hop leaves the brick. Pointer jumping
// to the fixpoint leaves every vertex pointing at its terminal u; the partial
// label is u (root) or u's out-of-brick hop target (an exit vertex).
template <bool kTMA>
__global__ void __launch_bounds__(A_THREADS, 1)
    k_tile_segment(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ field, FDims d,
                   uint32_t* __restrict__ desc, uint32_t* __restrict__ asc, uint32_t* __restrict__ maxima,
                   uint32_t* __restrict__ minima, uint64_t ext_cap, uint32_t* __restrict__ exits,
                   uint64_t exit_cap, ACounters* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char a_smem_raw[];
  // TMA destinations must be 128-byte aligned: round the window up (the
  // launch reserves kASmemAlign extra bytes for this).
  unsigned char* a_smem = a_smem_raw + ((1024u - (smem_u32(a_smem_raw) & 1023u)) & 1023u);
  float* f = reinterpret_cast<float*>(a_smem);          // HN floats (phase 1)
  uint16_t* Pd = reinterpret_cast<uint16_t*>(a_smem);   // TN (phase 2+, aliases f)
  uint16_t* Pa = Pd + TN;                               // TN
  uint8_t* hop = a_smem + 4 * HN;                       // TN: up | down << 4 (15 = self)
  __shared__ __align__(8) uint64_t s_bar;

  const uint32_t bt = blockIdx.x;
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const int gx0 = int(tx * TX), gy0 = int(ty * TY), gz0 = int(tz * TZ);
  const int lane = threadIdx.x & 31;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;

  // 1. halo'd brick of f
  if (kTMA) {
    const uint32_t bar = smem_u32(&s_bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(HN * 4))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4}], [%5];" ::"r"(smem_u32(f)),
          "l"(&tmap), "r"(gx0 - HXO), "r"(gy0 - 1), "r"(gz0 - 1), "r"(bar)
          : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(
            bar)
        : "memory");
  } else {
    for (int i0 = 0; i0 < HN; i0 += 8 * A_THREADS) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * A_THREADS + int(threadIdx.x);
        const int hx = i % HX, hy = (i / HX) % HY, hz = i / (HX * HY);
        const int gx = gx0 + hx - HXO, gy = gy0 + hy - 1, gz = gz0 + hz - 1;
        v[k] = __int_as_float(0x7fc00000);
        if (i < HN && gx >= 0 && gx < int(d.X) && gy >= 0 && gy < int(d.Y) && gz >= 0 && gz < int(d.Z))
          v[k] = __ldg(field + (uint32_t(gx) + d.X * (uint32_t(gy) + d.Y * uint32_t(gz))));
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * A_THREADS + int(threadIdx.x);
        if (i < HN) f[i] = v[k];
      }
    }
  }
  __syncthreads();

  // 2. steepest hops. Stencil s = 0..13 in ascending id-delta order
  //    (complex.cpp:78-88); the vertex itself sits between s = 6 and s = 7.
  //    With M = max f over the neighbours, steepest-up under (f, id) order is
  //    the highest s with f == M when M > f(v), or when M == f(v) and s > 6;
  //    otherwise v. Steepest-down mirrors it (lowest s, s < 7).
  constexpr uint32_t kOff[14] = {0x00, 0x01, 0x04, 0x05, 0x10, 0x11, 0x14,
                                 0x16, 0x19, 0x1a, 0x25, 0x26, 0x29, 0x2a};
  const int gx = gx0 + lx, gy = gy0 + ly;
  const bool col_ok = gx < int(d.X) && gy < int(d.Y);
#pragma unroll 1
  for (int lz = 0; lz < TZ; ++lz) {
    const int l = lx + TX * ly + TX * TY * lz;
    const int gz = gz0 + lz;
    if (!col_ok || gz >= int(d.Z)) {
      hop[l] = 0xff;
      continue;
    }
    const int h = (lz + 1) * HX * HY + (ly + 1) * HX + (lx + HXO);
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
    uint32_t su = 15, sd = 15;
#pragma unroll
    for (int s = 0; s < 14; ++s) su = fn[s] == M ? uint32_t(s) : su;  // highest s attaining M
#pragma unroll
    for (int s = 13; s >= 0; --s) sd = fn[s] == m ? uint32_t(s) : sd;  // lowest s attaining m
    if (!(M > fv || (M == fv && su > 6))) su = 15;
    if (!(m < fv || (m == fv && sd < 7))) sd = 15;
    hop[l] = uint8_t(su | (sd << 4));
  }
  __syncthreads();

  // 3. pointers (f is dead from here on)
  auto target = [&](int l, uint32_t s) -> int {  // in-brick hop target or l itself
    if (s == 15) return l;
    const uint32_t o = kOffTable(int(s));
    const int dx = int(o & 3) - 1, dy = int((o >> 2) & 3) - 1, dz = int((o >> 4) & 3) - 1;
    const int mx = (l & 31) + dx, my = ((l >> 5) & 31) + dy, mz = (l >> 10) + dz;
    const bool inside = mx >= 0 && mx < TX && my >= 0 && my < TY && mz >= 0 && mz < TZ;
    return inside ? l + dx + TX * dy + TX * TY * dz : l;
  };
#pragma unroll 4
  for (int lz = 0; lz < TZ; ++lz) {
    const int l = lx + TX * ly + TX * TY * lz;
    const uint32_t c = hop[l];
    Pd[l] = uint16_t(target(l, c & 15));
    Pa[l] = uint16_t(target(l, c >> 4));
  }
  __syncthreads();
  for (;;) {
    bool changed = false;
#pragma unroll 8
    for (int lz = 0; lz < TZ; ++lz) {
      const int l = lx + TX * ly + TX * TY * lz;
      const uint16_t p = Pd[l], q = Pd[p];
      if (q != p) {
        Pd[l] = q;
        changed = true;
      }
      const uint16_t pa = Pa[l], qa = Pa[pa];
      if (qa != pa) {
        Pa[l] = qa;
        changed = true;
      }
    }
    if (!__syncthreads_or(changed)) break;
  }

  // 4. partial labels, roots, exit vertices
  const uint32_t base_g = uint32_t(gx0) + d.X * (uint32_t(gy0) + d.Y * uint32_t(gz0));
  auto gid = [&](int u) -> uint32_t { return base_g + uint32_t(u & 31) + d.X * (uint32_t((u >> 5) & 31) + d.Y * uint32_t(u >> 10)); };
  auto gdelta = [&](uint32_t s) -> int {
    const uint32_t o = kOffTable(int(s));
    return (int(o & 3) - 1) + int(d.X) * (int((o >> 2) & 3) - 1) + int(d.XY) * (int((o >> 4) & 3) - 1);
  };
  auto append = [&](bool hit, uint32_t value, unsigned long long* counter, uint32_t* list, uint64_t cap) {
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (!m) return;
    unsigned long long b0 = 0;
    const int leader = __ffs(m) - 1;
    if (lane == leader) b0 = atomicAdd(counter, (unsigned long long)__popc(m));
    b0 = __shfl_sync(0xffffffffu, b0, leader);
    const uint64_t pos = b0 + __popc(m & ((1u << lane) - 1));
    if (hit && pos < cap) list[pos] = value;
  };
#pragma unroll 1
  for (int lz = 0; lz < TZ; ++lz) {
    const int l = lx + TX * ly + TX * TY * lz;
    const uint32_t c = hop[l];
    const bool valid = c != 0xff;
    const uint32_t gv = gid(l);
    uint32_t ld = 0, la = 0;
    bool xd = false, xa = false;
    uint32_t ed = 0, ea = 0;
    if (valid) {
      const int ud = Pd[l], ua = Pa[l];
      const uint32_t cd = hop[ud] & 15, ca = hop[ua] >> 4;
      ld = gid(ud) + (cd == 15 ? 0 : uint32_t(gdelta(cd)));
      la = gid(ua) + (ca == 15 ? 0 : uint32_t(gdelta(ca)));
      desc[gv] = ld;
      asc[gv] = la;
      // this vertex's own hop leaves the brick -> its target is an exit vertex
      const uint32_t sd = c & 15, sa = c >> 4;
      xd = sd != 15 && target(l, sd) == l;
      xa = sa != 15 && target(l, sa) == l;
      if (xd) ed = gv + uint32_t(gdelta(sd));
      if (xa) ea = gv + uint32_t(gdelta(sa));
    }
    append(valid && (c & 15) == 15, gv, &ctr->n_max, maxima, ext_cap);
    append(valid && (c >> 4) == 15, gv, &ctr->n_min, minima, ext_cap);
    append(xd, ed, &ctr->n_exit, exits, exit_cap);
    append(xa && !(xd && ea == ed), ea, &ctr->n_exit, exits, exit_cap);
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
    // Warp-cooperative emission: the chunk's T records are dealt out one per
    // lane, so every store instruction writes 32 consecutive records.
    const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
    const uint64_t chunk_base = tile_base + s_chunk[ch];
    const uint32_t cr = uint32_t((float(q) + 0.5f) * inv_cx), cx = q - cr * CX;
    const uint32_t bq = cx + X * cr;  // cube base index in the staged slab
    for (uint32_t j0 = 0; j0 < T; j0 += 32) {
      const uint32_t j = j0 + lane;
      // lane owning record j = number of lanes whose inclusive count is <= j
      // (binary search over the warp's nondecreasing prefix via shuffles)
      int src = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, inc, src + step - 1);
        if (v <= j) src += step;
      }
      const uint32_t c6 = __shfl_sync(0xffffffffu, code6, src & 31);
      const uint32_t ex = __shfl_sync(0xffffffffu, inc - cnt, src & 31);
      const uint32_t b = __shfl_sync(0xffffffffu, bq, src & 31);
      if (j >= T) continue;
      uint32_t k = j - ex;
      int t = 0;
      uint32_t cs = s_cases[c6 & 31];
#pragma unroll
      for (int tt = 0; tt < 5; ++tt) {
        if (k < (cs & 15)) break;
        k -= cs & 15;
        ++t;
        cs = s_cases[(c6 >> (5 * t)) & 31];
      }
      const uint32_t rowi = (cs >> 4) + k;
      const uint32_t row = s_rows[rowi];
      // tet t = cube corners {0, cb, cc, 7}; corner c -> slab offset
      const uint32_t cb = (0x442211u >> (4 * t)) & 15, cc = (0x656353u >> (4 * t)) & 15;
      auto corner = [&](uint32_t p) { return p == 0 ? 0u : (p == 1 ? cb : (p == 2 ? cc : 7u)); };
      auto off = [&](uint32_t c) { return (c & 1) + X * ((c >> 1) & 1) + LZ * (c >> 2); };
      const uint32_t la = s_ms[b + off(corner((row >> 12) & 3))];
      const uint32_t lb = s_ms[b + off(corner((row >> 14) & 3))];
      const uint64_t pos = chunk_base + j;
      if (pos < out_cap) {
        const uint64_t cr64 = ((cell_base + 6ull * (ch * 32 + uint32_t(src)) + t) << 6) | uint64_t(rowi);
        uint4 rec;
        rec.x = uint32_t(cr64);
        rec.y = uint32_t(cr64 >> 32);
        rec.z = min(la, lb);
        rec.w = max(la, lb);
        *reinterpret_cast<uint4*>(out + pos) = rec;
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
    CK(cudaFuncSetAttribute(k_tile_segment<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kASmem));
    CK(cudaFuncSetAttribute(k_tile_segment<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kASmem));
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

  // TMA descriptor of the field (3-D, float32, NaN out-of-bounds fill). The
  // global row pitch must be a 16-byte multiple, i.e. X % 4 == 0; otherwise
  // the brick is staged by an unrolled load loop.
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  bool use_tma = (g.X % 4) == 0 && (reinterpret_cast<uintptr_t>(field) & 15) == 0 && c.use_tma;
  if (use_tma) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        encode = reinterpret_cast<EncodeFn>(fn);
    }
    const cuuint64_t gdim[3] = {cuuint64_t(g.X), cuuint64_t(g.Y), cuuint64_t(g.Z)};
    const cuuint64_t gstride[2] = {cuuint64_t(g.X) * 4, cuuint64_t(g.X) * cuuint64_t(g.Y) * 4};
    const cuuint32_t box[3] = {HX, HY, HZ};
    const cuuint32_t estride[3] = {1, 1, 1};
    use_tma = encode && encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(field), gdim, gstride,
                               box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA) == CUDA_SUCCESS;
  }
  c.stats[4] = use_tma ? 1 : 0;

  // Device counters: [0, 64) ACounters, int flag at +128, ticket at +160,
  // triangle total at +192 (bytes).
  char* ctr_base = static_cast<char*>(c.get(S_FLAGS, 1024));
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
    if (use_tma)
      k_tile_segment<true><<<unsigned(ntiles), A_THREADS, kASmem, c.stream>>>(tmap, field, d, desc, asc, maxima,
                                                                           minima, ext_cap, E, exit_cap, ctr);
    else
      k_tile_segment<false><<<unsigned(ntiles), A_THREADS, kASmem, c.stream>>>(tmap, field, d, desc, asc, maxima,
                                                                            minima, ext_cap, E, exit_cap, ctr);
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
