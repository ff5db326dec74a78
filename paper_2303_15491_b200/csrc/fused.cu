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
// Field box in shared memory: x from gx0-4 (the TMA start coordinate in x
// must be 16-byte aligned on this platform, tools/tma_probe2.cu) to gx0+35,
// y and z from g0-1 to g0+32.
constexpr int HX = TX + 8, HY = TY + 2, HZ = TZ + 2;
constexpr int HXO = 4;            // x offset of the brick inside the field box
constexpr int HXY = HX * HY;
constexpr int HN = HXY * HZ;      // 46240 floats
// Pointer / hop-code index space: the brick plus a one-cell shell, 34^3
// cells (< 2^16, so pointers are u16). Shell cells are terminals: a chain
// that reaches one has left the brick, and the shell cell is the hop target.
constexpr int PX = TX + 2, PXY = PX * (TY + 2), PN = PXY * (TZ + 2);  // 34, 1156, 39304
constexpr int TN = TX * TY * TZ;
constexpr int A_THREADS = 1024;
constexpr int kCodeOff = 4 * HN;                // hop codes after the field box
constexpr int kASmem = 4 * HN + PN + 1024;      // + TMA alignment slack
static_assert(2 * 2 * PN <= 4 * HN, "pointer arrays must fit in the field box");
static_assert(kCodeOff % 16 == 0, "code array alignment");
constexpr uint8_t kExitMark = 0xfe;  // shell cell reached by some brick vertex
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

// Stencil s = 0..13 in ascending id-delta order (complex.cpp:78-88) as
// 2-bit-per-axis codes (dx+1 | (dy+1) << 2 | (dz+1) << 4); the vertex itself
// sits between s = 6 and s = 7.
__host__ __device__ constexpr uint32_t stencil_code(int s) {
  return s == 0 ? 0x00 : s == 1 ? 0x01 : s == 2 ? 0x04 : s == 3 ? 0x05 : s == 4 ? 0x10 : s == 5 ? 0x11
       : s == 6 ? 0x14 : s == 7 ? 0x16 : s == 8 ? 0x19 : s == 9 ? 0x1a : s == 10 ? 0x25 : s == 11 ? 0x26
       : s == 12 ? 0x29 : 0x2a;
}

struct ACounters {
  unsigned long long n_max, n_min, n_exit;
  int overflow;
  uint32_t bad;
};

// ---------------------------------------------------------------- pass A --
// One CTA (1024 threads, one per (x, y) column of 32 vertices) per 32^3
// brick.
//  1. The field box (40 x 34 x 34 floats) arrives by one TMA tensor copy whose
//     out-of-volume elements are NaN: fmaxf/fminf ignore NaN and NaN == x is
//     false, so a missing neighbour is never selected.
//  2. Steepest hops (segmentation.cpp:60-85). Each thread walks its column in
//     z keeping the 7 stencil columns in registers (7 shared loads per
//     vertex). With M = max f over the neighbours, steepest-up under the
//     (f, id) order is the highest s with f == M when M > f(v), or when
//     M == f(v) and s > 6; otherwise none. Steepest-down mirrors it (lowest
//     s, s < 7). Result: one byte per cell, up | down << 4 (15 = none).
//  3. f is dead; its shared memory becomes two u16 pointer arrays over the
//     34^3 shelled brick. Pointers start two hops ahead; shell cells point at
//     themselves.
//  4. Pointer jumping to the fixpoint (segmentation.cpp:87-168 restated as
//     parallel path compression): every vertex ends at its terminal, an
//     in-brick extremum or the shell cell where its chain leaves the brick.
//     The global id of that terminal is the vertex's partial label.
//  5. Extrema and the distinct exit (shell) cells are appended to global
//     lists, aggregated per brick.
template <bool kTMA>
__global__ void __launch_bounds__(A_THREADS, 1)
    k_tile_segment(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ field, FDims d,
                   uint32_t* __restrict__ desc, uint32_t* __restrict__ asc, uint32_t* __restrict__ maxima,
                   uint32_t* __restrict__ minima, uint64_t ext_cap, uint32_t* __restrict__ exits,
                   uint64_t exit_cap, ACounters* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char a_smem_raw[];
  // TMA destinations must be 128-byte aligned: round the window up (the
  // launch reserves 1024 extra bytes for this).
  unsigned char* a_smem = a_smem_raw + ((1024u - (smem_u32(a_smem_raw) & 1023u)) & 1023u);
  float* f = reinterpret_cast<float*>(a_smem);         // HN floats (steps 1-2)
  uint16_t* Pd = reinterpret_cast<uint16_t*>(a_smem);  // PN (steps 3+, aliases f)
  uint16_t* Pa = Pd + PN;                              // PN
  uint8_t* code = a_smem + kCodeOff;                   // PN
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_delta[16];
  __shared__ uint32_t s_wcnt[A_THREADS / 32][3];
  __shared__ unsigned long long s_lbase[3];

  const uint32_t bt = blockIdx.x;
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const int gx0 = int(tx * TX), gy0 = int(ty * TY), gz0 = int(tz * TZ);
  const int tid = int(threadIdx.x);
  const int lane = tid & 31;
  const int lx = tid & 31, ly = tid >> 5;

  // 1. field box
  if (kTMA) {
    const uint32_t bar = smem_u32(&s_bar);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(HN * 4))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4}], [%5];" ::"r"(smem_u32(f)),
          "l"(&tmap), "r"(gx0 - HXO), "r"(gy0 - 1), "r"(gz0 - 1), "r"(bar)
          : "memory");
    }
  } else {
    for (int i0 = 0; i0 < HN; i0 += 8 * A_THREADS) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * A_THREADS + tid;
        const int hx = i % HX, hy = (i / HX) % HY, hz = i / HXY;
        const int gx = gx0 + hx - HXO, gy = gy0 + hy - 1, gz = gz0 + hz - 1;
        v[k] = __int_as_float(0x7fc00000);
        if (i < HN && gx >= 0 && gx < int(d.X) && gy >= 0 && gy < int(d.Y) && gz >= 0 && gz < int(d.Z))
          v[k] = __ldg(field + (uint32_t(gx) + d.X * (uint32_t(gy) + d.Y * uint32_t(gz))));
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * A_THREADS + tid;
        if (i < HN) f[i] = v[k];
      }
    }
  }
  // while the box is in flight: no-hop codes everywhere (step 2 overwrites
  // the in-volume brick cells) and the stencil deltas of the pointer space
  for (int i = 4 * tid; i < PN; i += 4 * A_THREADS) *reinterpret_cast<uint32_t*>(code + i) = 0xffffffffu;
  if (tid < 16) {
    int dl = 0;
    if (tid < 14) {
      const uint32_t o = stencil_code(tid);
      dl = (int(o & 3) - 1) + PX * (int((o >> 2) & 3) - 1) + PXY * (int((o >> 4) & 3) - 1);
    }
    s_delta[tid] = dl;  // code 15 (none) -> 0
  }
  if (kTMA)
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(&s_bar))
        : "memory");
  __syncthreads();

  // 2. steepest hops
  const int gx = gx0 + lx, gy = gy0 + ly;
  const bool col_ok = gx < int(d.X) && gy < int(d.Y);
  const int nz = min(TZ, int(d.Z) - gz0);  // in-volume layers of the brick
  const int hc = (lx + 1) + PX * (ly + 1);  // column in the pointer space (shell layer z = 0)
  const uint32_t gv0 = uint32_t(gx) + d.X * uint32_t(gy) + d.XY * uint32_t(gz0);
  if (col_ok) {
    // stencil columns (dx, dy): c0 (-1,-1) c1 (0,-1) c2 (-1,0) c3 (0,0)
    // c4 (1,0) c5 (0,1) c6 (1,1); s -> (column, plane):
    //   s0-3 = c0-c3 @ z-1, s4-6 = c0-c2 @ z, s7-9 = c4-c6 @ z, s10-13 = c3-c6 @ z+1
    const float* fc = f + (ly + 1) * HX + (lx + HXO);
    float a0m = fc[-1 - HX], a1m = fc[-HX], a2m = fc[-1], a3m = fc[0];
    float a0 = fc[HXY - 1 - HX], a1 = fc[HXY - HX], a2 = fc[HXY - 1], a3 = fc[HXY], a4 = fc[HXY + 1],
          a5 = fc[HXY + HX], a6 = fc[HXY + HX + 1];
#pragma unroll 4
    for (int lz = 0; lz < TZ; ++lz) {
      const float* p = fc + (lz + 2) * HXY;  // plane z+1
      const float a3p = p[0], a4p = p[1], a5p = p[HX], a6p = p[HX + 1];
      if (lz < nz) {
        const float fv = a3;
        if (!isfinite(fv)) atomicMin(&ctr->bad, gv0 + d.XY * uint32_t(lz));
        const float fn[14] = {a0m, a1m, a2m, a3m, a0, a1, a2, a4, a5, a6, a3p, a4p, a5p, a6p};
        float M = fn[0], m = fn[0];
#pragma unroll
        for (int s = 1; s < 14; ++s) {
          M = fmaxf(M, fn[s]);
          m = fminf(m, fn[s]);
        }
        uint32_t eu = 0, ed = 0;
#pragma unroll
        for (int s = 0; s < 14; ++s) {
          eu |= uint32_t(fn[s] == M) << s;
          ed |= uint32_t(fn[s] == m) << s;
        }
        // eu == 0 only when every neighbour is missing (M is NaN): no hop
        const uint32_t su = (M > fv || (M == fv && eu > 0x7fu)) ? uint32_t(31 - __clz(eu)) : 15u;
        const uint32_t sd = (m < fv || (m == fv && (ed & 0x7fu) != 0)) ? uint32_t(__ffs(ed) - 1) : 15u;
        code[hc + (lz + 1) * PXY] = uint8_t(su | (sd << 4));
      }
      a0m = a0;
      a1m = a1;
      a2m = a2;
      a3m = a3;
      a0 = p[-1 - HX];
      a1 = p[-HX];
      a2 = p[-1];
      a3 = a3p;
      a4 = a4p;
      a5 = a5p;
      a6 = a6p;
    }
  }
  __syncthreads();

  // 3. pointers two hops ahead (f is dead from here on). Shell cells point
  //    at themselves: the z-shell cells of this column here, the 132 shell
  //    columns by threads 0..131.
  uint32_t live_d = 0, live_a = 0;
  Pd[hc] = uint16_t(hc);
  Pa[hc] = uint16_t(hc);
  Pd[hc + (TZ + 1) * PXY] = uint16_t(hc + (TZ + 1) * PXY);
  Pa[hc + (TZ + 1) * PXY] = uint16_t(hc + (TZ + 1) * PXY);
  int shell_col = -1;
  if (tid < 4 * (PX - 1)) {  // 132 shell columns: rows y = 0, y = 33, then x = 0, x = 33
    shell_col = tid < PX ? tid : tid < 2 * PX ? (tid - PX) + PX * (PX - 1) : tid < 2 * PX + TY
                                                  ? PX * (tid - 2 * PX + 1)
                                                  : (PX - 1) + PX * (tid - 2 * PX - TY + 1);
    for (int z = 0; z < TZ + 2; ++z) {
      const int h = shell_col + z * PXY;
      Pd[h] = uint16_t(h);
      Pa[h] = uint16_t(h);
    }
  }
#pragma unroll 4
  for (int lz = 0; lz < TZ; ++lz) {
    const int h = hc + (lz + 1) * PXY;
    const uint32_t c = code[h];
    int td = h, ta = h;
    if ((c & 15) != 15) {
      const int t1 = h + s_delta[c & 15];
      const uint32_t c2 = code[t1] & 15;
      td = t1 + s_delta[c2];
      live_d |= uint32_t(c2 != 15) << lz;
    }
    if ((c >> 4) != 15) {
      const int t1 = h + s_delta[c >> 4];
      const uint32_t c2 = code[t1] >> 4;
      ta = t1 + s_delta[c2];
      live_a |= uint32_t(c2 != 15) << lz;
    }
    Pd[h] = uint16_t(td);
    Pa[h] = uint16_t(ta);
  }
  __syncthreads();

  // 4. pointer jumping; a vertex retires once its pointer is a terminal
  for (;;) {
    uint32_t m = live_d;
    while (m) {
      const int lz = __ffs(m) - 1;
      m &= m - 1;
      const int h = hc + (lz + 1) * PXY;
      const uint16_t p = Pd[h], q = Pd[p];
      if (q == p)
        live_d &= ~(1u << lz);
      else
        Pd[h] = q;
    }
    m = live_a;
    while (m) {
      const int lz = __ffs(m) - 1;
      m &= m - 1;
      const int h = hc + (lz + 1) * PXY;
      const uint16_t p = Pa[h], q = Pa[p];
      if (q == p)
        live_a &= ~(1u << lz);
      else
        Pa[h] = q;
    }
    if (!__syncthreads_or((live_d | live_a) != 0)) break;
  }

  // 5. partial labels; extrema; exit shell cells marked in the code array
  const uint32_t gbase = uint32_t(gx0 - 1) + d.X * uint32_t(gy0 - 1) + d.XY * uint32_t(gz0 - 1);
  auto gid = [&](uint32_t t, bool& shell) -> uint32_t {
    const uint32_t hz = t / PXY, r = t - hz * PXY, hy = r / PX, hx = r - hy * PX;
    shell = (hx - 1u) >= uint32_t(TX) || (hy - 1u) >= uint32_t(TY) || (hz - 1u) >= uint32_t(TZ);
    return gbase + hx + d.X * hy + d.XY * hz;
  };
  uint32_t mmax = 0, mmin = 0;
  if (col_ok) {
#pragma unroll 2
    for (int lz = 0; lz < nz; ++lz) {
      const int h = hc + (lz + 1) * PXY;
      const uint32_t c = code[h];
      const uint32_t gv = gv0 + d.XY * uint32_t(lz);
      bool sh_d, sh_a;
      const uint32_t td = Pd[h], ta = Pa[h];
      desc[gv] = gid(td, sh_d);
      asc[gv] = gid(ta, sh_a);
      if (sh_d) code[td] = kExitMark;
      if (sh_a) code[ta] = kExitMark;
      mmax |= uint32_t((c & 15) == 15) << lz;
      mmin |= uint32_t((c >> 4) == 15) << lz;
    }
  }
  __syncthreads();
  // exit cells: this column's two z-shell cells (bits 0, 1) and, for threads
  // 0..131, a whole shell column (bits 2..35)
  uint64_t mex = uint64_t(code[hc] == kExitMark) | uint64_t(code[hc + (TZ + 1) * PXY] == kExitMark) << 1;
  if (shell_col >= 0)
    for (int z = 0; z < TZ + 2; ++z) mex |= uint64_t(code[shell_col + z * PXY] == kExitMark) << (z + 2);

  uint32_t cnt[3] = {uint32_t(__popc(mmax)), uint32_t(__popc(mmin)), uint32_t(__popcll(mex))};
  uint32_t pre[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    uint32_t inc = cnt[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    pre[k] = inc - cnt[k];
    if (lane == 31) s_wcnt[tid >> 5][k] = inc;
  }
  __syncthreads();
  if (tid < 32) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t t = s_wcnt[lane][k];
      uint32_t inc = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      s_wcnt[lane][k] = inc - t;
      const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
      if (lane == 0) {
        unsigned long long* ctrk = k == 0 ? &ctr->n_max : (k == 1 ? &ctr->n_min : &ctr->n_exit);
        s_lbase[k] = total ? atomicAdd(ctrk, (unsigned long long)total) : 0ull;
      }
    }
  }
  __syncthreads();
  uint64_t pos[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) pos[k] = s_lbase[k] + s_wcnt[tid >> 5][k] + pre[k];
  uint32_t m = mmax;
  while (m) {
    const int lz = __ffs(m) - 1;
    m &= m - 1;
    if (pos[0] < ext_cap) maxima[pos[0]] = gv0 + d.XY * uint32_t(lz);
    ++pos[0];
  }
  m = mmin;
  while (m) {
    const int lz = __ffs(m) - 1;
    m &= m - 1;
    if (pos[1] < ext_cap) minima[pos[1]] = gv0 + d.XY * uint32_t(lz);
    ++pos[1];
  }
  while (mex) {
    const int b = __ffsll(mex) - 1;
    mex &= mex - 1;
    const int h = b == 0 ? hc : b == 1 ? hc + (TZ + 1) * PXY : shell_col + (b - 2) * PXY;
    bool sh;
    if (pos[2] < exit_cap) exits[pos[2]] = gid(uint32_t(h), sh);
    ++pos[2];
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
// Also writes the vertex's edge-equality mask: bit k-1 (k = 1..7, k = dx |
// dy << 1 | dz << 2) is set when the vertex and its +offset-k neighbour share
// a Morse-Smale region (equal (asc, desc) pair <=> equal dense id). Every tet
// edge is such a positive stencil edge, so a cube is one region iff its min
// corner's mask is 0x7f, and all 19 label equalities the 6 tet codes need
// are mask bits of the cube's corners 0..6.
// One block per x-row segment (blockIdx.x = segment, blockIdx.y = row
// y + Y*z), so coordinates need no division.
__global__ void __launch_bounds__(256) k_assign_ms(uint32_t X, uint32_t Y, uint32_t Z,
                                                   const uint32_t* __restrict__ desc,
                                                   const uint32_t* __restrict__ asc,
                                                   const unsigned long long* __restrict__ fset, uint64_t fmask,
                                                   const uint32_t* __restrict__ slot_id, uint32_t* __restrict__ ms,
                                                   uint8_t* __restrict__ emask) {
  const int lane = threadIdx.x & 31;
  const uint32_t XY = X * Y;
  const uint32_t nseg = (X + blockDim.x - 1) / blockDim.x;
  const uint32_t row = blockIdx.x / nseg, seg = blockIdx.x - row * nseg;
  const uint32_t y = row % Y, z = row / Y;
  const bool by = y + 1 < Y, bz = z + 1 < Z;
  const uint32_t x = seg * blockDim.x + threadIdx.x;
  const bool ok = x < X;
  const uint32_t v = row * X + x;
  const uint64_t key = ok ? ((uint64_t(__ldg(asc + v)) << 32) | __ldg(desc + v)) : kEmpty;
  // neighbour pairs first (independent loads in flight together)
  uint32_t nd[7], na[7];
  const bool bx = x + 1 < X;
#pragma unroll
  for (int o = 1; o < 8; ++o) {
    const bool in = ok && (!(o & 1) || bx) && (!(o & 2) || by) && (!(o & 4) || bz);
    const uint32_t u = v + ((o & 1) ? 1u : 0u) + ((o & 2) ? X : 0u) + ((o & 4) ? XY : 0u);
    nd[o - 1] = in ? __ldg(desc + u) : ~0u;
    na[o - 1] = in ? __ldg(asc + u) : ~0u;
  }
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int leader = __ffs(peers) - 1;
  uint32_t id = 0;
  if (lane == leader && key != kEmpty) id = __ldg(slot_id + set_find(fset, fmask, key));
  id = __shfl_sync(0xffffffffu, id, leader);
  if (!ok) return;
  ms[v] = id;
  const uint32_t kd = uint32_t(key), ka = uint32_t(key >> 32);
  uint32_t m = 0;
#pragma unroll
  for (int o = 0; o < 7; ++o) m |= uint32_t(nd[o] == kd && na[o] == ka) << o;
  emask[v] = uint8_t(m);
}

bool g_consts_ready[64] = {};

}  // namespace

// Host driver of the fused pipeline. Returns false when the dims are outside
// the fused path's envelope (then the caller uses the staged kernels).
bool fused_supported(const Grid& g) { return g.n < (int64_t(1) << 32) - 1; }

FusedOut fused_pipeline(Ctx& c, const Grid& g, const float* field, uint32_t* desc, uint32_t* asc, uint32_t* ms) {
  FusedOut o{};
  for (auto& s : c.stats) s = 0;
  if (c.device >= 0 && c.device < 64 && !g_consts_ready[c.device]) {
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

  // Device counters: [0, 64) ACounters, int flag at +128 (bytes).
  char* ctr_base = static_cast<char*>(c.get(S_FLAGS, 1024));
  ACounters* ctr = reinterpret_cast<ACounters*>(ctr_base);
  int* flag = reinterpret_cast<int*>(ctr_base + 128);
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
    uint8_t* emask = c.get_t<uint8_t>(S_MASK, g.n + 64);
    {
      const unsigned grid = unsigned((g.X + 255) / 256 * g.Y * g.Z);
      k_assign_ms<<<grid, 256, 0, c.stream>>>(d.X, d.Y, d.Z, desc, asc, fset, fcap - 1, slot_id, ms, emask);
    }
    CK_LAUNCH("k_assign_ms");
    c.mark(4);
    // ---- D2: ordered marching (count, scan, emit)
    o.n_tris = fused_march(c, g, ms, emask, &o.tris);
    c.mark(5);
    o.maxima = maxima;
    o.minima = minima;
    o.keys = keys;
    return o;
  }
}

}  // namespace plmss_b200
