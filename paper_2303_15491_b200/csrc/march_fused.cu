// Pass D2 of the fused pipeline: ordered multi-label marching tetrahedra from
// the per-vertex edge-equality masks written by k_assign_ms.
//
// Cubes are processed in 32-cube chunks in the reference cell order
// (cube-major, x fastest: marching.cpp:116-133; lane i <-> cube 32*chunk+i).
//   k_march_count : chunk -> number of separator triangles. A cube is one
//                   region iff its min corner's mask is 0x7f (all 7 positive
//                   edges equal); otherwise the 6 tet codes come from 19
//                   mask bits through a 64-entry equality-pattern table.
//   exclusive scan of the chunk counts (u64) -> output offsets, exact total.
//   k_march_emit  : chunks with triangles recompute their codes and deal
//                   the records out one per lane (consecutive lanes write
//                   consecutive 16-byte records), region labels gathered
//                   from ms at the two corners each recipe row separates.
#include "common.cuh"
#include "tet_tables.h"

namespace plmss_b200 {
namespace {

__constant__ uint32_t c_mrows[PLMSS_TET_ROWS];
__constant__ uint16_t c_mcases[32];

struct MDims {
  uint32_t X, XY, CX, CY;
  uint32_t nxc;  // 32-cube chunks per cube row (a row = fixed cy, cz)
};

constexpr int M_THREADS = 256;

// Chunk ch covers cubes cx = 32*xs + lane of cube row r = cy + CY*cz, with
// (r, xs) = divmod(ch, nxc): chunk order is the reference cell order.
struct ChunkPos {
  uint64_t q0;  // cube id of lane 0
  uint32_t v0;  // min-corner vertex of lane 0's cube
  uint32_t n;   // cubes in the chunk
};

// Warps walk whole cube rows (one division per row, none per chunk).
__device__ __forceinline__ ChunkPos chunk_pos(uint32_t r, uint32_t cy, uint32_t cz, uint32_t xs,
                                              const MDims& d) {
  ChunkPos p;
  p.q0 = uint64_t(r) * d.CX + 32u * xs;
  p.v0 = 32u * xs + d.X * cy + d.XY * cz;
  p.n = min(32u, d.CX - 32u * xs);
  return p;
}

__device__ __forceinline__ void load_tables(uint16_t* s_tlut, uint16_t* s_cases, uint32_t* s_rows) {
  if (threadIdx.x < 32) s_cases[threadIdx.x] = c_mcases[threadIdx.x];
  if (s_rows && threadIdx.x < PLMSS_TET_ROWS) s_rows[threadIdx.x] = c_mrows[threadIdx.x];
  if (threadIdx.x < 64) {
    // equality pattern (b==a, c==a, c==b, d==a, d==b, d==c) of tet (a,b,c,d)
    // -> tetra_code (marching.cpp:28-44) | separator count << 5
    const uint32_t p = threadIdx.x;
    const int l1 = (p & 1) ? 0 : 1;
    const int l2 = (p & 2) ? 0 : ((p & 4) ? l1 : 2);
    const int l3 = (p & 8) ? 0 : ((p & 16) ? l1 : ((p & 32) ? l2 : 3));
    const int code = (l1 << 4) | (l2 << 2) | l3;
    s_tlut[p] = uint16_t(code | ((c_mcases[code] & 15) << 5));
  }
}

// Codes of the 6 tets of the cube at v0 (packed 5 bits each) and the count.
// Mask bit k-1 of a vertex = equal to its +k neighbour, k = dx|dy<<1|dz<<2;
// tets t = {0,1,3,7} {0,1,5,7} {0,2,3,7} {0,2,6,7} {0,4,5,7} {0,4,6,7}.
__device__ __forceinline__ uint32_t cube_codes(const uint8_t* __restrict__ emask, uint32_t v0, uint32_t X,
                                               uint32_t XY, const uint16_t* s_tlut, uint32_t& cnt) {
  const uint32_t m0 = __ldg(emask + v0);
  cnt = 0;
  if (m0 == 0x7fu) return 0;
  const uint32_t m1 = __ldg(emask + v0 + 1), m2 = __ldg(emask + v0 + X), m3 = __ldg(emask + v0 + X + 1),
                 m4 = __ldg(emask + v0 + XY), m5 = __ldg(emask + v0 + XY + 1), m6 = __ldg(emask + v0 + XY + X);
  const uint32_t e10 = m0 & 1, e20 = (m0 >> 1) & 1, e30 = (m0 >> 2) & 1, e40 = (m0 >> 3) & 1, e50 = (m0 >> 4) & 1,
                 e60 = (m0 >> 5) & 1, k7 = ((m0 >> 6) & 1) << 3;
  const uint32_t e31 = (m1 >> 1) & 1, e51 = (m1 >> 3) & 1, e71 = (m1 >> 5) & 1;
  const uint32_t e32 = m2 & 1, e62 = (m2 >> 3) & 1, e72 = (m2 >> 4) & 1;
  const uint32_t e54 = m4 & 1, e64 = (m4 >> 1) & 1, e74 = (m4 >> 2) & 1;
  const uint32_t e73 = (m3 >> 3) & 1, e75 = (m5 >> 1) & 1, e76 = m6 & 1;
  const uint32_t t0 = s_tlut[e10 | e30 << 1 | e31 << 2 | k7 | e71 << 4 | e73 << 5];
  const uint32_t t1 = s_tlut[e10 | e50 << 1 | e51 << 2 | k7 | e71 << 4 | e75 << 5];
  const uint32_t t2 = s_tlut[e20 | e30 << 1 | e32 << 2 | k7 | e72 << 4 | e73 << 5];
  const uint32_t t3 = s_tlut[e20 | e60 << 1 | e62 << 2 | k7 | e72 << 4 | e76 << 5];
  const uint32_t t4 = s_tlut[e40 | e50 << 1 | e54 << 2 | k7 | e74 << 4 | e75 << 5];
  const uint32_t t5 = s_tlut[e40 | e60 << 1 | e64 << 2 | k7 | e74 << 4 | e76 << 5];
  cnt = (t0 >> 5) + (t1 >> 5) + (t2 >> 5) + (t3 >> 5) + (t4 >> 5) + (t5 >> 5);
  return (t0 & 31) | (t1 & 31) << 5 | (t2 & 31) << 10 | (t3 & 31) << 15 | (t4 & 31) << 20 | (t5 & 31) << 25;
}

__global__ void __launch_bounds__(M_THREADS) k_march_count(MDims d, const uint8_t* __restrict__ emask,
                                                           uint64_t nchunks, uint64_t* __restrict__ counts) {
  __shared__ uint16_t s_tlut[64], s_cases[32];
  load_tables(s_tlut, s_cases, nullptr);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (M_THREADS / 32);
  const uint32_t nrows = uint32_t(nchunks / d.nxc);
  for (uint32_t r = blockIdx.x * (M_THREADS / 32) + (threadIdx.x >> 5); r < nrows; r += warps) {
    const uint32_t cz = r / d.CY, cy = r - cz * d.CY;
    for (uint32_t xs = 0; xs < d.nxc; ++xs) {
      const ChunkPos p = chunk_pos(r, cy, cz, xs, d);
      uint32_t cnt = 0;
      if (uint32_t(lane) < p.n) cube_codes(emask, p.v0 + lane, d.X, d.XY, s_tlut, cnt);
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0) counts[uint64_t(r) * d.nxc + xs] = cnt;
    }
  }
}

__global__ void __launch_bounds__(M_THREADS) k_march_emit(MDims d, const uint8_t* __restrict__ emask,
                                                          const uint32_t* __restrict__ ms, uint64_t nchunks,
                                                          const uint64_t* __restrict__ offsets, uint64_t total,
                                                          plmss_tri* __restrict__ out) {
  __shared__ uint16_t s_tlut[64], s_cases[32];
  __shared__ uint32_t s_rows[PLMSS_TET_ROWS];
  load_tables(s_tlut, s_cases, s_rows);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (M_THREADS / 32);
  const uint32_t nrows = uint32_t(nchunks / d.nxc);
  for (uint32_t r = blockIdx.x * (M_THREADS / 32) + (threadIdx.x >> 5); r < nrows; r += warps) {
   const uint32_t cz = r / d.CY, cy = r - cz * d.CY;
   for (uint32_t xs = 0; xs < d.nxc; ++xs) {
    const uint64_t ch = uint64_t(r) * d.nxc + xs;
    const uint64_t base = offsets[ch];
    const uint64_t T64 = (ch + 1 < nchunks ? offsets[ch + 1] : total) - base;
    if (T64 == 0) continue;
    const ChunkPos p = chunk_pos(r, cy, cz, xs, d);
    uint32_t cnt = 0, code6 = 0;
    const uint32_t v0 = p.v0 + lane;
    if (uint32_t(lane) < p.n) code6 = cube_codes(emask, v0, d.X, d.XY, s_tlut, cnt);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t T = uint32_t(T64);
    for (uint32_t j0 = 0; j0 < T; j0 += 32) {
      const uint32_t j = j0 + lane;
      // owning lane of record j = number of lanes whose inclusive count <= j
      int src = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t vv = __shfl_sync(0xffffffffu, inc, src + step - 1);
        if (vv <= j) src += step;
      }
      const uint32_t c6 = __shfl_sync(0xffffffffu, code6, src & 31);
      const uint32_t ex = __shfl_sync(0xffffffffu, inc - cnt, src & 31);
      const uint32_t b = __shfl_sync(0xffffffffu, v0, src & 31);
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
      // tet t = cube corners {0, cb, cc, 7}; corner c -> vertex offset
      const uint32_t cb = (0x442211u >> (4 * t)) & 15, cc = (0x656353u >> (4 * t)) & 15;
      auto corner = [&](uint32_t p) { return p == 0 ? 0u : (p == 1 ? cb : (p == 2 ? cc : 7u)); };
      auto off = [&](uint32_t c) { return (c & 1) + d.X * ((c >> 1) & 1) + d.XY * (c >> 2); };
      const uint32_t la = __ldg(ms + b + off(corner((row >> 12) & 3)));
      const uint32_t lb = __ldg(ms + b + off(corner((row >> 14) & 3)));
      const uint64_t cr64 = ((6ull * (p.q0 + uint32_t(src)) + t) << 6) | uint64_t(rowi);
      uint4 rec;
      rec.x = uint32_t(cr64);
      rec.y = uint32_t(cr64 >> 32);
      rec.z = min(la, lb);
      rec.w = max(la, lb);
      *reinterpret_cast<uint4*>(out + base + j) = rec;
    }
   }
  }
}

bool g_mconsts_ready[64] = {};

}  // namespace

int64_t fused_march(Ctx& c, const Grid& g, const uint32_t* ms, const uint8_t* emask, plmss_tri** out) {
  if (c.device >= 0 && c.device < 64 && !g_mconsts_ready[c.device]) {
    CK(cudaMemcpyToSymbol(c_mrows, kTetRowsPacked, sizeof(kTetRowsPacked)));
    CK(cudaMemcpyToSymbol(c_mcases, kTetCasePacked, sizeof(kTetCasePacked)));
    g_mconsts_ready[c.device] = true;
  }
  MDims d;
  d.X = uint32_t(g.X);
  d.XY = uint32_t(g.X * g.Y);
  d.CX = uint32_t(g.X - 1);
  d.CY = uint32_t(g.Y - 1);
  d.nxc = (d.CX + 31) / 32;
  const uint64_t nchunks = uint64_t(d.nxc) * uint64_t(g.Y - 1) * uint64_t(g.Z - 1);
  *out = nullptr;
  if (nchunks == 0) return 0;
  uint64_t* counts = c.get_t<uint64_t>(S_TMP1, nchunks);
  const uint64_t nrows = uint64_t(g.Y - 1) * uint64_t(g.Z - 1);
  const unsigned grid = unsigned(std::min<uint64_t>((nrows + 7) / 8, uint64_t(c.sm_count) * 32));
  k_march_count<<<grid, M_THREADS, 0, c.stream>>>(d, emask, nchunks, counts);
  CK_LAUNCH("k_march_count");
  const uint64_t total = exclusive_scan_u64(c, counts, int64_t(nchunks), true);
  plmss_tri* tris = c.get_t<plmss_tri>(S_TRIS, total ? total : 1);
  if (total) {
    k_march_emit<<<grid, M_THREADS, 0, c.stream>>>(d, emask, ms, nchunks, counts, total, tris);
    CK_LAUNCH("k_march_emit");
  }
  *out = tris;
  return int64_t(total);
}

}  // namespace plmss_b200
