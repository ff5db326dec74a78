// K4-K6: multi-label marching tetrahedra over the 6-tet Freudenthal cubes.
//
// Reference: index_separators / emit_geometry (marching.cpp:104-206),
// tetra_code (marching.cpp:28-44), recipes (marching_tables.cpp:48-127),
// cells (complex.cpp:203-218), emit_boundaries (marching.cpp:236-326).
//
// Cube corners are numbered by bits (x, y, z): corner k = v0 + (k&1) + X((k>>1)&1)
// + XY(k>>2). Tet t of the cube follows the axis permutation kTetAxisOrder[t]
// (complex.cpp:23-24), i.e. corners {0,1,3,7} {0,1,5,7} {0,2,3,7} {0,2,6,7}
// {0,4,5,7} {0,4,6,7}; cell id = 6 * cube + t with cube = cx + (X-1)(cy +
// (Y-1)cz), so thread order over cubes is the reference's cell-major order.
#include <algorithm>
#include <functional>
#include <vector>

#include <atomic>
#include <mutex>

#include "common.cuh"
#include "tet_tables.h"

namespace plmss_b200 {
namespace {

__constant__ uint32_t c_rows[PLMSS_TET_ROWS];
__constant__ uint16_t c_cases[32];
// corner index of tet vertex i of tet t
__constant__ uint8_t c_tet_corner[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7},
                                          {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

struct CDims {
  uint32_t X, Y, Z, XY;
  uint32_t CX, CY;  // cube extents in x, y
  uint64_t cubes;
};

CDims to_cdims(const Grid& g) {
  CDims d;
  d.X = uint32_t(g.X);
  d.Y = uint32_t(g.Y);
  d.Z = uint32_t(g.Z);
  d.XY = d.X * d.Y;
  d.CX = uint32_t(g.X - 1);
  d.CY = uint32_t(g.Y - 1);
  d.cubes = uint64_t(g.cubes);
  return d;
}

template <class L>
__device__ __forceinline__ int tet_code(L a, L b, L c, L d) {
  const int l1 = b == a ? 0 : 1;
  const int l2 = c == a ? 0 : (c == b ? l1 : 2);
  const int l3 = d == a ? 0 : (d == b ? l1 : (d == c ? l2 : 3));
  return (l1 << 4) | (l2 << 2) | l3;
}

__device__ __forceinline__ int case_count(int code) { return c_cases[code] & 15; }
__device__ __forceinline__ int case_first(int code) { return c_cases[code] >> 4; }

// Loads the 8 corner labels of cube q and returns the 6 tet codes packed
// 5 bits each plus the triangle count.
template <class L>
__device__ __forceinline__ void cube_codes(const L* __restrict__ lab, const CDims& d, uint64_t q, L (&cl)[8],
                                           int (&code)[6], int& count) {
  const uint32_t cx = uint32_t(q % d.CX);
  const uint64_t r = q / d.CX;
  const uint32_t cy = uint32_t(r % d.CY);
  const uint32_t cz = uint32_t(r / d.CY);
  const uint64_t v0 = uint64_t(cx) + uint64_t(d.X) * (cy + uint64_t(d.Y) * cz);
#pragma unroll
  for (int k = 0; k < 8; ++k)
    cl[k] = __ldg(lab + v0 + (k & 1) + ((k >> 1) & 1) * uint64_t(d.X) + (k >> 2) * uint64_t(d.XY));
  count = 0;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const int a = 0, b = (t < 2) ? 1 : (t < 4 ? 2 : 4);
    const int c = (t == 0 || t == 2) ? 3 : (t == 1 || t == 4 ? 5 : 6);
    code[t] = tet_code(cl[a], cl[b], cl[c], cl[7]);
    count += case_count(code[t]);
  }
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t& total) {
  __shared__ uint32_t ws[THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t t = lane < THREADS / 32 ? ws[lane] : 0;
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += u;
    }
    if (lane < THREADS / 32) ws[lane] = ti - t;
  }
  __syncthreads();
  const uint32_t excl = inc - v + ws[w];
  // total = exclusive prefix of the last warp + its inclusive sum
  __shared__ uint32_t tot;
  if (threadIdx.x == THREADS - 1) tot = excl + v;
  __syncthreads();
  total = tot;
  return excl;
}

constexpr int kMThreads = 256;

template <class L>
__global__ void __launch_bounds__(kMThreads) k_sep_count(const L* __restrict__ lab, CDims d,
                                                         uint8_t* __restrict__ codes,
                                                         uint64_t* __restrict__ block_counts) {
  const uint64_t q = uint64_t(blockIdx.x) * kMThreads + threadIdx.x;
  int cnt = 0;
  if (q < d.cubes) {
    L cl[8];
    int code[6];
    cube_codes(lab, d, q, cl, code, cnt);
    if (codes) {
#pragma unroll
      for (int t = 0; t < 6; ++t) codes[6 * q + t] = uint8_t(code[t]);
    }
  }
  uint32_t total;
  block_excl_scan_u32<kMThreads>(uint32_t(cnt), total);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = total;
}

template <class L>
struct RecOf;
template <>
struct RecOf<uint32_t> {
  using T = plmss_tri;
};
template <>
struct RecOf<int64_t> {
  using T = plmss_tri64;
};

template <class L>
__global__ void __launch_bounds__(kMThreads) k_sep_emit(const L* __restrict__ lab, CDims d,
                                                        const uint64_t* __restrict__ block_off,
                                                        typename RecOf<L>::T* __restrict__ out) {
  const uint64_t q = uint64_t(blockIdx.x) * kMThreads + threadIdx.x;
  int cnt = 0;
  L cl[8];
  int code[6];
  if (q < d.cubes) cube_codes(lab, d, q, cl, code, cnt);
  uint32_t total;
  const uint32_t excl = block_excl_scan_u32<kMThreads>(uint32_t(cnt), total);
  if (cnt == 0) return;
  uint64_t pos = block_off[blockIdx.x] + excl;
#pragma unroll 1
  for (int t = 0; t < 6; ++t) {
    const int n = case_count(code[t]);
    if (!n) continue;
    const int first = case_first(code[t]);
    const uint64_t cell = 6 * q + t;
    for (int r = 0; r < n; ++r) {
      const uint32_t row = c_rows[first + r];
      const L la = cl[c_tet_corner[t][(row >> 12) & 3]];
      const L lb = cl[c_tet_corner[t][(row >> 14) & 3]];
      typename RecOf<L>::T rec;
      rec.cell_row = (cell << 6) | uint64_t(first + r);
      rec.lo = la < lb ? la : lb;
      rec.hi = la < lb ? lb : la;
      out[pos++] = rec;
    }
  }
}

// ------------------------------------------------------------ materialise --
struct MGeom {
  double sp[3], og[3];
};

__device__ __forceinline__ void vpos(const CDims& d, const MGeom& gm, uint64_t v, double p[3]) {
  const uint64_t x = v % d.X, y = (v / d.X) % d.Y, z = v / d.XY;
  const double c[3] = {double(x), double(y), double(z)};
#pragma unroll
  for (int k = 0; k < 3; ++k) p[k] = __dadd_rn(gm.og[k], __dmul_rn(gm.sp[k], c[k]));
}

template <class R>
__global__ void k_materialize(const R* __restrict__ tris, int64_t n, CDims d, MGeom gm,
                              double* __restrict__ points, int64_t* __restrict__ regions,
                              int64_t* __restrict__ cells) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const R rec = tris[i];
  const uint64_t cell = rec.cell_row >> 6;
  const uint32_t row = c_rows[rec.cell_row & 63];
  if (points) {
    const uint64_t q = cell / 6;
    const int t = int(cell % 6);
    const uint32_t cx = uint32_t(q % d.CX);
    const uint64_t r = q / d.CX;
    const uint32_t cy = uint32_t(r % d.CY), cz = uint32_t(r / d.CY);
    const uint64_t v0 = cx + uint64_t(d.X) * (cy + uint64_t(d.Y) * cz);
    double pv[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = c_tet_corner[t][k];
      vpos(d, gm, v0 + (c & 1) + ((c >> 1) & 1) * uint64_t(d.X) + (c >> 2) * uint64_t(d.XY), pv[k]);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int mask = (row >> (4 * k)) & 15;
      double s[3] = {0.0, 0.0, 0.0};
      int m = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (mask & (1 << j)) {
#pragma unroll
          for (int a = 0; a < 3; ++a) s[a] = __dadd_rn(s[a], pv[j][a]);
          ++m;
        }
#pragma unroll
      for (int a = 0; a < 3; ++a) points[9 * i + 3 * k + a] = __ddiv_rn(s[a], double(m));
    }
  }
  if (regions) {
    regions[2 * i] = int64_t(rec.lo);
    regions[2 * i + 1] = int64_t(rec.hi);
  }
  if (cells) cells[i] = int64_t(cell);
}

// -------------------------------------------------------------- boundaries --
// Faces are enumerated per minimum vertex w0: (w0, w0+A, w0+B) with corner
// masks A strictly inside B (12 types). Sorting by (v0, v1, v2) equals
// sorting by (w0, A, B) because the id delta of a mask is monotone in the
// mask for X, Y >= 2. Each face lies in one or two tets; a tet emits it iff
// the face labels agree and its fourth vertex label differs (the unique
// "lone" corner of marching.cpp:258-275). The lowest such cell is kept, which
// is what the reference's sort + unique produces (marching.cpp:289-296).
struct FaceTet {
  uint8_t origin_neg;  // cube origin = w0 - (mask)
  uint8_t t;           // tet index in that cube
  uint8_t fourth_pos;  // fourth vertex = w0 + pos - neg
  uint8_t fourth_neg;
};
struct FaceType {
  uint8_t A, B, ntets, pad;
  FaceTet tet[2];
};
__constant__ FaceType c_faces[12];

int perm_index(int p0, int p1) { return 2 * p0 + (p1 > (3 - p0 - p1) ? 1 : 0); }
int axis_of(int single) { return single == 1 ? 0 : (single == 2 ? 1 : 2); }

std::vector<FaceType> build_face_types() {
  std::vector<FaceType> out;
  for (int A = 1; A < 8; ++A)
    for (int B = A + 1; B < 8; ++B) {
      if ((A & B) != A) continue;
      FaceType f{};
      f.A = uint8_t(A);
      f.B = uint8_t(B);
      const int na = __builtin_popcount(A), nb = __builtin_popcount(B);
      auto add = [&](int origin_neg, int c1, int c2, int fpos, int fneg) {
        // chain 0 < c1 < c2 < 7 of the cube: permutation (c1, c2\c1, 7\c2)
        const int p0 = axis_of(c1), p1 = axis_of(c2 & ~c1);
        FaceTet ft{uint8_t(origin_neg), uint8_t(perm_index(p0, p1)), uint8_t(fpos), uint8_t(fneg)};
        f.tet[f.ntets++] = ft;
      };
      if (na == 1 && nb == 2) {
        add(0, A, B, 7, 0);                   // levels 0,1,2 of the cube at w0
        const int s = 7 & ~B;                 // levels 1,2,3 of the cube at w0 - s
        add(s, s, s | A, 0, s);
      } else if (na == 1 && nb == 3) {
        for (int e = 1; e < 8; e <<= 1)
          if (!(A & e)) add(0, A, A | e, A | e, 0);
      } else if (na == 2 && nb == 3) {
        for (int e = 1; e < 8; e <<= 1)
          if (A & e) add(0, e, A, e, 0);
      } else {
        continue;
      }
      out.push_back(f);
    }
  return out;
}

struct VDims {
  uint32_t X, Y, Z, XY, n;
  uint32_t CX, CY;
};

template <class L>
__device__ __forceinline__ int face_of(const L* __restrict__ lab, const VDims& d, uint32_t w0, uint32_t x,
                                       uint32_t y, uint32_t z, int f, bool has_filter, L filter,
                                       uint64_t& best_cell, L& tag) {
  const FaceType& ft = c_faces[f];
  auto off = [&](int m) { return (m & 1) + ((m >> 1) & 1) * d.X + (m >> 2) * d.XY; };
  auto inb = [&](int pos, int neg) {
    if ((pos & 1) && x + 1 >= d.X) return false;
    if ((pos & 2) && y + 1 >= d.Y) return false;
    if ((pos & 4) && z + 1 >= d.Z) return false;
    if ((neg & 1) && x == 0) return false;
    if ((neg & 2) && y == 0) return false;
    if ((neg & 4) && z == 0) return false;
    return true;
  };
  if (!inb(ft.B, 0)) return 0;
  const L l0 = __ldg(lab + w0);
  const L la = __ldg(lab + w0 + off(ft.A));
  const L lb = __ldg(lab + w0 + off(ft.B));
  if (l0 != la || l0 != lb) return 0;
  if (has_filter && l0 != filter) return 0;
  best_cell = ~uint64_t(0);
  for (int k = 0; k < ft.ntets; ++k) {
    const FaceTet& tt = ft.tet[k];
    // cube at w0 needs its max corner inside; cube at w0 - s needs w0 - s
    // inside (its max corner is w0 + B, inside since the face exists).
    if (!(tt.origin_neg == 0 ? inb(7, 0) : inb(0, tt.origin_neg))) continue;
    const uint32_t f4 = w0 + off(tt.fourth_pos) - off(tt.fourth_neg);
    if (__ldg(lab + f4) == l0) continue;
    const uint32_t o = w0 - off(tt.origin_neg);
    const uint32_t ox = o % d.X, oy = (o / d.X) % d.Y, oz = o / d.XY;
    const uint64_t cell = 6 * (uint64_t(ox) + uint64_t(d.CX) * (oy + uint64_t(d.CY) * oz)) + tt.t;
    if (cell < best_cell) best_cell = cell;
  }
  if (best_cell == ~uint64_t(0)) return 0;
  tag = l0;
  return 1;
}

template <class L>
__global__ void __launch_bounds__(kMThreads) k_bnd(const L* __restrict__ lab, VDims d, bool has_filter, L filter,
                                                   uint64_t* __restrict__ block_counts,
                                                   const uint64_t* __restrict__ block_off,
                                                   uint32_t* __restrict__ faces, L* __restrict__ tags,
                                                   int64_t* __restrict__ cells, uint8_t* __restrict__ used) {
  const uint32_t w0 = blockIdx.x * kMThreads + threadIdx.x;
  uint32_t mask = 0;
  uint64_t cellv[12];
  L tagv = 0;
  if (w0 < d.n) {
    const uint32_t x = w0 % d.X, y = (w0 / d.X) % d.Y, z = w0 / d.XY;
#pragma unroll 1
    for (int f = 0; f < 12; ++f) {
      uint64_t bc;
      L tg;
      if (face_of(lab, d, w0, x, y, z, f, has_filter, filter, bc, tg)) {
        mask |= 1u << f;
        cellv[f] = bc;
        tagv = tg;
      }
    }
  }
  uint32_t total;
  const uint32_t excl = block_excl_scan_u32<kMThreads>(uint32_t(__popc(mask)), total);
  if (block_counts) {
    if (threadIdx.x == 0) block_counts[blockIdx.x] = total;
    return;
  }
  uint64_t pos = block_off[blockIdx.x] + excl;
  auto off = [&](int m) { return (m & 1) + ((m >> 1) & 1) * d.X + (m >> 2) * d.XY; };
  for (int f = 0; f < 12; ++f) {
    if (!(mask & (1u << f))) continue;
    const uint32_t va = w0 + off(c_faces[f].A), vb = w0 + off(c_faces[f].B);
    faces[3 * pos] = w0;
    faces[3 * pos + 1] = va;
    faces[3 * pos + 2] = vb;
    if (tags) tags[pos] = tagv;
    if (cells) cells[pos] = int64_t(cellv[f]);
    if (used) {
      used[w0] = 1;
      used[va] = 1;
      used[vb] = 1;
    }
    ++pos;
  }
}

constexpr int kCRows = 16;
constexpr int kCTile = kMThreads * kCRows;

__global__ void __launch_bounds__(kMThreads) k_count_used(const uint8_t* __restrict__ used, uint32_t n,
                                                          uint64_t* __restrict__ counts) {
  const uint32_t base = blockIdx.x * kCTile;
  uint32_t c = 0;
  for (int r = 0; r < kCRows; ++r) {
    const uint32_t i = base + r * kMThreads + threadIdx.x;
    if (i < n && used[i]) ++c;
  }
  uint32_t total;
  block_excl_scan_u32<kMThreads>(c, total);
  if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kMThreads) k_write_used(const uint8_t* __restrict__ used, VDims d,
                                                          const uint64_t* __restrict__ off, MGeom gm,
                                                          uint32_t* __restrict__ rank, double* __restrict__ pts) {
  __shared__ uint32_t wc[kMThreads / 32];
  __shared__ uint32_t wp[kMThreads / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t base = blockIdx.x * kCTile;
  uint64_t running = off[blockIdx.x];
  CDims cd;
  cd.X = d.X;
  cd.Y = d.Y;
  cd.Z = d.Z;
  cd.XY = d.XY;
  for (int r = 0; r < kCRows; ++r) {
    const uint32_t i = base + r * kMThreads + threadIdx.x;
    const bool hit = i < d.n && used[i];
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wc[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int k = 0; k < kMThreads / 32; ++k) {
        wp[k] = s;
        s += wc[k];
      }
      wp[kMThreads / 32] = s;
    }
    __syncthreads();
    if (hit) {
      const uint64_t pos = running + wp[w] + __popc(m & ((1u << lane) - 1));
      rank[i] = uint32_t(pos);
      if (pts) vpos(cd, gm, i, pts + 3 * pos);
    }
    running += wp[kMThreads / 32];
    __syncthreads();
  }
}

__global__ void k_face_indices(const uint32_t* __restrict__ faces, int64_t nf, const uint32_t* __restrict__ rank,
                               int64_t* __restrict__ idx) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < 3 * nf) idx[i] = rank[faces[i]];
}

// Separator counts per cell range [bounds[i], bounds[i+1]) (EmitPlan's
// per-worker counts): shared-memory accumulators, one global add per range.
constexpr int kMaxRanges = 1024;

template <class L>
__global__ void __launch_bounds__(kMThreads) k_count_ranges(const L* __restrict__ lab, CDims d,
                                                            const int64_t* __restrict__ bounds, int nr,
                                                            unsigned long long* __restrict__ counts) {
  __shared__ unsigned long long s_cnt[kMaxRanges];
  __shared__ int64_t s_b[kMaxRanges + 1];
  for (int i = threadIdx.x; i < nr; i += kMThreads) s_cnt[i] = 0;
  for (int i = threadIdx.x; i <= nr; i += kMThreads) s_b[i] = bounds[i];
  __syncthreads();
  const uint64_t q = uint64_t(blockIdx.x) * kMThreads + threadIdx.x;
  if (q < d.cubes) {
    L cl[8];
    int code[6], cnt;
    cube_codes(lab, d, q, cl, code, cnt);
    if (cnt) {
#pragma unroll 1
      for (int t = 0; t < 6; ++t) {
        const int n = case_count(code[t]);
        if (!n) continue;
        const int64_t cell = int64_t(6 * q + t);
        int lo = 0, hi = nr;  // range r with s_b[r] <= cell < s_b[r+1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) / 2;
          if (s_b[mid] <= cell)
            lo = mid;
          else
            hi = mid;
        }
        atomicAdd(&s_cnt[lo], (unsigned long long)n);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nr; i += kMThreads)
    if (s_cnt[i]) atomicAdd(&counts[i], s_cnt[i]);
}

std::atomic<bool> g_tables_ready[64] = {};
std::mutex g_tables_mu;

void ensure_tables(Ctx& c) {
  if (c.device >= 0 && c.device < 64 && g_tables_ready[c.device].load(std::memory_order_acquire)) return;
  // one upload per device even when several host threads arrive together
  std::lock_guard<std::mutex> lock(g_tables_mu);
  if (c.device >= 0 && c.device < 64 && g_tables_ready[c.device].load(std::memory_order_acquire)) return;
  // Uploaded on the context stream and waited for: a plain cudaMemcpyToSymbol
  // runs on the legacy stream, which a non-blocking context stream does not
  // wait on (the first count kernel then saw half-written tables).
  CK(cudaMemcpyToSymbolAsync(c_rows, kTetRowsPacked, sizeof(kTetRowsPacked), 0, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyToSymbolAsync(c_cases, kTetCasePacked, sizeof(kTetCasePacked), 0, cudaMemcpyHostToDevice, c.stream));
  const std::vector<FaceType> ft = build_face_types();
  if (ft.size() != 12) fail(PLMSS_ERR_LOGIC, "face type table must have 12 entries");
  CK(cudaMemcpyToSymbolAsync(c_faces, ft.data(), sizeof(FaceType) * 12, 0, cudaMemcpyHostToDevice, c.stream));
  c.sync();
  if (c.device >= 0 && c.device < 64) g_tables_ready[c.device].store(true, std::memory_order_release);
}

template <class L>
int64_t sep_count(Ctx& c, const Grid& g, const L* lab, uint8_t* codes, uint64_t** block_off, int64_t* nblocks) {
  ensure_tables(c);
  const CDims d = to_cdims(g);
  const int64_t nb = (g.cubes + kMThreads - 1) / kMThreads;
  uint64_t* bc = c.get_t<uint64_t>(S_TMP0, nb > 0 ? nb : 1);
  if (nb > 0) {
    k_sep_count<L><<<(unsigned)nb, kMThreads, 0, c.stream>>>(lab, d, codes, bc);
    CK_LAUNCH("k_sep_count");
  }
  const uint64_t total = exclusive_scan_u64(c, bc, nb, true);
  *block_off = bc;
  *nblocks = nb;
  return int64_t(total);
}

}  // namespace

void count_by_cell_ranges(Ctx& c, const Grid& g, int label_type, const void* labels, const int64_t* h_bounds,
                          int nranges, int64_t* h_counts) {
  ensure_tables(c);
  if (nranges < 1 || nranges > kMaxRanges) fail(PLMSS_ERR_INVALID_ARGUMENT, "1..1024 cell ranges supported");
  const CDims d = to_cdims(g);
  int64_t* d_b = c.get_t<int64_t>(S_TMP1, nranges + 1);
  unsigned long long* d_cnt = c.get_t<unsigned long long>(S_TMP2, nranges);
  CK(cudaMemcpyAsync(d_b, h_bounds, sizeof(int64_t) * (nranges + 1), cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * nranges, c.stream));
  const int64_t nb = (g.cubes + kMThreads - 1) / kMThreads;
  if (nb > 0) {
    if (label_type == 0)
      k_count_ranges<uint32_t><<<(unsigned)nb, kMThreads, 0, c.stream>>>(static_cast<const uint32_t*>(labels), d,
                                                                          d_b, nranges, d_cnt);
    else
      k_count_ranges<int64_t><<<(unsigned)nb, kMThreads, 0, c.stream>>>(static_cast<const int64_t*>(labels), d,
                                                                         d_b, nranges, d_cnt);
    CK_LAUNCH("k_count_ranges");
  }
  CK(cudaMemcpyAsync(h_counts, d_cnt, sizeof(int64_t) * nranges, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
}

int64_t index_separators(Ctx& c, const Grid& g, int label_type, const void* labels, uint8_t* codes) {
  uint64_t* off;
  int64_t nb;
  if (label_type == 0) return sep_count(c, g, static_cast<const uint32_t*>(labels), codes, &off, &nb);
  if (label_type == 1) return sep_count(c, g, static_cast<const int64_t*>(labels), codes, &off, &nb);
  fail(PLMSS_ERR_INVALID_ARGUMENT, "unknown label type");
}

int64_t emit_separators(Ctx& c, const Grid& g, int label_type, const void* labels,
                        const std::function<void*(int64_t)>& get_out) {
  uint64_t* off;
  int64_t nb;
  const CDims d = to_cdims(g);
  if (label_type == 0) {
    auto* lab = static_cast<const uint32_t*>(labels);
    const int64_t total = sep_count(c, g, lab, nullptr, &off, &nb);
    void* out = get_out(total);
    if (out && nb > 0 && total > 0) {
      k_sep_emit<uint32_t><<<(unsigned)nb, kMThreads, 0, c.stream>>>(lab, d, off, static_cast<plmss_tri*>(out));
      CK_LAUNCH("k_sep_emit");
    }
    return total;
  }
  if (label_type == 1) {
    auto* lab = static_cast<const int64_t*>(labels);
    const int64_t total = sep_count(c, g, lab, nullptr, &off, &nb);
    void* out = get_out(total);
    if (out && nb > 0 && total > 0) {
      k_sep_emit<int64_t><<<(unsigned)nb, kMThreads, 0, c.stream>>>(lab, d, off, static_cast<plmss_tri64*>(out));
      CK_LAUNCH("k_sep_emit");
    }
    return total;
  }
  fail(PLMSS_ERR_INVALID_ARGUMENT, "unknown label type");
}

void materialize(Ctx& c, const Grid& g, const double* sp, const double* og, int label_type, const void* tris,
                 int64_t n, double* points, int64_t* regions, int64_t* cells) {
  ensure_tables(c);
  if (n <= 0) return;
  MGeom gm;
  for (int k = 0; k < 3; ++k) {
    gm.sp[k] = sp ? sp[k] : 1.0;
    gm.og[k] = og ? og[k] : 0.0;
  }
  const CDims d = to_cdims(g);
  if (label_type == 0)
    k_materialize<plmss_tri><<<blocks_for(n, 256), 256, 0, c.stream>>>(static_cast<const plmss_tri*>(tris), n, d,
                                                                        gm, points, regions, cells);
  else
    k_materialize<plmss_tri64><<<blocks_for(n, 256), 256, 0, c.stream>>>(static_cast<const plmss_tri64*>(tris), n,
                                                                          d, gm, points, regions, cells);
  CK_LAUNCH("k_materialize");
}

template <class L>
static void boundaries_impl(Ctx& c, const Grid& g, const MGeom& gm, const L* lab, int has_filter, L filter,
                            uint32_t* faces, L* tags, int64_t* cells, double* points, int64_t* indices,
                            int64_t* n_faces, int64_t* n_points) {
  ensure_tables(c);
  VDims d;
  d.X = uint32_t(g.X);
  d.Y = uint32_t(g.Y);
  d.Z = uint32_t(g.Z);
  d.XY = d.X * d.Y;
  d.n = uint32_t(g.n);
  d.CX = uint32_t(g.X - 1);
  d.CY = uint32_t(g.Y - 1);
  const int64_t nb = (g.n + kMThreads - 1) / kMThreads;
  uint64_t* bc = c.get_t<uint64_t>(S_TMP0, nb);
  k_bnd<L><<<(unsigned)nb, kMThreads, 0, c.stream>>>(lab, d, has_filter != 0, filter, bc, nullptr, nullptr, nullptr,
                                                    nullptr, nullptr);
  CK_LAUNCH("k_bnd(count)");
  const int64_t nf = int64_t(exclusive_scan_u64(c, bc, nb, true));
  *n_faces = nf;
  // Faces always materialise into scratch (used-vertex marking needs them).
  uint32_t* fbuf = faces ? faces : c.get_t<uint32_t>(S_TMP1, 3 * std::max<int64_t>(nf, 1));
  uint8_t* used = c.get_t<uint8_t>(S_BITMAP, g.n);
  CK(cudaMemsetAsync(used, 0, g.n, c.stream));
  k_bnd<L><<<(unsigned)nb, kMThreads, 0, c.stream>>>(lab, d, has_filter != 0, filter, nullptr, bc, fbuf, tags, cells,
                                                    used);
  CK_LAUNCH("k_bnd(emit)");
  const int64_t ub = (g.n + kCTile - 1) / kCTile;
  uint64_t* uc = c.get_t<uint64_t>(S_TMP2, ub);
  k_count_used<<<(unsigned)ub, kMThreads, 0, c.stream>>>(used, d.n, uc);
  CK_LAUNCH("k_count_used");
  *n_points = int64_t(exclusive_scan_u64(c, uc, ub, true));
  if (!faces) return;
  uint32_t* rank = c.get_t<uint32_t>(S_RANK_MAX, g.n);
  k_write_used<<<(unsigned)ub, kMThreads, 0, c.stream>>>(used, d, uc, gm, rank, points);
  CK_LAUNCH("k_write_used");
  if (indices && nf > 0) {
    k_face_indices<<<blocks_for(3 * nf, 256), 256, 0, c.stream>>>(fbuf, nf, rank, indices);
    CK_LAUNCH("k_face_indices");
  }
}

void emit_boundaries(Ctx& c, const Grid& g, const double* sp, const double* og, int label_type, const void* labels,
                     int has_filter, int64_t filter, uint32_t* faces, void* tags, int64_t* cells, double* points,
                     int64_t* indices, int64_t* n_faces, int64_t* n_points) {
  MGeom gm;
  for (int k = 0; k < 3; ++k) {
    gm.sp[k] = sp ? sp[k] : 1.0;
    gm.og[k] = og ? og[k] : 0.0;
  }
  if (label_type == 0)
    boundaries_impl<uint32_t>(c, g, gm, static_cast<const uint32_t*>(labels), has_filter, uint32_t(filter), faces,
                              static_cast<uint32_t*>(tags), cells, points, indices, n_faces, n_points);
  else if (label_type == 1)
    boundaries_impl<int64_t>(c, g, gm, static_cast<const int64_t*>(labels), has_filter, filter, faces,
                             static_cast<int64_t*>(tags), cells, points, indices, n_faces, n_points);
  else
    fail(PLMSS_ERR_INVALID_ARGUMENT, "unknown label type");
}

}  // namespace plmss_b200
