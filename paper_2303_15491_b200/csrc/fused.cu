// Fused B200 pipeline (the benchmarked path), four brick passes.
//
//  A  k_tile_segment : per 32^3 brick, steepest hops and in-shared-memory path
//                      compression (segmentation.cpp:60-168). Every vertex
//                      ends at a brick terminal: an extremum of the brick or
//                      the shell cell where its chain leaves the brick. Each
//                      brick writes its terminal table TT (exits, maxima,
//                      minima as brick-major cell indices) and, per vertex and
//                      direction, the u16 index of its terminal in that table
//                      (LT, brick-major), plus the global extremum lists.
//  B  k_tt_*         : the exit entries of all terminal tables form a forest
//                      whose roots are the extremum entries: successor of an
//                      exit = the terminal of that cell in its own brick;
//                      pointer jumping to the roots, then each entry's final
//                      label (a global vertex id).
//  C  k_brick<false> : per brick (+1 halo layer in x, y, z), final labels of
//                      every vertex = table entry of its LT index; distinct
//                      (asc, desc) pairs into the region set; separator
//                      triangles counted per 32-cube row chunk.
//     unique pairs sorted -> dense MS ids; chunk counts scanned -> offsets.
//  D  k_brick<true>  : same labels again, MS ids, desc/asc/ms written, and the
//                      separator records emitted in the reference cell order
//                      (marching.cpp:116-215) at their chunk offsets.
//
// Correctness: every table entry lies on its vertex's steepest chain and the
// chain's terminal extremum is unique, so any order of these
// resolutions reproduces the reference labels exactly.
#include <math.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <type_traits>

#include <cuda.h>

#include "common.cuh"
#include "tet_tables.h"

namespace plmss_b200 {

// Checked build (libplmss_b200_checked.so, _build.build_cuda(checked=True)):
// bounds of every computed index into a table, list, bitmap or output of the
// fused and z-slab passes are asserted on the device; the first failure's
// code is reported by the host driver as PLMSS_ERR_LOGIC. compute-sanitizer
// is not available on the GPU pool, this is its stand-in (tools/checked_run.py).
#ifdef PLMSS_CHECKED
__device__ unsigned long long g_check_fail;
#define DCHECK(cond, code)                                                                 \
  do {                                                                                     \
    if (!(cond)) atomicCAS(&::plmss_b200::g_check_fail, 0ull, (unsigned long long)(code)); \
  } while (0)
#else
#define DCHECK(cond, code) \
  do {                     \
  } while (0)
#endif

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
// x-face copies of LT: after the ntiles * TN words of LT, per brick the words
// of its x = 0 and x = 31 faces, (side, z, y)-major, so that pass B's gathers
// along a neighbour's x-face (consecutive exits step in y) are coalesced
constexpr int kFaceX = 2 * TY * TZ;
constexpr int A_THREADS = 1024;
constexpr int kCodeOff = 4 * HN;                // hop codes after the field box
constexpr int kTabOff = kCodeOff + (PN + 15) / 16 * 16;  // code byte -> pointer delta, up and down
// CTA-wide scalars and scan scratch, also in the dynamic window: with no
// static shared memory the window starts at a fixed, 1024-byte aligned offset
// (checked at run time), so every shared access is an immediate offset from
// the symbol (a runtime-aligned base is rematerialised in the loops under
// register pressure)
struct AStat {
  uint64_t bar;
  unsigned long long lbase[3];
  uint32_t wcnt[A_THREADS / 32][3];
  uint32_t tot[3];
  uint32_t eoff[7][A_THREADS / 32];
};
constexpr int kStatOff = kTabOff + 2 * 256 * 4;
constexpr int kASmem = kStatOff + int((sizeof(AStat) + 15) / 16 * 16);
static_assert(2 * 2 * PN <= 4 * HN, "pointer arrays must fit in the field box");
static_assert(kCodeOff % 16 == 0, "code array alignment");
constexpr uint8_t kExitMark = 0xfe;  // shell cell reached by some brick vertex
constexpr uint64_t kEmpty = ~uint64_t(0);

struct FDims {
  uint32_t X, Y, Z, XY, n;
  uint32_t tx, ty, tz;  // tile counts
  // Field buffer layers relative to the grid: local z in [zf0, zf0 + zfn)
  // (a z-slab's halo layers: zf0 = -1 with a rank below, zfn = Z + halos).
  int32_t zf0;
  uint32_t zfn;
  // z-slab pipeline: table entries >= pbase (= bricks << 15) are portals,
  // pbase + side * XY + x + X * y for the vertex (x, y) of the halo layer
  // below (side 0) / above (side 1) that a chain reaches; 0 = no portals.
  uint32_t pbase;
};


__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// 1.0f when a == b, else 0.0f (also for NaN): one FSET instruction.
__device__ __forceinline__ float feq(float a, float b) {
  float r;
  asm("set.eq.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// m |= bit when (a op b): a compare and one predicated OR
__device__ __forceinline__ void or_if_ne(uint32_t& m, uint32_t a, uint32_t b, uint32_t bit) {
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %1, %2;\n @q or.b32 %0, %0, %3;\n}" : "+r"(m) : "r"(a), "r"(b), "r"(bit));
}
__device__ __forceinline__ void or_if_eq(uint32_t& m, uint32_t a, uint32_t b, uint32_t bit) {
  asm("{\n .reg .pred q;\n setp.eq.u32 q, %1, %2;\n @q or.b32 %0, %0, %3;\n}" : "+r"(m) : "r"(a), "r"(b), "r"(bit));
}
__device__ __forceinline__ void or_if_ge(uint32_t& m, uint32_t a, uint32_t b, uint32_t bit) {
  asm("{\n .reg .pred q;\n setp.ge.u32 q, %1, %2;\n @q or.b32 %0, %0, %3;\n}" : "+r"(m) : "r"(a), "r"(b), "r"(bit));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Stencil s = 0..13 in ascending id-delta order (complex.cpp:78-88): s < 7
// are the corners k = dx + 2 dy + 4 dz of the lower unit cube
// [x-1, x] x [y-1, y] x [z-1, z] of v (s = k), s >= 7 the corners k of the
// upper cube [x, x+1] x ... (s = 6 + k); the vertex itself sits between s = 6
// and s = 7. Hop codes store cube positions p = s + (s >= 7), p = 7 for
// "no hop" (v is the lower cube's corner 7 and the upper cube's corner 0).

// Shell cell j of the 34^3 pointer space, j in [0, kShell): the z = 0 and
// z = 33 layers, then the side walls layer by layer (rows y = 0, y = 33,
// then columns x = 0, x = 33).
constexpr int kShell = 2 * 34 * 34 + 32 * 4 * 33;  // 6536
__device__ __forceinline__ uint32_t shell_cell(uint32_t j) {
  constexpr uint32_t L = 34 * 34, W = 4 * 33;
  if (j < 2 * L) return j < L ? j : j - L + 33 * L;
  const uint32_t k = j - 2 * L, hz = 1 + k / W, c = k - (hz - 1) * W;
  const uint32_t col = c < 34 ? c : c < 68 ? (c - 34) + 34 * 33 : c < 100 ? 34 * (c - 67) : 33 + 34 * (c - 99);
  return col + hz * L;
}
constexpr int kShellPerThread = (kShell + 1023) / 1024;  // 7

struct ACounters {
  unsigned long long n_max, n_min, n_exit, n_tt;
  int overflow;
  uint32_t bad;
};

// Steepest hops of one (x, y) column of 32 vertices (segmentation.cpp:60-85)
// from a shared-memory field box with row stride kHX and plane stride kHXY;
// fc = the column's vertex at brick layer -1 (the box's first plane). Per
// in-volume layer lz < nz: emit(lz, up | down << 4), 15 = no hop. The thread
// walks its column in z keeping the 7 stencil columns in registers (7 shared
// loads per vertex). With M = max f over the neighbours, steepest-up under
// the (f, id) order is the highest s with f == M when M > f(v), or when
// M == f(v) and s > 6; otherwise none. Steepest-down mirrors it (lowest s,
// s < 7). NaN (missing) neighbours never win.
template <int kHX, int kHXY, class Emit>
__device__ __forceinline__ void hop_column(const float* __restrict__ fc, const int nz, const uint32_t gv0,
                                           const uint32_t XY, ACounters* __restrict__ ctr, Emit&& emit) {
    // stencil columns (dx, dy): c0 (-1,-1) c1 (0,-1) c2 (-1,0) c3 (0,0)
    // c4 (1,0) c5 (0,1) c6 (1,1); s -> (column, plane):
    //   s0-3 = c0-c3 @ z-1, s4-6 = c0-c2 @ z, s7-9 = c4-c6 @ z, s10-13 = c3-c6 @ z+1
    float a0m = fc[-1 - kHX], a1m = fc[-kHX], a2m = fc[-1], a3m = fc[0];
    float a0 = fc[kHXY - 1 - kHX], a1 = fc[kHXY - kHX], a2 = fc[kHXY - 1], a3 = fc[kHXY], a4 = fc[kHXY + 1],
          a5 = fc[kHXY + kHX], a6 = fc[kHXY + kHX + 1];
#pragma unroll 4
    for (int lz = 0; lz < TZ; ++lz) {
      const float* p = fc + (lz + 2) * kHXY;  // plane z+1
      const float a3p = p[0], a4p = p[1], a5p = p[kHX], a6p = p[kHX + 1];
      if (lz < nz) {
        const float fv = a3;
        if (!isfinite(fv)) atomicMin(&ctr->bad, gv0 + XY * uint32_t(lz));
        const float fn[14] = {a0m, a1m, a2m, a3m, a0, a1, a2, a4, a5, a6, a3p, a4p, a5p, a6p};
        // Maxima / minima of the lower (s < 7, ids below v) and upper
        // (s >= 7) halves. The highest s attaining M lies in the upper half
        // iff the upper half attains M; the lowest s attaining m lies in the
        // lower half iff that one does. NaN (missing) neighbours never win.
        float Ml = fn[0], ml = fn[0], Mh = fn[7], mh = fn[7];
#pragma unroll
        for (int s = 1; s < 7; ++s) {
          Ml = fmaxf(Ml, fn[s]);
          ml = fminf(ml, fn[s]);
          Mh = fmaxf(Mh, fn[7 + s]);
          mh = fminf(mh, fn[7 + s]);
        }
        const float M = fmaxf(Ml, Mh), m = fminf(ml, mh);
        const bool up_hi = Mh == M, dn_lo = ml == m;
        // which of the chosen half's 7 neighbours attain M (m): 1.0 / 0.0
        // flags (PTX set, one ALU op each) summed with weights 2^i
        // (2^(6-i)) on the FMA pipe; the highest weight present is the
        // float's exponent. Exact: distinct powers of two below 2^7.
        float au = 0.f, ad = 0.f;
#pragma unroll
        for (int i = 0; i < 7; ++i) {
          au = __fmaf_rn(feq(up_hi ? fn[7 + i] : fn[i], M), float(1 << i), au);
          ad = __fmaf_rn(feq(dn_lo ? fn[i] : fn[7 + i], m), float(1 << (6 - i)), ad);
        }
        // au == 0 only when every neighbour is missing (M is NaN): no hop
        const uint32_t hu = uint32_t(__float_as_int(au) >> 23) - 127u + (up_hi ? 7u : 0u);  // highest s attaining M
        const uint32_t hd = (dn_lo ? 6u : 13u) - (uint32_t(__float_as_int(ad) >> 23) - 127u);  // lowest s attaining m
        // hop code: cube positions (s < 7 -> s, s >= 7 -> s + 1, none -> 7)
        const uint32_t pu = (M > fv || (M == fv && up_hi)) ? hu + (hu >= 7u) : 7u;
        const uint32_t pd = (m < fv || (m == fv && dn_lo)) ? hd + (hd >= 7u) : 7u;
        emit(lz, uint8_t(pu | (pd << 4)));
      }
      a0m = a0;
      a1m = a1;
      a2m = a2;
      a3m = a3;
      a0 = p[-1 - kHX];
      a1 = p[-kHX];
      a2 = p[-1];
      a3 = a3p;
      a4 = a4p;
      a5 = a5p;
      a6 = a6p;
    }
  }

// Cube-shared steepest hops (the same result as hop_column, fewer ALU-pipe
// instructions). The 14 neighbours of v are the corners of its upper unit
// cube [x, x+1] x [y, y+1] x [z, z+1] and of its lower one [x-1, x] x ...,
// v itself excepted; in id order they are the lower cube's corners
// k = dx + 2 dy + 4 dz (s = 0..6), v, then the upper cube's (s = 6 + k). A
// cube is two 2x2 quads stacked in z; a quad is reused by the next layer's
// cube, so per vertex two quads, two cube merges and one final merge per
// direction. Within every merge the second operand's corners all have higher
// ids than the first's, so "the highest id attaining the maximum" (the
// simulation of simplicity order, F5) is: take the second operand iff it
// attains the maximum (FMNMX + FSET on the ALU pipe); the winner rides
// along as a power-of-two weight updated by FFMAs (FMA pipe): measured
// faster than the per-vertex equality masks of hop_column and than corner
// indices blended by FFMA. NaN (missing) neighbours never attain a maximum
// or minimum.
// Quad: W = sum over the corners attaining the
// extremum of 2^bit (max: bit = corner, min: bit = 3 - corner), so the
// highest set bit is the winner; merges scale the preferred operand's weight
// past the other's bits (x16 within a cube, x128 between the cubes), and the
// final position is the float exponent of W.
struct HopW {
  float M, WM, m, Wm;
};
__device__ __forceinline__ HopW hop_quad_w(float a, float b, float c, float d) {
  HopW q;
  q.M = fmaxf(fmaxf(a, b), fmaxf(c, d));  // FMNMX3 + FMNMX (nvcc fuses the chain)
  q.m = fminf(fminf(a, b), fminf(c, d));
  q.WM = __fmaf_rn(feq(d, q.M), 8.f, __fmaf_rn(feq(c, q.M), 4.f, __fmaf_rn(feq(b, q.M), 2.f, feq(a, q.M))));
  q.Wm = __fmaf_rn(feq(a, q.m), 8.f, __fmaf_rn(feq(b, q.m), 4.f, __fmaf_rn(feq(c, q.m), 2.f, feq(d, q.m))));
  return q;
}
// max prefers hi (higher ids), min prefers lo
__device__ __forceinline__ HopW hop_cube_w(const HopW& lo, const HopW& hi) {
  HopW c;
  c.M = fmaxf(lo.M, hi.M);
  c.WM = __fmaf_rn(feq(hi.M, c.M), __fmaf_rn(16.f, hi.WM, -lo.WM), lo.WM);
  c.m = fminf(lo.m, hi.m);
  c.Wm = __fmaf_rn(feq(lo.m, c.m), __fmaf_rn(16.f, lo.Wm, -hi.Wm), hi.Wm);
  return c;
}
__device__ __forceinline__ uint32_t w_exp(float w) { return (__float_as_uint(w) >> 23) - 127u; }

// Hop code of a vertex from its lower and upper unit cubes: positions lower
// cube corner k -> k, upper cube corner k -> 7 + k (v itself -> 7: no hop);
// the code is pu | pd << 4, straight from the weights' exponents:
// pu = e_u - 127, pd = 14 - (e_d - 127)
__device__ __forceinline__ uint8_t hop_code(const HopW& cl, const HopW& cu) {
  const float M = fmaxf(cl.M, cu.M), m = fminf(cl.m, cu.m);
  const uint32_t eu = __float_as_uint(__fmaf_rn(feq(cu.M, M), __fmaf_rn(128.f, cu.WM, -cl.WM), cl.WM)) >> 23;
  const uint32_t ed = __float_as_uint(__fmaf_rn(feq(cl.m, m), __fmaf_rn(128.f, cl.Wm, -cu.Wm), cu.Wm)) >> 23;
  return uint8_t(eu + 16u * (141u - ed) - 127u);
}

template <int kHX, int kHXY, class Emit>
__device__ __forceinline__ void hop_column_cube(const float* __restrict__ fc, const int nz, const uint32_t gv0,
                                                const uint32_t XY, ACounters* __restrict__ ctr, Emit&& emit) {
  HopW L = hop_quad_w(fc[-1 - kHX], fc[-kHX], fc[-1], fc[0]);
  const float* p0 = fc + kHXY;
  float b0 = p0[-1 - kHX], b1 = p0[-kHX], b2 = p0[-1], b3 = p0[0];
  HopW U = hop_quad_w(b3, p0[1], p0[kHX], p0[kHX + 1]);
#pragma unroll 2
  for (int lz = 0; lz < TZ; ++lz) {
    const float* p = fc + (lz + 2) * kHXY;
    const float n0 = p[-1 - kHX], n1 = p[-kHX], n2 = p[-1], n3 = p[0], n4 = p[1], n5 = p[kHX], n6 = p[kHX + 1];
    const HopW Ln = hop_quad_w(b0, b1, b2, b3);
    const HopW Un = hop_quad_w(n3, n4, n5, n6);
    if (lz < nz) {
      const float fv = b3;
      if (!isfinite(fv)) atomicMin(&ctr->bad, gv0 + XY * uint32_t(lz));
      emit(lz, hop_code(hop_cube_w(L, Ln), hop_cube_w(U, Un)));
    }
    L = Ln;
    U = Un;
    b0 = n0;
    b1 = n1;
    b2 = n2;
    b3 = n3;
  }
}

// Cube-shared hops of two diagonal neighbours v1 = (x, y) and v2 = (x+1, y+1)
// over brick layers [z0, z0 + nl): the upper cube of v1 at layer z is the
// lower cube of v2 at layer z + 1, so per layer three new quads (columns
// (x-1, y-1), (x, y), (x+1, y+1)) and three cube merges serve two vertices
// (hop_column_cube: two of each per vertex), and ten shared loads instead of
// fourteen. fc = v1's column at box plane 0; ok1 / ok2: the columns lie in
// the volume; emit(which, lz, code).
template <int kHX, int kHXY, class Emit>
__device__ __forceinline__ void hop_pair_cube(const float* __restrict__ fc, const int z0, const int nl,
                                              const bool ok1, const bool ok2, const uint32_t gv1,
                                              const uint32_t gv2, const uint32_t XY, ACounters* __restrict__ ctr,
                                              Emit&& emit) {
  constexpr int D = kHX + 1;  // (x, y) -> (x+1, y+1)
  const float* p = fc + z0 * kHXY;  // plane P0 - 1 (P0 = z0 + 1: first vertex plane)
  // A = Q(x-1, y-1) at plane P0 - 1; B = Q(x, y) at P0 - 1 and P0; D = Q(x+1, y+1) at P0
  HopW A = hop_quad_w(p[-D], p[-kHX], p[-1], p[0]);
  const HopW B0 = hop_quad_w(p[0], p[1], p[kHX], p[D]);
  p += kHXY;
  float f1 = p[0], f2 = p[D];  // v1, v2 at plane P0
  HopW B = hop_quad_w(f1, p[1], p[kHX], f2);
  HopW Dq = hop_quad_w(f2, p[D + 1], p[D + kHX], p[2 * D]);
  HopW cB = hop_cube_w(B0, B);  // lower cube of v2 at P0
#pragma unroll 2
  for (int i = 0; i < nl; ++i) {
    const int lz = z0 + i;
    const float* q = fc + (lz + 1) * kHXY;  // plane P
    const float* n = q + kHXY;              // plane P + 1
    const float g1 = n[0], g2 = n[D];
    const HopW An = hop_quad_w(q[-D], q[-kHX], q[-1], f1);
    const HopW Bn = hop_quad_w(g1, n[1], n[kHX], g2);
    const HopW Dn = hop_quad_w(g2, n[D + 1], n[D + kHX], n[2 * D]);
    const HopW cu1 = hop_cube_w(B, Bn);
    if (ok1) {
      if (!isfinite(f1)) atomicMin(&ctr->bad, gv1 + XY * uint32_t(lz));
      emit(0, lz, hop_code(hop_cube_w(A, An), cu1));
    }
    if (ok2) {
      if (!isfinite(f2)) atomicMin(&ctr->bad, gv2 + XY * uint32_t(lz));
      emit(1, lz, hop_code(cB, hop_cube_w(Dq, Dn)));
    }
    A = An;
    B = Bn;
    Dq = Dn;
    cB = cu1;
    f1 = g1;
    f2 = g2;
  }
}

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
template <bool kTMA, bool kCodes = false, bool kCube = false>
__global__ void __launch_bounds__(A_THREADS, 1)
    k_tile_segment(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ field,
                   const uint8_t* __restrict__ gcodes, FDims d,
                   uint32_t* __restrict__ maxima, uint32_t* __restrict__ minima, uint32_t* __restrict__ max_tt,
                   uint32_t* __restrict__ min_tt, uint64_t ext_cap,
                   uint32_t* __restrict__ TT, uint64_t tt_cap, uint4* __restrict__ TB, uint32_t* __restrict__ lt,
                   ACounters* __restrict__ ctr) {
  extern __shared__ __align__(1024) unsigned char a_smem[];
  float* f = reinterpret_cast<float*>(a_smem);         // HN floats (steps 1-2)
  uint16_t* Pd = reinterpret_cast<uint16_t*>(a_smem);  // PN (steps 3+, aliases f)
  uint16_t* Pa = Pd + PN;                              // PN
  uint8_t* code = a_smem + kCodeOff;                   // PN
  // per code byte: pointer deltas of its up and down hops (one 8-byte load
  // for both directions of the same byte)
  int2* dtab = reinterpret_cast<int2*>(a_smem + kTabOff);
  AStat& st = *reinterpret_cast<AStat*>(a_smem + kStatOff);
  uint64_t& s_bar = st.bar;
  uint32_t(&s_wcnt)[A_THREADS / 32][3] = st.wcnt;
  uint32_t(&s_tot)[3] = st.tot;
  uint32_t(&s_eoff)[kShellPerThread][A_THREADS / 32] = st.eoff;
  unsigned long long(&s_lbase)[3] = st.lbase;

  const int tid = int(threadIdx.x);
  const int lane = tid & 31;
  const int lx = tid & 31, ly = tid >> 5;
  // TMA destinations must be 128-byte aligned
  if (tid == 0 && (smem_u32(a_smem) & 127u)) __trap();
  if ((kTMA || kCodes) && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t ntiles = d.tx * d.ty * d.tz;
  uint32_t phase = 0;
  // x-face copies of the LT words (kFaceX), staged in the dead code bytes
  // during step 6 and written out coalesced while the next brick's box is in
  // flight: thread tid moves words tid and tid + 1024, exactly the words its
  // own part of the code fill overwrites next
  uint32_t* fstage = reinterpret_cast<uint32_t*>(code);
  uint32_t prev_bt = ~0u;
  auto flush_faces = [&] {
#ifndef PLMSS_NO_FACEX
    if (prev_bt != ~0u) {
      uint32_t* fo = lt + uint64_t(ntiles) * TN + uint64_t(prev_bt) * kFaceX;
      // the x = 31 face is staged with y ^ 16 (a different bank from the
      // x = 0 word of the same (y, z)): un-swizzled here, still one segment
      fo[tid] = fstage[tid];
      fo[A_THREADS + (tid ^ 16)] = fstage[tid + A_THREADS];
    }
#endif
  };
  static_assert(kFaceX == 2 * A_THREADS && kFaceX * 4 <= PN, "face staging");
  // persistent: one CTA per SM walks the bricks
  for (uint32_t bt = blockIdx.x; bt < ntiles; bt += gridDim.x, phase ^= 1u) {
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const int gx0 = int(tx * TX), gy0 = int(ty * TY), gz0 = int(tz * TZ);

  // 1. field box (kCodes: the brick's hop codes, one 32 KB bulk copy into
  //    the pointer area; k_hop_codes computed them)
  if (kCodes) {
    if (tid == 0) {
      const uint32_t bar = smem_u32(&s_bar);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(TN))
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(Pd)),
          "l"(gcodes + (uint64_t(bt) << 15)), "r"(uint32_t(TN)), "r"(bar)
          : "memory");
    }
  } else if (kTMA) {
    const uint32_t bar = smem_u32(&s_bar);
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(HN * 4))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4}], [%5];" ::"r"(smem_u32(f)),
          "l"(&tmap), "r"(gx0 - HXO), "r"(gy0 - 1), "r"(gz0 - 1 - d.zf0), "r"(bar)
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
        if (i < HN && gx >= 0 && gx < int(d.X) && gy >= 0 && gy < int(d.Y) && gz >= d.zf0 &&
            gz < d.zf0 + int(d.zfn))
          v[k] = __ldg(field + (uint32_t(gx) + d.X * (uint32_t(gy) + d.Y * uint32_t(gz - d.zf0))));
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k * A_THREADS + tid;
        if (i < HN) f[i] = v[k];
      }
    }
  }
  // while the box is in flight: no-hop codes everywhere (step 2 overwrites
  // the in-volume brick cells) and the pointer delta of each code byte per
  // direction (0 for "none" and for shell bytes 0xff / kExitMark)
  flush_faces();
  for (int i = 4 * tid; i < PN; i += 4 * A_THREADS) *reinterpret_cast<uint32_t*>(code + i) = 0xffffffffu;
  if (tid < 512) {
    // hop codes hold cube positions: lower cube corner k = dx + 2 dy + 4 dz
    // of [x-1, x] x [y-1, y] x [z-1, z] -> k, upper cube corner k -> 7 + k,
    // 7 = no hop (v itself)
    const uint32_t c = uint32_t(tid & 255), pn = tid < 256 ? (c & 15) : (c >> 4);
    int dl = 0;
    if (pn != 7 && pn < 15 && c < kExitMark) {
      const int k = pn < 7 ? int(pn) : int(pn) - 7, o = pn < 7 ? -1 : 0;
      dl = ((k & 1) + o) + PX * (((k >> 1) & 1) + o) + PXY * ((k >> 2) + o);
    }
    reinterpret_cast<int*>(dtab)[2 * c + (tid >> 8)] = dl;
  }
  if (kTMA || kCodes) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(&s_bar)), "r"(phase)
        : "memory");
  }
  __syncthreads();

  // 2. steepest hops
  const int gx = gx0 + lx, gy = gy0 + ly;
  const bool col_ok = gx < int(d.X) && gy < int(d.Y);
  const int nz = min(TZ, int(d.Z) - gz0);  // in-volume layers of the brick
  const int hc = (lx + 1) + PX * (ly + 1);  // column in the pointer space (shell layer z = 0)
  const uint32_t gv0 = uint32_t(gx) + d.X * uint32_t(gy) + d.XY * uint32_t(gz0);
#ifndef PLMSS_NO_HOP_PAIRS
  if (!kCodes && kCube) {
    // diagonal pairs (x, y), (x+1, y+1), y even, x < 31, over half the
    // layers each (warps 0-30); the 32 columns left over ((31, y even) and
    // (0, y odd)) one per lane of warp 31 over all layers
    if (tid < 992) {
      const int zh = tid >= 496, rq = tid - 496 * zh, r = rq / 31, x = rq - 31 * r, y = 2 * r;
      const int z0 = 16 * zh, nl = min(16, nz - z0);
      const int ax = gx0 + x, ay = gy0 + y;
      const bool ok1 = ax < int(d.X) && ay < int(d.Y), ok2 = ax + 1 < int(d.X) && ay + 1 < int(d.Y);
      const int h1 = (x + 1) + PX * (y + 1);
      if (nl > 0 && (ok1 || ok2))
        hop_pair_cube<HX, HXY>(f + (y + 1) * HX + (x + HXO), z0, nl, ok1, ok2,
                               uint32_t(ax) + d.X * uint32_t(ay) + d.XY * uint32_t(gz0),
                               uint32_t(ax + 1) + d.X * uint32_t(ay + 1) + d.XY * uint32_t(gz0), d.XY, ctr,
                               [&](int which, int lz, uint8_t b) {
                                 DCHECK(h1 + which * (PX + 1) + (lz + 1) * PXY < PN, 104);
                                 code[h1 + which * (PX + 1) + (lz + 1) * PXY] = b;
                               });
    } else {
      const int l = tid - 992, x = l < 16 ? 31 : 0, y = l < 16 ? 2 * l : 2 * (l - 16) + 1;
      const int ax = gx0 + x, ay = gy0 + y;
      const int h1 = (x + 1) + PX * (y + 1);
      if (ax < int(d.X) && ay < int(d.Y))
        hop_column_cube<HX, HXY>(f + (y + 1) * HX + (x + HXO), nz,
                                 uint32_t(ax) + d.X * uint32_t(ay) + d.XY * uint32_t(gz0), d.XY, ctr,
                                 [&](int lz, uint8_t b) { code[h1 + (lz + 1) * PXY] = b; });
    }
  } else
#endif
  if (!kCodes && col_ok) {
    if (kCube)
      hop_column_cube<HX, HXY>(f + (ly + 1) * HX + (lx + HXO), nz, gv0, d.XY, ctr,
                               [&](int lz, uint8_t b) { code[hc + (lz + 1) * PXY] = b; });
    else
      hop_column<HX, HXY>(f + (ly + 1) * HX + (lx + HXO), nz, gv0, d.XY, ctr,
                          [&](int lz, uint8_t b) { code[hc + (lz + 1) * PXY] = b; });
  }
  if (kCodes) {
    // the brick's codes (k_hop_codes, brick-major) staged in the pointer area
    const uint8_t* st = reinterpret_cast<const uint8_t*>(Pd);
#pragma unroll 8
    for (int lz = 0; lz < TZ; ++lz) code[hc + (lz + 1) * PXY] = st[(lz << 10) | (ly << 5) | lx];
  }
  __syncthreads();

  // 3. pointers four hops ahead (f is dead from here on). Shell cells point
  //    at themselves: the z-shell cells of this column here, the 132 shell
  //    columns by threads 0..131. A shell cell that is the hop target of a
  //    brick vertex is an exit: its code byte becomes kExitMark (readers
  //    treat 0xff and kExitMark alike).
  uint32_t live_d = 0, live_a = 0, mmax = 0, mmin = 0;
#pragma unroll
  for (int i = 0; i < kShellPerThread; ++i) {
    const uint32_t j = uint32_t(tid + i * A_THREADS);
    if (j < uint32_t(kShell)) {
      const uint32_t h = shell_cell(j);
      Pd[h] = uint16_t(h);
      Pa[h] = uint16_t(h);
    }
  }
#ifdef PLMSS_INIT_UNROLL4
#pragma unroll 4
#else
#pragma unroll 2
#endif
  for (int lz = 0; lz < TZ; ++lz) {
    const int h = hc + (lz + 1) * PXY;
    const uint32_t c = code[h];
    const int2 dc = dtab[c];
    int u = h + dc.x, w = h + dc.y;
    const uint32_t cu = code[u], cw = code[w];
    // (no hop: u == h, whose own byte is a vertex code, or 0xff outside the
    // volume, where the mark is harmless: no chain ever enters such a cell)
    if (cu >= kExitMark) code[u] = kExitMark;
    if (cw >= kExitMark) code[w] = kExitMark;
    const int du = dtab[cu].x, dw = dtab[cw].y;
    Pd[h] = uint16_t(u + du);
    Pa[h] = uint16_t(w + dw);
    const uint32_t bit = 1u << lz;
    or_if_ne(live_d, uint32_t(du), 0u, bit);  // pointer two hops ahead may not be a terminal
    or_if_ne(live_a, uint32_t(dw), 0u, bit);
    // extremum iff no hop (delta 0; out-of-volume bytes are masked below)
    or_if_eq(mmax, uint32_t(dc.x), 0u, bit);
    or_if_eq(mmin, uint32_t(dc.y), 0u, bit);
  }
  {
    const uint32_t vmask = col_ok ? (nz >= 32 ? 0xffffffffu : ((1u << nz) - 1u)) : 0u;
    mmax &= vmask;
    mmin &= vmask;
  }
  __syncthreads();

  // 4. pointer jumping, P <- P^3 per round in both directions (measured
  //    faster than P^2, P^4 and P^6 on the bench field); a vertex retires once
  //    both its pointers are terminals; each thread runs its own rounds
  for (;;) {
    uint32_t m = live_d | live_a, nd = 0, na = 0;
    // two vertices per iteration: up to four independent load chains, each
    // direction only while it is live
#ifdef PLMSS_JUMP4
    // four vertices per iteration: up to eight independent load chains
    while (m) {
      int lzv[4];
      uint32_t bv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lzv[k] = m ? 31 - __clz(m) : lzv[k > 0 ? k - 1 : 0];
        bv[k] = 1u << lzv[k];
        m &= ~bv[k];
      }
      int hv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) hv[k] = hc + (lzv[k] + 1) * PXY;
      const uint32_t any = bv[0] | bv[1] | bv[2] | bv[3];
      if (live_d & any) {
        uint32_t p1[4], p2[4], p3[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) p1[k] = Pd[hv[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k) p2[k] = Pd[p1[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k) p3[k] = Pd[p2[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          Pd[hv[k]] = uint16_t(p3[k]);
          or_if_ne(nd, p3[k], p2[k], bv[k]);
        }
      }
      if (live_a & any) {
        uint32_t q1[4], q2[4], q3[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) q1[k] = Pa[hv[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k) q2[k] = Pa[q1[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k) q3[k] = Pa[q2[k]];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          Pa[hv[k]] = uint16_t(q3[k]);
          or_if_ne(na, q3[k], q2[k], bv[k]);
        }
      }
    }
#else
    while (m) {
      const int lz = 31 - __clz(m);
      const uint32_t bit = 1u << lz;
      m ^= bit;
      const int lz2 = m ? 31 - __clz(m) : lz;  // a second live vertex, or the first again
      const uint32_t bit2 = 1u << lz2;
      m &= ~bit2;
      const int h = hc + (lz + 1) * PXY, h2 = hc + (lz2 + 1) * PXY;
      if (live_d & (bit | bit2)) {
        const uint32_t p1 = Pd[h], r1 = Pd[h2];
        DCHECK(p1 < PN && r1 < PN, 101);
        const uint32_t p2 = Pd[p1], r2 = Pd[r1];
        DCHECK(p2 < PN && r2 < PN, 101);
        const uint32_t p3 = Pd[p2], r3 = Pd[r2];
        Pd[h] = uint16_t(p3);
        Pd[h2] = uint16_t(r3);
        or_if_ne(nd, p3, p2, bit);
        or_if_ne(nd, r3, r2, bit2);
      }
      if (live_a & (bit | bit2)) {
        const uint32_t q1 = Pa[h], s1 = Pa[h2];
        DCHECK(q1 < PN && s1 < PN, 102);
        const uint32_t q2 = Pa[q1], s2 = Pa[s1];
        DCHECK(q2 < PN && s2 < PN, 102);
        const uint32_t q3 = Pa[q2], s3 = Pa[s2];
        Pa[h] = uint16_t(q3);
        Pa[h2] = uint16_t(s3);
        or_if_ne(na, q3, q2, bit);
        or_if_ne(na, s3, s2, bit2);
      }
    }
#endif
    live_d = nd;
    live_a = na;
    // asynchronous rounds (no barrier per round: measured 0.2 ms faster on
    // cfg5): a vertex's convergence is local — its pointer is a terminal —
    // and pointers only ever advance along their chains, so other threads'
    // partly advanced pointers only shorten the walk
    if (!(live_d | live_a)) break;
  }
  __syncthreads();

  // 5. terminal table of the brick: TT[base ..) = exit cells, then maxima,
  //    then minima (brick-major cell indices), one atomic per brick. Exit
  //    cells: shell cells tid + 1024 i (kShellPerThread per thread). The local index of every
  //    terminal is written into the pointer arrays AT the terminal (exits in
  //    both, extrema in their own direction's array).
  uint32_t mex = 0;  // bit i: shell cell tid + 1024 i is an exit
#pragma unroll
  for (int i = 0; i < kShellPerThread; ++i) {
    const uint32_t j = uint32_t(tid + i * A_THREADS);
    if (j < uint32_t(kShell)) mex |= uint32_t(code[shell_cell(j)] == kExitMark) << i;
  }
  // exits are numbered in shell order (j): per (i, warp) counts, scanned
  // below by warp 0
#pragma unroll
  for (int i = 0; i < kShellPerThread; ++i) {
    const uint32_t b = __ballot_sync(0xffffffffu, (mex >> i) & 1u);
    if (lane == 0) s_eoff[i][tid >> 5] = uint32_t(__popc(b));
  }

  const uint32_t cnt[3] = {uint32_t(__popc(mex)), uint32_t(__popc(mmax)), uint32_t(__popc(mmin))};
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
      if (lane == 31) s_tot[k] = inc;
    }
    {
      uint32_t run = 0;
#pragma unroll
      for (int i = 0; i < kShellPerThread; ++i) {
        const uint32_t v = s_eoff[i][lane];
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += u;
        }
        s_eoff[i][lane] = run + inc - v;
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncwarp();
    if (lane == 0) {
      const uint32_t te = s_tot[0], tm = s_tot[1], tn = s_tot[2];
      const unsigned long long base = atomicAdd(&ctr->n_tt, (unsigned long long)(te + tm + tn));
      s_lbase[0] = base;
      s_lbase[1] = tm ? atomicAdd(&ctr->n_max, (unsigned long long)tm) : 0ull;
      s_lbase[2] = tn ? atomicAdd(&ctr->n_min, (unsigned long long)tn) : 0ull;
      if (te) atomicAdd(&ctr->n_exit, (unsigned long long)te);
      TB[bt] = make_uint4(uint32_t(base), te, tm, tn);
    }
  }
  __syncthreads();
  const uint32_t te = s_tot[0], tm = s_tot[1];
  const uint64_t tbase = s_lbase[0];
  uint32_t lk[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) lk[k] = s_wcnt[tid >> 5][k] + pre[k];
  lk[1] += te;
  lk[2] += te + tm;
  uint64_t gpos_max = s_lbase[1] + (lk[1] - te), gpos_min = s_lbase[2] + (lk[2] - te - tm);
  const uint32_t bm0 = bt << 15;  // brick-major index of the brick's cell 0
#pragma unroll 1
  for (int b = 0; b < kShellPerThread; ++b) {
    const bool ex = (mex >> b) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, ex);
    if (!ex) continue;
    lk[0] = s_eoff[b][tid >> 5] + __popc(bal & ((1u << lane) - 1u));
    const uint32_t h = shell_cell(uint32_t(tid + b * A_THREADS));
    // the shell cell's brick and local coordinates (shell index 0 -> 31 of
    // the previous brick, 33 -> 0 of the next)
    const int hz = int(h / PXY), r = int(h) - hz * PXY, hy = r / PX, hx = r - hy * PX;
    const uint32_t nb = uint32_t(int(tx) + ((hx - 1) >> 5)) +
                        d.tx * (uint32_t(int(ty) + ((hy - 1) >> 5)) + d.ty * uint32_t(int(tz) + ((hz - 1) >> 5)));
    uint32_t bm = (nb << 15) | uint32_t((hx - 1) & 31) | uint32_t((hy - 1) & 31) << 5 |
                  uint32_t((hz - 1) & 31) << 10;
    // z-slab: a chain leaving the slab through a halo layer (only halo
    // layers hold real values outside the slab in z) -> portal entry
    const int gzc = gz0 + hz - 1;
    if (d.pbase && (gzc < 0 || gzc >= int(d.Z)))
      bm = d.pbase + (gzc < 0 ? 0u : d.XY) + uint32_t(gx0 + hx - 1) + d.X * uint32_t(gy0 + hy - 1);
    if (tbase + lk[0] < tt_cap) TT[tbase + lk[0]] = bm;
    Pd[h] = uint16_t(lk[0]);
    Pa[h] = uint16_t(lk[0]);
  }
  uint32_t m = mmax;
  while (m) {
    const int lz = __ffs(m) - 1;
    m &= m - 1;
    if (tbase + lk[1] < tt_cap) TT[tbase + lk[1]] = bm0 | uint32_t(lx + TX * ly + TX * TY * lz);
    if (gpos_max < ext_cap) {
      maxima[gpos_max] = gv0 + d.XY * uint32_t(lz);
      max_tt[gpos_max] = uint32_t(tbase + lk[1]);
    }
    Pd[hc + (lz + 1) * PXY] = uint16_t(lk[1]);
    ++lk[1];
    ++gpos_max;
  }
  m = mmin;
  while (m) {
    const int lz = __ffs(m) - 1;
    m &= m - 1;
    if (tbase + lk[2] < tt_cap) TT[tbase + lk[2]] = bm0 | uint32_t(lx + TX * ly + TX * TY * lz);
    if (gpos_min < ext_cap) {
      minima[gpos_min] = gv0 + d.XY * uint32_t(lz);
      min_tt[gpos_min] = uint32_t(tbase + lk[2]);
    }
    Pa[hc + (lz + 1) * PXY] = uint16_t(lk[2]);
    ++lk[2];
    ++gpos_min;
  }
  __syncthreads();

  // 6. LT: the terminal index of every in-volume vertex (an extremum reads
  //    its own entry, any other vertex its terminal's)
  if (col_ok) {
    uint32_t* ol = lt + bm0 + lx + TX * ly;
#ifdef PLMSS_NO_FACEX
    const bool face = false;
#else
    const bool face = lx == 0 || lx == TX - 1;
#endif
    uint32_t* of = fstage + (lx ? TY * TZ + (ly ^ 16) : ly);
#pragma unroll 4
    for (int lz = 0; lz < nz; ++lz) {
      const int h = hc + (lz + 1) * PXY;
      const uint32_t bit = 1u << lz;
      const uint32_t pd = Pd[h], pa = Pa[h];
      DCHECK(pd < PN && pa < PN, 103);
      // both directions' terminal indices in one word: desc | asc << 16
      const uint32_t w = uint32_t((mmax & bit) ? pd : Pd[pd]) | uint32_t((mmin & bit) ? pa : Pa[pa]) << 16;
      ol[TX * TY * lz] = w;
      if (face) of[TY * lz] = w;
    }
  }
  prev_bt = bt;
  __syncthreads();  // shared memory is reused by the next brick
  }
  flush_faces();
}

// Pass A1 (split mode, PLMSS_OPT_PASS_A_SPLIT): the steepest hops alone, at
// high occupancy. CTA = 8 rows x 32 columns x 32 layers of a brick; its field
// box (40 x 10 x 34 floats, 53 KB) arrives by one TMA copy (OOB = NaN), four
// CTAs per SM; codes out in the brick-major layout k_tile_segment<*, true>
// bulk-copies (one byte per padded brick cell, 0xff outside the volume).
constexpr int HR = 8;
constexpr int CXY = HX * (HR + 2);
constexpr int CN = CXY * HZ;
constexpr int kCSmem = CN * 4 + 128;

template <bool kTMA, bool kCube = false>
__global__ void __launch_bounds__(32 * HR, 4)
    k_hop_codes(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ field, const FDims d,
                uint8_t* __restrict__ codes, ACounters* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char h_smem_raw[];
  float* f = reinterpret_cast<float*>(h_smem_raw + ((128u - (smem_u32(h_smem_raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = int(threadIdx.x), lx = tid & 31, ly = tid >> 5;
  const uint32_t bt = blockIdx.x / (TY / HR), rg = blockIdx.x % (TY / HR);
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const int gx0 = int(tx * TX), gy0 = int(ty * TY + rg * HR), gz0 = int(tz * TZ);
  const int gx = gx0 + lx, gy = gy0 + ly;
  const bool col_ok = gx < int(d.X) && gy < int(d.Y);
  const int nz = min(TZ, int(d.Z) - gz0);
  uint8_t* out = codes + ((uint64_t(bt) << 15) | uint32_t((rg * HR + ly) << 5) | uint32_t(lx));
  if (gy0 < int(d.Y)) {
    if (kTMA) {
      if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar)),
                     "r"(uint32_t(CN * 4))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(smem_u32(f)),
            "l"(&tmap), "r"(gx0 - HXO), "r"(gy0 - 1), "r"(gz0 - 1 - d.zf0), "r"(smem_u32(&s_bar))
            : "memory");
      }
      __syncthreads();
      asm volatile(
          "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(
              smem_u32(&s_bar))
          : "memory");
    } else {
      for (int i = tid; i < CN; i += 32 * HR) {
        const int hx = i % HX, hy = (i / HX) % (HR + 2), hz = i / CXY;
        const int x = gx0 + hx - HXO, y = gy0 + hy - 1, z = gz0 + hz - 1;
        float v = __int_as_float(0x7fc00000);
        if (x >= 0 && x < int(d.X) && y >= 0 && y < int(d.Y) && z >= d.zf0 && z < d.zf0 + int(d.zfn))
          v = __ldg(field + (uint32_t(x) + d.X * (uint32_t(y) + d.Y * uint32_t(z - d.zf0))));
        f[i] = v;
      }
      __syncthreads();
    }
    if (col_ok) {
      const uint32_t gv0 = uint32_t(gx) + d.X * uint32_t(gy) + d.XY * uint32_t(gz0);
      if (kCube)
        hop_column_cube<HX, CXY>(f + (ly + 1) * HX + (lx + HXO), nz, gv0, d.XY, ctr,
                                 [&](int lz, uint8_t b) { out[lz << 10] = b; });
      else
        hop_column<HX, CXY>(f + (ly + 1) * HX + (lx + HXO), nz, gv0, d.XY, ctr,
                            [&](int lz, uint8_t b) { out[lz << 10] = b; });
    }
  }
  for (int lz = col_ok ? nz : 0; lz < TZ; ++lz) out[lz << 10] = 0xff;  // outside the volume: no hop
}

// ---------------------------------------------------------------- pass B --
// Terminal-table forest. Entry k of brick b is an exit (shell cell c, a
// vertex of a neighbouring brick b') or an extremum of b. The successor of an
// exit is the terminal of c in b': TB[b'].base + LT[c]; an extremum is its
// own successor. Chains follow the steepest paths, so the graph is a forest
// rooted at the extremum entries.
// A resolved entry holds its extremum's rank with kFinal set; an exit
// entry starts as its successor's index.
constexpr uint32_t kFinal = 0x80000000u;

constexpr uint32_t kPortal = 0x40000000u;  // with kFinal: a z-slab portal (pbase-relative index below)

__global__ void __launch_bounds__(256) k_tt_succ(const uint4* __restrict__ TB, const uint32_t* __restrict__ TT,
                                                 const uint32_t* __restrict__ lt, const uint32_t* __restrict__ RK,
                                                 uint32_t* __restrict__ SD, uint32_t* __restrict__ SA,
                                                 uint32_t pbase, uint64_t nt) {
  const uint4 h = TB[blockIdx.x];
  const uint32_t n = h.y + h.z + h.w;
  const uint32_t* TBw = reinterpret_cast<const uint32_t*>(TB);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t k = h.x + i;
    uint32_t sd, sa;
    if (i < h.y) {
      const uint32_t bm = __ldg(TT + k);
      if (pbase && bm >= pbase) {
        sd = sa = kFinal | kPortal | (bm - pbase);  // resolved across ranks (slab_resolve)
      } else {
        DCHECK((bm >> 15) < gridDim.x, 201);
        const uint32_t nb = __ldg(TBw + 4 * (bm >> 15));
        // desc | asc << 16; x-face cells from the face copy (grid = ntiles)
        const uint32_t cx = bm & 31u;
        const uint32_t l =
#ifdef PLMSS_NO_FACEX
            false
#else
            (cx == 0 || cx == TX - 1)
#endif
                ? __ldg(lt + uint64_t(gridDim.x) * TN + uint64_t(bm >> 15) * kFaceX + (cx ? TY * TZ : 0) +
                        ((bm >> 5) & 31u) + TY * ((bm >> 10) & 31u))
                : __ldg(lt + bm);
        sd = nb + (l & 0xffffu);
        sa = nb + (l >> 16);
        DCHECK(sd < nt && sa < nt, 202);
      }
    } else {
      // a maximum is only reached by descending-manifold chains, a minimum
      // only by ascending ones
      const uint32_t r = __ldg(RK + k) | kFinal;
      const bool is_max = i < h.y + h.z;
      sd = is_max ? r : kFinal;
      sa = is_max ? kFinal : r;
    }
    DCHECK(k < nt, 203);
    SD[k] = sd;
    SA[k] = sa;
  }
}

// Chain following on the successor arrays: each entry walks up to kChase
// links (both directions interleaved for memory-level parallelism) and
// stores the furthest entry reached. Values read from entries other threads
// have already advanced only shorten the walk; every value lies on the
// entry's chain, so concurrent updates are safe.
constexpr int kChase = 64;

__global__ void __launch_bounds__(256) k_tt_jump(uint64_t nt, uint32_t* __restrict__ SD, uint32_t* __restrict__ SA,
                                                 int* __restrict__ changed) {
  // two entries per thread (i, i + half): four independent chains in flight
  const uint64_t half = (nt + 1) / 2;
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool ch = false;
  if (i < half) {
    const uint64_t j = i + half;
    const bool two = j < nt;
    const uint32_t d0 = SD[i], a0 = SA[i];
    const uint32_t e0 = two ? SD[j] : kFinal, b0 = two ? SA[j] : kFinal;
    uint32_t xd = d0, xa = a0, yd = e0, ya = b0;
#pragma unroll 4
    for (int k = 0; k < kChase && !(xd & xa & yd & ya & kFinal); ++k) {
      DCHECK(((xd & kFinal) || xd < nt) && ((xa & kFinal) || xa < nt) && ((yd & kFinal) || yd < nt) &&
                 ((ya & kFinal) || ya < nt), 301);
      if (!(xd & kFinal)) xd = SD[xd];
      if (!(xa & kFinal)) xa = SA[xa];
      if (!(yd & kFinal)) yd = SD[yd];
      if (!(ya & kFinal)) ya = SA[ya];
    }
    if (xd != d0) SD[i] = xd;
    if (xa != a0) SA[i] = xa;
    if (two) {
      if (yd != e0) SD[j] = yd;
      if (ya != b0) SA[j] = ya;
    }
    ch = !(xd & xa & yd & ya & kFinal);
  }
  if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

// (list bit | gid, table entry) pairs of both extremum lists for one radix sort:
// maxima first (list bit 0), then minima (list bit 1 above the id bits)
__global__ void k_list_pairs(const uint32_t* __restrict__ maxima, const uint32_t* __restrict__ max_tt, int64_t n_max,
                             const uint32_t* __restrict__ minima, const uint32_t* __restrict__ min_tt, int64_t n_min,
                             int bits, uint64_t* __restrict__ keys, uint64_t* __restrict__ vals) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n_max) {
    keys[i] = maxima[i];
    vals[i] = max_tt[i];
  } else if (i < n_max + n_min) {
    keys[i] = (uint64_t(1) << bits) | minima[i - n_max];
    vals[i] = min_tt[i - n_max];
  }
}

// sorted pairs -> the two ascending lists and the rank (within its list) of
// every extremum table entry
__global__ void k_rank_lists(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, int64_t n_max,
                             int64_t n_min, int bits, uint32_t* __restrict__ maxima,
                             uint32_t* __restrict__ minima, uint32_t* __restrict__ RK, uint32_t id0) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_max + n_min) return;
  // id0: the slab's first vertex id (z-slab lists are global)
  if (i < n_max) {
    maxima[i] = uint32_t(keys[i]) + id0;
    RK[vals[i]] = uint32_t(i);
  } else {
    minima[i - n_max] = uint32_t(keys[i] ^ (uint64_t(1) << bits)) + id0;  // without the list bit
    RK[vals[i]] = uint32_t(i - n_max);
  }
}

// Both extremum lists sorted ascending (in place) and the rank of each of
// their table entries (RK), by one radix sort of the concatenated lists keyed
// (list, id): half the launches of a sort per list, and these launches are
// latency-bound (~2·10^4 entries). n_ids bounds the ids (radix bits).
static void sort_extrema(Ctx& c, uint32_t* maxima, const uint32_t* max_tt, int64_t n_max, uint32_t* minima,
                         const uint32_t* min_tt, int64_t n_min, uint64_t n_ids, uint32_t* RK, uint32_t id0) {
  const int64_t k = n_max + n_min;
  if (k < 1) return;
  uint64_t* kk = c.get_t<uint64_t>(S_SORT_A, k);
  uint64_t* vv = c.get_t<uint64_t>(S_SORT_B, k);
  int bits = 0;
  while ((uint64_t(1) << bits) < n_ids) ++bits;
  k_list_pairs<<<blocks_for(k, 256), 256, 0, c.stream>>>(maxima, max_tt, n_max, minima, min_tt, n_min, bits, kk, vv);
  CK_LAUNCH("k_list_pairs");
  if (k > 1) radix_sort_pairs(c, kk, vv, k, bits + 1);
  k_rank_lists<<<blocks_for(k, 256), 256, 0, c.stream>>>(kk, vv, n_max, n_min, bits, maxima, minima, RK, id0);
  CK_LAUNCH("k_rank_lists");
}

// Dense region bitmap (key = rank_min * n_max + rank_max, n_max * n_min <=
// 2^32): popcount per word, then per-word exclusive prefix (the dense MS id
// of the word's first set bit) and the region keys (asc << 32 | desc, in
// ascending order = the reference's sorted pair order).
constexpr int kWB = 1024;  // words per block
__global__ void __launch_bounds__(256) k_bitmap_count(const uint32_t* __restrict__ bm, uint64_t nw,
                                                      uint64_t* __restrict__ bsum) {
  const uint64_t w0 = uint64_t(blockIdx.x) * kWB;
  uint32_t c = 0;
  for (int k = threadIdx.x; k < kWB; k += 256)
    if (w0 + k < nw) c += __popc(bm[w0 + k]);
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int q = 0; q < 8; ++q) t += ws[q];
    bsum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kWB) k_bitmap_ids(const uint32_t* __restrict__ bm, uint64_t nw,
                                                    const uint64_t* __restrict__ boff, uint32_t nmax,
                                                    const uint32_t* __restrict__ maxs,
                                                    const uint32_t* __restrict__ mins, uint32_t* __restrict__ prefix,
                                                    uint64_t* __restrict__ keys, bool rank_keys = false) {
  __shared__ uint32_t ws[kWB / 32];
  const uint64_t wi = uint64_t(blockIdx.x) * kWB + threadIdx.x;
  const uint32_t word = wi < nw ? bm[wi] : 0u;
  const uint32_t c = __popc(word);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) ws[wp] = inc;
  __syncthreads();
  if (wp == 0) {
    const uint32_t t = ws[lane];
    uint32_t s2 = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, s2, o);
      if (lane >= o) s2 += u;
    }
    ws[lane] = s2 - t;
  }
  __syncthreads();
  if (wi >= nw) return;
  uint64_t id = boff[blockIdx.x] + ws[wp] + (inc - c);
  prefix[wi] = uint32_t(id);
  uint32_t m = word;
  while (m) {
    const uint32_t b = __ffs(m) - 1;
    m &= m - 1;
    const uint64_t key = wi * 32 + b;
    const uint32_t ra = uint32_t(key / nmax), rd = uint32_t(key - uint64_t(ra) * nmax);
    // region key in vertex ids, or (z-slab) the rank pair
    keys[id++] = rank_keys ? (uint64_t(ra) << 32 | rd) : (uint64_t(__ldg(mins + ra)) << 32) | __ldg(maxs + rd);
  }
}

// hash mode: sorted rank-pair keys -> region keys in vertex ids
__global__ void k_keys_to_gid(uint64_t* __restrict__ keys, int64_t r, const uint32_t* __restrict__ maxs,
                              const uint32_t* __restrict__ mins) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < r) {
    const uint64_t k = keys[i];
    keys[i] = (uint64_t(__ldg(mins + (k >> 32))) << 32) | __ldg(maxs + uint32_t(k));
  }
}

// ------------------------------------------------- region set compaction --
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

__global__ void k_set_ids(const uint64_t* __restrict__ sorted_slots, int64_t r, uint32_t* __restrict__ slot_id) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < r) slot_id[sorted_slots[i]] = uint32_t(i);
}

// ------------------------------------------------------------ passes C, D --
// One CTA per brick of 32^3 cubes; the vertex layers z = 0..32 of the brick
// plus its +x / +y halo (33 x 33 vertices per layer) are loaded kBatch layers
// at a time into a ring of kBatch + 1 layers in shared memory (all of a
// batch's loads in flight together). Every vertex's final pair is the table
// entry of its LT index: (FA[base + lta[v]], FD[base + ltd[v]]), base = its
// brick's table. Then warp w handles cube row y = w of each cube layer whose
// two vertex layers are present, lane = cube x (one 32-cube chunk of the
// reference cell order).
// A CTA takes RY = 4 cube rows of a brick (warp w <-> row w): small CTAs,
// many per SM, so one CTA's barriers overlap the others' work.
constexpr int RY = 8, B_THREADS = 32 * RY;
constexpr int LW = TX + 1, LQ = LW * (RY + 1);  // 33 x 17 = 561 vertices per layer
constexpr int kBatch = 8, kRing = 16;  // ring >= kBatch + 1, power of two
static_assert(kRing >= kBatch + 1 && (kRing & (kRing - 1)) == 0, "ring size");
__constant__ uint32_t c_mrows[PLMSS_TET_ROWS];
__constant__ uint16_t c_mcases[32];

// equality pattern (b==a, c==a, c==b, d==a, d==b, d==c) of tet (a,b,c,d)
// -> tetra_code (marching.cpp:28-44) | separator count << 5
__device__ __forceinline__ void load_march_tables(uint16_t* s_tlut, uint16_t* s_cases, uint32_t* s_rows) {
  if (threadIdx.x < 32) s_cases[threadIdx.x] = c_mcases[threadIdx.x];
  if (threadIdx.x < PLMSS_TET_ROWS) s_rows[threadIdx.x] = c_mrows[threadIdx.x];
  if (threadIdx.x < 64) {
    const uint32_t p = threadIdx.x;
    const int l1 = (p & 1) ? 0 : 1;
    const int l2 = (p & 2) ? 0 : ((p & 4) ? l1 : 2);
    const int l3 = (p & 8) ? 0 : ((p & 16) ? l1 : ((p & 32) ? l2 : 3));
    const int code = (l1 << 4) | (l2 << 2) | l3;
    s_tlut[p] = uint16_t(code | ((c_mcases[code] & 15) << 5));
  }
}

// The 6 tet codes (5 bits each) and separator count of a cube from its
// corner labels, corner c = dx | dy << 1 | dz << 2; tets t = {0,1,3,7}
// {0,1,5,7} {0,2,3,7} {0,2,6,7} {0,4,5,7} {0,4,6,7} (complex.cpp:203-218).
template <class L>
__device__ __forceinline__ uint32_t cube_codes(const L (&c)[8], const uint16_t* s_tlut, uint32_t& cnt) {
  const uint32_t e01 = c[1] == c[0], e02 = c[2] == c[0], e04 = c[4] == c[0], e07 = (c[7] == c[0]) << 3;
  const uint32_t e03 = c[3] == c[0], e05 = c[5] == c[0], e06 = c[6] == c[0];
  const uint32_t e13 = c[3] == c[1], e15 = c[5] == c[1], e23 = c[3] == c[2], e26 = c[6] == c[2];
  const uint32_t e45 = c[5] == c[4], e46 = c[6] == c[4];
  const uint32_t e17 = c[7] == c[1], e27 = c[7] == c[2], e47 = c[7] == c[4];
  const uint32_t e37 = c[7] == c[3], e57 = c[7] == c[5], e67 = c[7] == c[6];
  const uint32_t t0 = s_tlut[e01 | e03 << 1 | e13 << 2 | e07 | e17 << 4 | e37 << 5];
  const uint32_t t1 = s_tlut[e01 | e05 << 1 | e15 << 2 | e07 | e17 << 4 | e57 << 5];
  const uint32_t t2 = s_tlut[e02 | e03 << 1 | e23 << 2 | e07 | e27 << 4 | e37 << 5];
  const uint32_t t3 = s_tlut[e02 | e06 << 1 | e26 << 2 | e07 | e27 << 4 | e67 << 5];
  const uint32_t t4 = s_tlut[e04 | e05 << 1 | e45 << 2 | e07 | e47 << 4 | e57 << 5];
  const uint32_t t5 = s_tlut[e04 | e06 << 1 | e46 << 2 | e07 | e47 << 4 | e67 << 5];
  cnt = (t0 >> 5) + (t1 >> 5) + (t2 >> 5) + (t3 >> 5) + (t4 >> 5) + (t5 >> 5);
  return (t0 & 31) | (t1 & 31) << 5 | (t2 & 31) << 10 | (t3 & 31) << 15 | (t4 & 31) << 20 | (t5 & 31) << 25;
}

// Marching tables in global memory (L1-resident), built once per device by
// k_march_init: equality-pattern LUT, recipe cases and rows, and the
// two-label cube tables (corner membership m8 with bit 0 set, indexed m8 >> 1:
// separator count, records as tet << 8 | recipe row).
__device__ uint16_t g_tlut[64], g_cases[32];
__device__ uint32_t g_rows[PLMSS_TET_ROWS];
__device__ uint8_t g_two_cnt[128];
__device__ uint16_t g_two_rec[128 * 12];

__global__ void k_march_init() {
  __shared__ uint16_t s_tlut[64], s_cases[32];
  __shared__ uint32_t s_rows[PLMSS_TET_ROWS];
  load_march_tables(s_tlut, s_cases, s_rows);
  __syncthreads();
  const int tid = int(threadIdx.x);
  if (tid < 64) g_tlut[tid] = s_tlut[tid];
  if (tid < 32) g_cases[tid] = s_cases[tid];
  if (tid < PLMSS_TET_ROWS) g_rows[tid] = s_rows[tid];
  if (tid < 128) {
    // corner i carries label 0 when bit i of m8 is set (bit 0 always is)
    const uint32_t m8 = uint32_t(tid) << 1 | 1u;
    uint32_t lab[8];
    for (int i = 0; i < 8; ++i) lab[i] = (m8 >> i) & 1u ? 0u : 1u;
    uint32_t cnt;
    const uint32_t code6 = cube_codes(lab, s_tlut, cnt);
    g_two_cnt[tid] = uint8_t(cnt);
    uint32_t r = 0;
    for (int t = 0; t < 6; ++t) {
      const uint32_t cs = s_cases[(code6 >> (5 * t)) & 31];
      for (uint32_t k = 0; k < (cs & 15); ++k) g_two_rec[tid * 12 + r++] = uint16_t(uint32_t(t) << 8 | ((cs >> 4) + k));
    }
  }
}

// Insert k; returns its slot (new or existing), ~0 on probe overflow.
__device__ __forceinline__ uint64_t set_insert_slot(unsigned long long* __restrict__ t, uint64_t mask, uint64_t k) {
  uint64_t s = mix64(k) & mask;
#pragma unroll 1
  for (int probe = 0; probe < 1024; ++probe) {
    const unsigned long long cur = t[s];
    if (cur == k) return s;
    if (cur == kEmpty) {
      const unsigned long long prev = atomicCAS(t + s, kEmpty, k);
      if (prev == kEmpty || prev == k) return s;
    }
    s = (s + 1) & mask;
  }
  return ~uint64_t(0);
}

struct BrickArgs {
  FDims d;
  uint32_t brick0;  // first brick of the launch (z-slab pipelining)
  uint32_t nxc;  // 32-cube chunks per cube row
  const uint4* TB;
  const uint32_t* lt;             // per vertex: desc | asc << 16 terminal indices (brick-major)
  const uint32_t *FD, *FA;        // per table entry: rank of the maximum / minimum
  const uint32_t *maxs, *mins;    // sorted extremum lists (rank -> vertex id)
  uint32_t nmax;                  // dense mode: key = rank_min * nmax + rank_max
  uint32_t nmin;                  // (checked build: bounds)
  uint64_t nt, nw;                // table entries, bitmap words (checked build: bounds)
  uint32_t* bitmap;               // dense mode: region bitmap
  unsigned long long* fset;       // hash mode: region set of (rank_min << 32 | rank_max)
  uint64_t fmask;
  uint16_t* chunk;                // separator count per 32-cube chunk (<= 32 * 90)
  uint8_t* cls;                   // per cube: 0 one region, m8 two labels, 0xff more
  uint32_t *desc, *asc, *ms;      // ms holds the region token until k_ms_ids (null: labels only)
  int* overflow;
  // count pass with ids (PLMSS_OPT_IDS_IN_COUNT): ms holds the tokens, the
  // count pass writes every owned vertex's dense id into ids_out (dense:
  // bitmap word prefix, hash: slot -> id), so no id pass over ms is needed
  uint32_t* ids_out;
  const uint32_t *prefix, *slot_id;
};

// region token -> dense MS id, the count pass's copy of token_id
__device__ __forceinline__ uint32_t brick_token_id(const BrickArgs& a, uint32_t k) {
  if (a.prefix) return __ldg(a.prefix + (k >> 5)) + __popc(__ldg(a.bitmap + (k >> 5)) & ((1u << (k & 31)) - 1u));
  if (a.slot_id) return __ldg(a.slot_id + k);
  return k;  // ms already holds the ids (copied out)
}

// Pass C1 (k_tokens): every vertex's final pair from its LT indices and its
// brick's table, written as desc/asc (vertex ids of the two extrema) and as
// a region token in ms: the dense key (rank_min * nmax + rank_max) or the
// vertex's slot in the region hash set; equal tokens <=> equal (asc, desc)
// pairs. Thread per (x, y) column of a brick, kTokZ layers of loads in
// flight per step; the last pair of the column is cached (runs along z).
constexpr int kTokRows = 8, kTokZ = 8;

template <bool kDense>
__global__ void __launch_bounds__(32 * kTokRows) k_tokens(const BrickArgs a) {
  using Key = typename std::conditional<kDense, uint32_t, unsigned long long>::type;
  const FDims& d = a.d;
  const uint32_t bt = a.brick0 + blockIdx.x / (TY / kTokRows);
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const uint32_t lx = threadIdx.x & 31, ly = (blockIdx.x % (TY / kTokRows)) * kTokRows + (threadIdx.x >> 5);
  const uint32_t gx = tx * TX + lx, gy = ty * TY + ly, gz0 = tz * TZ;
  if (gx >= d.X || gy >= d.Y) return;
  const int nz = int(min(uint32_t(TZ), d.Z - gz0));
  const uint32_t base = __ldg(reinterpret_cast<const uint32_t*>(a.TB) + 4 * bt);
  const uint32_t* pl = a.lt + ((size_t(bt) << 15) | ly << 5 | lx);
  const uint32_t* fd = a.FD + base;
  const uint32_t* fa = a.FA + base;
  uint32_t gv = gx + d.X * (gy + d.Y * gz0);
  Key lkey = Key(~Key(0));
  uint32_t ltok = 0;
  uint2 lgv = make_uint2(0, 0);
  for (int z0 = 0; z0 < nz; z0 += kTokZ) {
    uint32_t ld[kTokZ], la[kTokZ];
#pragma unroll
    for (int i = 0; i < kTokZ; ++i) {
      if (z0 + i < nz) {
        const uint32_t l = __ldg(pl + (z0 + i) * TX * TY);
        ld[i] = l & 0xffffu;
        la[i] = l >> 16;
      }
    }
#pragma unroll
    for (int i = 0; i < kTokZ; ++i) {
      if (z0 + i < nz) {
        DCHECK(base + ld[i] < a.nt && base + la[i] < a.nt, 403);
        ld[i] = __ldg(fd + ld[i]);  // rank of the maximum | kFinal
        la[i] = __ldg(fa + la[i]);  // rank of the minimum | kFinal
      }
    }
#pragma unroll
    for (int i = 0; i < kTokZ; ++i) {
      if (z0 + i >= nz) break;
      // An entry the speculative forest sweep left unresolved holds a table
      // index, not a rank: no set insert and no extremum gather for it (the
      // pass is redone after the forest converges).
      if (!(ld[i] & la[i] & kFinal)) {
        if (a.desc) a.desc[gv] = a.asc[gv] = 0u;
        if (a.ms) a.ms[gv] = 0u;
        lkey = Key(~Key(0));
        gv += d.XY;
        continue;
      }
      ld[i] &= ~kFinal;
      la[i] &= ~kFinal;
      DCHECK(ld[i] < a.nmax && la[i] < a.nmin, 401);
      const Key key = kDense ? Key(la[i] * a.nmax + ld[i]) : Key((uint64_t(la[i]) << 32) | ld[i]);
      if (key != lkey) {
        if (!a.ms) {
          // labels only (fused_segment): no region set
        } else if (kDense) {
          ltok = uint32_t(key);
          const uint32_t bit = 1u << (ltok & 31);
          DCHECK((ltok >> 5) < a.nw, 402);
          uint32_t* wp = a.bitmap + (ltok >> 5);
          if (!(*wp & bit)) atomicOr(wp, bit);
        } else {
          const uint64_t slot = set_insert_slot(a.fset, a.fmask, uint64_t(key));
          if (slot == ~uint64_t(0)) *a.overflow = 1;
          ltok = uint32_t(slot);
        }
        if (a.desc) lgv = make_uint2(__ldg(a.maxs + ld[i]), __ldg(a.mins + la[i]));
        lkey = key;
      }
      if (a.desc) {
        a.desc[gv] = lgv.x;
        a.asc[gv] = lgv.y;
      }
      if (a.ms) a.ms[gv] = ltok;
      gv += d.XY;
    }
  }
}

// k_tokens with the CTA's terminal indices (8 rows x 32 layers of its brick,
// 2 x 16 KB) staged by two 2-D TMA tensor copies instead of per-thread loads.
constexpr int kTokSmem = 2 * TZ * 32 * kTokRows * 2;  // both index arrays
// kMode 0: region tokens (dense key / hash slot) and the labels; 1: mark
// only (region bitmap bits, no writes: a gather only where a column's LT
// word changes); 2: the dense ids straight into ms (bitmap and prefix
// complete) and the labels.
template <bool kDense, int kMode = 0>
__device__ __forceinline__ void tokens_tma_body(const CUtensorMap& mlt, const BrickArgs& a, const uint32_t blk,
                                                unsigned char* smem) {
  using Key = typename std::conditional<kDense, uint32_t, unsigned long long>::type;
  uint32_t(*sl)[32 * kTokRows] = reinterpret_cast<uint32_t(*)[32 * kTokRows]>(smem);  // 128-byte aligned
  __shared__ __align__(8) uint64_t s_bar;
  const FDims& d = a.d;
  const uint32_t grp = blk % (TY / kTokRows);
  const uint32_t bt = a.brick0 + blk / (TY / kTokRows);
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const uint32_t lx = threadIdx.x & 31, ly = grp * kTokRows + (threadIdx.x >> 5);
  const uint32_t bar = smem_u32(&s_bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(uint32_t(kTokSmem))
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(&sl[0][0])),
        "l"(&mlt), "r"(grp * 32 * kTokRows), "r"(bt * TZ), "r"(bar)
        : "memory");
  }
  const uint32_t base = __ldg(reinterpret_cast<const uint32_t*>(a.TB) + 4 * bt);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(bar)
      : "memory");
  const uint32_t gx = tx * TX + lx, gy = ty * TY + ly, gz0 = tz * TZ;
  if (gx >= d.X || gy >= d.Y) return;
  const int nz = int(min(uint32_t(TZ), d.Z - gz0));
  const uint32_t l = threadIdx.x;  // column within the CTA's rows
  const uint32_t* fd = a.FD + base;
  const uint32_t* fa = a.FA + base;
  if (kMode == 1) {
    static_assert(kDense || kMode != 1, "mark mode is dense only");
    // kTokZ layers per group: all table gathers in flight first (a repeated
    // word hits L1), then the bits where the column's word changed
    uint32_t llv = ~0u;
#pragma unroll 1
    for (int z0 = 0; z0 < nz; z0 += kTokZ) {
      uint32_t lv[kTokZ], rd[kTokZ], ra[kTokZ];
#pragma unroll
      for (int i = 0; i < kTokZ; ++i) {
        lv[i] = sl[min(z0 + i, nz - 1)][l];  // past the volume: a valid word, not used
        DCHECK(base + (lv[i] & 0xffffu) < a.nt && base + (lv[i] >> 16) < a.nt, 405);
        rd[i] = __ldg(fd + (lv[i] & 0xffffu));
        ra[i] = __ldg(fa + (lv[i] >> 16));
      }
#pragma unroll
      for (int i = 0; i < kTokZ; ++i) {
        if (z0 + i >= nz) break;
        if (lv[i] == llv) continue;
        llv = lv[i];
        if (!(rd[i] & ra[i] & kFinal)) continue;  // unresolved (speculative sweep): redone
        const uint32_t key = (ra[i] & ~kFinal) * a.nmax + (rd[i] & ~kFinal);
        DCHECK((rd[i] & ~kFinal) < a.nmax && (ra[i] & ~kFinal) < a.nmin && (key >> 5) < a.nw, 406);
        const uint32_t bit = 1u << (key & 31);
        uint32_t* wp = a.bitmap + (key >> 5);
        if (!(*wp & bit)) atomicOr(wp, bit);
      }
    }
    return;
  }
  uint32_t gv = gx + d.X * (gy + d.Y * gz0);
  Key lkey = Key(~Key(0));
  uint32_t ltok = 0;
  uint2 lgv = make_uint2(0, 0);
  // kTokZ layers per group, unguarded for full bricks
  auto group = [&](auto full, const int z0) {
    constexpr bool kF = decltype(full)::value;
    uint32_t ld[kTokZ], la[kTokZ];
#pragma unroll
    for (int i = 0; i < kTokZ; ++i) {
      if (kF || z0 + i < nz) {
        const uint32_t lv = sl[z0 + i][l];
        DCHECK(base + (lv & 0xffffu) < a.nt && base + (lv >> 16) < a.nt, 404);
        ld[i] = __ldg(fd + (lv & 0xffffu));  // rank of the maximum | kFinal
        la[i] = __ldg(fa + (lv >> 16));      // rank of the minimum | kFinal
      }
    }
#pragma unroll
    for (int i = 0; i < kTokZ; ++i) {
      if (!kF && z0 + i >= nz) break;
      // An entry the speculative forest sweep left unresolved holds a table
      // index, not a rank: no set insert and no extremum gather for it (the
      // pass is redone after the forest converges).
      if (!(ld[i] & la[i] & kFinal)) {
        if (a.desc) a.desc[gv] = a.asc[gv] = 0u;
        if (a.ms) a.ms[gv] = 0u;
        lkey = Key(~Key(0));
        gv += d.XY;
        continue;
      }
      ld[i] &= ~kFinal;
      la[i] &= ~kFinal;
      DCHECK(ld[i] < a.nmax && la[i] < a.nmin, 401);
      const Key key = kDense ? Key(la[i] * a.nmax + ld[i]) : Key((uint64_t(la[i]) << 32) | ld[i]);
      if (key != lkey) {
        if (!a.ms) {
          // labels only (fused_segment): no region set
        } else if (kMode == 2) {
          DCHECK((uint32_t(key) >> 5) < a.nw, 402);
          ltok = brick_token_id(a, uint32_t(key));
        } else if (kDense) {
          ltok = uint32_t(key);
          const uint32_t bit = 1u << (ltok & 31);
          DCHECK((ltok >> 5) < a.nw, 402);
          uint32_t* wp = a.bitmap + (ltok >> 5);
          if (!(*wp & bit)) atomicOr(wp, bit);
        } else {
          const uint64_t slot = set_insert_slot(a.fset, a.fmask, uint64_t(key));
          if (slot == ~uint64_t(0)) *a.overflow = 1;
          ltok = uint32_t(slot);
        }
        if (a.desc) lgv = make_uint2(__ldg(a.maxs + ld[i]), __ldg(a.mins + la[i]));
        lkey = key;
      }
      if (a.desc) {
        a.desc[gv] = lgv.x;
        a.asc[gv] = lgv.y;
      }
      if (a.ms) a.ms[gv] = ltok;
      gv += d.XY;
    }
  };
  if (nz == TZ) {
#pragma unroll 1
    for (int z0 = 0; z0 < TZ; z0 += kTokZ) group(std::true_type{}, z0);
  } else {
#pragma unroll 1
    for (int z0 = 0; z0 < nz; z0 += kTokZ) group(std::false_type{}, z0);
  }
}

// Pass C2 (k_brick): cube classes and separator counts per 32-cube chunk
// from the region tokens. CTA = RY cube rows of a brick; the vertex layers
// z = 0..32 of those rows plus the +x / +y halo stream through a shared-memory
// ring kBatch layers at a time; warp w handles cube row w, lane = cube x.
__global__ void __launch_bounds__(B_THREADS, 4) k_brick(const BrickArgs a) {
  __shared__ uint32_t ring[kRing * LQ];
  const FDims& d = a.d;
  const uint32_t bt = a.brick0 + blockIdx.x / (TY / RY), yb = (blockIdx.x % (TY / RY)) * RY;  // brick, first row
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const uint32_t gx0 = tx * TX, gy0 = ty * TY + yb, gz0 = tz * TZ;
  if (gy0 >= d.Y) return;  // rows of a brick cut by the volume
  const int tid = int(threadIdx.x), lane = tid & 31, w = tid >> 5;
  const int nl = int(min(uint32_t(TZ + 1), d.Z - gz0));  // vertex layers of the brick + halo
  // this thread's cube column: x = lane, y = w
  const uint32_t cy = gy0 + uint32_t(w);
  const bool row_ok = cy + 1 < d.Y && tx < a.nxc;
  const bool cube_ok = row_ok && gx0 + uint32_t(lane) + 1 < d.X;
  // this thread's cube class and its row's chunk count, advanced one cube
  // layer at a time
  const uint64_t CX = d.X - 1, CXY = uint64_t(d.X - 1) * (d.Y - 1);
  uint8_t* clsp = a.cls + (uint64_t(gx0) + lane + CX * cy + CXY * gz0);
  uint16_t* chp = a.chunk + (uint64_t(cy) + uint64_t(d.Y - 1) * gz0) * a.nxc + tx;
  const uint64_t chstep = uint64_t(d.Y - 1) * a.nxc;
  uint32_t pf[4] = {0, 0, 0, 0};  // top face of this thread's previous cube
  bool have_prev = false;
  // the (up to two) ring columns this thread loads: q = tid, tid + B_THREADS
  const uint32_t* col[2];
  bool col_ok[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int q = tid + p * B_THREADS;
    const int x = q % LW, y = q / LW;
    const uint32_t gx = gx0 + uint32_t(x), gy = gy0 + uint32_t(y);
    col_ok[p] = q < LQ && gx < d.X && gy < d.Y;
    col[p] = a.ms + (uint64_t(gx) + uint64_t(d.X) * (uint64_t(gy) + uint64_t(d.Y) * gz0));
  }

  for (int z0 = 0; z0 < nl; z0 += kBatch) {
    const int zn = min(kBatch, nl - z0);
    // ---- load layers z0 .. z0+zn-1 of the tokens
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int q = tid + p * B_THREADS;
      if (q >= LQ) break;
      uint32_t t[kBatch];
#pragma unroll
      for (int i = 0; i < kBatch; ++i)
        t[i] = (i < zn && col_ok[p]) ? __ldg(col[p] + uint64_t(z0 + i) * d.XY) : ~0u;
#pragma unroll
      for (int i = 0; i < kBatch; ++i)
        if (i < zn) ring[((z0 + i) & (kRing - 1)) * LQ + q] = t[i];
    }
    __syncthreads();
    if (a.ids_out && gx0 + uint32_t(lane) < d.X && cy < d.Y) {
      // the owned layers of this thread's vertex column (x = lane, y = w)
      uint32_t lt = ~0u, lid = 0;
      const uint64_t vo = uint64_t(gx0 + lane) + uint64_t(d.X) * (uint64_t(cy) + uint64_t(d.Y) * gz0);
      // the brick's own layers, and the grid's last layer when it is this
      // brick's layer 32 (a z-slab's extra layer)
      for (int z = z0; z < z0 + zn && (z < TZ || gz0 + uint32_t(z) == d.Z - 1); ++z) {
        const uint32_t tk = ring[(z & (kRing - 1)) * LQ + w * LW + lane];
        if (tk != lt) {
          lt = tk;
          lid = brick_token_id(a, tk);
        }
        a.ids_out[vo + uint64_t(z) * d.XY] = lid;
      }
    }
    // ---- cube layers z-1 whose two vertex layers are loaded
    for (int z = max(z0, 1); z < z0 + zn; ++z) {
      const uint32_t* lo = ring + ((z - 1) & (kRing - 1)) * LQ;
      const uint32_t* cur = ring + (z & (kRing - 1)) * LQ;
      const int o = w * LW + lane;
      uint32_t cnt = 0;
      if (cube_ok) {
        uint32_t c[8];
        // bottom face = the previous cube layer's top face (registers)
        if (have_prev) {
          c[0] = pf[0];
          c[1] = pf[1];
          c[2] = pf[2];
          c[3] = pf[3];
        } else {
          c[0] = lo[o];
          c[1] = lo[o + 1];
          c[2] = lo[o + LW];
          c[3] = lo[o + LW + 1];
        }
        c[4] = cur[o];
        c[5] = cur[o + 1];
        c[6] = cur[o + LW];
        c[7] = cur[o + LW + 1];
        pf[0] = c[4];
        pf[1] = c[5];
        pf[2] = c[6];
        pf[3] = c[7];
        have_prev = true;
        const bool uni = c[1] == c[0] && c[2] == c[0] && c[3] == c[0] && c[4] == c[0] && c[5] == c[0] &&
                         c[6] == c[0] && c[7] == c[0];
        uint32_t cls = 0;
        if (!uni) {
          // corners equal to corner 0 (bit i)
          uint32_t m8 = 1u;
#pragma unroll
          for (int i = 1; i < 8; ++i) m8 |= uint32_t(c[i] == c[0]) << i;
          // the lowest corner with another label; two labels iff every
          // corner carries one of the two (the common case on a separator)
          uint32_t b = c[7];
#pragma unroll
          for (int i = 6; i >= 1; --i) b = (m8 >> i) & 1u ? b : c[i];
          uint32_t mb = 0u;
#pragma unroll
          for (int i = 1; i < 8; ++i) mb |= uint32_t(c[i] == b) << i;
          if ((m8 | mb) == 0xffu) {
            cnt = g_two_cnt[m8 >> 1];
            cls = m8;
          } else {
            cube_codes(c, g_tlut, cnt);
            cls = 0xffu;
          }
        }
        *clsp = uint8_t(cls);
      }
      const uint32_t tot = __any_sync(0xffffffffu, cnt != 0) ? __reduce_add_sync(0xffffffffu, cnt) : 0u;
      if (lane == 0 && row_ok) *chp = uint16_t(tot);
      clsp += CXY;
      chp += chstep;
    }
    __syncthreads();
  }
}

// k_brick with the tokens staged by 3-D TMA tensor copies: batch b (cube
// layers 8b .. 8b+7) needs vertex layers 8b .. 8b+8 of the CTA's rows plus
// the +x / +y halo; one box {36 (x, padded), RY + 1, kBatch + 1} per batch,
// double-buffered so the next batch's copy overlaps this batch's cubes.
constexpr int TLW = 36;  // padded ring row (16-byte multiple of u32)
constexpr int kBrickBufWords = ((kBatch + 1) * (RY + 1) * TLW + 31) / 32 * 32;  // one staged batch
constexpr int kBrickSmem = 2 * kBrickBufWords * 4;
// Record count of a cube with three or more labels (rare): out of line so
// the unrolled count loop stays small in the instruction cache.
__device__ __noinline__ uint32_t general_count(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t c4,
                                               uint32_t c5, uint32_t c6, uint32_t c7) {
  const uint32_t c[8] = {c0, c1, c2, c3, c4, c5, c6, c7};
  uint32_t cnt = 0;
  cube_codes(c, g_tlut, cnt);
  return cnt;
}

__device__ __forceinline__ void brick_tma_body(const CUtensorMap& mtok, const BrickArgs& a, const uint32_t blk,
                                               unsigned char* smem) {
  // each buffer starts on a 128-byte boundary (TMA destination)
  constexpr int kBufWords = kBrickBufWords;
  uint32_t(*bufraw)[kBufWords] = reinterpret_cast<uint32_t(*)[kBufWords]>(smem);  // 128-byte aligned
  using Buf = uint32_t[kBatch + 1][RY + 1][TLW];
  Buf* buf[2] = {reinterpret_cast<Buf*>(bufraw[0]), reinterpret_cast<Buf*>(bufraw[1])};
  __shared__ __align__(8) uint64_t s_bar[2];
  const FDims& d = a.d;
  const uint32_t bt = a.brick0 + blk / (TY / RY), yb = (blk % (TY / RY)) * RY;  // brick, first row
  const uint32_t tx = bt % d.tx, ty = (bt / d.tx) % d.ty, tz = bt / (d.tx * d.ty);
  const uint32_t gx0 = tx * TX, gy0 = ty * TY + yb, gz0 = tz * TZ;
  if (gy0 >= d.Y) return;  // rows of a brick cut by the volume
  const int tid = int(threadIdx.x), lane = tid & 31, w = tid >> 5;
  const int ncl = int(min(uint32_t(TZ), d.Z - 1 - gz0));  // cube layers of the brick
  const int nb = (ncl + kBatch - 1) / kBatch;
  // this thread's cube column: x = lane, y = w
  const uint32_t cy = gy0 + uint32_t(w);
  const bool row_ok = cy + 1 < d.Y && tx < a.nxc;
  const bool cube_ok = row_ok && gx0 + uint32_t(lane) + 1 < d.X;
  const uint64_t CX = d.X - 1, CXY = uint64_t(d.X - 1) * (d.Y - 1);
  uint8_t* clsp = a.cls + (uint64_t(gx0) + lane + CX * cy + CXY * gz0);
  uint16_t* chp = a.chunk + (uint64_t(cy) + uint64_t(d.Y - 1) * gz0) * a.nxc + tx;
  const uint64_t chstep = uint64_t(d.Y - 1) * a.nxc;
  uint32_t pf[1] = {0};  // corner 0 of this thread's previous cube's top face
  uint32_t pu = 0;       // ... and whether its four labels agree (0 / 1)
  __shared__ uint16_t s_q[RY][kBatch * 32];  // per warp: queued non-uniform cubes (layer << 5 | lane)
  __shared__ uint32_t s_lt[RY][kBatch];      // per warp: record total of each cube layer of the batch
  // ids (a.ids_out): this thread's vertex column
  const bool vert_ok = gx0 + uint32_t(lane) < d.X && cy < d.Y;
  const uint64_t ids_v0 = uint64_t(gx0 + lane) + uint64_t(d.X) * (uint64_t(cy) + uint64_t(d.Y) * gz0);
  if (a.ids_out && vert_ok && ncl == 0 && gz0 == d.Z - 1) {
    // a brick made of the volume's last vertex layer only: no cube layers
    a.ids_out[ids_v0] = brick_token_id(a, __ldg(a.ms + ids_v0));
  }
  if (lane < kBatch) s_lt[w][lane] = 0u;
  if (tid == 0) {
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int b) {
    const uint32_t bar = smem_u32(&s_bar[b & 1]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"(uint32_t(sizeof(Buf)))
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(bufraw[b & 1])),
        "l"(&mtok), "r"(int(gx0)), "r"(int(gy0)), "r"(int(gz0) + b * kBatch), "r"(bar)
        : "memory");
  };
  if (tid == 0 && nb > 0) issue(0);
  // one cube layer; the bottom face is the previous layer's top face, so a
  // cube is uniform iff its top face is, the bottom one was, and one
  // vertical edge agrees. Uniform cubes get class 0 here; the others are
  // queued per warp (layer, lane) and classified after the batch with every
  // lane busy (separator cubes are a few lanes of a row: classifying them
  // in place would run the two-label path at low lane occupancy).
  int qn = 0;  // warp-uniform: queued cubes of this batch
  auto face = [&](const uint32_t(&cur)[RY + 1][TLW], const int cl) {
    bool nu = false;
    if (cube_ok) {
      const uint32_t c4 = cur[w][lane], c5 = cur[w][lane + 1], c6 = cur[w + 1][lane], c7 = cur[w + 1][lane + 1];
      const uint32_t tu = c5 == c4 && c6 == c4 && c7 == c4;
      nu = !((tu & pu) && c4 == pf[0]);
      pf[0] = c4;
      pu = tu;
      if (!nu) *clsp = 0;
    }
    const uint32_t q = __ballot_sync(0xffffffffu, nu);
    if (nu) s_q[w][qn + __popc(q & ((1u << lane) - 1u))] = uint16_t(cl << 5 | lane);
    qn += __popc(q);
    clsp += CXY;
  };
  // the queued cubes of a batch: corners from the staged layers, class byte,
  // record count into the layer's total
  auto classify = [&](const Buf& bb, uint8_t* cls0) {
    for (int i0 = 0; i0 < qn; i0 += 32) {
      if (i0 + lane < qn) {
        const uint32_t e = s_q[w][i0 + lane], cl = e >> 5, x = e & 31u;
        DCHECK(cl < uint32_t(kBatch) && qn <= kBatch * 32, 601);
        uint32_t c[8];
        c[0] = bb[cl][w][x];
        c[1] = bb[cl][w][x + 1];
        c[2] = bb[cl][w + 1][x];
        c[3] = bb[cl][w + 1][x + 1];
        c[4] = bb[cl + 1][w][x];
        c[5] = bb[cl + 1][w][x + 1];
        c[6] = bb[cl + 1][w + 1][x];
        c[7] = bb[cl + 1][w + 1][x + 1];
        // corners equal to corner 0 (bit i)
        uint32_t m8 = 1u;
#pragma unroll
        for (int i = 1; i < 8; ++i) m8 |= uint32_t(c[i] == c[0]) << i;
        // the lowest corner with another label; two labels iff every
        // corner carries one of the two (the common case on a separator)
        uint32_t bl = c[7];
#pragma unroll
        for (int i = 6; i >= 1; --i) bl = (m8 >> i) & 1u ? bl : c[i];
        uint32_t mb = 0u;
#pragma unroll
        for (int i = 1; i < 8; ++i) mb |= uint32_t(c[i] == bl) << i;
        uint32_t cnt, cls;
        if ((m8 | mb) == 0xffu) {
          cnt = g_two_cnt[m8 >> 1];
          cls = m8;
        } else {
          cnt = general_count(c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
          cls = 0xffu;
        }
        cls0[uint64_t(cl) * CXY + x] = uint8_t(cls);
        if (cnt) atomicAdd(&s_lt[w][cl], cnt);
      }
    }
  };
  for (int b = 0; b < nb; ++b) {
    if (tid == 0 && b + 1 < nb) issue(b + 1);  // the other buffer was released by the barrier below
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(&s_bar[b & 1])),
        "r"(uint32_t((b >> 1) & 1))
        : "memory");
    const Buf& bb = *buf[b & 1];
    if (b == 0 && cube_ok) {
      pf[0] = bb[0][w][lane];
      pu = bb[0][w][lane + 1] == pf[0] && bb[0][w + 1][lane] == pf[0] && bb[0][w + 1][lane + 1] == pf[0];
    }
    const int cn = min(kBatch, ncl - b * kBatch);
    uint8_t* const cls0 = clsp - uint64_t(lane);  // class byte of this batch's cube (0, row w, layer 0)
    qn = 0;
    if (cn == kBatch) {
#pragma unroll 2
      for (int cl = 0; cl < kBatch; ++cl) face(bb[cl + 1], cl);
    } else {
#pragma unroll 1
      for (int cl = 0; cl < cn; ++cl) face(bb[cl + 1], cl);
    }
    __syncwarp();
    classify(bb, cls0);
    __syncwarp();
    const uint32_t btot = lane < kBatch ? s_lt[w][lane] : 0u;
    __syncwarp();
    if (lane < kBatch) s_lt[w][lane] = 0u;
    if (a.ids_out && vert_ok) {
      // this thread's vertex column: the batch's bottom layers, and the
      // volume's top layer when the batch ends there
      const int nv = cn + ((gz0 + uint32_t(b * kBatch + cn) == d.Z - 1) ? 1 : 0);
      uint32_t* op = a.ids_out + (ids_v0 + uint64_t(b * kBatch) * d.XY);
      uint32_t lt = ~0u, lid = 0;
      for (int i = 0; i < nv; ++i, op += d.XY) {
        const uint32_t tk = bb[i][w][lane];
        if (tk != lt) {
          lt = tk;
          lid = brick_token_id(a, tk);
        }
        *op = lid;
      }
    }
    // the batch's chunk counts, one store per layer from lanes 0 .. cn-1
    if (lane < cn && row_ok) chp[uint64_t(lane) * chstep] = uint16_t(btot);
    chp += uint64_t(kBatch) * chstep;
    __syncthreads();  // buffer b & 1 is free for batch b + 2
  }
}

#ifndef PLMSS_BRICK_MINB
#define PLMSS_BRICK_MINB 6
#endif
#ifndef PLMSS_TOK_MINB
#define PLMSS_TOK_MINB 4
#endif
__global__ void __launch_bounds__(B_THREADS, PLMSS_BRICK_MINB) k_brick_tma(const __grid_constant__ CUtensorMap mtok,
                                                             const BrickArgs a) {
  __shared__ __align__(128) unsigned char smem[kBrickSmem];
  brick_tma_body(mtok, a, blockIdx.x, smem);
}

template <bool kDense, int kMode = 0>
__global__ void __launch_bounds__(32 * kTokRows, PLMSS_TOK_MINB) k_tokens_tma(const __grid_constant__ CUtensorMap mlt,
                                                                const BrickArgs a) {
  __shared__ __align__(128) unsigned char smem[kTokSmem];
  tokens_tma_body<kDense, kMode>(mlt, a, blockIdx.x, smem);
}

// Pass C, one launch per brick z-layer s: the tokens of layer s and the
// count pass of layer s - 2 (whose tokens and following layer are complete),
// CTAs interleaved so that the memory-bound token work and the issue-bound
// cube classification share every SM.
static_assert(TY / kTokRows == TY / RY && 32 * kTokRows == B_THREADS, "token and count items must match");
template <int kMode = 0>
__global__ void __launch_bounds__(B_THREADS, 5) k_slab_tma(const __grid_constant__ CUtensorMap mlt,
                                                           const __grid_constant__ CUtensorMap mtok,
                                                           const BrickArgs ta, const BrickArgs ca) {
  __shared__ __align__(128) unsigned char smem[kTokSmem > kBrickSmem ? kTokSmem : kBrickSmem];
  if (blockIdx.x & 1)
    brick_tma_body(mtok, ca, blockIdx.x >> 1, smem);
  else
    tokens_tma_body<true, kMode>(mlt, ta, blockIdx.x >> 1, smem);
}

// Region token -> dense MS id.
template <bool kDense>
__device__ __forceinline__ uint32_t token_id(uint32_t k, const uint32_t* __restrict__ bitmap,
                                             const uint32_t* __restrict__ prefix, const uint32_t* __restrict__ slot_id) {
  if (kDense) return __ldg(prefix + (k >> 5)) + __popc(__ldg(bitmap + (k >> 5)) & ((1u << (k & 31)) - 1u));
  return __ldg(slot_id + k);
}

// Record total of every group of 32 consecutive chunks (the emit warps'
// unit), scanned into the groups' record offsets.
__global__ void __launch_bounds__(256) k_group_sums(const uint16_t* __restrict__ cnt, uint64_t nchunks,
                                                    uint64_t* __restrict__ gsum) {
  const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t c0 = g * 32;
  if (c0 >= nchunks) return;
  uint32_t t = 0;
  if (c0 + 32 <= nchunks) {
    const uint4* p = reinterpret_cast<const uint4*>(cnt + c0);  // 64-byte aligned
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 v = __ldg(p + k);
      t += (v.x & 0xffffu) + (v.x >> 16) + (v.y & 0xffffu) + (v.y >> 16) + (v.z & 0xffffu) + (v.z >> 16) +
           (v.w & 0xffffu) + (v.w >> 16);
    }
  } else {
    for (uint64_t c = c0; c < nchunks; ++c) t += cnt[c];
  }
  gsum[g] = t;
}

// group record offsets (exclusive) into gbase; returns the record total
uint64_t group_offsets(Ctx& c, const uint16_t* cnt, uint64_t nchunks, uint64_t* gbase) {
  const uint64_t ngroups = (nchunks + 31) / 32;
  k_group_sums<<<unsigned((ngroups + 255) / 256), 256, 0, c.stream>>>(cnt, nchunks, gbase);
  CK_LAUNCH("k_group_sums");
  return exclusive_scan_u64(c, gbase, int64_t(ngroups), true);
}

// Emission grid: warp tasks of whole 32-chunk groups, split into 2, 4, .. 32
// tasks per group while there are fewer than ~256 warp tasks per SM (small
// volumes: cfg1 has 248 groups of ~13 k records each). Sets ea.cshift.
struct EmitArgs;
unsigned emit_grid(const Ctx& c, EmitArgs& ea);

struct EmitArgs {
  uint32_t X, Y, Z, nxc;
  uint64_t nchunks, total;
  uint64_t cube0;        // global id of cube 0 (z-slab pipeline; 0 otherwise)
  const uint16_t* cnt;   // records per chunk
  const uint64_t* gbase; // exclusive record offset of every group of 32 chunks
  uint32_t cshift;       // a warp task = 32 >> cshift chunks of a group (small volumes: more tasks)
  const uint8_t* cls;
  const uint32_t* ids;   // ms (dense MS ids)
  plmss_tri* out;
};

// Pass D: separator records of every chunk with records, at its offset, in
// the reference order (cube-major, tets in order, recipe rows in order:
// marching.cpp:116-215). Warps walk whole cube rows; lane = cube of the chunk;
// records are dealt out one per lane (consecutive lanes write consecutive
// 16-byte records).
// Rare emission paths (cubes with three or more labels), out of line: the
// tet codes with the record count (count << 32 | codes), and a record's tet,
// recipe row and the two cube corners whose labels it separates
// (t | rowi << 8 | corner a << 16 | corner b << 24).
__device__ __noinline__ uint64_t general_codes(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t c4,
                                               uint32_t c5, uint32_t c6, uint32_t c7) {
  const uint32_t c[8] = {c0, c1, c2, c3, c4, c5, c6, c7};
  uint32_t cnt = 0;
  const uint32_t code6 = cube_codes(c, g_tlut, cnt);
  return uint64_t(cnt) << 32 | code6;
}
__device__ __noinline__ uint32_t general_record(uint32_t c6, uint32_t k) {
  uint32_t t = 0;
  uint32_t cs = g_cases[c6 & 31];
#pragma unroll
  for (int tt = 0; tt < 5; ++tt) {
    if (k < (cs & 15)) break;
    k -= cs & 15;
    ++t;
    cs = g_cases[(c6 >> (5 * t)) & 31];
  }
  const uint32_t rowi = (cs >> 4) + k;
  const uint32_t row = g_rows[rowi];
  // tet t = cube corners {0, cb, cc, 7}
  const uint32_t cb = (0x442211u >> (4 * t)) & 15, cc = (0x656353u >> (4 * t)) & 15;
  auto corner = [&](uint32_t p) { return p == 0 ? 0u : (p == 1 ? cb : (p == 2 ? cc : 7u)); };
  return t | rowi << 8 | corner((row >> 12) & 3) << 16 | corner((row >> 14) & 3) << 24;
}

// kSplit: warp tasks of 32 >> cshift chunks (small volumes), else whole groups
template <bool kSplit>
__global__ void __launch_bounds__(256) k_emit_chunks(const EmitArgs a) {
  __shared__ uint8_t s_own[256 / 32][32];  // record window position -> lane of the cube starting there
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t CX = a.X - 1, CY = a.Y - 1, XY = a.X * a.Y;
  const uint64_t ngroups = (a.nchunks + 31) / 32;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
  auto corner_off = [&](uint32_t cn) { return (cn & 1) + a.X * ((cn >> 1) & 1) + XY * (cn >> 2); };
  // warps take groups of 32 consecutive chunks; one coalesced load of their
  // offsets and one division per lane for their coordinates, then only the
  // chunks with records
  // (nchunks < 2^32: task and group indices fit 32 bits)
  const uint32_t cshift = kSplit ? a.cshift : 0u;
  const uint64_t ntasks = ngroups << cshift;
  const uint32_t tmask = 0xffffffffu >> (32u - (32u >> cshift));  // this task's chunks, before the shift
  for (uint64_t task = uint64_t(blockIdx.x) * (blockDim.x / 32) + wib; task < ntasks; task += warps) {
    const uint64_t grp = task >> cshift;
    const uint64_t chl = grp * 32 + uint64_t(lane);
    const uint32_t ccnt = chl < a.nchunks ? uint32_t(a.cnt[chl]) : 0u;
    uint32_t todo = __ballot_sync(0xffffffffu, ccnt != 0);
    if (kSplit) todo &= tmask << ((uint32_t(task) << (5u - cshift)) & 31u);
    if (!todo) continue;
    // the chunk's offset: the group's base plus the warp's exclusive prefix
    uint32_t cinc = ccnt;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, cinc, s);
      if (lane >= s) cinc += t;
    }
    const uint64_t my_off = __ldg(a.gbase + grp) + (cinc - ccnt);
    // this lane's chunk: cube row r = (cz, cy), x segment xs (nchunks < 2^32)
    const uint32_t c32 = uint32_t(chl), r_l = c32 / a.nxc, xs_l = c32 - r_l * a.nxc;
    const uint32_t cz_l = r_l / CY, cy_l = r_l - cz_l * CY;
    const uint32_t x0_l = 32 * xs_l;
    const uint32_t v0_l = x0_l + a.X * cy_l + XY * cz_l;  // min corner of the chunk's first cube
    const uint32_t q0_l = x0_l + CX * r_l;  // cube ids < n < 2^32
    const uint32_t T_l = ccnt;
    // one busy chunk ahead: its classes and the ids of its cubes' four
    // corner rows (lane i: corners 0, 2, 4, 6 of cube i; corners 1, 3, 5, 7
    // come from lane i + 1, lane 31 loads them) are loaded while the current
    // chunk is emitted
    struct Pre {
      uint32_t cls, v0, q0, r[4], e[4];
    };
    const uint32_t X = a.X;
    auto fetch = [&](int k, Pre& p) {
      const uint32_t cx = __shfl_sync(0xffffffffu, x0_l, k) + uint32_t(lane);
      p.v0 = __shfl_sync(0xffffffffu, v0_l, k) + uint32_t(lane);
      p.q0 = __shfl_sync(0xffffffffu, q0_l, k);
      const uint32_t v0 = p.v0;
      p.cls = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) p.r[i] = p.e[i] = 0;
      if (cx <= CX) {  // the vertex past the last cube is that cube's corner 1
        p.r[0] = __ldg(a.ids + v0);
        p.r[1] = __ldg(a.ids + (v0 + X));
        p.r[2] = __ldg(a.ids + (v0 + XY));
        p.r[3] = __ldg(a.ids + (v0 + XY + X));
      }
      if (cx < CX) {
        p.cls = a.cls[p.q0 + uint32_t(lane)];
        if (lane == 31) {
          p.e[0] = __ldg(a.ids + (v0 + 1));
          p.e[1] = __ldg(a.ids + (v0 + X + 1));
          p.e[2] = __ldg(a.ids + (v0 + XY + 1));
          p.e[3] = __ldg(a.ids + (v0 + XY + X + 1));
        }
      }
    };
    int kc = __ffs(todo) - 1;
    todo &= todo - 1;
    Pre cur;
    fetch(kc, cur);
    for (;;) {
      const bool more = todo != 0;  // warp-uniform
      int kn = 0;
      Pre nxt;
      if (more) {
        kn = __ffs(todo) - 1;
        todo &= todo - 1;
        fetch(kn, nxt);
      }
      const uint64_t base = __shfl_sync(0xffffffffu, my_off, kc);
      const uint32_t T = __shfl_sync(0xffffffffu, T_l, kc);
      const uint32_t q0 = cur.q0;  // cube id of lane 0's cube
      const uint32_t v0 = cur.v0;  // this lane's min corner
      const uint32_t cls = cur.cls;
      uint32_t c[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        c[2 * i] = cur.r[i];
        const uint32_t nb = __shfl_down_sync(0xffffffffu, cur.r[i], 1);
        c[2 * i + 1] = lane == 31 ? cur.e[i] : nb;
      }
      uint32_t cnt = 0, code6 = 0, lo2 = 0, hi2 = 0;
      if (cls == 0xffu) {
        const uint64_t g = general_codes(c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
        code6 = uint32_t(g);
        cnt = uint32_t(g >> 32);
      } else if (cls != 0) {
        // two labels: corner 0's and that of the lowest corner outside its set
        cnt = g_two_cnt[cls >> 1];
        code6 = 0x80000000u | cls;
        uint32_t ib = c[7];
#pragma unroll
        for (int i = 6; i >= 1; --i) ib = (cls >> i) & 1u ? ib : c[i];
        lo2 = min(c[0], ib);
        hi2 = max(c[0], ib);
      }
      uint32_t inc = cnt;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, s);
        if (lane >= s) inc += t;
      }
      const uint32_t ex = inc - cnt;  // this cube's first record
      int carry = 0;                  // owner of the window's records before its first start
      for (uint32_t j0 = 0; j0 < T; j0 += 32) {
        // owner of record j0 + lane = the cube with the last start at or before it
        const bool st = cnt != 0 && ex - j0 < 32u;
        if (st) s_own[wib][ex - j0] = uint8_t(lane);
        const uint32_t S = __reduce_or_sync(0xffffffffu, st ? 1u << (ex - j0) : 0u);
        __syncwarp();
        const uint32_t m = S & (0xffffffffu >> (31 - lane));
        const int src = m ? int(s_own[wib][31 - __clz(m)]) : carry;
        carry = __shfl_sync(0xffffffffu, src, 31);
        __syncwarp();
        const uint32_t j = j0 + uint32_t(lane);
        const uint32_t c6 = __shfl_sync(0xffffffffu, code6, src);
        const uint32_t exs = __shfl_sync(0xffffffffu, ex, src);
        const uint32_t l2 = __shfl_sync(0xffffffffu, lo2, src);
        const uint32_t h2 = __shfl_sync(0xffffffffu, hi2, src);
        if (j >= T) continue;
        uint32_t k = j - exs;
        uint32_t t, rowi, la, lb;
        if (c6 >> 31) {
          // two-label cube: record list from the table, one region pair
          const uint32_t e = g_two_rec[((c6 & 0xffu) >> 1) * 12 + k];
          t = e >> 8;
          rowi = e & 0xffu;
          la = l2;
          lb = h2;
        } else {
          const uint32_t r = general_record(c6, k);
          t = r & 0xffu;
          rowi = (r >> 8) & 0xffu;
          const uint32_t vs = v0 - uint32_t(lane) + uint32_t(src);
          la = __ldg(a.ids + (vs + corner_off((r >> 16) & 0xffu)));
          lb = __ldg(a.ids + (vs + corner_off(r >> 24)));
        }
        const uint64_t cr64 = ((6ull * (a.cube0 + uint64_t(q0 + uint32_t(src))) + t) << 6) | uint64_t(rowi);
        DCHECK(base + j < a.total, 501);
        *reinterpret_cast<uint4*>(a.out + base + j) =
            make_uint4(uint32_t(cr64), uint32_t(cr64 >> 32), min(la, lb), max(la, lb));
      }
      if (!more) break;
      kc = kn;
      cur = nxt;
    }
  }
}

unsigned emit_grid(const Ctx& c, EmitArgs& ea) {
  const uint64_t ngroups = (ea.nchunks + 31) / 32, target = uint64_t(c.sm_count) * 256;
  ea.cshift = 0;
  while (ea.cshift < 5 && (ngroups << ea.cshift) < target) ++ea.cshift;
  const uint64_t tasks = ngroups << ea.cshift;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((tasks + 7) / 8, uint64_t(c.sm_count) * 256)));
}

// ms: region token -> dense id, in place (4 vertices per thread, the last
// lookup cached: runs of one region are the norm).
template <bool kDense>
__global__ void __launch_bounds__(256) k_ms_ids(uint32_t* __restrict__ ms, uint64_t n,
                                                const uint32_t* __restrict__ bitmap,
                                                const uint32_t* __restrict__ prefix,
                                                const uint32_t* __restrict__ slot_id) {
  const uint64_t i0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i0 >= n) return;
  uint32_t lt = ~0u, lid = 0;
  if (i0 + 4 <= n) {
    uint4 v = *reinterpret_cast<const uint4*>(ms + i0);
    uint32_t* e = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e[k] != lt) {
        lt = e[k];
        lid = token_id<kDense>(lt, bitmap, prefix, slot_id);
      }
      e[k] = lid;
    }
    *reinterpret_cast<uint4*>(ms + i0) = v;
  } else {
    for (uint64_t i = i0; i < n; ++i) ms[i] = token_id<kDense>(ms[i], bitmap, prefix, slot_id);
  }
}

// ------------------------------------------------- z-slab pipeline (e) --
// A rank's slab is a grid of its own (owned layers, local vertex ids) whose
// field buffer carries the neighbours' boundary layers as halos; chains that
// leave the slab end at portal entries (k_tt_succ), resolved across ranks
// through the gathered boundary layers (k_slab_patch).

// Resolved value of the owned first (side 0) / last (side 1) layer vertex
// (x, y): [desc first, desc last, asc first, asc last] x XY words, each
// kFinal | slab-local rank, or kFinal | kPortal | portal index.
__global__ void k_slab_boundary(const FDims d, const uint4* __restrict__ TB, const uint32_t* __restrict__ lt,
                                const uint32_t* __restrict__ SD,
                                const uint32_t* __restrict__ SA, uint32_t* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 2ull * d.XY) return;
  const uint32_t side = uint32_t(i / d.XY), xy = uint32_t(i - uint64_t(side) * d.XY);
  const uint32_t x = xy % d.X, y = xy / d.X, z = side ? d.Z - 1 : 0;
  const uint32_t bt = (x >> 5) + d.tx * ((y >> 5) + d.ty * (z >> 5));
  const uint32_t bm = bt << 15 | (x & 31) | (y & 31) << 5 | (z & 31) << 10;
  const uint32_t base = __ldg(reinterpret_cast<const uint32_t*>(TB) + 4 * bt);
  const uint32_t l = __ldg(lt + bm);
  out[i] = SD[base + (l & 0xffffu)];
  out[2ull * d.XY + i] = SA[base + (l >> 16)];
}

// The final value of portal p of rank r: follow it through the gathered
// boundary layers G[world][4][XY] (steepest chains are strictly monotone, so
// the walk ends) and offset the extremum's slab rank by its rank's prefix.
__device__ uint32_t slab_chase(const uint32_t* __restrict__ G, uint32_t dir, int r, uint32_t p, uint32_t XY,
                               int world, const uint32_t* __restrict__ pre, int* __restrict__ err) {
#pragma unroll 1
  for (int it = 0; it < (1 << 24); ++it) {
    const uint32_t side = p >= XY ? 1u : 0u, xy = p - side * XY;
    const int r2 = side ? r + 1 : r - 1;  // the rank owning the halo layer
    if (r2 < 0 || r2 >= world) break;
    // its first layer when the chain went up, its last when it went down
    const uint32_t v = __ldg(G + (uint64_t(r2) * 4 + dir * 2 + (side ? 0u : 1u)) * XY + xy);
    if (!(v & kFinal)) break;
    if (!(v & kPortal)) return kFinal | ((v & ~kFinal) + __ldg(pre + r2));
    r = r2;
    p = v & ~(kFinal | kPortal);
  }
  atomicExch(err, 1);
  return kFinal;
}

// Every table entry of this rank -> kFinal | global extremum rank.
__global__ void k_slab_patch(uint64_t nt, uint32_t* __restrict__ SD, uint32_t* __restrict__ SA,
                             const uint32_t* __restrict__ G, int world, int rank, uint32_t XY,
                             const uint32_t* __restrict__ pre_max, const uint32_t* __restrict__ pre_min,
                             int* __restrict__ err) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  uint32_t* S[2] = {SD, SA};
  const uint32_t* pre[2] = {pre_max, pre_min};
#pragma unroll
  for (uint32_t dir = 0; dir < 2; ++dir) {
    uint32_t v = S[dir][i];
    if (!(v & kFinal)) {
      atomicExch(err, 2);  // the slab forest had not converged
      continue;
    }
    if (v & kPortal)
      v = slab_chase(G, dir, rank, v & ~(kFinal | kPortal), XY, world, pre[dir], err);
    else
      v = kFinal | ((v & ~kFinal) + __ldg(pre[dir] + rank));
    S[dir][i] = v;
  }
}

// Dense region bitmap from gathered rank-pair keys (rank_min << 32 | rank_max).
__global__ void k_set_bits(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ bitmap,
                           uint32_t nmax) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  const uint64_t b = (k >> 32) * uint64_t(nmax) + uint32_t(k);
  const uint32_t bit = 1u << (b & 31);
  uint32_t* w = bitmap + (b >> 5);
  if (!(*w & bit)) atomicOr(w, bit);
}

// sorted keys -> 1 at the first occurrence of each value
__global__ void k_first_flags(const uint64_t* __restrict__ k, int64_t n, uint64_t* __restrict__ flags) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}
__global__ void k_compact_first(const uint64_t* __restrict__ k, int64_t n, const uint64_t* __restrict__ pos,
                                uint64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && (i == 0 || k[i] != k[i - 1])) out[pos[i]] = k[i];
}

// hash mode: every occupied slot of the slab's region set -> its position in
// the global sorted unique keys
__global__ void k_slot_ids(const unsigned long long* __restrict__ fset, uint64_t fcap,
                           const uint64_t* __restrict__ ukeys, int64_t R, uint32_t* __restrict__ slot_id) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= fcap) return;
  const unsigned long long k = fset[i];
  if (k == kEmpty) return;
  int64_t lo = 0, hi = R;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (__ldg(ukeys + m) < k) lo = m + 1; else hi = m;
  }
  slot_id[i] = uint32_t(lo);
}

std::atomic<bool> g_consts_ready[64] = {};
std::mutex g_consts_mu;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn tensor_map_encoder() {
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<EncodeFn>(fn);
  }
  return encode;
}

// LT as a 2-D tensor (1024 cells of a brick layer, ntiles * 32 layers) for
// the token pass: one box = 8 rows x 32 layers of a brick
bool encode_lt_map(Ctx& c, uint64_t ntiles, uint32_t* lt, CUtensorMap* mlt) {
  if (!c.use_tma || !tensor_map_encoder()) return false;
  const cuuint64_t gdim[2] = {cuuint64_t(TX * TY), cuuint64_t(ntiles) * TZ};
  const cuuint64_t gstride[1] = {cuuint64_t(TX * TY) * 4};
  const cuuint32_t box[2] = {cuuint32_t(32 * kTokRows), cuuint32_t(TZ)};
  const cuuint32_t estride[2] = {1, 1};
  return tensor_map_encoder()(mlt, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, lt, gdim, gstride, box, estride,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Host driver of the fused pipeline. Returns false when the dims are outside
// the fused path's envelope (then the caller uses the staged kernels).
bool fused_supported(const Grid& g) {
  // u32 vertex ids, and u32 brick-major cell indices (bricks padded to 32^3)
  const int64_t bricks = ((g.X + TX - 1) / TX) * ((g.Y + TY - 1) / TY) * ((g.Z + TZ - 1) / TZ);
  return g.n < (int64_t(1) << 32) - 1 && bricks * TN <= (int64_t(1) << 32);
}

// One-time per device: kernel attributes, recipe tables, marching tables.
static void ensure_consts(Ctx& c) {
  if (c.device >= 0 && c.device < 64 && !g_consts_ready[c.device].load(std::memory_order_acquire)) {
    // one upload per device even when several host threads arrive together
    std::lock_guard<std::mutex> lock(g_consts_mu);
    if (!g_consts_ready[c.device].load(std::memory_order_acquire)) {
      CK(cudaFuncSetAttribute(k_tile_segment<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kASmem));
      CK(cudaFuncSetAttribute(k_tile_segment<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kASmem));
      CK(cudaFuncSetAttribute(k_tile_segment<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kASmem));
      CK(cudaFuncSetAttribute(k_hop_codes<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmem));
      CK(cudaFuncSetAttribute(k_hop_codes<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmem));
      CK(cudaFuncSetAttribute(k_hop_codes<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmem));
      CK(cudaFuncSetAttribute(k_tile_segment<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kASmem));
      CK(cudaFuncSetAttribute(k_tile_segment<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kASmem));
      CK(cudaFuncSetAttribute(k_hop_codes<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmem));
      // on the context stream (a non-blocking stream does not wait on the legacy one)
      CK(cudaMemcpyToSymbolAsync(c_mrows, kTetRowsPacked, sizeof(kTetRowsPacked), 0, cudaMemcpyHostToDevice,
                                 c.stream));
      CK(cudaMemcpyToSymbolAsync(c_mcases, kTetCasePacked, sizeof(kTetCasePacked), 0, cudaMemcpyHostToDevice,
                                 c.stream));
      k_march_init<<<1, 128, 0, c.stream>>>();
      CK_LAUNCH("k_march_init");
      c.sync();  // other contexts (other streams) may use the tables next
      g_consts_ready[c.device].store(true, std::memory_order_release);
    }
  }
}

// Pass A launch: the fused kernel, or (PLMSS_OPT_PASS_A_SPLIT) the hop-code
// kernel followed by the brick compression fed by the codes.
static void launch_pass_a(Ctx& c, const FDims& d, uint64_t ntiles, bool use_tma, const CUtensorMap& tmap,
                          const float* field, uint32_t* maxima, uint32_t* minima, uint32_t* max_tt, uint32_t* min_tt,
                          uint64_t ext_cap, uint32_t* TT, uint64_t tt_cap, uint4* TB, uint32_t* lt,
                          ACounters* ctr) {
  const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(c.sm_count)));
  if (c.pass_a_split) {
    uint8_t* codes = c.get_t<uint8_t>(S_CODES, ntiles * TN);
    CUtensorMap hmap;
    memset(&hmap, 0, sizeof hmap);
    bool hop_tma = false;
    if (use_tma) {
      const cuuint64_t gdim[3] = {cuuint64_t(d.X), cuuint64_t(d.Y), cuuint64_t(d.zfn)};
      const cuuint64_t gstride[2] = {cuuint64_t(d.X) * 4, cuuint64_t(d.X) * cuuint64_t(d.Y) * 4};
      const cuuint32_t box[3] = {HX, HR + 2, HZ};
      const cuuint32_t estride[3] = {1, 1, 1};
      hop_tma = tensor_map_encoder()(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(field), gdim,
                                     gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA) == CUDA_SUCCESS;
    }
    const unsigned hgrid = unsigned(ntiles * (TY / HR));
    if (hop_tma && c.hop_cube)
      k_hop_codes<true, true><<<hgrid, 32 * HR, kCSmem, c.stream>>>(hmap, field, d, codes, ctr);
    else if (hop_tma)
      k_hop_codes<true><<<hgrid, 32 * HR, kCSmem, c.stream>>>(hmap, field, d, codes, ctr);
    else if (c.hop_cube)
      k_hop_codes<false, true><<<hgrid, 32 * HR, kCSmem, c.stream>>>(hmap, field, d, codes, ctr);
    else
      k_hop_codes<false><<<hgrid, 32 * HR, kCSmem, c.stream>>>(hmap, field, d, codes, ctr);
    CK_LAUNCH("k_hop_codes");
    k_tile_segment<false, true><<<grid, A_THREADS, kASmem, c.stream>>>(
        tmap, field, codes, d, maxima, minima, max_tt, min_tt, ext_cap, TT, tt_cap, TB, lt, ctr);
    CK_LAUNCH("k_tile_segment");
    return;
  }
  if (use_tma && c.hop_cube)
    k_tile_segment<true, false, true><<<grid, A_THREADS, kASmem, c.stream>>>(
        tmap, field, nullptr, d, maxima, minima, max_tt, min_tt, ext_cap, TT, tt_cap, TB, lt, ctr);
  else if (use_tma)
    k_tile_segment<true><<<grid, A_THREADS, kASmem, c.stream>>>(tmap, field, nullptr, d, maxima, minima, max_tt,
                                                                min_tt, ext_cap, TT, tt_cap, TB, lt, ctr);
  else if (c.hop_cube)
    k_tile_segment<false, false, true><<<grid, A_THREADS, kASmem, c.stream>>>(
        tmap, field, nullptr, d, maxima, minima, max_tt, min_tt, ext_cap, TT, tt_cap, TB, lt, ctr);
  else
    k_tile_segment<false><<<grid, A_THREADS, kASmem, c.stream>>>(tmap, field, nullptr, d, maxima, minima, max_tt,
                                                                 min_tt, ext_cap, TT, tt_cap, TB, lt, ctr);
  CK_LAUNCH("k_tile_segment");
}

// Checked build: fail on the first device bounds check that did not hold.
static void check_device(Ctx& c, const char* where) {
#ifdef PLMSS_CHECKED
  unsigned long long v = 0;
  CK(cudaMemcpyFromSymbolAsync(&v, g_check_fail, sizeof v, 0, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (v) {
    const unsigned long long zero = 0;
    CK(cudaMemcpyToSymbolAsync(g_check_fail, &zero, sizeof zero, 0, cudaMemcpyHostToDevice, c.stream));
    c.sync();
    fail(PLMSS_ERR_LOGIC, std::string("device bounds check ") + std::to_string(v) + " failed in " + where);
  }
#else
  (void)c;
  (void)where;
#endif
}

FusedOut fused_pipeline(Ctx& c, const Grid& g, const float* field, uint32_t* desc, uint32_t* asc, uint32_t* ms) {
  FusedOut o{};
  for (auto& s : c.stats) s = 0;
  ensure_consts(c);
  FDims d{};
  d.X = uint32_t(g.X);
  d.Y = uint32_t(g.Y);
  d.Z = uint32_t(g.Z);
  d.XY = d.X * d.Y;
  d.n = uint32_t(g.n);
  d.tx = uint32_t((g.X + TX - 1) / TX);
  d.ty = uint32_t((g.Y + TY - 1) / TY);
  d.tz = uint32_t((g.Z + TZ - 1) / TZ);
  d.zf0 = 0;
  d.zfn = d.Z;
  d.pbase = 0;
  const uint64_t ntiles = uint64_t(d.tx) * d.ty * d.tz;

  // TMA descriptor of the field (3-D, float32, NaN out-of-bounds fill). The
  // global row pitch must be a 16-byte multiple, i.e. X % 4 == 0; otherwise
  // the brick is staged by an unrolled load loop.
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  bool use_tma = (g.X % 4) == 0 && (reinterpret_cast<uintptr_t>(field) & 15) == 0 && c.use_tma;
  if (use_tma) {
    const EncodeFn encode = tensor_map_encoder();
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
  uint32_t* lt = c.get_t<uint32_t>(S_LTD, ntiles * (TN + kFaceX));  // desc | asc << 16, then the x faces
  // LT as a 2-D tensor (1024 cells of a brick layer, ntiles * 32 layers) for
  // the token pass: one box = 8 rows x 32 layers of a brick
  CUtensorMap mlt;
  const bool lt_tma = encode_lt_map(c, ntiles, lt, &mlt);
  uint4* TB = c.get_t<uint4>(S_TB, ntiles);
  for (int attempt = 0;; ++attempt) {
    const uint64_t ext_cap = c.fused_ext_cap ? c.fused_ext_cap : uint64_t(g.n / 4 + 1024);
    uint32_t* maxima = c.get_t<uint32_t>(S_MAXIMA, ext_cap);
    uint32_t* minima = c.get_t<uint32_t>(S_MINIMA, ext_cap);
    uint32_t* max_tt = c.get_t<uint32_t>(S_RANK_MAX, ext_cap);
    uint32_t* min_tt = c.get_t<uint32_t>(S_RANK_MIN, ext_cap);
    const uint64_t tt_cap = c.fused_exit_cap ? c.fused_exit_cap : uint64_t(g.n / 4 + 1024);
    uint32_t* TT = c.get_t<uint32_t>(S_TMP0, tt_cap);
    CK(cudaMemsetAsync(ctr, 0, sizeof(ACounters), c.stream));
    CK(cudaMemsetAsync(&ctr->bad, 0xff, 4, c.stream));
    c.mark(0);
    launch_pass_a(c, d, ntiles, use_tma, tmap, field, maxima, minima, max_tt, min_tt, ext_cap, TT, tt_cap, TB, lt,
                  ctr);
    c.mark(1);
    ACounters h;
    CK(cudaMemcpyAsync(c.h_pinned, ctr, sizeof(ACounters), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    memcpy(&h, c.h_pinned, sizeof h);
    if (h.bad != 0xffffffffu)
      fail(PLMSS_ERR_INVALID_ARGUMENT, "non-finite scalar value at vertex " + std::to_string(h.bad));
    bool retry = false;
    if (h.n_tt > tt_cap) {
      c.fused_exit_cap = h.n_tt + h.n_tt / 4 + 1024;
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
    const uint64_t nt = h.n_tt;
    // ---- extrema lists sorted ascending; rank of every extremum table entry
    uint32_t* RK = c.get_t<uint32_t>(S_RK, nt);
    sort_extrema(c, maxima, max_tt, o.n_max, minima, min_tt, o.n_min, uint64_t(g.n), RK, 0u);
    c.mark(2);
    // ---- B: terminal-table forest -> extremum rank of every table entry
    uint32_t* SD = c.get_t<uint32_t>(S_SD, nt);
    uint32_t* SA = c.get_t<uint32_t>(S_SA, nt);
    k_tt_succ<<<unsigned(ntiles), 256, 0, c.stream>>>(TB, TT, lt, RK, SD, SA, 0u, nt);
    CK_LAUNCH("k_tt_succ");
    // Two sweeps are enqueued without waiting (they converge on smooth
    // fields); passes C and D follow speculatively and the convergence flag
    // of the last sweep is checked at the end — if it is set, the sweeps
    // continue to the fixpoint and C, D are redone.
    int* jflag = reinterpret_cast<int*>(ctr_base + 192);
    o.sweeps = 0;
    auto sweep = [&]() {
      CK(cudaMemsetAsync(jflag, 0, 4, c.stream));
      k_tt_jump<<<blocks_for(int64_t((nt + 1) / 2), 256), 256, 0, c.stream>>>(nt, SD, SA, jflag);
      CK_LAUNCH("k_tt_jump");
      ++o.sweeps;
    };
    if (c.spec_sweeps == 0) CK(cudaMemsetAsync(jflag, 0xff, 4, c.stream));  // "not converged"
    for (int i = 0; i < c.spec_sweeps; ++i) sweep();
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(c.h_pinned) + 64, jflag, 4, cudaMemcpyDeviceToHost, c.stream));
    for (int pass = 0;; ++pass) {
    c.mark(3);
    // ---- C: region tokens, desc/asc, cube classes, separator counts per chunk
    BrickArgs ba{};
    ba.d = d;
    ba.nxc = uint32_t((g.X - 1 + 31) / 32);
    ba.TB = TB;
    ba.lt = lt;
    ba.FD = SD;
    ba.FA = SA;
    ba.maxs = maxima;
    ba.mins = minima;
    ba.nmax = uint32_t(o.n_max);
    ba.nmin = uint32_t(o.n_min);
    ba.nt = nt;
    ba.desc = desc;
    ba.asc = asc;
    ba.ms = ms;
    ba.overflow = flag;
    const uint64_t nchunks = uint64_t(ba.nxc) * uint64_t(g.Y - 1) * uint64_t(g.Z - 1);
    uint16_t* chunk = c.get_t<uint16_t>(S_TMP1, nchunks ? nchunks : 1);
    ba.chunk = chunk;
    ba.cls = c.get_t<uint8_t>(S_MASK, uint64_t(g.cubes ? g.cubes : 1));
    const unsigned cgrid = unsigned((TY / RY) * ntiles);
    const unsigned tgrid = unsigned((TY / kTokRows) * ntiles);
    // tokens as a 3-D tensor for the count pass: in ms (ids rewritten in
    // place by k_ms_ids), or (PLMSS_OPT_IDS_IN_COUNT) in a scratch array the
    // count pass translates into ms
    // PLMSS_OPT_IDS_IN_COUNT 2 (mark mode, dense keys with TMA): a mark pass
    // builds the region bitmap from LT and the tables alone, so the token
    // pass writes dense ids straight into ms and the count pass (no id
    // writes) runs interleaved with it, layer by layer
    const bool mark_mode = c.ids_mode == 2 && lt_tma && (g.X % 4) == 0 &&
                           uint64_t(o.n_max) * uint64_t(o.n_min) < (uint64_t(1) << 32) && c.combine_path != 2;
    const bool ids_in_count = !mark_mode && c.ids_mode != 0;
    uint32_t* tokbuf = ids_in_count ? c.get_t<uint32_t>(S_TOKENS, uint64_t(g.n)) : ms;
    ba.ms = tokbuf;
    // (the count pass writing the labels from the tokens, the token pass
    // skipping them, measured slower on cfg5: 7.36 vs 7.22 ms for the two
    // passes, so the token pass writes them)
    CUtensorMap mtok;
    bool tok_tma = lt_tma && (g.X % 4) == 0;
    if (tok_tma) {
      const cuuint64_t gdim[3] = {cuuint64_t(g.X), cuuint64_t(g.Y), cuuint64_t(g.Z)};
      const cuuint64_t gstride[2] = {cuuint64_t(g.X) * 4, cuuint64_t(g.X) * cuuint64_t(g.Y) * 4};
      const cuuint32_t box[3] = {cuuint32_t(TLW), cuuint32_t(RY + 1), cuuint32_t(kBatch + 1)};
      const cuuint32_t estride[3] = {1, 1, 1};
      tok_tma = tensor_map_encoder()(&mtok, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, tokbuf, gdim, gstride, box, estride,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                CUDA_SUCCESS;
    }
    const uint64_t nbits = uint64_t(o.n_max) * uint64_t(o.n_min);
    const bool dense = nbits < (uint64_t(1) << 32) && c.combine_path != 2;  // PLMSS_OPT_COMBINE_PATH 2: hash
    uint64_t* keys = nullptr;
    int64_t R = 0;
    uint32_t *bitmap = nullptr, *prefix = nullptr, *slot_id = nullptr;
    if (dense) {
      // rank-product bitmap: no hashing, ids by prefix popcount
      const uint64_t nw = (nbits + 31) / 32;
      bitmap = c.get_t<uint32_t>(S_BITMAP, nw);
      CK(cudaMemsetAsync(bitmap, 0, nw * 4, c.stream));
      ba.bitmap = bitmap;
      ba.nw = nw;
      // z-slab pipeline: tokens of brick layer s on the main stream; the
      // count pass of layer s-1 (which reads layer s's first vertex layer)
      // on the side stream as soon as they are written
      const uint32_t bpl = d.tx * d.ty;
      const unsigned items = bpl * (TY / kTokRows);
      if (mark_mode) {
        k_tokens_tma<true, 1><<<tgrid, 32 * kTokRows, 0, c.stream>>>(mlt, ba);
        CK_LAUNCH("k_mark");
      } else if (ids_in_count) {
        // all tokens first; the count pass (ids) runs once the set is complete
        if (lt_tma)
          k_tokens_tma<true><<<tgrid, 32 * kTokRows, 0, c.stream>>>(mlt, ba);
        else
          k_tokens<true><<<tgrid, 32 * kTokRows, 0, c.stream>>>(ba);
        CK_LAUNCH("k_tokens");
      } else if (lt_tma && tok_tma) {
        // one stream: launch L = tokens of layer L with the count pass of
        // layer L - 2 in the same grid (see k_slab_tma), then the last two
        // count passes together
        for (uint32_t L = 0; L < d.tz; ++L) {
          BrickArgs ts = ba;
          ts.brick0 = L * bpl;
          if (L >= 2) {
            BrickArgs cs = ba;
            cs.brick0 = (L - 2) * bpl;
            k_slab_tma<><<<2 * items, B_THREADS, 0, c.stream>>>(mlt, mtok, ts, cs);
            CK_LAUNCH("k_slab_tma");
          } else {
            k_tokens_tma<true><<<items, 32 * kTokRows, 0, c.stream>>>(mlt, ts);
            CK_LAUNCH("k_tokens");
          }
        }
        BrickArgs cs = ba;
        const uint32_t c0 = d.tz >= 2 ? d.tz - 2 : 0;
        cs.brick0 = c0 * bpl;
        k_brick_tma<<<(d.tz - c0) * items, B_THREADS, 0, c.stream>>>(mtok, cs);
        CK_LAUNCH("k_brick");
        CK(cudaEventRecord(c.join, c.stream));
      } else
      for (uint32_t sl = 0; sl <= d.tz; ++sl) {
        if (sl < d.tz) {
          BrickArgs bs = ba;
          bs.brick0 = sl * bpl;
          if (lt_tma)
            k_tokens_tma<true><<<bpl * (TY / kTokRows), 32 * kTokRows, 0, c.stream>>>(mlt, bs);
          else
            k_tokens<true><<<bpl * (TY / kTokRows), 32 * kTokRows, 0, c.stream>>>(bs);
          CK_LAUNCH("k_tokens");
          CK(cudaEventRecord(c.slab_event(sl), c.stream));
        }
        if (sl >= 1) {
          BrickArgs bs = ba;
          bs.brick0 = (sl - 1) * bpl;
          CK(cudaStreamWaitEvent(c.side, c.slab_event(std::min(sl, d.tz - 1)), 0));
          if (tok_tma)
            k_brick_tma<<<bpl * (TY / RY), B_THREADS, 0, c.side>>>(mtok, bs);
          else
            k_brick<<<bpl * (TY / RY), B_THREADS, 0, c.side>>>(bs);
          CK_LAUNCH("k_brick");
        }
        if (sl == d.tz) CK(cudaEventRecord(c.join, c.side));
      }
      const int64_t nb = int64_t((nw + kWB - 1) / kWB);
      uint64_t* bsum = c.get_t<uint64_t>(S_HASH_V, nb);
      k_bitmap_count<<<unsigned(nb), 256, 0, c.stream>>>(bitmap, nw, bsum);
      CK_LAUNCH("k_bitmap_count");
      R = int64_t(exclusive_scan_u64(c, bsum, nb, true));
      keys = c.get_t<uint64_t>(S_KEYS, R);
      prefix = c.get_t<uint32_t>(S_HASH_K, nw);
      k_bitmap_ids<<<unsigned(nb), kWB, 0, c.stream>>>(bitmap, nw, bsum, ba.nmax, maxima, minima, prefix, keys);
      CK_LAUNCH("k_bitmap_ids");
      c.stats[2] = -int64_t(nw);
    } else {
      uint64_t fcap = 1024;
      {
        const uint64_t want = c.fused_pair_hint ? c.fused_pair_hint * 2 : uint64_t(1) << 20;
        while (fcap < want) fcap <<= 1;
      }
      unsigned long long* fset = nullptr;
      for (int tries = 0;; ++tries) {
        // tokens are u32 slots
        if (fcap > (uint64_t(1) << 32)) fail(PLMSS_ERR_LOGIC, "region set larger than 2^32 slots");
        fset = c.get_t<unsigned long long>(S_HASH_V, fcap);
        CK(cudaMemsetAsync(fset, 0xff, fcap * 8, c.stream));
        CK(cudaMemsetAsync(flag, 0, 4, c.stream));
        ba.fset = fset;
        ba.fmask = fcap - 1;
        if (lt_tma)
          k_tokens_tma<false><<<tgrid, 32 * kTokRows, 0, c.stream>>>(mlt, ba);
        else
          k_tokens<false><<<tgrid, 32 * kTokRows, 0, c.stream>>>(ba);
        CK_LAUNCH("k_tokens");
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
      R = int64_t(exclusive_scan_u64(c, fcounts, fb, true));
      c.fused_pair_hint = uint64_t(R);
      keys = c.get_t<uint64_t>(S_KEYS, R);
      uint64_t* slots = c.get_t<uint64_t>(S_SORT_B, R);
      k_write_occ<<<unsigned(fb), kCThreads, 0, c.stream>>>(fset, fcap, fcounts, keys, slots);
      CK_LAUNCH("k_write_occ");
      int kb = 32;
      while ((uint64_t(1) << (kb - 32)) < uint64_t(std::max(o.n_min, int64_t(1)))) ++kb;
      radix_sort_pairs(c, keys, slots, R, kb);
      slot_id = c.get_t<uint32_t>(S_BITMAP, fcap);
      k_set_ids<<<blocks_for(R, 256), 256, 0, c.stream>>>(slots, R, slot_id);
      CK_LAUNCH("k_set_ids");
      k_keys_to_gid<<<blocks_for(R, 256), 256, 0, c.stream>>>(keys, R, maxima, minima);
      CK_LAUNCH("k_keys_to_gid");
      c.stats[2] = int64_t(fcap);
    }
    o.n_regions = R;
    if (mark_mode) {
      // token pass in id mode (labels + dense ids into ms) for brick layer
      // L with the count pass of layer L - 2 in the same grid, then the
      // last two count passes
      BrickArgs ia = ba;
      ia.prefix = prefix;
      const uint32_t bpl = d.tx * d.ty;
      const unsigned items = bpl * (TY / kTokRows);
      if (tok_tma) {
        for (uint32_t L = 0; L < d.tz; ++L) {
          BrickArgs ts = ia;
          ts.brick0 = L * bpl;
          if (L >= 2) {
            BrickArgs cs = ba;
            cs.brick0 = (L - 2) * bpl;
            k_slab_tma<2><<<2 * items, B_THREADS, 0, c.stream>>>(mlt, mtok, ts, cs);
            CK_LAUNCH("k_slab_tma");
          } else {
            k_tokens_tma<true, 2><<<items, 32 * kTokRows, 0, c.stream>>>(mlt, ts);
            CK_LAUNCH("k_tokens");
          }
        }
        BrickArgs cs = ba;
        const uint32_t c0 = d.tz >= 2 ? d.tz - 2 : 0;
        cs.brick0 = c0 * bpl;
        k_brick_tma<<<(d.tz - c0) * items, B_THREADS, 0, c.stream>>>(mtok, cs);
        CK_LAUNCH("k_brick");
      } else {
        k_tokens_tma<true, 2><<<tgrid, 32 * kTokRows, 0, c.stream>>>(mlt, ia);
        CK_LAUNCH("k_tokens");
        k_brick<<<cgrid, B_THREADS, 0, c.stream>>>(ba);
        CK_LAUNCH("k_brick");
      }
    } else if (ids_in_count) {
      // cube classes, separator counts and the dense ids of every vertex
      BrickArgs cb = ba;
      cb.ids_out = ms;
      cb.bitmap = bitmap;
      cb.prefix = dense ? prefix : nullptr;
      cb.slot_id = slot_id;
      if (tok_tma)
        k_brick_tma<<<cgrid, B_THREADS, 0, c.stream>>>(mtok, cb);
      else
        k_brick<<<cgrid, B_THREADS, 0, c.stream>>>(cb);
      CK_LAUNCH("k_brick");
    } else if (dense) {
      CK(cudaStreamWaitEvent(c.stream, c.join, 0));  // count passes done
    } else {
      // cube classes and separator counts from the tokens
      if (tok_tma)
        k_brick_tma<<<cgrid, B_THREADS, 0, c.stream>>>(mtok, ba);
      else
        k_brick<<<cgrid, B_THREADS, 0, c.stream>>>(ba);
      CK_LAUNCH("k_brick");
    }
    const uint64_t ngroups = (nchunks + 31) / 32;
    uint64_t* gbase = c.get_t<uint64_t>(S_CHUNK_G, ngroups ? ngroups : 1);
    const uint64_t total = nchunks ? group_offsets(c, chunk, nchunks, gbase) : 0;
    c.mark(4);
    // ---- D: ms tokens -> dense ids; separator records at their chunk offsets
    if (!ids_in_count && !mark_mode) {
      const unsigned mgrid = unsigned((uint64_t(g.n) + 1023) / 1024);
      if (dense)
        k_ms_ids<true><<<mgrid, 256, 0, c.stream>>>(ms, uint64_t(g.n), bitmap, prefix, slot_id);
      else
        k_ms_ids<false><<<mgrid, 256, 0, c.stream>>>(ms, uint64_t(g.n), bitmap, prefix, slot_id);
      CK_LAUNCH("k_ms_ids");
    }
    plmss_tri* tris = c.get_t<plmss_tri>(S_TRIS, total ? total : 1);
    if (total) {
      EmitArgs ea{};
      ea.X = d.X;
      ea.Y = d.Y;
      ea.Z = d.Z;
      ea.nxc = ba.nxc;
      ea.nchunks = nchunks;
      ea.total = total;
      ea.cnt = chunk;
      ea.gbase = gbase;
      ea.cls = ba.cls;
      ea.ids = ms;
      ea.out = tris;
      const unsigned egrid = emit_grid(c, ea);
      if (ea.cshift)
        k_emit_chunks<true><<<egrid, 256, 0, c.stream>>>(ea);
      else
        k_emit_chunks<false><<<egrid, 256, 0, c.stream>>>(ea);
      CK_LAUNCH("k_emit_chunks");
    }
    c.mark(5);
    c.sync();
    if (*reinterpret_cast<int*>(reinterpret_cast<char*>(c.h_pinned) + 64) != 0) {
      // not converged in two sweeps: finish the forest, redo C and D
      if (pass > 0) fail(PLMSS_ERR_LOGIC, "terminal forest did not converge");
      for (;;) {
        sweep();
        CK(cudaMemcpyAsync(reinterpret_cast<char*>(c.h_pinned) + 64, jflag, 4, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (*reinterpret_cast<int*>(reinterpret_cast<char*>(c.h_pinned) + 64) == 0) break;
        if (o.sweeps > 64) fail(PLMSS_ERR_LOGIC, "terminal forest did not converge");
      }
      continue;
    }
    check_device(c, "fused_pipeline");
    o.n_tris = int64_t(total);
    o.tris = tris;
    o.maxima = maxima;
    o.minima = minima;
    o.keys = keys;
    return o;
    }
  }
}


// segment (segmentation.hpp:74-76) on the fused passes: pass A, the extremum
// lists, the forest to its fixpoint, then a token pass that writes only the
// labels (global vertex ids of the maximum / minimum of every vertex). Keys
// are float32 values; OrderField ranks arrive bit-cast to float32 (ranks
// < 2^30: non-negative finite floats whose order is the rank order, no ties).
void fused_segment(Ctx& c, const Grid& g, const float* field, uint32_t* desc, uint32_t* asc, uint32_t* maxima_out,
                   uint32_t* minima_out, int64_t* n_max_out, int64_t* n_min_out, int32_t* sweeps_out) {
  ensure_consts(c);
  FDims d{};
  d.X = uint32_t(g.X);
  d.Y = uint32_t(g.Y);
  d.Z = uint32_t(g.Z);
  d.XY = d.X * d.Y;
  d.n = uint32_t(g.n);
  d.tx = uint32_t((g.X + TX - 1) / TX);
  d.ty = uint32_t((g.Y + TY - 1) / TY);
  d.tz = uint32_t((g.Z + TZ - 1) / TZ);
  d.zf0 = 0;
  d.zfn = d.Z;
  d.pbase = 0;
  const uint64_t ntiles = uint64_t(d.tx) * d.ty * d.tz;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  bool use_tma = (g.X % 4) == 0 && (reinterpret_cast<uintptr_t>(field) & 15) == 0 && c.use_tma;
  if (use_tma) {
    const EncodeFn encode = tensor_map_encoder();
    const cuuint64_t gdim[3] = {cuuint64_t(g.X), cuuint64_t(g.Y), cuuint64_t(g.Z)};
    const cuuint64_t gstride[2] = {cuuint64_t(g.X) * 4, cuuint64_t(g.X) * cuuint64_t(g.Y) * 4};
    const cuuint32_t box[3] = {HX, HY, HZ};
    const cuuint32_t estride[3] = {1, 1, 1};
    use_tma = encode && encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(field), gdim, gstride,
                               box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA) == CUDA_SUCCESS;
  }
  char* ctr_base = static_cast<char*>(c.get(S_FLAGS, 1024));
  ACounters* ctr = reinterpret_cast<ACounters*>(ctr_base);
  uint32_t* lt = c.get_t<uint32_t>(S_LTD, ntiles * (TN + kFaceX));  // desc | asc << 16, then the x faces
  uint4* TB = c.get_t<uint4>(S_TB, ntiles);
  uint32_t *maxima = nullptr, *minima = nullptr, *max_tt = nullptr, *min_tt = nullptr, *TT = nullptr;
  ACounters h;
  for (int attempt = 0;; ++attempt) {
    const uint64_t ext_cap = c.fused_ext_cap ? c.fused_ext_cap : uint64_t(g.n / 4 + 1024);
    maxima = c.get_t<uint32_t>(S_MAXIMA, ext_cap);
    minima = c.get_t<uint32_t>(S_MINIMA, ext_cap);
    max_tt = c.get_t<uint32_t>(S_RANK_MAX, ext_cap);
    min_tt = c.get_t<uint32_t>(S_RANK_MIN, ext_cap);
    const uint64_t tt_cap = c.fused_exit_cap ? c.fused_exit_cap : uint64_t(g.n / 4 + 1024);
    TT = c.get_t<uint32_t>(S_TMP0, tt_cap);
    CK(cudaMemsetAsync(ctr, 0, sizeof(ACounters), c.stream));
    CK(cudaMemsetAsync(&ctr->bad, 0xff, 4, c.stream));
    launch_pass_a(c, d, ntiles, use_tma, tmap, field, maxima, minima, max_tt, min_tt, ext_cap, TT, tt_cap, TB, lt,
                  ctr);
    CK(cudaMemcpyAsync(c.h_pinned, ctr, sizeof(ACounters), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    memcpy(&h, c.h_pinned, sizeof h);
    if (h.bad != 0xffffffffu)
      fail(PLMSS_ERR_INVALID_ARGUMENT, "non-finite scalar value at vertex " + std::to_string(h.bad));
    bool retry = false;
    if (h.n_tt > tt_cap) {
      c.fused_exit_cap = h.n_tt + h.n_tt / 4 + 1024;
      retry = true;
    }
    if (h.n_max > ext_cap || h.n_min > ext_cap) {
      c.fused_ext_cap = std::max(h.n_max, h.n_min) + 1024;
      retry = true;
    }
    if (!retry) break;
    if (attempt > 6) fail(PLMSS_ERR_LOGIC, "fused segment capacity retries exhausted");
  }
  const int64_t n_max = int64_t(h.n_max), n_min = int64_t(h.n_min);
  const uint64_t nt = h.n_tt;
  uint32_t* RK = c.get_t<uint32_t>(S_RK, nt);
  sort_extrema(c, maxima, max_tt, n_max, minima, min_tt, n_min, uint64_t(g.n), RK, 0u);
  uint32_t* SD = c.get_t<uint32_t>(S_SD, nt);
  uint32_t* SA = c.get_t<uint32_t>(S_SA, nt);
  k_tt_succ<<<unsigned(ntiles), 256, 0, c.stream>>>(TB, TT, lt, RK, SD, SA, 0u, nt);
  CK_LAUNCH("k_tt_succ");
  int* jflag = reinterpret_cast<int*>(ctr_base + 192);
  int sweeps = 0;
  for (;;) {
    CK(cudaMemsetAsync(jflag, 0, 4, c.stream));
    k_tt_jump<<<blocks_for(int64_t((nt + 1) / 2), 256), 256, 0, c.stream>>>(nt, SD, SA, jflag);
    CK_LAUNCH("k_tt_jump");
    ++sweeps;
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(c.h_pinned) + 64, jflag, 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (*reinterpret_cast<int*>(reinterpret_cast<char*>(c.h_pinned) + 64) == 0) break;
    if (sweeps > 64) fail(PLMSS_ERR_LOGIC, "terminal forest did not converge");
  }
  BrickArgs ba{};
  ba.d = d;
  ba.nxc = uint32_t((g.X - 1 + 31) / 32);
  ba.TB = TB;
  ba.lt = lt;
  ba.FD = SD;
  ba.FA = SA;
  ba.maxs = maxima;
  ba.mins = minima;
  ba.nmax = uint32_t(n_max);
  ba.nmin = uint32_t(n_min);
  ba.nt = nt;
  ba.desc = desc;
  ba.asc = asc;
  ba.ms = nullptr;  // labels only
  CUtensorMap mlt;
  const bool lt_tma = encode_lt_map(c, ntiles, lt, &mlt);
  const unsigned tgrid = unsigned((TY / kTokRows) * ntiles);
  if (lt_tma)
    k_tokens_tma<true><<<tgrid, 32 * kTokRows, 0, c.stream>>>(mlt, ba);
  else
    k_tokens<true><<<tgrid, 32 * kTokRows, 0, c.stream>>>(ba);
  CK_LAUNCH("k_tokens");
  if (maxima_out && n_max)
    CK(cudaMemcpyAsync(maxima_out, maxima, size_t(n_max) * 4, cudaMemcpyDeviceToDevice, c.stream));
  if (minima_out && n_min)
    CK(cudaMemcpyAsync(minima_out, minima, size_t(n_min) * 4, cudaMemcpyDeviceToDevice, c.stream));
  check_device(c, "fused_segment");
  c.sync();
  if (n_max_out) *n_max_out = n_max;
  if (n_min_out) *n_min_out = n_min;
  if (sweeps_out) *sweeps_out = sweeps;
}

}  // namespace plmss_b200

// ===================================================== z-slab pipeline (e) ==
// The fused passes on one rank's slab (include/plmss_b200.h, stages 1-4).
namespace plmss_b200 {
namespace {

FDims slab_dims(const SlabState& st) {
  FDims d{};
  const int64_t nz = st.z1 - st.z0;
  d.X = uint32_t(st.g.X);
  d.Y = uint32_t(st.g.Y);
  d.Z = uint32_t(nz);
  d.XY = d.X * d.Y;
  d.n = uint32_t(st.g.X * st.g.Y * nz);
  d.tx = uint32_t((st.g.X + TX - 1) / TX);
  d.ty = uint32_t((st.g.Y + TY - 1) / TY);
  d.tz = uint32_t((nz + TZ - 1) / TZ);
  d.zf0 = -st.has_down;
  d.zfn = uint32_t(nz + st.has_down + st.has_up);
  d.pbase = uint32_t(uint64_t(d.tx) * d.ty * d.tz << 15);
  return d;
}


bool encode_tok_map(Ctx& c, uint32_t* ms, uint32_t X, uint32_t Y, uint32_t Z, CUtensorMap* m) {
  if (!c.use_tma || !tensor_map_encoder() || (X % 4) != 0 || (reinterpret_cast<uintptr_t>(ms) & 15) != 0)
    return false;
  const cuuint64_t gdim[3] = {cuuint64_t(X), cuuint64_t(Y), cuuint64_t(Z)};
  const cuuint64_t gstride[2] = {cuuint64_t(X) * 4, cuuint64_t(X) * cuuint64_t(Y) * 4};
  const cuuint32_t box[3] = {cuuint32_t(TLW), cuuint32_t(RY + 1), cuuint32_t(kBatch + 1)};
  const cuuint32_t estride[3] = {1, 1, 1};
  return tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, ms, gdim, gstride, box, estride,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void need_stage(const Ctx& c, int s, const char* what) {
  if (c.slab.stage != s)
    fail(PLMSS_ERR_LOGIC, std::string(what) + " called out of order (z-slab stage " + std::to_string(c.slab.stage) +
                              " completed, " + std::to_string(s) + " required)");
}

}  // namespace

// Stage 1: pass A on the slab's bricks, the extremum lists, the forest.
void slab_segment(Ctx& c, const Grid& g, int64_t z0, int64_t z1, const float* field, plmss_slab_info* info) {
  if (!fused_supported(g)) fail(PLMSS_ERR_INVALID_ARGUMENT, "grid outside the fused pipeline's envelope");
  if (z0 < 0 || z1 > g.Z || z0 >= z1) fail(PLMSS_ERR_INVALID_ARGUMENT, "slab layers outside the grid");
  if (z0 % TZ != 0 || (z1 % TZ != 0 && z1 != g.Z))
    fail(PLMSS_ERR_INVALID_ARGUMENT, "slabs must be whole 32-layer brick layers (z0 % 32 == 0, z1 % 32 == 0 or z1 == Z)");
  ensure_consts(c);
  for (auto& s : c.stats) s = 0;
  SlabState& st = c.slab;
  st = SlabState{};
  st.g = g;
  st.z0 = z0;
  st.z1 = z1;
  st.has_down = z0 > 0;
  st.has_up = z1 < g.Z;
  const FDims d = slab_dims(st);
  const uint64_t ntiles = uint64_t(d.tx) * d.ty * d.tz;
  st.ntiles = ntiles;
  if ((ntiles << 15) + 2 * uint64_t(d.XY) >= (uint64_t(1) << 32) || 2 * uint64_t(d.XY) >= (uint64_t(1) << 30))
    fail(PLMSS_ERR_INVALID_ARGUMENT, "slab too large for u32 portal entries");

  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  bool use_tma = (g.X % 4) == 0 && (reinterpret_cast<uintptr_t>(field) & 15) == 0 && c.use_tma;
  if (use_tma) {
    const EncodeFn encode = tensor_map_encoder();
    const cuuint64_t gdim[3] = {cuuint64_t(g.X), cuuint64_t(g.Y), cuuint64_t(d.zfn)};
    const cuuint64_t gstride[2] = {cuuint64_t(g.X) * 4, cuuint64_t(g.X) * cuuint64_t(g.Y) * 4};
    const cuuint32_t box[3] = {HX, HY, HZ};
    const cuuint32_t estride[3] = {1, 1, 1};
    use_tma = encode && encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(field), gdim, gstride,
                               box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA) == CUDA_SUCCESS;
  }
  c.stats[4] = use_tma ? 1 : 0;
  char* ctr_base = static_cast<char*>(c.get(S_FLAGS, 1024));
  ACounters* ctr = reinterpret_cast<ACounters*>(ctr_base);
  uint32_t* lt = c.get_t<uint32_t>(S_LTD, ntiles * (TN + kFaceX));  // desc | asc << 16, then the x faces
  uint4* TB = c.get_t<uint4>(S_TB, ntiles);
  const uint64_t nloc = uint64_t(d.n);
  uint32_t *maxima = nullptr, *minima = nullptr, *max_tt = nullptr, *min_tt = nullptr, *TT = nullptr;
  ACounters h;
  for (int attempt = 0;; ++attempt) {
    const uint64_t ext_cap = c.fused_ext_cap ? c.fused_ext_cap : uint64_t(nloc / 4 + 1024);
    maxima = c.get_t<uint32_t>(S_MAXIMA, ext_cap);
    minima = c.get_t<uint32_t>(S_MINIMA, ext_cap);
    max_tt = c.get_t<uint32_t>(S_RANK_MAX, ext_cap);
    min_tt = c.get_t<uint32_t>(S_RANK_MIN, ext_cap);
    const uint64_t tt_cap = c.fused_exit_cap ? c.fused_exit_cap : uint64_t(nloc / 4 + 1024);
    TT = c.get_t<uint32_t>(S_TMP0, tt_cap);
    CK(cudaMemsetAsync(ctr, 0, sizeof(ACounters), c.stream));
    CK(cudaMemsetAsync(&ctr->bad, 0xff, 4, c.stream));
    launch_pass_a(c, d, ntiles, use_tma, tmap, field, maxima, minima, max_tt, min_tt, ext_cap, TT, tt_cap, TB, lt,
                  ctr);
    CK(cudaMemcpyAsync(c.h_pinned, ctr, sizeof(ACounters), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    memcpy(&h, c.h_pinned, sizeof h);
    if (h.bad != 0xffffffffu)
      fail(PLMSS_ERR_INVALID_ARGUMENT,
           "non-finite scalar value at vertex " + std::to_string(uint64_t(h.bad) + uint64_t(z0) * d.XY));
    bool retry = false;
    if (h.n_tt > tt_cap) {
      c.fused_exit_cap = h.n_tt + h.n_tt / 4 + 1024;
      retry = true;
    }
    if (h.n_max > ext_cap || h.n_min > ext_cap) {
      c.fused_ext_cap = std::max(h.n_max, h.n_min) + 1024;
      retry = true;
    }
    if (!retry) break;
    if (attempt > 6) fail(PLMSS_ERR_LOGIC, "z-slab pass A capacity retries exhausted");
  }
  if (h.n_max >= (1ull << 30) || h.n_min >= (1ull << 30))
    fail(PLMSS_ERR_INVALID_ARGUMENT, "z-slab: more than 2^30 extrema in one slab");
  c.stats[0] = int64_t(h.n_exit);
  st.n_max_l = int64_t(h.n_max);
  st.n_min_l = int64_t(h.n_min);
  const uint64_t nt = h.n_tt;
  st.nt = nt;
  // extremum lists sorted by id (global ids: + z0 * XY), rank of every extremum entry
  uint32_t* RK = c.get_t<uint32_t>(S_RK, nt);
  sort_extrema(c, maxima, max_tt, st.n_max_l, minima, min_tt, st.n_min_l, nloc, RK, uint32_t(uint64_t(z0) * d.XY));
  // the forest inside the slab, to its fixpoint (portals are roots)
  uint32_t* SD = c.get_t<uint32_t>(S_SD, nt);
  uint32_t* SA = c.get_t<uint32_t>(S_SA, nt);
  k_tt_succ<<<unsigned(ntiles), 256, 0, c.stream>>>(TB, TT, lt, RK, SD, SA, d.pbase, nt);
  CK_LAUNCH("k_tt_succ");
  int* jflag = reinterpret_cast<int*>(ctr_base + 192);
  for (;;) {
    CK(cudaMemsetAsync(jflag, 0, 4, c.stream));
    k_tt_jump<<<blocks_for(int64_t((nt + 1) / 2), 256), 256, 0, c.stream>>>(nt, SD, SA, jflag);
    CK_LAUNCH("k_tt_jump");
    ++st.sweeps;
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(c.h_pinned) + 64, jflag, 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (*reinterpret_cast<int*>(reinterpret_cast<char*>(c.h_pinned) + 64) == 0) break;
    if (st.sweeps > 64) fail(PLMSS_ERR_LOGIC, "z-slab terminal forest did not converge");
  }
  uint32_t* bnd = c.get_t<uint32_t>(S_SLAB_BND, 4 * uint64_t(d.XY));
  k_slab_boundary<<<blocks_for(2 * int64_t(d.XY), 256), 256, 0, c.stream>>>(d, TB, lt, SD, SA, bnd);
  CK_LAUNCH("k_slab_boundary");
  // no device sync: the boundary layers and lists are ordered on the context
  // stream, where the caller's collectives read them
  check_device(c, "slab_segment");
  st.stage = 1;
  if (info) {
    *info = plmss_slab_info{};
    info->n_maxima = st.n_max_l;
    info->n_minima = st.n_min_l;
    info->d_maxima = maxima;
    info->d_minima = minima;
    info->d_boundary = bnd;
    info->sweeps = st.sweeps;
  }
}

// Stage 2: portals -> global ranks; desc / asc; region tokens; the slab's pairs.
void slab_resolve(Ctx& c, const uint32_t* G, int world, int rank, const int64_t* max_counts,
                  const int64_t* min_counts, const uint32_t* maxs_g, const uint32_t* mins_g, uint32_t* desc,
                  uint32_t* asc, uint32_t* ms, plmss_slab_info* info) {
  need_stage(c, 1, "slab_resolve");
  SlabState& st = c.slab;
  if (world < 1 || rank < 0 || rank >= world || !G || !max_counts || !min_counts || !desc || !asc || !ms)
    fail(PLMSS_ERR_INVALID_ARGUMENT, "slab_resolve: bad arguments");
  const FDims d = slab_dims(st);
  // rank prefixes of the extremum counts (rank order == vertex id order)
  std::vector<uint32_t> pre(2 * size_t(world) + 2, 0);
  int64_t smax = 0, smin = 0;
  for (int r = 0; r < world; ++r) {
    pre[r] = uint32_t(smax);
    pre[world + 1 + r] = uint32_t(smin);
    smax += max_counts[r];
    smin += min_counts[r];
  }
  if (max_counts[rank] != st.n_max_l || min_counts[rank] != st.n_min_l)
    fail(PLMSS_ERR_INVALID_ARGUMENT, "slab_resolve: this rank's counts differ from slab_segment's");
  if (smax >= (int64_t(1) << 30) || smin >= (int64_t(1) << 30))
    fail(PLMSS_ERR_INVALID_ARGUMENT, "z-slab: more than 2^30 extrema");
  st.n_max_g = smax;
  st.n_min_g = smin;
  st.maxs_g = maxs_g;
  st.mins_g = mins_g;
  st.desc = desc;
  st.asc = asc;
  st.ms = ms;
  uint32_t* d_pre = c.get_t<uint32_t>(S_SCAN_C, pre.size());
  CK(cudaMemcpyAsync(d_pre, pre.data(), pre.size() * 4, cudaMemcpyHostToDevice, c.stream));
  char* ctr_base = static_cast<char*>(c.get(S_FLAGS, 1024));
  int* err = reinterpret_cast<int*>(ctr_base + 256);
  int* flag = reinterpret_cast<int*>(ctr_base + 128);
  CK(cudaMemsetAsync(err, 0, 4, c.stream));
  uint32_t* SD = static_cast<uint32_t*>(c.buf[S_SD]);
  uint32_t* SA = static_cast<uint32_t*>(c.buf[S_SA]);
  k_slab_patch<<<blocks_for(int64_t(st.nt), 256), 256, 0, c.stream>>>(st.nt, SD, SA, G, world, rank, d.XY, d_pre,
                                                                     d_pre + world + 1, err);
  CK_LAUNCH("k_slab_patch");
  CK(cudaMemcpyAsync(reinterpret_cast<char*>(c.h_pinned) + 96, err, 4, cudaMemcpyDeviceToHost, c.stream));
  // tokens
  BrickArgs ba{};
  ba.d = d;
  ba.nxc = uint32_t((st.g.X - 1 + 31) / 32);
  ba.TB = static_cast<const uint4*>(c.buf[S_TB]);
  ba.lt = static_cast<const uint32_t*>(c.buf[S_LTD]);
  ba.FD = SD;
  ba.FA = SA;
  ba.maxs = maxs_g;
  ba.mins = mins_g;
  ba.nmax = uint32_t(smax);
  ba.nmin = uint32_t(smin);
  ba.nt = st.nt;
  ba.desc = desc;
  ba.asc = asc;
  ba.ms = ms;
  ba.overflow = flag;
  CUtensorMap mlt;
  const bool lt_tma = encode_lt_map(c, st.ntiles, static_cast<uint32_t*>(c.buf[S_LTD]), &mlt);
  const unsigned tgrid = unsigned((TY / kTokRows) * st.ntiles);
  const uint64_t nbits = uint64_t(smax) * uint64_t(smin);
  st.dense = nbits < (uint64_t(1) << 32) && c.combine_path != 2;
  if (st.dense) {
    const uint64_t nw = (nbits + 31) / 32;
    uint32_t* bitmap = c.get_t<uint32_t>(S_BITMAP, nw);
    CK(cudaMemsetAsync(bitmap, 0, nw * 4, c.stream));
    ba.bitmap = bitmap;
    ba.nw = nw;
    if (lt_tma)
      k_tokens_tma<true><<<tgrid, 32 * kTokRows, 0, c.stream>>>(mlt, ba);
    else
      k_tokens<true><<<tgrid, 32 * kTokRows, 0, c.stream>>>(ba);
    CK_LAUNCH("k_tokens");
    // the slab's pairs, as rank keys in key order
    const int64_t nb = int64_t((nw + kWB - 1) / kWB);
    uint64_t* bsum = c.get_t<uint64_t>(S_HASH_V, nb);
    k_bitmap_count<<<unsigned(nb), 256, 0, c.stream>>>(bitmap, nw, bsum);
    CK_LAUNCH("k_bitmap_count");
    st.n_keys = int64_t(exclusive_scan_u64(c, bsum, nb, true));
    st.keys = c.get_t<uint64_t>(S_KEYS, st.n_keys);
    uint32_t* prefix = c.get_t<uint32_t>(S_HASH_K, nw);
    k_bitmap_ids<<<unsigned(nb), kWB, 0, c.stream>>>(bitmap, nw, bsum, ba.nmax, maxs_g, mins_g, prefix, st.keys,
                                                      true);
    CK_LAUNCH("k_bitmap_ids");
  } else {
    uint64_t fcap = 1024;
    {
      const uint64_t want = c.fused_pair_hint ? c.fused_pair_hint * 2 : uint64_t(1) << 20;
      while (fcap < want) fcap <<= 1;
    }
    unsigned long long* fset = nullptr;
    for (int tries = 0;; ++tries) {
      if (fcap > (uint64_t(1) << 32)) fail(PLMSS_ERR_LOGIC, "region set larger than 2^32 slots");
      fset = c.get_t<unsigned long long>(S_HASH_V, fcap);
      CK(cudaMemsetAsync(fset, 0xff, fcap * 8, c.stream));
      CK(cudaMemsetAsync(flag, 0, 4, c.stream));
      ba.fset = fset;
      ba.fmask = fcap - 1;
      if (lt_tma)
        k_tokens_tma<false><<<tgrid, 32 * kTokRows, 0, c.stream>>>(mlt, ba);
      else
        k_tokens<false><<<tgrid, 32 * kTokRows, 0, c.stream>>>(ba);
      CK_LAUNCH("k_tokens");
      CK(cudaMemcpyAsync(c.h_pinned, flag, 4, cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      if (*reinterpret_cast<int*>(c.h_pinned) == 0) break;
      if (fcap >= 4 * uint64_t(d.n) || tries > 8) fail(PLMSS_ERR_LOGIC, "region set overflow");
      fcap <<= 2;
    }
    st.fcap = fcap;
    const int64_t fb = int64_t((fcap + kCTile - 1) / kCTile);
    uint64_t* fcounts = c.get_t<uint64_t>(S_TMP2, fb);
    k_count_occ<<<unsigned(fb), kCThreads, 0, c.stream>>>(fset, fcap, fcounts);
    CK_LAUNCH("k_count_occ");
    st.n_keys = int64_t(exclusive_scan_u64(c, fcounts, fb, true));
    c.fused_pair_hint = uint64_t(st.n_keys);
    st.keys = c.get_t<uint64_t>(S_KEYS, st.n_keys);
    k_write_occ<<<unsigned(fb), kCThreads, 0, c.stream>>>(fset, fcap, fcounts, st.keys, nullptr);
    CK_LAUNCH("k_write_occ");
  }
  // the patch kernel's error flag was copied out before the key compaction,
  // whose scan synchronised the stream
  const int e = *reinterpret_cast<volatile int*>(reinterpret_cast<char*>(c.h_pinned) + 96);
  if (e) fail(PLMSS_ERR_LOGIC, e == 2 ? "z-slab forest entry unresolved" : "z-slab portal chain broken");
  check_device(c, "slab_resolve");
  st.stage = 2;
  if (info) {
    info->n_maxima = smax;
    info->n_minima = smin;
    info->n_keys = st.n_keys;
    info->d_keys = st.keys;
    info->dense = st.dense ? 1 : 0;
  }
}

// Stage 3: the gathered pairs -> global dense ids (combine_ms order) in ms.
void slab_ids(Ctx& c, const uint64_t* keys_all, int64_t n_keys_all, plmss_slab_info* info) {
  need_stage(c, 2, "slab_ids");
  SlabState& st = c.slab;
  if (n_keys_all < 0 || (n_keys_all > 0 && !keys_all)) fail(PLMSS_ERR_INVALID_ARGUMENT, "slab_ids: bad keys");
  const FDims d = slab_dims(st);
  const uint64_t nown = uint64_t(d.n);
  const unsigned mgrid = unsigned((nown + 1023) / 1024);
  if (st.dense) {
    const uint64_t nbits = uint64_t(st.n_max_g) * uint64_t(st.n_min_g);
    const uint64_t nw = (nbits + 31) / 32;
    uint32_t* bitmap = static_cast<uint32_t*>(c.buf[S_BITMAP]);  // holds this slab's pairs already
    if (n_keys_all)
      k_set_bits<<<blocks_for(n_keys_all, 256), 256, 0, c.stream>>>(keys_all, n_keys_all, bitmap,
                                                                     uint32_t(st.n_max_g));
    CK_LAUNCH("k_set_bits");
    const int64_t nb = int64_t((nw + kWB - 1) / kWB);
    uint64_t* bsum = c.get_t<uint64_t>(S_HASH_V, nb);
    k_bitmap_count<<<unsigned(nb), 256, 0, c.stream>>>(bitmap, nw, bsum);
    CK_LAUNCH("k_bitmap_count");
    st.R = int64_t(exclusive_scan_u64(c, bsum, nb, true));
    st.keys = c.get_t<uint64_t>(S_KEYS, st.R);
    uint32_t* prefix = c.get_t<uint32_t>(S_HASH_K, nw);
    k_bitmap_ids<<<unsigned(nb), kWB, 0, c.stream>>>(bitmap, nw, bsum, uint32_t(st.n_max_g), st.maxs_g, st.mins_g,
                                                      prefix, st.keys, false);
    CK_LAUNCH("k_bitmap_ids");
    // ms keeps the (globally consistent) dense-key tokens: the count pass of
    // slab_emit writes the ids, the halo layer exchanged is tokens too
    st.bitmap = bitmap;
    st.prefix = prefix;
    (void)mgrid;
  } else {
    // sort + unique of the gathered rank pairs
    const int64_t n = std::max<int64_t>(n_keys_all, 1);
    uint64_t* kk = c.get_t<uint64_t>(S_SORT_A, n);
    uint64_t* vv = c.get_t<uint64_t>(S_SORT_B, n);  // (radix_sort_pairs uses S_SORT_C / S_SORT_D)
    if (n_keys_all) CK(cudaMemcpyAsync(kk, keys_all, n_keys_all * 8, cudaMemcpyDeviceToDevice, c.stream));
    int kb = 32;
    while ((uint64_t(1) << (kb - 32)) < uint64_t(std::max<int64_t>(st.n_min_g, 1))) ++kb;
    if (n_keys_all > 1) radix_sort_pairs(c, kk, vv, n_keys_all, kb);
    uint64_t* pos = c.get_t<uint64_t>(S_SORT_D, n);
    k_first_flags<<<blocks_for(n, 256), 256, 0, c.stream>>>(kk, n_keys_all, pos);
    CK_LAUNCH("k_first_flags");
    st.R = n_keys_all ? int64_t(exclusive_scan_u64(c, pos, n_keys_all, true)) : 0;
    st.keys = c.get_t<uint64_t>(S_KEYS, std::max<int64_t>(st.R, 1));
    k_compact_first<<<blocks_for(n, 256), 256, 0, c.stream>>>(kk, n_keys_all, pos, st.keys);
    CK_LAUNCH("k_compact_first");
    uint32_t* slot_id = c.get_t<uint32_t>(S_BITMAP, st.fcap);
    k_slot_ids<<<blocks_for(int64_t(st.fcap), 256), 256, 0, c.stream>>>(
        static_cast<const unsigned long long*>(c.buf[S_HASH_V]), st.fcap, st.keys, st.R, slot_id);
    CK_LAUNCH("k_slot_ids");
    k_ms_ids<false><<<mgrid, 256, 0, c.stream>>>(st.ms, nown, nullptr, nullptr, slot_id);
    CK_LAUNCH("k_ms_ids");
    if (st.R) k_keys_to_gid<<<blocks_for(st.R, 256), 256, 0, c.stream>>>(st.keys, st.R, st.maxs_g, st.mins_g);
    CK_LAUNCH("k_keys_to_gid");
  }
  check_device(c, "slab_ids");  // (stream-ordered: no device sync)
  st.stage = 3;
  if (info) {
    info->n_regions = st.R;
    info->d_region_keys = st.keys;
  }
}

// Stage 4: separator records of the owned cube layers (+ the layer shared
// with the next rank), global cell ids.
void slab_emit(Ctx& c, uint32_t* ids, plmss_slab_info* info) {
  need_stage(c, 3, "slab_emit");
  if (!ids) fail(PLMSS_ERR_INVALID_ARGUMENT, "slab_emit: ids output is null");
  SlabState& st = c.slab;
  FDims d = slab_dims(st);
  const uint32_t Zc = d.Z + uint32_t(st.has_up);  // vertex layers in ms
  d.Z = Zc;
  const uint64_t ncl = Zc - 1;                    // cube layers
  const uint32_t nxc = uint32_t((st.g.X - 1 + 31) / 32);
  const uint64_t nchunks = uint64_t(nxc) * uint64_t(st.g.Y - 1) * ncl;
  uint64_t total = 0;
  plmss_tri* tris = nullptr;
  if (nchunks) {
    BrickArgs ba{};
    ba.d = d;
    ba.nxc = nxc;
    uint16_t* chunk = c.get_t<uint16_t>(S_TMP1, nchunks);
    ba.chunk = chunk;
    uint64_t* gbase = c.get_t<uint64_t>(S_CHUNK_G, (nchunks + 31) / 32);
    ba.cls = c.get_t<uint8_t>(S_MASK, uint64_t(st.g.X - 1) * uint64_t(st.g.Y - 1) * ncl);
    ba.ms = st.ms;
    // dense: ms holds the tokens -> ids; hash: ms holds the ids -> copied
    ba.ids_out = ids;
    ba.bitmap = st.dense ? st.bitmap : nullptr;
    ba.prefix = st.dense ? st.prefix : nullptr;
    ba.slot_id = nullptr;
    const unsigned cgrid = unsigned((TY / RY) * st.ntiles);
    CUtensorMap mtok;
    if (encode_tok_map(c, st.ms, d.X, d.Y, Zc, &mtok))
      k_brick_tma<<<cgrid, B_THREADS, 0, c.stream>>>(mtok, ba);
    else
      k_brick<<<cgrid, B_THREADS, 0, c.stream>>>(ba);
    CK_LAUNCH("k_brick");
    total = group_offsets(c, chunk, nchunks, gbase);
    tris = c.get_t<plmss_tri>(S_TRIS, total ? total : 1);
    if (total) {
      EmitArgs ea{};
      ea.X = d.X;
      ea.Y = d.Y;
      ea.Z = Zc;
      ea.nxc = nxc;
      ea.nchunks = nchunks;
      ea.total = total;
      ea.cube0 = uint64_t(st.z0) * uint64_t(st.g.X - 1) * uint64_t(st.g.Y - 1);
      ea.cnt = chunk;
      ea.gbase = gbase;
      ea.cls = ba.cls;
      ea.ids = ids;
      ea.out = tris;
      const unsigned egrid = emit_grid(c, ea);
      if (ea.cshift)
        k_emit_chunks<true><<<egrid, 256, 0, c.stream>>>(ea);
      else
        k_emit_chunks<false><<<egrid, 256, 0, c.stream>>>(ea);
      CK_LAUNCH("k_emit_chunks");
    }
  } else {
    // no cube layer (a one-layer slab at the top of the volume): the ids of
    // the owned layer straight from ms
    tris = c.get_t<plmss_tri>(S_TRIS, 1);
    const uint64_t nv = uint64_t(Zc) * d.XY;
    CK(cudaMemcpyAsync(ids, st.ms, nv * 4, cudaMemcpyDeviceToDevice, c.stream));
    if (st.dense) {
      k_ms_ids<true><<<unsigned((nv + 1023) / 1024), 256, 0, c.stream>>>(ids, nv, st.bitmap, st.prefix, nullptr);
      CK_LAUNCH("k_ms_ids");
    }
  }
  c.sync();
  st.n_tris = int64_t(total);
  st.tris = tris;
  check_device(c, "slab_emit");
  st.stage = 4;
  if (info) {
    info->n_tris = st.n_tris;
    info->d_tris = tris;
  }
}

}  // namespace plmss_b200
