/* CPU restatement for FULL-SIZE grids — TEST INFRASTRUCTURE ONLY.
 *
 * The same reference algorithms as plmss_oracle.c, restated for the BASELINE
 * configs at full size (up to 1024^3 = 2^30 vertices on a 62 GB host):
 * uint32 vertex ids instead of int64, float32 values compared as (f, id)
 * (exact: float widens to double exactly), OpenMP workers the
 * way the reference uses std::thread workers (results are identical for any
 * worker count, proj/include/plmss/segmentation.hpp:70-73). Pinned against
 * plmss_oracle.c and the compiled reference in tests/test_oracle_pin.py.
 *
 * Also the host half of the input definition include/plmss_synth.h
 * (orc_synth), which must give the device generator's bytes.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "plmss_oracle.h"
#include "plmss_synth.h"

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------- the input -- */

/* include/plmss_synth.h, host loop: rows (y, z) in parallel, Gaussians in
 * order, every product and sum rounded separately (-ffp-contract=off). */
int orc_synth(const int64_t dims[3], int kind, const double* gauss, int ng, double noise, uint64_t seed,
              int levels, int64_t z0, int64_t nz, float* out) {
  const int64_t X = dims[0], Y = dims[1], Z = dims[2];
  if (z0 < 0 || nz < 1 || z0 + nz > Z) return 1;
  if (levels > 0 && (z0 != 0 || nz != Z)) return 1;
  const int64_t rows = Y * nz;
  if (kind == 1) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t x = 0; x < X; ++x) {
        const uint64_t v = (uint64_t)(x + X * (r + Y * z0));
        out[r * X + x] = (float)plmss_synth_uniform01(seed, v);
      }
  } else {
    float* tab = (float*)malloc(sizeof(float) * (size_t)ng * (size_t)(X + Y + Z + 1) + 16);
    float *ex = tab, *ey = ex + (size_t)ng * X, *ez = ey + (size_t)ng * Y, *am = ez + (size_t)ng * Z;
    for (int k = 0; k < ng; ++k) {
      const double* p = gauss + 5 * k;
      plmss_synth_axis_table(p[0], p[3], X, ex + (size_t)k * X);
      plmss_synth_axis_table(p[1], p[3], Y, ey + (size_t)k * Y);
      plmss_synth_axis_table(p[2], p[3], Z, ez + (size_t)k * Z);
      am[k] = (float)p[4];
    }
#pragma omp parallel
    {
      float* s = (float*)malloc(sizeof(float) * (size_t)X);
#pragma omp for schedule(static)
      for (int64_t r = 0; r < rows; ++r) {
        const int64_t y = r % Y, z = z0 + r / Y;
        for (int64_t x = 0; x < X; ++x) s[x] = 0.0f;
        for (int k = 0; k < ng; ++k) {
          const float w = am[k] * (ey[(size_t)k * Y + y] * ez[(size_t)k * Z + z]);
          const float* exk = ex + (size_t)k * X;
          for (int64_t x = 0; x < X; ++x) s[x] = s[x] + exk[x] * w;
        }
        for (int64_t x = 0; x < X; ++x) {
          const uint64_t v = (uint64_t)(x + X * (y + Y * z));
          const double u = plmss_synth_uniform01(seed, v);
          out[r * X + x] = (float)((double)s[x] + noise * (2.0 * u - 1.0));
        }
      }
      free(s);
    }
    free(tab);
  }
  if (levels > 0) {
    const int64_t n = X * Y * Z;
    float lo = out[0], hi = out[0];
    for (int64_t i = 1; i < n; ++i) {
      lo = out[i] < lo ? out[i] : lo;
      hi = out[i] > hi ? out[i] : hi;
    }
    const double dlo = lo, dhi = hi;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      const double t = dhi > dlo ? ((double)out[i] - dlo) / (dhi - dlo) : 0.0;
      const double fl = t * (double)levels;
      int q = (int)fl; /* floor: t >= 0 */
      if ((double)q > fl) --q;
      q = q < 0 ? 0 : (q >= levels ? levels - 1 : q);
      out[i] = (float)q;
    }
  }
  return 0;
}

/* ---------------------------------------------------------- segmentation -- */

/* Stencil in ascending id-delta order (proj/src/complex.cpp:45-89): the 14
 * offsets of {-1,0,1}^3 \ 0 whose nonzero components share a sign. */
static const int kSt[14][3] = {{-1, -1, -1}, {0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {-1, -1, 0},
                               {0, -1, 0},   {-1, 0, 0},  {1, 0, 0},   {0, 1, 0},  {1, 1, 0},
                               {0, 0, 1},    {1, 0, 1},   {0, 1, 1},   {1, 1, 1}};

/* seed_hops_both (proj/src/segmentation.cpp:60-85) over float values in the
 * (f, id) order. Returns the lowest non-finite vertex or -1
 * (proj/src/orderfield.cpp:14-18). */
int64_t orc_seed_hops_f32(const int64_t dims[3], const float* f, uint32_t* desc, uint32_t* asc) {
  const int64_t X = dims[0], Y = dims[1], Z = dims[2], n = X * Y * Z;
  int64_t bad = -1;
  for (int64_t v = 0; v < n && bad < 0; ++v)
    if (!(f[v] - f[v] == 0.0f)) bad = v;
  if (bad >= 0) return bad;
  int64_t delta[14];
  for (int s = 0; s < 14; ++s) delta[s] = kSt[s][0] + X * (kSt[s][1] + Y * (int64_t)kSt[s][2]);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < Y * Z; ++r) {
    const int64_t y = r % Y, z = r / Y;
    for (int64_t x = 0; x < X; ++x) {
      const int64_t v = x + X * r;
      int64_t up = v, dn = v;
      float fu = f[v], fd = f[v];
      for (int s = 0; s < 14; ++s) {
        const int64_t nx = x + kSt[s][0], ny = y + kSt[s][1], nz = z + kSt[s][2];
        if (nx < 0 || nx >= X || ny < 0 || ny >= Y || nz < 0 || nz >= Z) continue;
        const int64_t u = v + delta[s];
        const float fw = f[u];
        if (fw > fu || (fw == fu && u > up)) {
          up = u;
          fu = fw;
        } else if (fw < fd || (fw == fd && u < dn)) {
          dn = u;
          fd = fw;
        }
      }
      desc[v] = (uint32_t)up;
      asc[v] = (uint32_t)dn;
    }
  }
  return -1;
}

static inline uint32_t ld_relaxed(const uint32_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
static inline void st_relaxed(uint32_t* p, uint32_t v) { __atomic_store_n(p, v, __ATOMIC_RELAXED); }

/* Step 2 (proj/src/segmentation.cpp:87-105, driver :144-156) with workers:
 * each sweep splits the active list into contiguous per-worker ranges, does
 * label <- label[label] in both directions with relaxed atomics (:14-20) and
 * keeps a vertex while either direction has not settled. Returns sweeps. */
int orc_compress_u32(int64_t n, uint32_t* desc, uint32_t* asc) {
  uint32_t* act = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  int64_t na = 0;
  for (int64_t v = 0; v < n; ++v)
    if (desc[v] != (uint32_t)v || asc[v] != (uint32_t)v) act[na++] = (uint32_t)v;
  int sweeps = 0;
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  int64_t* kept = (int64_t*)calloc((size_t)nt, sizeof(int64_t));
  while (na > 0) {
#pragma omp parallel num_threads(nt)
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      const int64_t b = na * t / nt, e = na * (t + 1) / nt;
      int64_t k = b;
      for (int64_t i = b; i < e; ++i) {
        const uint32_t v = act[i];
        const uint32_t d2 = ld_relaxed(desc + ld_relaxed(desc + v));
        st_relaxed(desc + v, d2);
        int settled = ld_relaxed(desc + d2) == d2;
        const uint32_t a2 = ld_relaxed(asc + ld_relaxed(asc + v));
        st_relaxed(asc + v, a2);
        settled = settled && ld_relaxed(asc + a2) == a2;
        if (!settled) act[k++] = v;
      }
      kept[t] = k - b;
    }
    int64_t m = 0;
    for (int t = 0; t < nt; ++t) {
      const int64_t b = na * t / nt;
      if (m != b && kept[t]) memmove(act + m, act + b, sizeof(uint32_t) * (size_t)kept[t]);
      m += kept[t];
    }
    na = m;
    ++sweeps;
  }
  free(kept);
  free(act);
  return sweeps;
}

/* maxima / minima ascending (proj/src/segmentation.cpp:158-166). */
int64_t orc_extrema_u32(int64_t n, const uint32_t* labels, uint32_t* out) {
  int64_t k = 0;
  for (int64_t v = 0; v < n; ++v)
    if (labels[v] == (uint32_t)v) {
      if (out) out[k] = (uint32_t)v;
      ++k;
    }
  return k;
}

/* ------------------------------------------------------------ combine_ms -- */

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static inline uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

typedef struct {
  uint64_t* k;
  uint32_t* id;
  uint64_t mask, used;
} kset_t;

static void kset_init(kset_t* s, uint64_t cap) {
  s->k = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  s->id = NULL;
  memset(s->k, 0xff, sizeof(uint64_t) * cap);
  s->mask = cap - 1;
  s->used = 0;
}

static uint64_t kset_find(const kset_t* s, uint64_t key) {
  uint64_t i = mix64(key) & s->mask;
  while (s->k[i] != key && s->k[i] != ~0ull) i = (i + 1) & s->mask;
  return i;
}

static void kset_insert(kset_t* s, uint64_t key) {
  if (2 * (s->used + 1) > s->mask + 1) { /* grow */
    kset_t t;
    kset_init(&t, 2 * (s->mask + 1));
    for (uint64_t i = 0; i <= s->mask; ++i)
      if (s->k[i] != ~0ull) t.k[kset_find(&t, s->k[i])] = s->k[i];
    t.used = s->used;
    free(s->k);
    *s = t;
  }
  const uint64_t i = kset_find(s, key);
  if (s->k[i] == ~0ull) {
    s->k[i] = key;
    ++s->used;
  }
}

/* combine_ms (proj/src/segmentation.cpp:170-196): region_keys = the sorted
 * distinct (asc, desc) pairs (packed asc << 32 | desc: lexicographic order =
 * ms_key order, proj/include/plmss/segmentation.hpp:19-30); ms[v] = index of
 * v's pair (the lower_bound of :190-194, found through a hash of the pairs).
 * keys_out (capacity keys_cap) gets the sorted keys. Returns R. */
int64_t orc_combine_ms_u32(int64_t n, const uint32_t* asc, const uint32_t* desc, uint32_t* ms, uint64_t* keys_out,
                           int64_t keys_cap) {
  kset_t s;
  kset_init(&s, 1u << 16);
  uint64_t last = ~0ull;
  for (int64_t v = 0; v < n; ++v) {
    const uint64_t key = ((uint64_t)asc[v] << 32) | desc[v];
    if (key != last) kset_insert(&s, key);
    last = key;
  }
  const int64_t R = (int64_t)s.used;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(R > 0 ? R : 1));
  int64_t r = 0;
  for (uint64_t i = 0; i <= s.mask; ++i)
    if (s.k[i] != ~0ull) keys[r++] = s.k[i];
  qsort(keys, (size_t)R, sizeof(uint64_t), cmp_u64);
  s.id = (uint32_t*)malloc(sizeof(uint32_t) * (s.mask + 1));
  for (int64_t i = 0; i < R; ++i) s.id[kset_find(&s, keys[i])] = (uint32_t)i;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    const uint64_t key = ((uint64_t)asc[v] << 32) | desc[v];
    ms[v] = s.id[kset_find(&s, key)];
  }
  if (keys_out) memcpy(keys_out, keys, sizeof(uint64_t) * (size_t)(R < keys_cap ? R : keys_cap));
  free(keys);
  free(s.id);
  free(s.k);
  return R;
}

/* ------------------------------------------------------------ separators -- */

/* Cube tets (proj/src/complex.cpp:23-24, cell() :203-218): corners of cube
 * corner index dx | dy << 1 | dz << 2, axis orders xyz xzy yxz yzx zxy zyx. */
static const int kTetCorner[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7},
                                     {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

/* Records of cube layers [cz0, cz1) in the reference emission order
 * (cell-major, recipe rows in order: proj/src/marching.cpp:116-206); row =
 * index of the recipe in the reference's kTetraData (marching_tables.cpp:48-116),
 * lo / hi = (min, max) of the labels at pairA / pairB (:84-90). labels are
 * indexed by global vertex id. out == NULL: count only. Returns the count. */
int64_t orc_separator_records(const int64_t dims[3], const uint32_t* labels, int64_t cz0, int64_t cz1,
                              orc_tri* out) {
  const int64_t X = dims[0], Y = dims[1], CX = X - 1, CY = Y - 1;
  int row0[32], rowc[32];
  uint8_t rows[32][12][5];
  {
    int off = 0;
    for (int code = 0; code < 32; ++code) rowc[code] = 0;
    /* kTetraData order = the order of codes in the restated table */
    static const int order[14] = {3, 8, 16, 21, 10, 17, 20, 11, 19, 23, 24, 25, 26, 27};
    for (int i = 0; i < 14; ++i) {
      const int code = order[i];
      rowc[code] = orc_tetra_case(code, &rows[code][0][0]);
      row0[code] = off;
      off += rowc[code];
    }
  }
  const int64_t nrows = CY * (cz1 - cz0);
  int64_t* cnt = (int64_t*)calloc((size_t)(nrows + 1), sizeof(int64_t));
  for (int pass = 0; pass < (out ? 2 : 1); ++pass) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < nrows; ++r) {
      const int64_t cy = r % CY, cz = cz0 + r / CY;
      int64_t w = pass ? cnt[r] : 0;
      for (int64_t cx = 0; cx < CX; ++cx) {
        const int64_t v0 = cx + X * (cy + Y * cz);
        const int64_t cube = cx + CX * (cy + CY * cz);
        uint32_t cl[8];
        for (int c = 0; c < 8; ++c) cl[c] = labels[v0 + (c & 1) + X * ((c >> 1) & 1) + X * Y * (c >> 2)];
        for (int t = 0; t < 6; ++t) {
          int64_t l[4];
          for (int i = 0; i < 4; ++i) l[i] = cl[kTetCorner[t][i]];
          const int code = orc_tetra_code(l, NULL);
          const int nr = code < 32 ? rowc[code] : 0;
          if (!pass) {
            w += nr;
            continue;
          }
          for (int k = 0; k < nr; ++k, ++w) {
            const uint8_t* row = rows[code][k];
            const uint32_t a = (uint32_t)l[row[3]], b = (uint32_t)l[row[4]];
            out[w].cellrow = ((uint64_t)(6 * cube + t) << 6) | (uint64_t)(row0[code] + k);
            out[w].lo = a < b ? a : b;
            out[w].hi = a < b ? b : a;
          }
        }
      }
      if (!pass) cnt[r + 1] = w;
    }
    if (!pass)
      for (int64_t r = 0; r < nrows; ++r) cnt[r + 1] += cnt[r];
  }
  const int64_t total = cnt[nrows];
  free(cnt);
  return total;
}
