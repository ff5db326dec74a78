/* CPU restatement of the PLMSS hot path — TEST INFRASTRUCTURE ONLY.
 * See plmss_oracle.h for the contract. Citations are relative to
 * /root/reference/ (proj/...). Compiled with -ffp-contract=off so the point
 * arithmetic is the reference's separately rounded mul/add/div.
 */
#include "plmss_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ grid -- */

typedef struct {
  int64_t d[3];
  int dim;         /* 3, or 2 when exactly one axis has extent 1 */
  int ax0, ax1;    /* active axes in 2-D */
  int nst;         /* stencil size: 14 (3-D) or 6 (2-D) */
  int st[14][3];   /* offsets, sorted by id delta */
  int64_t delta[14];
} grid_t;

/* Stencil rule: offsets in {-1,0,1}^3 \ 0 whose nonzero components share a
 * sign (proj/src/complex.cpp:45-89, rule :53-64); 2-D: same rule in the
 * active plane (:66-77); enumeration sorted by id delta (:78-88). */
static void grid_init(grid_t* g, const int64_t dims[3]) {
  int wide = 0, k = 0;
  memcpy(g->d, dims, sizeof g->d);
  for (int a = 0; a < 3; ++a) wide += dims[a] >= 2;
  g->dim = wide == 3 ? 3 : 2;
  g->ax0 = 0;
  g->ax1 = 1;
  if (g->dim == 2) {
    int q = 0;
    for (int a = 0; a < 3; ++a)
      if (dims[a] >= 2) (q == 0 ? (g->ax0 = a) : (g->ax1 = a)), ++q;
  }
  g->nst = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int o[3] = {dx, dy, dz};
        if (!dx && !dy && !dz) continue;
        int pos = dx > 0 || dy > 0 || dz > 0, neg = dx < 0 || dy < 0 || dz < 0;
        if (pos && neg) continue;
        if (g->dim == 2) {
          int off = 0;
          for (int a = 0; a < 3; ++a)
            if (a != g->ax0 && a != g->ax1 && o[a] != 0) off = 1;
          if (off) continue;
        }
        memcpy(g->st[g->nst], o, sizeof o);
        g->delta[g->nst] = dx + dims[0] * (dy + dims[1] * (int64_t)dz);
        ++g->nst;
      }
  /* insertion sort by delta */
  for (int i = 1; i < g->nst; ++i)
    for (int j = i; j > 0 && g->delta[j - 1] > g->delta[j]; --j) {
      int64_t td = g->delta[j];
      int to[3];
      g->delta[j] = g->delta[j - 1];
      g->delta[j - 1] = td;
      memcpy(to, g->st[j], sizeof to);
      memcpy(g->st[j], g->st[j - 1], sizeof to);
      memcpy(g->st[j - 1], to, sizeof to);
    }
  (void)k;
}

/* ----------------------------------------------------------------- order -- */

static const double* g_sort_vals;
static int cmp_by_value(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  double fa = g_sort_vals[a], fb = g_sort_vals[b];
  if (fa != fb) return fa < fb ? -1 : 1; /* -0.0 == +0.0 falls through */
  return a < b ? -1 : (a > b);
}

/* compute_order (proj/src/orderfield.cpp:12-32): finite check naming the
 * lowest bad vertex, sort ids by (value, id), rank[byValue[i]] = i. */
int64_t orc_compute_order(const double* values, int64_t n, int64_t* rank) {
  for (int64_t v = 0; v < n; ++v)
    if (!isfinite(values[v])) return v;
  int64_t* by = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) by[i] = i;
  g_sort_vals = values;
  qsort(by, (size_t)n, sizeof(int64_t), cmp_by_value);
  for (int64_t i = 0; i < n; ++i) rank[by[i]] = i;
  free(by);
  return -1;
}

/* u "higher than" v under simulation of simplicity: (f(u), u) > (f(v), v)
 * lexicographically; on ranks this is rank(u) > rank(v) (F5 in SURVEY.md). */
static int higher(const void* keys, int kind, int64_t u, int64_t v) {
  if (kind == 1) return ((const int64_t*)keys)[u] > ((const int64_t*)keys)[v];
  double fu = ((const double*)keys)[u], fv = ((const double*)keys)[v];
  if (fu != fv) return fu > fv;
  return u > v;
}

/* ---------------------------------------------------------- segmentation -- */

/* seed_hops_both (proj/src/segmentation.cpp:60-85) with for_each_neighbor
 * (proj/include/plmss/complex.hpp:84-101): neighbours in ascending id order,
 * up = strictly highest, down = strictly lowest, self when none. */
void orc_seed_hops(const int64_t dims[3], const void* keys, int key_kind, int64_t* desc,
                   int64_t* asc) {
  grid_t g;
  grid_init(&g, dims);
  const int64_t n = dims[0] * dims[1] * dims[2];
  for (int64_t v = 0; v < n; ++v) {
    int64_t x = v % dims[0], y = (v / dims[0]) % dims[1], z = v / (dims[0] * dims[1]);
    int64_t up = v, down = v;
    for (int s = 0; s < g.nst; ++s) {
      int64_t nx = x + g.st[s][0], ny = y + g.st[s][1], nz = z + g.st[s][2];
      if (nx < 0 || nx >= dims[0] || ny < 0 || ny >= dims[1] || nz < 0 || nz >= dims[2]) continue;
      int64_t u = v + g.delta[s];
      if (higher(keys, key_kind, u, up))
        up = u;
      else if (higher(keys, key_kind, down, u))
        down = u;
    }
    desc[v] = up;
    asc[v] = down;
  }
}

/* Step 2 (proj/src/segmentation.cpp:87-105 and :144-156), single worker:
 * sweep the active list in order, label <- label[label] for both arrays, keep
 * a vertex while either direction has not settled. */
int orc_compress(int64_t n, int64_t* desc, int64_t* asc) {
  int64_t* act = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t na = 0;
  int sweeps = 0;
  for (int64_t v = 0; v < n; ++v)
    if (desc[v] != v || asc[v] != v) act[na++] = v;
  while (na > 0) {
    int64_t keep = 0;
    for (int64_t i = 0; i < na; ++i) {
      int64_t v = act[i];
      int64_t d2 = desc[desc[v]];
      desc[v] = d2;
      int settled = desc[d2] == d2;
      int64_t a2 = asc[asc[v]];
      asc[v] = a2;
      settled = settled && asc[a2] == a2;
      if (!settled) act[keep++] = v;
    }
    na = keep;
    ++sweeps;
  }
  free(act);
  return sweeps;
}

/* maxima/minima lists, ascending (proj/src/segmentation.cpp:158-166). */
int64_t orc_extrema(int64_t n, const int64_t* labels, int64_t* out) {
  int64_t k = 0;
  for (int64_t v = 0; v < n; ++v)
    if (labels[v] == v) {
      if (out) out[k] = v;
      ++k;
    }
  return k;
}

/* ------------------------------------------------------------ combine_ms -- */

typedef struct {
  uint64_t hi, lo;
} key128;

static int cmp_key(const void* pa, const void* pb) {
  const key128 *a = (const key128*)pa, *b = (const key128*)pb;
  if (a->hi != b->hi) return a->hi < b->hi ? -1 : 1;
  if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
  return 0;
}

/* combine_ms (proj/src/segmentation.cpp:170-196) with ms_key
 * (proj/include/plmss/segmentation.hpp:21-24): key = (min << 64) | max,
 * sorted unique keys = region table, region id = lower_bound index. */
int64_t orc_combine_ms(int64_t n, const int64_t* asc, const int64_t* desc, int64_t* ms_region,
                       int64_t* keys_out) {
  key128* k = (key128*)malloc(sizeof(key128) * (size_t)(n > 0 ? n : 1));
  for (int64_t v = 0; v < n; ++v) {
    k[v].hi = (uint64_t)asc[v];
    k[v].lo = (uint64_t)desc[v];
  }
  qsort(k, (size_t)n, sizeof(key128), cmp_key);
  int64_t r = 0;
  for (int64_t i = 0; i < n; ++i)
    if (r == 0 || cmp_key(&k[r - 1], &k[i]) != 0) k[r++] = k[i];
  for (int64_t v = 0; v < n; ++v) {
    key128 q = {(uint64_t)asc[v], (uint64_t)desc[v]};
    int64_t lo = 0, hi = r;
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (cmp_key(&k[mid], &q) < 0)
        lo = mid + 1;
      else
        hi = mid;
    }
    ms_region[v] = lo;
  }
  if (keys_out)
    for (int64_t i = 0; i < r; ++i) {
      keys_out[2 * i] = (int64_t)k[i].hi;
      keys_out[2 * i + 1] = (int64_t)k[i].lo;
    }
  free(k);
  return r;
}

/* ----------------------------------------------------------------- codes -- */

/* tetra_code (proj/src/marching.cpp:28-44): local[i] = local of the first
 * earlier j with an equal label, else i; code = l1<<4 | l2<<2 | l3. */
int orc_tetra_code(const int64_t labels[4], int local_out[4]) {
  int local[4] = {0, 0, 0, 0};
  for (int i = 1; i < 4; ++i) {
    local[i] = i;
    for (int j = 0; j < i; ++j)
      if (labels[i] == labels[j]) {
        local[i] = local[j];
        break;
      }
  }
  if (local_out) memcpy(local_out, local, sizeof local);
  return (local[1] << 4) | (local[2] << 2) | local[3];
}

/* triangle_code (proj/src/marching.cpp:14-26). */
int orc_triangle_code(const int64_t l[3]) {
  int l1 = l[1] == l[0] ? 0 : 1;
  int l2 = l[2] == l[0] ? 0 : (l[2] == l[1] ? l1 : 2);
  return (l1 << 2) | l2;
}

/* Separator recipes restated from proj/src/marching_tables.cpp:48-127 (3-D)
 * and :36-46 (2-D). Corner masks: bit i = cell vertex i; edge midpoint = 2
 * bits, face barycentre = 3, cell barycentre = 4. Listed per code as
 * {mask0, mask1, mask2, pairA, pairB}. */
typedef struct {
  int code, count;
  uint8_t rows[12][5];
} tet_case_t;

static const tet_case_t kTet[] = {
    {3, 1, {{9, 10, 12, 0, 3}}},
    {8, 1, {{5, 6, 12, 0, 2}}},
    {16, 1, {{3, 6, 10, 0, 1}}},
    {21, 1, {{3, 5, 9, 0, 1}}},
    {10, 2, {{5, 9, 6, 0, 2}, {9, 6, 10, 0, 2}}},
    {17, 2, {{3, 9, 6, 0, 1}, {9, 6, 12, 0, 1}}},
    {20, 2, {{3, 5, 10, 0, 1}, {5, 10, 12, 0, 1}}},
    {11, 5, {{13, 14, 5, 0, 2}, {14, 5, 6, 0, 2}, {13, 14, 9, 0, 3}, {14, 9, 10, 0, 3},
             {13, 14, 12, 2, 3}}},
    {19, 5, {{11, 14, 3, 0, 1}, {14, 3, 6, 0, 1}, {11, 14, 9, 0, 3}, {14, 9, 12, 0, 3},
             {11, 14, 10, 1, 3}}},
    {23, 5, {{11, 13, 3, 0, 1}, {13, 3, 5, 0, 1}, {11, 13, 10, 1, 3}, {13, 10, 12, 1, 3},
             {11, 13, 9, 0, 3}}},
    {24, 5, {{7, 14, 3, 0, 1}, {14, 3, 10, 0, 1}, {7, 14, 5, 0, 2}, {14, 5, 12, 0, 2},
             {7, 14, 6, 1, 2}}},
    {25, 5, {{7, 13, 3, 0, 1}, {13, 3, 9, 0, 1}, {7, 13, 6, 1, 2}, {13, 6, 12, 1, 2},
             {7, 13, 5, 0, 2}}},
    {26, 5, {{7, 11, 5, 0, 2}, {11, 5, 9, 0, 2}, {7, 11, 6, 1, 2}, {11, 6, 10, 1, 2},
             {7, 11, 3, 0, 1}}},
    {27, 12, {{15, 7, 3, 0, 1}, {15, 7, 5, 0, 2}, {15, 7, 6, 1, 2}, {15, 11, 3, 0, 1},
              {15, 11, 9, 0, 3}, {15, 11, 10, 1, 3}, {15, 13, 5, 0, 2}, {15, 13, 9, 0, 3},
              {15, 13, 12, 2, 3}, {15, 14, 6, 1, 2}, {15, 14, 10, 1, 3}, {15, 14, 12, 2, 3}}},
};

typedef struct {
  int code, count;
  uint8_t rows[3][4];
} tri_case_t;

static const tri_case_t kTri[] = {
    {2, 1, {{5, 6, 0, 2}}},
    {4, 1, {{3, 6, 0, 1}}},
    {5, 1, {{3, 5, 0, 1}}},
    {6, 3, {{7, 3, 0, 1}, {7, 6, 1, 2}, {7, 5, 0, 2}}},
};

static const tet_case_t* tet_case(int code) {
  for (size_t i = 0; i < sizeof kTet / sizeof kTet[0]; ++i)
    if (kTet[i].code == code) return &kTet[i];
  return NULL;
}
static const tri_case_t* tri_case(int code) {
  for (size_t i = 0; i < sizeof kTri / sizeof kTri[0]; ++i)
    if (kTri[i].code == code) return &kTri[i];
  return NULL;
}

int orc_tetra_case(int code, uint8_t* out) {
  const tet_case_t* c = tet_case(code);
  if (!c) return 0;
  if (out) memcpy(out, c->rows, (size_t)c->count * 5);
  return c->count;
}

int orc_triangle_case(int code, uint8_t* out) {
  const tri_case_t* c = tri_case(code);
  if (!c) return 0;
  if (out) memcpy(out, c->rows, (size_t)c->count * 4);
  return c->count;
}

/* ----------------------------------------------------------------- cells -- */

/* Cube tetrahedra: monotone lattice paths in permutation order
 * (proj/src/complex.cpp:23-24, cell() :203-218). */
static const int kAxisOrder[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                     {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

int64_t orc_num_cells(const int64_t d[3]) {
  grid_t g;
  grid_init(&g, d);
  if (g.dim == 3) return 6 * (d[0] - 1) * (d[1] - 1) * (d[2] - 1);
  return 2 * (d[g.ax0] - 1) * (d[g.ax1] - 1);
}

static int cell_of(const grid_t* g, int64_t c, int64_t out[4]) {
  const int64_t* d = g->d;
  const int64_t step[3] = {1, d[0], d[0] * d[1]};
  if (g->dim == 3) {
    int64_t cube = c / 6;
    int t = (int)(c % 6);
    int64_t cx = cube % (d[0] - 1), cy = (cube / (d[0] - 1)) % (d[1] - 1),
            cz = cube / ((d[0] - 1) * (d[1] - 1));
    int64_t v = cx + step[1] * cy + step[2] * cz;
    out[0] = v;
    for (int i = 0; i < 3; ++i) {
      v += step[kAxisOrder[t][i]];
      out[i + 1] = v;
    }
    return 4;
  }
  /* 2-D (proj/src/complex.cpp:219-231) */
  int64_t sq = c / 2;
  int t = (int)(c % 2);
  int64_t u = sq % (d[g->ax0] - 1), w = sq / (d[g->ax0] - 1);
  int64_t p = u * step[g->ax0] + w * step[g->ax1];
  out[0] = p;
  out[1] = p + (t == 0 ? step[g->ax0] : step[g->ax1]);
  out[2] = p + step[g->ax0] + step[g->ax1];
  out[3] = -1;
  return 3;
}

int orc_cell(const int64_t dims[3], int64_t c, int64_t out[4]) {
  grid_t g;
  grid_init(&g, dims);
  return cell_of(&g, c, out);
}

/* position (proj/src/complex.cpp:235-244): origin + spacing * coord, each
 * component a rounded multiply then a rounded add. */
static void position(const grid_t* g, const double sp[3], const double og[3], int64_t v,
                     double p[3]) {
  int64_t x = v % g->d[0], y = (v / g->d[0]) % g->d[1], z = v / (g->d[0] * g->d[1]);
  double c[3] = {(double)x, (double)y, (double)z};
  for (int k = 0; k < 3; ++k) {
    volatile double m = sp[k] * c[k];
    p[k] = og[k] + m;
  }
}

/* ------------------------------------------------------------ separators -- */

/* index_separators (proj/src/marching.cpp:104-134), one worker. */
int64_t orc_index_separators(const int64_t dims[3], const int64_t* labels, uint8_t* codes) {
  grid_t g;
  grid_init(&g, dims);
  int64_t nc = orc_num_cells(dims), total = 0;
  for (int64_t c = 0; c < nc; ++c) {
    int64_t v[4], l[4] = {0, 0, 0, 0};
    int ar = cell_of(&g, c, v), code;
    for (int i = 0; i < ar; ++i) l[i] = labels[v[i]];
    if (ar == 4) {
      code = orc_tetra_code(l, NULL);
      total += orc_tetra_case(code, NULL);
    } else {
      code = orc_triangle_code(l);
      total += orc_triangle_case(code, NULL);
    }
    if (codes) codes[c] = (uint8_t)code;
  }
  return total;
}

/* recipe_point (proj/src/marching.cpp:71-82): sum of the masked vertex
 * positions in ascending corner order starting from +0.0, divided by count. */
static void recipe_point(const grid_t* g, const double sp[3], const double og[3],
                         const int64_t* v, int ar, int mask, double out[3]) {
  double s[3] = {0.0, 0.0, 0.0};
  int n = 0;
  for (int i = 0; i < ar; ++i)
    if (mask & (1 << i)) {
      double p[3];
      position(g, sp, og, v[i], p);
      for (int k = 0; k < 3; ++k) s[k] = s[k] + p[k];
      ++n;
    }
  for (int k = 0; k < 3; ++k) out[k] = s[k] / (double)n;
}

/* emit_geometry (proj/src/marching.cpp:136-206): cell-major soup, region pair
 * = (min, max) of labels at pairA/pairB (:84-90), source cell = c. */
void orc_emit_geometry(const int64_t dims[3], const double spacing[3], const double origin[3],
                       const int64_t* labels, const uint8_t* codes, double* points,
                       int64_t* regions, int64_t* source_cells) {
  grid_t g;
  grid_init(&g, dims);
  int64_t nc = orc_num_cells(dims), prim = 0;
  for (int64_t c = 0; c < nc; ++c) {
    int64_t v[4];
    int ar = cell_of(&g, c, v);
    int code = codes[c];
    if (ar == 4) {
      const tet_case_t* tc = tet_case(code);
      if (!tc) continue;
      for (int r = 0; r < tc->count; ++r, ++prim) {
        const uint8_t* row = tc->rows[r];
        for (int k = 0; k < 3; ++k) recipe_point(&g, spacing, origin, v, 4, row[k], points + 9 * prim + 3 * k);
        int64_t la = labels[v[row[3]]], lb = labels[v[row[4]]];
        regions[2 * prim] = la < lb ? la : lb;
        regions[2 * prim + 1] = la < lb ? lb : la;
        source_cells[prim] = c;
      }
    } else {
      const tri_case_t* tc = tri_case(code);
      if (!tc) continue;
      for (int r = 0; r < tc->count; ++r, ++prim) {
        const uint8_t* row = tc->rows[r];
        for (int k = 0; k < 2; ++k) recipe_point(&g, spacing, origin, v, 3, row[k], points + 6 * prim + 3 * k);
        int64_t la = labels[v[row[2]]], lb = labels[v[row[3]]];
        regions[2 * prim] = la < lb ? la : lb;
        regions[2 * prim + 1] = la < lb ? lb : la;
        source_cells[prim] = c;
      }
    }
  }
}

/* ------------------------------------------------------------ boundaries -- */

typedef struct {
  int64_t v[3], tag, cell;
} bface_t;

static int cmp_face(const void* pa, const void* pb) {
  const bface_t *a = (const bface_t*)pa, *b = (const bface_t*)pb;
  for (int k = 0; k < 3; ++k)
    if (a->v[k] != b->v[k]) return a->v[k] < b->v[k] ? -1 : 1;
  if (a->tag != b->tag) return a->tag < b->tag ? -1 : 1;
  if (a->cell != b->cell) return a->cell < b->cell ? -1 : 1;
  return 0;
}

static int cmp_i64(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  return a < b ? -1 : (a > b);
}

/* emit_boundaries (proj/src/marching.cpp:236-326): a tet emits the face of
 * the first "lone" corner whose other three corners share a label that the
 * lone one does not; triangles emit the analogous edge. Sort by (face, tag,
 * cell), keep one per (face, tag) — lowest cell — then points are the sorted
 * unique used vertices. */
void orc_emit_boundaries(const int64_t dims[3], const double spacing[3], const double origin[3],
                         const int64_t* labels, int has_filter, int64_t filter, int64_t sizes[2],
                         int64_t* faces_out, int64_t* tags, int64_t* cells, double* points,
                         int64_t* indices) {
  grid_t g;
  grid_init(&g, dims);
  int64_t nc = orc_num_cells(dims), nf = 0, cap = 1024;
  bface_t* f = (bface_t*)malloc(sizeof(bface_t) * (size_t)cap);
  for (int64_t c = 0; c < nc; ++c) {
    int64_t v[4], l[4];
    int ar = cell_of(&g, c, v);
    for (int i = 0; i < ar; ++i) l[i] = labels[v[i]];
    for (int lone = 0; lone < ar; ++lone) {
      bface_t b;
      if (ar == 4) {
        int64_t shared = l[(lone + 1) % 4];
        int all = 1;
        for (int i = 0; i < 4; ++i)
          if (i != lone && l[i] != shared) all = 0;
        if (!all || l[lone] == shared) continue;
        if (has_filter && shared != filter) break;
        int k = 0;
        for (int i = 0; i < 4; ++i)
          if (i != lone) b.v[k++] = v[i];
        b.tag = shared;
      } else {
        int i = (lone + 1) % 3, j = (lone + 2) % 3;
        if (l[i] != l[j] || l[lone] == l[i]) continue;
        if (has_filter && l[i] != filter) break;
        b.v[0] = v[i] < v[j] ? v[i] : v[j];
        b.v[1] = v[i] < v[j] ? v[j] : v[i];
        b.v[2] = -1;
        b.tag = l[i];
      }
      b.cell = c;
      if (nf == cap) {
        cap *= 2;
        f = (bface_t*)realloc(f, sizeof(bface_t) * (size_t)cap);
      }
      f[nf++] = b;
      break;
    }
  }
  qsort(f, (size_t)nf, sizeof(bface_t), cmp_face);
  int64_t u = 0;
  for (int64_t i = 0; i < nf; ++i)
    if (u == 0 || !(f[u - 1].v[0] == f[i].v[0] && f[u - 1].v[1] == f[i].v[1] &&
                    f[u - 1].v[2] == f[i].v[2] && f[u - 1].tag == f[i].tag))
      f[u++] = f[i];
  nf = u;
  const int ar = g.dim == 3 ? 3 : 2;
  int64_t* used = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nf * ar + 1));
  int64_t nu = 0;
  for (int64_t i = 0; i < nf; ++i)
    for (int k = 0; k < ar; ++k) used[nu++] = f[i].v[k];
  qsort(used, (size_t)nu, sizeof(int64_t), cmp_i64);
  int64_t w = 0;
  for (int64_t i = 0; i < nu; ++i)
    if (w == 0 || used[w - 1] != used[i]) used[w++] = used[i];
  nu = w;
  sizes[0] = nf;
  sizes[1] = nu;
  if (faces_out || tags || cells || points || indices) {
    for (int64_t i = 0; i < nf; ++i) {
      for (int k = 0; k < ar; ++k) {
        if (faces_out) faces_out[ar * i + k] = f[i].v[k];
        if (indices) {
          int64_t lo = 0, hi = nu;
          while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (used[mid] < f[i].v[k])
              lo = mid + 1;
            else
              hi = mid;
          }
          indices[ar * i + k] = lo;
        }
      }
      if (tags) tags[i] = f[i].tag;
      if (cells) cells[i] = f[i].cell;
    }
    if (points)
      for (int64_t i = 0; i < nu; ++i) position(&g, spacing, origin, used[i], points + 3 * i);
  }
  free(used);
  free(f);
}
