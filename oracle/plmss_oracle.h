/* CPU restatement of the PLMSS hot path — TEST INFRASTRUCTURE ONLY.
 *
 * This is the checker the B200 path is compared against (tests/, smoke() and
 * bench.py's cpu_baseline leg only). The product library never links it.
 * Every function restates one reference function; the citation is on the
 * definition in plmss_oracle.c. It is itself pinned against (a) the golden
 * vectors of the reference's own tests (proj/tests/fixtures.hpp, the code
 * KATs in proj/tests/test_marching.cpp) and (b) the reference library compiled
 * unchanged from /root/reference (oracle/_ref/libplmss_ref.so), see
 * tests/test_oracle_pin.py.
 *
 * Conventions: ids and labels are int64 (proj/include/plmss/types.hpp:9-16);
 * dims = {X, Y, Z}, vertex id = x + X*(y + Y*z); scalar values are double
 * (float32 inputs are widened exactly, proj/src/io.cpp:101-104). Grids may be
 * 3-D or 2-D (exactly one dim == 1), like SimplicialComplex3::implicit_grid.
 */
#ifndef PLMSS_ORACLE_H
#define PLMSS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rank = position in the sort by (value, id). Returns -1, or the lowest
 * non-finite vertex (no ranks written then). */
int64_t orc_compute_order(const double* values, int64_t n, int64_t* rank);

/* Step 1 (fused both directions). key_kind 0: keys are double values compared
 * as (value, id); 1: keys are int64 ranks. desc/asc get the hop targets. */
void orc_seed_hops(const int64_t dims[3], const void* keys, int key_kind, int64_t* desc,
                   int64_t* asc);

/* Step 2: sweeps of label <- label[label] over an active list. Returns sweeps. */
int orc_compress(int64_t n, int64_t* desc, int64_t* asc);

/* Self-pointing vertices of `labels`, ascending. Returns count. */
int64_t orc_extrema(int64_t n, const int64_t* labels, int64_t* out);

/* Dense MS ids; keys_out gets (min, max) pairs (2*R int64). Returns R. */
int64_t orc_combine_ms(int64_t n, const int64_t* asc, const int64_t* desc, int64_t* ms_region,
                       int64_t* keys_out);

int orc_tetra_code(const int64_t labels[4], int local_out[4]);
int orc_triangle_code(const int64_t labels[3]);
/* Rows of a code: 5 bytes (p0,p1,p2,pairA,pairB) for tets, 4 (p0,p1,pairA,pairB) for triangles. */
int orc_tetra_case(int code, uint8_t* out);
int orc_triangle_case(int code, uint8_t* out);

int64_t orc_num_cells(const int64_t dims[3]);
/* Vertices of cell c (ascending); returns the arity (3 or 4). */
int orc_cell(const int64_t dims[3], int64_t c, int64_t out[4]);

/* Indexing phase: codes per cell; returns the total primitive count. */
int64_t orc_index_separators(const int64_t dims[3], const int64_t* labels, uint8_t* codes);
/* Geometry phase into reference layout (points: 3 doubles per corner,
 * arity corners per primitive; regions 2 per primitive; source cells). */
void orc_emit_geometry(const int64_t dims[3], const double spacing[3], const double origin[3],
                       const int64_t* labels, const uint8_t* codes, double* points,
                       int64_t* regions, int64_t* source_cells);

/* Boundaries. Call with all outputs NULL to get sizes[0]=faces, sizes[1]=points,
 * then again with buffers. faces_out: arity vertex ids per face (sorted order),
 * tags, cells; points: positions of the sorted unique used vertices; indices
 * into them. */
void orc_emit_boundaries(const int64_t dims[3], const double spacing[3], const double origin[3],
                         const int64_t* labels, int has_filter, int64_t filter, int64_t sizes[2],
                         int64_t* faces_out, int64_t* tags, int64_t* cells, double* points,
                         int64_t* indices);

/* ---- full-size grids (plmss_oracle_big.c): uint32 ids, float32 values,
 * OpenMP workers. ---- */

/* One separator triangle: (global cell << 6 | recipe row), region pair. */
typedef struct {
  uint64_t cellrow;
  uint32_t lo, hi;
} orc_tri;

/* The input definition of include/plmss_synth.h, vertex layers [z0, z0+nz). */
int orc_synth(const int64_t dims[3], int kind, const double* gauss, int ng, double noise, uint64_t seed,
              int levels, int64_t z0, int64_t nz, float* out);
int64_t orc_seed_hops_f32(const int64_t dims[3], const float* f, uint32_t* desc, uint32_t* asc);
int orc_compress_u32(int64_t n, uint32_t* desc, uint32_t* asc);
int64_t orc_extrema_u32(int64_t n, const uint32_t* labels, uint32_t* out);
int64_t orc_combine_ms_u32(int64_t n, const uint32_t* asc, const uint32_t* desc, uint32_t* ms, uint64_t* keys_out,
                           int64_t keys_cap);
int64_t orc_separator_records(const int64_t dims[3], const uint32_t* labels, int64_t cz0, int64_t cz1,
                              orc_tri* out);

#ifdef __cplusplus
}
#endif
#endif
