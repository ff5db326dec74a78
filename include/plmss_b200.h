/* plmss_b200 — B200-native (sm_100a) PL Morse-Smale segmentation hot path.
 *
 * C-ABI drop-in boundary. Plain pointers, sizes and status codes; no C++ or
 * torch types cross it. Each entry point names the reference interface it
 * replaces (paths relative to the reference repo, proj/include/plmss/...).
 * The C++ facade (paper_2303_15491_b200/csrc/dropin/plmss_dropin.cpp) maps
 * these back onto the reference's own C++ signatures and exception types.
 *
 * Conventions
 *  - dims = {X, Y, Z}; vertex id v = x + X*(y + Y*z) (x fastest), as
 *    SimplicialComplex3::implicit_grid (complex.hpp:52-55, complex.cpp:91-126).
 *    Only 3-D grids (all dims >= 2) with X*Y*Z < 2^32 are accepted.
 *  - Device pointers are prefixed d_, host pointers h_. All device work is
 *    issued on the context's stream; functions return after the work that
 *    produces host-visible scalars (counts) has completed.
 *  - Vertex ids, extremum labels and dense region ids are uint32 on device;
 *    the reference's int64 VertexId/Label (types.hpp:9-16) are widened by the
 *    facade.
 *  - Status: PLMSS_OK, or an error whose text plmss_b200_last_error() returns
 *    (thread-local). Error classes mirror the reference exceptions:
 *    INVALID_ARGUMENT <-> std::invalid_argument, LOGIC <-> std::logic_error,
 *    OUT_OF_RANGE <-> std::out_of_range.
 *  - There is no CPU fallback: without a CUDA device every call fails with
 *    PLMSS_ERR_CUDA.
 */
#ifndef PLMSS_B200_H
#define PLMSS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum plmss_status {
  PLMSS_OK = 0,
  PLMSS_ERR_INVALID_ARGUMENT = 1,
  PLMSS_ERR_LOGIC = 2,
  PLMSS_ERR_OUT_OF_RANGE = 3,
  PLMSS_ERR_CUDA = 4,
  PLMSS_ERR_NOMEM = 5,
  PLMSS_ERR_FORMAT = 6, /* io.hpp FormatError: malformed file or dims  */
  PLMSS_ERR_IO = 7      /* io.hpp IoError: open / read / write failure */
};

/* Scalar key types accepted by segmentation. */
enum plmss_key_type {
  PLMSS_KEY_F32 = 0,  /* float values, compared as (value, id)            */
  PLMSS_KEY_F64 = 1,  /* double values, compared as (value, id)           */
  PLMSS_KEY_RANK = 2  /* int64 OrderField ranks (orderfield.hpp:23-30)    */
};

/* plmss::Direction (segmentation.hpp:14). */
enum plmss_direction { PLMSS_ASCENDING = 0, PLMSS_DESCENDING = 1, PLMSS_BOTH = 2 };

/* Compact separator record (16 B), written in the reference's output order:
 * cell-major, then table row (marching.cpp:136-206, F7 in SURVEY.md).
 *   cell_row = cell_id << 6 | row, row in [0, 52) indexes the recipe table
 *              of marching_tables.cpp:48-116 regrouped by ascending code
 *              (plmss_b200_tet_table() exports it);
 *   lo, hi   = sorted region pair (marching.cpp:84-90).
 * plmss_b200_materialize_separators() expands it to the reference layout. */
typedef struct plmss_tri {
  uint64_t cell_row;
  uint32_t lo, hi;
} plmss_tri;

/* Same record for int64 label fields (API path with arbitrary labels). */
typedef struct plmss_tri64 {
  uint64_t cell_row;
  int64_t lo, hi;
} plmss_tri64;

typedef struct plmss_ctx plmss_ctx;

/* Host copy of the device recipe table: rows[52] packed as
 * p0 | p1<<4 | p2<<8 | pairA<<12 | pairB<<14, cases[32] = first_row<<4 | count.
 * Needs no GPU (used by the CPU tests to pin the table to the reference). */
void plmss_b200_tet_table(uint32_t rows[52], uint16_t cases[32]);

const char* plmss_b200_last_error(void);
/* Library version string and the SM architecture it was compiled for. */
const char* plmss_b200_version(void);
/* Total kernel launches issued by this library so far (all contexts). */
unsigned long long plmss_b200_launch_count(void);

/* Context = device + stream + grow-only scratch arena. stream may be NULL
 * (the context then creates its own non-blocking stream). */
int plmss_b200_ctx_create(int device, void* stream, plmss_ctx** out);
void plmss_b200_ctx_destroy(plmss_ctx* ctx);
/* Bytes of device scratch currently held by the context. */
size_t plmss_b200_ctx_scratch_bytes(const plmss_ctx* ctx);
/* Frees the context's scratch arena (every result pointer it handed out
 * becomes invalid) and trims the device memory pool. */
int plmss_b200_ctx_release(plmss_ctx* ctx);
/* Device time (ms) of the last kernel stage named by `stage` (see
 * plmss_b200_pipeline): 0 hops, 1 compress, 2 extrema, 3 combine, 4 marching.
 * Only filled when timing is enabled. */
int plmss_b200_ctx_set_timing(plmss_ctx* ctx, int enable);
int plmss_b200_ctx_stage_ms(const plmss_ctx* ctx, float out[8]);
/* Diagnostics of the last fused pipeline call: [0] exit-graph entries,
 * [1] pass-A capacity retries, [2] region-set capacity (negative: bitmap
 * words), [4] TMA field loads used. */
int plmss_b200_ctx_stats(const plmss_ctx* ctx, int64_t out[8]);

/* ---- order field --------------------------------------------------------
 * Replaces compute_order (orderfield.hpp:35, orderfield.cpp:12-32): d_rank[v]
 * = position of v in the sort by (value, id). Fails with INVALID_ARGUMENT
 * "non-finite scalar value at vertex i" (lowest i). key_type F32 or F64. */
int plmss_b200_compute_order(plmss_ctx* ctx, int key_type, const void* d_values, int64_t n,
                             int64_t* d_rank);

/* ---- segmentation -------------------------------------------------------
 * Replaces segment() (segmentation.hpp:74-76, segmentation.cpp:109-168):
 * steepest-neighbour hops over the 14-neighbour Freudenthal stencil with
 * (key, id) simulation of simplicity, then path compression to the fixpoint.
 * d_desc / d_asc (N each) may be NULL when the direction does not ask for
 * them. d_maxima / d_minima receive the extrema ascending (capacity N) and
 * may be NULL; counts go to *n_maxima / *n_minima. *sweeps = compression
 * sweeps (schedule-dependent, not part of parity). */
int plmss_b200_segment(plmss_ctx* ctx, const int64_t dims[3], int key_type, const void* d_keys,
                       int direction, uint32_t* d_desc, uint32_t* d_asc, uint32_t* d_maxima,
                       uint32_t* d_minima, int64_t* n_maxima, int64_t* n_minima, int32_t* sweeps);

/* Slab segmentation for the z-slab multi-GPU decomposition: the grid is one
 * rank's slab extended by its halo layers; when halo_lo (halo_hi) is set the
 * first (last) z layer is a copy of the neighbour rank's boundary layer and
 * its vertices are made terminals (hop = self), so after compression every
 * owned vertex points at a root of its own slab or at a halo vertex whose
 * label the neighbour resolves (paper_2303_15491_b200/distributed.py). */
int plmss_b200_segment_slab(plmss_ctx* ctx, const int64_t dims[3], int key_type, const void* d_keys,
                            int halo_lo, int halo_hi, uint32_t* d_desc, uint32_t* d_asc, int32_t* sweeps);

/* ---- z-slab pipeline (multi-GPU) --------------------------
 * The fused pipeline on one rank's z-slab, in four stages; the caller runs
 * the exchanges between them (paper_2303_15491_b200/distributed.py, NCCL):
 *   1 slab_segment : pass A on the slab's bricks (field halo layers as real
 *                    data), sorted extremum lists, the terminal forest inside
 *                    the slab; chains leaving the slab end at portals.
 *     -> all_gather counts, extremum lists, boundary layers
 *   2 slab_resolve : portals resolved through every rank's boundary layers,
 *                    desc / asc (global vertex ids), region tokens, the slab's
 *                    distinct rank pairs.
 *     -> all_gather the rank pairs
 *   3 slab_ids     : the global region table (combine_ms order); the hash
 *                    mode writes the dense ids into ms, the dense mode keeps
 *                    its (globally consistent) region tokens there.
 *     -> the next rank's first layer of ms into ms's extra layer
 *   4 slab_emit    : the dense ids of the owned vertices (+ the extra layer)
 *                    into d_ids, separator records of the owned cube layers,
 *                    global cell ids, reference order.
 * No reference counterpart (the reference is one process, parallel.hpp:27-57
 * splits work among threads); results equal the single-volume pipeline's.
 * Slabs are whole 32-layer brick layers: z0 % 32 == 0, z1 % 32 == 0 or
 * z1 == Z. All device pointers handed to a stage must stay valid until
 * slab_emit returns. */
typedef struct plmss_slab_info {
  int64_t n_maxima, n_minima;      /* stage 1: the slab's; stage 2+: global */
  const uint32_t* d_maxima;        /* stage 1: the slab's sorted extrema (global vertex ids) */
  const uint32_t* d_minima;
  const uint32_t* d_boundary;      /* stage 1: [desc, asc] x [first, last owned layer] x X*Y words */
  int64_t n_keys;                  /* stage 2: the slab's distinct (rank_min << 32 | rank_max) */
  const uint64_t* d_keys;
  int64_t n_regions;               /* stage 3: global region count and keys (asc << 32 | desc, sorted) */
  const uint64_t* d_region_keys;
  int64_t n_tris;                  /* stage 4: this slab's separator records */
  const plmss_tri* d_tris;
  int32_t sweeps;                  /* forest sweeps inside the slab */
  int32_t dense;                   /* 1: rank-product bitmap, 0: region hash set */
} plmss_slab_info;

/* d_field: vertex layers [z0 - 1, z1 + 1) clipped to [0, Z) (halos of the
 * ranks below / above). */
int plmss_b200_slab_segment(plmss_ctx* ctx, const int64_t dims[3], int64_t z0, int64_t z1, const float* d_field,
                            plmss_slab_info* info);
/* d_boundary_all: every rank's d_boundary, rank order (world * 4 * X*Y);
 * h_max_counts / h_min_counts: every rank's n_maxima / n_minima (host);
 * d_maxima_all / d_minima_all: the concatenated lists (rank order = id
 * order). Outputs: d_desc, d_asc (owned vertices), d_ms (owned vertices +
 * one more layer when z1 < Z; region tokens until slab_ids). */
int plmss_b200_slab_resolve(plmss_ctx* ctx, const uint32_t* d_boundary_all, int world, int rank,
                            const int64_t* h_max_counts, const int64_t* h_min_counts, const uint32_t* d_maxima_all,
                            const uint32_t* d_minima_all, uint32_t* d_desc, uint32_t* d_asc, uint32_t* d_ms,
                            plmss_slab_info* info);
/* d_keys_all: every rank's d_keys concatenated (duplicates allowed). */
int plmss_b200_slab_ids(plmss_ctx* ctx, const uint64_t* d_keys_all, int64_t n_keys_all, plmss_slab_info* info);
/* The layer z1 of d_ms holds the next rank's first layer of d_ms (z1 < Z);
 * d_ids has the layout of d_ms and receives the dense MS ids. */
int plmss_b200_slab_emit(plmss_ctx* ctx, uint32_t* d_ids, plmss_slab_info* info);

/* Step 1 only (detail::seed_hops_both, segmentation.cpp:60-85): hop targets. */
int plmss_b200_seed_hops(plmss_ctx* ctx, const int64_t dims[3], int key_type, const void* d_keys,
                         uint32_t* d_desc, uint32_t* d_asc);

/* One path-compression sweep over an active list (detail::compress_sweep /
 * compress_sweep_both, segmentation.cpp:48-58, 87-105): label <- label[label]
 * for every active vertex (d_asc may be NULL), in place and concurrently like
 * the reference's workers; d_next receives the still-unsettled vertices in
 * list order, *n_next their count. */
int plmss_b200_compress_sweep(plmss_ctx* ctx, uint32_t* d_desc, uint32_t* d_asc, const uint32_t* d_active,
                              int64_t n_active, uint32_t* d_next, int64_t* n_next);

/* ---- Morse-Smale combine ------------------------------------------------
 * Replaces combine_ms (segmentation.hpp:80, segmentation.cpp:170-196):
 * d_ms[v] = rank of (asc[v], desc[v]) among the distinct pairs in
 * lexicographic order; d_region_keys[r] = asc << 32 | desc of region r
 * (the reference's MsKey = min << 64 | max, segmentation.hpp:21-24, narrowed
 * to u32 halves). d_region_keys capacity: N. */
int plmss_b200_combine_ms(plmss_ctx* ctx, int64_t n, const uint32_t* d_asc, const uint32_t* d_desc,
                          uint32_t* d_ms, uint64_t* d_region_keys, int64_t* n_regions);

/* ---- marching tetrahedra ------------------------------------------------
 * label_type: 0 = uint32 labels, 1 = int64 labels.
 * index_separators (marching.hpp:101-102, marching.cpp:104-134): per-cell
 * codes (d_codes, 6(X-1)(Y-1)(Z-1) bytes, may be NULL) and the total. */
int plmss_b200_index_separators(plmss_ctx* ctx, const int64_t dims[3], int label_type,
                                const void* d_labels, uint8_t* d_codes, int64_t* total);

/* Separator primitives per contiguous cell range [bounds[i], bounds[i+1])
 * (nranges + 1 bounds) — the per-worker counts of EmitPlan
 * (marching.hpp:81-93, marching.cpp:116-133), computed on the device. */
int plmss_b200_count_by_cell_ranges(plmss_ctx* ctx, const int64_t dims[3], int label_type,
                                    const void* d_labels, const int64_t* h_bounds, int nranges,
                                    int64_t* h_counts);

/* emit_separators (marching.hpp:115-117, marching.cpp:136-215): compact
 * records in reference order. d_out has room for `capacity` records
 * (plmss_tri for label_type 0, plmss_tri64 for 1); *total is always set; if
 * total > capacity nothing is written and PLMSS_ERR_LOGIC is returned. */
int plmss_b200_emit_separators(plmss_ctx* ctx, const int64_t dims[3], int label_type,
                               const void* d_labels, void* d_out, int64_t capacity,
                               int64_t* total);

/* Expand records to the reference SeparatingMesh layout (marching.hpp:65-76):
 * d_points 9 doubles per triangle (3 corners x xyz, Eigen column-major),
 * d_regions 2 int64, d_source_cells 1 int64 (any may be NULL). Points follow
 * recipe_point (marching.cpp:71-82) bit for bit: ascending-corner sum from
 * +0.0 of origin + spacing*coord, divided by the corner count. */
int plmss_b200_materialize_separators(plmss_ctx* ctx, const int64_t dims[3], const double spacing[3],
                                      const double origin[3], int label_type, const void* d_tris,
                                      int64_t n, double* d_points, int64_t* d_regions,
                                      int64_t* d_source_cells);

/* The same SeparatingMesh arrays streamed chunk by chunk into a host sink
 * (outputs larger than device or host memory: cfg3's 5.4 G triangles are
 * ~520 GB of geometry). The sink gets triangles [first, first + count):
 * points 9 doubles, regions 2 int64, source cells 1 int64 per triangle, in
 * pinned host buffers valid until it returns; a nonzero return stops the
 * stream (PLMSS_ERR_LOGIC). chunk <= 0: 4 Mi triangles. The device
 * materialisation and copy of the next chunk overlap the sink. */
typedef int (*plmss_geometry_sink)(void* user, int64_t first, int64_t count, const double* points,
                                   const int64_t* regions, const int64_t* source_cells);
int plmss_b200_materialize_separators_chunked(plmss_ctx* ctx, const int64_t dims[3], const double spacing[3],
                                              const double origin[3], int label_type, const void* d_tris,
                                              int64_t n, int64_t chunk, plmss_geometry_sink sink, void* user);

/* emit_boundaries (marching.hpp:123-126, marching.cpp:236-326): faces whose
 * 3 vertices share a label that the 4th tet vertex lacks, one per face
 * (lowest generating cell), in (v0, v1, v2) order. Two calls: with
 * d_faces == NULL only *n_faces / *n_points are computed. Outputs: d_faces
 * 3 uint32 vertex ids per face, d_tags (label_type width), d_cells int64,
 * d_points 3 doubles per sorted unique used vertex, d_indices 3 int64 per
 * face. */
int plmss_b200_emit_boundaries(plmss_ctx* ctx, const int64_t dims[3], const double spacing[3],
                               const double origin[3], int label_type, const void* d_labels,
                               int has_filter, int64_t filter, uint32_t* d_faces, void* d_tags,
                               int64_t* d_cells, double* d_points, int64_t* d_indices,
                               int64_t* n_faces, int64_t* n_points);

/* ---- fused full pipeline (the benchmarked path) --------------------------
 * run_benchmark's MorseSmale pass (bench.cpp:66-87) minus compute_order:
 * f32 field -> desc, asc, maxima, minima, ms_region, region_keys, separator
 * records. Outputs live in the context until the next call; fetch with
 * plmss_b200_result(). */
typedef struct plmss_result {
  const uint32_t* d_desc;
  const uint32_t* d_asc;
  const uint32_t* d_ms;
  const uint32_t* d_maxima;
  const uint32_t* d_minima;
  const uint64_t* d_region_keys;
  const plmss_tri* d_tris;
  int64_t n_vertices, n_maxima, n_minima, n_regions, n_tris;
  int32_t sweeps;
} plmss_result;

int plmss_b200_pipeline(plmss_ctx* ctx, const int64_t dims[3], const float* d_field);
int plmss_b200_result(const plmss_ctx* ctx, plmss_result* out);
/* Copies `bytes` from a device pointer (e.g. a plmss_result array) to dst
 * (host when to_host != 0, else device) on the context stream, then syncs. */
int plmss_b200_copy(plmss_ctx* ctx, void* dst, const void* d_src, int64_t bytes, int to_host);

/* Tuning / test options:
 *   PLMSS_OPT_COMBINE_PATH  0 auto, 1 bitmap, 2 hash (staged combine_ms, and the
 *                           fused pipeline's region keys);
 *   PLMSS_OPT_PIPELINE_PATH 0 fused tile pipeline when the dims allow it,
 *                           1 staged kernels (segment/combine/emit);
 *   PLMSS_OPT_TMA           1 (default) TMA tensor loads of the field bricks,
 *                           0 plain load loop (both are exact);
 *   PLMSS_OPT_SPECULATIVE_SWEEPS  forest sweeps enqueued before the fused
 *                           pipeline's passes C and D (default 1); if the
 *                           forest has not converged by then, the sweeps
 *                           continue and C, D are redone (0 forces that path);
 *   PLMSS_OPT_PASS_A_SPLIT  1: pass A as two kernels (hop codes at high
 *                           occupancy, then the brick compression from the
 *                           codes), 0: one fused kernel (both are exact);
 *   PLMSS_OPT_HOP_CUBE      1 (default): steepest hops from shared 2x2 quads / unit
 *                           cubes, 0: per-vertex equality masks (both exact);
 *   PLMSS_OPT_IDS_IN_COUNT  1 (default): region tokens in a scratch array, the count pass
 *                           writes the dense ids (no in-place id pass over
 *                           ms), 0: tokens in ms, counts interleaved with the
 *                           token pass, then the id pass; 2: a mark pass builds
 *                           the region bitmap first, the token pass writes the
 *                           ids into ms, counts interleaved (dense keys; all
 *                           exact). */
/* pipeline_host over a sequence of volumes of the same dims, double-buffered:
 * two internal contexts (own non-blocking streams, created on first use,
 * options copied from ctx) take alternate volumes on two host threads, so
 * volume i+1's upload and compute overlap volume i's download (host <-> device
 * copies run in both directions at once). Each volume's outputs and counts
 * as in pipeline_host; result device pointers are not valid after return.
 * Returns the first failing volume's status (each one's in ->status). */
typedef struct plmss_host_volume {
  const float* h_field;
  uint32_t *h_desc, *h_asc, *h_ms, *h_maxima, *h_minima;
  uint64_t* h_region_keys;
  plmss_tri* h_tris;
  int64_t tri_capacity;
  plmss_result result;
  int32_t status;
} plmss_host_volume;
int plmss_b200_pipeline_host_batch(plmss_ctx* ctx, const int64_t dims[3], plmss_host_volume* volumes, int64_t n);

/* ---- callers either side of the path ------------------
 * weld_points (marching.hpp:138-140, marching.cpp:400-417): merges
 * bitwise-identical points of a separator soup in place, the first occurrence
 * of each point keeping its place in order; d_points is (n_points, 3) float64
 * (the reference's column-major Matrix3Xd), d_indices are remapped.
 * *n_unique receives the new point count. Out-of-range indices:
 * PLMSS_ERR_OUT_OF_RANGE. */
int plmss_b200_weld_points(plmss_ctx* ctx, double* d_points, int64_t n_points, int64_t* d_indices,
                           int64_t n_indices, int64_t* n_unique);

/* read_volume (io.hpp:46-55, io.cpp:90-124): headerless little-endian raw
 * volume, x fastest, streamed through pinned staging buffers into device
 * memory: d_out is float64 (out_f64 = 1, like the reference's ScalarField) or
 * float32 (out_f64 = 0, the pipeline's input; refused for f64le files). File
 * size != X*Y*Z*sizeof(dtype): PLMSS_ERR_FORMAT with the reference's text. */
enum plmss_dtype {
  PLMSS_DTYPE_F32LE = 0,
  PLMSS_DTYPE_F64LE = 1,
  PLMSS_DTYPE_U8 = 2,
  PLMSS_DTYPE_U16LE = 3,
  PLMSS_DTYPE_I16LE = 4
};
int plmss_b200_read_volume(plmss_ctx* ctx, const char* path, const int64_t dims[3], int dtype, int out_f64,
                           void* d_out);

/* write_labels (io.hpp:66-70, io.cpp:216-235): "PLMSSLBL", u32 1, u64 n, then
 * (u64 asc, u64 desc) per vertex, from device label arrays (label_type 0 =
 * uint32, 1 = int64), streamed in chunks. */
int plmss_b200_write_labels(plmss_ctx* ctx, const char* path, int label_type, const void* d_asc,
                            const void* d_desc, int64_t n);

/* write_surface_obj (io.hpp:79-83, io.cpp:268-299): the reference's OBJ text
 * ("v %.17g %.17g %.17g", "g rA_rB" on region changes, 1-based "f"/"l"
 * lines) from device arrays: points (n_points, 3) float64, indices
 * (n_prims * verts_per_prim) int64, regions (n_prims, 2) int64. */
int plmss_b200_write_surface_obj(plmss_ctx* ctx, const char* path, const double* d_points, int64_t n_points,
                                 const int64_t* d_indices, const int64_t* d_regions, int64_t n_prims,
                                 int verts_per_prim);

/* write_surface_obj(path, emit_separators(...)) of the reference (io.cpp:268-299
 * over the SeparatingMesh, marching.hpp:65-76) straight from the compact
 * records, streamed: points materialised on the device chunk by chunk, the
 * identity faces and region groups formatted on host threads. Byte-identical
 * to the reference file; the mesh is never held whole. */
int plmss_b200_write_separators_obj(plmss_ctx* ctx, const char* path, const int64_t dims[3],
                                    const double spacing[3], const double origin[3], int label_type,
                                    const void* d_tris, int64_t n);

enum plmss_option {
  PLMSS_OPT_COMBINE_PATH = 1,
  PLMSS_OPT_PIPELINE_PATH = 2,
  PLMSS_OPT_TMA = 3,
  PLMSS_OPT_SPECULATIVE_SWEEPS = 4,
  PLMSS_OPT_PASS_A_SPLIT = 5,
  PLMSS_OPT_HOP_CUBE = 6,
  PLMSS_OPT_IDS_IN_COUNT = 7
};
int plmss_b200_ctx_set_option(plmss_ctx* ctx, int option, int64_t value);

/* End-to-end variant over HOST buffers: pinned or pageable h_field in; the
 * label arrays (N each, any may be NULL), extrema, region keys and separator
 * records are copied back to host buffers of the given capacities (counts are
 * always reported in *out). */
int plmss_b200_pipeline_host(plmss_ctx* ctx, const int64_t dims[3], const float* h_field,
                             uint32_t* h_desc, uint32_t* h_asc, uint32_t* h_ms,
                             uint32_t* h_maxima, uint32_t* h_minima, uint64_t* h_region_keys,
                             plmss_tri* h_tris, int64_t tri_capacity, plmss_result* out);

/* ---- synthetic inputs (benchmark/test harness utility) -------------------
 * The input definition of include/plmss_synth.h (bit-identical to its host
 * loop): value(x,y,z) = sum_k amp_k * ex_k(x) * ey_k(y) * ez_k(z) (separable
 * Gaussians, float32 axis tables) + noise_amp * (2u - 1), u uniform in [0, 1)
 * from a splitmix64 hash of (seed, v); kind 1 = i.i.d. uniform [0, 1) from
 * the same hash (no Gaussians); levels > 0 quantises to that many levels over
 * [min, max]. gaussians: n_gauss x 5 doubles (cx, cy, cz, sigma, amp). */
int plmss_b200_synth(plmss_ctx* ctx, const int64_t dims[3], int kind, const double* h_gaussians,
                     int n_gauss, double noise_amp, uint64_t seed, int levels, float* d_field);
/* Vertex layers [z0, z0 + nz) of the same field (no quantisation) into
 * d_field (X * Y * nz floats): a rank's slab plus halo layers. */
int plmss_b200_synth_layers(plmss_ctx* ctx, const int64_t dims[3], int kind, const double* h_gaussians,
                            int n_gauss, double noise_amp, uint64_t seed, int64_t z0, int64_t nz, float* d_field);

#ifdef __cplusplus
}
#endif
#endif /* PLMSS_B200_H */
