// Shared definitions of the plmss_b200 library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <functional>
#include <vector>
#include <stdexcept>
#include <string>

#include "plmss_b200.h"

namespace plmss_b200 {

// ---------------------------------------------------------------- errors ---
// Exceptions inside the library; capi.cu converts them to status codes.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(e == cudaErrorMemoryAllocation ? PLMSS_ERR_NOMEM : PLMSS_ERR_CUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
}
// Kernel launches issued by this library (reported by bench.py).
extern unsigned long long g_launches;
#define CK(x) ::plmss_b200::cuda_check((x), #x)
// Launch trace (measurement aid, PLMSS_KTRACE=1): the fused pipeline sets
// g_trace_stream, and every launch on it is followed by an event, so the
// gaps between kernels in the real (concurrent, warm-cache) pipeline can be
// read off — which ncu's serialised launch list cannot show.
extern thread_local cudaStream_t g_trace_stream;
void trace_launch(const char* name);
void trace_begin(cudaStream_t s);
void trace_end();
#define CK_LAUNCH(name)                                      \
  do {                                                       \
    __atomic_fetch_add(&::plmss_b200::g_launches, 1ull, __ATOMIC_RELAXED); \
    ::plmss_b200::cuda_check(cudaGetLastError(), name);      \
    if (::plmss_b200::g_trace_stream) ::plmss_b200::trace_launch(name); \
  } while (0)

// ------------------------------------------------------------------ grid ---
struct Grid {
  int64_t X, Y, Z;   // vertex extents
  int64_t n;         // vertices
  int64_t cubes;     // (X-1)(Y-1)(Z-1)
  int64_t cells;     // 6 * cubes
};

inline Grid make_grid(const int64_t* dims) {
  if (!dims) fail(PLMSS_ERR_INVALID_ARGUMENT, "dims is null");
  for (int a = 0; a < 3; ++a)
    if (dims[a] < 1)
      fail(PLMSS_ERR_INVALID_ARGUMENT, "grid dims must be positive, got " + std::to_string(dims[a]) +
                                           " on axis " + std::to_string(a));
  for (int a = 0; a < 3; ++a)
    if (dims[a] < 2)
      fail(PLMSS_ERR_INVALID_ARGUMENT,
           "the B200 path handles 3-D implicit grids only (every dim >= 2)");
  Grid g;
  g.X = dims[0];
  g.Y = dims[1];
  g.Z = dims[2];
  g.n = g.X * g.Y * g.Z;
  if (g.n >= (int64_t(1) << 32) - 1)
    fail(PLMSS_ERR_INVALID_ARGUMENT, "grid has >= 2^32-1 vertices; uint32 vertex ids required");
  g.cubes = (g.X - 1) * (g.Y - 1) * (g.Z - 1);
  g.cells = 6 * g.cubes;
  return g;
}

// --------------------------------------------------------------- context ---
enum Slot {
  S_DESC, S_ASC, S_MS, S_MAXIMA, S_MINIMA, S_KEYS, S_TRIS,  // pipeline results
  S_FLAGS,        // small device counters / flags
  S_SCAN_A, S_SCAN_B, S_SCAN_C,  // scan partials
  S_RANK_MAX, S_RANK_MIN,        // extremum -> rank maps (N, sparse use)
  S_BITMAP, S_HASH_K, S_HASH_V, S_SORT_A, S_SORT_B, S_SORT_C, S_SORT_D,
  S_TMP0, S_TMP1, S_TMP2, S_FIELD, S_MASK,
  S_LTD, S_LTA, S_TB, S_SD, S_SA, S_RK,  // fused pipeline: terminal indices, brick headers, table labels
  S_SLAB_BND,                             // z-slab pipeline: boundary layers
  S_CODES,                                // split pass A: hop codes (1 B per padded brick cell)
  S_TOKENS,                               // region tokens when the count pass writes the ids
  S_CHUNK_G,                              // record offset of every 32-chunk group
  S_COUNT
};

// State of the z-slab pipeline between its four C-ABI stages (fused.cu).
struct SlabState {
  int stage = 0;            // last completed stage (0: none)
  Grid g{};                 // the global grid
  int64_t z0 = 0, z1 = 0;   // owned vertex layers
  int has_down = 0, has_up = 0;
  uint64_t ntiles = 0, nt = 0;
  int64_t n_max_l = 0, n_min_l = 0, n_max_g = 0, n_min_g = 0;
  bool dense = true;
  uint64_t fcap = 0;        // hash mode: region set slots
  int64_t n_keys = 0, R = 0, n_tris = 0;
  int sweeps = 0;
  const uint32_t *maxs_g = nullptr, *mins_g = nullptr;
  uint32_t *desc = nullptr, *asc = nullptr, *ms = nullptr;
  uint32_t *bitmap = nullptr, *prefix = nullptr;  // dense mode: the global region bitmap and word prefix
  uint64_t* keys = nullptr;
  plmss_tri* tris = nullptr;
};

struct Ctx {
  int device = 0;
  SlabState slab;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* buf[S_COUNT] = {};
  size_t cap[S_COUNT] = {};
  uint64_t* h_pinned = nullptr;  // small pinned host staging for counters
  // pinned staging for the file streams (io.cu), kept across calls: pinning
  // costs more than the copy of a small volume
  unsigned char* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  unsigned char* stage(size_t bytes) {
    if (h_stage_bytes < bytes) {
      if (h_stage) CK(cudaFreeHost(h_stage));
      h_stage = nullptr;
      h_stage_bytes = 0;
      CK(cudaMallocHost(reinterpret_cast<void**>(&h_stage), bytes));
      h_stage_bytes = bytes;
    }
    return h_stage;
  }
  bool timing = false;
  float stage_ms[8] = {};
  cudaEvent_t ev[9] = {};
  // side stream for the z-slab pipelining of pass C, with its events
  cudaStream_t side = nullptr;
  cudaEvent_t join = nullptr;
  std::vector<cudaEvent_t> slab_ev;
  cudaEvent_t slab_event(size_t i) {
    while (slab_ev.size() <= i) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      slab_ev.push_back(e);
    }
    return slab_ev[i];
  }
  plmss_result result{};
  int sm_count = 148;
  int combine_path = 0;  // PLMSS_OPT_COMBINE_PATH
  int pipeline_path = 0; // PLMSS_OPT_PIPELINE_PATH: 0 fused when supported, 1 staged
  bool use_tma = true;   // PLMSS_OPT_TMA
  int spec_sweeps = 1;   // PLMSS_OPT_SPECULATIVE_SWEEPS
  bool pass_a_split = false;  // PLMSS_OPT_PASS_A_SPLIT
  bool hop_cube = true;       // PLMSS_OPT_HOP_CUBE
  int ids_mode = 1;           // PLMSS_OPT_IDS_IN_COUNT (0, 1, 2: mark pass)
  // Adaptive capacities of the fused pipeline (remembered between calls).
  uint64_t fused_exit_cap = 0, fused_pair_hint = 0, fused_tri_cap = 0, fused_ext_cap = 0;
  // Diagnostics of the last fused call: [0] exit entries, [1] pass-A retries,
  // [2] region-set capacity, [3] finalize retries.
  int64_t stats[8] = {};

  void* get(Slot s, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (cap[s] < bytes) {
      if (buf[s]) CK(cudaFreeAsync(buf[s], stream));
      buf[s] = nullptr;
      cap[s] = 0;
      size_t want = bytes + bytes / 8;  // headroom for repeated growth
      CK(cudaMallocAsync(&buf[s], want, stream));
      cap[s] = want;
    }
    return buf[s];
  }
  template <class T>
  T* get_t(Slot s, size_t count) {
    return static_cast<T*>(get(s, count * sizeof(T)));
  }
  void sync() { CK(cudaStreamSynchronize(stream)); }
  // stage boundaries of the fused pipeline: CUDA events (stage_ms) when
  // timing, and NVTX ranges (ncu --nvtx --nvtx-include "plmss.passA/")
  bool nvtx_open = false;
  void mark(int i) {
    if (timing) CK(cudaEventRecord(ev[i], stream));
    static const char* const kStage[5] = {"plmss.passA", "plmss.extrema_sort", "plmss.exit_resolve",
                                          "plmss.finalize_ids", "plmss.march"};
    if (nvtx_open) nvtxRangePop();
    nvtx_open = i < 5;
    if (nvtx_open) nvtxRangePushA(kStage[i]);
  }
};

inline unsigned blocks_for(int64_t n, int threads, int64_t cap = int64_t(1) << 31) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b < cap ? b : cap);
}

// --------------------------------------------- internal entry points ------
// segment.cu
void seed_hops(Ctx& c, const Grid& g, int key_type, const void* keys, uint32_t* desc, uint32_t* asc,
               uint32_t* bad_vertex /*device, may be null*/);
int compress(Ctx& c, int64_t n, uint32_t* desc, uint32_t* asc);
void terminal_layers(Ctx& c, const Grid& g, bool lo, bool hi, uint32_t* desc, uint32_t* asc);
// Ordered compaction of self-pointing vertices: count (keeps block offsets
// in S_TMP1), then write the list and/or the extremum -> rank map.
int64_t count_extrema(Ctx& c, int64_t n, const uint32_t* labels);
void write_extrema(Ctx& c, int64_t n, const uint32_t* labels, uint32_t* out, uint32_t* rank_map);
void compute_order(Ctx& c, int key_type, const void* values, int64_t n, int64_t* rank);
// One sweep over an active list; returns the unsettled count written to next.
int64_t compress_sweep_list(Ctx& c, uint32_t* desc, uint32_t* asc, const uint32_t* active, int64_t na,
                            uint32_t* next);

// combine.cu
// get_keys(R) returns the region-key buffer (or nullptr).
int64_t combine_ms(Ctx& c, int64_t n, const uint32_t* asc, const uint32_t* desc, uint32_t* ms,
                   const std::function<uint64_t*(int64_t)>& get_keys, const uint32_t* minima, int64_t n_min, const uint32_t* maxima,
                   int64_t n_max, const uint32_t* rank_min, const uint32_t* rank_max);

// marching.cu
int64_t index_separators(Ctx& c, const Grid& g, int label_type, const void* labels, uint8_t* codes);
void count_by_cell_ranges(Ctx& c, const Grid& g, int label_type, const void* labels, const int64_t* h_bounds,
                          int nranges, int64_t* h_counts);
// get_out(total) returns the record buffer (or nullptr to only count).
int64_t emit_separators(Ctx& c, const Grid& g, int label_type, const void* labels,
                        const std::function<void*(int64_t)>& get_out);
void materialize(Ctx& c, const Grid& g, const double* sp, const double* og, int label_type,
                 const void* tris, int64_t n, double* points, int64_t* regions, int64_t* cells);
void emit_boundaries(Ctx& c, const Grid& g, const double* sp, const double* og, int label_type,
                     const void* labels, int has_filter, int64_t filter, uint32_t* faces, void* tags,
                     int64_t* cells, double* points, int64_t* indices, int64_t* n_faces,
                     int64_t* n_points);

// scan.cu — device-wide exclusive scan of uint64 (in place allowed); returns total.
uint64_t exclusive_scan_u64(Ctx& c, uint64_t* data, int64_t n, bool want_total = true);
// stable LSD radix sort of (u64 key, u64 value) pairs; `bits` significant key bits.
void radix_sort_pairs(Ctx& c, uint64_t* keys, uint64_t* vals, int64_t n, int bits);

// fused.cu — the benchmarked single-GPU pipeline.
struct FusedOut {
  int64_t n_max, n_min, n_regions, n_tris;
  int sweeps;
  uint32_t *maxima, *minima;
  uint64_t* keys;
  plmss_tri* tris;
};
bool fused_supported(const Grid& g);
void fused_segment(Ctx& c, const Grid& g, const float* field, uint32_t* desc, uint32_t* asc, uint32_t* maxima_out,
                   uint32_t* minima_out, int64_t* n_max_out, int64_t* n_min_out, int32_t* sweeps_out);
FusedOut fused_pipeline(Ctx& c, const Grid& g, const float* field, uint32_t* desc, uint32_t* asc, uint32_t* ms);
// z-slab pipeline (multi-GPU), fused.cu; the stages of include/plmss_b200.h
void slab_segment(Ctx& c, const Grid& g, int64_t z0, int64_t z1, const float* field, plmss_slab_info* info);
void slab_resolve(Ctx& c, const uint32_t* G, int world, int rank, const int64_t* max_counts,
                  const int64_t* min_counts, const uint32_t* maxs_g, const uint32_t* mins_g, uint32_t* desc,
                  uint32_t* asc, uint32_t* ms, plmss_slab_info* info);
void slab_ids(Ctx& c, const uint64_t* keys_all, int64_t n_keys_all, plmss_slab_info* info);
void slab_emit(Ctx& c, uint32_t* ids, plmss_slab_info* info);

// synth.cu
// io.cu: callers either side of the path
int64_t weld_points(Ctx& c, double* d_points, int64_t n, int64_t* d_indices, int64_t m);
void read_volume(Ctx& c, const char* path, const int64_t dims[3], int dtype, int out_f64, void* d_out);
void write_labels(Ctx& c, const char* path, int label_type, const void* d_asc, const void* d_desc, int64_t n);
void write_surface_obj(Ctx& c, const char* path, const double* d_points, int64_t n_points, const int64_t* d_indices,
                       const int64_t* d_regions, int64_t n_prims, int verts_per_prim);
void write_separators_obj(Ctx& c, const char* path, const Grid& g, const double* sp, const double* og,
                          int label_type, const void* d_tris, int64_t n);
void materialize_chunks(Ctx& c, const Grid& g, const double* sp, const double* og, int label_type,
                        const void* d_tris, int64_t n, int64_t chunk, plmss_geometry_sink sink, void* user);
void synth(Ctx& c, const Grid& g, int kind, const double* h_gauss, int n_gauss, double noise_amp,
           uint64_t seed, int levels, float* field, int64_t z0, int64_t nz);

}  // namespace plmss_b200
