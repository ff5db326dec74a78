// extern "C" boundary of libplmss_b200.so (declared in include/plmss_b200.h).
// Converts internal exceptions to status codes + a thread-local message.
#include <string.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#include <string>
#include <thread>
#include <mutex>

#include "common.cuh"
#include "tet_tables.h"

using namespace plmss_b200;

unsigned long long plmss_b200::g_launches = 0;
thread_local cudaStream_t plmss_b200::g_trace_stream = nullptr;
namespace plmss_b200 {
namespace {
struct TraceRec {
  const char* name;
  cudaEvent_t ev;
};
thread_local std::vector<TraceRec> g_trace;
}  // namespace
void trace_launch(const char* name) {
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, g_trace_stream);
  g_trace.push_back({name, e});
}
// start: events from here on; stop: sync, print each launch's time since the
// previous event (launch + any gap before it) to stderr, release
void trace_begin(cudaStream_t s) {
  g_trace_stream = s;
  trace_launch("begin");
}
void trace_end() {
  if (!g_trace_stream) return;
  cudaStreamSynchronize(g_trace_stream);
  for (size_t i = 1; i < g_trace.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, g_trace[i - 1].ev, g_trace[i].ev);
    fprintf(stderr, "[ktrace] %-22s %8.4f ms\n", g_trace[i].name, ms);
  }
  for (auto& r : g_trace) cudaEventDestroy(r.ev);
  g_trace.clear();
  g_trace_stream = nullptr;
}
}  // namespace plmss_b200

struct plmss_ctx {
  Ctx c;
  // pipeline_host_batch: two internal contexts (own non-blocking streams)
  // that take alternate volumes on two host threads
  plmss_ctx* peer[2] = {nullptr, nullptr};
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PLMSS_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return PLMSS_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PLMSS_ERR_CUDA;
  }
}

Ctx& C(plmss_ctx* p) {
  if (!p) fail(PLMSS_ERR_INVALID_ARGUMENT, "null context");
  return p->c;
}

void set_device(Ctx& c) { CK(cudaSetDevice(c.device)); }

void finish_timing(Ctx& c, int marks) {
  if (!c.timing) return;
  c.sync();
  for (int i = 0; i + 1 < marks; ++i) CK(cudaEventElapsedTime(&c.stage_ms[i], c.ev[i], c.ev[i + 1]));
}

// Segmentation stages shared by plmss_b200_segment and the pipeline.
struct SegOut {
  int64_t n_max = 0, n_min = 0;
  int sweeps = 0;
};

SegOut run_segment(Ctx& c, const Grid& g, int key_type, const void* keys, int direction, uint32_t* desc,
                   uint32_t* asc, const std::function<uint32_t*(int64_t)>& get_maxima,
                   const std::function<uint32_t*(int64_t)>& get_minima, uint32_t* rank_max, uint32_t* rank_min) {
  SegOut o;
  const bool want_desc = direction != PLMSS_ASCENDING, want_asc = direction != PLMSS_DESCENDING;
  uint32_t* bad = static_cast<uint32_t*>(c.get(S_FLAGS, 64)) + 8;
  if (key_type != PLMSS_KEY_RANK) CK(cudaMemsetAsync(bad, 0xff, sizeof(uint32_t), c.stream));
  c.mark(0);
  seed_hops(c, g, key_type, keys, want_desc ? desc : nullptr, want_asc ? asc : nullptr,
            key_type != PLMSS_KEY_RANK ? bad : nullptr);
  c.mark(1);
  if (key_type != PLMSS_KEY_RANK) {
    CK(cudaMemcpyAsync(c.h_pinned + 2, bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const uint32_t b = *reinterpret_cast<uint32_t*>(c.h_pinned + 2);
    if (b != 0xffffffffu) fail(PLMSS_ERR_INVALID_ARGUMENT, "non-finite scalar value at vertex " + std::to_string(b));
  }
  o.sweeps = compress(c, g.n, want_desc ? desc : nullptr, want_asc ? asc : nullptr);
  c.mark(2);
  if (want_desc) {
    o.n_max = count_extrema(c, g.n, desc);
    write_extrema(c, g.n, desc, get_maxima(o.n_max), rank_max);
  }
  if (want_asc) {
    o.n_min = count_extrema(c, g.n, asc);
    write_extrema(c, g.n, asc, get_minima(o.n_min), rank_min);
  }
  c.mark(3);
  return o;
}

}  // namespace

extern "C" {

const char* plmss_b200_last_error(void) { return g_err.c_str(); }

const char* plmss_b200_version(void) { return "plmss_b200 0.1 (sm_100a)"; }

unsigned long long plmss_b200_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

void plmss_b200_tet_table(uint32_t rows[52], uint16_t cases[32]) {
  memcpy(rows, kTetRowsPacked, sizeof(kTetRowsPacked));
  memcpy(cases, kTetCasePacked, sizeof(kTetCasePacked));
}

int plmss_b200_ctx_create(int device, void* stream, plmss_ctx** out) {
  return guarded([&] {
    if (!out) fail(PLMSS_ERR_INVALID_ARGUMENT, "null out");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) fail(PLMSS_ERR_INVALID_ARGUMENT, "no such CUDA device");
    auto* p = new plmss_ctx();
    Ctx& c = p->c;
    c.device = device;
    try {
      CK(cudaSetDevice(device));
      if (stream) {
        c.stream = static_cast<cudaStream_t>(stream);
      } else {
        CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        c.own_stream = true;
      }
      CK(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming));
      CK(cudaMallocHost(&c.h_pinned, 64 * sizeof(uint64_t)));
      for (auto& e : c.ev) CK(cudaEventCreate(&e));
      CK(cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, device));
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

void plmss_b200_ctx_destroy(plmss_ctx* p) {
  if (p)
    for (auto& q : p->peer)
      if (q) {
        plmss_b200_ctx_destroy(q);
        q = nullptr;
      }
  if (!p) return;
  Ctx& c = p->c;
  cudaSetDevice(c.device);
  cudaStreamSynchronize(c.stream);
  for (auto& b : c.buf)
    if (b) cudaFreeAsync(b, c.stream);
  cudaStreamSynchronize(c.stream);
  for (auto& e : c.ev)
    if (e) cudaEventDestroy(e);
  if (c.side) {
    cudaStreamSynchronize(c.side);
    cudaStreamDestroy(c.side);
  }
  if (c.join) cudaEventDestroy(c.join);
  for (auto& e : c.slab_ev) cudaEventDestroy(e);
  if (c.h_pinned) cudaFreeHost(c.h_pinned);
  if (c.h_stage) cudaFreeHost(c.h_stage);
  if (c.own_stream) cudaStreamDestroy(c.stream);
  delete p;
}

size_t plmss_b200_ctx_scratch_bytes(const plmss_ctx* p) {
  if (!p) return 0;
  size_t s = 0;
  for (size_t x : p->c.cap) s += x;
  return s;
}

int plmss_b200_ctx_release(plmss_ctx* p) {
  return guarded([&] {
    if (p)
      for (auto* q : p->peer)
        if (q) {
          const int s2 = plmss_b200_ctx_release(q);
          if (s2) fail(s2, plmss_b200_last_error());
        }
    Ctx& c = C(p);
    set_device(c);
    c.sync();
    for (int s = 0; s < S_COUNT; ++s) {
      if (c.buf[s]) CK(cudaFreeAsync(c.buf[s], c.stream));
      c.buf[s] = nullptr;
      c.cap[s] = 0;
    }
    c.sync();
    c.result = plmss_result{};
    c.slab = SlabState{};
    // return the freed blocks of the context's pool to the device
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess) CK(cudaMemPoolTrimTo(pool, 0));
  });
}

int plmss_b200_ctx_set_timing(plmss_ctx* p, int enable) {
  return guarded([&] { C(p).timing = enable != 0; });
}

int plmss_b200_ctx_stage_ms(const plmss_ctx* p, float out[8]) {
  return guarded([&] {
    if (!p) fail(PLMSS_ERR_INVALID_ARGUMENT, "null context");
    memcpy(out, p->c.stage_ms, sizeof(p->c.stage_ms));
  });
}

int plmss_b200_ctx_stats(const plmss_ctx* p, int64_t out[8]) {
  return guarded([&] {
    if (!p) fail(PLMSS_ERR_INVALID_ARGUMENT, "null context");
    memcpy(out, p->c.stats, sizeof(p->c.stats));
  });
}

int plmss_b200_compute_order(plmss_ctx* p, int key_type, const void* d_values, int64_t n, int64_t* d_rank) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (n < 0) fail(PLMSS_ERR_INVALID_ARGUMENT, "negative size");
    compute_order(c, key_type, d_values, n, d_rank);
    c.sync();
  });
}

int plmss_b200_seed_hops(plmss_ctx* p, const int64_t dims[3], int key_type, const void* d_keys, uint32_t* d_desc,
                         uint32_t* d_asc) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    seed_hops(c, g, key_type, d_keys, d_desc, d_asc, nullptr);
    c.sync();
  });
}

int plmss_b200_segment_slab(plmss_ctx* p, const int64_t dims[3], int key_type, const void* d_keys, int halo_lo,
                            int halo_hi, uint32_t* d_desc, uint32_t* d_asc, int32_t* sweeps) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    if (!d_desc || !d_asc) fail(PLMSS_ERR_INVALID_ARGUMENT, "d_desc and d_asc required");
    uint32_t* bad = static_cast<uint32_t*>(c.get(S_FLAGS, 64)) + 8;
    if (key_type != PLMSS_KEY_RANK) CK(cudaMemsetAsync(bad, 0xff, sizeof(uint32_t), c.stream));
    seed_hops(c, g, key_type, d_keys, d_desc, d_asc, key_type != PLMSS_KEY_RANK ? bad : nullptr);
    terminal_layers(c, g, halo_lo != 0, halo_hi != 0, d_desc, d_asc);
    const int s = compress(c, g.n, d_desc, d_asc);
    if (key_type != PLMSS_KEY_RANK) {
      CK(cudaMemcpyAsync(c.h_pinned + 2, bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, c.stream));
      c.sync();
      const uint32_t b = *reinterpret_cast<uint32_t*>(c.h_pinned + 2);
      if (b != 0xffffffffu) fail(PLMSS_ERR_INVALID_ARGUMENT, "non-finite scalar value at vertex " + std::to_string(b));
    }
    c.sync();
    if (sweeps) *sweeps = s;
  });
}

int plmss_b200_compress_sweep(plmss_ctx* p, uint32_t* d_desc, uint32_t* d_asc, const uint32_t* d_active,
                              int64_t n_active, uint32_t* d_next, int64_t* n_next) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (!d_desc || (n_active > 0 && (!d_active || !d_next))) fail(PLMSS_ERR_INVALID_ARGUMENT, "null argument");
    const int64_t k = compress_sweep_list(c, d_desc, d_asc, d_active, n_active, d_next);
    c.sync();
    if (n_next) *n_next = k;
  });
}

// OrderField ranks -> float32 keys with the same order (bit patterns of
// non-negative floats order like the integers); flags a rank outside [0, 2^30).
__global__ void k_rank_keys(const int64_t* __restrict__ rank, int64_t n, float* __restrict__ out,
                            int* __restrict__ bad) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = rank[i];
  if (r < 0 || r >= (int64_t(1) << 30)) *bad = 1;
  out[i] = __uint_as_float(uint32_t(r) & 0x3fffffffu);
}

int plmss_b200_segment(plmss_ctx* p, const int64_t dims[3], int key_type, const void* d_keys, int direction,
                       uint32_t* d_desc, uint32_t* d_asc, uint32_t* d_maxima, uint32_t* d_minima,
                       int64_t* n_maxima, int64_t* n_minima, int32_t* sweeps) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    if (direction < 0 || direction > 2) fail(PLMSS_ERR_INVALID_ARGUMENT, "bad direction");
    if (direction != PLMSS_ASCENDING && !d_desc) fail(PLMSS_ERR_INVALID_ARGUMENT, "d_desc required");
    if (direction != PLMSS_DESCENDING && !d_asc) fail(PLMSS_ERR_INVALID_ARGUMENT, "d_asc required");
    // The fused passes (fused.cu fused_segment) for float32 values and
    // OrderField ranks on grids inside the fused envelope; float64 values and
    // PLMSS_OPT_PIPELINE_PATH 1 take the staged kernels.
    if (c.pipeline_path == 0 && fused_supported(g) && (key_type == PLMSS_KEY_F32 || key_type == PLMSS_KEY_RANK)) {
      const float* f = static_cast<const float*>(d_keys);
      bool ok = true;
      if (key_type == PLMSS_KEY_RANK) {
        float* fk = c.get_t<float>(S_FIELD, g.n);
        int* bad = reinterpret_cast<int*>(static_cast<char*>(c.get(S_FLAGS, 1024)) + 320);
        CK(cudaMemsetAsync(bad, 0, 4, c.stream));
        k_rank_keys<<<blocks_for(g.n, 256), 256, 0, c.stream>>>(static_cast<const int64_t*>(d_keys), g.n, fk, bad);
        CK_LAUNCH("k_rank_keys");
        CK(cudaMemcpyAsync(c.h_pinned + 3, bad, 4, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        ok = *reinterpret_cast<int*>(c.h_pinned + 3) == 0;
        f = fk;
      }
      if (ok) {
        uint32_t* dd = d_desc ? d_desc : c.get_t<uint32_t>(S_DESC, g.n);
        uint32_t* da = d_asc ? d_asc : c.get_t<uint32_t>(S_ASC, g.n);
        int64_t nmx = 0, nmn = 0;
        int32_t sw = 0;
        fused_segment(c, g, f, dd, da, direction != PLMSS_ASCENDING ? d_maxima : nullptr,
                      direction != PLMSS_DESCENDING ? d_minima : nullptr, &nmx, &nmn, &sw);
        if (n_maxima) *n_maxima = direction != PLMSS_ASCENDING ? nmx : 0;
        if (n_minima) *n_minima = direction != PLMSS_DESCENDING ? nmn : 0;
        if (sweeps) *sweeps = sw;
        return;
      }
    }
    SegOut o = run_segment(
        c, g, key_type, d_keys, direction, d_desc, d_asc, [&](int64_t) { return d_maxima; },
        [&](int64_t) { return d_minima; }, nullptr, nullptr);
    c.sync();
    if (n_maxima) *n_maxima = o.n_max;
    if (n_minima) *n_minima = o.n_min;
    if (sweeps) *sweeps = o.sweeps;
  });
}

int plmss_b200_combine_ms(plmss_ctx* p, int64_t n, const uint32_t* d_asc, const uint32_t* d_desc, uint32_t* d_ms,
                          uint64_t* d_region_keys, int64_t* n_regions) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (!d_asc || !d_desc) fail(PLMSS_ERR_INVALID_ARGUMENT, "combine_ms needs both ascending and descending labels");
    if (n <= 0 || n >= (int64_t(1) << 32) - 1) fail(PLMSS_ERR_INVALID_ARGUMENT, "bad vertex count");
    // Extremum lists and rank maps from the (converged) label arrays.
    uint32_t* rmax = c.get_t<uint32_t>(S_RANK_MAX, n);
    uint32_t* rmin = c.get_t<uint32_t>(S_RANK_MIN, n);
    const int64_t nmax = count_extrema(c, n, d_desc);
    uint32_t* maxima = c.get_t<uint32_t>(S_MAXIMA, nmax);
    write_extrema(c, n, d_desc, maxima, rmax);
    const int64_t nmin = count_extrema(c, n, d_asc);
    uint32_t* minima = c.get_t<uint32_t>(S_MINIMA, nmin);
    write_extrema(c, n, d_asc, minima, rmin);
    const int64_t R = combine_ms(
        c, n, d_asc, d_desc, d_ms, [&](int64_t) { return d_region_keys; }, minima, nmin, maxima, nmax, rmin, rmax);
    c.sync();
    if (n_regions) *n_regions = R;
  });
}

int plmss_b200_index_separators(plmss_ctx* p, const int64_t dims[3], int label_type, const void* d_labels,
                                uint8_t* d_codes, int64_t* total) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    const int64_t t = index_separators(c, g, label_type, d_labels, d_codes);
    c.sync();
    if (total) *total = t;
  });
}

int plmss_b200_count_by_cell_ranges(plmss_ctx* p, const int64_t dims[3], int label_type, const void* d_labels,
                                    const int64_t* h_bounds, int nranges, int64_t* h_counts) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    if (!h_bounds || !h_counts) fail(PLMSS_ERR_INVALID_ARGUMENT, "null bounds/counts");
    count_by_cell_ranges(c, g, label_type, d_labels, h_bounds, nranges, h_counts);
  });
}

int plmss_b200_emit_separators(plmss_ctx* p, const int64_t dims[3], int label_type, const void* d_labels,
                               void* d_out, int64_t capacity, int64_t* total) {
  int64_t t = 0;
  int st = guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    t = emit_separators(c, g, label_type, d_labels,
                        [&](int64_t tot) -> void* { return tot <= capacity ? d_out : nullptr; });
    c.sync();
    if (total) *total = t;
    if (t > capacity)
      fail(PLMSS_ERR_LOGIC, "geometry phase exceeds indexed primitive count (capacity " + std::to_string(capacity) +
                                ", need " + std::to_string(t) + ")");
  });
  return st;
}

int plmss_b200_materialize_separators(plmss_ctx* p, const int64_t dims[3], const double spacing[3],
                                      const double origin[3], int label_type, const void* d_tris, int64_t n,
                                      double* d_points, int64_t* d_regions, int64_t* d_source_cells) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    materialize(c, g, spacing, origin, label_type, d_tris, n, d_points, d_regions, d_source_cells);
    c.sync();
  });
}

int plmss_b200_emit_boundaries(plmss_ctx* p, const int64_t dims[3], const double spacing[3], const double origin[3],
                               int label_type, const void* d_labels, int has_filter, int64_t filter,
                               uint32_t* d_faces, void* d_tags, int64_t* d_cells, double* d_points,
                               int64_t* d_indices, int64_t* n_faces, int64_t* n_points) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    int64_t nf = 0, np = 0;
    if (label_type == 0 && has_filter && (filter < 0 || filter > int64_t(0xffffffffu))) {
      // No uint32 label can carry this tag: empty result.
    } else {
      emit_boundaries(c, g, spacing, origin, label_type, d_labels, has_filter, filter, d_faces, d_tags, d_cells,
                      d_points, d_indices, &nf, &np);
      c.sync();
    }
    if (n_faces) *n_faces = nf;
    if (n_points) *n_points = np;
  });
}

int plmss_b200_pipeline(plmss_ctx* p, const int64_t dims[3], const float* d_field) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    uint32_t* desc = c.get_t<uint32_t>(S_DESC, g.n);
    uint32_t* asc = c.get_t<uint32_t>(S_ASC, g.n);
    uint32_t* ms = c.get_t<uint32_t>(S_MS, g.n);
    if (c.pipeline_path == 0 && fused_supported(g)) {
      static const bool ktrace = getenv("PLMSS_KTRACE") != nullptr;
      if (ktrace) trace_begin(c.stream);
      const FusedOut fo = fused_pipeline(c, g, d_field, desc, asc, ms);
      if (ktrace) trace_end();
      c.sync();
      finish_timing(c, 6);
      plmss_result& r = c.result;
      r.d_desc = desc;
      r.d_asc = asc;
      r.d_ms = ms;
      r.d_maxima = fo.maxima;
      r.d_minima = fo.minima;
      r.d_region_keys = fo.keys;
      r.d_tris = fo.tris;
      r.n_vertices = g.n;
      r.n_maxima = fo.n_max;
      r.n_minima = fo.n_min;
      r.n_regions = fo.n_regions;
      r.n_tris = fo.n_tris;
      r.sweeps = fo.sweeps;
      return;
    }
    uint32_t* rmax = c.get_t<uint32_t>(S_RANK_MAX, g.n);
    uint32_t* rmin = c.get_t<uint32_t>(S_RANK_MIN, g.n);
    uint32_t *maxima = nullptr, *minima = nullptr;
    SegOut o = run_segment(
        c, g, PLMSS_KEY_F32, d_field, PLMSS_BOTH, desc, asc,
        [&](int64_t k) { return maxima = c.get_t<uint32_t>(S_MAXIMA, k); },
        [&](int64_t k) { return minima = c.get_t<uint32_t>(S_MINIMA, k); }, rmax, rmin);
    uint64_t* keys = nullptr;
    const int64_t R = combine_ms(
        c, g.n, asc, desc, ms, [&](int64_t r) { return keys = c.get_t<uint64_t>(S_KEYS, r); }, minima, o.n_min,
        maxima, o.n_max, rmin, rmax);
    c.mark(4);
    plmss_tri* tris = nullptr;
    const int64_t T = emit_separators(c, g, 0, ms, [&](int64_t t) -> void* {
      return tris = c.get_t<plmss_tri>(S_TRIS, t);
    });
    c.mark(5);
    c.sync();
    finish_timing(c, 6);
    plmss_result& r = c.result;
    r.d_desc = desc;
    r.d_asc = asc;
    r.d_ms = ms;
    r.d_maxima = maxima;
    r.d_minima = minima;
    r.d_region_keys = keys;
    r.d_tris = tris;
    r.n_vertices = g.n;
    r.n_maxima = o.n_max;
    r.n_minima = o.n_min;
    r.n_regions = R;
    r.n_tris = T;
    r.sweeps = o.sweeps;
  });
}

int plmss_b200_copy(plmss_ctx* p, void* dst, const void* d_src, int64_t bytes, int to_host) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (bytes < 0) fail(PLMSS_ERR_INVALID_ARGUMENT, "negative size");
    if (bytes == 0) return;
    if (!dst || !d_src) fail(PLMSS_ERR_INVALID_ARGUMENT, "null pointer");
    CK(cudaMemcpyAsync(dst, d_src, size_t(bytes), to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                       c.stream));
    c.sync();
  });
}

int plmss_b200_ctx_set_option(plmss_ctx* p, int option, int64_t value) {
  return guarded([&] {
    Ctx& c = C(p);
    if (option == PLMSS_OPT_COMBINE_PATH) {
      if (value < 0 || value > 2) fail(PLMSS_ERR_INVALID_ARGUMENT, "combine path must be 0, 1 or 2");
      c.combine_path = int(value);
      return;
    }
    if (option == PLMSS_OPT_SPECULATIVE_SWEEPS) {
      if (value < 0 || value > 64) fail(PLMSS_ERR_INVALID_ARGUMENT, "speculative sweeps must be in [0, 64]");
      c.spec_sweeps = int(value);
      return;
    }
    if (option == PLMSS_OPT_TMA) {
      c.use_tma = value != 0;
      return;
    }
    if (option == PLMSS_OPT_PASS_A_SPLIT) {
      c.pass_a_split = value != 0;
      return;
    }
    if (option == PLMSS_OPT_HOP_CUBE) {
      c.hop_cube = value != 0;
      return;
    }
    if (option == PLMSS_OPT_IDS_IN_COUNT) {
      if (value < 0 || value > 2) fail(PLMSS_ERR_INVALID_ARGUMENT, "ids mode must be 0, 1 or 2");
      c.ids_mode = int(value);
      return;
    }
    if (option == PLMSS_OPT_PIPELINE_PATH) {
      if (value < 0 || value > 1) fail(PLMSS_ERR_INVALID_ARGUMENT, "pipeline path must be 0 or 1");
      c.pipeline_path = int(value);
      return;
    }
    fail(PLMSS_ERR_INVALID_ARGUMENT, "unknown option");
  });
}

int plmss_b200_result(const plmss_ctx* p, plmss_result* out) {
  return guarded([&] {
    if (!p || !out) fail(PLMSS_ERR_INVALID_ARGUMENT, "null argument");
    *out = p->c.result;
  });
}

int plmss_b200_pipeline_host(plmss_ctx* p, const int64_t dims[3], const float* h_field, uint32_t* h_desc,
                             uint32_t* h_asc, uint32_t* h_ms, uint32_t* h_maxima, uint32_t* h_minima,
                             uint64_t* h_region_keys, plmss_tri* h_tris, int64_t tri_capacity, plmss_result* out) {
  int st = guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    if (!h_field) fail(PLMSS_ERR_INVALID_ARGUMENT, "null field");
    float* f = c.get_t<float>(S_FIELD, g.n);
    CK(cudaMemcpyAsync(f, h_field, g.n * sizeof(float), cudaMemcpyHostToDevice, c.stream));
  });
  if (st) return st;
  st = plmss_b200_pipeline(p, dims, static_cast<const float*>(p->c.buf[S_FIELD]));
  if (st) return st;
  return guarded([&] {
    Ctx& c = p->c;
    const plmss_result& r = c.result;
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
    };
    d2h(h_desc, r.d_desc, r.n_vertices * 4);
    d2h(h_asc, r.d_asc, r.n_vertices * 4);
    d2h(h_ms, r.d_ms, r.n_vertices * 4);
    d2h(h_maxima, r.d_maxima, r.n_maxima * 4);
    d2h(h_minima, r.d_minima, r.n_minima * 4);
    d2h(h_region_keys, r.d_region_keys, r.n_regions * 8);
    if (h_tris && r.n_tris <= tri_capacity) d2h(h_tris, r.d_tris, r.n_tris * sizeof(plmss_tri));
    c.sync();
    if (out) *out = r;
    if (h_tris && r.n_tris > tri_capacity)
      fail(PLMSS_ERR_LOGIC, "separator records exceed the host capacity (" + std::to_string(r.n_tris) + ")");
  });
}

int plmss_b200_pipeline_host_batch(plmss_ctx* p, const int64_t dims[3], plmss_host_volume* vols, int64_t n) {
  int st = guarded([&] {
    if (!p) fail(PLMSS_ERR_INVALID_ARGUMENT, "null context");
    if (n < 0 || (n > 0 && !vols)) fail(PLMSS_ERR_INVALID_ARGUMENT, "bad volume list");
    for (auto& q : p->peer)
      if (!q) {
        const int s2 = plmss_b200_ctx_create(p->c.device, nullptr, &q);
        if (s2) fail(s2, "peer context: " + std::string(plmss_b200_last_error()));
      }
    for (auto* q : p->peer) {  // the caller's options
      q->c.combine_path = p->c.combine_path;
      q->c.pipeline_path = p->c.pipeline_path;
      q->c.use_tma = p->c.use_tma;
      q->c.spec_sweeps = p->c.spec_sweeps;
      q->c.pass_a_split = p->c.pass_a_split;
      q->c.hop_cube = p->c.hop_cube;
      q->c.ids_mode = p->c.ids_mode;
    }
  });
  if (st) return st;
  int first_err = 0;
  std::string first_msg;
  std::mutex mu;
  auto worker = [&](int k) {
    for (int64_t i = k; i < n; i += 2) {
      plmss_host_volume& v = vols[i];
      v.status = plmss_b200_pipeline_host(p->peer[k], dims, v.h_field, v.h_desc, v.h_asc, v.h_ms, v.h_maxima,
                                          v.h_minima, v.h_region_keys, v.h_tris, v.tri_capacity, &v.result);
      if (v.status) {
        std::lock_guard<std::mutex> lock(mu);
        if (!first_err) {
          first_err = v.status;
          first_msg = plmss_b200_last_error();
        }
        return;
      }
    }
  };
  std::thread t1(worker, 1);
  worker(0);
  t1.join();
  if (first_err) g_err = first_msg;
  return first_err;
}

int plmss_b200_synth(plmss_ctx* p, const int64_t dims[3], int kind, const double* h_gaussians, int n_gauss,
                     double noise_amp, uint64_t seed, int levels, float* d_field) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    synth(c, g, kind, h_gaussians, n_gauss, noise_amp, seed, levels, d_field, 0, g.Z);
  });
}

int plmss_b200_synth_layers(plmss_ctx* p, const int64_t dims[3], int kind, const double* h_gaussians, int n_gauss,
                            double noise_amp, uint64_t seed, int64_t z0, int64_t nz, float* d_field) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    const Grid g = make_grid(dims);
    synth(c, g, kind, h_gaussians, n_gauss, noise_amp, seed, 0, d_field, z0, nz);
  });
}

int plmss_b200_materialize_separators_chunked(plmss_ctx* p, const int64_t dims[3], const double spacing[3],
                                              const double origin[3], int label_type, const void* d_tris,
                                              int64_t n, int64_t chunk, plmss_geometry_sink sink, void* user) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (label_type != 0 && label_type != 1) fail(PLMSS_ERR_INVALID_ARGUMENT, "label_type must be 0 or 1");
    materialize_chunks(c, make_grid(dims), spacing, origin, label_type, d_tris, n, chunk, sink, user);
  });
}

int plmss_b200_write_separators_obj(plmss_ctx* p, const char* path, const int64_t dims[3], const double spacing[3],
                                    const double origin[3], int label_type, const void* d_tris, int64_t n) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (label_type != 0 && label_type != 1) fail(PLMSS_ERR_INVALID_ARGUMENT, "label_type must be 0 or 1");
    write_separators_obj(c, path, make_grid(dims), spacing, origin, label_type, d_tris, n);
  });
}

// ---- z-slab pipeline (fused.cu slab_*) ----------------------------------
int plmss_b200_slab_segment(plmss_ctx* p, const int64_t dims[3], int64_t z0, int64_t z1, const float* d_field,
                            plmss_slab_info* info) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (!d_field) fail(PLMSS_ERR_INVALID_ARGUMENT, "field is null");
    slab_segment(c, make_grid(dims), z0, z1, d_field, info);
  });
}

int plmss_b200_slab_resolve(plmss_ctx* p, const uint32_t* d_boundary_all, int world, int rank,
                            const int64_t* h_max_counts, const int64_t* h_min_counts, const uint32_t* d_maxima_all,
                            const uint32_t* d_minima_all, uint32_t* d_desc, uint32_t* d_asc, uint32_t* d_ms,
                            plmss_slab_info* info) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    slab_resolve(c, d_boundary_all, world, rank, h_max_counts, h_min_counts, d_maxima_all, d_minima_all, d_desc,
                 d_asc, d_ms, info);
  });
}

int plmss_b200_slab_ids(plmss_ctx* p, const uint64_t* d_keys_all, int64_t n_keys_all, plmss_slab_info* info) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    slab_ids(c, d_keys_all, n_keys_all, info);
  });
}

int plmss_b200_slab_emit(plmss_ctx* p, uint32_t* d_ids, plmss_slab_info* info) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    slab_emit(c, d_ids, info);
  });
}

int plmss_b200_weld_points(plmss_ctx* p, double* d_points, int64_t n_points, int64_t* d_indices, int64_t n_indices,
                           int64_t* n_unique) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if ((n_points && !d_points) || (n_indices && !d_indices)) fail(PLMSS_ERR_INVALID_ARGUMENT, "null array");
    const int64_t u = weld_points(c, d_points, n_points, d_indices, n_indices);
    if (n_unique) *n_unique = u;
  });
}

int plmss_b200_read_volume(plmss_ctx* p, const char* path, const int64_t dims[3], int dtype, int out_f64,
                           void* d_out) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (!dims || !d_out) fail(PLMSS_ERR_INVALID_ARGUMENT, "null dims or output");
    read_volume(c, path, dims, dtype, out_f64, d_out);
  });
}

int plmss_b200_write_labels(plmss_ctx* p, const char* path, int label_type, const void* d_asc, const void* d_desc,
                            int64_t n) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    if (label_type != 0 && label_type != 1) fail(PLMSS_ERR_INVALID_ARGUMENT, "label_type must be 0 or 1");
    write_labels(c, path, label_type, d_asc, d_desc, n);
  });
}

int plmss_b200_write_surface_obj(plmss_ctx* p, const char* path, const double* d_points, int64_t n_points,
                                 const int64_t* d_indices, const int64_t* d_regions, int64_t n_prims,
                                 int verts_per_prim) {
  return guarded([&] {
    Ctx& c = C(p);
    set_device(c);
    write_surface_obj(c, path, d_points, n_points, d_indices, d_regions, n_prims, verts_per_prim);
  });
}

}  // extern "C"
