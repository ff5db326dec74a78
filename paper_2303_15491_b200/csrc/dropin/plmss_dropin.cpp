// C++ drop-in for the reference hot path: the plmss:: entry points declared
// in the reference headers (proj/include/plmss/{orderfield,segmentation,
// marching}.hpp), implemented on the B200 through the C-ABI of
// include/plmss_b200.h. Link this library instead of the reference's
// orderfield.cpp / segmentation.cpp / marching.cpp / marching_tables.cpp;
// complex.cpp, io.cpp, bench.cpp and synth.cpp stay the reference's own
// (INTEGRATION.md). Scope: implicit 3-D grids; anything else throws
// std::invalid_argument (there is no CPU fallback). Status codes map back
// to the reference exception types with the reference messages.
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "plmss/marching.hpp"
#include "plmss/orderfield.hpp"
#include "plmss/parallel.hpp"
#include "plmss/segmentation.hpp"
#include "plmss_b200.h"

namespace plmss {
namespace {

[[noreturn]] void rethrow(int st) {
  const std::string msg = plmss_b200_last_error();
  switch (st) {
    case PLMSS_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case PLMSS_ERR_LOGIC:
      throw std::logic_error(msg);
    case PLMSS_ERR_OUT_OF_RANGE:
      throw std::out_of_range(msg);
    default:
      throw std::runtime_error("plmss B200: " + msg);
  }
}

void check(int st) {
  if (st != PLMSS_OK) rethrow(st);
}

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("plmss B200: ") + what + ": " + cudaGetErrorString(e));
}

// One context per host thread keeps the functions reentrant.
plmss_ctx* ctx() {
  struct Holder {
    plmss_ctx* c = nullptr;
    ~Holder() {
      if (c) plmss_b200_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c) check(plmss_b200_ctx_create(0, nullptr, &h.c));
  return h.c;
}

// Device buffer owned for the duration of one call.
template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) {
    if (n) cuda(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  void up(const T* h, size_t n);
  void down(T* h, size_t n) const;
};

std::array<int64_t, 3> grid_of(const SimplicialComplex3& complex) {
  if (!complex.is_implicit_grid() || complex.dimension() != 3)
    throw std::invalid_argument(
        "the plmss B200 drop-in handles implicit 3-D grids only (explicit meshes and 2-D grids are out of scope)");
  const auto& d = complex.grid_dims();
  return {d[0], d[1], d[2]};
}

// ---- host <-> device transfers through pinned staging, host side on threads
// (the reference containers are pageable std::vector / Eigen storage: a plain
// cudaMemcpy from them runs at pageable speed on one thread).
constexpr size_t kStage = size_t(64) << 20;

unsigned host_threads() { return std::max(1u, std::min(16u, std::thread::hardware_concurrency())); }

template <class F>
void parallel_for(int64_t n, F&& f) {  // f(begin, end)
  const unsigned nt = n < (int64_t(1) << 16) ? 1u : host_threads();
  if (nt == 1) {
    f(int64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t b = std::min(n, int64_t(t) * per), e = std::min(n, b + per);
    if (b < e) th.emplace_back([&f, b, e] { f(b, e); });
  }
  for (auto& x : th) x.join();
}

// ---- large host outputs. The reference containers are value-initialised by
// resize() on one thread; at geometry sizes (cfg2: 12 GB of mesh) that is
// page-fault bound, the kernel zeroing every 4 KB page on first touch. The
// storage is reserved first, its pages faulted in on all host threads (2 MB
// pages where the kernel allows them), and only then sized.
void prefault(void* p, size_t bytes) {
  if (!p || bytes < (size_t(64) << 20)) return;
  constexpr uintptr_t kHuge = uintptr_t(2) << 20;
  const uintptr_t b = reinterpret_cast<uintptr_t>(p), e = b + bytes;
  const uintptr_t hb = (b + kHuge - 1) & ~(kHuge - 1), he = e & ~(kHuge - 1);
  if (he > hb) madvise(reinterpret_cast<void*>(hb), he - hb, MADV_HUGEPAGE);  // advice only
  unsigned char* c = static_cast<unsigned char*>(p);
  parallel_for(int64_t((bytes + 4095) / 4096), [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) c[std::min(size_t(i) * 4096, bytes - 1)] = 0;
  });
}

template <class T>
void resize_out(std::vector<T>& v, size_t n) {
  static_assert(std::is_trivially_copyable_v<T>, "raw storage prefault");
  if (v.capacity() < n) {
    v.reserve(n);
    prefault(v.data() + v.size(), (n - v.size()) * sizeof(T));
  }
  v.resize(n);
}

struct Stage {
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  Stage() {
    for (auto& b : buf) cuda(cudaMallocHost(reinterpret_cast<void**>(&b), kStage), "cudaMallocHost");
    cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : ev) cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  }
};

Stage& stage() {
  thread_local Stage s;  // one per host thread, like the contexts
  return s;
}

// Device -> host: chunk k is copied into pinned buffer k % 2 while the host
// threads convert chunk k - 1 out of the other one. conv(dst_index0,
// staged source, count) writes count source elements.
template <class S, class Conv>
void down_conv(const S* d_src, int64_t n, Conv&& conv) {
  if (n <= 0) return;
  Stage& g = stage();
  cuda(cudaDeviceSynchronize(), "sync");
  const int64_t per = int64_t(kStage / sizeof(S));
  const int64_t nch = (n + per - 1) / per;
  for (int64_t k = 0; k <= nch; ++k) {
    if (k < nch) {
      const int64_t i0 = k * per, cnt = std::min(per, n - i0);
      cuda(cudaMemcpyAsync(g.buf[k & 1], d_src + i0, size_t(cnt) * sizeof(S), cudaMemcpyDeviceToHost, g.st), "D2H");
      cuda(cudaEventRecord(g.ev[k & 1], g.st), "event");
    }
    if (k >= 1) {
      const int64_t j = k - 1, i0 = j * per, cnt = std::min(per, n - i0);
      cuda(cudaEventSynchronize(g.ev[j & 1]), "event sync");
      const S* src = reinterpret_cast<const S*>(g.buf[j & 1]);
      parallel_for(cnt, [&](int64_t b, int64_t e) { conv(i0 + b, src + b, e - b); });
    }
  }
}

// Host -> device: the host threads fill pinned buffer k % 2 (conversion
// included) while chunk k - 1 is in flight. fill(dst staged, src_index0, count).
template <class D, class Fill>
void up_conv(D* d_dst, int64_t n, Fill&& fill) {
  if (n <= 0) return;
  Stage& g = stage();
  const int64_t per = int64_t(kStage / sizeof(D));
  const int64_t nch = (n + per - 1) / per;
  for (int64_t k = 0; k < nch; ++k) {
    const int64_t i0 = k * per, cnt = std::min(per, n - i0);
    if (k >= 2) cuda(cudaEventSynchronize(g.ev[k & 1]), "event sync");  // buffer k % 2 free again
    D* dst = reinterpret_cast<D*>(g.buf[k & 1]);
    parallel_for(cnt, [&](int64_t b, int64_t e) { fill(dst + b, i0 + b, e - b); });
    cuda(cudaMemcpyAsync(d_dst + i0, dst, size_t(cnt) * sizeof(D), cudaMemcpyHostToDevice, g.st), "H2D");
    cuda(cudaEventRecord(g.ev[k & 1], g.st), "event");
  }
  cuda(cudaStreamSynchronize(g.st), "sync");
}

template <class T>
void down_copy(T* h_dst, const T* d_src, int64_t n) {
  down_conv(d_src, n, [&](int64_t i0, const T* s, int64_t c) { std::memcpy(h_dst + i0, s, size_t(c) * sizeof(T)); });
}
template <class T>
void up_copy(T* d_dst, const T* h_src, int64_t n) {
  up_conv(d_dst, n, [&](T* d, int64_t i0, int64_t c) { std::memcpy(d, h_src + i0, size_t(c) * sizeof(T)); });
}
// labels: device uint32 <-> host int64
void down_widen(int64_t* h_dst, const uint32_t* d_src, int64_t n) {
  down_conv(d_src, n, [&](int64_t i0, const uint32_t* s, int64_t c) {
    for (int64_t i = 0; i < c; ++i) h_dst[i0 + i] = s[i];
  });
}
void up_narrow(uint32_t* d_dst, const int64_t* h_src, int64_t n) {
  up_conv(d_dst, n, [&](uint32_t* d, int64_t i0, int64_t c) {
    for (int64_t i = 0; i < c; ++i) d[i] = static_cast<uint32_t>(h_src[i0 + i]);
  });
}

template <class T>
void DevBuf<T>::up(const T* h, size_t n) {
  if (n < (size_t(1) << 16))
    cuda(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  else
    up_copy(p, h, int64_t(n));
}
template <class T>
void DevBuf<T>::down(T* h, size_t n) const {
  if (n < (size_t(1) << 16))
    cuda(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  else
    down_copy(h, p, int64_t(n));
}

std::vector<uint32_t> narrow(std::span<const int64_t> v) {
  std::vector<uint32_t> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = static_cast<uint32_t>(v[i]);
  return out;
}

std::vector<int64_t> widen(const std::vector<uint32_t>& v) { return std::vector<int64_t>(v.begin(), v.end()); }

void check_labels(const SimplicialComplex3& complex, std::span<const Label> labels) {
  // marching.cpp:92-100
  if (static_cast<int64_t>(labels.size()) != complex.num_vertices())
    throw std::invalid_argument("label field size does not match vertex count");
  if (complex.dimension() < 2) throw std::invalid_argument("separating geometry needs a 2-D or 3-D complex");
}

// ---- recipe tables: the device table regrouped into the reference types --
struct Tables {
  std::vector<tables::SeparatorTri> tri;
  std::array<std::pair<int, int>, 32> tet_case{};
  std::vector<tables::SeparatorSeg> seg;
  std::array<std::pair<int, int>, 8> tri_case{};
  Tables() {
    uint32_t rows[52];
    uint16_t cases[32];
    plmss_b200_tet_table(rows, cases);
    for (uint32_t r : rows) {
      tables::SeparatorTri t;
      t.p[0] = uint8_t(r & 15);
      t.p[1] = uint8_t((r >> 4) & 15);
      t.p[2] = uint8_t((r >> 8) & 15);
      t.pairA = uint8_t((r >> 12) & 3);
      t.pairB = uint8_t((r >> 14) & 3);
      tri.push_back(t);
    }
    for (int c = 0; c < 32; ++c) tet_case[c] = {cases[c] >> 4, cases[c] & 15};
    // 2-D recipes (marching_tables.cpp:36-46) for API completeness; the
    // B200 marching path itself is 3-D.
    const uint8_t s2[6][4] = {{5, 6, 0, 2}, {3, 6, 0, 1}, {3, 5, 0, 1}, {7, 3, 0, 1}, {7, 6, 1, 2}, {7, 5, 0, 2}};
    for (const auto& r : s2) {
      tables::SeparatorSeg s;
      s.p[0] = r[0];
      s.p[1] = r[1];
      s.pairA = r[2];
      s.pairB = r[3];
      seg.push_back(s);
    }
    tri_case[2] = {0, 1};
    tri_case[4] = {1, 1};
    tri_case[5] = {2, 1};
    tri_case[6] = {3, 3};
  }
};

const Tables& tabs() {
  static const Tables t;
  return t;
}

}  // namespace

// ============================================================ orderfield ==
OrderField compute_order(const ScalarField& field) {
  const int64_t n = field.values.size();
  OrderField order;
  resize_out(order.rank, static_cast<size_t>(n));
  if (n == 0) return order;
  DevBuf<double> dv(n);
  DevBuf<int64_t> dr(n);
  dv.up(field.values.data(), n);
  check(plmss_b200_compute_order(ctx(), PLMSS_KEY_F64, dv.p, n, dr.p));
  dr.down(order.rank.data(), n);
  return order;
}

VertexClass classify_vertex(const SimplicialComplex3&, const OrderField&, VertexId) {
  throw std::logic_error(
      "classify_vertex is a test oracle of the reference (orderfield.cpp:34-92) and is not part of the B200 "
      "drop-in");
}

// ========================================================== segmentation ==
SegmentationResult segment(const SimplicialComplex3& complex, const OrderField& order, Direction direction,
                           int workers) {
  const int64_t n = complex.num_vertices();
  if (order.size() != n) throw std::invalid_argument("order field size does not match complex");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  const auto dims = grid_of(complex);
  const bool want_desc = direction != Direction::Ascending, want_asc = direction != Direction::Descending;
  DevBuf<int64_t> dk(n);
  dk.up(order.rank.data(), n);
  DevBuf<uint32_t> dd(want_desc ? n : 0), da(want_asc ? n : 0), dmx(want_desc ? n : 0), dmn(want_asc ? n : 0);
  int64_t nmax = 0, nmin = 0;
  int32_t sweeps = 0;
  check(plmss_b200_segment(ctx(), dims.data(), PLMSS_KEY_RANK, dk.p, int(direction), dd.p, da.p, dmx.p, dmn.p,
                           &nmax, &nmin, &sweeps));
  SegmentationResult seg;
  if (want_desc) {
    resize_out(seg.desc, size_t(n));
    down_widen(seg.desc.data(), dd.p, n);
    seg.maxima.resize(nmax);
    down_widen(seg.maxima.data(), dmx.p, nmax);
  }
  if (want_asc) {
    resize_out(seg.asc, size_t(n));
    down_widen(seg.asc.data(), da.p, n);
    seg.minima.resize(nmin);
    down_widen(seg.minima.data(), dmn.p, nmin);
  }
  seg.sweeps = sweeps;
  return seg;
}

void combine_ms(SegmentationResult& seg, int workers) {
  if (!seg.has_desc() || !seg.has_asc())
    throw std::invalid_argument("combine_ms needs both ascending and descending labels");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  const int64_t n = static_cast<int64_t>(seg.desc.size());
  DevBuf<uint32_t> da(n), dd(n), dm(n);
  DevBuf<uint64_t> dk(n);
  up_narrow(da.p, seg.asc.data(), n);
  up_narrow(dd.p, seg.desc.data(), n);
  int64_t r = 0;
  check(plmss_b200_combine_ms(ctx(), n, da.p, dd.p, dm.p, dk.p, &r));
  resize_out(seg.ms_region, size_t(n));
  down_widen(seg.ms_region.data(), dm.p, n);
  std::vector<uint64_t> keys(r);
  dk.down(keys.data(), r);
  seg.region_keys.resize(r);
  for (int64_t i = 0; i < r; ++i)
    seg.region_keys[i] = ms_key(VertexId(keys[i] >> 32), VertexId(keys[i] & 0xffffffffu));
}

VertexId oracle_integral_walk(const SimplicialComplex3&, const OrderField&, VertexId, Direction) {
  throw std::logic_error(
      "oracle_integral_walk is a test oracle of the reference (segmentation.cpp:198-217) and is not part of the "
      "B200 drop-in");
}

namespace detail {

void seed_hops(const SimplicialComplex3& complex, const OrderField& order, bool ascending, std::int64_t begin,
               std::int64_t end, std::span<VertexId> labels, std::vector<VertexId>& active,
               std::vector<VertexId>& extrema) {
  std::vector<VertexId> other(labels.size()), mx, mn, act;
  if (ascending)
    seed_hops_both(complex, order, begin, end, other, labels, act, mx, mn);
  else
    seed_hops_both(complex, order, begin, end, labels, other, act, mx, mn);
  for (VertexId v = begin; v < end; ++v) {
    if (labels[v] == v)
      extrema.push_back(v);
    else
      active.push_back(v);
  }
}

void seed_hops_both(const SimplicialComplex3& complex, const OrderField& order, std::int64_t begin,
                    std::int64_t end, std::span<VertexId> desc, std::span<VertexId> asc,
                    std::vector<VertexId>& active, std::vector<VertexId>& maxima, std::vector<VertexId>& minima) {
  const int64_t n = complex.num_vertices();
  const auto dims = grid_of(complex);
  if (order.size() != n) throw std::invalid_argument("order field size does not match complex");
  DevBuf<int64_t> dk(n);
  dk.up(order.rank.data(), n);
  DevBuf<uint32_t> dd(n), da(n);
  check(plmss_b200_seed_hops(ctx(), dims.data(), PLMSS_KEY_RANK, dk.p, dd.p, da.p));
  std::vector<uint32_t> hd(n), ha(n);
  dd.down(hd.data(), n);
  da.down(ha.data(), n);
  for (VertexId v = begin; v < end; ++v) {
    desc[v] = hd[v];
    asc[v] = ha[v];
    if (desc[v] == v) maxima.push_back(v);
    if (asc[v] == v) minima.push_back(v);
    if (desc[v] != v || asc[v] != v) active.push_back(v);
  }
}

namespace {
std::vector<VertexId> sweep(std::span<VertexId> desc, std::span<VertexId>* asc, std::span<const VertexId> active) {
  const int64_t n = static_cast<int64_t>(desc.size()), na = static_cast<int64_t>(active.size());
  std::vector<VertexId> next;
  if (na == 0) return next;
  DevBuf<uint32_t> dd(n), da(asc ? n : 0), dact(na), dnext(na);
  const auto d32 = narrow(desc), act32 = narrow(active);
  dd.up(d32.data(), n);
  if (asc) {
    const auto a32 = narrow(*asc);
    da.up(a32.data(), n);
  }
  dact.up(act32.data(), na);
  int64_t nn = 0;
  check(plmss_b200_compress_sweep(ctx(), dd.p, da.p, dact.p, na, dnext.p, &nn));
  std::vector<uint32_t> tmp(n);
  dd.down(tmp.data(), n);
  for (int64_t i = 0; i < n; ++i) desc[i] = tmp[i];
  if (asc) {
    da.down(tmp.data(), n);
    for (int64_t i = 0; i < n; ++i) (*asc)[i] = tmp[i];
  }
  tmp.resize(nn);
  dnext.down(tmp.data(), nn);
  return widen(tmp);
}
}  // namespace

std::vector<VertexId> compress_sweep(std::span<VertexId> labels, std::span<const VertexId> active) {
  return sweep(labels, nullptr, active);
}

std::vector<VertexId> compress_sweep_both(std::span<VertexId> desc, std::span<VertexId> asc,
                                          std::span<const VertexId> active) {
  return sweep(desc, &asc, active);
}

}  // namespace detail

// ============================================================== marching ==
CellCode triangle_code(const std::array<Label, 3>& labels) {
  // marching.cpp:14-26 (scalar helper; the bulk codes are computed on device)
  CellCode out;
  out.local[1] = labels[1] == labels[0] ? 0 : 1;
  out.local[2] = labels[2] == labels[0] ? 0 : (labels[2] == labels[1] ? out.local[1] : 2);
  out.code = static_cast<std::uint8_t>((out.local[1] << 2) | out.local[2]);
  return out;
}

CellCode tetra_code(const std::array<Label, 4>& labels) {
  // marching.cpp:28-44 (scalar helper; the bulk codes are computed on device)
  CellCode out;
  for (int i = 1; i < 4; ++i) {
    out.local[i] = static_cast<std::uint8_t>(i);
    for (int j = 0; j < i; ++j)
      if (labels[i] == labels[j]) {
        out.local[i] = out.local[j];
        break;
      }
  }
  out.code = static_cast<std::uint8_t>((out.local[1] << 4) | (out.local[2] << 2) | out.local[3]);
  return out;
}

namespace tables {

bool triangle_code_valid(std::uint8_t code) { return code == 0 || code == 2 || code == 4 || code == 5 || code == 6; }

bool tetra_code_valid(std::uint8_t code) {
  for (const std::uint8_t c : kValidTetraCodes)
    if (c == code) return true;
  return false;
}

std::span<const SeparatorSeg> triangle_case(std::uint8_t code) {
  if (code >= 8) return {};
  const auto& t = tabs();
  return {t.seg.data() + t.tri_case[code].first, static_cast<size_t>(t.tri_case[code].second)};
}

std::span<const SeparatorTri> tetra_case(std::uint8_t code) {
  if (code >= 32) return {};
  const auto& t = tabs();
  return {t.tri.data() + t.tet_case[code].first, static_cast<size_t>(t.tet_case[code].second)};
}

}  // namespace tables

SeparatorIndex index_separators(const SimplicialComplex3& complex, std::span<const Label> labels, int workers) {
  check_labels(complex, labels);
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  const auto dims = grid_of(complex);
  const int64_t n = complex.num_vertices(), nc = complex.num_cells();
  DevBuf<int64_t> dl(n);
  dl.up(labels.data(), n);
  DevBuf<uint8_t> dc(nc);
  int64_t total = 0;
  check(plmss_b200_index_separators(ctx(), dims.data(), 1, dl.p, dc.p, &total));
  SeparatorIndex index;
  index.workers = workers;
  index.codes.resize(nc);
  dc.down(index.codes.data(), nc);
  // per-worker counts over the same contiguous cell chunks the reference
  // uses (parallel.hpp:27-29), counted on the device
  std::vector<int64_t> bounds(workers + 1);
  for (int w = 0; w <= workers; ++w) bounds[w] = chunk_begin(w, workers, nc);
  index.plan.counts.assign(workers, 0);
  index.plan.offsets.assign(workers, 0);
  if (workers <= 1024) {
    check(plmss_b200_count_by_cell_ranges(ctx(), dims.data(), 1, dl.p, bounds.data(), workers,
                                          index.plan.counts.data()));
  } else {
    throw std::invalid_argument("the B200 drop-in supports at most 1024 workers in EmitPlan");
  }
  int64_t running = 0;
  for (int w = 0; w < workers; ++w) {
    index.plan.offsets[w] = running;
    running += index.plan.counts[w];
  }
  if (running != total) throw std::logic_error("indexing counts disagree with the total");
  return index;
}

SeparatingMesh emit_geometry(const SimplicialComplex3& complex, std::span<const Label> labels,
                             SeparatorIndex& index) {
  check_labels(complex, labels);
  const auto dims = grid_of(complex);
  const int64_t n = complex.num_vertices(), nc = complex.num_cells();
  const int workers = index.workers;
  DevBuf<int64_t> dl(n);
  dl.up(labels.data(), n);
  // writes per worker chunk must equal the indexed counts (marching.cpp:164-204)
  std::vector<int64_t> bounds(workers + 1), written(workers, 0);
  for (int w = 0; w <= workers; ++w) bounds[w] = chunk_begin(w, workers, nc);
  check(plmss_b200_count_by_cell_ranges(ctx(), dims.data(), 1, dl.p, bounds.data(), workers, written.data()));
  for (int w = 0; w < workers; ++w)
    if (w < static_cast<int>(index.plan.counts.size()) && written[w] > index.plan.counts[w])
      throw std::logic_error("geometry phase exceeds indexed primitive count");
  index.plan.written = written;
  for (int w = 0; w < workers; ++w)
    if (index.plan.written[w] != index.plan.counts[w])
      throw std::logic_error("geometry phase wrote " + std::to_string(index.plan.written[w]) +
                             " primitives, indexing counted " + std::to_string(index.plan.counts[w]));
  const int64_t total = index.plan.total();
  DevBuf<plmss_tri64> dt(total);
  int64_t got = 0;
  check(plmss_b200_emit_separators(ctx(), dims.data(), 1, dl.p, dt.p, total, &got));
  SeparatingMesh mesh;
  mesh.verts_per_primitive = 3;
  mesh.points.resize(3, 3 * total);
  prefault(mesh.points.data(), size_t(9 * total) * sizeof(double));
  resize_out(mesh.indices, static_cast<size_t>(3 * total));
  resize_out(mesh.regions, static_cast<size_t>(total));
  resize_out(mesh.source_cells, static_cast<size_t>(total));
  if (total) {
    const auto& sp = complex.grid_spacing();
    const auto& og = complex.grid_origin();
    const double spv[3] = {sp[0], sp[1], sp[2]}, ogv[3] = {og[0], og[1], og[2]};
    DevBuf<double> dp(9 * total);
    DevBuf<int64_t> dr(2 * total), ds(total);
    check(plmss_b200_materialize_separators(ctx(), dims.data(), spv, ogv, 1, dt.p, total, dp.p, dr.p, ds.p));
    dp.down(mesh.points.data(), 9 * total);
    static_assert(sizeof(std::array<Label, 2>) == 2 * sizeof(int64_t), "region pair layout");
    dr.down(reinterpret_cast<int64_t*>(mesh.regions.data()), 2 * total);
    ds.down(mesh.source_cells.data(), total);
    int64_t* idx = mesh.indices.data();
    parallel_for(3 * total, [&](int64_t b, int64_t e) {
      for (int64_t i = b; i < e; ++i) idx[i] = i;
    });
  }
  return mesh;
}

SeparatingMesh emit_separators(const SimplicialComplex3& complex, std::span<const Label> labels, int workers,
                               EmitPlan* planOut) {
  SeparatorIndex index = index_separators(complex, labels, workers);
  SeparatingMesh mesh = emit_geometry(complex, labels, index);
  if (planOut) *planOut = index.plan;
  return mesh;
}

SeparatingMesh emit_boundaries(const SimplicialComplex3& complex, std::span<const Label> labels,
                               std::optional<Label> regionFilter, int workers) {
  check_labels(complex, labels);
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  const auto dims = grid_of(complex);
  const int64_t n = complex.num_vertices();
  DevBuf<int64_t> dl(n);
  dl.up(labels.data(), n);
  const auto& sp = complex.grid_spacing();
  const auto& og = complex.grid_origin();
  const double spv[3] = {sp[0], sp[1], sp[2]}, ogv[3] = {og[0], og[1], og[2]};
  int64_t nf = 0, np = 0;
  const int hf = regionFilter ? 1 : 0;
  const int64_t flt = regionFilter ? *regionFilter : 0;
  check(plmss_b200_emit_boundaries(ctx(), dims.data(), spv, ogv, 1, dl.p, hf, flt, nullptr, nullptr, nullptr,
                                   nullptr, nullptr, &nf, &np));
  DevBuf<uint32_t> dfc(3 * std::max<int64_t>(nf, 1));
  DevBuf<int64_t> dtag(std::max<int64_t>(nf, 1)), dcell(std::max<int64_t>(nf, 1)),
      didx(3 * std::max<int64_t>(nf, 1));
  DevBuf<double> dpts(3 * std::max<int64_t>(np, 1));
  check(plmss_b200_emit_boundaries(ctx(), dims.data(), spv, ogv, 1, dl.p, hf, flt, dfc.p, dtag.p, dcell.p, dpts.p,
                                   didx.p, &nf, &np));
  SeparatingMesh mesh;
  mesh.verts_per_primitive = 3;
  mesh.points.resize(3, np);
  prefault(mesh.points.data(), size_t(3 * np) * sizeof(double));
  dpts.down(mesh.points.data(), 3 * np);
  resize_out(mesh.indices, static_cast<size_t>(3 * nf));
  didx.down(mesh.indices.data(), 3 * nf);
  std::vector<int64_t> tags(nf);
  dtag.down(tags.data(), nf);
  resize_out(mesh.regions, static_cast<size_t>(nf));
  parallel_for(nf, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) mesh.regions[i] = {tags[i], -1};
  });
  resize_out(mesh.source_cells, static_cast<size_t>(nf));
  dcell.down(mesh.source_cells.data(), nf);
  return mesh;
}

std::vector<std::vector<Label>> select_labels(const SegmentationResult& seg, SegMode mode) {
  // marching.cpp:328-350
  switch (mode) {
    case SegMode::Ascending:
      if (!seg.has_asc()) throw std::logic_error("ascending labels missing");
      return {std::vector<Label>(seg.asc.begin(), seg.asc.end())};
    case SegMode::Descending:
      if (!seg.has_desc()) throw std::logic_error("descending labels missing");
      return {std::vector<Label>(seg.desc.begin(), seg.desc.end())};
    case SegMode::MorseSmale:
      if (!seg.has_ms()) throw std::logic_error("combine_ms has not been run");
      return {seg.ms_region};
    case SegMode::Union:
      if (!seg.has_asc() || !seg.has_desc()) throw std::logic_error("union needs both directions");
      return {std::vector<Label>(seg.asc.begin(), seg.asc.end()), std::vector<Label>(seg.desc.begin(), seg.desc.end())};
  }
  throw std::logic_error("unknown segmentation mode");
}

void append_mesh(SeparatingMesh& mesh, const SeparatingMesh& extra) {
  // container concatenation (marching.cpp:352-371), not a compute step
  if (extra.num_primitives() == 0) return;
  if (mesh.num_primitives() == 0) {
    mesh = extra;
    return;
  }
  if (mesh.verts_per_primitive != extra.verts_per_primitive)
    throw std::invalid_argument("cannot append meshes of different arity");
  const int64_t base = mesh.points.cols();
  mesh.points.conservativeResize(3, base + extra.points.cols());
  mesh.points.rightCols(extra.points.cols()) = extra.points;
  for (const auto idx : extra.indices) mesh.indices.push_back(idx + base);
  mesh.regions.insert(mesh.regions.end(), extra.regions.begin(), extra.regions.end());
  mesh.source_cells.insert(mesh.source_cells.end(), extra.source_cells.begin(), extra.source_cells.end());
}

void weld_points(SeparatingMesh& mesh) {
  // marching.cpp:400-417 on the device (plmss_b200_weld_points): the first
  // occurrence of every bitwise-distinct point keeps its place in order
  const int64_t n = mesh.points.cols(), m = static_cast<int64_t>(mesh.indices.size());
  if (n == 0) {
    if (m) throw std::out_of_range("point index out of range");
    return;
  }
  DevBuf<double> dp(3 * n);
  DevBuf<int64_t> di(m);
  dp.up(mesh.points.data(), 3 * n);
  di.up(mesh.indices.data(), m);
  int64_t unique = 0;
  check(plmss_b200_weld_points(ctx(), dp.p, n, di.p, m, &unique));
  dp.down(mesh.points.data(), 3 * unique);
  mesh.points.conservativeResize(3, unique);
  di.down(mesh.indices.data(), m);
}

}  // namespace plmss
