// ctypes-facing C wrapper around the reference PLMSS library — TEST
// INFRASTRUCTURE ONLY (oracle). Never linked into the product library.
//
// It is compiled twice by oracle/Makefile:
//   * with -Dplmss=plmss_ref against the UNMODIFIED reference sources under
//     /root/reference/proj/src  -> oracle/_ref/libplmss_ref.so  (CPU oracle and
//     the `bench.py --impl reference` arm);
//   * with the reference's own complex/bench sources plus the GPU drop-in facade
//     (paper_2303_15491_b200/csrc/dropin/) in place of orderfield/segmentation/
//     marching -> build/libplmss_dropin_harness.so, so the very same calls run the
//     reference API against the B200 implementation.
//
// Every entry point forwards to the reference public API declared in
// proj/include/plmss/{orderfield,segmentation,marching,bench}.hpp and converts
// C++ exceptions into (status, message): 1 invalid_argument, 2 logic_error,
// 3 out_of_range, 4 other, 6 io FormatError, 7 io IoError.
#include <array>
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "plmss/bench.hpp"
#include "plmss/complex.hpp"
#include "plmss/io.hpp"
#include "plmss/marching.hpp"
#include "plmss/orderfield.hpp"
#include "plmss/segmentation.hpp"

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return 3;
  } catch (const std::logic_error& e) {
    g_error = e.what();
    return 2;
  } catch (const plmss::FormatError& e) {
    g_error = e.what();
    return 6;
  } catch (const plmss::IoError& e) {
    g_error = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 4;
  }
}

plmss::SimplicialComplex3 make_grid(const int64_t* dims, const double* spacing,
                                    const double* origin) {
  Eigen::Vector3d sp = spacing ? Eigen::Vector3d(spacing[0], spacing[1], spacing[2])
                               : Eigen::Vector3d::Ones();
  Eigen::Vector3d og = origin ? Eigen::Vector3d(origin[0], origin[1], origin[2])
                              : Eigen::Vector3d::Zero();
  return plmss::SimplicialComplex3::implicit_grid({dims[0], dims[1], dims[2]}, sp, og);
}

plmss::OrderField order_from(const int64_t* rank, int64_t n) {
  plmss::OrderField o;
  o.rank.assign(rank, rank + n);
  return o;
}

struct MeshOut {
  plmss::SeparatingMesh mesh;
  plmss::EmitPlan plan;
  std::vector<std::uint8_t> codes;
};

}  // namespace

extern "C" {

const char* cap_last_error() { return g_error.c_str(); }

int cap_compute_order(const double* values, int64_t n, int64_t* rank_out) {
  return guarded([&] {
    plmss::ScalarField f;
    f.values.resize(n);
    for (int64_t i = 0; i < n; ++i) f.values[i] = values[i];
    const plmss::OrderField o = plmss::compute_order(f);
    std::memcpy(rank_out, o.rank.data(), sizeof(int64_t) * static_cast<size_t>(n));
  });
}

// direction: 0 ascending, 1 descending, 2 both (plmss::Direction order).
int cap_segment(const int64_t* dims, const int64_t* rank, int64_t n, int direction,
                int workers, int do_combine, void** handle) {
  return guarded([&] {
    const auto grid = make_grid(dims, nullptr, nullptr);
    auto* seg = new plmss::SegmentationResult(plmss::segment(
        grid, order_from(rank, n), static_cast<plmss::Direction>(direction), workers));
    if (do_combine) {
      try {
        plmss::combine_ms(*seg, workers);
      } catch (...) {
        delete seg;
        throw;
      }
    }
    *handle = seg;
  });
}

// which: 0 desc, 1 asc, 2 maxima, 3 minima, 4 ms_region, 5 region_keys (2 x u64
// per key: min then max), 6 sweeps (1 value).
int64_t cap_seg_size(void* handle, int which) {
  auto* s = static_cast<plmss::SegmentationResult*>(handle);
  switch (which) {
    case 0: return static_cast<int64_t>(s->desc.size());
    case 1: return static_cast<int64_t>(s->asc.size());
    case 2: return static_cast<int64_t>(s->maxima.size());
    case 3: return static_cast<int64_t>(s->minima.size());
    case 4: return static_cast<int64_t>(s->ms_region.size());
    case 5: return static_cast<int64_t>(s->region_keys.size()) * 2;
    case 6: return 1;
  }
  return -1;
}

void cap_seg_copy(void* handle, int which, int64_t* out) {
  auto* s = static_cast<plmss::SegmentationResult*>(handle);
  auto cp = [&](const std::vector<int64_t>& v) {
    if (!v.empty()) std::memcpy(out, v.data(), sizeof(int64_t) * v.size());
  };
  switch (which) {
    case 0: cp(s->desc); break;
    case 1: cp(s->asc); break;
    case 2: cp(s->maxima); break;
    case 3: cp(s->minima); break;
    case 4: cp(s->ms_region); break;
    case 5:
      for (size_t i = 0; i < s->region_keys.size(); ++i) {
        out[2 * i] = plmss::ms_key_min(s->region_keys[i]);
        out[2 * i + 1] = plmss::ms_key_max(s->region_keys[i]);
      }
      break;
    case 6: out[0] = s->sweeps; break;
  }
}

void cap_seg_free(void* handle) { delete static_cast<plmss::SegmentationResult*>(handle); }

// detail:: step functions (segmentation.hpp:90-121) of whichever library this
// file is linked against (the compiled reference or the B200 drop-in).
// mode 0 / 1: seed_hops descending / ascending into desc; 2: seed_hops_both.
int cap_seed_hops(const int64_t* dims, const int64_t* rank, int64_t n, int mode, int64_t begin, int64_t end,
                  int64_t* desc, int64_t* asc, int64_t* active, int64_t* n_active, int64_t* ext1, int64_t* n_ext1,
                  int64_t* ext2, int64_t* n_ext2) {
  return guarded([&] {
    const auto grid = make_grid(dims, nullptr, nullptr);
    const auto order = order_from(rank, n);
    std::vector<plmss::VertexId> d(size_t(n), -1), a(size_t(n), -1), act, e1, e2;
    if (mode == 2)
      plmss::detail::seed_hops_both(grid, order, begin, end, d, a, act, e1, e2);
    else
      plmss::detail::seed_hops(grid, order, mode == 1, begin, end, d, act, e1);
    std::memcpy(desc, d.data(), sizeof(int64_t) * size_t(n));
    if (asc) std::memcpy(asc, a.data(), sizeof(int64_t) * size_t(n));
    auto out = [](const std::vector<plmss::VertexId>& v, int64_t* dst, int64_t* cnt) {
      *cnt = int64_t(v.size());
      if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(int64_t) * v.size());
    };
    out(act, active, n_active);
    out(e1, ext1, n_ext1);
    out(e2, ext2, n_ext2);
  });
}

// One compress_sweep (asc == NULL) / compress_sweep_both, labels in place.
int cap_compress_sweep(int64_t* desc, int64_t* asc, int64_t n, const int64_t* active, int64_t na, int64_t* next,
                       int64_t* n_next) {
  return guarded([&] {
    std::span<plmss::VertexId> d(desc, size_t(n));
    std::span<const plmss::VertexId> act(active, size_t(na));
    const std::vector<plmss::VertexId> nx =
        asc ? plmss::detail::compress_sweep_both(d, std::span<plmss::VertexId>(asc, size_t(n)), act)
            : plmss::detail::compress_sweep(d, act);
    *n_next = int64_t(nx.size());
    if (!nx.empty()) std::memcpy(next, nx.data(), sizeof(int64_t) * nx.size());
  });
}

int cap_oracle_walk(const int64_t* dims, const int64_t* rank, int64_t n, int64_t v,
                    int direction, int64_t* out) {
  return guarded([&] {
    const auto grid = make_grid(dims, nullptr, nullptr);
    *out = plmss::oracle_integral_walk(grid, order_from(rank, n), v,
                                       static_cast<plmss::Direction>(direction));
  });
}

int cap_tetra_code(const int64_t* labels4, int32_t* code, int32_t* local4) {
  return guarded([&] {
    const auto c = plmss::tetra_code({labels4[0], labels4[1], labels4[2], labels4[3]});
    *code = c.code;
    for (int i = 0; i < 4; ++i) local4[i] = c.local[i];
  });
}

int cap_triangle_code(const int64_t* labels3, int32_t* code) {
  return guarded([&] { *code = plmss::triangle_code({labels3[0], labels3[1], labels3[2]}).code; });
}

// Table rows for a tetra code as 5 bytes each (p0,p1,p2,pairA,pairB). Returns count.
int cap_tetra_case(int code, uint8_t* out) {
  const auto rows = plmss::tables::tetra_case(static_cast<std::uint8_t>(code));
  int i = 0;
  for (const auto& r : rows) {
    out[5 * i + 0] = r.p[0];
    out[5 * i + 1] = r.p[1];
    out[5 * i + 2] = r.p[2];
    out[5 * i + 3] = r.pairA;
    out[5 * i + 4] = r.pairB;
    ++i;
  }
  return i;
}

int cap_triangle_case(int code, uint8_t* out) {
  const auto rows = plmss::tables::triangle_case(static_cast<std::uint8_t>(code));
  int i = 0;
  for (const auto& r : rows) {
    out[4 * i + 0] = r.p[0];
    out[4 * i + 1] = r.p[1];
    out[4 * i + 2] = r.pairA;
    out[4 * i + 3] = r.pairB;
    ++i;
  }
  return i;
}

// kind: 0 separators (index_separators + emit_geometry), 1 boundaries.
int cap_emit(const int64_t* dims, const double* spacing, const double* origin,
             const int64_t* labels, int64_t n, int kind, int workers, int has_filter,
             int64_t filter, void** handle) {
  return guarded([&] {
    const auto grid = make_grid(dims, spacing, origin);
    std::span<const plmss::Label> lab(labels, static_cast<size_t>(n));
    auto* out = new MeshOut();
    try {
      if (kind == 0) {
        plmss::SeparatorIndex index = plmss::index_separators(grid, lab, workers);
        out->mesh = plmss::emit_geometry(grid, lab, index);
        out->plan = index.plan;
        out->codes = index.codes;
      } else {
        std::optional<plmss::Label> f;
        if (has_filter) f = filter;
        out->mesh = plmss::emit_boundaries(grid, lab, f, workers);
      }
    } catch (...) {
      delete out;
      throw;
    }
    *handle = out;
  });
}

// sizes: [n_primitives, n_points, verts_per_primitive, n_codes, plan_total]
void cap_mesh_sizes(void* handle, int64_t* sizes) {
  auto* m = static_cast<MeshOut*>(handle);
  sizes[0] = m->mesh.num_primitives();
  sizes[1] = m->mesh.num_points();
  sizes[2] = m->mesh.verts_per_primitive;
  sizes[3] = static_cast<int64_t>(m->codes.size());
  sizes[4] = m->plan.total();
}

void cap_mesh_copy(void* handle, double* points, int64_t* indices, int64_t* regions,
                   int64_t* source_cells, uint8_t* codes) {
  auto* m = static_cast<MeshOut*>(handle);
  const auto& mesh = m->mesh;
  if (points && mesh.num_points() > 0)
    std::memcpy(points, mesh.points.data(), sizeof(double) * 3 * static_cast<size_t>(mesh.num_points()));
  if (indices && !mesh.indices.empty())
    std::memcpy(indices, mesh.indices.data(), sizeof(int64_t) * mesh.indices.size());
  if (regions)
    for (size_t i = 0; i < mesh.regions.size(); ++i) {
      regions[2 * i] = mesh.regions[i][0];
      regions[2 * i + 1] = mesh.regions[i][1];
    }
  if (source_cells && !mesh.source_cells.empty())
    std::memcpy(source_cells, mesh.source_cells.data(), sizeof(int64_t) * mesh.source_cells.size());
  if (codes && !m->codes.empty()) std::memcpy(codes, m->codes.data(), m->codes.size());
}

void cap_mesh_free(void* handle) { delete static_cast<MeshOut*>(handle); }

// Runs the reference benchmark protocol (proj/src/bench.cpp:46-103) on one
// worker count; phases_out = trimmed-mean [order, seg, combine, index, geometry].
int cap_run_benchmark(const int64_t* dims, const double* values, int workers, int repeats,
                      int mode, double* phases_out) {
  return guarded([&] {
    const auto grid = make_grid(dims, nullptr, nullptr);
    plmss::ScalarField f;
    const int64_t n = dims[0] * dims[1] * dims[2];
    f.values.resize(n);
    for (int64_t i = 0; i < n; ++i) f.values[i] = values[i];
    const auto rep = plmss::run_benchmark(grid, f, {workers}, repeats, "cap",
                                          static_cast<plmss::SegMode>(mode));
    const auto& m = rep.rows.front().mean;
    phases_out[0] = m.order;
    phases_out[1] = m.segmentation;
    phases_out[2] = m.combine;
    phases_out[3] = m.index;
    phases_out[4] = m.geometry;
  });
}

// One pass of the benchmarked pipeline exactly as run_benchmark's inner loop
// (proj/src/bench.cpp:62-87): compute_order, segment(Both), combine_ms,
// select_labels(mode), index_separators + emit_geometry per field. Phase
// wall times (s) go to phases_out[5]; counts_out = [regions, primitives].
int cap_run_once(const int64_t* dims, const float* values, int workers, int mode, double* phases_out,
                 int64_t* counts_out) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
    const auto grid = make_grid(dims, nullptr, nullptr);
    plmss::ScalarField f;
    const int64_t n = dims[0] * dims[1] * dims[2];
    f.values.resize(n);
    for (int64_t i = 0; i < n; ++i) f.values[i] = values[i];
    auto mark = clk::now();
    const plmss::OrderField order = plmss::compute_order(f);
    phases_out[0] = secs(mark);
    mark = clk::now();
    plmss::SegmentationResult seg = plmss::segment(grid, order, plmss::Direction::Both, workers);
    phases_out[1] = secs(mark);
    mark = clk::now();
    plmss::combine_ms(seg, workers);
    phases_out[2] = secs(mark);
    phases_out[3] = phases_out[4] = 0;
    int64_t prims = 0;
    for (const auto& labels : plmss::select_labels(seg, static_cast<plmss::SegMode>(mode))) {
      mark = clk::now();
      plmss::SeparatorIndex index = plmss::index_separators(grid, labels, workers);
      phases_out[3] += secs(mark);
      mark = clk::now();
      prims += plmss::emit_geometry(grid, labels, index).num_primitives();
      phases_out[4] += secs(mark);
    }
    counts_out[0] = seg.num_regions();
    counts_out[1] = prims;
  });
}

// weld_points (marching.cpp:400-417) on a soup given as (n, 3) points and
// indices; both are overwritten, *n_unique = points kept.
int cap_weld(double* points, int64_t n, int64_t* indices, int64_t m, int64_t* n_unique) {
  return guarded([&] {
    plmss::SeparatingMesh mesh;
    mesh.points.resize(3, n);
    if (n) std::memcpy(mesh.points.data(), points, sizeof(double) * 3 * static_cast<size_t>(n));
    mesh.indices.assign(indices, indices + m);
    plmss::weld_points(mesh);
    *n_unique = mesh.points.cols();
    if (mesh.points.cols())
      std::memcpy(points, mesh.points.data(), sizeof(double) * 3 * static_cast<size_t>(mesh.points.cols()));
    if (m) std::memcpy(indices, mesh.indices.data(), sizeof(int64_t) * static_cast<size_t>(m));
  });
}

// read_volume (io.cpp:90-124): values as doubles into out (X*Y*Z).
int cap_read_volume(const char* path, const int64_t* dims, const char* dtype, double* out) {
  return guarded([&] {
    plmss::VolumeSpec spec;
    spec.path = path;
    spec.dims = {dims[0], dims[1], dims[2]};
    spec.dtype = plmss::parse_dtype(dtype);
    const plmss::VolumeData d = plmss::read_volume(spec);
    std::memcpy(out, d.field.values.data(), sizeof(double) * static_cast<size_t>(d.field.values.size()));
  });
}

int cap_write_labels(const char* path, const int64_t* asc, const int64_t* desc, int64_t n) {
  return guarded([&] {
    plmss::SegmentationResult seg;
    seg.asc.assign(asc, asc + n);
    seg.desc.assign(desc, desc + n);
    plmss::write_labels(seg, path);
  });
}

// write_surface_obj (io.cpp:268-299); regions are (n_prims, 2).
int cap_write_obj(const char* path, const double* points, int64_t n_points, const int64_t* indices,
                  const int64_t* regions, int64_t n_prims, int verts_per_prim) {
  return guarded([&] {
    plmss::SeparatingMesh mesh;
    mesh.verts_per_primitive = verts_per_prim;
    mesh.points.resize(3, n_points);
    if (n_points) std::memcpy(mesh.points.data(), points, sizeof(double) * 3 * static_cast<size_t>(n_points));
    mesh.indices.assign(indices, indices + n_prims * verts_per_prim);
    mesh.regions.resize(static_cast<size_t>(n_prims));
    for (int64_t i = 0; i < n_prims; ++i) mesh.regions[i] = {regions[2 * i], regions[2 * i + 1]};
    mesh.source_cells.assign(static_cast<size_t>(n_prims), 0);
    plmss::write_surface_obj(mesh, path);
  });
}

// Separator records of cube layers [cz0, cz1) of a (X, Y, Z) grid from the
// reference itself: emit_separators (marching.cpp:208-215) on the z-chunk
// grid implicit_grid({X, Y, cz1 - cz0 + 1}, spacing 1, origin (0, 0, cz0))
// over the label slice of vertex layers [cz0, cz1], each
// triangle converted to the 16-byte record (global cell << 6 | recipe row,
// lo, hi). The recipe row of the k-th triangle of cell c is
// tetra_case(code(c))[k] (marching.cpp:160-195 emits a cell's rows in table
// order); the row is CHECKED by recomputing its three corner points (mean of
// the masked tet vertex positions, ascending corner order) and its region
// pair against the reference's own output, bit for bit. out == nullptr:
// count only. *count = records.
struct RecordsOut {
  struct Rec {
    uint64_t cellrow;
    uint32_t lo, hi;
  };
  std::vector<Rec> rec;
  // the reference mesh of the chunk (global cell ids), for geometry digests
  std::vector<double> points;
  std::vector<int64_t> regions, cells;
};

int cap_records_chunk(const int64_t* dims, const int64_t* labels, int64_t cz0, int64_t cz1, int workers,
                      void** handle, int64_t* count) {
  return guarded([&] {
    const int64_t X = dims[0], Y = dims[1];
    const int64_t nzv = cz1 - cz0 + 1;
    const int64_t cdims[3] = {X, Y, nzv};
    const double og[3] = {0.0, 0.0, double(cz0)};
    const auto grid = make_grid(cdims, nullptr, og);
    std::span<const plmss::Label> lab(labels, static_cast<size_t>(X * Y * nzv));
    const plmss::SeparatingMesh mesh = plmss::emit_separators(grid, lab, workers);
    const int64_t np = mesh.num_primitives();
    auto* res = new RecordsOut();
    *handle = res;
    *count = np;
    res->rec.resize(size_t(np));
    res->regions.resize(2 * size_t(np));
    res->cells.resize(size_t(np));
    res->points.assign(mesh.points.data(), mesh.points.data() + 3 * mesh.points.cols());  // column-major 3 x N
    // kTetraData row offsets (the GPU table numbering, marching_tables.cpp:48-116)
    const auto* data0 = plmss::tables::tetra_case(3).data();
    RecordsOut::Rec* rec = res->rec.data();
    const int64_t cell_base = 6 * (X - 1) * (Y - 1) * cz0;
    int64_t prev_cell = -1, k = 0;
    for (int64_t j = 0; j < np; ++j) {
      const int64_t c = mesh.source_cells[j];
      k = c == prev_cell ? k + 1 : 0;
      prev_cell = c;
      const auto verts = grid.cell(c);
      std::array<plmss::Label, 4> l{};
      for (int i = 0; i < 4; ++i) l[i] = labels[verts[i]];
      const auto code = plmss::tetra_code(l).code;
      const auto rows = plmss::tables::tetra_case(code);
      if (k >= int64_t(rows.size())) throw std::logic_error("cap_records_chunk: row count");
      const auto& row = rows[k];
      for (int q = 0; q < 3; ++q) {
        Eigen::Vector3d sum = Eigen::Vector3d::Zero();
        int cnt = 0;
        for (int i = 0; i < 4; ++i)
          if (row.p[q] & (1 << i)) {
            sum += grid.position(verts[i]);
            ++cnt;
          }
        const Eigen::Vector3d pt = sum / double(cnt);
        for (int a = 0; a < 3; ++a)
          if (pt[a] != mesh.points(a, mesh.indices[3 * j + q]))
            throw std::logic_error("cap_records_chunk: recipe point mismatch at triangle " + std::to_string(j));
      }
      const plmss::Label la = l[row.pairA], lb = l[row.pairB];
      if (mesh.regions[j][0] != std::min(la, lb) || mesh.regions[j][1] != std::max(la, lb))
        throw std::logic_error("cap_records_chunk: region pair mismatch");
      rec[j].cellrow = (uint64_t(cell_base + c) << 6) | uint64_t(&row - data0);
      res->regions[2 * j] = mesh.regions[j][0];
      res->regions[2 * j + 1] = mesh.regions[j][1];
      res->cells[j] = cell_base + c;
      rec[j].lo = uint32_t(mesh.regions[j][0]);
      rec[j].hi = uint32_t(mesh.regions[j][1]);
    }
  });
}

void cap_records_copy(void* handle, void* out) {
  auto* r = static_cast<RecordsOut*>(handle);
  if (!r->rec.empty()) std::memcpy(out, r->rec.data(), r->rec.size() * sizeof(RecordsOut::Rec));
}

void cap_records_free(void* handle) { delete static_cast<RecordsOut*>(handle); }

// The chunk's SeparatingMesh arrays: points (3 per corner, 9 per triangle),
// regions (2 per triangle), source cells (global).
void cap_records_geometry(void* handle, double* points, int64_t* regions, int64_t* cells) {
  auto* r = static_cast<RecordsOut*>(handle);
  if (points && !r->points.empty()) std::memcpy(points, r->points.data(), r->points.size() * sizeof(double));
  if (regions && !r->regions.empty()) std::memcpy(regions, r->regions.data(), r->regions.size() * sizeof(int64_t));
  if (cells && !r->cells.empty()) std::memcpy(cells, r->cells.data(), r->cells.size() * sizeof(int64_t));
}

}  // extern "C"
