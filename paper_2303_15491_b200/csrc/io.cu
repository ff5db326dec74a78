// Callers either side of the hot path:
//  * weld_points (marching.cpp:400-417): merge bitwise-identical separator
//    points, first occurrence wins, indices remapped — on the device;
//  * read_volume (io.cpp:90-124): a raw little-endian volume streamed from
//    the file through pinned staging buffers straight into device memory
//    (f32 for the pipeline, or f64 like the reference's ScalarField);
//  * write_labels (io.cpp:216-235) and write_surface_obj (io.cpp:268-299):
//    the reference file formats written from device arrays, streamed in
//    chunks (device -> pinned host -> file), OBJ text formatted by host
//    threads in order.
#include <errno.h>
#include <fcntl.h>
#include <stdio.h>
#include <string.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <exception>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace plmss_b200 {

namespace {

// ------------------------------------------------------------ weld_points --
// Open-addressing table of point indices keyed by the point's 3 x 64 bits.
// A slot holds some index of its point class; atomicMin keeps the lowest, so
// once all inserts are done the slot names the class's first occurrence.
constexpr unsigned long long kNoSlot = ~0ull;

__device__ __forceinline__ uint64_t point_hash(uint64_t x, uint64_t y, uint64_t z) {
  uint64_t h = x * 0x9E3779B97F4A7C15ull ^ (y + 0x632BE59BD9B4E019ull) * 0xC2B2AE3D27D4EB4Full ^
               (z + 0x165667B19E3779F9ull) * 0xD6E8FEB86659FD93ull;
  h ^= h >> 32;
  h *= 0xD6E8FEB86659FD93ull;
  h ^= h >> 29;
  return h;
}

__device__ __forceinline__ bool same_point(const uint64_t* __restrict__ p, uint64_t j, uint64_t x, uint64_t y,
                                           uint64_t z) {
  return p[3 * j] == x && p[3 * j + 1] == y && p[3 * j + 2] == z;
}

__global__ void k_weld_insert(const uint64_t* __restrict__ p, int64_t n, unsigned long long* __restrict__ table,
                              uint64_t mask) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t x = p[3 * i], y = p[3 * i + 1], z = p[3 * i + 2];
  for (uint64_t h = point_hash(x, y, z) & mask;; h = (h + 1) & mask) {
    unsigned long long cur = table[h];
    if (cur == kNoSlot) {
      cur = atomicCAS(&table[h], kNoSlot, (unsigned long long)i);
      if (cur == kNoSlot) return;
    }
    // every index a slot ever holds belongs to the same point class
    if (same_point(p, cur, x, y, z)) {
      atomicMin(&table[h], (unsigned long long)i);
      return;
    }
  }
}

// rep[i] = first occurrence of point i's class; flag[i] = 1 when i is it
__global__ void k_weld_rep(const uint64_t* __restrict__ p, int64_t n, const unsigned long long* __restrict__ table,
                           uint64_t mask, int64_t* __restrict__ rep, uint64_t* __restrict__ flag) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t x = p[3 * i], y = p[3 * i + 1], z = p[3 * i + 2];
  for (uint64_t h = point_hash(x, y, z) & mask;; h = (h + 1) & mask) {
    const unsigned long long cur = table[h];
    if (same_point(p, cur, x, y, z)) {
      rep[i] = int64_t(cur);
      flag[i] = cur == (unsigned long long)i;
      return;
    }
  }
}

// first occurrences move to their rank (into a copy); rep becomes the remap
__global__ void k_weld_compact(const uint64_t* __restrict__ p, int64_t n, const int64_t* __restrict__ rep,
                               const uint64_t* __restrict__ rank, uint64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || rep[i] != i) return;
  const uint64_t r = rank[i];
  out[3 * r] = p[3 * i];
  out[3 * r + 1] = p[3 * i + 1];
  out[3 * r + 2] = p[3 * i + 2];
}

__global__ void k_weld_remap(int64_t* __restrict__ idx, int64_t m, const int64_t* __restrict__ rep,
                             const uint64_t* __restrict__ rank, int64_t n, int* __restrict__ bad) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t v = idx[k];
  if (v < 0 || v >= n) {
    *bad = 1;
    return;
  }
  idx[k] = int64_t(rank[rep[v]]);
}

// ------------------------------------------------------------ read_volume --
__global__ void k_convert_volume(const unsigned char* __restrict__ src, int64_t count, int dtype, int out_f64,
                                 void* __restrict__ dst) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double v;
  switch (dtype) {
    case PLMSS_DTYPE_F32LE: v = double(reinterpret_cast<const float*>(src)[i]); break;
    case PLMSS_DTYPE_F64LE: v = reinterpret_cast<const double*>(src)[i]; break;
    case PLMSS_DTYPE_U8: v = double(src[i]); break;
    case PLMSS_DTYPE_U16LE: v = double(reinterpret_cast<const uint16_t*>(src)[i]); break;
    default: v = double(reinterpret_cast<const int16_t*>(src)[i]); break;
  }
  if (out_f64)
    static_cast<double*>(dst)[i] = v;
  else  // exact for every dtype but f64 (refused by the host side)
    static_cast<float*>(dst)[i] = float(v);
}

size_t dtype_bytes(int dtype) {
  switch (dtype) {
    case PLMSS_DTYPE_F32LE: return 4;
    case PLMSS_DTYPE_F64LE: return 8;
    case PLMSS_DTYPE_U8: return 1;
    case PLMSS_DTYPE_U16LE:
    case PLMSS_DTYPE_I16LE: return 2;
  }
  fail(PLMSS_ERR_FORMAT, "unknown dtype " + std::to_string(dtype) + " (expected f32le, f64le, u8, u16le, or i16le)");
}

struct File {
  int fd = -1;
  File(const char* path, int flags, const std::string& what) {
    fd = ::open(path, flags, 0644);
    if (fd < 0) fail(PLMSS_ERR_IO, "cannot open " + std::string(path) + what);
  }
  ~File() {
    if (fd >= 0) ::close(fd);
  }
};

void write_all(int fd, const void* data, size_t bytes, const char* path) {
  const char* p = static_cast<const char*>(data);
  while (bytes) {
    const ssize_t w = ::write(fd, p, bytes);
    if (w < 0 && errno == EINTR) continue;
    if (w <= 0) fail(PLMSS_ERR_IO, "write failed on " + std::string(path));
    p += w;
    bytes -= size_t(w);
  }
}

void pwrite_all(int fd, const void* data, size_t bytes, uint64_t off, const char* path) {
  const char* p = static_cast<const char*>(data);
  while (bytes) {
    const ssize_t w = ::pwrite(fd, p, bytes, off_t(off));
    if (w < 0 && errno == EINTR) continue;
    if (w <= 0) fail(PLMSS_ERR_IO, "write failed on " + std::string(path));
    p += w;
    off += uint64_t(w);
    bytes -= size_t(w);
  }
}

// Runs fn(t) on nt host threads; the first failure is rethrown.
void on_threads(unsigned nt, const std::function<void(unsigned)>& fn) {
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(nt);
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      try {
        fn(t);
      } catch (...) {
        err[t] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

unsigned host_threads() { return std::max(1u, std::min(16u, std::thread::hardware_concurrency())); }

constexpr size_t kChunk = size_t(64) << 20;  // staging chunk (bytes)

}  // namespace

int64_t weld_points(Ctx& c, double* d_points, int64_t n, int64_t* d_indices, int64_t m) {
  if (n < 0 || m < 0) fail(PLMSS_ERR_INVALID_ARGUMENT, "negative size");
  if (n == 0) {
    if (m) fail(PLMSS_ERR_OUT_OF_RANGE, "point index out of range");
    return 0;
  }
  uint64_t cap = 1024;
  while (cap < 2 * uint64_t(n)) cap <<= 1;
  auto* table = c.get_t<unsigned long long>(S_HASH_V, cap);
  auto* rep = c.get_t<int64_t>(S_SORT_A, n);
  auto* rank = c.get_t<uint64_t>(S_SORT_B, n);
  auto* copy = c.get_t<uint64_t>(S_SORT_C, 3 * uint64_t(n));
  int* bad = static_cast<int*>(c.get(S_FLAGS, 1024)) + 40;
  const uint64_t* p = reinterpret_cast<const uint64_t*>(d_points);
  CK(cudaMemsetAsync(table, 0xff, cap * 8, c.stream));
  CK(cudaMemsetAsync(bad, 0, 4, c.stream));
  k_weld_insert<<<blocks_for(n, 256), 256, 0, c.stream>>>(p, n, table, cap - 1);
  CK_LAUNCH("k_weld_insert");
  k_weld_rep<<<blocks_for(n, 256), 256, 0, c.stream>>>(p, n, table, cap - 1, rep, rank);
  CK_LAUNCH("k_weld_rep");
  const int64_t unique = int64_t(exclusive_scan_u64(c, rank, n, true));  // flags -> ranks of first occurrences
  k_weld_compact<<<blocks_for(n, 256), 256, 0, c.stream>>>(p, n, rep, rank, copy);
  CK_LAUNCH("k_weld_compact");
  if (m) {
    k_weld_remap<<<blocks_for(m, 256), 256, 0, c.stream>>>(d_indices, m, rep, rank, n, bad);
    CK_LAUNCH("k_weld_remap");
  }
  CK(cudaMemcpyAsync(d_points, copy, size_t(unique) * 24, cudaMemcpyDeviceToDevice, c.stream));
  CK(cudaMemcpyAsync(c.h_pinned + 3, bad, 4, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (*reinterpret_cast<int*>(c.h_pinned + 3)) fail(PLMSS_ERR_OUT_OF_RANGE, "point index out of range");
  return unique;
}

void read_volume(Ctx& c, const char* path, const int64_t dims[3], int dtype, int out_f64, void* d_out) {
  if (!path) fail(PLMSS_ERR_INVALID_ARGUMENT, "null path");
  const int64_t n = dims[0] * dims[1] * dims[2];
  if (dims[0] <= 0 || dims[1] <= 0 || dims[2] <= 0) fail(PLMSS_ERR_FORMAT, "volume dims must be positive");
  const size_t elem = dtype_bytes(dtype);
  if (!out_f64 && dtype == PLMSS_DTYPE_F64LE)
    fail(PLMSS_ERR_INVALID_ARGUMENT, "f64le volumes need a float64 destination");
  const uint64_t expected = uint64_t(n) * elem;
  struct stat st;
  if (::stat(path, &st) != 0) fail(PLMSS_ERR_IO, "cannot stat " + std::string(path) + ": " + strerror(errno));
  if (uint64_t(st.st_size) != expected)
    fail(PLMSS_ERR_FORMAT, std::string(path) + ": expected " + std::to_string(expected) + " bytes, got " +
                               std::to_string(uint64_t(st.st_size)));
  File f(path, O_RDONLY, "");
  // two pinned chunks: the file read of one overlaps the copy + conversion
  // of the other
  const size_t chunk = kChunk / 8 * 8;
  unsigned char* stage = c.stage(2 * chunk);
  unsigned char* dev = c.get_t<unsigned char>(S_TMP0, 2 * chunk);
  cudaEvent_t done[2];
  for (auto& e : done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  try {
    uint64_t off = 0;
    for (int k = 0; off < expected; ++k) {
      const int b = k & 1;
      const size_t len = size_t(std::min<uint64_t>(chunk, expected - off));
      CK(cudaEventSynchronize(done[b]));  // buffer b is free again
      // the chunk is read by several threads (one page-cache copy stream is
      // slower than PCIe)
      const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
      const size_t part = (len / nt + 4095) / 4096 * 4096;
      std::vector<std::thread> th;
      std::vector<int> ok(nt, 1);
      for (unsigned t = 0; t < nt; ++t) {
        const size_t p0 = std::min(len, size_t(t) * part), p1 = std::min(len, p0 + part);
        th.emplace_back([&, t, p0, p1] {
          size_t got = p0;
          while (got < p1) {
            const ssize_t r = ::pread(f.fd, stage + b * chunk + got, p1 - got, off_t(off + got));
            if (r < 0 && errno == EINTR) continue;
            if (r <= 0) {
              ok[t] = 0;
              return;
            }
            got += size_t(r);
          }
        });
      }
      for (auto& x : th) x.join();
      for (int v : ok)
        if (!v) fail(PLMSS_ERR_IO, "short read on " + std::string(path));
      CK(cudaMemcpyAsync(dev + b * chunk, stage + b * chunk, len, cudaMemcpyHostToDevice, c.stream));
      const int64_t cnt = int64_t(len / elem), first = int64_t(off / elem);
      void* dst = out_f64 ? static_cast<void*>(static_cast<double*>(d_out) + first)
                          : static_cast<void*>(static_cast<float*>(d_out) + first);
      k_convert_volume<<<blocks_for(cnt, 256), 256, 0, c.stream>>>(dev + b * chunk, cnt, dtype, out_f64, dst);
      CK_LAUNCH("k_convert_volume");
      CK(cudaEventRecord(done[b], c.stream));
      off += len;
    }
    c.sync();
  } catch (...) {
    cudaStreamSynchronize(c.stream);
    for (auto& e : done) cudaEventDestroy(e);
    throw;
  }
  for (auto& e : done) CK(cudaEventDestroy(e));
}

void write_labels(Ctx& c, const char* path, int label_type, const void* d_asc, const void* d_desc, int64_t n) {
  if (!path) fail(PLMSS_ERR_INVALID_ARGUMENT, "null path");
  if (!d_asc || !d_desc || n < 0)
    fail(PLMSS_ERR_INVALID_ARGUMENT, "label output needs matching ascending and descending arrays");
  const size_t w = label_type == 0 ? 4 : 8;
  File f(path, O_WRONLY | O_CREAT | O_TRUNC, " for writing");
  unsigned char head[20] = {'P', 'L', 'M', 'S', 'S', 'L', 'B', 'L', 1, 0, 0, 0};
  for (int i = 0; i < 8; ++i) head[12 + i] = uint8_t(uint64_t(n) >> (8 * i));
  write_all(f.fd, head, sizeof head, path);
  const int64_t per = int64_t(kChunk / 16);
  unsigned char* raw = c.stage(2 * size_t(per) * w);
  std::vector<uint64_t> rec;
  const unsigned nt = host_threads();
  for (int64_t v0 = 0; v0 < n; v0 += per) {
    const int64_t cnt = std::min(per, n - v0);
    CK(cudaMemcpyAsync(raw, static_cast<const char*>(d_asc) + v0 * w, size_t(cnt) * w, cudaMemcpyDeviceToHost,
                       c.stream));
    CK(cudaMemcpyAsync(raw + size_t(per) * w, static_cast<const char*>(d_desc) + v0 * w, size_t(cnt) * w,
                       cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    rec.resize(2 * size_t(cnt));
    auto at = [&](const unsigned char* base, int64_t i) -> uint64_t {
      if (w == 4) return reinterpret_cast<const uint32_t*>(base)[i];
      return reinterpret_cast<const uint64_t*>(base)[i];
    };
    // records packed and written at their file offsets by host threads
    // (little-endian host: a record is the two words themselves)
    const int64_t part = (cnt + nt - 1) / nt;
    on_threads(nt, [&](unsigned t) {
      const int64_t b = std::min(cnt, int64_t(t) * part), e = std::min(cnt, b + part);
      for (int64_t i = b; i < e; ++i) {
        rec[2 * i] = at(raw, i);
        rec[2 * i + 1] = at(raw + size_t(per) * w, i);
      }
      if (e > b) pwrite_all(f.fd, rec.data() + 2 * b, size_t(e - b) * 16, 20 + uint64_t(v0 + b) * 16, path);
    });
  }
}

// The reference OBJ text (io.cpp:268-299) from two chunk fetchers: points
// [p0, p0 + cnt) into host doubles, primitives [q0, q0 + cnt) into host
// indices and region pairs. Formatting on host threads, written in order.
using PointFetch = std::function<void(int64_t, int64_t, double*)>;
using PrimFetch = std::function<void(int64_t, int64_t, int64_t*, int64_t*)>;

static void write_obj_core(Ctx& c, const char* path, int64_t n_points, int64_t n_prims, int verts_per_prim,
                           int64_t point_chunk, int64_t prim_chunk, const PointFetch& fetch_points,
                           const PrimFetch& fetch_prims) {
  File f(path, O_WRONLY | O_CREAT | O_TRUNC, " for writing");
  uint64_t fpos = 0;  // file offset of the next part
  {
    const std::string head = "# separating geometry: " + std::to_string(n_points) + " points, " +
                             std::to_string(n_prims) + (verts_per_prim == 3 ? " triangles\n" : " segments\n");
    write_all(f.fd, head.data(), head.size(), path);
    fpos = head.size();
  }
  const unsigned nthreads = host_threads();
  // format [0, cnt) items of a chunk on nthreads threads, then write in order
  auto parallel_format = [&](int64_t cnt, const std::function<void(int64_t, int64_t, std::string&)>& fmt) {
    std::vector<std::string> parts(nthreads);
    const int64_t per = (cnt + nthreads - 1) / nthreads;
    on_threads(nthreads, [&](unsigned t) {
      const int64_t b = std::min(cnt, int64_t(t) * per), e = std::min(cnt, b + per);
      fmt(b, e, parts[t]);
    });
    std::vector<uint64_t> at(nthreads);
    for (unsigned t = 0; t < nthreads; ++t) {
      at[t] = fpos;
      fpos += parts[t].size();
    }
    on_threads(nthreads, [&](unsigned t) { pwrite_all(f.fd, parts[t].data(), parts[t].size(), at[t], path); });
  };
  // points: "v %.17g %.17g %.17g"
  {
    const int64_t per = point_chunk;
    std::vector<double> hpv(size_t(std::max<int64_t>(per, 1)) * 3);
    const double* hp = hpv.data();
    for (int64_t p0 = 0; p0 < n_points; p0 += per) {
      const int64_t cnt = std::min(per, n_points - p0);
      fetch_points(p0, cnt, hpv.data());
      parallel_format(cnt, [&](int64_t b, int64_t e, std::string& s) {
        char line[96];
        s.reserve(size_t(e - b) * 60);
        for (int64_t i = b; i < e; ++i) {
          const int len = snprintf(line, sizeof line, "v %.17g %.17g %.17g\n", hp[3 * i], hp[3 * i + 1], hp[3 * i + 2]);
          s.append(line, size_t(len));
        }
      });
    }
  }
  // primitives: "g rA[_rB]" whenever the region pair changes, then
  // "f i j k" / "l i j" with 1-based indices
  {
    const int64_t per = prim_chunk;
    const int vp = verts_per_prim;
    std::vector<int64_t> hiv(size_t(std::max<int64_t>(per, 1)) * vp), hrv(size_t(std::max<int64_t>(per, 1)) * 2);
    const int64_t* hi = hiv.data();
    const int64_t* hr = hrv.data();
    int64_t prev[2] = {-2, -2};  // region pair of the primitive before the chunk
    for (int64_t q0 = 0; q0 < n_prims; q0 += per) {
      const int64_t cnt = std::min(per, n_prims - q0);
      fetch_prims(q0, cnt, hiv.data(), hrv.data());
      const int64_t p0a = prev[0], p0b = prev[1];
      parallel_format(cnt, [&](int64_t b, int64_t e, std::string& s) {
        int64_t ca = b ? hr[2 * (b - 1)] : p0a, cb = b ? hr[2 * (b - 1) + 1] : p0b;
        s.reserve(size_t(e - b) * 40);
        char line[96];
        for (int64_t i = b; i < e; ++i) {
          if (hr[2 * i] != ca || hr[2 * i + 1] != cb) {
            ca = hr[2 * i];
            cb = hr[2 * i + 1];
            const int len = cb >= 0 ? snprintf(line, sizeof line, "g r%lld_r%lld\n", (long long)ca, (long long)cb)
                                    : snprintf(line, sizeof line, "g r%lld\n", (long long)ca);
            s.append(line, size_t(len));
          }
          int len = 0;
          if (vp == 3)
            len = snprintf(line, sizeof line, "f %lld %lld %lld\n", (long long)(hi[3 * i] + 1),
                           (long long)(hi[3 * i + 1] + 1), (long long)(hi[3 * i + 2] + 1));
          else
            len = snprintf(line, sizeof line, "l %lld %lld\n", (long long)(hi[2 * i] + 1), (long long)(hi[2 * i + 1] + 1));
          s.append(line, size_t(len));
        }
      });
      prev[0] = hr[2 * (cnt - 1)];
      prev[1] = hr[2 * (cnt - 1) + 1];
    }
  }
}

void write_surface_obj(Ctx& c, const char* path, const double* d_points, int64_t n_points, const int64_t* d_indices,
                       const int64_t* d_regions, int64_t n_prims, int verts_per_prim) {
  if (!path) fail(PLMSS_ERR_INVALID_ARGUMENT, "null path");
  if (verts_per_prim != 2 && verts_per_prim != 3) fail(PLMSS_ERR_INVALID_ARGUMENT, "verts_per_prim must be 2 or 3");
  if (n_points < 0 || n_prims < 0) fail(PLMSS_ERR_INVALID_ARGUMENT, "negative size");
  const int vp = verts_per_prim;
  unsigned char* stage = c.stage(kChunk);
  write_obj_core(
      c, path, n_points, n_prims, vp, int64_t(kChunk / 24), int64_t(kChunk / (8 * vp + 16)),
      [&](int64_t p0, int64_t cnt, double* out) {
        CK(cudaMemcpyAsync(stage, d_points + 3 * p0, size_t(cnt) * 24, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        memcpy(out, stage, size_t(cnt) * 24);
      },
      [&](int64_t q0, int64_t cnt, int64_t* idx, int64_t* reg) {
        CK(cudaMemcpyAsync(stage, d_indices + q0 * vp, size_t(cnt) * vp * 8, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(stage + size_t(cnt) * vp * 8, d_regions + 2 * q0, size_t(cnt) * 16, cudaMemcpyDeviceToHost,
                           c.stream));
        c.sync();
        memcpy(idx, stage, size_t(cnt) * vp * 8);
        memcpy(reg, stage + size_t(cnt) * vp * 8, size_t(cnt) * 16);
      });
}

// The reference write_surface_obj of emit_separators' mesh, streamed from the
// compact records: points materialised on the device chunk by chunk
// (marching.cu materialize), faces are the identity soup (3j, 3j+1, 3j+2),
// regions from the records — the SeparatingMesh (marching.hpp:65-76) is
// never held whole, on the device or on the host.
void write_separators_obj(Ctx& c, const char* path, const Grid& g, const double* sp, const double* og,
                          int label_type, const void* d_tris, int64_t n) {
  if (!path) fail(PLMSS_ERR_INVALID_ARGUMENT, "null path");
  if (n < 0 || (n > 0 && !d_tris)) fail(PLMSS_ERR_INVALID_ARGUMENT, "bad separator records");
  const size_t rec = label_type == 0 ? sizeof(plmss_tri) : sizeof(plmss_tri64);
  const int64_t per_tri = int64_t(kChunk / 72);  // triangles per points chunk
  double* d_pts = c.get_t<double>(S_TMP2, size_t(per_tri) * 9);
  int64_t* d_reg = c.get_t<int64_t>(S_SCAN_C, size_t(per_tri) * 2);
  unsigned char* stage = c.stage(kChunk);
  write_obj_core(
      c, path, 3 * n, n, 3, 3 * per_tri, per_tri,
      [&](int64_t p0, int64_t cnt, double* out) {  // p0, cnt: multiples of 3 except at the end
        const int64_t t0 = p0 / 3, tn = (cnt + 2) / 3;
        materialize(c, g, sp, og, label_type, static_cast<const char*>(d_tris) + size_t(t0) * rec, tn, d_pts, nullptr,
                    nullptr);
        CK(cudaMemcpyAsync(stage, d_pts, size_t(cnt) * 24, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        memcpy(out, stage, size_t(cnt) * 24);
      },
      [&](int64_t q0, int64_t cnt, int64_t* idx, int64_t* reg) {
        materialize(c, g, sp, og, label_type, static_cast<const char*>(d_tris) + size_t(q0) * rec, cnt, nullptr, d_reg,
                    nullptr);
        CK(cudaMemcpyAsync(stage, d_reg, size_t(cnt) * 16, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        memcpy(reg, stage, size_t(cnt) * 16);
        for (int64_t i = 0; i < 3 * cnt; ++i) idx[i] = 3 * q0 + i;
      });
}

// The SeparatingMesh arrays of the records, chunk by chunk into a host sink:
// device materialisation of chunk k+1 and its copy overlap the sink's work
// on chunk k (two pinned buffers).
void materialize_chunks(Ctx& c, const Grid& g, const double* sp, const double* og, int label_type,
                        const void* d_tris, int64_t n, int64_t chunk, plmss_geometry_sink sink, void* user) {
  if (!sink) fail(PLMSS_ERR_INVALID_ARGUMENT, "null sink");
  if (n < 0 || (n > 0 && !d_tris)) fail(PLMSS_ERR_INVALID_ARGUMENT, "bad separator records");
  if (chunk <= 0) chunk = int64_t(1) << 22;
  chunk = std::min(chunk, std::max<int64_t>(n, 1));
  const size_t rec = label_type == 0 ? sizeof(plmss_tri) : sizeof(plmss_tri64);
  const size_t per = size_t(chunk) * (72 + 16 + 8);  // points, regions, cells per triangle
  char* dbuf = static_cast<char*>(c.get(S_TMP2, 2 * per));
  char* hbuf = nullptr;
  CK(cudaMallocHost(reinterpret_cast<void**>(&hbuf), 2 * per));
  cudaEvent_t ev[2] = {};
  int status = 0;
  try {
    for (int k = 0; k < 2; ++k) CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    auto parts = [&](char* base, int64_t cnt, double*& p, int64_t*& r, int64_t*& cl) {
      p = reinterpret_cast<double*>(base);
      r = reinterpret_cast<int64_t*>(base + size_t(cnt) * 72);
      cl = reinterpret_cast<int64_t*>(base + size_t(cnt) * 88);
    };
    const int64_t nch = (n + chunk - 1) / chunk;
    for (int64_t k = 0; k <= nch && status == 0; ++k) {
      if (k < nch) {
        const int64_t t0 = k * chunk, cnt = std::min(chunk, n - t0);
        const int s = int(k & 1);
        double* p;
        int64_t *r, *cl;
        parts(dbuf + s * per, cnt, p, r, cl);
        materialize(c, g, sp, og, label_type, static_cast<const char*>(d_tris) + size_t(t0) * rec, cnt, p, r, cl);
        CK(cudaMemcpyAsync(hbuf + s * per, dbuf + s * per, size_t(cnt) * 96, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaEventRecord(ev[s], c.stream));
      }
      if (k >= 1) {  // hand chunk k-1 to the sink while chunk k is in flight
        const int64_t t0 = (k - 1) * chunk, cnt = std::min(chunk, n - t0);
        const int s = int((k - 1) & 1);
        CK(cudaEventSynchronize(ev[s]));
        double* p;
        int64_t *r, *cl;
        parts(hbuf + s * per, cnt, p, r, cl);
        status = sink(user, t0, cnt, p, r, cl);
      }
    }
    c.sync();
  } catch (...) {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    cudaFreeHost(hbuf);
    throw;
  }
  for (auto e : ev) cudaEventDestroy(e);
  CK(cudaFreeHost(hbuf));
  if (status) fail(PLMSS_ERR_LOGIC, "geometry sink stopped the stream (status " + std::to_string(status) + ")");
}

}  // namespace plmss_b200
