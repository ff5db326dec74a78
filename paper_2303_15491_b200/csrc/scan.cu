// Device-wide primitives: exclusive scan (uint64) and stable LSD radix sort
// of (uint64 key, uint64 value) pairs. Hand-written; no CUB.
#include "common.cuh"

namespace plmss_b200 {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total.
template <int THREADS>
__device__ __forceinline__ void block_excl_scan(uint64_t v, uint64_t& excl) {
  __shared__ uint64_t warp_tot[THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t inc = warp_incl_scan(v);
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint64_t t = lane < THREADS / 32 ? warp_tot[lane] : 0;
    uint64_t ti = warp_incl_scan(t);
    if (lane < THREADS / 32) warp_tot[lane] = ti - t;
  }
  __syncthreads();
  excl = inc - v + warp_tot[w];
  __syncthreads();
}

// Scans each tile in place (exclusive) and writes the tile total.
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(uint64_t* data, int64_t n, uint64_t* tile_tot) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
  uint64_t v[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? data[base + i] : 0;
    s += v[i];
  }
  __shared__ uint64_t last_incl;
  uint64_t excl;
  block_excl_scan<kScanThreads>(s, excl);
  if (threadIdx.x == kScanThreads - 1) last_incl = excl + s;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) data[base + i] = excl;
    excl += v[i];
  }
  if (threadIdx.x == 0 && tile_tot) tile_tot[blockIdx.x] = last_incl;
}

__global__ void k_add_offsets(uint64_t* data, int64_t n, const uint64_t* tile_off) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) data[i] += tile_off[i / kScanTile];
}

void scan_rec(Ctx& c, uint64_t* data, int64_t n, int depth) {
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles <= 1) {
    k_scan_tiles<<<1, kScanThreads, 0, c.stream>>>(data, n, nullptr);
    CK_LAUNCH("k_scan_tiles");
    return;
  }
  Slot slot = depth == 0 ? S_SCAN_A : (depth == 1 ? S_SCAN_B : S_SCAN_C);
  if (depth > 2) fail(PLMSS_ERR_LOGIC, "scan too deep");
  uint64_t* tot = c.get_t<uint64_t>(slot, tiles);
  k_scan_tiles<<<(unsigned)tiles, kScanThreads, 0, c.stream>>>(data, n, tot);
  CK_LAUNCH("k_scan_tiles");
  scan_rec(c, tot, tiles, depth + 1);
  k_add_offsets<<<blocks_for(n, 256), 256, 0, c.stream>>>(data, n, tot);
  CK_LAUNCH("k_add_offsets");
}

// ------------------------------------------------------------ radix sort --
constexpr int kSortThreads = 256;
constexpr int kSortRows = 8;  // keys per thread (striped)
constexpr int kSortTile = kSortThreads * kSortRows;

__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const uint64_t* keys, int64_t n, int shift,
                                                             uint64_t* counts, int64_t nblocks) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kSortTile;
#pragma unroll
  for (int r = 0; r < kSortRows; ++r) {
    int64_t i = base + r * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  counts[int64_t(threadIdx.x) * nblocks + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const uint64_t* keys_in, const uint64_t* vals_in,
                                                                uint64_t* keys_out, uint64_t* vals_out,
                                                                int64_t n, int shift, const uint64_t* offsets,
                                                                int64_t nblocks) {
  __shared__ uint32_t warp_cnt[kSortThreads / 32][256];
  __shared__ uint64_t digit_base[256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  digit_base[threadIdx.x] = offsets[int64_t(threadIdx.x) * nblocks + blockIdx.x];
  const int64_t base = int64_t(blockIdx.x) * kSortTile;
  for (int r = 0; r < kSortRows; ++r) {
    for (int k = threadIdx.x; k < (kSortThreads / 32) * 256; k += kSortThreads) (&warp_cnt[0][0])[k] = 0;
    __syncthreads();
    const int64_t i = base + r * kSortThreads + threadIdx.x;
    const bool valid = i < n;
    uint64_t key = valid ? keys_in[i] : 0;
    uint64_t val = valid ? vals_in[i] : 0;
    const unsigned d = valid ? unsigned((key >> shift) & 255) : 256u;  // 256 = invalid group
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned below = peers & ((1u << lane) - 1);
    const int rank_in_warp = __popc(below);
    if (valid && below == 0) warp_cnt[w][d] = __popc(peers);
    __syncthreads();
    // thread t = digit t: exclusive prefix over warps, then advance the base.
    {
      const int dg = threadIdx.x;
      uint32_t run = 0;
#pragma unroll
      for (int ww = 0; ww < kSortThreads / 32; ++ww) {
        uint32_t t = warp_cnt[ww][dg];
        warp_cnt[ww][dg] = run;
        run += t;
      }
      // digit_base updated after everyone read it below; stash row total.
      __syncthreads();
      if (valid) {
        uint64_t dst = digit_base[d] + warp_cnt[w][d] + rank_in_warp;
        keys_out[dst] = key;
        vals_out[dst] = val;
      }
      __syncthreads();
      digit_base[dg] += run;
    }
    __syncthreads();
  }
}

}  // namespace

uint64_t exclusive_scan_u64(Ctx& c, uint64_t* data, int64_t n, bool want_total) {
  if (n <= 0) return 0;
  uint64_t last = 0;
  if (want_total) {
    CK(cudaMemcpyAsync(c.h_pinned, data + n - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.stream));
  }
  scan_rec(c, data, n, 0);
  if (want_total) {
    CK(cudaMemcpyAsync(c.h_pinned + 1, data + n - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    last = c.h_pinned[0] + c.h_pinned[1];
  }
  return last;
}

void radix_sort_pairs(Ctx& c, uint64_t* keys, uint64_t* vals, int64_t n, int bits) {
  if (n <= 1 || bits <= 0) return;
  const int64_t nblocks = (n + kSortTile - 1) / kSortTile;
  uint64_t* k2 = c.get_t<uint64_t>(S_SORT_C, n);
  uint64_t* v2 = c.get_t<uint64_t>(S_SORT_D, n);
  uint64_t* counts = c.get_t<uint64_t>(S_TMP2, 256 * nblocks);
  uint64_t *ka = keys, *va = vals, *kb = k2, *vb = v2;
  const int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    k_radix_hist<<<(unsigned)nblocks, kSortThreads, 0, c.stream>>>(ka, n, shift, counts, nblocks);
    CK_LAUNCH("k_radix_hist");
    exclusive_scan_u64(c, counts, 256 * nblocks, false);
    k_radix_scatter<<<(unsigned)nblocks, kSortThreads, 0, c.stream>>>(ka, va, kb, vb, n, shift, counts, nblocks);
    CK_LAUNCH("k_radix_scatter");
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (ka != keys) {
    CK(cudaMemcpyAsync(keys, ka, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, c.stream));
    CK(cudaMemcpyAsync(vals, va, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, c.stream));
  }
}

}  // namespace plmss_b200
