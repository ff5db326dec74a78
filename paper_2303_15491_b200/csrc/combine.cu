// K3: Morse-Smale region ids with dense compaction.
//
// Reference (segmentation.cpp:170-196): key = (asc << 64 | desc), region
// table = sorted unique keys, region id = lower_bound index. Here the pair is
// first mapped to its order-preserving compressed index
//     k(v) = rank_min(asc[v]) * n_max + rank_max(desc[v])  in [0, n_min*n_max)
// (ranks = positions in the sorted extremum lists, so (asc, desc)
// lexicographic order == k order). Distinct k are then found either
//   * with a bitmap over [0, n_min*n_max) when that fits (smooth fields):
//     region id = popcount prefix of the bitmap, no sort at all; or
//   * with an open-addressing hash table + radix sort of the R unique keys
//     (noise-like fields where n_min*n_max is huge).
// Both produce exactly the reference's dense ids and region table.
#include "common.cuh"

namespace plmss_b200 {
namespace {

constexpr uint64_t kEmpty = ~uint64_t(0);
constexpr int64_t kBitmapMaxBits = int64_t(1) << 31;

__device__ __forceinline__ uint64_t pair_index(uint32_t v, const uint32_t* __restrict__ asc,
                                               const uint32_t* __restrict__ desc,
                                               const uint32_t* __restrict__ rmin,
                                               const uint32_t* __restrict__ rmax, uint64_t n_max) {
  const uint32_t a = asc[v], d = desc[v];
  return uint64_t(__ldg(rmin + a)) * n_max + __ldg(rmax + d);
}

__global__ void __launch_bounds__(256) k_mark_bitmap(uint32_t n, const uint32_t* __restrict__ asc,
                                                     const uint32_t* __restrict__ desc,
                                                     const uint32_t* __restrict__ rmin,
                                                     const uint32_t* __restrict__ rmax, uint64_t n_max,
                                                     uint32_t* __restrict__ bm) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = v < n;
  const uint64_t k = ok ? pair_index(v, asc, desc, rmin, rmax, n_max) : kEmpty;
  const unsigned peers = __match_any_sync(0xffffffffu, k);
  const int lane = threadIdx.x & 31;
  if (ok && (peers & ((1u << lane) - 1)) == 0) {
    const uint32_t bit = 1u << (k & 31);
    uint32_t* w = bm + (k >> 5);
    if ((*w & bit) == 0) atomicOr(w, bit);
  }
}

__global__ void k_word_popc(const uint32_t* __restrict__ bm, int64_t words, uint64_t* __restrict__ pc) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < words) pc[i] = __popc(bm[i]);
}

__global__ void __launch_bounds__(256) k_assign_bitmap(uint32_t n, const uint32_t* __restrict__ asc,
                                                       const uint32_t* __restrict__ desc,
                                                       const uint32_t* __restrict__ rmin,
                                                       const uint32_t* __restrict__ rmax, uint64_t n_max,
                                                       const uint32_t* __restrict__ bm,
                                                       const uint64_t* __restrict__ pre,
                                                       uint32_t* __restrict__ ms) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const uint64_t k = pair_index(v, asc, desc, rmin, rmax, n_max);
  const uint64_t w = k >> 5;
  const uint32_t below = __ldg(bm + w) & ((1u << (k & 31)) - 1u);
  ms[v] = static_cast<uint32_t>(__ldg(pre + w) + __popc(below));
}

__global__ void k_bitmap_keys(const uint32_t* __restrict__ bm, int64_t words, const uint64_t* __restrict__ pre,
                              const uint32_t* __restrict__ minima, const uint32_t* __restrict__ maxima,
                              uint64_t n_max, uint64_t* __restrict__ keys) {
  const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= words) return;
  uint32_t bits = bm[w];
  uint64_t id = pre[w];
  while (bits) {
    const int b = __ffs(bits) - 1;
    bits &= bits - 1;
    const uint64_t k = uint64_t(w) * 32 + b;
    keys[id++] = (uint64_t(minima[k / n_max]) << 32) | maxima[k % n_max];
  }
}

// ---------------------------------------------------------------- hash ---
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

__global__ void __launch_bounds__(256) k_hash_insert(uint32_t n, const uint32_t* __restrict__ asc,
                                                     const uint32_t* __restrict__ desc,
                                                     const uint32_t* __restrict__ rmin,
                                                     const uint32_t* __restrict__ rmax, uint64_t n_max,
                                                     unsigned long long* __restrict__ table, uint64_t mask,
                                                     int* __restrict__ overflow) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = v < n;
  const uint64_t k = ok ? pair_index(v, asc, desc, rmin, rmax, n_max) : kEmpty;
  const unsigned peers = __match_any_sync(0xffffffffu, k);
  const int lane = threadIdx.x & 31;
  if (!ok || (peers & ((1u << lane) - 1)) != 0) return;
  uint64_t s = mix64(k) & mask;
  for (uint64_t probe = 0; probe <= mask; ++probe) {
    const unsigned long long cur = table[s];
    if (cur == k) return;
    if (cur == kEmpty) {
      const unsigned long long prev = atomicCAS(table + s, kEmpty, k);
      if (prev == kEmpty || prev == k) return;
    }
    s = (s + 1) & mask;
    if (probe > 4096) break;
  }
  *overflow = 1;
}

__device__ __forceinline__ uint64_t hash_find(const unsigned long long* __restrict__ table, uint64_t mask,
                                              uint64_t k) {
  uint64_t s = mix64(k) & mask;
  while (table[s] != k) s = (s + 1) & mask;
  return s;
}

constexpr int kCThreads = 256;
constexpr int kCRows = 16;
constexpr int kCTile = kCThreads * kCRows;

__global__ void __launch_bounds__(kCThreads) k_count_occupied(const unsigned long long* __restrict__ t,
                                                              int64_t n, uint64_t* __restrict__ counts) {
  const int64_t base = int64_t(blockIdx.x) * kCTile;
  uint32_t c = 0;
  for (int r = 0; r < kCRows; ++r) {
    const int64_t i = base + r * kCThreads + threadIdx.x;
    if (i < n && t[i] != kEmpty) ++c;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[kCThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kCThreads / 32; ++w) s += ws[w];
    counts[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kCThreads) k_write_occupied(const unsigned long long* __restrict__ t,
                                                              int64_t n, const uint64_t* __restrict__ off,
                                                              uint64_t* __restrict__ keys,
                                                              uint64_t* __restrict__ slots) {
  __shared__ uint32_t wc[kCThreads / 32];
  __shared__ uint32_t wp[kCThreads / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = int64_t(blockIdx.x) * kCTile;
  uint64_t running = off[blockIdx.x];
  for (int r = 0; r < kCRows; ++r) {
    const int64_t i = base + r * kCThreads + threadIdx.x;
    const unsigned long long k = i < n ? t[i] : kEmpty;
    const bool hit = k != kEmpty;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wc[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int q = 0; q < kCThreads / 32; ++q) {
        wp[q] = s;
        s += wc[q];
      }
      wp[kCThreads / 32] = s;
    }
    __syncthreads();
    if (hit) {
      const uint64_t pos = running + wp[w] + __popc(m & ((1u << lane) - 1));
      keys[pos] = k;
      slots[pos] = static_cast<uint64_t>(i);
    }
    running += wp[kCThreads / 32];
    __syncthreads();
  }
}

__global__ void k_hash_set_ids(const uint64_t* __restrict__ sorted_slots, int64_t r,
                               uint32_t* __restrict__ slot_id) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < r) slot_id[sorted_slots[i]] = static_cast<uint32_t>(i);
}

__global__ void __launch_bounds__(256) k_hash_assign(uint32_t n, const uint32_t* __restrict__ asc,
                                                     const uint32_t* __restrict__ desc,
                                                     const uint32_t* __restrict__ rmin,
                                                     const uint32_t* __restrict__ rmax, uint64_t n_max,
                                                     const unsigned long long* __restrict__ table,
                                                     uint64_t mask, const uint32_t* __restrict__ slot_id,
                                                     uint32_t* __restrict__ ms) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const uint64_t k = pair_index(v, asc, desc, rmin, rmax, n_max);
  ms[v] = slot_id[hash_find(table, mask, k)];
}

__global__ void k_keys_from_sorted(const uint64_t* __restrict__ sk, int64_t r, const uint32_t* __restrict__ minima,
                                   const uint32_t* __restrict__ maxima, uint64_t n_max,
                                   uint64_t* __restrict__ keys) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < r) keys[i] = (uint64_t(minima[sk[i] / n_max]) << 32) | maxima[sk[i] % n_max];
}

int bit_length(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

}  // namespace

int64_t combine_ms(Ctx& c, int64_t n, const uint32_t* asc, const uint32_t* desc, uint32_t* ms,
                   const std::function<uint64_t*(int64_t)>& get_keys, const uint32_t* minima, int64_t n_min, const uint32_t* maxima, int64_t n_max,
                   const uint32_t* rank_min, const uint32_t* rank_max) {
  if (n <= 0) return 0;
  const uint32_t nn = static_cast<uint32_t>(n);
  const unsigned nb = blocks_for(n, 256);
  const uint64_t P = uint64_t(n_min) * uint64_t(n_max);
  const bool bitmap = c.combine_path == 1 || (c.combine_path == 0 && P <= uint64_t(kBitmapMaxBits));
  if (c.combine_path == 1 && P > uint64_t(kBitmapMaxBits) * 4)
    fail(PLMSS_ERR_INVALID_ARGUMENT, "bitmap combine path forced but n_min * n_max is too large");
  if (bitmap) {
    const int64_t words = static_cast<int64_t>((P + 31) / 32);
    uint32_t* bm = c.get_t<uint32_t>(S_BITMAP, words);
    uint64_t* pre = c.get_t<uint64_t>(S_HASH_K, words);
    CK(cudaMemsetAsync(bm, 0, words * sizeof(uint32_t), c.stream));
    k_mark_bitmap<<<nb, 256, 0, c.stream>>>(nn, asc, desc, rank_min, rank_max, n_max, bm);
    CK_LAUNCH("k_mark_bitmap");
    k_word_popc<<<blocks_for(words, 256), 256, 0, c.stream>>>(bm, words, pre);
    CK_LAUNCH("k_word_popc");
    const int64_t R = static_cast<int64_t>(exclusive_scan_u64(c, pre, words, true));
    if (ms) {
      k_assign_bitmap<<<nb, 256, 0, c.stream>>>(nn, asc, desc, rank_min, rank_max, n_max, bm, pre, ms);
      CK_LAUNCH("k_assign_bitmap");
    }
    uint64_t* keys = get_keys(R);
    if (keys) {
      k_bitmap_keys<<<blocks_for(words, 256), 256, 0, c.stream>>>(bm, words, pre, minima, maxima, n_max, keys);
      CK_LAUNCH("k_bitmap_keys");
    }
    return R;
  }
  // Hash path.
  int* overflow = static_cast<int*>(c.get(S_FLAGS, 64));
  uint64_t cap = 1024;
  const uint64_t start = std::min<uint64_t>(uint64_t(n), uint64_t(1) << 24) * 2;
  while (cap < start) cap <<= 1;
  unsigned long long* table = nullptr;
  for (;;) {
    table = c.get_t<unsigned long long>(S_HASH_K, cap);
    CK(cudaMemsetAsync(table, 0xff, cap * sizeof(uint64_t), c.stream));
    CK(cudaMemsetAsync(overflow, 0, sizeof(int), c.stream));
    k_hash_insert<<<nb, 256, 0, c.stream>>>(nn, asc, desc, rank_min, rank_max, n_max, table, cap - 1, overflow);
    CK_LAUNCH("k_hash_insert");
    CK(cudaMemcpyAsync(c.h_pinned, overflow, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (*reinterpret_cast<int*>(c.h_pinned) == 0) break;
    if (cap >= 4 * uint64_t(n)) fail(PLMSS_ERR_LOGIC, "region hash table overflow");
    cap <<= 2;
  }
  const int64_t tb = static_cast<int64_t>((cap + kCTile - 1) / kCTile);
  uint64_t* counts = c.get_t<uint64_t>(S_TMP1, tb);
  k_count_occupied<<<(unsigned)tb, kCThreads, 0, c.stream>>>(table, cap, counts);
  CK_LAUNCH("k_count_occupied");
  const int64_t R = static_cast<int64_t>(exclusive_scan_u64(c, counts, tb, true));
  uint64_t* uk = c.get_t<uint64_t>(S_SORT_A, R);
  uint64_t* us = c.get_t<uint64_t>(S_SORT_B, R);
  k_write_occupied<<<(unsigned)tb, kCThreads, 0, c.stream>>>(table, cap, counts, uk, us);
  CK_LAUNCH("k_write_occupied");
  radix_sort_pairs(c, uk, us, R, bit_length(P - 1));
  uint32_t* slot_id = c.get_t<uint32_t>(S_HASH_V, cap);
  k_hash_set_ids<<<blocks_for(R, 256), 256, 0, c.stream>>>(us, R, slot_id);
  CK_LAUNCH("k_hash_set_ids");
  if (ms) {
    k_hash_assign<<<nb, 256, 0, c.stream>>>(nn, asc, desc, rank_min, rank_max, n_max, table, cap - 1, slot_id, ms);
    CK_LAUNCH("k_hash_assign");
  }
  uint64_t* keys = get_keys(R);
  if (keys) {
    k_keys_from_sorted<<<blocks_for(R, 256), 256, 0, c.stream>>>(uk, R, minima, maxima, n_max, keys);
    CK_LAUNCH("k_keys_from_sorted");
  }
  return R;
}

}  // namespace plmss_b200
