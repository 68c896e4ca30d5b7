// Unique-color reduction for large images (reference: build_histogram,
// histogram.hpp:65-99) as a partitioned histogram: no global atomics, no
// 128 MiB bin table, no scattered bitmap ORs.
//
//   H1 k_part_count    source block s (a contiguous range of R pixels) counts
//                      its pixels per bucket = Morton code >> 13 (2048
//                      buckets of 8192 bins) in shared memory -> cnt[s][b]
//   H2 k_part_scan     bucket-major exclusive scan -> off[s][b] (where source
//                      block s writes bucket b) and bucket starts
//   H3 k_part_scatter  each pixel becomes one 32-bit entry in its bucket:
//                      (pixel - s*R) << 13 | low 13 Morton bits
//   H4 k_part_build    one CTA per bucket: a shared-memory table of its 8192
//                      bins {count, first pixel} from its entries (shared
//                      atomics), then the non-empty bins in Morton order ->
//                      samples {key, count, first pixel} (decoupled look-back
//                      across buckets for the output offset), and first[bin]
//                      into the 2^24-entry first-pixel table
//   H5 k_first_flags   pixel i is a first occurrence iff first[bin(i)] == i:
//                      the P-bit first-occurrence bitmap, written word by word
//
// The samples come out in the same Morton order as the bin-table path
// (k_bins_compact), carrying their first pixel index instead of their
// first-occurrence rank; ranks follow from the bitmap's prefix popcounts
// (k_bitmap_scan), and only where needed: init_centers' K chosen ranks
// (k_select_ranks) and the build_histogram API (k_rank_from_bitmap). The
// empty-cluster reseed compares first pixels, which orders samples exactly as
// their ranks do.
#pragma once
#include "common.cuh"
#include "hist.cuh"

namespace cqb {

constexpr int PB_BITS = 11;                        // buckets: Morton code >> PB_SUB
constexpr int PB_N = 1 << PB_BITS;                 // 2048
constexpr int PB_SUB = 24 - PB_BITS;               // 13: bins per bucket = 8192
constexpr int PB_BINS = 1 << PB_SUB;
constexpr int PB_LOCAL = 32 - PB_SUB;              // 19 bits of pixel offset per source block
constexpr uint64_t PB_RANGE_MAX = 1ull << PB_LOCAL;
constexpr int PB_THREADS = 1024;                   // H1 / H3 / H5
constexpr int PB_BUILD_THREADS = 512;              // H4
constexpr size_t PB_BUILD_SMEM = 2 * PB_BINS * sizeof(uint32_t);  // count + first per bin

// Source blocks: at least one per SM, each at most 2^19 pixels (multiples of
// 16 pixels, the vector-load chunk).
struct PartGeom {
  uint32_t blocks;
  uint64_t range;
};
inline PartGeom part_geom(uint64_t P, int num_sms) {
  uint64_t g = std::max<uint64_t>((uint64_t)num_sms, (P + PB_RANGE_MAX - 1) / PB_RANGE_MAX);
  uint64_t r = ((P + g - 1) / g + 15) / 16 * 16;
  g = (P + r - 1) / r;
  return PartGeom{(uint32_t)std::max<uint64_t>(g, 1), r};
}

__device__ __forceinline__ uint32_t part_bucket(uint32_t m) { return m >> PB_SUB; }

// H1
__global__ void __launch_bounds__(PB_THREADS) k_part_count(const uint8_t* __restrict__ img, uint64_t P, uint64_t R,
                                                           uint32_t* __restrict__ cnt) {
  __shared__ uint32_t h[PB_N];
  for (int b = threadIdx.x; b < PB_N; b += PB_THREADS) h[b] = 0u;
  __syncthreads();
  const uint64_t p0 = (uint64_t)blockIdx.x * R, p1 = min(P, p0 + R);
  for (uint64_t c = p0 / PX_PER_THREAD + threadIdx.x; c * PX_PER_THREAD < p1; c += PB_THREADS) {
    uint32_t keys[PX_PER_THREAD];
    const int n = load_chunk_keys(img, p1, c, keys);
    uint32_t cur = part_bucket(morton_of_key(keys[0])), run = 1;
#pragma unroll
    for (int s = 1; s < PX_PER_THREAD; ++s) {
      if (s < n) {
        const uint32_t b = part_bucket(morton_of_key(keys[s]));
        if (b == cur) {
          ++run;
        } else {
          atomicAdd(&h[cur], run);
          cur = b;
          run = 1;
        }
      }
    }
    atomicAdd(&h[cur], run);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < PB_N; b += PB_THREADS) cnt[(size_t)blockIdx.x * PB_N + b] = h[b];
}

// H2: one CTA of PB_THREADS; thread t owns buckets t, t + PB_THREADS.
// off[s][b] = start[b] + sum_{s' < s} cnt[s'][b]; start[PB_N] = P.
__global__ void __launch_bounds__(PB_THREADS) k_part_scan(const uint32_t* __restrict__ cnt, uint32_t blocks,
                                                          uint32_t* __restrict__ off, uint32_t* __restrict__ start) {
  constexpr int PER = PB_N / PB_THREADS;
  __shared__ uint32_t warp_tot[PB_THREADS / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  uint32_t tot[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) tot[q] = 0u;
#pragma unroll 4
  for (uint32_t s = 0; s < blocks; ++s)
#pragma unroll
    for (int q = 0; q < PER; ++q) tot[q] += cnt[(size_t)s * PB_N + q * PB_THREADS + t];
  // exclusive scan over buckets in order b = q * PB_THREADS + t
  uint32_t base = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    uint32_t incl = tot[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    uint32_t before = 0, all = 0;
    for (int w = 0; w < PB_THREADS / 32; ++w) {
      const uint32_t v = warp_tot[w];
      before += w < wid ? v : 0u;
      all += v;
    }
    const uint32_t st = base + before + incl - tot[q];
    start[q * PB_THREADS + t] = st;
    tot[q] = st;  // becomes the running offset
    base += all;
    __syncthreads();
  }
  if (t == 0) start[PB_N] = base;
#pragma unroll 4
  for (uint32_t s = 0; s < blocks; ++s)
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const size_t i = (size_t)s * PB_N + q * PB_THREADS + t;
      const uint32_t c = cnt[i];
      off[i] = tot[q];
      tot[q] += c;
    }
}

// H3
__global__ void __launch_bounds__(PB_THREADS) k_part_scatter(const uint8_t* __restrict__ img, uint64_t P, uint64_t R,
                                                             const uint32_t* __restrict__ off,
                                                             uint32_t* __restrict__ entries) {
  __shared__ uint32_t cur[PB_N];
  for (int b = threadIdx.x; b < PB_N; b += PB_THREADS) cur[b] = off[(size_t)blockIdx.x * PB_N + b];
  __syncthreads();
  const uint64_t p0 = (uint64_t)blockIdx.x * R, p1 = min(P, p0 + R);
  for (uint64_t c = p0 / PX_PER_THREAD + threadIdx.x; c * PX_PER_THREAD < p1; c += PB_THREADS) {
    uint32_t keys[PX_PER_THREAD];
    const int n = load_chunk_keys(img, p1, c, keys);
    const uint32_t local0 = (uint32_t)(c * PX_PER_THREAD - p0);
#pragma unroll
    for (int s = 0; s < PX_PER_THREAD; ++s) {
      if (s < n) {
        const uint32_t m = morton_of_key(keys[s]);
        const uint32_t pos = atomicAdd(&cur[part_bucket(m)], 1u);
        entries[pos] = ((local0 + s) << PB_SUB) | (m & (PB_BINS - 1));
      }
    }
  }
}

// H4: one CTA per bucket, taken in ticket order (the look-back needs every
// earlier bucket's CTA to have started).
__global__ void __launch_bounds__(PB_BUILD_THREADS) k_part_build(
    const uint32_t* __restrict__ entries, const uint32_t* __restrict__ off, const uint32_t* __restrict__ start,
    uint32_t blocks, uint64_t R, uint32_t* __restrict__ m_keys, uint32_t* __restrict__ m_counts,
    uint32_t* __restrict__ m_first, uint32_t* __restrict__ first_tab, unsigned long long* tile_state,
    unsigned int* ticket, unsigned long long* n_unique) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* cnt = sm;              // [PB_BINS]
  uint32_t* fst = sm + PB_BINS;    // [PB_BINS]
  constexpr int NW = PB_BUILD_THREADS / 32;
  __shared__ uint32_t s_bucket, s_prefix;
  __shared__ uint32_t s_warp[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_bucket = atomicAdd(ticket, 1u);
  for (int i = tid; i < PB_BINS; i += PB_BUILD_THREADS) {
    cnt[i] = 0u;
    fst[i] = 0xFFFFFFFFu;
  }
  __syncthreads();
  const uint32_t bucket = s_bucket;
  // entries: one segment per source block, warp-strided over the segments
  for (uint32_t s = wid; s < blocks; s += NW) {
    const uint32_t lo = off[(size_t)s * PB_N + bucket];
    const uint32_t hi = s + 1 < blocks ? off[(size_t)(s + 1) * PB_N + bucket] : start[bucket + 1];
    const uint32_t base = (uint32_t)((uint64_t)s * R);
    for (uint32_t e = lo + lane; e < hi; e += 32) {
      const uint32_t v = entries[e];
      const uint32_t bin = v & (PB_BINS - 1);
      atomicAdd(&cnt[bin], 1u);
      atomicMin(&fst[bin], base + (v >> PB_SUB));
    }
  }
  __syncthreads();
  // emission in Morton order, coalesced: PER rounds of PB_BUILD_THREADS
  // consecutive bins; the bucket's total first (for the look-back)
  constexpr int PER = PB_BINS / PB_BUILD_THREADS;  // 16
  uint32_t mine = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) mine += cnt[q * PB_BUILD_THREADS + tid] != 0u;
  mine = warp_sum(mine);
  if (lane == 0) s_warp[wid] = mine;
  __syncthreads();
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) total += s_warp[w];
  if (wid == 0) {  // decoupled look-back over the earlier buckets
    uint32_t prefix = 0;
    if (bucket == 0) {
      if (lane == 0) atomicExch(tile_state, LB_PRE | total);
    } else {
      if (lane == 0) atomicExch(tile_state + bucket, LB_AGG | total);
      int j = (int)bucket - 1;
      while (true) {
        const int idx = j - lane;
        unsigned long long st = idx >= 0 ? lb_load(tile_state + idx) : (LB_PRE | 0ull);
        while (__any_sync(0xffffffffu, (st >> 32) == 0)) {
          if ((st >> 32) == 0) st = lb_load(tile_state + idx);
        }
        const uint32_t pmask = __ballot_sync(0xffffffffu, (st >> 32) == 2);
        const uint32_t val = (uint32_t)st;
        if (pmask) {
          const int first_p = __ffs(pmask) - 1;
          prefix += warp_sum(lane <= first_p ? val : 0u);
          break;
        }
        prefix += warp_sum(val);
        j -= 32;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(tile_state + bucket, LB_PRE | (prefix + total));
      }
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t running = s_prefix;
  const uint32_t mbase = bucket << PB_SUB;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll 1
  for (int q = 0; q < PER; ++q) {
    const uint32_t bin = q * PB_BUILD_THREADS + tid;
    const uint32_t c = cnt[bin];
    const unsigned bal = __ballot_sync(0xffffffffu, c != 0u);
    __syncthreads();  // s_warp reuse
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    uint32_t before = 0, round = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t v = s_warp[w];
      before += w < wid ? v : 0u;
      round += v;
    }
    if (c) {
      const uint32_t pos = running + before + __popc(bal & lt);
      const uint32_t f = fst[bin];
      m_keys[pos] = key_of_morton(mbase + bin);
      m_counts[pos] = c;
      m_first[pos] = f;
      if (first_tab) first_tab[mbase + bin] = f;
    }
    running += round;
  }
  if (bucket == PB_N - 1 && tid == 0) *n_unique = (unsigned long long)(s_prefix + total);
}

// H5: thread w builds bitmap word w (pixels 32w .. 32w+31).
__global__ void __launch_bounds__(256) k_first_flags(const uint8_t* __restrict__ img, uint64_t P,
                                                     const uint32_t* __restrict__ first_tab,
                                                     uint32_t* __restrict__ bitmap) {
  const uint64_t n_words = (P + 31) / 32;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_words;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t keys[PX_PER_THREAD];
      const uint64_t c = 2 * w + h;
      const int n = c * PX_PER_THREAD < P ? load_chunk_keys(img, P, c, keys) : 0;
      uint32_t f[PX_PER_THREAD];
#pragma unroll
      for (int s = 0; s < PX_PER_THREAD; ++s) f[s] = s < n ? __ldg(first_tab + morton_of_key(keys[s])) : 0xFFFFFFFFu;
#pragma unroll
      for (int s = 0; s < PX_PER_THREAD; ++s)
        word |= (f[s] == (uint32_t)(c * PX_PER_THREAD + s) ? 1u : 0u) << (h * PX_PER_THREAD + s);
    }
    bitmap[w] = word;
  }
}

}  // namespace cqb
