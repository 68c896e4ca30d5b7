// Unique-color data reduction (reference: build_histogram,
// histogram.hpp:65-99): a 2^24-bin direct histogram with first-occurrence
// tracking, then bin-space compaction into Morton order, then the
// first-occurrence ranks (histogram.hpp:77-92) from a bitmap of
// first pixel indices. No sort, and only K1 reads the pixels.
//
// Bin table layout (HBM, 128 MiB, kept all-zero between calls), indexed by
// the MORTON code of the color (morton_of_key):
//   bins[m].x = pixel count          (atomicAdd, RED.ADD)
//   bins[m].y = ~first pixel index   (atomicMax of the complement = min index)
// Both words share one 8-B slot, so each pixel touches one 32-B sector.
// K2b scans the table in bin (= Morton) order, emits the samples in that
// spatially coherent order with their first pixel, sets that pixel's bit in
// a P-bit bitmap, and zeroes every touched bin, so no 128 MiB clear is ever
// paid per call. K2c/K2d turn first pixels into ranks (set bits below).
#pragma once
#include "common.cuh"

namespace cqb {

__device__ __forceinline__ void bin_add(uint2* __restrict__ bins, uint32_t key, uint32_t run, uint32_t first,
                                        uint32_t mlo, uint32_t mhi, uint32_t* __restrict__ occ) {
  const uint32_t m = morton_of_key(key);
  if (m - mlo >= mhi - mlo) return;  // outside this pass's slice of the table
  uint32_t* b = reinterpret_cast<uint32_t*>(bins + m);
  atomicAdd(b, run);
  atomicMax(b + 1, ~first);
  if (occ) atomicOr(&occ[m >> 5], 1u << (m & 31));
}

// K1: one thread per 16-pixel chunk (grid-stride). Consecutive equal colors
// within a thread's chunk are run-length aggregated into one atomic pair.
// Only bins in the Morton slice [mlo, mhi) are updated: large images run K1
// once per half of the 128 MiB table, so each pass's atomics stay in the
// 126 MB L2 instead of re-fetching sectors from HBM.
// With `occ`, K1 also marks every touched bin in a 2^24-bit occupancy map
// (2 MiB), so small images can compact the table without scanning 128 MiB.
// px0: index of img's first pixel in the whole image (K1 over one slice of
// an image whose H2D copy is still in flight, cqb_quantize_ex).
template <bool kStream = false>
__device__ __forceinline__ void hist_count_chunks(const uint8_t* __restrict__ img, uint64_t P,
                                                  uint2* __restrict__ bins, uint32_t mlo, uint32_t mhi,
                                                  uint32_t* __restrict__ occ, uint64_t c0, uint64_t cstride,
                                                  uint32_t px0 = 0) {
  const uint64_t nchunk = (P + PX_PER_THREAD - 1) / PX_PER_THREAD;
  for (uint64_t c = c0; c < nchunk; c += cstride) {
    uint32_t keys[PX_PER_THREAD];
    const int n = load_chunk_keys<kStream>(img, P, c, keys);
    const uint32_t base = px0 + (uint32_t)(c * PX_PER_THREAD);
    uint32_t cur = keys[0], run = 1, start = base;
#pragma unroll
    for (int s = 1; s < PX_PER_THREAD; ++s) {
      if (s < n) {
        if (keys[s] == cur) {
          ++run;
        } else {
          bin_add(bins, cur, run, start, mlo, mhi, occ);
          cur = keys[s];
          run = 1;
          start = base + s;
        }
      }
    }
    bin_add(bins, cur, run, start, mlo, mhi, occ);
  }
}

template <bool kStream = false>
__global__ void __launch_bounds__(HIST_THREADS) k_hist_count(const uint8_t* __restrict__ img, uint64_t P,
                                                              uint2* __restrict__ bins, uint32_t mlo, uint32_t mhi,
                                                              uint32_t* __restrict__ occ, uint32_t px0 = 0) {
  hist_count_chunks<kStream>(img, P, bins, mlo, mhi, occ, (uint64_t)blockIdx.x * HIST_THREADS + threadIdx.x,
                    (uint64_t)gridDim.x * HIST_THREADS, px0);
}

// Decoupled look-back state word: flag in the high 32 bits, value low.
constexpr unsigned long long LB_AGG = 1ull << 32;
constexpr unsigned long long LB_PRE = 2ull << 32;

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Fill the bin table from a first-occurrence-ordered histogram (host
// histogram APIs): bins[morton(key_r)] = {count_r, r}.
__global__ void k_bins_scatter(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ counts,
                               const unsigned long long* __restrict__ n_unique, uint2* __restrict__ bins) {
  const uint64_t n = *n_unique;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    bins[morton_of_key(keys[i])] = make_uint2(counts[i], (uint32_t)i);
}

// K2b: bin-space compaction in Morton order. Each touched bin (count > 0)
// becomes one sample {key, count, first-occurrence rank}; the bin is zeroed.
// A warp streams 512 consecutive bins as 8 coalesced 512-B steps (one 16-B
// load = 2 bins per lane); in-order output offsets come from two ballots per
// step. Tiles of 8192 bins (16 warps), decoupled look-back across tiles.
#ifndef CQB_BC_THREADS
#define CQB_BC_THREADS 512
#endif
constexpr int BC_THREADS = CQB_BC_THREADS;
#ifndef CQB_BC_STEPS
#define CQB_BC_STEPS 8
#endif
constexpr int BC_STEPS = CQB_BC_STEPS;
constexpr int BIN_TILE = (BC_THREADS / 32) * 64 * BC_STEPS;
constexpr int N_BIN_TILES = (1 << 24) / BIN_TILE;

//
// Two modes for the second bin word y:
//  * bitmap == nullptr: y is the sample's rank (k_bins_scatter of a host
//    histogram); it is emitted as m_rank.
//  * bitmap != nullptr: y = ~first pixel index (straight from K1); the first
//    index is emitted in m_rank (k_rank_from_bitmap turns it into the rank)
//    and its bit is set in the P-bit first-occurrence bitmap.
__global__ void __launch_bounds__(BC_THREADS) k_bins_compact(uint2* __restrict__ bins, uint32_t* __restrict__ m_keys,
                                                             uint32_t* __restrict__ m_counts,
                                                             uint32_t* __restrict__ m_rank,
                                                             unsigned long long* tile_state, unsigned int* ticket,
                                                             unsigned long long* n_unique,
                                                             uint32_t* __restrict__ bitmap, int first_mode,
                                                             uint32_t tile_base = 0) {
  // tile_base: the launch compacts tiles [tile_base, tile_base + gridDim.x)
  // of the table (a Morton range), its output starting at index 0
  constexpr int NW = BC_THREADS / 32;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[NW];
  __shared__ uint32_t s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t wbase = (tile_base + tile) * BIN_TILE + wid * (64 * BC_STEPS);
  const unsigned lt = (1u << lane) - 1u;
  uint4 v[BC_STEPS];
  uint32_t off[BC_STEPS];
  uint32_t wcount = 0;
#pragma unroll
  for (int q = 0; q < BC_STEPS; ++q) {
    v[q] = reinterpret_cast<const uint4*>(bins + wbase + q * 64)[lane];
    const unsigned b0 = __ballot_sync(0xffffffffu, v[q].x != 0u);
    const unsigned b1 = __ballot_sync(0xffffffffu, v[q].z != 0u);
    off[q] = wcount + __popc(b0 & lt) + __popc(b1 & lt);
    wcount += __popc(b0) + __popc(b1);
  }
  if (lane == 0) s_warp[wid] = wcount;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < NW ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < NW) s_warp[lane] = w;  // inclusive
  }
  __syncthreads();
  const uint32_t block_total = s_warp[NW - 1];
  const uint32_t wexcl = wid ? s_warp[wid - 1] : 0;
  if (wid == 0) {
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(tile_state, LB_PRE | block_total);
    } else {
      if (lane == 0) atomicExch(tile_state + tile, LB_AGG | block_total);
      int j = (int)tile - 1;
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
        atomicExch(tile_state + tile, LB_PRE | (prefix + block_total));
      }
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  const uint32_t base_out = s_prefix + wexcl;
#pragma unroll
  for (int q = 0; q < BC_STEPS; ++q) {
    const bool f0 = v[q].x != 0u, f1 = v[q].z != 0u;
    if (f0 | f1) {
      uint32_t pos = base_out + off[q];
      const uint32_t bin = wbase + q * 64 + 2 * lane;
      if (f0) {
        m_keys[pos] = key_of_morton(bin);
        m_counts[pos] = v[q].x;
        const uint32_t y = first_mode ? ~v[q].y : v[q].y;
        m_rank[pos] = y;
        if (bitmap) atomicOr(&bitmap[y >> 5], 1u << (y & 31));
        ++pos;
      }
      if (f1) {
        m_keys[pos] = key_of_morton(bin + 1);
        m_counts[pos] = v[q].z;
        const uint32_t y = first_mode ? ~v[q].w : v[q].w;
        m_rank[pos] = y;
        if (bitmap) atomicOr(&bitmap[y >> 5], 1u << (y & 31));
      }
      reinterpret_cast<uint4*>(bins + wbase + q * 64)[lane] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  if (tile == gridDim.x - 1 && tid == 0) *n_unique = (unsigned long long)(s_prefix + block_total);
}

// K2b for sparse tables (small images): the same Morton-order samples as
// k_bins_compact, found through K1's occupancy map. A thread owns 4 map words
// (128 bins); set bits are counted, scanned (decoupled look-back over tiles),
// and each touched bin is read, emitted {key, count, first pixel}, zeroed,
// and its first pixel marked in the first-occurrence bitmap. The occupancy
// words are cleared for the next call. Reads 2 MiB + the touched bins only.
constexpr int OC_THREADS = 256;
constexpr int OC_WPT = 1;                            // occupancy words per thread
constexpr int OC_WORDS = OC_THREADS * OC_WPT;        // occupancy words per tile
constexpr int N_OCC_TILES = (1 << 19) / OC_WORDS;   // 2^24 bins / 32 per word

__global__ void __launch_bounds__(OC_THREADS) k_occ_compact(uint32_t* __restrict__ occ, uint2* __restrict__ bins,
                                                            uint32_t* __restrict__ m_keys,
                                                            uint32_t* __restrict__ m_counts,
                                                            uint32_t* __restrict__ m_first,
                                                            unsigned long long* tile_state, unsigned int* ticket,
                                                            unsigned long long* n_unique,
                                                            uint32_t* __restrict__ bitmap) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[OC_THREADS / 32];
  __shared__ uint32_t s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t w0 = tile * OC_WORDS + tid * OC_WPT;
  uint32_t words[OC_WPT];
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < OC_WPT; ++q) {
    words[q] = occ[w0 + q];
    cnt += __popc(words[q]);
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < OC_THREADS / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    if (lane < OC_THREADS / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const uint32_t block_total = s_warp[OC_THREADS / 32 - 1];
  const uint32_t excl = incl - cnt + (wid ? s_warp[wid - 1] : 0);
  if (wid == 0) {
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(tile_state, LB_PRE | block_total);
    } else {
      if (lane == 0) atomicExch(tile_state + tile, LB_AGG | block_total);
      int j = (int)tile - 1;
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
        atomicExch(tile_state + tile, LB_PRE | (prefix + block_total));
      }
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  if (cnt) {
    uint32_t pos = s_prefix + excl;
    int q = 0;
    // batches of up to 8 touched bins: their loads are issued together
    // (memory-level parallelism for the scattered bin reads)
    while (true) {
      uint32_t ms[8];
      int nb = 0;
      while (nb < 8 && q < OC_WPT) {
        if (words[q] == 0u) {
          ++q;
          continue;
        }
        ms[nb++] = (w0 + q) * 32 + (__ffs(words[q]) - 1);
        words[q] &= words[q] - 1u;
      }
      if (nb == 0) break;
      uint2 v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < nb) v[e] = bins[ms[e]];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (e < nb) {
          const uint32_t f = ~v[e].y;
          m_keys[pos] = key_of_morton(ms[e]);
          m_counts[pos] = v[e].x;
          m_first[pos] = f;
          if (bitmap)
            asm volatile("red.global.or.b32 [%0], %1;" ::"l"(bitmap + (f >> 5)), "r"(1u << (f & 31)) : "memory");
          bins[ms[e]] = make_uint2(0u, 0u);
          ++pos;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < OC_WPT; ++e) occ[w0 + e] = 0u;
  }
  if (tile == N_OCC_TILES - 1 && tid == 0) *n_unique = (unsigned long long)(s_prefix + block_total);
}

// First-occurrence ranks from the P-bit bitmap of first pixel indices
// (histogram.hpp:77-92 orders the unique colors by first occurrence): the
// rank of a color whose first pixel is f is the number of set bits below f.
// BS_WORDS words per tile; pre[w] = set bits in words < w (decoupled
// look-back over tiles).
constexpr int BS_THREADS = 256;
constexpr int BS_PER_THREAD = 16;
constexpr int BS_WORDS = BS_THREADS * BS_PER_THREAD;

__global__ void __launch_bounds__(BS_THREADS) k_bitmap_scan(const uint32_t* __restrict__ bitmap, uint32_t n_words,
                                                            uint32_t* __restrict__ pre,
                                                            unsigned long long* tile_state, unsigned int* ticket) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[BS_THREADS / 32];
  __shared__ uint32_t s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t w0 = tile * BS_WORDS + tid * BS_PER_THREAD;
  uint32_t c[BS_PER_THREAD];
  uint32_t cnt = 0;
  if (w0 + BS_PER_THREAD <= n_words) {
#pragma unroll
    for (int q = 0; q < BS_PER_THREAD; q += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(bitmap + w0 + q);
      c[q] = __popc(v.x);
      c[q + 1] = __popc(v.y);
      c[q + 2] = __popc(v.z);
      c[q + 3] = __popc(v.w);
    }
  } else {
#pragma unroll
    for (int q = 0; q < BS_PER_THREAD; ++q) c[q] = w0 + q < n_words ? __popc(bitmap[w0 + q]) : 0u;
  }
#pragma unroll
  for (int q = 0; q < BS_PER_THREAD; ++q) cnt += c[q];
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < BS_THREADS / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    if (lane < BS_THREADS / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const uint32_t block_total = s_warp[BS_THREADS / 32 - 1];
  const uint32_t excl = incl - cnt + (wid ? s_warp[wid - 1] : 0);
  if (wid == 0) {
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(tile_state, LB_PRE | block_total);
    } else {
      if (lane == 0) atomicExch(tile_state + tile, LB_AGG | block_total);
      int j = (int)tile - 1;
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
        atomicExch(tile_state + tile, LB_PRE | (prefix + block_total));
      }
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = s_prefix + excl;
#pragma unroll
  for (int q = 0; q < BS_PER_THREAD; ++q) {
    if (w0 + q < n_words) pre[w0 + q] = run;
    run += c[q];
  }
}

// Morton sample s (first pixel f in m_rank[s]) -> its first-occurrence rank
// r, in place. With r_keys (the build_histogram API only), also scatters the
// histogram into first-occurrence order (keys, counts, first index): random
// 4-B writes, ~0.7 ms at N' = 10.6M, so the quantize path skips it.
//
// With `chosen` (k sorted-able distinct ranks from k_init_centers, which ran
// after K2b), the sample whose rank is chosen[i] also becomes initial center
// i (kmeans.hpp:67-68): init's gather fused into this pass.
template <typename Gather>
__device__ __forceinline__ void rank_pass(const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ pre,
                                          const uint32_t* __restrict__ m_keys, const uint32_t* __restrict__ m_counts,
                                          uint32_t* __restrict__ m_rank, uint32_t n, uint32_t* __restrict__ r_keys,
                                          uint32_t* __restrict__ r_counts, uint32_t* __restrict__ r_first,
                                          Gather gather) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const uint32_t f = m_rank[s];
    const uint32_t w = f >> 5;
    const uint32_t r = pre[w] + __popc(bitmap[w] & ((1u << (f & 31)) - 1u));
    m_rank[s] = r;
    gather(r, s);
    if (r_keys) {
      r_keys[r] = m_keys[s];
      r_counts[r] = m_counts[s];
      r_first[r] = f;
    }
  }
}

__global__ void __launch_bounds__(256) k_rank_from_bitmap(
    const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ pre, const uint32_t* __restrict__ m_keys,
    const uint32_t* __restrict__ m_counts, uint32_t* __restrict__ m_rank, const unsigned long long* __restrict__ n_unique,
    uint32_t* __restrict__ r_keys, uint32_t* __restrict__ r_counts, uint32_t* __restrict__ r_first,
    const uint32_t* __restrict__ chosen, const int* __restrict__ status, int k, double* __restrict__ centers) {
  // the K chosen ranks in a 1024-slot open-addressing table (load <= 1/4):
  // ~1 shared load per sample instead of a binary search
  constexpr uint32_t HS = 1024, EMPTY = 0xFFFFFFFFu;
  __shared__ uint32_t hk[HS];
  __shared__ uint32_t hv[HS];
  auto slot0 = [](uint32_t r) { return (r * 2654435761u) >> 22; };
  const uint32_t n = (uint32_t)*n_unique;
  const bool do_gather = chosen && *status == 0 && k <= 256;
  if (do_gather) {
    const int tid = threadIdx.x;
    for (uint32_t h = tid; h < HS; h += blockDim.x) hk[h] = EMPTY;
    __syncthreads();
    if (tid < k) {  // chosen ranks are distinct
      const uint32_t r0 = chosen[tid];
      uint32_t h = slot0(r0);
      while (atomicCAS(&hk[h], EMPTY, r0) != EMPTY) h = (h + 1) & (HS - 1);
      hv[h] = (uint32_t)tid;
    }
    __syncthreads();
    rank_pass(bitmap, pre, m_keys, m_counts, m_rank, n, r_keys, r_counts, r_first, [&](uint32_t r, uint32_t s) {
      uint32_t h = slot0(r);
      uint32_t v;
      while ((v = hk[h]) != r && v != EMPTY) h = (h + 1) & (HS - 1);
      if (v == r) {
        const int i = (int)hv[h];
        const uint32_t key = m_keys[s];
        centers[3 * i + 0] = (double)key_r(key);
        centers[3 * i + 1] = (double)key_g(key);
        centers[3 * i + 2] = (double)key_b(key);
      }
    });
  } else {
    rank_pass(bitmap, pre, m_keys, m_counts, m_rank, n, r_keys, r_counts, r_first, [](uint32_t, uint32_t) {});
  }
}

// ---------------------------------------------------------------------------
// init_centers' gather (kmeans.hpp:58-68) without first-occurrence ranks.
// Center i is the sample of first-occurrence rank chosen[i] (k_init_centers),
// i.e. the sample with the chosen[i]-th smallest first pixel index f. Only
// the samples' first pixels (m_first) are needed:
//   RS1 k_first_coarse  histogram of f >> cs (NC <= 4096 coarse pixel blocks)
//   RS2 k_init_select   init_centers' chosen ranks; prefix of the coarse counts;
//                       rank r -> (block, residual);
//                       the distinct target blocks get a slot
//   RS3 k_first_mark    a bitmap of the first pixels inside the target blocks
//   RS4 k_rank_pick     the residual-th set bit of the center's block = its
//                       first pixel; the center is that pixel's color
// Two coalesced passes over N' first indices plus K bitmaps of 2^cs bits.
constexpr int RS_NC = 4096;
__host__ __device__ inline int rank_select_shift(uint64_t P) {  // smallest cs >= 5 with P >> cs <= RS_NC
  int cs = 5;
  while ((P + (1ull << cs) - 1) >> cs > (uint64_t)RS_NC) ++cs;
  return cs;
}

__global__ void __launch_bounds__(1024) k_first_coarse(const uint32_t* __restrict__ m_first,
                                                      const unsigned long long* __restrict__ n_unique, int cs,
                                                      uint32_t* __restrict__ coarse) {
  __shared__ uint32_t h[RS_NC];
  for (int i = threadIdx.x; i < RS_NC; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const uint64_t n = *n_unique, n4 = n / 4;
  const uint4* f4 = reinterpret_cast<const uint4*>(m_first);  // 16-B aligned allocation
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n4; s += 2 * T) {
    const uint4 v = __ldg(f4 + s);  // two independent 16-B loads in flight per thread
    const uint4 u = s + T < n4 ? __ldg(f4 + s + T) : make_uint4(0u, 0u, 0u, 0u);
    atomicAdd(&h[v.x >> cs], 1u);
    atomicAdd(&h[v.y >> cs], 1u);
    atomicAdd(&h[v.z >> cs], 1u);
    atomicAdd(&h[v.w >> cs], 1u);
    if (s + T < n4) {
      atomicAdd(&h[u.x >> cs], 1u);
      atomicAdd(&h[u.y >> cs], 1u);
      atomicAdd(&h[u.z >> cs], 1u);
      atomicAdd(&h[u.w >> cs], 1u);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - 4 * n4) atomicAdd(&h[m_first[4 * n4 + threadIdx.x] >> cs], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < RS_NC; i += blockDim.x)
    if (h[i]) atomicAdd(&coarse[i], h[i]);
}

// One CTA of RS_THREADS. slot_of[b]: the bitmap slot of target block b (or
// 0xFFFF); target[i] = slot << 16 | residual... split in two arrays.
constexpr int RS_THREADS = 1024;
__device__ __forceinline__ void rank_targets_block(const uint32_t* __restrict__ coarse, int nc,
                                                   const uint32_t* __restrict__ chosen,
                                                   const int* __restrict__ status, int k,
                                                   uint16_t* __restrict__ slot_of, uint32_t* __restrict__ tgt_block,
                                                   uint32_t* __restrict__ tgt_resid,
                                                   uint32_t* __restrict__ slot_bits, int words_per_slot) {
  constexpr int PER = RS_NC / RS_THREADS;  // 4 coarse blocks per thread
  __shared__ uint32_t pre[RS_NC + 1];
  __shared__ uint16_t so[RS_NC];
  __shared__ uint32_t tb[KMAX];
  __shared__ uint32_t warp_tot[RS_THREADS / 32];
  __shared__ int n_slots;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  uint32_t c[PER], sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    c[q] = t * PER + q < nc ? coarse[t * PER + q] : 0u;
    sum += c[q];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) warp_tot[wid] = incl;
  if (t == 0) n_slots = 0;
  __syncthreads();
  uint32_t run = incl - sum;
  for (int w = 0; w < wid; ++w) run += warp_tot[w];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    pre[t * PER + q] = run;
    run += c[q];
    so[t * PER + q] = 0xFFFFu;
  }
  if (t == RS_THREADS - 1) pre[RS_NC] = run;
  __syncthreads();
  const bool ok = *status == 0;
  if (ok && t < k) {  // the block holding rank r: the last b with pre[b] <= r
    const uint32_t r = chosen[t];
    int lo = 0, hi = nc;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= r) lo = mid;
      else hi = mid;
    }
    tb[t] = (uint32_t)lo;
    tgt_block[t] = (uint32_t)lo;
    tgt_resid[t] = r - pre[lo];
  }
  __syncthreads();
  // distinct target blocks get consecutive slots: flag them, then rank the
  // flags (thread t owns blocks t*PER .. t*PER+PER-1)
  if (ok && t < k) so[tb[t]] = 0u;
  __syncthreads();
  uint32_t f = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) f += so[t * PER + q] == 0u;
  uint32_t fi = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, fi, o);
    if (lane >= o) fi += u;
  }
  __syncthreads();
  if (lane == 31) warp_tot[wid] = fi;
  __syncthreads();
  uint32_t slot = fi - f;
  for (int w = 0; w < wid; ++w) slot += warp_tot[w];
#pragma unroll
  for (int q = 0; q < PER; ++q)
    if (so[t * PER + q] == 0u) so[t * PER + q] = (uint16_t)slot++;
  if (t == RS_THREADS - 1) n_slots = (int)slot;
  __syncthreads();
  for (int i = t; i < RS_NC; i += RS_THREADS) slot_of[i] = so[i];
  for (int i = t; i < n_slots * words_per_slot; i += RS_THREADS) slot_bits[i] = 0u;
}

__global__ void __launch_bounds__(1024) k_first_mark(const uint32_t* __restrict__ m_first,
                                                    const unsigned long long* __restrict__ n_unique, int cs,
                                                    const uint16_t* __restrict__ slot_of, int words_per_slot,
                                                    uint32_t* __restrict__ slot_bits) {
  __shared__ uint16_t so[RS_NC];
  for (int i = threadIdx.x; i < RS_NC; i += blockDim.x) so[i] = slot_of[i];
  __syncthreads();
  const uint64_t n = *n_unique, n4 = n / 4;
  const uint32_t mask = (1u << cs) - 1u;
  auto mark = [&](uint32_t f) {
    const uint32_t sl = so[f >> cs];
    if (sl != 0xFFFFu) atomicOr(&slot_bits[sl * words_per_slot + ((f & mask) >> 5)], 1u << (f & 31));
  };
  const uint4* f4 = reinterpret_cast<const uint4*>(m_first);
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n4; s += 2 * T) {
    const uint4 v = __ldg(f4 + s);
    const uint4 u = s + T < n4 ? __ldg(f4 + s + T) : make_uint4(0u, 0u, 0u, 0u);
    mark(v.x);
    mark(v.y);
    mark(v.z);
    mark(v.w);
    if (s + T < n4) {
      mark(u.x);
      mark(u.y);
      mark(u.z);
      mark(u.w);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < n - 4 * n4) mark(m_first[4 * n4 + threadIdx.x]);
}

// One warp per center.
__global__ void k_rank_pick(const uint32_t* __restrict__ slot_bits, int words_per_slot, int cs,
                            const uint16_t* __restrict__ slot_of, const uint32_t* __restrict__ tgt_block,
                            const uint32_t* __restrict__ tgt_resid, const uint8_t* __restrict__ img,
                            const int* __restrict__ status, int k, double* __restrict__ centers) {
  const int i = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (i >= k || *status != 0) return;
  const uint32_t b = tgt_block[i];
  const uint32_t* bits = slot_bits + (size_t)slot_of[b] * words_per_slot;
  uint32_t need = tgt_resid[i];  // set bits to skip before the one we want
  for (int w0 = 0; w0 < words_per_slot; w0 += 32) {
    const uint32_t word = w0 + lane < words_per_slot ? bits[w0 + lane] : 0u;
    const uint32_t pc = __popc(word);
    uint32_t incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    if (need < tot) {
      const unsigned owner = __ballot_sync(0xffffffffu, incl > need && incl - pc <= need);
      const int src = __ffs(owner) - 1;
      if (lane == src) {
        uint32_t wd = word;
        for (uint32_t d = need - (incl - pc); d; --d) wd &= wd - 1u;
        const uint64_t px = ((uint64_t)b << cs) + (uint64_t)(w0 + lane) * 32 + (__ffs(wd) - 1);
        centers[3 * i + 0] = (double)img[3 * px];
        centers[3 * i + 1] = (double)img[3 * px + 1];
        centers[3 * i + 2] = (double)img[3 * px + 2];
      }
      return;
    }
    need -= tot;
  }
}

// weights[i] = double(count) * (1.0 / double(P))  — histogram.hpp:94-97.
__global__ void k_hist_weights(const uint32_t* __restrict__ counts, const unsigned long long* __restrict__ n_unique,
                               uint64_t P, double* __restrict__ weights) {
  const uint64_t n = *n_unique;
  const double inv_total = 1.0 / (double)P;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    weights[i] = __dmul_rn((double)counts[i], inv_total);
}

// ---------------------------------------------------------------------------
// Pixel-row sharded histogram (config 4 across GPUs; capi.cu cqb_hist_rows /
// cqb_hist_merge). Samples travel between ranks as {key, count, first pixel}
// u32 triplets; rank o owns the bins of Morton range [o 2^24 / W, (o+1) 2^24 / W).

__host__ __device__ __forceinline__ uint32_t owner_morton_lo(int o, int world) {
  return (uint32_t)(((unsigned long long)o << 24) / (unsigned long long)world);
}

// Morton-ordered SoA samples -> triplets, and the W + 1 owner boundaries
// (first sample index of each owner's Morton range; bounds[W] = n).
__global__ void k_pack_triplets(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ counts,
                                const uint32_t* __restrict__ first, const unsigned long long* __restrict__ n_ptr,
                                uint32_t* __restrict__ out, int world, unsigned long long* __restrict__ bounds) {
  const unsigned long long n = *n_ptr;
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (unsigned long long i = tid; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
    out[3 * i] = keys[i];
    out[3 * i + 1] = counts[i];
    out[3 * i + 2] = first[i];
  }
  if (bounds && tid <= (unsigned long long)world) {
    const int o = (int)tid;
    unsigned long long a = 0, b = n;  // first i with morton(keys[i]) >= lo(o)
    if (o == world) {
      a = n;
    } else {
      const uint32_t m = owner_morton_lo(o, world);
      while (a < b) {
        const unsigned long long mid = (a + b) >> 1;
        if (morton_of_key(keys[mid]) < m) a = mid + 1;
        else b = mid;
      }
    }
    bounds[o] = a;
  }
}

// Received triplets (any order, keys may repeat across source ranks) into the
// bin table: count sum, first-pixel min, occupancy bit (k_occ_compact then
// emits them in Morton order).
__global__ void k_merge_triplets(const uint32_t* __restrict__ in, unsigned long long n, uint2* __restrict__ bins,
                                 uint32_t* __restrict__ occ) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t key = in[3 * i], cnt = in[3 * i + 1], f = in[3 * i + 2];
    const uint32_t m = morton_of_key(key);
    uint32_t* b = reinterpret_cast<uint32_t*>(bins + m);
    atomicAdd(b, cnt);
    atomicMax(b + 1, ~f);
    atomicOr(&occ[m >> 5], 1u << (m & 31));
  }
}

// The whole image's triplets (owners' lists concatenated) -> SoA samples.
__global__ void k_unpack_triplets(const uint32_t* __restrict__ in, unsigned long long n, uint32_t* __restrict__ keys,
                                  uint32_t* __restrict__ counts, uint32_t* __restrict__ first,
                                  unsigned long long* __restrict__ n_ptr) {
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) *n_ptr = n;
  for (unsigned long long i = tid; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
    keys[i] = in[3 * i];
    counts[i] = in[3 * i + 1];
    first[i] = in[3 * i + 2];
  }
}

}  // namespace cqb
