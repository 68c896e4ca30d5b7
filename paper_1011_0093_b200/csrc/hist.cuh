// K1 + K2: unique-color data reduction (reference: build_histogram,
// histogram.hpp:65-99) — 2^24-bin direct histogram with first-occurrence
// tracking, then pixel-space compaction that emits the unique colors in
// FIRST-OCCURRENCE order (histogram.hpp:77-92) with no sort.
//
// Bin table layout (HBM, 128 MiB, kept all-zero between calls), indexed by
// the MORTON code of the color (morton_of_key):
//   bins[m].x = pixel count          (atomicAdd, RED.ADD)
//   bins[m].y = ~first pixel index   (atomicMax of the complement = min index);
//               K2 then overwrites it with the first-occurrence RANK.
// Both words share one 8-B slot, so each pixel touches one 32-B sector.
// K2b scans the table in bin (= Morton) order, emits the samples in that
// spatially coherent order with their rank, and zeroes every touched bin, so
// no 128 MiB clear is ever paid per call.
#pragma once
#include "common.cuh"

namespace cqb {

__device__ __forceinline__ void bin_add(uint2* __restrict__ bins, uint32_t key, uint32_t run, uint32_t first) {
  uint32_t* b = reinterpret_cast<uint32_t*>(bins + morton_of_key(key));
  atomicAdd(b, run);
  atomicMax(b + 1, ~first);
}

// K1: one thread per 16-pixel chunk (grid-stride). Consecutive equal colors
// within a thread's chunk are run-length aggregated into one atomic pair.
__global__ void __launch_bounds__(HIST_THREADS) k_hist_count(const uint8_t* __restrict__ img, uint64_t P,
                                                              uint2* __restrict__ bins) {
  const uint64_t nchunk = (P + PX_PER_THREAD - 1) / PX_PER_THREAD;
  for (uint64_t c = (uint64_t)blockIdx.x * HIST_THREADS + threadIdx.x; c < nchunk;
       c += (uint64_t)gridDim.x * HIST_THREADS) {
    uint32_t keys[PX_PER_THREAD];
    const int n = load_chunk_keys(img, P, c, keys);
    const uint32_t base = (uint32_t)(c * PX_PER_THREAD);
    uint32_t cur = keys[0], run = 1, start = base;
#pragma unroll
    for (int s = 1; s < PX_PER_THREAD; ++s) {
      if (s < n) {
        if (keys[s] == cur) {
          ++run;
        } else {
          bin_add(bins, cur, run, start);
          cur = keys[s];
          run = 1;
          start = base + s;
        }
      }
    }
    bin_add(bins, cur, run, start);
  }
}

// Decoupled look-back state word: flag in the high 32 bits, value low.
constexpr unsigned long long LB_AGG = 1ull << 32;
constexpr unsigned long long LB_PRE = 2ull << 32;

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// K2: pixel-space compaction. Pixel i is the representative of its color iff
// bins[key_i] records i as the first occurrence; the exclusive prefix count of
// representatives in scan order IS the first-occurrence rank. Single pass,
// decoupled look-back over tiles of TILE_PX pixels (tile ids from a ticket so
// predecessors are always resident). Emits keys[], counts[] (and optionally
// the first pixel index) in first-occurrence order; the last tile writes N'.
__global__ void __launch_bounds__(HIST_THREADS) k_hist_compact(
    const uint8_t* __restrict__ img, uint64_t P, uint2* __restrict__ bins, uint32_t* __restrict__ out_keys,
    uint32_t* __restrict__ out_counts, uint32_t* __restrict__ out_first, unsigned long long* tile_state,
    unsigned int* ticket, unsigned long long* n_unique, uint32_t ntiles) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[HIST_THREADS / 32];
  __shared__ uint32_t s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t c = (uint64_t)tile * HIST_THREADS + tid;

  uint32_t keys[PX_PER_THREAD];
  uint32_t cnts[PX_PER_THREAD];
  uint32_t mask = 0;
  const uint64_t nchunk = (P + PX_PER_THREAD - 1) / PX_PER_THREAD;
  const uint32_t base = (uint32_t)(c * PX_PER_THREAD);
  if (c < nchunk) {
    const int n = load_chunk_keys(img, P, c, keys);
#pragma unroll
    for (int s = 0; s < PX_PER_THREAD; ++s) {
      cnts[s] = 0;
      if (s < n) {
        const uint2 b = bins[morton_of_key(keys[s])];
        if (b.y == ~(base + s)) {
          mask |= 1u << s;
          cnts[s] = b.x;
        }
      }
    }
  }
  const uint32_t cnt = __popc(mask);

  // block exclusive scan of per-thread representative counts
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < HIST_THREADS / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    if (lane < HIST_THREADS / 32) s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t block_total = s_warp[HIST_THREADS / 32 - 1];
  const uint32_t excl = incl - cnt + (wid ? s_warp[wid - 1] : 0);

  // decoupled look-back (warp 0)
  if (wid == 0) {
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) {
        __threadfence();
        atomicExch(tile_state, LB_PRE | block_total);
      }
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
  __threadfence();
  uint32_t rank = s_prefix + excl;
  if (mask) {
#pragma unroll
    for (int s = 0; s < PX_PER_THREAD; ++s) {
      if (mask & (1u << s)) {
        out_keys[rank] = keys[s];
        out_counts[rank] = cnts[s];
        if (out_first) out_first[rank] = base + s;
        // record the rank in the bin for the Morton-order pass (K2b). Other
        // pixels of this color compare ~their index against it, which can
        // never equal a rank < 2^24 while P < 2^32 - 2^24.
        bins[morton_of_key(keys[s])].y = rank;
        ++rank;
      }
    }
  }
  if (tile == ntiles - 1 && tid == 0) *n_unique = (unsigned long long)(s_prefix + block_total);
}

// Returns the touched bins to zero (used when no map pass follows).
__global__ void k_bins_reset(const uint32_t* __restrict__ keys, const unsigned long long* __restrict__ n_unique,
                             uint2* __restrict__ bins) {
  const uint64_t n = *n_unique;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    bins[morton_of_key(keys[i])] = make_uint2(0u, 0u);
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
constexpr int BC_THREADS = 512;
constexpr int BC_STEPS = 8;
constexpr int BIN_TILE = (BC_THREADS / 32) * 64 * BC_STEPS;
constexpr int N_BIN_TILES = (1 << 24) / BIN_TILE;

__global__ void __launch_bounds__(BC_THREADS) k_bins_compact(uint2* __restrict__ bins, uint32_t* __restrict__ m_keys,
                                                             uint32_t* __restrict__ m_counts,
                                                             uint32_t* __restrict__ m_rank,
                                                             unsigned long long* tile_state, unsigned int* ticket,
                                                             unsigned long long* n_unique) {
  constexpr int NW = BC_THREADS / 32;
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[NW];
  __shared__ uint32_t s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t wbase = tile * BIN_TILE + wid * (64 * BC_STEPS);
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
        m_rank[pos] = v[q].y;
        ++pos;
      }
      if (f1) {
        m_keys[pos] = key_of_morton(bin + 1);
        m_counts[pos] = v[q].z;
        m_rank[pos] = v[q].w;
      }
      reinterpret_cast<uint4*>(bins + wbase + q * 64)[lane] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  if (tile == N_BIN_TILES - 1 && tid == 0) *n_unique = (unsigned long long)(s_prefix + block_total);
}

// weights[i] = double(count) * (1.0 / double(P))  — histogram.hpp:94-97.
__global__ void k_hist_weights(const uint32_t* __restrict__ counts, const unsigned long long* __restrict__ n_unique,
                               uint64_t P, double* __restrict__ weights) {
  const uint64_t n = *n_unique;
  const double inv_total = 1.0 / (double)P;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    weights[i] = __dmul_rn((double)counts[i], inv_total);
}

}  // namespace cqb
