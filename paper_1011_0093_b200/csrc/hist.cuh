// K1 + K2: unique-color data reduction (reference: build_histogram,
// histogram.hpp:65-99) — 2^24-bin direct histogram with first-occurrence
// tracking, then pixel-space compaction that emits the unique colors in
// FIRST-OCCURRENCE order (histogram.hpp:77-92) with no sort.
//
// Bin table layout (HBM, 128 MiB, kept all-zero between calls):
//   bins[key].x = pixel count          (atomicAdd, RED.ADD)
//   bins[key].y = ~first pixel index   (atomicMax of the complement = min index)
// Both words share one 8-B slot, so each pixel touches one 32-B sector.
// The table is returned to zero by k_bins_reset / k_map_unique over the N'
// touched keys, so no 128 MiB clear is ever paid per call.
#pragma once
#include "common.cuh"

namespace cqb {

__device__ __forceinline__ void bin_add(uint2* __restrict__ bins, uint32_t key, uint32_t run, uint32_t first) {
  uint32_t* b = reinterpret_cast<uint32_t*>(bins + key);
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
    const uint8_t* __restrict__ img, uint64_t P, const uint2* __restrict__ bins, uint32_t* __restrict__ out_keys,
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
        const uint2 b = __ldg(bins + keys[s]);
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
    bins[keys[i]] = make_uint2(0u, 0u);
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
