// Small images: everything between K1 and the WSM loop in ONE cooperative
// launch (replaces k_occ_compact, k_bitmap_scan, k_init_centers and
// k_rank_from_bitmap, i.e. four launches and their look-back chains, by three
// grid barriers). Same outputs, same semantics:
//
//   A. count the set bits of the bin-occupancy map per block (contiguous
//      slices of the map, so block order = Morton order)          | grid.sync
//   B. emit the Morton-order samples {key, count, first pixel}, zero the
//      touched bins and map words, mark the first pixels in the
//      first-occurrence bitmap (histogram.hpp:65-99 with no sort)   | grid.sync
//   C. per-word popcount prefix of the bitmap; meanwhile block 0 runs
//      init_centers (kmeans.hpp:53-74; needs only N')               | grid.sync
//   D. first-occurrence rank of every sample (set bits below its first pixel)
//      and the gather of the K initial centers by rank.
#pragma once
#include <cooperative_groups.h>

#include <cstddef>

#include "hist.cuh"
#include "wsm.cuh"

namespace cqb {

constexpr int PREP_THREADS = 1024;
// zero_state clears exactly these run scalars; keep in sync with WsmState
static_assert(offsetof(WsmState, stop_it) + sizeof(int) - offsetof(WsmState, evals) == 40, "WsmState run scalars changed");

struct PrepParams {
  const uint8_t* img;       // with hist: K1 runs here too (phase 0)
  uint64_t P;
  int hist;
  uint32_t* occ;            // 2^19 words
  uint2* bins;
  uint32_t* m_keys;
  uint32_t* m_counts;
  uint32_t* m_rank;         // first pixel, then rank
  unsigned long long* n_unique;
  uint32_t* bitmap;         // P bits, zeroed by the host
  uint32_t* pre;            // P/32 words
  uint32_t n_words;         // ceil(P / 32)
  uint32_t* block_counts;   // [3 * gridDim.x] scratch
  uint32_t* units;          // [gridDim.x][4 * per_block] scratch: the block's non-empty units (word * 4 + byte)
  uint32_t* wofs;           // [2^19] scratch: in-block offset of each occupancy word's first sample
  const unsigned long long* draws;
  int ndraws;
  int k;
  WsmState* st;
  uint32_t* r_keys;         // optional (build_histogram API): first-occurrence order
  uint32_t* r_counts;
  uint32_t* r_first;
  unsigned long long* stamps;  // profiling: globaltimer at each phase boundary (block 0)
  int zero_state;              // also zero the bitmap, the moment sums and the run scalars (no host memsets)
};

__device__ __forceinline__ void prep_stamp(const PrepParams& Q, int i) {
  if (Q.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    Q.stamps[i] = t;
  }
}

// Block-wide exclusive scan of one u32 per thread (PREP_THREADS threads);
// returns the exclusive prefix, writes the block total to *total.
__device__ __forceinline__ uint32_t prep_block_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t ex = incl - v + (wid ? s_warp[wid - 1] : 0u);
  *total = s_warp[PREP_THREADS / 32 - 1];
  __syncthreads();  // s_warp reusable
  return ex;
}

__global__ void __launch_bounds__(PREP_THREADS, 1) k_prep_small(PrepParams Q) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t s_warp[PREP_THREADS / 32];
  __shared__ uint32_t s_base;
  __shared__ uint32_t sr[KMAX], si[KMAX], sc[KMAX];
  const int tid = threadIdx.x;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  prep_stamp(Q, 0);
  if (Q.hist) {  // ---- 0: K1 (k_hist_count's work) in the same launch
    // chunk c -> block c % G: the few chunks of a small image spread over all SMs
    hist_count_chunks(Q.img, Q.P, Q.bins, 0u, 1u << 24, Q.occ, (uint64_t)tid * G + b, (uint64_t)G * PREP_THREADS);
    grid.sync();
  }

  // ---- A: set bits per block over a contiguous slice of the occupancy map
  constexpr uint32_t OCC_WORDS_ALL = 1u << 19;
  const uint32_t per_block = (OCC_WORDS_ALL + G - 1) / G;
  const uint32_t wb0 = min(b * per_block, OCC_WORDS_ALL), wb1 = min(wb0 + per_block, OCC_WORDS_ALL);
  const uint32_t wpt = (per_block + PREP_THREADS - 1) / PREP_THREADS;  // words per thread (contiguous)
  const uint32_t wt0 = min(wb0 + tid * wpt, wb1), wt1 = min(wt0 + wpt, wb1);
  uint32_t cnt = 0, ucnt = 0;
  for (uint32_t w = wt0; w < wt1; ++w) {
    const uint32_t word = Q.occ[w];
    cnt += __popc(word);
    ucnt += (word & 0xFFu ? 1u : 0u) + (word & 0xFF00u ? 1u : 0u) + (word & 0xFF0000u ? 1u : 0u) + (word >> 24 ? 1u : 0u);
  }
  if (Q.zero_state) {  // replaces the host memsets of the quantize path
    for (uint32_t w = b * PREP_THREADS + tid; w < Q.n_words; w += G * PREP_THREADS) Q.bitmap[w] = 0u;
    if (b == 0) {
      for (int i = tid; i < 5 * KMAX; i += PREP_THREADS) Q.st->acc[i] = 0ull;
      if (tid == 0) {
        Q.st->evals = 0ull;
        Q.st->mse_err = 0ull;
        Q.st->sse = 0.0;
        Q.st->iterations = 0;
        Q.st->status = ST_OK;
        Q.st->n_empty_events = 0;
        Q.st->stop_it = 0;
      }
    }
  }
  uint32_t btotal, utotal;
  const uint32_t tex = prep_block_scan(cnt, s_warp, &btotal);
  const uint32_t uex = prep_block_scan(ucnt, s_warp, &utotal);
  {
    // the block's non-empty units, in Morton order, into its own list (phase B
    // deals them out over the whole grid: work follows the samples, not the map)
    uint32_t* ul = Q.units + (size_t)b * 4 * per_block;
    uint32_t run = tex, urun = uex;
    for (uint32_t w = wt0; w < wt1; ++w) {
      const uint32_t word = Q.occ[w];
      Q.wofs[w] = run;
      run += __popc(word);
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j)
        if ((word >> (8 * j)) & 0xFFu) ul[urun++] = w * 4 + j;
    }
  }
  if (tid == 0) {
    Q.block_counts[b] = btotal;
    Q.block_counts[2 * G + b] = utotal;
  }
  prep_stamp(Q, 1);
  grid.sync();
  prep_stamp(Q, 2);

  // ---- B: emit samples in Morton order. The non-empty units (8 bins of one
  // occupancy word) listed in phase A are dealt out over blocks 1..G-1 by
  // their global index, so every thread gets about N'/(8 x threads) units
  // however the colors cluster; a unit's output offset = its word's block
  // base + the word's in-block offset (phase A) + the set bits below it.
  // Block 0 runs init_centers meanwhile (it needs only N').
  __shared__ uint32_t s_bbase[MAXBLK];
  __shared__ uint32_t s_ubase[MAXBLK + 1];
  if (tid == 0) {
    uint32_t base = 0, ubase = 0;
    for (uint32_t c = 0; c < G; ++c) {
      s_bbase[c] = base;
      base += Q.block_counts[c];
      s_ubase[c] = ubase;
      ubase += Q.block_counts[2 * G + c];
    }
    s_ubase[G] = ubase;
    if (b == 0) *Q.n_unique = base;
    s_base = base;
  }
  __syncthreads();
  if (b == 0 && G > 1) {
    if (Q.k > 0) init_centers_block(nullptr, s_base, Q.k, Q.draws, Q.ndraws, Q.st);  // chosen ranks only
  } else {
    const uint32_t nunits = s_ubase[G];
    const uint32_t B0 = G > 1 ? 1u : 0u, NB = G - B0;
    for (uint32_t g = (b - B0) * PREP_THREADS + tid; g < nunits; g += NB * PREP_THREADS) {
      uint32_t lo = 0, hi = G;  // the block c whose list holds unit g: s_ubase[c] <= g < s_ubase[c + 1]
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_ubase[mid] <= g) lo = mid;
        else hi = mid;
      }
      const uint32_t unit = Q.units[(size_t)lo * 4 * per_block + (g - s_ubase[lo])];
      const uint32_t w = unit >> 2, j = unit & 3u;
      const uint32_t word = Q.occ[w];
      const uint32_t mine = word & (0xFFu << (8 * j));
      uint32_t pos = s_bbase[w / per_block] + Q.wofs[w] + __popc(word & ((1u << (8 * j)) - 1u));
      uint32_t ms[8];
      int nb = 0;
      uint32_t bits = mine;
      while (bits) {
        ms[nb++] = w * 32 + (__ffs(bits) - 1);
        bits &= bits - 1u;
      }
      uint2 v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < nb) v[e] = Q.bins[ms[e]];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (e < nb) {
          const uint32_t f = ~v[e].y;
          Q.m_keys[pos] = key_of_morton(ms[e]);
          Q.m_counts[pos] = v[e].x;
          Q.m_rank[pos] = f;
          asm volatile("red.global.or.b32 [%0], %1;" ::"l"(Q.bitmap + (f >> 5)), "r"(1u << (f & 31)) : "memory");
          Q.bins[ms[e]] = make_uint2(0u, 0u);
          ++pos;
        }
      }
    }
  }
  prep_stamp(Q, 3);
  if (Q.stamps) {  // per-block end of phase B (profiling)
    __syncthreads();
    if (tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      Q.stamps[-MAXBLK + (int)b] = t;
    }
  }
  grid.sync();
  prep_stamp(Q, 4);

  // ---- C: bitmap prefix (counts per block, then per-word prefix) + init
  const uint32_t n = (uint32_t)*Q.n_unique;
  const uint32_t pb = (Q.n_words + G - 1) / G;
  const uint32_t xb0 = min(b * pb, Q.n_words), xb1 = min(xb0 + pb, Q.n_words);
  const uint32_t xpt = (pb + PREP_THREADS - 1) / PREP_THREADS;
  const uint32_t xt0 = min(xb0 + tid * xpt, xb1), xt1 = min(xt0 + xpt, xb1);
  uint32_t bc = 0;
  for (uint32_t w = xt0; w < xt1; ++w) bc += __popc(Q.bitmap[w]);
  uint32_t xtotal;
  const uint32_t xex = prep_block_scan(bc, s_warp, &xtotal);
  if (tid == 0) Q.block_counts[G + b] = xtotal;
  for (uint32_t w = wb0 + tid; w < wb1; w += PREP_THREADS) Q.occ[w] = 0u;  // all-zero between calls
  prep_stamp(Q, 5);
  if (G == 1 && Q.k > 0) init_centers_block(nullptr, n, Q.k, Q.draws, Q.ndraws, Q.st);  // (one block: here)
  prep_stamp(Q, 6);
  grid.sync();
  prep_stamp(Q, 7);
  if (tid == 0) {
    uint32_t base = 0;
    for (uint32_t c = 0; c < b; ++c) base += Q.block_counts[G + c];
    s_base = base;
  }
  __syncthreads();
  {
    uint32_t run = s_base + xex;
    for (uint32_t w = xt0; w < xt1; ++w) {
      Q.pre[w] = run;
      run += __popc(Q.bitmap[w]);
    }
  }
  prep_stamp(Q, 8);
  grid.sync();
  prep_stamp(Q, 9);

  // ---- D: ranks + initial centers by rank
  const int k = Q.k;  // 0: no init (histogram only)
  const bool gather = k > 0 && Q.st->status == ST_OK;
  if (gather) {
    const uint32_t r0 = tid < k ? Q.st->chosen[tid] : 0u;
    if (tid < k) sc[tid] = r0;
    __syncthreads();
    if (tid < k) {
      int pos = 0;
      for (int u = 0; u < k; ++u) pos += sc[u] < r0;  // chosen ranks are distinct
      sr[pos] = r0;
      si[pos] = (uint32_t)tid;
    }
    __syncthreads();
  }
  for (uint32_t s = b * PREP_THREADS + tid; s < n; s += G * PREP_THREADS) {
    const uint32_t f = Q.m_rank[s];
    const uint32_t w = f >> 5;
    const uint32_t r = Q.pre[w] + __popc(Q.bitmap[w] & ((1u << (f & 31)) - 1u));
    Q.m_rank[s] = r;
    if (Q.r_keys) {
      Q.r_keys[r] = Q.m_keys[s];
      Q.r_counts[r] = Q.m_counts[s];
      Q.r_first[r] = f;
    }
    if (gather && k > 0) {
      int lo = 0, hi = k;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sr[mid] < r) lo = mid + 1;
        else hi = mid;
      }
      if (lo < k && sr[lo] == r) {
        const int i = (int)si[lo];
        const uint32_t key = Q.m_keys[s];
        Q.st->C[0][3 * i + 0] = (double)key_r(key);
        Q.st->C[0][3 * i + 1] = (double)key_g(key);
        Q.st->C[0][3 * i + 2] = (double)key_b(key);
      }
    }
  }
  prep_stamp(Q, 10);
}

}  // namespace cqb
