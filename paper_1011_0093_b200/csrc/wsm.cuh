// K3-K5 + loop: Weighted Sort-Means on device (reference: init_centers,
// ClusterState::update_center_tables, assign_sort_means, update_centers and
// run_weighted_kmeans — kmeans.hpp:43-74, 132-184, 201-239, 245-296, 336-376).
//
// One cooperative persistent kernel runs the whole iteration loop:
//
//   prologue : tables(C_1)                                   | grid.sync
//   iter it  : assign(it)  -> per-block exact moment deltas -> acc | grid.sync
//              finalize(it) redundantly in EVERY block (new centers, empty
//              reseed, moment-form SSE, termination) + tables(C_{it+1})
//                                                            | grid.sync
//
// Exactness contract:
//  * distances are FP64 without FMA (dist2_rn), tables sorted by (d, index),
//    sort-means break `d[p][t] >= 4*prev` and tie rule `dist < min ||
//    (dist == min && t < best)` exactly as kmeans.hpp:211-236;
//  * iteration 1 (labels all 0, integer centers) is integer-exact, run as a
//    dense dp4a argmin whose labels equal the sort-means scan from p = 0
//    (p = 0 is the lowest index, so the midpoint quirk cannot occur) and whose
//    dist_evals are recovered exactly by a binary search of row 0;
//  * cluster sums are exact u64 (Σc·r, Σc·g, Σc·b, Σc, Σc·|x|²): order- and
//    sharding-independent; centers = FP64 S/N (bit-identical to the
//    reference's FP64 weighted sums whenever P is a power of two);
//  * SSE uses the exact moment identity Σ_k Q_k − 2c_k·S_k + |c_k|²N_k in
//    double-double with a fixed reduction tree: deterministic, within ~1 ulp
//    of the true value (the reference's sequential sum differs by its own
//    rounding, ~1e-16 relative).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "map.cuh"

#ifndef CQB_DIAG_FALLBACK
#define CQB_DIAG_FALLBACK 0
#endif
#ifndef CQB_Q0
#define CQB_Q0 1  // large path: first row quads staged in shared memory
#endif
#ifndef CQB_DIAG_COUNTS
#define CQB_DIAG_COUNTS 1  // per-iteration changed / active sample counts for the profiling timeline
#endif
#ifndef CQB_D1_PPT
#define CQB_D1_PPT 4  // iteration 1 (dense, integer): samples per thread per step
#endif
#ifndef CQB_Q0_SMALL
#define CQB_Q0_SMALL 0  // ... also on the small path
#endif
#ifndef CQB_NQ
#define CQB_NQ 4  // ... how many (entries 1..4*NQ)
#endif
#ifndef CQB_EDIFF
#define CQB_EDIFF 1  // large path: candidates evaluated in difference form from per-row-entry tables (rowE)
#endif
#ifndef CQB_EDIFF_SMALL
#define CQB_EDIFF_SMALL 0  // ... also on the small path
#endif
#ifndef CQB_MOVEQ
#define CQB_MOVEQ 1  // large path: moment deltas of moving samples queued per warp and applied 32 at a time
#endif
#ifndef CQB_MOVEQ_SMALL
#define CQB_MOVEQ_SMALL 0  // ... also on the small path
#endif
#ifndef CQB_SCHED_LARGE
#define CQB_SCHED_LARGE 1  // longest-first chunk order on the large path too, for sparse sample sets (LoopSmem::sched_on)
#endif
#ifndef CQB_C4W
#define CQB_C4W 1  // scan_f32e: the first row entry's distance rides in c4[p].w (no row-quad load for points without candidates)
#endif
#ifndef CQB_B0F_LARGE
#define CQB_B0F_LARGE 0  // large path: block 0 loads a cluster's five moments once for the centers and the SSE (cfg4 -0.4%, cfg3 +1.1%: off)
#endif
#ifndef CQB_MAP_STAGE
#define CQB_MAP_STAGE 1  // large path: the map epilogue's first row entries staged in shared memory
#endif
#ifndef CQB_NQE
#define CQB_NQE 4  // quads of rowE entries staged in shared memory with the first row quads (<= CQB_NQ)
#endif


namespace cqb {

namespace cg = cooperative_groups;

constexpr int ROW32 = KMAX + 4;  // FP32 row stride (entries): 16-B aligned rows with room for the +inf tail

struct WsmState {
  double C[2][3 * KMAX];                  // center buffers [k*3 + ch]
  unsigned long long acc[5 * KMAX];       // exact sums [field*KMAX + k]: Sr, Sg, Sb, N, Q
  double sortedD[KMAX * KMAX];            // row p: d(c_p, c_order[p][j]) ascending
  // The same rows for scan_f32, without the self entry: position i holds
  // entry i + 1 (FP32 distance, order byte), positions k-1 .. ROW32-1 hold
  // +inf, so a scan reads aligned quads (one 16-B + one 4-B load per four
  // entries) and stops at the row's end without a bounds check.
  alignas(16) float rowD32[KMAX * ROW32];
  alignas(16) uint8_t rowO[KMAX * ROW32];
  // Difference form of the same entries (scan_f32<kE>): position i of row p
  // holds {m, w} of entry i + 1 = center t, with D(x, c_t) - D(x, c_p) =
  // w + (x - fl32(c_p)) . m exactly for m = -2 (c_t - c_p), w = |c_t -
  // fl32(c_p)|^2 - |c_p - fl32(c_p)|^2 (computed in FP64, rounded to FP32).
  alignas(16) float4 rowE[KMAX * KMAX];
  uint8_t order[KMAX * KMAX];             // row p: [p, others by (d, index)]
  double final_C[3 * KMAX];
  uint32_t chosen[KMAX];                  // init: chosen sample indices
  unsigned long long cand_d[2][MAXBLK];   // reseed candidates (d bits, rank, key)
  unsigned int cand_i[2][MAXBLK];
  unsigned int cand_k[2][MAXBLK];
  // the loop's grid barrier: arrivals in the low 32 bits (monotonic within a
  // launch, zeroed by block 0 before the prologue barrier), block 0's stop
  // decision in the high half; alone in its 128-B line
  alignas(128) unsigned long long bar;
  unsigned long long bar_pad[15];
  unsigned long long evals;               // point + pair distance evaluations
  unsigned long long mse_err;             // Σ count * int distance (map pass)
  double sse;
  int iterations;
  int status;
  int n_empty_events;
  int stop_it;                            // iteration at which block 0 decided to stop
};

// Sample arrays are in MORTON order (k_bins_compact); rank[i] is sample i's
// first-occurrence rank, used wherever the reference breaks ties by sample
// index (empty-cluster reseed, kmeans.hpp:277-289).
struct LoopParams {
  const uint32_t* keys;
  const uint32_t* counts;
  const uint32_t* rank;
  uint8_t* labels;
  const unsigned long long* n_ptr;  // N' on device
  unsigned long long shard_lo;      // this rank's sample range (single GPU: 0..N')
  unsigned long long shard_hi_or_max;
  unsigned long long total;         // P (pixels)
  int k;
  int mode;       // 0 fixed, 1 convergent
  int max_iters;
  double eps;
  int cap;
  int dense_first;  // iteration 1: labels all 0 and integer centers
  WsmState* st;
  double* sse_hist;
  int hist_cap;
  double* traj;
  int traj_cap;
  unsigned long long* timeline;  // optional: per-iteration globaltimer stamps (8 per iteration)
  int moments_only;  // sharded step: stop after assign + flush (global sums = this shard's moments)
  const uint8_t* cand;     // iteration 1: per 16^3 color cell, the centers that can be nearest (null: dense)
  // map epilogue (quantize path; null lut: none): k_map_tables + k_map_unique fused into the loop's tail
  int* map_sortedDr;
  uint8_t* map_orderR;
  uint32_t* map_palkey;
  uint8_t* map_lut;
  uint32_t* map_cellw;     // coarse map table (null: none): per-cell words, zeroed in the prologue
  uint8_t* map_coarse;     // its compact form (labels + MIXED bits) for k_map_pixels_coarse
  const uint16_t* cand_n;  // per cell: count, or CAND_OVERFLOW
  int debug_flags;   // diagnostics only (tools/ablate.py): 1 = skip the candidate scan (results wrong)
  unsigned long long* block_times;  // optional: phase stamps of iteration stamp_iter [phase][block]
  int stamp_iter;
  // Sharded loop with the moment exchange inside the kernel (xch.cuh; X != 0
  // instantiations only): xw ranks, each owning the contiguous sample range
  // shard_range(N', xw, rank). xrank >= 0: one process per GPU, this is rank
  // xrank and xbox[r] is rank r's exchange window mapped over NVLink (IPC).
  // xrank < 0: xw block groups of this one cooperative launch act as the
  // ranks (single-GPU emulation), xbox[g] = group g's window, xacc the
  // groups' moment sums [xw][5*KMAX].
  int res_cap;  // resident-sample kernels: samples per block reserved in dynamic shared memory
  int xw;
  int xrank;
  unsigned long long xch_timeout_ns;  // peer wait limit of the in-kernel exchange
  unsigned long long* xbox[8];
  unsigned long long* xacc;
};

// ---------------------------------------------------------------------------
// init_centers on device (kmeans.hpp:53-70): partial Fisher–Yates over
// iota(N') using the raw mt19937_64 stream computed on the host (the stream is
// independent of N'). bounded_rand's rejection + modulo (:43-49) are evaluated
// for all k draws in parallel (a rejection, probability < N'/2^64 per draw,
// diverts to the exact sequential path); the k swaps then run in one thread
// with positions >= k held in a small open-addressing map.
// The chosen indices of init_centers for one block (blockDim >= k <= KM; all
// threads of the block must call it). Returns early, uniformly, on an error
// status.
template <int KM>
__device__ void fisher_yates_block(unsigned long long n, int k, const unsigned long long* __restrict__ draws,
                                   int ndraws, uint32_t* __restrict__ chosen_out, int* status) {
  // Partial Fisher-Yates (kmeans.hpp:58-68): for i < k, j_i = i + bounded_rand(N'-i),
  // swap(idx[i], idx[j_i]), center i = colors[idx[i]]. Position i is final
  // after step i (later steps swap positions >= i+1), so with
  //   W(i)  = idx[i] just before step i = W(m) for the last m < i with j_m = i, else i
  //   c_i   = idx[j_i] just before step i = W(m) for the last m < i with j_m = j_i, else j_i
  // every chosen index follows from the j's in parallel (pointer jumping for W).
  __shared__ unsigned long long jv[KM];
  __shared__ int ptr[2][KM];
  __shared__ uint32_t wv[2][KM];
  __shared__ int s_rejected;
  const int tid = threadIdx.x;
  if ((unsigned long long)k > n) {
    if (tid == 0) *status = ST_K_EXCEEDS_N;
    return;
  }
  if (tid == 0) s_rejected = 0;
  __syncthreads();
  for (int i = tid; i < k; i += blockDim.x) {
    const unsigned long long bound = n - (unsigned long long)i;
    const unsigned long long limit = ~0ull - (~0ull % bound);
    const unsigned long long r = i < ndraws ? draws[i] : ~0ull;
    if (r >= limit) s_rejected = 1;
    jv[i] = (unsigned long long)i + r % bound;
  }
  __syncthreads();
  if (tid == 0 && s_rejected) {  // exact sequential draw consumption (bounded_rand rejection, :43-49)
    int di = 0;
    for (int i = 0; i < k; ++i) {
      const unsigned long long bound = n - (unsigned long long)i;
      const unsigned long long limit = ~0ull - (~0ull % bound);
      unsigned long long r;
      do {
        if (di >= ndraws) {
          *status = ST_DRAWS_EXHAUSTED;
          s_rejected = 2;
          break;
        }
        r = draws[di++];
      } while (r >= limit);
      if (s_rejected == 2) break;
      jv[i] = (unsigned long long)i + r % bound;
    }
  }
  __syncthreads();
  if (s_rejected == 2) return;
  const int i = tid;
  int pred = -1, same = -1;
  if (i < k) {
    const unsigned long long ji = jv[i];
    for (int m = 0; m < i; ++m) {
      const unsigned long long jm = jv[m];
      if (jm == (unsigned long long)i) pred = m;
      if (jm == ji) same = m;
    }
    ptr[0][i] = pred;
    wv[0][i] = (uint32_t)i;
  }
  __syncthreads();
  int cur = 0;
  for (int round = 0; (1 << round) <= KM; ++round) {  // 2^rounds > KM: every chain resolved
    if (i < k) {
      const int p = ptr[cur][i];
      ptr[cur ^ 1][i] = p < 0 ? -1 : ptr[cur][p];
      wv[cur ^ 1][i] = p < 0 ? wv[cur][i] : wv[cur][p];
    }
    __syncthreads();
    cur ^= 1;
  }
  if (i < k) chosen_out[i] = same < 0 ? (uint32_t)jv[i] : wv[cur][same];
}

// init_centers for the histogram path: chosen sample ranks into st->chosen,
// and (with first-occurrence-ordered keys) the centers themselves.
__device__ void init_centers_block(const uint32_t* __restrict__ keys, unsigned long long n, int k,
                                   const unsigned long long* __restrict__ draws, int ndraws, WsmState* st) {
  fisher_yates_block<KMAX>(n, k, draws, ndraws, st->chosen, &st->status);
  __syncthreads();
  if (st->status != ST_OK) return;
  const int i = threadIdx.x;
  if (keys && i < k) {  // first-occurrence-ordered keys available: gather here
    const uint32_t key = keys[st->chosen[i]];
    st->C[0][3 * i + 0] = (double)key_r(key);
    st->C[0][3 * i + 1] = (double)key_g(key);
    st->C[0][3 * i + 2] = (double)key_b(key);
  }
}


__global__ void __launch_bounds__(KMAX) k_init_centers(const uint32_t* __restrict__ keys,
                                                      const unsigned long long* __restrict__ n_ptr, int k,
                                                      const unsigned long long* __restrict__ draws, int ndraws,
                                                      WsmState* st) {
  init_centers_block(keys, *n_ptr, k, draws, ndraws, st);
}

// init_centers' K chosen ranks (above), then RS2 of the rank selection
// (hist.cuh): one launch for both single-block steps.
__global__ void __launch_bounds__(RS_THREADS) k_init_select(const unsigned long long* __restrict__ n_ptr, int k,
                                                           const unsigned long long* __restrict__ draws,
                                                           int ndraws, WsmState* st,
                                                           const uint32_t* __restrict__ coarse, int nc,
                                                           uint16_t* __restrict__ slot_of,
                                                           uint32_t* __restrict__ tgt_block,
                                                           uint32_t* __restrict__ tgt_resid,
                                                           uint32_t* __restrict__ slot_bits, int words_per_slot) {
  init_centers_block(nullptr, *n_ptr, k, draws, ndraws, st);
  __syncthreads();
  rank_targets_block(coarse, nc, st->chosen, &st->status, k, slot_of, tgt_block, tgt_resid, slot_bits,
                     words_per_slot);
}

// Initial centers from the Morton-order samples: center i = the sample whose
// first-occurrence rank is chosen[i] (kmeans.hpp:67-68). Each block sorts the
// K chosen ranks in shared memory; every sample binary-searches its rank.
__global__ void __launch_bounds__(KMAX) k_gather_chosen(const uint32_t* __restrict__ m_keys,
                                                         const uint32_t* __restrict__ m_rank,
                                                         const unsigned long long* __restrict__ n_ptr, int k,
                                                         WsmState* st) {
  __shared__ uint32_t sr[KMAX];
  __shared__ uint32_t si[KMAX];
  __shared__ uint32_t sc[KMAX];
  if (st->status != ST_OK) return;
  const int tid = threadIdx.x;
  const uint32_t r0 = tid < k ? st->chosen[tid] : 0u;
  if (tid < k) sc[tid] = r0;
  __syncthreads();
  if (tid < k) {
    int pos = 0;
    for (int u = 0; u < k; ++u) pos += sc[u] < r0;  // chosen ranks are distinct
    sr[pos] = r0;
    si[pos] = (uint32_t)tid;
  }
  __syncthreads();
  const uint32_t n = (uint32_t)*n_ptr;
  for (uint32_t s = blockIdx.x * blockDim.x + tid; s < n; s += gridDim.x * blockDim.x) {
    const uint32_t r = m_rank[s];
    int lo = 0, hi = k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sr[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    if (lo < k && sr[lo] == r) {
      const int i = (int)si[lo];
      const uint32_t key = m_keys[s];
      st->C[0][3 * i + 0] = (double)key_r(key);
      st->C[0][3 * i + 1] = (double)key_g(key);
      st->C[0][3 * i + 2] = (double)key_b(key);
    }
  }
}

// ---------------------------------------------------------------------------
// Shared-memory working set of one persistent block.
//
// Cluster moments are accumulated as exact integers in TWO per-block arrays
// (plus / minus) of u64 values split into (lo, hi) u32 words: shared-memory
// 64-bit atomics are CAS loops on sm_100a, 32-bit ones are native, and the
// carry out of `lo` is propagated by the thread that produced it. From the
// second iteration of a launch only points whose label CHANGED touch the
// accumulators (subtract from the old cluster, add to the new one), so the
// per-iteration atomic work falls with the label churn (a few % of N').
struct LoopSmem {
  double cx[KMAX], cy[KMAX], cz[KMAX];   // centers of the current assignment
  double nx[KMAX], ny[KMAX], nz[KMAX];   // next centers (finalize)
  uint2 accp[5 * KMAX];                  // block-local moment deltas (+)
  uint2 accm[5 * KMAX];                  // block-local moment deltas (-)
  int2 cb[KMAX];                         // dense path: {packed center, cc*256 + k}
  uint32_t row0[KMAX];                   // dense path: sorted d(c_0, .) as integers
  double rowd[2][KMAX];                  // tables scratch (two rows per pass)
  int rank_part[2][2][KMAX];             // tables: [row][half of u-range][t]
  uint8_t rowo[2][KMAX];                 // tables: permutation being repaired (kept: the block's rows' order)
  int rowo_row[2];                       // row whose final permutation rowo[r] holds (-1: none)
  unsigned long long red_u64[LOOP_THREADS / 32];
  double red_hi[LOOP_THREADS / 32], red_lo[LOOP_THREADS / 32];
  int red_i[LOOP_THREADS / 32];
  int red_j[LOOP_THREADS / 32];
  int empty_list[KMAX];
  unsigned int taken[KMAX];
  int n_empty;
  unsigned int wq;                       // assign: next chunk of this block's list
  unsigned long long barv;               // grid barrier: the counter value that released this block
  int stop_flag;                         // block 0: stop after this iteration
  unsigned long long* stamp;             // profiling: block_times in the stamped iteration, else null
  unsigned int part_b, part_g;           // emulated ranks (X == 2): block index in its group, group size
  int debug;                             // LoopParams::debug_flags
  int f32ok;                             // FP32 screening valid: every center |c| < 256
  int sched_on;                          // large path: longest-first chunk order in use (sparse sample sets)
};
#define SUB_STAMP(phase)                                                         \
  do {                                                                           \
    if (threadIdx.x == 0 && S.stamp) S.stamp[(phase) * gridDim.x + blockIdx.x] = globaltimer(); \
  } while (0)

// Per-block phase stamps for one iteration (profiling): bt[phase * G + block].
#define BLOCK_STAMP(phase)                                                                   \
  do {                                                                                       \
    if (L.block_times && it == L.stamp_iter && threadIdx.x == 0)                                        \
      L.block_times[(phase) * gridDim.x + blockIdx.x] = globaltimer();                     \
  } while (0)

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Entry (p -> e) of WsmState::rowE from the FP64 centers (FP64 throughout; the
// FP32 roundings of the four results are the only errors scan_f32 accounts for).
__device__ __forceinline__ float4 ediff_entry(const LoopSmem& S, int p, int e) {
  const double fx = (double)__double2float_rn(S.cx[p]), fy = (double)__double2float_rn(S.cy[p]),
               fz = (double)__double2float_rn(S.cz[p]);
  const double gx = S.cx[e] - fx, gy = S.cy[e] - fy, gz = S.cz[e] - fz;
  const double hx = S.cx[p] - fx, hy = S.cy[p] - fy, hz = S.cz[p] - fz;
  const double w = (gx * gx + gy * gy + gz * gz) - (hx * hx + hy * hy + hz * hz);
  return make_float4(__double2float_rn(-2.0 * (S.cx[e] - S.cx[p])), __double2float_rn(-2.0 * (S.cy[e] - S.cy[p])),
                     __double2float_rn(-2.0 * (S.cz[e] - S.cz[p])), __double2float_rn(w));
}

// Rows pa (and pb, or -1) of the center tables (kmeans.hpp:147-168):
// d[p][t] = dist2(c_p, c_t) and the order row [p, others sorted by
// (d, index)]. The block's 1024 threads take two rows per pass.
//
// Incremental path (like the reference's insertion repair, :169-180): the
// previous permutation is re-checked under the new distances; if it is
// still strictly increasing in (d, index) it IS the unique sorted order and
// only the distances are rewritten. Otherwise (early iterations) the row is
// re-sorted by rank counting, half of the block per row, u-range split in 2.
__device__ void tables_rows2(LoopSmem& S, WsmState* st, int pa, int pb, int k, bool incremental, bool keep,
                             bool want_e, bool tail_sync = true) {
  static_assert(LOOP_THREADS == 4 * KMAX || LOOP_THREADS == 2 * KMAX, "tables layout: 512 or 1024 threads");
  const int tid = threadIdx.x;
  const int r = tid >> 9;                     // which row of the pair
  const int t = tid & (KMAX - 1);             // element / position
  const int h = (tid >> 8) & 1;               // half of the u-range
  const int p = r ? pb : pa;
  const bool lead = p >= 0 && h == 0;         // one thread per (row, element)
  // the previous permutation: still in shared memory when this block owns the
  // same row in the same slot every iteration (one pass), else from L2
  const bool have = keep && S.rowo_row[r] == p;
  if (lead && t < k) {
    S.rowd[r][t] = t == p ? 0.0 : dist2_rn(S.cx[p], S.cy[p], S.cz[p], S.cx[t], S.cy[t], S.cz[t]);
    if (incremental && !have) S.rowo[r][t] = st->order[p * KMAX + t];
  }
  __syncthreads();
  SUB_STAMP(10);
  bool resort = !incremental;
  if (incremental) {
    // Odd-even transposition sort of positions 1..k-1 starting from the
    // previous permutation, by (d, index). A row that is still in order
    // converges in one round; repair is capped, then falls back to a full
    // rank-count sort.
    int rounds = 0;
    bool again = true;
    while (again && rounds < 32) {
      int swapped = 0;
#pragma unroll
      for (int ph = 0; ph < 2; ++ph) {
        const int pos = 1 + ph + 2 * t;
        if (lead && pos + 1 < k) {
          const int ea = S.rowo[r][pos], eb = S.rowo[r][pos + 1];
          const double da = S.rowd[r][ea], db = S.rowd[r][eb];
          if (db < da || (db == da && eb < ea)) {
            S.rowo[r][pos] = (uint8_t)eb;
            S.rowo[r][pos + 1] = (uint8_t)ea;
            swapped = 1;
          }
        }
        // the second phase's barrier is the round's vote (bar.red.or orders shared memory too)
        if (ph == 0) __syncthreads();
      }
      again = __syncthreads_or(swapped) != 0;
      ++rounds;
    }
    resort = again;
    SUB_STAMP(11);
    if (!resort && lead && t < k) {
      const int e = S.rowo[r][t];
      st->sortedD[p * KMAX + t] = S.rowd[r][e];
      if (t > 0) {
        st->rowD32[p * ROW32 + t - 1] = __double2float_rn(S.rowd[r][e]);
        st->rowO[p * ROW32 + t - 1] = (uint8_t)e;
        if (want_e) st->rowE[p * KMAX + t - 1] = ediff_entry(S, p, e);
      }
      st->order[p * KMAX + t] = (uint8_t)e;
    }
  }
  if (resort) {  // full rank-count sort (uniform across the block)
    if (p >= 0 && t < k) {
      int cnt = 0;
      if (t != p) {
        const double dt = S.rowd[r][t];
        const int u0 = h * (KMAX / 2), u1 = min(k, u0 + KMAX / 2);
        for (int u = u0; u < u1; ++u) {
          const double du = S.rowd[r][u];
          cnt += (u != p) & ((du < dt) | ((du == dt) & (u < t)));
        }
      }
      S.rank_part[r][h][t] = cnt;
    }
    __syncthreads();
    if (lead && t < k) {
      const int rank = t == p ? 0 : 1 + S.rank_part[r][0][t] + S.rank_part[r][1][t];
      st->sortedD[p * KMAX + rank] = S.rowd[r][t];
      if (rank > 0) {
        st->rowD32[p * ROW32 + rank - 1] = __double2float_rn(S.rowd[r][t]);
        st->rowO[p * ROW32 + rank - 1] = (uint8_t)t;
        if (want_e) st->rowE[p * KMAX + rank - 1] = ediff_entry(S, p, t);
      }
      st->order[p * KMAX + rank] = (uint8_t)t;
      S.rowo[r][rank] = (uint8_t)t;
    }
  }
  if (threadIdx.x == 0) {
    S.rowo_row[0] = keep ? pa : -1;
    S.rowo_row[1] = keep ? pb : -1;
  }
  if (tail_sync) __syncthreads();  // else the caller's next step begins with a block barrier
}

// Rows are owned by blocks 1..G-1 (block 0 runs the SSE / termination
// finalize meanwhile); a single-block grid does everything itself.
__device__ __forceinline__ void tables_all(LoopSmem& S, WsmState* st, int k, bool incremental, bool want_e) {
  const int G = (int)gridDim.x;
  const int first = G == 1 ? 0 : (int)blockIdx.x - 1;
  const int stride = G == 1 ? 1 : G - 1;
  if (first < 0) return;
  // one pass per block (the rows never move between slots): keep the permutations in shared memory
  const bool keep = LOOP_THREADS == 4 * KMAX && 2 * stride >= k && !(S.debug & 2048);
  for (int p = first; p < k; p += 2 * stride) {
    const int q = p + stride;
    if (LOOP_THREADS == 4 * KMAX) {
      // the last pass skips its trailing barrier: the grid barrier (or
      // grid.sync) after tables_all starts with one
      tables_rows2(S, st, p, q < k ? q : -1, k, incremental, keep, want_e, p + 2 * stride < k);
    } else {  // 512 threads: one row per pass
      tables_rows2(S, st, p, -1, k, incremental, false, want_e);
      if (q < k) tables_rows2(S, st, q, -1, k, incremental, false, want_e);
    }
  }
}

// u64 += v on a (lo, hi) pair of shared u32 words, native 32-bit atomics only.
__device__ __forceinline__ void sadd64(uint2* a, unsigned long long v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(&a->x, lo);
  const uint32_t c = (uint32_t)(old + lo) < old ? 1u : 0u;
  if (hi + c) atomicAdd(&a->y, hi + c);
}

// A sample moving from cluster `from` to cluster `to`: its five moments
// subtracted (accm) and added (accp). The ten low-word atomics are issued
// back to back (independent round trips in flight), then the carries and
// high words follow as fire-and-forget adds.
__device__ __forceinline__ void acc_move(uint2* accm, uint2* accp, int from, int to, uint32_t key, uint32_t cnt) {
  const unsigned long long c = cnt;
  const uint32_t r = key_r(key), g = key_g(key), b = key_b(key);
  const unsigned long long v[5] = {c * r, c * g, c * b, c, c * (unsigned long long)(r * r + g * g + b * b)};
  uint32_t om[5], op[5];
#pragma unroll
  for (int f = 0; f < 5; ++f) {
    om[f] = atomicAdd(&accm[f * KMAX + from].x, (uint32_t)v[f]);
    op[f] = atomicAdd(&accp[f * KMAX + to].x, (uint32_t)v[f]);
  }
#pragma unroll
  for (int f = 0; f < 5; ++f) {
    const uint32_t lo = (uint32_t)v[f], hi = (uint32_t)(v[f] >> 32);
    const uint32_t cm = hi + ((uint32_t)(om[f] + lo) < om[f] ? 1u : 0u);
    const uint32_t cp = hi + ((uint32_t)(op[f] + lo) < op[f] ? 1u : 0u);
    if (cm) atomicAdd(&accm[f * KMAX + from].y, cm);
    if (cp) atomicAdd(&accp[f * KMAX + to].y, cp);
  }
}

// The five exact moments of one sample: Σc·r, Σc·g, Σc·b, Σc, Σc·|x|².
__device__ __forceinline__ void acc_point(uint2* acc, int k, uint32_t key, uint32_t cnt) {
  const unsigned long long c = cnt;
  const uint32_t r = key_r(key), g = key_g(key), b = key_b(key);
  sadd64(&acc[0 * KMAX + k], c * r);
  sadd64(&acc[1 * KMAX + k], c * g);
  sadd64(&acc[2 * KMAX + k], c * b);
  sadd64(&acc[3 * KMAX + k], c);
  sadd64(&acc[4 * KMAX + k], c * (unsigned long long)(r * r + g * g + b * b));
}

// Work distribution: the Morton-ordered samples are dealt out in 32-sample
// warp segments round-robin over all warps of the grid (grid-stride at warp
// granularity). A segment is a compact patch of color space, so the warp's
// lanes share their previous center, row and most candidates (broadcast
// shared-memory reads, little divergence), while the round-robin spreads the
// expensive regions (Voronoi boundaries) evenly over the blocks.
__device__ __forceinline__ unsigned long long grid_threads() { return (unsigned long long)gridDim.x * blockDim.x; }
// The block's part of the grid: the whole grid, or (X == 2, emulated ranks)
// block group blockIdx.x / (gridDim.x / xw). Read from the special registers
// at each use, so the X == 0 kernels keep no extra live registers.
template <int X>
__device__ __forceinline__ unsigned int part_size(const LoopSmem& S) {
  if constexpr (X == 2) return S.part_g;
  else return gridDim.x;
}
template <int X>
__device__ __forceinline__ unsigned int part_block(const LoopSmem& S) {
  if constexpr (X == 2) return S.part_b;
  else return blockIdx.x;
}

// Full accumulation of one point per lane; when every valid lane of the warp
// carries the same label (the common case in Morton order) the five moments
// are warp-reduced and one lane does the five atomics.
__device__ __forceinline__ void acc_point_warp(uint2* acc, bool valid, int lab, uint32_t key, uint32_t cnt) {
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!act) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(act) - 1;
  const int l0 = __shfl_sync(0xffffffffu, lab, leader);
  if (__all_sync(0xffffffffu, !valid || lab == l0)) {
    const unsigned long long c = valid ? cnt : 0u;
    const uint32_t r = key_r(key), g = key_g(key), b = key_b(key);
    unsigned long long f0 = c * r, f1 = c * g, f2 = c * b, f3 = c,
                       f4 = c * (unsigned long long)(r * r + g * g + b * b);
    f0 = warp_sum(f0);
    f1 = warp_sum(f1);
    f2 = warp_sum(f2);
    f3 = warp_sum(f3);
    f4 = warp_sum(f4);
    if (lane == leader) {
      sadd64(&acc[0 * KMAX + l0], f0);
      sadd64(&acc[1 * KMAX + l0], f1);
      sadd64(&acc[2 * KMAX + l0], f2);
      sadd64(&acc[3 * KMAX + l0], f3);
      sadd64(&acc[4 * KMAX + l0], f4);
    }
  } else if (valid) {
    acc_point(acc, lab, key, cnt);
  }
}

// Iteration 1 candidates. The RGB cube is cut into 16^3 cells of 16^3
// colors. For a cell, c_t can be the nearest center of some color in it only
// if mindist2(cell, c_t) <= min_u maxdist2(cell, c_u): any color x in the
// cell has d(x, nearest) <= maxdist2(cell, c_u) for every u, and d(x, c_t) >=
// mindist2(cell, c_t). The test is non-strict, so ties stay in, and it is
// integer arithmetic on integer centers: the candidate list always contains
// the lexicographic (d, index) minimum. One block per cell, one thread per
// center; a cell with more than CAND_CAP candidates falls back to all k.
#ifndef CQB_CAND_BITS
#define CQB_CAND_BITS 4  // iteration-1 cells per axis = 2^bits (cell side 256 >> bits colors)
#endif
constexpr int CAND_AXIS = 1 << CQB_CAND_BITS, CAND_SIDE = 256 >> CQB_CAND_BITS;
constexpr int CAND_CELLS = CAND_AXIS * CAND_AXIS * CAND_AXIS;
__device__ __forceinline__ int cand_cell(uint32_t key) {
  constexpr int sh = 8 - CQB_CAND_BITS, m = CAND_AXIS - 1;
  return (int)((((key >> (16 + sh)) & m) << (2 * CQB_CAND_BITS)) | (((key >> (8 + sh)) & m) << CQB_CAND_BITS) |
               ((key >> sh) & m));
}
constexpr int CAND_CAP = 64;
constexpr uint16_t CAND_OVERFLOW = 0xFFFF;

__global__ void __launch_bounds__(KMAX) k_grid_cands(const WsmState* __restrict__ st, int k,
                                                     uint8_t* __restrict__ cand, uint16_t* __restrict__ cand_n) {
  __shared__ int s_min[KMAX / 32];
  __shared__ int s_cnt[KMAX / 32];
  const int cell = blockIdx.x, t = threadIdx.x, lane = t & 31, wid = t >> 5;
  if (st->status != ST_OK) return;
  const int lo[3] = {(cell >> (2 * CQB_CAND_BITS)) * CAND_SIDE, ((cell >> CQB_CAND_BITS) & (CAND_AXIS - 1)) * CAND_SIDE,
                     (cell & (CAND_AXIS - 1)) * CAND_SIDE};
  int mind2 = 0, maxd2 = 0x7fffffff;
  if (t < k) {
    maxd2 = 0;
    for (int ch = 0; ch < 3; ++ch) {
      const int c = (int)st->C[0][3 * t + ch];  // initial centers are sample colors: integers
      const int a = lo[ch], b = lo[ch] + CAND_SIDE - 1;
      const int below = a - c, above = c - b;
      const int dn = below > 0 ? below : (above > 0 ? above : 0);
      const int fa = c - a, fb = b - c;
      const int far = max(fa < 0 ? -fa : fa, fb < 0 ? -fb : fb);
      mind2 += dn * dn;
      maxd2 += far * far;
    }
  }
  int m = maxd2;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) s_min[wid] = m;
  __syncthreads();
  int bound = s_min[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) bound = min(bound, s_min[w]);
  const bool c_in = t < k && mind2 <= bound;
  const unsigned bal = __ballot_sync(0xffffffffu, c_in);
  if (lane == 0) s_cnt[wid] = __popc(bal);
  __syncthreads();
  int before = 0, total = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (w < wid) before += s_cnt[w];
    total += s_cnt[w];
  }
  if (c_in) {
    const int pos = before + __popc(bal & ((1u << lane) - 1u));
    if (pos < CAND_CAP) cand[cell * CAND_CAP + pos] = (uint8_t)t;
  }
  if (t == 0) cand_n[cell] = total > CAND_CAP ? CAND_OVERFLOW : (uint16_t)total;
}

// Iteration 1, dense + integer-exact (see header). Full accumulation.
template <int X>
__device__ void assign_dense_first(LoopSmem& S, const LoopParams& L, unsigned long long lo, unsigned long long hi,
                                   unsigned long long& evals) {
  const unsigned int pb = part_block<X>(S), pG = part_size<X>(S);
  const int k = L.k;
  const unsigned long long bhi = hi;
  const unsigned long long T = (unsigned long long)pG * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int cc0 = S.cb[0].y >> 8;  // |c_0|^2
  const uint32_t c0 = (uint32_t)S.cb[0].x;
  constexpr int PPT = CQB_D1_PPT;
  for (unsigned long long base = lo + (unsigned long long)pb * blockDim.x + threadIdx.x; base - lane < bhi;
       base += PPT * T) {
    uint32_t x[PPT];
    int best[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const unsigned long long i = base + q * T;
      x[q] = i < bhi ? L.keys[i] : 0u;
      best[q] = 0x7fffffff;
    }
    if (L.cand) {  // only the cell's candidate centers (k_grid_cands)
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const uint32_t xk = x[q];
        const int cell = cand_cell(xk);
        const int nc = L.cand_n[cell];
        if (nc == CAND_OVERFLOW) {
          for (int t = 0; t < k; ++t) {
            const int2 cb = S.cb[t];
            best[q] = min(best[q], cb.y - 512 * key_dot(xk, (uint32_t)cb.x));
          }
        } else {
          const uint8_t* cl = L.cand + cell * CAND_CAP;
          for (int c = 0; c < nc; ++c) {
            const int2 cb = S.cb[cl[c]];
            best[q] = min(best[q], cb.y - 512 * key_dot(xk, (uint32_t)cb.x));
          }
        }
      }
    } else {
      for (int t = 0; t < k; ++t) {
        const int2 cb = S.cb[t];
#pragma unroll
        for (int q = 0; q < PPT; ++q) best[q] = min(best[q], cb.y - 512 * key_dot(x[q], (uint32_t)cb.x));
      }
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const unsigned long long i = base + q * T;
      const bool valid = i < bhi;
      const int lab = best[q] & 255;
      uint32_t cnt = 0;
      if (valid) {
        const int xx = key_dot(x[q], x[q]);
        const uint32_t prev0 = (uint32_t)(xx + cc0 - 2 * key_dot(x[q], c0));
        const uint32_t bound = 4u * prev0;
        // # of j >= 1 with d(c_0, c_order[0][j]) < bound  (row 0 ascending)
        int lo_j = 1, hi_j = k;
        while (lo_j < hi_j) {
          const int mid = (lo_j + hi_j) >> 1;
          if (S.row0[mid] < bound) lo_j = mid + 1;
          else hi_j = mid;
        }
        evals += (unsigned long long)lo_j;  // 1 (prev) + (lo_j - 1) candidates (KM/FKM: replaced by the host)
        L.labels[i] = (uint8_t)lab;
        cnt = L.counts[i];
      }
      acc_point_warp(S.accp, valid, lab, x[q], cnt);
    }
  }
}

// Iterations >= 2 (or the first of a teacher-forced launch, full = true):
// FP64 sort-means scan from the previous label (kmeans.hpp:211-236).
//
// The reference scan evaluates exactly the row entries before the first j
// with d[p][t_j] >= 4*prev (:220-226); rows are sorted, so the break index J
// is found by binary search over the staged prefix and the J-1 candidates are
// evaluated independently (the lexicographic (dist, index) minimum does not
// depend on evaluation order). A scan that runs past the staged prefix
// ("deep" point, < 1% of points) is finished by the whole warp: 32 row
// entries per coalesced L2 read, break located by ballot, candidates
// evaluated one per lane, lexicographic minimum by shuffle reduction.
__device__ __forceinline__ void lex_min(double& md, int& mb, double d, int t) {
  if (d < md || (d == md && t < mb)) {
    md = d;
    mb = t;
  }
}

constexpr int DBG_NO_F32 = 1 << 17;   // debug flag: FP64 scans only (A/B of the FP32 screening)
constexpr int DBG_NO_SCHED_LARGE = 1 << 24;  // debug flag: large path without the longest-first chunk order (A/B)

// ---------------------------------------------------------------------------
// FP32 screening of the sort-means scan (iterations >= 2), certified against
// the reference's FP64 decisions; a lane whose decision the FP32 values
// cannot certify redoes its point with the exact FP64 scan (scan_fp64).
//
// Error bound. x is an integer color, c an FP64 center with |c| < 256 (every
// center of a run is a mean of colors or a color; checked per launch), cf =
// fl32(c) with |c - cf| <= 2^-17. The FP32 distance d = fma(b,b, fma(g,g,
// r*r)) of the FP32 differences a_i = fl(x_i - cf_i) satisfies, against the
// exact distance D (and so against the reference's FP64 dist2, which is
// within ~5 ulp64 of D):
//   |d - D| <= 2^-16 L1 + 2^-21 d + 2^-26,   L1 = sum_i |x_i - c_i| <= sqrt(3 D)
// (2 |c - cf| L1 + 2u D from the differences, 3u d from the three roundings,
// u = 2^-24; second-order terms sit in the constants' slack). With
// sqrt(3 D) <= sqrt(3) (D / 32 + 8) (AM-GM at D = 256) this is at most
//   Elin(d) = 1.3030e-6 d + 2.1150e-4,
// increasing in d with slope < 1. Decisions (every comparison below absorbs
// its own FP32 rounding: each FFMA rounds once):
//  * break at row entry j: d64[p][t_j] >= 4 prev64 is certain when
//    fl32(d64) >= pu = fl(4 (1 + 2^-18) prev + 8.52e-4) >= 4 (prev + Elin)(1 + u),
//    and the scan certainly continues when fl32(d64) < pl =
//    fl(4 (1 - 2^-18) prev - 8.52e-4); in between the point is ambiguous;
//  * the argmin: the FP32 best b is the exact (d, index) minimum when every
//    other evaluated distance has d_t - Elin(d_t) > d_b + Elin(d_b); with d2
//    the second smallest FP32 distance it suffices that
//    fl((1 - 2^-19) d2 - 2.12e-4) > fl((1 + 2^-19) d_b + 2.12e-4)
//    (an FP32 tie never certifies).
// A certified point has the reference's label and break index J (so its
// dist_evals) exactly; sums stay exact integers.
constexpr float F32_INF = __builtin_huge_valf();
constexpr float F32_PU_A = 4.0f + 0x1p-16f, F32_PL_A = 4.0f - 0x1p-16f, F32_P_B = 8.52e-4f;
constexpr float F32_C_LO = 1.0f - 0x1p-19f, F32_C_HI = 1.0f + 0x1p-19f, F32_C_B = 2.12e-4f;

// Channel C (0 = blue .. 2 = red) of a packed key as a float: one I2F.U8 with
// a byte selector (exact; a quarter-rate pipe, but one issue slot - the scan
// is issue-bound - against PRMT + FADD for the 0x4B0000xx - 2^23 form).
#ifndef CQB_I2F
#define CQB_I2F 1
#endif
template <int C>
__device__ __forceinline__ float key_chan_f32(uint32_t key) {
#if CQB_I2F
  return (float)((key >> (8 * C)) & 0xFFu);
#else
  return __fsub_rn(__uint_as_float(__byte_perm(key, 0x4B000000u, 0x7440u | (unsigned)C)), 8388608.0f);
#endif
}
__device__ __forceinline__ float u8_to_float(uint32_t v) {  // exact, no I2F
  return __fsub_rn(__uint_as_float(0x4B000000u | v), 8388608.0f);
}
__device__ __forceinline__ float dist32(float x0, float x1, float x2, float4 c) {
  const float a = __fsub_rn(x0, c.x), b = __fsub_rn(x1, c.y), d = __fsub_rn(x2, c.z);
  return __fmaf_rn(d, d, __fmaf_rn(b, b, __fmul_rn(a, a)));
}

// Longest-first chunk order (dynamic shared memory). A chunk's scan cost
// changes little between iterations, so each block hands its chunks to the
// warps in decreasing order of last iteration's cost (the largest break index
// J in the chunk): the expensive chunks start first and the block's tail -
// one warp finishing a deep chunk while the others idle - shrinks. Order only
// affects timing; every sum is an exact integer and labels are per point.
constexpr int SCHED_MAX = 4096;  // chunks per block (N' <= 2^24 at 148 blocks needs 3543)
constexpr int SCHED_BUCKETS = 64;
struct ChunkSched {
  uint16_t order[SCHED_MAX];
  uint8_t cost[SCHED_MAX];
  uint32_t bucket[SCHED_BUCKETS];
};
// Dynamic shared memory of the loop kernels (the static LoopSmem is at the
// 48 KB static limit): the FP32 centers of scan_f32, then the chunk order.
struct LoopDyn {
  float4 c4[KMAX];  // centers of the current assignment rounded to FP32
  float4 q0[CQB_NQ][KMAX];  // large path: entries 1..4*NQ of every FP32 row (staged per pass)
#if !CQB_EDIFF || CQB_Q0_SMALL
  uint32_t o0[CQB_NQ][KMAX];  // (scan_f32 only: scan_f32e reads no order bytes)
#endif
  ChunkSched sched;
};
// ... followed, in the kernels whose scan is scan_f32e / whose moves are queued, by
struct LoopDynLarge {
  LoopDyn base;
  // entries 1..4*NQE of every rowE row, row-major with one entry of padding
  // per row (coalesced staging copy; lanes on neighbouring rows hit different
  // banks)
  float4 e0[KMAX * (4 * CQB_NQE + 1)];
  // per-warp list of moving samples awaiting their moment deltas:
  // {count index | new label << 24, key | old label << 24}
  uint32_t mq[LOOP_THREADS / 32][32][2];
};
constexpr bool kSmallUsesLarge = CQB_EDIFF_SMALL || CQB_MOVEQ_SMALL;
constexpr size_t LOOP_DYN_LARGE = sizeof(LoopDynLarge);                                  // PPT >= 2 kernels
constexpr size_t LOOP_DYN_SMALL = kSmallUsesLarge ? sizeof(LoopDynLarge) : sizeof(LoopDyn);  // PPT == 1 kernels
__device__ __forceinline__ LoopDyn& loop_dyn_smem() {
  extern __shared__ __align__(16) unsigned char loop_dyn[];
  return *reinterpret_cast<LoopDyn*>(loop_dyn);
}
__device__ __forceinline__ LoopDynLarge& loop_dyn_large() {
  extern __shared__ __align__(16) unsigned char loop_dyn[];
  return *reinterpret_cast<LoopDynLarge*>(loop_dyn);
}
__device__ __forceinline__ ChunkSched& chunk_sched() { return loop_dyn_smem().sched; }
__device__ __forceinline__ float4* loop_c4() { return loop_dyn_smem().c4; }
// Resident samples (small sample sets): the block's chunks - its fixed share
// of the Morton-ordered samples - stay in dynamic shared memory for the whole
// loop (key, count, label; local index = chunk * 32 + lane), so a scan starts
// without the L2 round trip for its sample. Global labels are still written
// on every change (stores do not stall), so reseed, the map epilogue and the
// API read them as before. Capacity: res_cap samples per block (host-sized).
struct ResSamples {
  uint32_t* key;
  uint32_t* cnt;
  uint8_t* lab;
};
__device__ __forceinline__ ResSamples res_samples(int cap) {
  extern __shared__ __align__(16) unsigned char loop_dyn[];
  unsigned char* b = loop_dyn + ((LOOP_DYN_SMALL + 15) & ~size_t(15));
  return {reinterpret_cast<uint32_t*>(b), reinterpret_cast<uint32_t*>(b) + cap,
          reinterpret_cast<uint8_t*>(reinterpret_cast<uint32_t*>(b) + 2 * cap)};
}
__host__ __device__ constexpr size_t res_smem_bytes(int cap) {
  return ((LOOP_DYN_SMALL + 15) & ~size_t(15)) + (size_t)cap * 9;
}

// Counting sort of this block's chunks by cost, descending (block-wide).
__device__ void sched_sort(uint32_t my_ch) {
  ChunkSched& C = chunk_sched();
  const int tid = threadIdx.x;
  for (int b = tid; b < SCHED_BUCKETS; b += blockDim.x) C.bucket[b] = 0u;
  __syncthreads();
  for (uint32_t j = tid; j < my_ch; j += blockDim.x) atomicAdd(&C.bucket[min((int)C.cost[j], SCHED_BUCKETS - 1)], 1u);
  __syncthreads();
  if (tid < 32) {  // exclusive prefix over buckets, high cost first
    uint32_t a = C.bucket[SCHED_BUCKETS - 1 - 2 * tid], b = C.bucket[SCHED_BUCKETS - 2 - 2 * tid];
    uint32_t v = a + b, incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (tid >= o) incl += u;
    }
    const uint32_t ex = incl - v;
    C.bucket[SCHED_BUCKETS - 1 - 2 * tid] = ex;
    C.bucket[SCHED_BUCKETS - 2 - 2 * tid] = ex + a;
  }
  __syncthreads();
  for (uint32_t j = tid; j < my_ch; j += blockDim.x)
    C.order[atomicAdd(&C.bucket[min((int)C.cost[j], SCHED_BUCKETS - 1)], 1u)] = (uint16_t)j;
  __syncthreads();
}

// Sort-means scans past DEEP_J entries switch to a
// search for the break index with DEEP_P independent probes per round, then
// evaluate the candidates below it with no per-entry check: a deep scan is a
// few L2 round trips instead of one per two entries.
#ifndef CQB_DEEP_J
#define CQB_DEEP_J 17
#endif
#ifndef CQB_DEEP_P
#define CQB_DEEP_P 3
#endif
constexpr int DEEP_J = CQB_DEEP_J;
#ifndef CQB_LOOP_BARRIER
#define CQB_LOOP_BARRIER 1
#endif
constexpr int DEEP_P = CQB_DEEP_P;

// One point's sort-means scan in FP32. Returns its break index J (>= 1) and
// sets `best` when both decisions are certified, else 0 (redo in FP64).
// c4: FP32 centers; rq / oq: row p of the FP32 distances / order bytes
// without the self entry (WsmState::rowD32 / rowO), read four entries at a time.
template <bool kDeep, int DEEP_J_, int DEEP_P_, bool kQ0 = false>
__device__ __forceinline__ int scan_f32(const float4* __restrict__ c4, const float4* __restrict__ rq,
                                        const uint32_t* __restrict__ oq, int k, uint32_t key, int p, int& best_out,
                                        unsigned int& n_active) {
  const float x0 = key_chan_f32<2>(key), x1 = key_chan_f32<1>(key), x2 = key_chan_f32<0>(key);
  const float prev = dist32(x0, x1, x2, c4[p]);
  const float pu = __fmaf_rn(prev, F32_PU_A, F32_P_B);
  const float pl = __fmaf_rn(prev, F32_PL_A, -F32_P_B);
  best_out = p;
  float4 D;  // entries 1..4
  uint32_t T;
#if !CQB_EDIFF || CQB_Q0_SMALL
  if constexpr (kQ0) {  // staged in shared memory
    D = loop_dyn_smem().q0[0][p];
    T = loop_dyn_smem().o0[0][p];
  } else
#endif
  {
    D = rq[0];
    T = oq[0];
  }
  // the common case: no candidate (kmeans.hpp:220-226 breaks at j = 1); k = 1: D.x = +inf
  if (D.x >= pl) return D.x >= pu ? 1 : 0;
  if (CQB_DIAG_COUNTS) n_active += 1;
  float bd = prev, d2 = F32_INF;
  int best = p;
  auto eval = [&](uint32_t t) {
    const float d = dist32(x0, x1, x2, c4[t]);
    d2 = fminf(d2, fmaxf(bd, d));
    best = d < bd ? (int)t : best;
    bd = fminf(bd, d);
  };
  int j = 1;  // the next entry to test; entry j is a certain candidate at the loop head
  int qi = 0;
  float Db;   // the break entry's distance
  for (;;) {
    eval(T & 0xFFu);
    if (D.y >= pl) { Db = D.y; j += 1; break; }
    eval((T >> 8) & 0xFFu);
    if (D.z >= pl) { Db = D.z; j += 2; break; }
    eval((T >> 16) & 0xFFu);
    if (D.w >= pl) { Db = D.w; j += 3; break; }
    eval(T >> 24);
    j += 4;
    ++qi;
#if !CQB_EDIFF || CQB_Q0_SMALL
    if (kQ0 && qi < CQB_NQ) {
      D = loop_dyn_smem().q0[qi][p];
      T = loop_dyn_smem().o0[qi][p];
    } else
#endif
    {
      D = rq[qi];
      T = oq[qi];
    }
    if (D.x >= pl) { Db = D.x; break; }
    if (kDeep && j > DEEP_J_) {
      // deep scan: the first entry e >= j with distance >= pl (rows are sorted,
      // fl32 is monotone, and the +inf tail ends the row), by DEEP_P_
      // independent probes per round; then j .. e-1 are candidates
      const float* rf = reinterpret_cast<const float*>(rq) - 1;  // rf[e] = entry e
      const uint8_t* ro = reinterpret_cast<const uint8_t*>(oq) - 1;
      int a = j, b = k;
      while (a < b) {
        int na = a, nb = b;
#pragma unroll
        for (int u = DEEP_P_; u >= 1; --u) {
          const int m = a + ((b - a) * u) / (DEEP_P_ + 1);
          if (m >= a && m < b) {
            if (rf[m] >= pl) nb = m;
            else if (m + 1 > na) na = m + 1;
          }
        }
        if (na == a && nb == b) {
          if (rf[a] >= pl) nb = a;
          else na = a + 1;
        }
        a = na < nb ? na : nb;
        b = nb;
      }
      for (int i2 = j; i2 < b; ++i2) eval(ro[i2]);
      j = b;
      Db = rf[b];  // +inf at the row's end (b = k)
      break;
    }
  }
  if (Db < pu) return 0;  // the break itself is uncertain
  if (!(__fmaf_rn(d2, F32_C_LO, -F32_C_B) > __fmaf_rn(bd, F32_C_HI, F32_C_B))) return 0;
  best_out = best;
  return j;
}

// The same scan with the candidates evaluated in DIFFERENCE form: for the
// point's own center p and row entry j -> center t,
//   Delta_t = D(x, c_t) - D(x, c_p) = w + a . m,  a = x - fl32(c_p),
// with {m, w} = WsmState::rowE[p][j - 1] (ediff_entry). One 16-B load and three
// FFMAs per candidate (no order byte, no center gather, no subtractions), on
// the differences a_i the own-center distance already produced. The break
// tests are those of scan_f32 (prev in the six-operation form, same pl / pu).
//
// Error bound of diff = fma(a0, m0, fma(a1, m1, fma(a2, m2, w))), u = 2^-24:
// w carries one FP32 rounding (u |w*|), every product a_i m_i two (a_i and
// m_i: 2u S, S = sum |a_i m_i|), and each of the three FFMAs rounds a partial
// sum of magnitude <= |w*| + S: |diff - Delta| <= (4 |w*| + 5 S) u (1 + O(u))
// + 1e-9 (the FP64 roundings of the table and of the reference's own dist2).
// An evaluated entry has D(c_p, c_t) < 4 prev (its fl32 is below pl), hence
// |w*| <= D(c_p, c_t) + 0.012 and S <= |a| |m| = 2 sqrt(prev' D(c_p, c_t))
// with prev' = |a*|^2 <= prev (1 + 6u): both are at most 4 prev (1 + 1e-6) +
// 0.012, and |diff - Delta| <= E = 36 u prev + 1e-8 = 2.15e-6 prev + 1e-8
// (tests/test_ediff_bound_cpu.py samples it: random and reflected-center
// inputs stay below 0.75 E). The own center has Delta = 0 exactly. The FP32
// best (index 0 = own) is the reference's lexicographic (d, index) minimum
// when the second smallest difference exceeds the smallest by more than 2 E;
// the test below uses 4.4e-6 prev + 2.5e-6 (> 2 E (1 + u) plus the
// subtraction's rounding). A tie never certifies.
constexpr float F32_E_A = 4.4e-6f, F32_E_B = 2.5e-6f;
// 16-B load from a 32-bit shared-window address (the dynamic block's base is
// converted once per assign pass; addressing through generic pointers made the
// compiler rebuild the window base, S2R + three more instructions, per point)
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
template <bool kDeep, int DEEP_J_, int DEEP_P_, bool kQ0 = false>
__device__ __forceinline__ int scan_f32e(const uint32_t sb, const float4* __restrict__ rq,
                                         const uint32_t* __restrict__ oq, const float4* __restrict__ re, int k,
                                         uint32_t key, int p, int& best_out, unsigned int& n_active) {
  // sb: shared-window address of the loop's dynamic block (LoopDyn)
  const uint32_t sp = sb + (uint32_t)p * 16u;  // + row p of c4 / q0[.]
  const uint32_t se = sb + (uint32_t)offsetof(LoopDynLarge, e0) + (uint32_t)p * (16u * (4 * CQB_NQE + 1));
  const float4 cp = lds128(sp + (uint32_t)offsetof(LoopDyn, c4));
  const float a0 = __fsub_rn(key_chan_f32<2>(key), cp.x), a1 = __fsub_rn(key_chan_f32<1>(key), cp.y),
              a2 = __fsub_rn(key_chan_f32<0>(key), cp.z);
  const float prev = __fmaf_rn(a2, a2, __fmaf_rn(a1, a1, __fmul_rn(a0, a0)));  // = dist32(x, c4[p])
  const float pu = __fmaf_rn(prev, F32_PU_A, F32_P_B);
  const float pl = __fmaf_rn(prev, F32_PL_A, -F32_P_B);
  best_out = p;
  float4 D;  // entries 1..4
  if (CQB_C4W && kQ0) {
    if (cp.w >= pl) return cp.w >= pu ? 1 : 0;
    D = lds128(sp + (uint32_t)offsetof(LoopDyn, q0));
  } else {
    if constexpr (kQ0) D = lds128(sp + (uint32_t)offsetof(LoopDyn, q0));
    else D = rq[0];
    if (D.x >= pl) return D.x >= pu ? 1 : 0;
  }
  if (CQB_DIAG_COUNTS) n_active += 1;
  float bd = 0.f, d2 = F32_INF;  // smallest / second smallest difference (own center: 0)
  int best = 0;                  // row entry of the smallest (0 = own center)
  auto eval = [&](const float4 E, int e) {
    const float d = __fmaf_rn(a0, E.x, __fmaf_rn(a1, E.y, __fmaf_rn(a2, E.z, E.w)));
    d2 = fminf(d2, fmaxf(bd, d));
    best = d < bd ? e : best;
    bd = fminf(bd, d);
  };
  // Quad qi = entries 4 qi + 1 .. 4 qi + 4, its distances in D; the first is a
  // certain candidate at the loop head; every exit records the break index
  // and the break entry's distance.
  int qi = 0;
  int j;
  float Db;
  auto leave = [&](int jv, float dv) {
    j = jv;
    Db = dv;
  };
  // ld(c): the rowE entry of 4 qi + 1 + c; true = the scan broke inside the quad
  auto quad = [&](auto ld) -> bool {
    eval(ld(0), 4 * qi + 1);
    if (D.y >= pl) { leave(4 * qi + 2, D.y); return true; }
    eval(ld(1), 4 * qi + 2);
    if (D.z >= pl) { leave(4 * qi + 3, D.z); return true; }
    eval(ld(2), 4 * qi + 3);
    if (D.w >= pl) { leave(4 * qi + 4, D.w); return true; }
    eval(ld(3), 4 * qi + 4);
    return false;
  };
  for (;;) {
    if (kQ0 && qi < CQB_NQE) {
      const uint32_t es = se + 64u * (uint32_t)qi;
      if (quad([&](int c) { return lds128(es + 16u * (uint32_t)c); })) break;
    } else {
      const float4* eg = re + 4 * qi;
      if (quad([&](int c) { return eg[c]; })) break;
    }
    ++qi;
    if (kQ0 && qi < CQB_NQ) D = lds128(sp + (uint32_t)offsetof(LoopDyn, q0) + (uint32_t)qi * (16u * KMAX));
    else D = rq[qi];
    if (D.x >= pl) { leave(4 * qi + 1, D.x); break; }
    if (kDeep && 4 * qi + 1 > DEEP_J_) {  // deep scan (as in scan_f32)
      const float* rf = reinterpret_cast<const float*>(rq) - 1;  // rf[e] = entry e
      int a = 4 * qi + 1, b = k;
      while (a < b) {
        int na = a, nb = b;
#pragma unroll
        for (int u = DEEP_P_; u >= 1; --u) {
          const int m = a + ((b - a) * u) / (DEEP_P_ + 1);
          if (m >= a && m < b) {
            if (rf[m] >= pl) nb = m;
            else if (m + 1 > na) na = m + 1;
          }
        }
        if (na == a && nb == b) {
          if (rf[a] >= pl) nb = a;
          else na = a + 1;
        }
        a = na < nb ? na : nb;
        b = nb;
      }
      for (int i2 = 4 * qi + 1; i2 < b; ++i2) eval(re[i2 - 1], i2);
      leave(b, rf[b]);  // +inf at the row's end (b = k)
      break;
    }
  }
  if (Db < pu) return 0;  // the break itself is uncertain
  if (!(__fsub_rn(d2, bd) > __fmaf_rn(prev, F32_E_A, F32_E_B))) return 0;
  if (best) best_out = (int)(reinterpret_cast<const uint8_t*>(oq) - 1)[best];
  return j;
}

// One point's sort-means scan in FP64 with the reference's exact semantics
// (kmeans.hpp:211-236). Out of line: it is the rare path (scan_f32 not
// certified, or centers outside its range) and keeps its registers out of the
// FP32 loop. Returns J | best << 12 | active << 24.
__device__ __noinline__ int scan_fp64(const LoopSmem& S, const double* __restrict__ rd, const uint8_t* __restrict__ ro,
                                      int k, uint32_t key, int p, int debug_flags) {
  int best = p, J = 1, active = 0;
  const double x0 = u8_to_double(key_r(key)), x1 = u8_to_double(key_g(key)), x2 = u8_to_double(key_b(key));
  double mind = dist2_rn(x0, x1, x2, S.cx[p], S.cy[p], S.cz[p]);  // prev
  const double bound = 4.0 * mind;
  bool deep = false;
  // the reference's scan (kmeans.hpp:217-231), two entries per step
  if (k > 1 && rd[1] < bound && !(debug_flags & 1)) {
    active = 1;
    int j = 1;
    for (;;) {
      const double d0 = rd[j];
      const double d1 = j + 1 < k ? rd[j + 1] : bound;
      const int t0 = ro[j];
      const int t1 = j + 1 < k ? ro[j + 1] : 0;
      if (d0 >= bound) break;
      lex_min(mind, best, dist2_rn(x0, x1, x2, S.cx[t0], S.cy[t0], S.cz[t0]), t0);
      ++j;
      if (d1 >= bound) break;
      lex_min(mind, best, dist2_rn(x0, x1, x2, S.cx[t1], S.cy[t1], S.cz[t1]), t1);
      ++j;
      if (j >= k) break;
      if (j >= DEEP_J) {  // deep scan: find the break index, then evaluate without checks
        deep = true;
        break;
      }
    }
    if (deep) {
      // J = min{i in [j, k) : rd[i] >= bound}, or k: the row is sorted, so
      // DEEP_P independent probes per round cut [lo, hi] to 1/(DEEP_P+1)
      int a = j, b = k;
      while (a < b) {
        int na = a, nb = b;
#pragma unroll
        for (int u = DEEP_P; u >= 1; --u) {
          const int m = a + ((b - a) * u) / (DEEP_P + 1);
          if (m >= a && m < b) {
            if (rd[m] >= bound) nb = m;
            else if (m + 1 > na) na = m + 1;
          }
        }
        if (na == a && nb == b) {  // interval too small for distinct probes: step
          if (rd[a] >= bound) nb = a;
          else na = a + 1;
        }
        a = na < nb ? na : nb;
        b = nb;
      }
      // candidates j .. b-1 are below the bound: the serial scan's set
      for (int i2 = j; i2 < b; ++i2) {
        const int t = ro[i2];
        lex_min(mind, best, dist2_rn(x0, x1, x2, S.cx[t], S.cy[t], S.cz[t]), t);
      }
      j = b;
    }
    J = j;
  }
  return J | (best << 12) | (active << 24);
}

// SCHED: longest-first chunk order (always for PPT == 1). The large path has
// both forms as separate copies of this function inside one kernel, chosen per
// launch by LoopSmem::sched_on: compiled into a single copy, the order's
// bookkeeping cost the other case 7% even when switched off (spills).
template <int PPT, int X, bool R, bool SCHED>
__device__ __forceinline__ void assign_sort_means(LoopSmem& S, const LoopParams& L, unsigned long long lo64,
                                  unsigned long long hi64, bool full, unsigned long long& evals,
                                  unsigned int& n_changed, unsigned int& n_active) {
  const unsigned int pb = part_block<X>(S), pG = part_size<X>(S);
  // Lane-local scan; 32-bit indexing (N' <= 2^24). The break index J is found
  // by exponential + binary search in the sorted row (most points stop at
  // J = 1 after one comparison), then the J - 1 candidates are evaluated.
  // PPT chunks per grab (one point per lane per chunk): 2 gives ILP for large
  // sample sets, 1 finer balance (shorter tails) for small ones.
  const uint32_t lo = (uint32_t)lo64, hi = (uint32_t)hi64;
  const int lane = threadIdx.x & 31;
  // Work split: 32-point Morton chunks dealt round-robin to the blocks
  // (chunk c -> block c % G), so every SM gets the same number of chunks
  // within one and samples every region of color space; inside a block the
  // chunks are handed to the warps dynamically (shared counter), PPT at a
  // time (small sample sets: longest first, sched_sort): a warp held up by
  // deep scans does not hold up the block.
  const uint32_t G = pG, W = blockDim.x >> 5, w = threadIdx.x >> 5;
  const uint32_t nch = (hi - lo + 31u) >> 5;
  // small sample sets: chunk costs recorded for the longest-first order
  constexpr bool kSched = SCHED;
  constexpr bool kDeep = true;
  constexpr bool kQ0 = (PPT >= 2 || CQB_Q0_SMALL) && CQB_Q0;
  constexpr bool kE = PPT >= 2 ? CQB_EDIFF != 0 : CQB_EDIFF_SMALL != 0;
  const uint32_t my_ch = nch > pb ? (nch - 1u - pb) / G + 1u : 0u;
  const double* __restrict__ gd = L.st->sortedD;
  const float4* __restrict__ rq32 = reinterpret_cast<const float4*>(L.st->rowD32);
  const uint32_t* __restrict__ oq32 = reinterpret_cast<const uint32_t*>(L.st->rowO);
  const float4* c4 = loop_c4();
  // (through an opaque move: the compiler would otherwise rebuild it from S2R per point)
  uint32_t dyn_sb;
  asm volatile("mov.u32 %0, %1;" : "=r"(dyn_sb) : "r"((uint32_t)__cvta_generic_to_shared(&loop_dyn_smem())));
  const uint8_t* __restrict__ go = L.st->order;
  // FP32 screening (scan_f32): sort-means scans whose centers all satisfy |c| < 256
  const bool use32 = S.f32ok;
  if constexpr (kQ0) {  // the rows' first quads into shared memory (the rows are final: grid barrier)
    for (int u = threadIdx.x; u < CQB_NQ * L.k; u += blockDim.x) {
      const int t = u % L.k, qq = u / L.k;
      loop_dyn_smem().q0[qq][t] = __ldcg(rq32 + t * (ROW32 / 4) + qq);
#if !CQB_EDIFF || CQB_Q0_SMALL
      if (!kE) loop_dyn_smem().o0[qq][t] = __ldcg(oq32 + t * (ROW32 / 4) + qq);
#endif
    }
    if (kE)
      for (int u = threadIdx.x; u < 4 * CQB_NQE * L.k; u += blockDim.x) {
        const int t = u / (4 * CQB_NQE), e = u % (4 * CQB_NQE);
        loop_dyn_large().e0[t * (4 * CQB_NQE + 1) + e] = __ldcg(L.st->rowE + t * KMAX + e);
      }
    __syncthreads();
    if (CQB_C4W && kE) {
      for (int t = threadIdx.x; t < L.k; t += blockDim.x) loop_dyn_smem().c4[t].w = loop_dyn_smem().q0[0][t].x;
      __syncthreads();
    }
  }
  const uint32_t* __restrict__ keys = L.keys;
  const uint32_t* __restrict__ counts = L.counts;
  uint8_t* __restrict__ labels = L.labels;
  const int k = L.k;
  uint32_t ev = 0;
  (void)W;
  (void)w;
  // Moving samples (label changed) are a few % of a pass, scattered over the
  // warps: applying their ten moment atomics on the spot runs ~70 warp
  // instructions for one or two lanes. They are queued per warp instead (two
  // words in a 32-slot shared list, positions from one ballot) and applied
  // together, one record per lane, when the next chunk's moves would not fit
  // (the counts are gathered then). The sums are exact integers, so the order
  // of the additions does not matter.
  constexpr bool kMQ = PPT >= 2 ? CQB_MOVEQ != 0 : CQB_MOVEQ_SMALL != 0;
  uint32_t qn = 0;  // queued records (warp-uniform)
  uint32_t(*mq)[2] = loop_dyn_large().mq[threadIdx.x >> 5];
  auto apply_moves = [&]() {  // all qn (<= 32) queued records
    __syncwarp();
    if ((uint32_t)lane < qn) {
      const uint32_t a = mq[lane][0], b = mq[lane][1];
      const uint32_t ci = a & 0xFFFFFFu;
      uint32_t cnt;
      if constexpr (R) cnt = res_samples(L.res_cap).cnt[ci];
      else cnt = counts[ci];
      acc_move(S.accm, S.accp, (int)(b >> 24), (int)(a >> 24), b & 0xFFFFFFu, cnt);
    }
    __syncwarp();
    qn = 0;
  };
  for (;;) {
    uint32_t j = 0;
    if (lane == 0) j = atomicAdd(&S.wq, (unsigned)PPT);
    j = __shfl_sync(0xffffffffu, j, 0);
    if (j >= my_ch) break;
    uint32_t key[PPT], idx[PPT], chunk[PPT];
    int lab[PPT], nlab[PPT];
    const bool sched = kSched && my_ch <= (uint32_t)SCHED_MAX;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      uint32_t jj = j + q;
      if (sched && jj < my_ch) jj = chunk_sched().order[jj];
      chunk[q] = jj;
      const uint32_t i = lo + ((pb + G * jj) << 5) + lane;
      const bool v = jj < my_ch && i < hi;
      idx[q] = v ? i : hi;
      if constexpr (R) {
        const ResSamples rs = res_samples(L.res_cap);
        const uint32_t li = (jj << 5) + lane;
        key[q] = v ? rs.key[li] : 0u;
        lab[q] = v ? (int)rs.lab[li] : 0;
      } else {
        key[q] = v ? keys[i] : 0u;
        lab[q] = v ? (int)labels[i] : 0;
      }
    }
    uint32_t J_of[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) J_of[q] = 0u;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      nlab[q] = lab[q];
      if (idx[q] >= hi) continue;
      const int p = lab[q];
      const uint8_t* ro = go + p * KMAX;
      int best = p;
      int J = 0;
      if (use32) {
        if constexpr (kE)
          J = scan_f32e<kDeep, DEEP_J, DEEP_P, kQ0>(dyn_sb, rq32 + p * (ROW32 / 4), oq32 + p * (ROW32 / 4),
                                                    L.st->rowE + p * KMAX, k, key[q], p, best, n_active);
        else
          J = scan_f32<kDeep, DEEP_J, DEEP_P, kQ0>(c4, rq32 + p * (ROW32 / 4), oq32 + p * (ROW32 / 4), k, key[q], p,
                                                   best, n_active);
      }
      if (J == 0) {  // FP64: uncertified FP32 screens, or screening off (rare)
        const int r = scan_fp64(S, gd + p * KMAX, ro, k, key[q], p, L.debug_flags);
        J = r & 0xFFF;
        best = (r >> 12) & 0xFF;
#if CQB_DIAG_FALLBACK  // diagnostics build: the timeline's "active" count = FP64 fallbacks of scan_f32
        n_active += use32 ? 1000000u : 0u;
#else
        if (CQB_DIAG_COUNTS) n_active += (unsigned)(r >> 24) & 1u;
#endif
      }
      ev += (uint32_t)J;  // prev + (J - 1) candidates: the reference's count
      J_of[q] = (uint32_t)J;
      nlab[q] = best;
    }
    if (kSched) {  // this chunk's cost for the next iteration's order
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const uint32_t c = __reduce_max_sync(0xffffffffu, idx[q] < hi ? (unsigned)J_of[q] : 0u);
        if (lane == 0 && chunk[q] < my_ch) chunk_sched().cost[chunk[q]] = (uint8_t)min(c, 255u);
      }
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const uint32_t i = idx[q];
      const bool v = i < hi;
      const bool ch = v && nlab[q] != lab[q];
      uint32_t cnt = 0;
      const bool now = full || !kMQ;  // the count is needed here (else when the queue is applied)
      uint32_t ci = i;  // where the sample's count lives
      if constexpr (R) {
        const ResSamples rs = res_samples(L.res_cap);
        const uint32_t li = (chunk[q] << 5) + lane;
        ci = li;
        if (v && (full || ch) && now) cnt = rs.cnt[li];
        if (ch) rs.lab[li] = (uint8_t)nlab[q];
      } else {
        if (v && (full || ch) && now) cnt = counts[i];
      }
      if (ch) {
        labels[i] = (uint8_t)nlab[q];
        if (CQB_DIAG_COUNTS) ++n_changed;
      }
      if (full) {
        acc_point_warp(S.accp, v, nlab[q], key[q], cnt);
      } else if constexpr (kMQ) {
        const unsigned m = __ballot_sync(0xffffffffu, ch);
        if (m) {
          if (qn + (uint32_t)__popc(m) > 32u) apply_moves();
          if (ch) {
            const uint32_t slot = qn + __popc(m & ((1u << lane) - 1u));
            mq[slot][0] = ci | ((uint32_t)nlab[q] << 24);
            mq[slot][1] = key[q] | ((uint32_t)lab[q] << 24);
          }
          qn += __popc(m);
        }
      } else if (ch) {
        acc_move(S.accm, S.accp, lab[q], nlab[q], key[q], cnt);
      }
    }
  }
  if (kMQ && qn) apply_moves();
  evals += ev;
}

// Block reduction of a double-double in a fixed tree (deterministic).
__device__ dd block_sum_dd(LoopSmem& S, dd v) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd w{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    v = dd_add(v, w);
  }
  __syncthreads();
  if (lane == 0) {
    S.red_hi[wid] = v.hi;
    S.red_lo[wid] = v.lo;
  }
  __syncthreads();
  dd tot{0.0, 0.0};
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot = dd_add(tot, dd{S.red_hi[w], S.red_lo[w]});
  return tot;
}

// One fixed-tree block reduction of (double-double, int, int).
__device__ void block_sum3(LoopSmem& S, dd& v, int& a, int& b) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd w{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    v = dd_add(v, w);
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  if (lane == 0) {
    S.red_hi[wid] = v.hi;
    S.red_lo[wid] = v.lo;
    S.red_i[wid] = a;
    S.red_j[wid] = b;
  }
  __syncthreads();
  if (wid == 0) {  // fixed shuffle tree over the (<= 32) warp partials
    const int nw = (int)(blockDim.x >> 5);
    dd x = lane < nw ? dd{S.red_hi[lane], S.red_lo[lane]} : dd{0.0, 0.0};
    int xa = lane < nw ? S.red_i[lane] : 0, xb = lane < nw ? S.red_j[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dd w{__shfl_xor_sync(0xffffffffu, x.hi, o), __shfl_xor_sync(0xffffffffu, x.lo, o)};
      x = dd_add(x, w);
      xa += __shfl_xor_sync(0xffffffffu, xa, o);
      xb += __shfl_xor_sync(0xffffffffu, xb, o);
    }
    if (lane == 0) {
      S.red_hi[0] = x.hi;
      S.red_lo[0] = x.lo;
      S.red_i[0] = xa;
      S.red_j[0] = xb;
    }
  }
  __syncthreads();
  v = dd{S.red_hi[0], S.red_lo[0]};
  a = S.red_i[0];
  b = S.red_j[0];
}

__device__ int block_sum_int(LoopSmem& S, int v) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) S.red_i[wid] = v;
  __syncthreads();
  int tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += S.red_i[w];
  return tot;
}

// Reseed candidate: lexicographic max of (d, -index) — update_centers'
// strict '>' scan in index order (kmeans.hpp:272-289).
__device__ __forceinline__ bool cand_better(double d, unsigned int i, double bd, unsigned int bi) {
  return d > bd || (d == bd && i < bi);
}

// ---------------------------------------------------------------------------
// In-kernel exchange between ranks (sharded loop, BASELINE config 4).
//
// Each rank owns an exchange window (XB_BYTES, cudaMalloc'd, exported by IPC
// handle so every peer maps it over NVLink/NVSwitch):
//   u64 flag[src]   at XB_FLAG + 16*src  (own 128-B line per source)
//   u64 seq         at XB_SEQ            (this rank's exchange counter, kept across launches)
//   u64 payload[2][XMAX][5*KMAX] at XB_PAY  (slot parity = exchange number & 1)
//   u8  labels[2^24] at byte XB_LAB_OFF  (the rank's sample labels during the loop; after the
//                                         map epilogue, every rank's final palette indices)
// Exchange number s: every source writes its payload into slot s&1 of every
// rank's window with plain stores, then (one thread, after bar.sync) a
// sys-scope acq_rel fence and a relaxed store of s into flag[source]; a
// receiver polls its own flags with sys-scope acquire loads until all are
// >= s and reads the payload from L2 (ld.cg). Slot s&1 is rewritten only by
// exchange s+2, which a source starts after receiving this rank's exchange
// s+1, sent after this rank finished reading exchange s; so two slots
// suffice, and the monotonic counters need no reset between launches (every
// rank makes the same exchanges: the decisions are computed from identical
// totals). One exchange per iteration carries the K x 5 exact moment sums;
// the rare empty-cluster reseed adds one per empty cluster (its candidate).
constexpr int XMAX = 8;
constexpr int XB_FLAG = 0;
constexpr int XB_SEQ = XMAX * 16;
constexpr int XB_PAY = XB_SEQ + 128;
constexpr int XB_SLOT = 5 * KMAX;
// the per-iteration moment exchange in "LL" words: each u64 sum travels as
// two words {32 data bits, the exchange number's low 32 bits}, so a receiver
// polls the data itself (8-B stores are single-copy atomic) — no sender
// fence, no flag round trip
constexpr int XB_LL_SLOT = 2 * 5 * KMAX;
constexpr int XB_LL = XB_PAY + 2 * XMAX * XB_SLOT;
constexpr size_t XB_LAB_OFF = 512 * 1024;
constexpr size_t XB_BYTES = XB_LAB_OFF + (size_t(1) << 24);
static_assert((XB_LL + 2 * XMAX * XB_LL_SLOT) * sizeof(unsigned long long) <= XB_LAB_OFF, "window layout");
#ifndef CQB_XLL
#define CQB_XLL 1
#endif
// A dead peer fails the call instead of hanging: LoopParams::xch_timeout_ns
// (cqb_xch_set_timeout; default 5 s), and 4x that for the first exchange of
// a launch, whose peers may still be starting their own launch.
constexpr unsigned long long XCH_TIMEOUT_NS = 5000000000ull;

__device__ __forceinline__ unsigned long long* xpay(unsigned long long* box, unsigned long long s, int src) {
  return box + XB_PAY + ((size_t)(s & 1) * XMAX + src) * XB_SLOT;
}
// Thread 0 only, after the payload stores are ordered by bar.sync: publish s.
__device__ __forceinline__ unsigned long long* xll(unsigned long long* box, unsigned long long s, int src) {
  return box + XB_LL + ((size_t)(s & 1) * XMAX + src) * XB_LL_SLOT;
}
// two LL words in one 16-B store (each 8-B half is single-copy atomic, which
// is all the protocol needs)
__device__ __forceinline__ void ll_store2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
// Spin until word p carries exchange tag `tag` (or the exchange failed).
__device__ __forceinline__ unsigned long long ll_wait(const unsigned long long* p, uint32_t tag, int* status,
                                                      unsigned long long t0, unsigned long long limit) {
  for (;;) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if ((uint32_t)(v >> 32) == tag) return v;
    if (*reinterpret_cast<volatile int*>(status) == ST_XCH_TIMEOUT) return 0ull;
    if (globaltimer() - t0 > limit) {
      atomicExch(status, ST_XCH_TIMEOUT);
      return 0ull;
    }
  }
}

__device__ __forceinline__ void xch_signal(unsigned long long* box, int src, unsigned long long s) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(box + XB_FLAG + 16 * src), "l"(s) : "memory");
}
// The per-iteration K x 5 moment all-reduce in LL words (block-wide; inline:
// out of line, the call's register save spills into the points loop): block pb < xw of every
// part sends its part's sums to part pb; every block sums the xw sources.
__device__ __forceinline__ void xch_moments_ll(unsigned long long* dst_box, unsigned long long* own, int part,
                                            unsigned int pb, int xw,
                                            unsigned long long s, int k, const unsigned long long* gacc,
                                            unsigned long long* tot, bool silent, int* status,
                                            unsigned long long limit) {
  const int tid = threadIdx.x;
  const uint32_t tag = (uint32_t)s;
  if (pb < (unsigned)xw && !silent) {
    unsigned long long* dst = xll(dst_box, s, part);
    const unsigned long long hi = (unsigned long long)tag << 32;
    for (int e = tid; e < 5 * KMAX; e += blockDim.x)
      if ((e & (KMAX - 1)) < k) {
        const unsigned long long v = __ldcg(&gacc[e]);
        ll_store2(dst + 2 * e, (v & 0xffffffffull) | hi, (v >> 32) | hi);
      }
  }
  const unsigned long long t0 = globaltimer();
  for (int e = tid; e < 5 * KMAX; e += blockDim.x)
    if ((e & (KMAX - 1)) < k) {
      // two sources' words in flight at a time; only late words are polled
      unsigned long long a = 0;
      for (int r = 0; r < xw; r += 2) {
        const unsigned long long* s0 = xll(own, s, r) + 2 * e;
        const unsigned long long* s1 = xll(own, s, r + 1) + 2 * e;
        ulonglong2 v0 = __ldcg(reinterpret_cast<const ulonglong2*>(s0));
        ulonglong2 v1 = r + 1 < xw ? __ldcg(reinterpret_cast<const ulonglong2*>(s1)) : make_ulonglong2(0ull, 0ull);
        if ((uint32_t)(v0.x >> 32) != tag) v0.x = ll_wait(s0, tag, status, t0, limit);
        if ((uint32_t)(v0.y >> 32) != tag) v0.y = ll_wait(s0 + 1, tag, status, t0, limit);
        a += (v0.x & 0xffffffffull) | ((v0.y & 0xffffffffull) << 32);
        if (r + 1 < xw) {
          if ((uint32_t)(v1.x >> 32) != tag) v1.x = ll_wait(s1, tag, status, t0, limit);
          if ((uint32_t)(v1.y >> 32) != tag) v1.y = ll_wait(s1 + 1, tag, status, t0, limit);
          a += (v1.x & 0xffffffffull) | ((v1.y & 0xffffffffull) << 32);
        }
      }
      tot[e] = a;
    }
  __syncthreads();
}

// Block-wide: wait until all xw sources published exchange s into `box`.
__device__ __forceinline__ void xch_wait(unsigned long long* box, int xw, unsigned long long s, int* status,
                                         unsigned long long timeout_ns) {
  if (threadIdx.x < (unsigned)xw) {
    const unsigned long long* f = box + XB_FLAG + 16 * threadIdx.x;
    const unsigned long long t0 = globaltimer();
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= s) break;
      if (*reinterpret_cast<volatile int*>(status) == ST_XCH_TIMEOUT) break;
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(status, ST_XCH_TIMEOUT);
        break;
      }
    }
  }
  __syncthreads();
}

// Empty-cluster reseed (kmeans.hpp:268-290), grid-wide, all blocks agree.
// Candidates are ordered by (distance desc, first-occurrence rank asc): the
// reference's strict '>' scan in sample order. Unique colors are distinct, so
// "color already taken" is "rank already taken". Sharded (X != 0): each part
// (rank) reduces its own candidates, the parts exchange them (xch above) and
// every block picks the same global best.
template <int X>
__device__ void reseed_empty(LoopSmem& S, const LoopParams& L, cg::grid_group& grid, unsigned long long lo,
                             unsigned long long hi, int part, unsigned long long& xs) {
  WsmState* st = L.st;
  const unsigned int pb = part_block<X>(S), pG = part_size<X>(S);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned long long T = (unsigned long long)pG * blockDim.x;
  for (int e = 0; e < S.n_empty; ++e) {
    double bd = -1.0;
    unsigned int bi = 0xffffffffu, bk = 0u;
    for (unsigned long long i = lo + (unsigned long long)pb * blockDim.x + threadIdx.x; i < hi; i += T) {
      const unsigned int rk = L.rank[i];
      bool used = false;
      for (int t = 0; t < e; ++t) used |= (S.taken[t] == rk);
      if (used) continue;
      const uint32_t key = L.keys[i];
      const int m = L.labels[i];
      const double d = dist2_rn((double)key_r(key), (double)key_g(key), (double)key_b(key), S.cx[m], S.cy[m], S.cz[m]);
      if (cand_better(d, rk, bd, bi)) {
        bd = d;
        bi = rk;
        bk = key;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const unsigned int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const unsigned int ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (cand_better(od, oi, bd, bi)) {
        bd = od;
        bi = oi;
        bk = ok;
      }
    }
    __syncthreads();
    if (lane == 0) {
      S.red_hi[wid] = bd;
      S.red_i[wid] = (int)bi;
      S.red_j[wid] = (int)bk;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double xd = -1.0;
      unsigned int xi = 0xffffffffu, xk = 0u;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        if (cand_better(S.red_hi[w], (unsigned int)S.red_i[w], xd, xi)) {
          xd = S.red_hi[w];
          xi = (unsigned int)S.red_i[w];
          xk = (unsigned int)S.red_j[w];
        }
      st->cand_d[e & 1][blockIdx.x] = __double_as_longlong(xd);
      st->cand_i[e & 1][blockIdx.x] = xi;
      st->cand_k[e & 1][blockIdx.x] = xk;
    }
    grid.sync();
    if constexpr (X == 0) {
      if (threadIdx.x == 0) {
        double xd = -1.0;
        unsigned int xi = 0xffffffffu, xk = 0u;
        for (unsigned int b = 0; b < gridDim.x; ++b) {
          const double d = __longlong_as_double((long long)st->cand_d[e & 1][b]);
          const unsigned int i = st->cand_i[e & 1][b];
          if (cand_better(d, i, xd, xi)) {
            xd = d;
            xi = i;
            xk = st->cand_k[e & 1][b];
          }
        }
        S.taken[e] = xi;
        const int ke = S.empty_list[e];
        S.nx[ke] = (double)key_r(xk);
        S.ny[ke] = (double)key_g(xk);
        S.nz[ke] = (double)key_b(xk);
      }
      __syncthreads();
      continue;
    }
    // this part's blocks are [blockIdx.x - pb, blockIdx.x - pb + pG)
    const unsigned int b0 = blockIdx.x - pb, nb = pG;
    double xd = -1.0;
    unsigned int xi = 0xffffffffu, xk = 0u;
    if (threadIdx.x == 0 && pb == 0) {
      for (unsigned int b = b0; b < b0 + nb; ++b) {
        const double d = __longlong_as_double((long long)st->cand_d[e & 1][b]);
        const unsigned int i = st->cand_i[e & 1][b];
        if (cand_better(d, i, xd, xi)) {
          xd = d;
          xi = i;
          xk = st->cand_k[e & 1][b];
        }
      }
    }
    if constexpr (X != 0) {
      const unsigned long long s = ++xs;
      if (threadIdx.x == 0 && pb == 0)
        for (int r = 0; r < L.xw; ++r) {
          unsigned long long* dst = xpay(L.xbox[r], s, part);
          dst[0] = (unsigned long long)__double_as_longlong(xd);
          dst[1] = xi;
          dst[2] = xk;
          xch_signal(L.xbox[r], part, s);
        }
      unsigned long long* own = L.xbox[part];
      xch_wait(own, L.xw, s, &st->status, L.xch_timeout_ns);
      if (threadIdx.x == 0) {
        xd = -1.0;
        xi = 0xffffffffu;
        xk = 0u;
        for (int r = 0; r < L.xw; ++r) {
          const unsigned long long* src = xpay(own, s, r);
          const double d = __longlong_as_double((long long)__ldcg(&src[0]));
          const unsigned int i = (unsigned int)__ldcg(&src[1]);
          if (cand_better(d, i, xd, xi)) {
            xd = d;
            xi = i;
            xk = (unsigned int)__ldcg(&src[2]);
          }
        }
      }
    }
    if (threadIdx.x == 0) {
      S.taken[e] = xi;
      const int ke = S.empty_list[e];
      S.nx[ke] = (double)key_r(xk);
      S.ny[ke] = (double)key_g(xk);
      S.nz[ke] = (double)key_b(xk);
    }
    __syncthreads();
  }
}

// Flush the block's moment deltas into the global exact sums (u64, modular).
__device__ void flush_moments(LoopSmem& S, unsigned long long* gacc, int k) {
  for (int e = threadIdx.x; e < 5 * KMAX; e += blockDim.x) {
    if ((e & (KMAX - 1)) >= k) continue;
    const uint2 a = S.accp[e], m = S.accm[e];
    const unsigned long long d = ((unsigned long long)a.y << 32 | a.x) - ((unsigned long long)m.y << 32 | m.x);
    if (d) atomicAdd(&gacc[e], d);
    S.accp[e] = make_uint2(0u, 0u);
    S.accm[e] = make_uint2(0u, 0u);
  }
}

// The persistent, cooperative WSM loop (run_weighted_kmeans, kmeans.hpp:336-376).
template <int X, bool STAGE>
__device__ void map_epilogue(LoopSmem& S, const LoopParams& L, cg::grid_group& grid, unsigned long long n,
                                          unsigned long long lo, unsigned long long hi, int part,
                                          unsigned long long& xs);

// One instantiation per assignment variant (WSM, KM, FKM): a single kernel
// with a runtime switch cost the WSM loop ~1.5% (register allocation).
// Grid barrier of the persistent loop (one per phase boundary). Thread 0 of
// each block: acq_rel fence (the block's writes, ordered by the preceding
// bar.sync, become visible), one relaxed add to the counter, then acquire
// loads until every block has arrived; the other threads wait at bar.sync.
// Same ordering as cooperative_groups' grid.sync, with a payload: block 0
// adds its stop decision to the high half, so no block needs a separate L2
// round trip to learn whether the loop ends. wait = false: arrive only (the
// block's writes are published; it does not wait for the others).
__device__ __forceinline__ unsigned long long loop_barrier(LoopSmem& S, unsigned long long* bar, unsigned int target,
                                                           unsigned long long add, bool wait = true) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(bar), "l"(add) : "memory");
    unsigned long long v = 0;
    while (wait) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
      if ((unsigned int)v >= target) break;
    }
    S.barv = v;
  }
  __syncthreads();
  return S.barv;
}

// X: 0 = one rank (or a host-driven shard step); 1 = one process per GPU,
// moments exchanged over NVLink inside the loop; 2 = the same exchange among
// L.xw block groups of this launch (single-GPU emulation of the ranks).
// R: resident samples (ResSamples; small sample sets, X == 0 only).
template <int PPT, int X, bool R = false>
__global__ void __launch_bounds__(LOOP_THREADS, CQB_LOOP_MINB) k_wsm_loop(LoopParams L) {
  __shared__ LoopSmem S;
  extern __shared__ __align__(16) unsigned char dyn[];
  cg::grid_group grid = cg::this_grid();
  constexpr bool kLoopE = PPT >= 2 ? CQB_EDIFF != 0 : CQB_EDIFF_SMALL != 0;  // assign_sort_means reads rowE
  WsmState* st = L.st;
  const int tid = threadIdx.x;
  const int k = L.k;
  if (st->status != ST_OK) return;  // uniform across the grid
  if (L.block_times && tid == 0) L.block_times[12 * gridDim.x + blockIdx.x] = globaltimer();  // kernel entry
  const unsigned long long n = *L.n_ptr;
  // this block's part of the grid: the whole grid, or (X == 2) block group
  // `part` of xw; the part's ranks own shard_range(n, xw, part)
  const int part = X == 2 ? (int)(blockIdx.x / (gridDim.x / (unsigned)L.xw)) : (X == 1 ? L.xrank : 0);
  if (X == 2 && tid == 0) {
    S.part_g = gridDim.x / (unsigned)L.xw;
    S.part_b = blockIdx.x % S.part_g;
  }
  unsigned long long lo, hi;
  if constexpr (X != 0) {
    lo = n * (unsigned long long)part / (unsigned long long)L.xw;
    hi = n * (unsigned long long)(part + 1) / (unsigned long long)L.xw;
  } else {
    lo = L.shard_lo < n ? L.shard_lo : n;
    hi = L.shard_hi_or_max < n ? L.shard_hi_or_max : n;
  }
  const double inv_P = 1.0 / (double)L.total;
  // exact running sums of this rank's samples (zeroed by the host per launch)
  unsigned long long* gacc = X == 2 ? L.xacc + (size_t)part * 5 * KMAX : st->acc;
  // sharded: the totals over all ranks, rebuilt in shared memory every iteration
  // (the block's delta arrays are idle between the flush and the next assign)
  unsigned long long* tot = X ? reinterpret_cast<unsigned long long*>(S.accp) : gacc;
  unsigned long long xs = 0;  // exchange counter (X != 0), identical in every block of every rank
  if constexpr (X != 0) xs = __ldcg(L.xbox[part] + XB_SEQ);
  unsigned long long* tl = L.timeline;
  const bool rec = tl && blockIdx.x == 0 && tid == 0;
  (void)dyn;

  int big = 0;  // a center outside (-256, 256): no FP32 screening in this launch (scan_f32's bound)
  for (int t = tid; t < k; t += blockDim.x) {
    S.cx[t] = st->C[0][3 * t];
    S.cy[t] = st->C[0][3 * t + 1];
    S.cz[t] = st->C[0][3 * t + 2];
    loop_c4()[t] = make_float4(__double2float_rn(S.cx[t]), __double2float_rn(S.cy[t]), __double2float_rn(S.cz[t]), 0.f);
    big |= !(fabs(S.cx[t]) < 256.0 && fabs(S.cy[t]) < 256.0 && fabs(S.cz[t]) < 256.0);
  }
  big = __syncthreads_or(big);
  for (int t = tid; t < 5 * KMAX; t += blockDim.x) {
    S.accp[t] = make_uint2(0u, 0u);
    S.accm[t] = make_uint2(0u, 0u);
  }
  for (int j = tid; j < SCHED_MAX; j += blockDim.x) {  // identity order until costs are known
      chunk_sched().order[j] = (uint16_t)j;
      chunk_sched().cost[j] = 0;
    }
  if (tid == 0) {
    S.stamp = nullptr;
    S.wq = 0u;
    S.debug = L.debug_flags;
    S.f32ok = !big && !(L.debug_flags & DBG_NO_F32);
    // Longest-first chunk order on the large path: it pays when chunk costs
    // are uneven (photo-like images: cfg3 -9%) and costs when they are even
    // (a sample set that fills color space, cfg4: +9%). Unique colors per
    // pixel tell the two apart: below 1/2 the samples are sparse in the cube.
    S.sched_on = CQB_SCHED_LARGE && n * 2 < L.total && !(L.debug_flags & DBG_NO_SCHED_LARGE);

    S.rowo_row[0] = S.rowo_row[1] = -1;
  }
  __syncthreads();
  if (L.block_times && tid == 0) {  // profiling: SM of this block, evaluations in stamp_iter
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    L.block_times[6 * gridDim.x + blockIdx.x] = smid;
    L.block_times[7 * gridDim.x + blockIdx.x] = 0ull;
  }
  // prologue: tables of the initial centers (all pairs evaluated: non-incremental)
  if constexpr (R) {  // the block's chunks into shared memory (labels: unless iteration 1 writes them)
    const ResSamples rs = res_samples(L.res_cap);
    const unsigned long long nch = (hi - lo + 31) >> 5;
    const unsigned long long my = nch > blockIdx.x ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    for (unsigned long long li = tid; li < my * 32; li += blockDim.x) {
      const unsigned long long i = lo + ((blockIdx.x + gridDim.x * (li >> 5)) << 5) + (li & 31);
      if (i < hi) {
        rs.key[li] = L.keys[i];
        rs.cnt[li] = L.counts[i];
        if (!L.dense_first) rs.lab[li] = L.labels[i];
      }
    }
  }
  if (L.map_cellw)  // the epilogue's coarse cells start empty (read only after the loop's barriers)
    for (uint32_t c = blockIdx.x * blockDim.x + tid; c < (uint32_t)COARSE_CELLS; c += gridDim.x * blockDim.x)
      L.map_cellw[c] = 0u;
  // scan_f32 rows: +inf after the k - 1 entries
  for (int p = blockIdx.x; p < k; p += gridDim.x)
      for (int i = k - 1 + tid; i < ROW32; i += blockDim.x) {
        st->rowD32[p * ROW32 + i] = F32_INF;
        st->rowO[p * ROW32 + i] = 0;
      }
  tables_all(S, st, k, false, kLoopE);
  unsigned long long evals = 0;  // this thread's point evaluations (flushed once at exit)
  // pair evaluations of the center tables (block 0 only); none in naive mode
  // (sharded over processes: counted by rank 0 only)
  unsigned long long pair_evals = (X == 1 && L.xrank != 0)
                                      ? 0ull
                                      : (unsigned long long)k * (unsigned long long)(k - 1) / 2;
  if (CQB_LOOP_BARRIER && blockIdx.x == 0 && tid == 0) st->bar = 0ull;  // before the prologue barrier
  grid.sync();
  unsigned int bar_target = 0;  // loop_barrier episodes x G

  double prev_sse = __longlong_as_double(0x7ff0000000000000LL);  // +inf (block 0)
  for (int it = 1;; ++it) {
    const bool rec_it = rec && it <= L.hist_cap;
    if (rec_it) tl[(it - 1) * 8 + 0] = globaltimer();
    BLOCK_STAMP(0);
    // ---------------- assign(it) ----------------
    if (it == 1 && L.dense_first) {
      for (int t = tid; t < k; t += blockDim.x) {
        const uint32_t key = ((uint32_t)S.cx[t] << 16) | ((uint32_t)S.cy[t] << 8) | (uint32_t)S.cz[t];
        S.cb[t] = make_int2((int)key, key_dot(key, key) * 256 + t);
        S.row0[t] = (uint32_t)st->sortedD[t];  // row 0 (p = 0), integer-valued
      }
      __syncthreads();
      if (rec_it) tl[(it - 1) * 8 + 1] = globaltimer();
      assign_dense_first<X>(S, L, lo, hi, evals);
    } else {
      // no block barrier here: the grid barrier that ended the previous
      // iteration already ordered everything this assign reads (S.wq was
      // reset after the previous assign)
      if (rec_it) tl[(it - 1) * 8 + 1] = globaltimer();
      unsigned int n_changed = 0, n_deep = 0;
      const unsigned long long ev0 = evals;
      if constexpr (PPT == 1) {
        assign_sort_means<PPT, X, R, true>(S, L, lo, hi, it == 1, evals, n_changed, n_deep);
      } else if (CQB_SCHED_LARGE && S.sched_on) {
        assign_sort_means<PPT, X, R, CQB_SCHED_LARGE != 0>(S, L, lo, hi, it == 1, evals, n_changed, n_deep);
      } else {
        assign_sort_means<PPT, X, R, false>(S, L, lo, hi, it == 1, evals, n_changed, n_deep);
      }
      if (L.block_times && it == L.stamp_iter) {
        const unsigned long long v = warp_sum(evals - ev0);
        if ((tid & 31) == 0) atomicAdd(&L.block_times[7 * gridDim.x + blockIdx.x], v);
      }
      if (rec_it || (tl && it <= L.hist_cap)) {  // diagnostics: label churn and deep scans
        const unsigned long long v = ((unsigned long long)warp_sum(n_deep) << 32) | warp_sum(n_changed);
        if ((tid & 31) == 0 && v) atomicAdd(&tl[(it - 1) * 8 + 7], v);
      }
    }
    __syncthreads();
    if (tid == 0) S.wq = 0u;  // every warp has left the chunk loop; the next assign reads it after two grid barriers
    if (rec_it) tl[(it - 1) * 8 + 2] = globaltimer();
    BLOCK_STAMP(1);
    flush_moments(S, gacc, k);
    // next iteration's longest-first chunk order (this block's chunks are
    // done); small sample sets only (latency-bound), re-sorted at iterations
    // 2, 4, 8, ... (costs drift slowly; the sort is not free)
    if ((PPT == 1 || (CQB_SCHED_LARGE && S.sched_on)) && it >= 2 && (it & (it - 1)) == 0) {
      const unsigned long long nn = hi - lo, nch = (nn + 31) >> 5;
      const uint32_t pb = part_block<X>(S), pG = part_size<X>(S);
      const uint32_t my_ch = nch > pb ? (uint32_t)((nch - 1 - pb) / pG + 1) : 0u;
      if (my_ch <= (uint32_t)SCHED_MAX) sched_sort(my_ch);
    }
    if (rec_it) tl[(it - 1) * 8 + 3] = globaltimer();
    BLOCK_STAMP(2);
    if (CQB_LOOP_BARRIER) {
      bar_target += gridDim.x;
      // sharded: only the sending blocks need every local flush; the others
      // read the totals from the exchange (each rank sends after its own
      // barrier), so they arrive without waiting
      const bool waits = X == 0 || part_block<X>(S) < (unsigned)L.xw;
      loop_barrier(S, &st->bar, bar_target, 1ull, waits);
    } else {
      grid.sync();
    }
    if (rec_it) tl[(it - 1) * 8 + 4] = globaltimer();
    BLOCK_STAMP(3);
    if (L.moments_only) break;
    if constexpr (R) {
      if (it == 1 && L.dense_first) {  // iteration 1 wrote the labels in its own (dense) order
        const ResSamples rs = res_samples(L.res_cap);
        const unsigned long long nch = (hi - lo + 31) >> 5;
        const unsigned long long my = nch > blockIdx.x ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
        for (unsigned long long li = tid; li < my * 32; li += blockDim.x) {
          const unsigned long long i = lo + ((blockIdx.x + gridDim.x * (li >> 5)) << 5) + (li & 31);
          if (i < hi) rs.lab[li] = __ldcg(&L.labels[i]);
        }
      }
    }
    if constexpr (X != 0) {  // all-reduce of the K x 5 moment sums over the ranks
      const unsigned long long s = ++xs;
      const unsigned int pb = part_block<X>(S);
      // (debug flag 32768, tests only: part 1 goes silent at iteration 3 - a dead peer)
      const bool silent = (L.debug_flags & 32768) && part == 1 && it >= 3;
      const unsigned long long limit = it == 1 ? 4 * L.xch_timeout_ns : L.xch_timeout_ns;
      if (CQB_XLL) {
        xch_moments_ll(pb < (unsigned)L.xw ? L.xbox[pb] : nullptr, L.xbox[part], part, pb, L.xw, s, k, gacc, tot,
                       silent, &st->status, limit);
      } else {
        if (pb < (unsigned)L.xw && !silent) {  // block pb of every part sends to rank pb
          unsigned long long* dst = xpay(L.xbox[pb], s, part);
          for (int e = tid; e < 5 * KMAX; e += blockDim.x)
            if ((e & (KMAX - 1)) < k) dst[e] = __ldcg(&gacc[e]);
          __syncthreads();
          if (tid == 0) xch_signal(L.xbox[pb], part, s);
        }
        unsigned long long* own = L.xbox[part];
        xch_wait(own, L.xw, s, &st->status, limit);
        for (int e = tid; e < 5 * KMAX; e += blockDim.x)
          if ((e & (KMAX - 1)) < k) {
            unsigned long long a = 0;
            for (int r = 0; r < L.xw; ++r) a += __ldcg(xpay(own, s, r) + e);
            tot[e] = a;
          }
        __syncthreads();
      }
    }

    // ---------------- finalize(it) ----------------
    // Every block: new centers S/N (FP64, exact integer inputs) + empty count.
    // One division per thread: unit u = (channel, cluster) over 3*KMAX units
    // (one unit per thread at 1024 threads), each loading its sum and N in one
    // L2 round trip.
    int empt_local = 0;
    // block 0 (SSE + termination): thread t loads all five moments of cluster
    // t in one L2 round trip and keeps them for the SSE below; the other
    // blocks split the 3k coordinates over their threads
    const bool b0f = (PPT == 1 || CQB_B0F_LARGE) && blockIdx.x == 0 && !(S.debug & 4096);
    unsigned long long mN = 0, mS0 = 0, mS1 = 0, mS2 = 0, mQ = 0;
    if (b0f && tid < k) {
      mN = ldmom<X != 0>(&tot[3 * KMAX + tid]);
      mS0 = ldmom<X != 0>(&tot[0 * KMAX + tid]);
      mS1 = ldmom<X != 0>(&tot[1 * KMAX + tid]);
      mS2 = ldmom<X != 0>(&tot[2 * KMAX + tid]);
      mQ = ldmom<X != 0>(&tot[4 * KMAX + tid]);
      if (mN) {
        S.nx[tid] = center_coord_v(mS0, mN, mS0, mS1, mS2, mQ, inv_P);
        S.ny[tid] = center_coord_v(mS1, mN, mS0, mS1, mS2, mQ, inv_P);
        S.nz[tid] = center_coord_v(mS2, mN, mS0, mS1, mS2, mQ, inv_P);
      } else {
        empt_local = 1;
      }
    }
    // blocks other than 0 need the old centers only for a reseed: they write
    // the new ones straight into the current set (one unit per thread), and
    // put the old ones back in the rare case that a cluster is empty
    const bool spec = LOOP_THREADS >= 3 * KMAX && blockIdx.x != 0 && !(S.debug & 8192);
    double oldc = 0.0;
    bool wrote = false;
    for (int u = tid; u < 3 * KMAX && !b0f; u += blockDim.x) {
      const int ch = u / KMAX, t = u % KMAX;
      if (t < k) {
        const unsigned long long N = ldmom<X != 0>(&tot[3 * KMAX + t]);
        const unsigned long long Sv = ldmom<X != 0>(&tot[ch * KMAX + t]);
        if (N) {
          const double c = center_coord<X != 0>(tot, KMAX, t, Sv, N, inv_P);
          (ch == 0 ? S.nx : (ch == 1 ? S.ny : S.nz))[t] = c;
          if (spec) {
            double* cur = ch == 0 ? S.cx : (ch == 1 ? S.cy : S.cz);
            oldc = cur[t];
            cur[t] = c;
            wrote = true;
          }
        } else if (ch == 0) {
          empt_local = 1;
        }
      }
    }
    const int empt = __syncthreads_count(empt_local);  // k <= blockDim: one cluster per thread
    const bool direct = spec && !empt;
    if (spec && empt) {  // rare: the reseed needs the old centers
      if (wrote) (tid < KMAX ? S.cx : (tid < 2 * KMAX ? S.cy : S.cz))[tid % KMAX] = oldc;
      __syncthreads();
    }
    BLOCK_STAMP(8);
    if (empt) {  // rare: empty clusters (uniform across the grid)
      if (tid == 0) {
        S.n_empty = empt;
        int m = 0;
        for (int t = 0; t < k; ++t)
          if (ldmom<X != 0>(&tot[3 * KMAX + t]) == 0ull) S.empty_list[m++] = t;
      }
      __syncthreads();
      reseed_empty<X>(S, L, grid, lo, hi, part, xs);
    }
    // Block 0: moment-form SSE, termination (kmeans.hpp:359-369), reporting.
    if (blockIdx.x == 0) {
      dd part{0.0, 0.0};
      int moved = 0, unused = 0;
      if (tid < k) {
        const int t = tid;
        moved += (S.nx[t] != S.cx[t]) | (S.ny[t] != S.cy[t]) | (S.nz[t] != S.cz[t]);
        if (!b0f) {
          mN = ldmom<X != 0>(&tot[3 * KMAX + t]);
          mS0 = ldmom<X != 0>(&tot[0 * KMAX + t]);
          mS1 = ldmom<X != 0>(&tot[1 * KMAX + t]);
          mS2 = ldmom<X != 0>(&tot[2 * KMAX + t]);
          mQ = ldmom<X != 0>(&tot[4 * KMAX + t]);
        }
        if (mN) {
          const double dn = (double)mN;
          const double Sr = (double)mS0, Sg = (double)mS1;
          const double Sb = (double)mS2, Q = (double)mQ;
          const double cr = S.cx[t], cgc = S.cy[t], cbc = S.cz[t];
          // Q - 2 c.S + |c|^2 N with the centers of THIS assignment
          dd cs = dd_add(dd_add(two_prod(cr, Sr), two_prod(cgc, Sg)), two_prod(cbc, Sb));
          dd c2 = dd_add(dd_add(two_prod(cr, cr), two_prod(cgc, cgc)), two_prod(cbc, cbc));
          dd term = dd_add(dd{Q, 0.0}, dd_scale(cs, -2.0));
          term = dd_add(term, dd_scale(c2, dn));
          part = dd_add(part, term);
        }
      }
      if (L.block_times && it == L.stamp_iter && tid == 0) L.block_times[15 * gridDim.x + 0] = globaltimer();
      block_sum3(S, part, moved, unused);
      if (L.block_times && it == L.stamp_iter && tid == 0) L.block_times[15 * gridDim.x + 1] = globaltimer();
      const double sse = fmax(__dadd_rn(part.hi, part.lo) * inv_P, 0.0);
      bool stop;
      if (L.mode == 0) {
        stop = it >= L.max_iters;
      } else {
        stop = (sse == 0.0) || ((prev_sse - sse) / sse <= L.eps) || (it >= L.cap);
      }
      prev_sse = sse;
      if (tid == 0) {
        if (it <= L.hist_cap) L.sse_hist[it - 1] = sse;
        st->iterations = it;
        st->sse = sse;
        if (empt) st->n_empty_events += empt;  // (rare: no global read-modify-write on the critical path)
        if (stop) st->stop_it = it;
        S.stop_flag = stop;
        // pair evaluations of the incremental table update (kmeans.hpp:137-155)
        if (!stop) {
          const unsigned long long still = (unsigned long long)(k - moved);
          pair_evals += (unsigned long long)k * (unsigned long long)(k - 1) / 2 - (still ? still * (still - 1) / 2 : 0ull);
        }
      }
      if (L.traj && it <= L.traj_cap)
        for (int t = tid; t < k; t += blockDim.x) {
          double* o = L.traj + ((size_t)(it - 1) * k + t) * 3;
          o[0] = S.nx[t];
          o[1] = S.ny[t];
          o[2] = S.nz[t];
        }
      if (stop)
        for (int t = tid; t < k; t += blockDim.x) {
          st->final_C[3 * t] = S.nx[t];
          st->final_C[3 * t + 1] = S.ny[t];
          st->final_C[3 * t + 2] = S.nz[t];
        }
    }
    if (L.block_times && it == L.stamp_iter && tid == 0 && blockIdx.x == 0) L.block_times[15 * gridDim.x + 2] = globaltimer();
    if (!direct) __syncthreads();  // (direct: the new centers were written before the count barrier)
    BLOCK_STAMP(9);
    if constexpr (X != 0)  // the delta accumulators again
      for (int e = tid; e < 5 * KMAX; e += blockDim.x) tot[e] = 0ull;
    if (!direct) {
      for (int t = tid; t < k; t += blockDim.x) {
        S.cx[t] = S.nx[t];
        S.cy[t] = S.ny[t];
        S.cz[t] = S.nz[t];
      }
      __syncthreads();
    }
    // FP32 copies for the next assign (read after the grid barrier); the new
    // centers are means of colors or colors, so |c| < 256 holds
    for (int t = tid; t < k; t += blockDim.x)
      loop_c4()[t] = make_float4(__double2float_rn(S.cx[t]), __double2float_rn(S.cy[t]), __double2float_rn(S.cz[t]), 0.f);
    if (rec_it) tl[(it - 1) * 8 + 5] = globaltimer();
    BLOCK_STAMP(4);
    if (tid == 0) S.stamp = (L.block_times && it == L.stamp_iter) ? L.block_times : nullptr;
    tables_all(S, st, k, true, kLoopE);  // wasted work on the final iteration only
    if (rec_it) tl[(it - 1) * 8 + 6] = globaltimer();
    BLOCK_STAMP(5);
    if (CQB_LOOP_BARRIER) {
      bar_target += gridDim.x;
      // block 0 also stops the whole grid, on the same iteration, when an
      // exchange timed out (every block then leaves through this barrier)
      const bool stop_here =
          blockIdx.x == 0 && (S.stop_flag || (X != 0 && *reinterpret_cast<volatile int*>(&st->status) != ST_OK));
      if ((loop_barrier(S, &st->bar, bar_target, 1ull + (stop_here ? (1ull << 32) : 0ull)) >> 32) != 0) break;
    } else {
      grid.sync();
      if (*reinterpret_cast<volatile int*>(&st->stop_it) == it) break;
    }
  }
  if (L.block_times && tid == 0) L.block_times[13 * gridDim.x + blockIdx.x] = globaltimer();  // loop exit
  // one evals flush per block (a per-warp atomic every iteration would
  // serialize thousands of same-address atomics in L2)
  evals = warp_sum(evals);
  __syncthreads();
  if ((tid & 31) == 0) S.red_u64[tid >> 5] = evals;
  __syncthreads();
  if (tid == 0) {
    unsigned long long tot = blockIdx.x == 0 ? pair_evals : 0ull;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += S.red_u64[w];
    atomicAdd(&st->evals, tot);
  }
  if constexpr (X != 0)
    if (part_block<X>(S) == 0 && tid == 0) L.xbox[part][XB_SEQ] = xs + (L.map_lut ? 1ull : 0ull);  // + the epilogue's exchange
  if constexpr (X != 0) {
    if (L.map_lut) map_epilogue<X, (PPT >= 2) && CQB_MAP_STAGE>(S, L, grid, n, lo, hi, part, xs);
  } else {
    unsigned long long none = 0;
    if (L.map_lut) map_epilogue<0, (PPT >= 2) && CQB_MAP_STAGE>(S, L, grid, hi, 0, 0, 0, none);
  }
  if (L.block_times && tid == 0) L.block_times[14 * gridDim.x + blockIdx.x] = globaltimer();  // kernel exit
}

// ---------------------------------------------------------------------------
// map_pixels' per-color work (image_ops.hpp:18-51) fused into the loop's tail,
// the same computation as k_map_tables + k_map_unique (map.cuh): rounded
// palette (lround, clamp), integer rows sorted by (d, index) - two rows per
// block, like the center tables - then, after a grid barrier, each unique
// color's exact argmin over the rounded palette from its final label with the
// strict break d(R_p, R_t) > 4 prev, the key -> index LUT and the exact
// u64 sum of count x error. Saves two launches on the quantize path.
// STAGE (large-image kernels, whose dynamic shared block has the room): the
// first MAPQ entries of every integer row are copied to shared memory after
// the rows' grid barrier, and a sample's scan reads them there (the rows are
// otherwise read entry by entry from L2: the epilogue took 180 us on cfg4).
constexpr int MAPQ = 16;
template <int X, bool STAGE>
__device__ void map_epilogue(LoopSmem& S, const LoopParams& L, cg::grid_group& grid, unsigned long long n,
                                          unsigned long long lo, unsigned long long hi, int part,
                                          unsigned long long& xs) {
  const int k = L.k, tid = threadIdx.x;
  const double* C = L.st->final_C;
  uint32_t* s_key = S.row0;        // rounded palette keys
  int* s_cc = S.empty_list;        // |R_t|^2
  int2* s_kc = S.cb;               // {key, |R_t|^2} (one load per evaluation)
  for (int t = tid; t < k; t += blockDim.x) {
    const uint32_t key = (round_chan(C[3 * t]) << 16) | (round_chan(C[3 * t + 1]) << 8) | round_chan(C[3 * t + 2]);
    s_key[t] = key;
    s_cc[t] = key_dot(key, key);
    s_kc[t] = make_int2((int)key, key_dot(key, key));
    if (blockIdx.x == 0) L.map_palkey[t] = key;
  }
  __syncthreads();
  {  // rows: same ownership as tables_all
    const int G = (int)gridDim.x;
    const int first = G == 1 ? 0 : (int)blockIdx.x - 1;
    const int stride = G == 1 ? 1 : G - 1;
    const int r = tid >> 9, t = tid & (KMAX - 1), h = (tid >> 8) & 1;
    for (int p0 = first; first >= 0 && p0 < k; p0 += 2 * stride) {
      const int p = r ? (p0 + stride < k ? p0 + stride : -1) : p0;
      if (p >= 0 && h == 0 && t < k) S.rowd[r][t] = (double)(s_cc[p] + s_cc[t] - 2 * key_dot(s_key[p], s_key[t]));
      __syncthreads();
      if (p >= 0 && t < k) {
        int cnt = 0;
        if (t != p) {
          const double dt = S.rowd[r][t];
          const int u0 = h * (KMAX / 2), u1 = min(k, u0 + KMAX / 2);
          for (int u = u0; u < u1; ++u) {
            const double du = S.rowd[r][u];
            cnt += (u != p) & ((du < dt) | ((du == dt) & (u < t)));
          }
        }
        S.rank_part[r][h][t] = cnt;
      }
      __syncthreads();
      if (p >= 0 && h == 0 && t < k) {
        const int rank = t == p ? 0 : 1 + S.rank_part[r][0][t] + S.rank_part[r][1][t];
        L.map_sortedDr[p * KMAX + rank] = t == p ? 0 : (int)S.rowd[r][t];
        L.map_orderR[p * KMAX + rank] = (uint8_t)t;
      }
      __syncthreads();
    }
  }
  grid.sync();
  // staged rows: entries 1..MAPQ of row p at q_d[p * (MAPQ + 1) + e] (padded: lanes on
  // neighbouring rows hit different banks), their order bytes at q_o[p * MAPQ + e]
  int* q_d = nullptr;
  uint8_t* q_o = nullptr;
  if constexpr (STAGE) {
    q_d = reinterpret_cast<int*>(loop_dyn_large().e0);
    q_o = reinterpret_cast<uint8_t*>(q_d + KMAX * (MAPQ + 1));
    static_assert(sizeof(LoopDynLarge::e0) >= KMAX * (MAPQ + 1) * 4 + KMAX * MAPQ, "staged map rows fit in the rowE stage");
    for (int u = tid; u < MAPQ * k; u += blockDim.x) {
      const int p = u / MAPQ, e = u % MAPQ;
      if (1 + e < k) {
        q_d[p * (MAPQ + 1) + e] = __ldcg(L.map_sortedDr + p * KMAX + 1 + e);
        q_o[p * MAPQ + e] = __ldcg(L.map_orderR + p * KMAX + 1 + e);
      }
    }
    __syncthreads();
  }
  // Sharded: each rank (part) maps its own samples [lo, hi). X = 1 sends the
  // palette indices into every rank's window (its label region, contiguous
  // stores), exchanges the partial error sums, and every rank then fills its
  // LUT for all samples from its window; X = 2 (one shared LUT) writes it
  // directly.
  const unsigned int pb = X == 2 ? part_block<X>(S) : blockIdx.x;
  const unsigned int pG = X == 2 ? part_size<X>(S) : gridDim.x;
  const unsigned long long a = X ? lo : 0ull, b = X ? hi : n;
  unsigned long long err = 0;
  // whole warps per step (consecutive Morton samples per warp: the coarse table's cell segments)
  const int lane = tid & 31;
  // the next step's sample (key, label, count) is loaded before this step's
  // scan: one L2 round trip per step hidden behind the previous scan
  const unsigned long long step = (unsigned long long)pG * blockDim.x;
  uint32_t nx = 0, ncnt = 0;
  int np = 0;
  auto fetch = [&](unsigned long long bs) {
    const unsigned long long i2 = bs + lane;
    if (i2 < b) {
      nx = L.keys[i2];
      np = X ? (int)__ldcg(&L.labels[i2]) : (int)L.labels[i2];
      ncnt = L.counts[i2];
    }
  };
  {
    const unsigned long long b0 = a + (unsigned long long)pb * blockDim.x + (tid & ~31);
    if (b0 < b) fetch(b0);
  }
  for (unsigned long long base = a + (unsigned long long)pb * blockDim.x + (tid & ~31); base < b; base += step) {
    const unsigned long long i = base + lane;
    const bool v = i < b;
    uint32_t x = nx;
    const int p = np;
    const uint32_t cnt = ncnt;
    if (base + step < b) fetch(base + step);
    int best = 0;
    if (v) {
      const int xx = key_dot(x, x);
      const int prev = xx + s_cc[p] - 2 * key_dot(x, s_key[p]);
      const int bound = 4 * prev;
      int mind = prev;
      best = p;
      const int* rowd = L.map_sortedDr + p * KMAX;
      const uint8_t* rowo = L.map_orderR + p * KMAX;
      auto eval = [&](int t) {
        const int2 kc = s_kc[t];
        const int d = xx + kc.y - 2 * key_dot(x, (uint32_t)kc.x);
        if (d < mind || (d == mind && t < best)) {
          mind = d;
          best = t;
        }
      };
      int j = 1;
      bool open = true;  // the scan has not met its break entry yet
      if constexpr (STAGE) {
        const int* qd = q_d + p * (MAPQ + 1);
        const uint8_t* qo = q_o + p * MAPQ;
        const int jm = min(k, MAPQ + 1);
        for (; j < jm; ++j) {
          if (qd[j - 1] > bound) { open = false; break; }
          eval(qo[j - 1]);
        }
      }
      if (open)
        for (; j < k; ++j) {
          if (rowd[j] > bound) break;
          eval(rowo[j]);
        }
      if constexpr (X == 1) {
        for (int r = 0; r < L.xw; ++r) (reinterpret_cast<uint8_t*>(L.xbox[r]) + XB_LAB_OFF)[i] = (uint8_t)best;
      } else {
        L.map_lut[x] = (uint8_t)best;
      }
      err += (unsigned long long)cnt * (unsigned long long)mind;
    }
    if (X != 1 && L.map_cellw) {
      const unsigned am = __ballot_sync(0xffffffffu, v);
      if (v) coarse_note(L.map_cellw, am, x, best);
    }
  }
  err = warp_sum(err);
  __syncthreads();
  if ((tid & 31) == 0) S.red_u64[tid >> 5] = err;
  __syncthreads();
  if (tid == 0) {
    unsigned long long tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += S.red_u64[w];
    if (tot) atomicAdd(&L.st->mse_err, tot);
  }
  if constexpr (X != 0) {
    grid.sync();  // this rank's indices and error partial are in place
    const unsigned long long s = ++xs;
    if (tid == 0 && blockIdx.x % pG == 0) {  // one sender per part
      if (X == 1) {
        const unsigned long long e = __ldcg(&L.st->mse_err);
        for (int r = 0; r < L.xw; ++r) *xpay(L.xbox[r], s, part) = e;
      }
      for (int r = 0; r < L.xw; ++r) xch_signal(L.xbox[r], part, s);
    }
    xch_wait(L.xbox[part], L.xw, s, &L.st->status, L.xch_timeout_ns);
    if constexpr (X == 1) {
      if (blockIdx.x == 0 && tid == 0) {  // the world's error sum (every rank reports the same MSE)
        unsigned long long e = 0;
        for (int r = 0; r < L.xw; ++r) e += __ldcg(xpay(L.xbox[part], s, r));
        L.st->mse_err = e;
      }
      const uint8_t* idx = reinterpret_cast<const uint8_t*>(L.xbox[part]) + XB_LAB_OFF;
      for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x + (tid & ~31); base < n;
           base += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = base + lane;
        const bool v = i < n;
        uint32_t x = 0;
        int best = 0;
        if (v) {
          x = L.keys[i];
          best = __ldcg(idx + i);
          L.map_lut[x] = (uint8_t)best;
        }
        if (L.map_cellw) {
          const unsigned am = __ballot_sync(0xffffffffu, v);
          if (v) coarse_note(L.map_cellw, am, x, best);
        }
      }
    }
  }
  if (L.map_cellw) {  // every cell noted: the compact table for k_map_pixels_coarse
    grid.sync();
    coarse_compact(L.map_cellw, L.map_coarse, blockIdx.x * blockDim.x + tid, gridDim.x * blockDim.x);
  }
}

// ---------------------------------------------------------------------------
// Sharded-run helpers (multi-GPU host driver, paper_1011_0093_b200/distributed.py).

// Device finalize of reduced moments (same math as the loop's finalize):
// new centers S/N, moment-form double-double SSE, ascending empty list.
// One block of KMAX threads.
__global__ void __launch_bounds__(KMAX) k_finalize(const unsigned long long* __restrict__ mom, const double* __restrict__ Cused,
                                                   int k, unsigned long long total, double* __restrict__ Cnew,
                                                   double* __restrict__ sse_out, int* __restrict__ n_empty_out,
                                                   int* __restrict__ empty_list) {
  __shared__ double s_hi[KMAX / 32], s_lo[KMAX / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  dd part{0.0, 0.0};
  int empty = 0;
  if (t < k) {
    const unsigned long long N = mom[3 * KMAX + t];
    if (N) {
      const double dn = (double)N;
      const double Sr = (double)mom[t], Sg = (double)mom[KMAX + t], Sb = (double)mom[2 * KMAX + t];
      const double Q = (double)mom[4 * KMAX + t];
      const double inv_P = 1.0 / (double)total;
      Cnew[3 * t] = center_coord(mom, KMAX, t, mom[t], N, inv_P);
      Cnew[3 * t + 1] = center_coord(mom, KMAX, t, mom[KMAX + t], N, inv_P);
      Cnew[3 * t + 2] = center_coord(mom, KMAX, t, mom[2 * KMAX + t], N, inv_P);
      const double cr = Cused[3 * t], cgc = Cused[3 * t + 1], cbc = Cused[3 * t + 2];
      dd cs = dd_add(dd_add(two_prod(cr, Sr), two_prod(cgc, Sg)), two_prod(cbc, Sb));
      dd c2 = dd_add(dd_add(two_prod(cr, cr), two_prod(cgc, cgc)), two_prod(cbc, cbc));
      dd term = dd_add(dd{Q, 0.0}, dd_scale(cs, -2.0));
      part = dd_add(term, dd_scale(c2, dn));
    } else {
      empty = 1;
      Cnew[3 * t] = Cused[3 * t];
      Cnew[3 * t + 1] = Cused[3 * t + 1];
      Cnew[3 * t + 2] = Cused[3 * t + 2];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd w{__shfl_xor_sync(0xffffffffu, part.hi, o), __shfl_xor_sync(0xffffffffu, part.lo, o)};
    part = dd_add(part, w);
  }
  const int ne = __syncthreads_count(empty);
  if (lane == 0) {
    s_hi[wid] = part.hi;
    s_lo[wid] = part.lo;
  }
  __syncthreads();
  if (t == 0) {
    dd tot{0.0, 0.0};
    for (int w = 0; w < KMAX / 32; ++w) tot = dd_add(tot, dd{s_hi[w], s_lo[w]});
    *sse_out = fmax(__dadd_rn(tot.hi, tot.lo) * (1.0 / (double)total), 0.0);
    *n_empty_out = ne;
    int m = 0;
    for (int c = 0; c < k; ++c)
      if (mom[3 * KMAX + c] == 0ull) empty_list[m++] = c;
  }
}

// Reseed candidate of a shard: lexicographic max of (dist to own center,
// -first-occurrence rank) over samples [lo, hi) whose rank is not taken.
__global__ void k_reseed_scan(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ rank,
                              const uint8_t* __restrict__ labels, unsigned long long lo, unsigned long long hi,
                              const double* __restrict__ C, const uint32_t* __restrict__ taken, int n_taken,
                              double* __restrict__ cand_d, unsigned int* __restrict__ cand_r,
                              unsigned int* __restrict__ cand_k) {
  __shared__ double sd[32];
  __shared__ unsigned int sr[32], sk[32];
  double bd = -1.0;
  unsigned int br = 0xffffffffu, bk = 0u;
  for (unsigned long long i = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned int rk = rank[i];
    bool used = false;
    for (int e = 0; e < n_taken; ++e) used |= taken[e] == rk;
    if (used) continue;
    const uint32_t key = keys[i];
    const int m = labels[i];
    const double d = dist2_rn((double)key_r(key), (double)key_g(key), (double)key_b(key), C[3 * m], C[3 * m + 1],
                              C[3 * m + 2]);
    if (cand_better(d, rk, bd, br)) {
      bd = d;
      br = rk;
      bk = key;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const unsigned int orr = __shfl_xor_sync(0xffffffffu, br, o);
    const unsigned int ok = __shfl_xor_sync(0xffffffffu, bk, o);
    if (cand_better(od, orr, bd, br)) {
      bd = od;
      br = orr;
      bk = ok;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sd[threadIdx.x >> 5] = bd;
    sr[threadIdx.x >> 5] = br;
    sk[threadIdx.x >> 5] = bk;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bd = sd[0];
    br = sr[0];
    bk = sk[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (cand_better(sd[w], sr[w], bd, br)) {
        bd = sd[w];
        br = sr[w];
        bk = sk[w];
      }
    cand_d[blockIdx.x] = bd;
    cand_r[blockIdx.x] = br;
    cand_k[blockIdx.x] = bk;
  }
}

__global__ void k_reseed_pick(const double* __restrict__ cand_d, const unsigned int* __restrict__ cand_r,
                              const unsigned int* __restrict__ cand_k, int nb, double* out_d,
                              unsigned int* out_r, unsigned int* out_k) {
  if (threadIdx.x != 0) return;
  double bd = -1.0;
  unsigned int br = 0xffffffffu, bk = 0u;
  for (int b = 0; b < nb; ++b)
    if (cand_better(cand_d[b], cand_r[b], bd, br)) {
      bd = cand_d[b];
      br = cand_r[b];
      bk = cand_k[b];
    }
  *out_d = bd;
  *out_r = br;
  *out_k = bk;
}

}  // namespace cqb
