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

namespace cqb {

namespace cg = cooperative_groups;

struct WsmState {
  double C[2][3 * KMAX];                  // center buffers [k*3 + ch]
  unsigned long long acc[5 * KMAX];       // exact sums [field*KMAX + k]: Sr, Sg, Sb, N, Q
  double sortedD[KMAX * KMAX];            // row p: d(c_p, c_order[p][j]) ascending
  uint8_t order[KMAX * KMAX];             // row p: [p, others by (d, index)]
  double final_C[3 * KMAX];
  uint32_t chosen[KMAX];                  // init: chosen sample indices
  unsigned long long cand_d[2][MAXBLK];   // reseed candidates (d bits, index)
  unsigned int cand_i[2][MAXBLK];
  unsigned long long evals;               // point + pair distance evaluations
  unsigned long long mse_err;             // Σ count * int distance (map pass)
  double sse;
  int iterations;
  int status;
  int n_empty_events;
};

struct LoopParams {
  const uint32_t* keys;
  const uint32_t* counts;
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
  unsigned long long* timeline;  // optional: per-iteration globaltimer stamps (5 per iteration)
};

// ---------------------------------------------------------------------------
// init_centers on device (kmeans.hpp:53-70): partial Fisher–Yates over
// iota(N') using the raw mt19937_64 stream computed on the host (the stream is
// independent of N'). bounded_rand's rejection + modulo (:43-49) are evaluated
// for all k draws in parallel (a rejection, probability < N'/2^64 per draw,
// diverts to the exact sequential path); the k swaps then run in one thread
// with positions >= k held in a small open-addressing map.
__global__ void __launch_bounds__(KMAX) k_init_centers(const uint32_t* __restrict__ keys,
                                                      const unsigned long long* __restrict__ n_ptr, int k,
                                                      const unsigned long long* __restrict__ draws, int ndraws,
                                                      WsmState* st) {
  constexpr int HS = 2 * KMAX;  // hash slots for positions >= k
  __shared__ unsigned long long jv[KMAX];
  __shared__ uint32_t lowv[KMAX];
  __shared__ unsigned long long hpos[HS];
  __shared__ uint32_t hval[HS];
  __shared__ int s_rejected;
  const int tid = threadIdx.x;
  const unsigned long long n = *n_ptr;
  if ((unsigned long long)k > n) {
    if (tid == 0) st->status = ST_K_EXCEEDS_N;
    return;
  }
  if (tid == 0) s_rejected = 0;
  for (int h = tid; h < HS; h += blockDim.x) hpos[h] = ~0ull;
  __syncthreads();
  for (int i = tid; i < k; i += blockDim.x) {
    lowv[i] = (uint32_t)i;
    const unsigned long long bound = n - (unsigned long long)i;
    const unsigned long long limit = ~0ull - (~0ull % bound);
    const unsigned long long r = i < ndraws ? draws[i] : ~0ull;
    if (r >= limit) s_rejected = 1;
    jv[i] = (unsigned long long)i + r % bound;
  }
  __syncthreads();
  if (tid == 0) {
    if (s_rejected) {  // exact sequential draw consumption
      int di = 0;
      for (int i = 0; i < k; ++i) {
        const unsigned long long bound = n - (unsigned long long)i;
        const unsigned long long limit = ~0ull - (~0ull % bound);
        unsigned long long r;
        do {
          if (di >= ndraws) {
            st->status = ST_DRAWS_EXHAUSTED;
            s_rejected = 2;
            break;
          }
          r = draws[di++];
        } while (r >= limit);
        if (s_rejected == 2) break;
        jv[i] = (unsigned long long)i + r % bound;
      }
    }
    if (s_rejected != 2) {
      for (int i = 0; i < k; ++i) {
        const unsigned long long j = jv[i];
        const uint32_t vi = lowv[i];
        uint32_t vj;
        if (j < (unsigned long long)k) {
          vj = lowv[j];
          lowv[j] = vi;
        } else {
          int h = (int)((j * 0x9E3779B97F4A7C15ull) >> 55);  // 9 bits -> [0, 512)
          while (hpos[h] != ~0ull && hpos[h] != j) h = (h + 1) & (HS - 1);
          vj = hpos[h] == j ? hval[h] : (uint32_t)j;
          hpos[h] = j;
          hval[h] = vi;
        }
        lowv[i] = vj;
      }
    }
  }
  __syncthreads();
  if (s_rejected == 2) return;
  for (int i = tid; i < k; i += blockDim.x) {
    const uint32_t key = keys[lowv[i]];
    st->C[0][3 * i + 0] = (double)key_r(key);
    st->C[0][3 * i + 1] = (double)key_g(key);
    st->C[0][3 * i + 2] = (double)key_b(key);
    st->chosen[i] = lowv[i];
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
  double rowd[KMAX];                     // tables scratch
  double red_hi[LOOP_THREADS / 32], red_lo[LOOP_THREADS / 32];
  int red_i[LOOP_THREADS / 32];
  int empty_list[KMAX];
  unsigned int taken[KMAX];
  int n_empty;
  double sse;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Row p of the center tables (kmeans.hpp:147-168): d[p][t] = dist2(c_p, c_t)
// and the order row [p, others sorted by (d, index)] by rank counting.
__device__ void tables_row(LoopSmem& S, WsmState* st, int p, int k) {
  const int tid = threadIdx.x;
  if (tid < k) S.rowd[tid] = tid == p ? 0.0 : dist2_rn(S.cx[p], S.cy[p], S.cz[p], S.cx[tid], S.cy[tid], S.cz[tid]);
  __syncthreads();
  if (tid < k) {
    int rank = 0;
    if (tid != p) {
      const double dt = S.rowd[tid];
      rank = 1;
      for (int u = 0; u < k; ++u) {
        const double du = S.rowd[u];
        rank += (u != p) & ((du < dt) | ((du == dt) & (u < tid)));
      }
    }
    st->sortedD[p * KMAX + rank] = S.rowd[tid];
    st->order[p * KMAX + rank] = (uint8_t)tid;
  }
  __syncthreads();
}

// u64 += v on a (lo, hi) pair of shared u32 words, native 32-bit atomics only.
__device__ __forceinline__ void sadd64(uint2* a, unsigned long long v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(&a->x, lo);
  const uint32_t c = (uint32_t)(old + lo) < old ? 1u : 0u;
  if (hi + c) atomicAdd(&a->y, hi + c);
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

// Iteration 1, dense + integer-exact (see header). Full accumulation.
__device__ void assign_dense_first(LoopSmem& S, const LoopParams& L, unsigned long long lo, unsigned long long hi,
                                   unsigned long long& evals) {
  const int k = L.k;
  const unsigned long long T = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long g0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int cc0 = S.cb[0].y >> 8;  // |c_0|^2
  const uint32_t c0 = (uint32_t)S.cb[0].x;
  constexpr int PPT = 4;
  for (unsigned long long base = lo + g0; base < hi; base += PPT * T) {
    uint32_t x[PPT];
    int best[PPT];
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const unsigned long long i = base + q * T;
      x[q] = i < hi ? L.keys[i] : 0u;
      best[q] = 0x7fffffff;
    }
    for (int t = 0; t < k; ++t) {
      const int2 cb = S.cb[t];
#pragma unroll
      for (int q = 0; q < PPT; ++q) best[q] = min(best[q], cb.y - 512 * key_dot(x[q], (uint32_t)cb.x));
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const unsigned long long i = base + q * T;
      if (i < hi) {
        const int lab = best[q] & 255;
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
        evals += (unsigned long long)lo_j;  // 1 (prev) + (lo_j - 1) candidates
        L.labels[i] = (uint8_t)lab;
        acc_point(S.accp, lab, x[q], L.counts[i]);
      }
    }
  }
}

// Iterations >= 2 (or the first of a teacher-forced launch, full = true):
// FP64 sort-means scan from the previous label (kmeans.hpp:211-236); tables
// in L2 (written by this kernel, read after the grid barrier).
__device__ void assign_sort_means(LoopSmem& S, const LoopParams& L, unsigned long long lo, unsigned long long hi,
                                  bool full, unsigned long long& evals) {
  const unsigned long long T = (unsigned long long)gridDim.x * blockDim.x;
  const double* __restrict__ sd = L.st->sortedD;
  const uint8_t* __restrict__ od = L.st->order;
  const int k = L.k;
  for (unsigned long long i = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += T) {
    const uint32_t key = L.keys[i];
    const int p = L.labels[i];
    const double x0 = (double)key_r(key), x1 = (double)key_g(key), x2 = (double)key_b(key);
    const double prev = dist2_rn(x0, x1, x2, S.cx[p], S.cy[p], S.cz[p]);
    const double bound = 4.0 * prev;
    double mind = prev;
    int best = p;
    unsigned long long ev = 1;
    const double* rowd = sd + p * KMAX;
    const uint8_t* rowo = od + p * KMAX;
    for (int j = 1; j < k; ++j) {
      const double dj = rowd[j];
      if (dj >= bound) break;
      const int t = rowo[j];
      const double d = dist2_rn(x0, x1, x2, S.cx[t], S.cy[t], S.cz[t]);
      ++ev;
      if (d < mind || (d == mind && t < best)) {
        mind = d;
        best = t;
      }
    }
    evals += ev;
    if (full) {
      if (best != p) L.labels[i] = (uint8_t)best;
      acc_point(S.accp, best, key, L.counts[i]);
    } else if (best != p) {
      L.labels[i] = (uint8_t)best;
      const uint32_t cnt = L.counts[i];
      acc_point(S.accm, p, key, cnt);
      acc_point(S.accp, best, key, cnt);
    }
  }
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

// Empty-cluster reseed (kmeans.hpp:268-290), grid-wide, all blocks agree.
__device__ void reseed_empty(LoopSmem& S, const LoopParams& L, cg::grid_group& grid, unsigned long long lo,
                             unsigned long long hi) {
  WsmState* st = L.st;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned long long T = (unsigned long long)gridDim.x * blockDim.x;
  for (int e = 0; e < S.n_empty; ++e) {
    double bd = -1.0;
    unsigned int bi = 0xffffffffu;
    for (unsigned long long i = lo + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += T) {
      bool used = false;
      for (int t = 0; t < e; ++t) used |= (S.taken[t] == (unsigned int)i);
      if (used) continue;
      const uint32_t key = L.keys[i];
      const int m = L.labels[i];
      const double d = dist2_rn((double)key_r(key), (double)key_g(key), (double)key_b(key), S.cx[m], S.cy[m], S.cz[m]);
      if (cand_better(d, (unsigned int)i, bd, bi)) {
        bd = d;
        bi = (unsigned int)i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const unsigned int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (cand_better(od, oi, bd, bi)) {
        bd = od;
        bi = oi;
      }
    }
    __syncthreads();
    if (lane == 0) {
      S.red_hi[wid] = bd;
      S.red_i[wid] = (int)bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double xd = -1.0;
      unsigned int xi = 0xffffffffu;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        if (cand_better(S.red_hi[w], (unsigned int)S.red_i[w], xd, xi)) {
          xd = S.red_hi[w];
          xi = (unsigned int)S.red_i[w];
        }
      st->cand_d[e & 1][blockIdx.x] = __double_as_longlong(xd);
      st->cand_i[e & 1][blockIdx.x] = xi;
    }
    grid.sync();
    if (threadIdx.x == 0) {
      double xd = -1.0;
      unsigned int xi = 0xffffffffu;
      for (unsigned int b = 0; b < gridDim.x; ++b) {
        const double d = __longlong_as_double((long long)st->cand_d[e & 1][b]);
        const unsigned int i = st->cand_i[e & 1][b];
        if (cand_better(d, i, xd, xi)) {
          xd = d;
          xi = i;
        }
      }
      S.taken[e] = xi;
      const int ke = S.empty_list[e];
      const uint32_t key = L.keys[xi];
      S.nx[ke] = (double)key_r(key);
      S.ny[ke] = (double)key_g(key);
      S.nz[ke] = (double)key_b(key);
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
__global__ void __launch_bounds__(LOOP_THREADS, 2) k_wsm_loop(LoopParams L) {
  __shared__ LoopSmem S;
  cg::grid_group grid = cg::this_grid();
  WsmState* st = L.st;
  const int tid = threadIdx.x;
  const int k = L.k;
  if (st->status != ST_OK) return;  // uniform across the grid
  const unsigned long long n = *L.n_ptr;
  const unsigned long long lo = L.shard_lo < n ? L.shard_lo : n;
  const unsigned long long hi = L.shard_hi_or_max < n ? L.shard_hi_or_max : n;
  const double inv_P = 1.0 / (double)L.total;
  unsigned long long* gacc = st->acc;  // exact running sums (zeroed by the host per launch)
  unsigned long long* tl = L.timeline;
  const bool rec = tl && blockIdx.x == 0 && tid == 0;

  for (int t = tid; t < k; t += blockDim.x) {
    S.cx[t] = st->C[0][3 * t];
    S.cy[t] = st->C[0][3 * t + 1];
    S.cz[t] = st->C[0][3 * t + 2];
  }
  for (int t = tid; t < 5 * KMAX; t += blockDim.x) {
    S.accp[t] = make_uint2(0u, 0u);
    S.accm[t] = make_uint2(0u, 0u);
  }
  __syncthreads();
  // prologue: tables of the initial centers (all pairs evaluated: non-incremental)
  for (int p = blockIdx.x; p < k; p += gridDim.x) tables_row(S, st, p, k);
  if (blockIdx.x == 0 && tid == 0) st->evals += (unsigned long long)k * (unsigned long long)(k - 1) / 2;
  grid.sync();

  double prev_sse = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  for (int it = 1;; ++it) {
    const bool rec_it = rec && it <= L.hist_cap;
    if (rec_it) tl[(it - 1) * 5 + 0] = globaltimer();
    // ---------------- assign(it) ----------------
    unsigned long long evals = 0;
    if (it == 1 && L.dense_first) {
      for (int t = tid; t < k; t += blockDim.x) {
        const uint32_t key = ((uint32_t)S.cx[t] << 16) | ((uint32_t)S.cy[t] << 8) | (uint32_t)S.cz[t];
        S.cb[t] = make_int2((int)key, key_dot(key, key) * 256 + t);
        S.row0[t] = (uint32_t)st->sortedD[t];  // row 0 (p = 0), integer-valued
      }
      __syncthreads();
      assign_dense_first(S, L, lo, hi, evals);
    } else {
      assign_sort_means(S, L, lo, hi, it == 1, evals);
    }
    evals = warp_sum(evals);
    if ((tid & 31) == 0 && evals) atomicAdd(&st->evals, evals);
    __syncthreads();
    flush_moments(S, gacc, k);
    if (rec_it) tl[(it - 1) * 5 + 1] = globaltimer();
    grid.sync();
    if (rec_it) tl[(it - 1) * 5 + 2] = globaltimer();

    // ---------------- finalize(it), redundantly per block ----------------
    dd part{0.0, 0.0};
    int empt = 0;
    for (int t = tid; t < k; t += blockDim.x) {
      const unsigned long long N = gacc[3 * KMAX + t];
      const double Sr = (double)gacc[0 * KMAX + t], Sg = (double)gacc[1 * KMAX + t], Sb = (double)gacc[2 * KMAX + t];
      if (N) {
        const double dn = (double)N;
        S.nx[t] = Sr / dn;
        S.ny[t] = Sg / dn;
        S.nz[t] = Sb / dn;
        // Q - 2 c.S + |c|^2 N with the centers of THIS assignment
        const double cr = S.cx[t], cgc = S.cy[t], cbc = S.cz[t];
        dd cs = dd_add(dd_add(two_prod(cr, Sr), two_prod(cgc, Sg)), two_prod(cbc, Sb));
        dd c2 = dd_add(dd_add(two_prod(cr, cr), two_prod(cgc, cgc)), two_prod(cbc, cbc));
        dd term = dd_add(dd{(double)gacc[4 * KMAX + t], 0.0}, dd_scale(cs, -2.0));
        term = dd_add(term, dd_scale(c2, dn));
        part = dd_add(part, term);
      } else {
        empt = 1;
      }
    }
    const dd tot = block_sum_dd(S, part);
    const int n_empty = block_sum_int(S, empt);
    if (tid == 0) {
      const double sse = __dadd_rn(tot.hi, tot.lo) * inv_P;
      S.sse = sse < 0.0 ? 0.0 : sse;
      S.n_empty = n_empty;
      if (n_empty) {
        int m = 0;
        for (int t = 0; t < k; ++t)
          if (gacc[3 * KMAX + t] == 0ull) S.empty_list[m++] = t;
      }
    }
    __syncthreads();
    if (S.n_empty) reseed_empty(S, L, grid, lo, hi);
    const double sse = S.sse;
    // termination (kmeans.hpp:359-369)
    bool stop;
    if (L.mode == 0) {
      stop = it >= L.max_iters;
    } else {
      stop = (sse == 0.0) || ((prev_sse - sse) / sse <= L.eps) || (it >= L.cap);
    }
    prev_sse = sse;
    if (blockIdx.x == 0) {
      if (tid == 0) {
        if (it <= L.hist_cap) L.sse_hist[it - 1] = sse;
        st->iterations = it;
        st->sse = sse;
        st->n_empty_events += S.n_empty;
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
    if (stop) break;
    // pair evaluations of the incremental table update (kmeans.hpp:137-155)
    int moved = 0;
    for (int t = tid; t < k; t += blockDim.x)
      moved += (S.nx[t] != S.cx[t]) | (S.ny[t] != S.cy[t]) | (S.nz[t] != S.cz[t]);
    const int n_moved = block_sum_int(S, moved);
    if (blockIdx.x == 0 && tid == 0) {
      const unsigned long long still = (unsigned long long)(k - n_moved);
      const unsigned long long all = (unsigned long long)k * (unsigned long long)(k - 1) / 2;
      st->evals += all - (still ? still * (still - 1) / 2 : 0ull);
    }
    __syncthreads();
    for (int t = tid; t < k; t += blockDim.x) {
      S.cx[t] = S.nx[t];
      S.cy[t] = S.ny[t];
      S.cz[t] = S.nz[t];
    }
    __syncthreads();
    if (rec_it) tl[(it - 1) * 5 + 3] = globaltimer();
    for (int p = blockIdx.x; p < k; p += gridDim.x) tables_row(S, st, p, k);
    if (rec_it) tl[(it - 1) * 5 + 4] = globaltimer();
    grid.sync();
  }
}

}  // namespace cqb
