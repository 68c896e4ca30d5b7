// Weighted k-means over an ARBITRARY weighted point set (reference:
// kmeans.hpp's span<const Vec3> overloads: init_centers :53-74,
// ClusterState::update_center_tables :132-184, assign_sort_means :201-239,
// update_centers :245-302, weighted_sse :306-317, run_weighted_kmeans /
// run_wsm_points :336-390). The histogram path (wsm.cuh) needs 8-bit colors
// and integer counts; this one takes FP64 points, FP64 weights and K up to
// PTS_KMAX, one kernel per step with the loop on the host (cqb_run_wsm_points).
//
// Exactness: distances are dist2_rn (FP64, no FMA) and the tables are sorted
// by (d, index) with self first, so memberships and dist_evals follow the
// reference's sort-means scan. update_centers reproduces the reference's
// sequential per-cluster sums bit for bit: the points are stably sorted by
// membership (counting sort, index order kept inside a cluster) and one thread
// per cluster accumulates w*x and w in index order, exactly the additions the
// reference's single loop makes into that cluster's sums. The weighted SSE is
// a fixed-order tree sum (deterministic, within a few ulp of the reference's
// sequential sum).
#pragma once
#include "common.cuh"

namespace cqb {

constexpr int PTS_KMAX = 1024;
constexpr int PTS_THREADS = 256;
constexpr int PTS_TILE = 1024;  // points per tile of the stable counting sort
constexpr int PTS_SORT_MEANS = 0, PTS_NAIVE = 1, PTS_FKM = 2;  // k_pts_assign modes

// Pixels as points (methods.hpp pixels_as_points; kmeans.hpp:413-416): the
// u8x3 raster widened to FP64 points of weight 1/P each.
__global__ void k_pts_from_rgb(const uint8_t* __restrict__ rgb, uint64_t P, double* __restrict__ X,
                               double* __restrict__ W) {
  const double w = 1.0 / (double)P;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (uint64_t)gridDim.x * blockDim.x) {
    X[3 * i] = (double)rgb[3 * i];
    X[3 * i + 1] = (double)rgb[3 * i + 1];
    X[3 * i + 2] = (double)rgb[3 * i + 2];
    W[i] = w;
  }
}

// Row p of the center tables: center_dists[p][t] = dist2(c_p, c_t) (zero
// diagonal, symmetric), order[p] = [p, others by (d, index)], sortedD[p][j] =
// center_dists[p][order[p][j]]. One block per row.
__global__ void __launch_bounds__(PTS_THREADS) k_pts_tables(const double* __restrict__ C, int k,
                                                            double* __restrict__ center_dists,
                                                            int32_t* __restrict__ order,
                                                            double* __restrict__ sortedD) {
  __shared__ double d[PTS_KMAX];
  const int p = blockIdx.x;
  const double px = C[3 * p], py = C[3 * p + 1], pz = C[3 * p + 2];
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const double v = t == p ? 0.0 : dist2_rn(px, py, pz, C[3 * t], C[3 * t + 1], C[3 * t + 2]);
    d[t] = v;
    center_dists[(size_t)p * k + t] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    int rank = 0;
    if (t != p) {  // self first even if another center coincides (kmeans.hpp:165)
      const double dt = d[t];
      rank = 1;
      for (int u = 0; u < k; ++u) rank += (u != p) & ((d[u] < dt) | ((d[u] == dt) & (u < t)));
    }
    order[(size_t)p * k + rank] = t;
    sortedD[(size_t)p * k + rank] = d[t];
  }
}

// The sorted distance rows of caller-supplied tables (ClusterState):
// sortedD[p][j] = center_dists[p][order[p][j]].
__global__ void __launch_bounds__(PTS_THREADS) k_pts_sorted_rows(const double* __restrict__ center_dists,
                                                                 const int32_t* __restrict__ order, int k,
                                                                 double* __restrict__ sortedD) {
  const int p = blockIdx.x;
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    sortedD[(size_t)p * k + j] = center_dists[(size_t)p * k + order[(size_t)p * k + j]];
}

// assign_sort_means (kmeans.hpp:201-239) over n points; per-block partial
// weighted SSE (fixed order) and the evaluation count.
__global__ void __launch_bounds__(PTS_THREADS) k_pts_assign(const double* __restrict__ X,
                                                            const double* __restrict__ W, uint64_t n,
                                                            const double* __restrict__ C, int k,
                                                            const int32_t* __restrict__ order,
                                                            const double* __restrict__ sortedD,
                                                            int32_t* __restrict__ m, double* __restrict__ sse_part,
                                                            unsigned long long* __restrict__ evals, int mode,
                                                            int kprime, int32_t* __restrict__ skip_rank,
                                                            double* __restrict__ prev_out) {
  __shared__ double cs[3 * PTS_KMAX];
  __shared__ double red[PTS_THREADS / 32];
  __shared__ unsigned long long red_e[PTS_THREADS / 32];
  for (int i = threadIdx.x; i < 3 * k; i += blockDim.x) cs[i] = C[i];
  __syncthreads();
  double sse = 0.0;
  unsigned long long ev = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double x0 = X[3 * i], x1 = X[3 * i + 1], x2 = X[3 * i + 2];
    if (mode == PTS_FKM) {  // run_fkm (fast_variants.hpp:42-55): order[m][0..k'), ties to the lowest index
      const int32_t* row = order + (size_t)m[i] * k;
      int best = row[0];
      double best_d = dist2_rn(x0, x1, x2, cs[3 * best], cs[3 * best + 1], cs[3 * best + 2]);
      for (int j = 1; j < kprime; ++j) {
        const int t = row[j];
        const double dist = dist2_rn(x0, x1, x2, cs[3 * t], cs[3 * t + 1], cs[3 * t + 2]);
        if (dist < best_d || (dist == best_d && t < best)) {
          best_d = dist;
          best = t;
        }
      }
      ev += (unsigned long long)kprime;
      m[i] = best;
      sse = __dadd_rn(sse, __dmul_rn(W[i], best_d));
      continue;
    }
    if (mode == PTS_NAIVE) {  // assign_naive (kmeans.hpp:89-102): strict '<' from c_0
      double best_d = dist2_rn(x0, x1, x2, cs[0], cs[1], cs[2]);
      int best = 0;
      for (int t = 1; t < k; ++t) {
        const double dist = dist2_rn(x0, x1, x2, cs[3 * t], cs[3 * t + 1], cs[3 * t + 2]);
        if (dist < best_d) {
          best_d = dist;
          best = t;
        }
      }
      ev += (unsigned long long)k;
      m[i] = best;
      sse = __dadd_rn(sse, __dmul_rn(W[i], best_d));
      continue;
    }
    const int p = m[i];
    const double prev = dist2_rn(x0, x1, x2, cs[3 * p], cs[3 * p + 1], cs[3 * p + 2]);
    double best_d = prev;
    int best = p;
    const double bound = 4.0 * prev;
    const int32_t* row = order + (size_t)p * k;
    const double* drow = sortedD + (size_t)p * k;
    int j = 1;
    for (; j < k; ++j) {
      if (drow[j] >= bound) break;
      const int t = row[j];
      const double dist = dist2_rn(x0, x1, x2, cs[3 * t], cs[3 * t + 1], cs[3 * t + 2]);
      if (dist < best_d || (dist == best_d && t < best)) {
        best_d = dist;
        best = t;
      }
    }
    ev += (unsigned long long)j;  // prev + (j - 1) candidates
    if (skip_rank) {
      skip_rank[i] = j < k ? j : -1;
      prev_out[i] = prev;
    }
    m[i] = best;
    sse = __dadd_rn(sse, __dmul_rn(W[i], best_d));
  }
  sse = warp_sum(sse);
  ev = warp_sum(ev);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = sse;
    red_e[threadIdx.x >> 5] = ev;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    unsigned long long e = 0;
    for (int w = 0; w < PTS_THREADS / 32; ++w) {
      s += red[w];
      e += red_e[w];
    }
    sse_part[blockIdx.x] = s;
    atomicAdd(evals, e);
  }
}

// weighted_sse (kmeans.hpp:306-317): per-block partials of sum w*dist2(x, c_m).
__global__ void __launch_bounds__(PTS_THREADS) k_pts_sse(const double* __restrict__ X, const double* __restrict__ W,
                                                         uint64_t n, const double* __restrict__ C,
                                                         const int32_t* __restrict__ m,
                                                         double* __restrict__ sse_part) {
  __shared__ double red[PTS_THREADS / 32];
  double sse = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = m[i];
    sse = __dadd_rn(sse, __dmul_rn(W[i], dist2_rn(X[3 * i], X[3 * i + 1], X[3 * i + 2], C[3 * c], C[3 * c + 1],
                                                  C[3 * c + 2])));
  }
  sse = warp_sum(sse);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sse;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < PTS_THREADS / 32; ++w) s += red[w];
    sse_part[blockIdx.x] = s;
  }
}

// Fixed-order sum of nb block partials (one thread: deterministic).
__global__ void k_pts_sum(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[b];
  *out = s;
}

// Stable counting sort by membership, step 1: per tile, per cluster counts.
__global__ void __launch_bounds__(PTS_THREADS) k_pts_tile_count(const int32_t* __restrict__ m, uint64_t n, int k,
                                                                uint32_t* __restrict__ cnt) {
  __shared__ uint32_t h[PTS_KMAX];
  for (int c = threadIdx.x; c < k; c += blockDim.x) h[c] = 0u;
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * PTS_TILE;
  for (uint64_t i = t0 + threadIdx.x; i < n && i < t0 + PTS_TILE; i += blockDim.x) atomicAdd(&h[m[i]], 1u);
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) cnt[(size_t)blockIdx.x * k + c] = h[c];
}

// Step 2 (one block of PTS_KMAX threads): cluster-major exclusive offsets
// off[tile][c] and cluster starts start[c] (start[k] = n).
__global__ void __launch_bounds__(PTS_KMAX) k_pts_offsets(const uint32_t* __restrict__ cnt, uint32_t tiles, int k,
                                                          uint32_t* __restrict__ off, uint32_t* __restrict__ start) {
  __shared__ uint32_t warp_tot[PTS_KMAX / 32];
  const int c = threadIdx.x, lane = c & 31, wid = c >> 5;
  uint32_t tot = 0;
  if (c < k)
    for (uint32_t t = 0; t < tiles; ++t) tot += cnt[(size_t)t * k + c];
  uint32_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  uint32_t run = incl - tot;
  for (int w = 0; w < wid; ++w) run += warp_tot[w];
  if (c < k) {
    start[c] = run;
    for (uint32_t t = 0; t < tiles; ++t) {
      const uint32_t v = cnt[(size_t)t * k + c];
      off[(size_t)t * k + c] = run;
      run += v;
    }
  }
  if (c == k - 1) start[k] = run;
}

// Step 3: one warp per tile places the tile's points in index order (32 at a
// time; peers by __match_any_sync keep their order): perm[pos] = i.
__global__ void k_pts_tile_scatter(const int32_t* __restrict__ m, uint64_t n, int k, const uint32_t* __restrict__ off,
                                   uint32_t* __restrict__ perm) {
  extern __shared__ uint32_t cur_all[];  // [warps per block][k]
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  uint32_t* cur = cur_all + (size_t)wib * k;
  const uint64_t t0 = tile * PTS_TILE;
  if (t0 >= n) return;
  for (int c = lane; c < k; c += 32) cur[c] = off[tile * k + c];
  __syncwarp();
  for (uint64_t b = t0; b < n && b < t0 + PTS_TILE; b += 32) {
    const uint64_t i = b + lane;
    const bool v = i < n && i < t0 + PTS_TILE;
    const int c = v ? m[i] : -1 - lane;  // invalid lanes: distinct dummy keys
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    const int before = __popc(peers & ((1u << lane) - 1u));
    uint32_t base = 0;
    if (v) base = cur[c];
    __syncwarp();
    if (v) {
      perm[base + before] = (uint32_t)i;
      if (before == 0) cur[c] = base + __popc(peers);  // the group's lowest lane advances the cursor
    }
    __syncwarp();
  }
}

// Step 4 (update_centers, kmeans.hpp:252-266): one thread per cluster sums
// w*x and w over its members in index order. Empty clusters are flagged.
__global__ void k_pts_sums(const double* __restrict__ X, const double* __restrict__ W,
                           const uint32_t* __restrict__ perm, const uint32_t* __restrict__ start, int k,
                           double* __restrict__ next, int* __restrict__ empty) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, ws = 0.0;
  for (uint32_t j = start[c]; j < start[c + 1]; ++j) {
    const uint32_t i = perm[j];
    const double w = W[i];
    s0 = __dadd_rn(s0, __dmul_rn(w, X[3 * i]));
    s1 = __dadd_rn(s1, __dmul_rn(w, X[3 * i + 1]));
    s2 = __dadd_rn(s2, __dmul_rn(w, X[3 * i + 2]));
    ws = __dadd_rn(ws, w);
  }
  const bool e = !(ws > 0.0);
  empty[c] = e;
  if (!e) {
    next[3 * c] = __ddiv_rn(s0, ws);
    next[3 * c + 1] = __ddiv_rn(s1, ws);
    next[3 * c + 2] = __ddiv_rn(s2, ws);
  }
}

// Empty-cluster reseed candidate (kmeans.hpp:272-290): per block, the point
// with the largest dist2(x_i, prev[m_i]) (strict '>': lowest index on ties)
// whose value differs from every point already taken this round.
__global__ void __launch_bounds__(PTS_THREADS) k_pts_reseed_scan(const double* __restrict__ X, uint64_t n,
                                                                 const double* __restrict__ prev,
                                                                 const int32_t* __restrict__ m,
                                                                 const double* __restrict__ taken, int n_taken,
                                                                 double* __restrict__ cand_d,
                                                                 unsigned long long* __restrict__ cand_i) {
  __shared__ double sd[PTS_THREADS / 32];
  __shared__ unsigned long long si[PTS_THREADS / 32];
  double bd = -1.0;
  unsigned long long bi = ~0ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double x0 = X[3 * i], x1 = X[3 * i + 1], x2 = X[3 * i + 2];
    const int c = m[i];
    const double d = dist2_rn(x0, x1, x2, prev[3 * c], prev[3 * c + 1], prev[3 * c + 2]);
    if (!(d > bd || (d == bd && i < bi))) continue;
    bool used = false;
    for (int t = 0; t < n_taken; ++t)
      used |= taken[3 * t] == x0 && taken[3 * t + 1] == x1 && taken[3 * t + 2] == x2;
    if (used) continue;
    bd = d;
    bi = i;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const unsigned long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (od > bd || (od == bd && oi < bi)) {
      bd = od;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sd[threadIdx.x >> 5] = bd;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < PTS_THREADS / 32; ++w)
      if (sd[w] > bd || (sd[w] == bd && si[w] < bi)) {
        bd = sd[w];
        bi = si[w];
      }
    cand_d[blockIdx.x] = bd;
    cand_i[blockIdx.x] = bi;
  }
}

// The winner among the blocks' candidates becomes cluster c's center and
// joins the taken list.
__global__ void k_pts_reseed_pick(const double* __restrict__ cand_d, const unsigned long long* __restrict__ cand_i,
                                  int nb, const double* __restrict__ X, int c, double* __restrict__ next,
                                  double* __restrict__ taken, int slot) {
  if (threadIdx.x != 0) return;
  double bd = -1.0;
  unsigned long long bi = ~0ull;
  for (int b = 0; b < nb; ++b)
    if (cand_d[b] > bd || (cand_d[b] == bd && cand_i[b] < bi)) {
      bd = cand_d[b];
      bi = cand_i[b];
    }
  if (bi == ~0ull) bi = 0;  // every point taken: the reference keeps best_i = 0
  for (int d = 0; d < 3; ++d) {
    next[3 * c + d] = X[3 * bi + d];
    taken[3 * slot + d] = X[3 * bi + d];
  }
}

// init_centers (kmeans.hpp:58-68) on points: center i = points[chosen[i]].
__global__ void k_pts_gather(const double* __restrict__ X, const uint32_t* __restrict__ chosen, int k,
                             const int* __restrict__ status, double* __restrict__ C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k || *status != 0) return;
  const uint64_t p = chosen[i];
  C[3 * i] = X[3 * p];
  C[3 * i + 1] = X[3 * p + 1];
  C[3 * i + 2] = X[3 * p + 2];
}

}  // namespace cqb
