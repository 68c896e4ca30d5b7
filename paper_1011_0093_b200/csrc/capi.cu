// Host side of the C ABI (include/colorq_b200.h): per-context device arena,
// stream, launch sequencing and result staging. No CPU fallback exists: every
// numeric result below comes from the sm_100a kernels in hist/wsm/map.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "../../include/colorq_b200.h"
#include "hist.cuh"
#include "map.cuh"
#include "wsm.cuh"
#include "prep.cuh"
#include "points.cuh"

using namespace cqb;

namespace {

constexpr int XFER_CHUNKS = 8;
#ifndef CQB_K1_GRID
#define CQB_K1_GRID 32  // K1 blocks per SM (grid-stride over 16-pixel chunks; 4/8/16/32: 249/247/231/226 us on cfg4)
#endif
constexpr int DBG_NO_COARSE = 1 << 21;  // (see below)
constexpr int DBG_K1_2PASS = 1 << 22;   // debug flag: K1 in two half-table passes (A/B)
constexpr int DBG_K1_1PASS = 1 << 23;   // debug flag: K1 in one pass (A/B)  // debug flag: k_map_pixels with per-pixel LUT gathers only (A/B)
constexpr int DBG_NO_XFER_OVERLAP = 1 << 19;  // debug flag: one H2D / D2H copy each, K1 after the H2D

struct Staging {  // pinned host mirror of the per-call results
  double centers[3 * KMAX];
  unsigned long long evals, mse_err, n_unique;
  double sse;
  int iterations, status, n_empty;
};

}  // namespace

struct cqb_ctx {
  int device = 0;
  std::vector<cqb_ctx*> lanes;  // cqb_quantize_batch: images in flight (config 5)
  cudaEvent_t join_ev = nullptr;  // cqb_quantize_batch: lanes wait for the caller's stream
  cudaEvent_t lane_done = nullptr;  // as a lane: end of its batch work
  cudaEvent_t join_ev_out() {
    if (!lane_done) cudaEventCreateWithFlags(&lane_done, cudaEventDisableTiming);
    return lane_done;
  }
  int num_sms = 0;
  int loop_blocks_max = 0;
  int grid_limit = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // cqb_quantize_ex on large images: host<->device copies in XFER_CHUNKS
  // slices on a second stream, overlapped with K1 (H2D) and the map (D2H)
  cudaStream_t xfer = nullptr;
  cudaEvent_t xev[2 * XFER_CHUNKS + 1] = {};
  bool k1_done = false;               // set only while cqb_quantize_ex enqueues: bins already counted
  uint8_t* h_index_dst = nullptr;     // set only while cqb_quantize_ex enqueues: chunked D2H targets
  uint8_t* h_rgb_dst = nullptr;
  uint8_t* h_err_dst = nullptr;

  uint2* bins = nullptr;  // 2^24 x {count, ~first}; all-zero between calls
  uint8_t* lut = nullptr; // 2^24 key -> palette index
  uint32_t* d_cellw = nullptr;   // coarse map table: per-cell words (map.cuh)
  uint8_t* d_coarse = nullptr;   // its compact form (labels + MIXED bits)
  bool coarse_built = false;     // set by launch_loop: the loop's epilogue wrote d_coarse for this call
  const uint32_t* ext_samples = nullptr;  // set only while cqb_quantize_sharded_samples enqueues: the
  uint64_t ext_n = 0;                     // whole image's Morton-ordered {key, count, first} triplets

  size_t cap_px = 0;
  uint8_t* d_img = nullptr;
  uint8_t* d_img2 = nullptr;
  uint8_t* d_index = nullptr;
  uint8_t* d_rgb = nullptr;
  size_t cap_tiles = 0;
  unsigned long long* tile_state = nullptr;  // [ntiles] + ticket at [cap_tiles]

  size_t cap_s = 0;
  uint32_t* d_keys = nullptr;
  uint32_t* d_counts = nullptr;
  uint32_t* d_first = nullptr;
  uint32_t* d_bitmap = nullptr;  // P-bit first-occurrence bitmap (+ pad)
  uint32_t* d_occ = nullptr;     // 2^24-bit bin occupancy map (small images; all-zero between calls)
  uint32_t* d_block_counts = nullptr;  // k_prep_small scratch [3 * MAXBLK]
  uint32_t* d_units = nullptr;         // k_prep_small scratch: non-empty 8-bin units, per-block lists
  uint32_t* d_wofs = nullptr;          // k_prep_small scratch [2^19]
  int prep_blocks = 0;                 // k_prep_small cooperative grid
  uint8_t* d_err = nullptr;       // error_image raster (cqb_quantize_ex / cqb_error_image)
  uint8_t* err_target = nullptr;  // set only while cqb_quantize_ex enqueues: fused error_image output
  bool fuse_map = false;          // set only while enqueue_quantize launches the loop: map epilogue
  uint8_t* d_cand = nullptr;      // iteration-1 candidate centers per 16^3 color cell
  uint16_t* d_cand_n = nullptr;
  uint32_t* d_bpre = nullptr;    // per-word set-bit prefix of d_bitmap
  uint8_t* d_labels = nullptr;    // Morton layout (loop + map)
  uint8_t* d_lab_rank = nullptr;  // first-occurrence layout (API in/out)
  uint32_t* d_mkeys = nullptr;    // Morton-ordered samples (K2b)
  uint32_t* d_mcounts = nullptr;
  uint32_t* d_mrank = nullptr;
  unsigned long long* bin_tile_state = nullptr;  // K2b look-back [N_BIN_TILES] + ticket
  // init_centers by rank selection over first pixels (hist.cuh RS1-RS4)
  uint32_t* rs_coarse = nullptr;       // [RS_NC]
  uint16_t* rs_slot_of = nullptr;      // [RS_NC]
  uint32_t* rs_tgt = nullptr;          // [2 * KMAX] target block, residual
  uint32_t* rs_slot_bits = nullptr;
  size_t cap_slot_bits = 0;
  // generic weighted points (points.cuh)
  struct Points {
    size_t cap_n = 0, cap_tiles = 0;
    int cap_k = 0;
    double* X = nullptr;            // 3n
    double* W = nullptr;            // n
    int32_t* m = nullptr;           // n memberships
    uint32_t* perm = nullptr;       // n, stable sort by membership
    int32_t* skip = nullptr;        // n audit: first skipped rank or -1
    double* prevd = nullptr;        // n audit: previous distance
    uint32_t* tcnt = nullptr;       // tiles x k
    uint32_t* toff = nullptr;
    double* C = nullptr;            // 3k current centers
    double* next = nullptr;         // 3k
    double* taken = nullptr;        // 3k
    double* dists = nullptr;        // k x k
    int32_t* order = nullptr;       // k x k
    double* sortedD = nullptr;      // k x k
    uint32_t* start = nullptr;      // k + 1
    int* empty = nullptr;           // k
    double* part = nullptr;         // block partials
    unsigned long long* cand_i = nullptr;
    double* scal = nullptr;         // [0] sse
    unsigned long long* evals = nullptr;
    uint32_t* chosen = nullptr;     // k
  } pts;
  double* d_weights = nullptr;
  unsigned long long* d_n = nullptr;  // N'

  WsmState* st = nullptr;
  double* d_hist = nullptr;
  int cap_hist = 0;
  unsigned long long* d_timeline = nullptr;  // 8 stamps per iteration (profiling)
  unsigned long long* d_block_times = nullptr;  // [8 iterations][MAXBLK] (profiling)
  // sharded-run scratch
  int shard_k = 0;
  uint64_t shard_total = 0;
  unsigned long long* d_mom = nullptr;  // 5*KMAX
  unsigned long long* h_mom = nullptr;  // pinned 5*KMAX + 1 (evals)
  double* d_Cnew = nullptr;
  double* d_scal = nullptr;             // sse + reseed outputs
  int* d_ints = nullptr;                // n_empty + empty list
  uint32_t* d_taken = nullptr;
  double* d_cand_d = nullptr;
  unsigned int* d_cand_r = nullptr;
  unsigned int* d_cand_k = nullptr;
  double* d_traj = nullptr;
  size_t cap_traj = 0;
  double* d_centers_in = nullptr;
  int* d_sortedDr = nullptr;
  uint8_t* d_orderR = nullptr;
  uint32_t* d_palkey = nullptr;
  // in-kernel sharded loop (cqb_xch_*, cqb_quantize_sharded)
  int xmode = 0;                      // 0 none, 1 one process per GPU (IPC windows), 2 emulated ranks
  int xw = 0, xrank = -1;
  unsigned long long* xwin = nullptr;  // own window (mode 1) / the xw windows (mode 2)
  unsigned long long* xpeer[8] = {};   // every rank's window as mapped here (own = xwin)
  unsigned long long* xacc = nullptr;  // mode 2: per-group moment sums
  bool xsharded = false;              // set only while cqb_quantize_sharded enqueues
  unsigned long long xch_timeout_ns = XCH_TIMEOUT_NS;  // cqb_xch_set_timeout
  uint64_t px_lo = 0, px_hi = 0;      // sharded: pixel range mapped by this rank

  unsigned long long* d_draws = nullptr;
  unsigned long long* h_draws = nullptr;
  int cap_draws = 0;
  bool draws_valid = false;
  uint64_t draws_seed = 0;
  int draws_n = 0;

  Staging* h_stage = nullptr;
  double* h_hist = nullptr;
  unsigned long long* h_scalar = nullptr;
  cudaEvent_t ev[4] = {};
  bool profiling = false;
  int stamp_iter = 3;
  int debug_flags = 0;  // diagnostics only (see LoopParams::debug_flags)
  cudaEvent_t pev[8] = {};  // stage boundaries when profiling
  int last_k = 0;
  uint64_t last_P = 0;  // pixels of the last enqueued quantize (MSE denominator)
  int last_hist_cap = 0;
  int launches = 0;
  std::string err;
};

namespace {

int fail(cqb_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? CQB_ERR_OOM : CQB_ERR_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                             \
  } while (0)

#define CKL()                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = cudaGetLastError();                                                         \
    if (e_ != cudaSuccess)                                                                       \
      return fail(ctx, CQB_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                     \
    ++ctx->launches;                                                                             \
  } while (0)

#define TRY(x)             \
  do {                     \
    int r_ = (x);          \
    if (r_ != CQB_OK) return r_; \
  } while (0)

template <typename T>
int grow(cqb_ctx* ctx, T** p, size_t n) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  CK(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T)));
  return CQB_OK;
}

int ensure_pixels(cqb_ctx* ctx, size_t P) {
  if (P <= ctx->cap_px) return CQB_OK;
  const size_t cap = (P + 15) / 16 * 16 + 64;
  TRY(grow(ctx, &ctx->d_img, 3 * cap));
  TRY(grow(ctx, &ctx->d_img2, 3 * cap));
  TRY(grow(ctx, &ctx->d_index, cap));
  TRY(grow(ctx, &ctx->d_rgb, 3 * cap));
  TRY(grow(ctx, &ctx->d_err, 3 * cap));
  TRY(grow(ctx, &ctx->d_bitmap, cap / 32 + 64));
  TRY(grow(ctx, &ctx->d_bpre, cap / 32 + 64));
  ctx->cap_px = cap;
  const size_t tiles = (P + TILE_PX - 1) / TILE_PX + 1;
  if (tiles > ctx->cap_tiles) {
    TRY(grow(ctx, &ctx->tile_state, tiles + 1));
    ctx->cap_tiles = tiles;
  }
  return CQB_OK;
}

int ensure_samples(cqb_ctx* ctx, size_t n) {
  if (n <= ctx->cap_s) return CQB_OK;
  const size_t cap = n + 64;
  TRY(grow(ctx, &ctx->d_keys, cap));
  TRY(grow(ctx, &ctx->d_counts, cap));
  TRY(grow(ctx, &ctx->d_first, cap));
  TRY(grow(ctx, &ctx->d_labels, cap));
  TRY(grow(ctx, &ctx->d_lab_rank, cap));
  TRY(grow(ctx, &ctx->d_mkeys, cap));
  TRY(grow(ctx, &ctx->d_mcounts, cap));
  TRY(grow(ctx, &ctx->d_mrank, cap));
  TRY(grow(ctx, &ctx->d_weights, cap));
  ctx->cap_s = cap;
  return CQB_OK;
}

int ensure_hist(cqb_ctx* ctx, int n) {
  if (n <= ctx->cap_hist) return CQB_OK;
  TRY(grow(ctx, &ctx->d_hist, (size_t)n));
  TRY(grow(ctx, &ctx->d_timeline, (size_t)n * 8));
  if (ctx->h_hist) cudaFreeHost(ctx->h_hist);
  ctx->h_hist = nullptr;
  CK(cudaMallocHost(&ctx->h_hist, sizeof(double) * (size_t)n));
  ctx->cap_hist = n;
  return CQB_OK;
}

int check_term(cqb_ctx* ctx, const cqb_termination* t) {
  if (!t) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "termination is null");
  if (t->mode == 1) {
    if (!(t->epsilon > 0)) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "convergent termination requires epsilon > 0");
    if (t->hard_cap < 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hard_cap must be >= 1");
  } else if (t->mode == 0) {
    if (t->max_iters < 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "max_iters must be >= 1");
  } else {
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "unknown termination mode %d", t->mode);
  }
  return CQB_OK;
}

int term_iters(const cqb_termination* t) { return t->mode == 1 ? t->hard_cap : t->max_iters; }

int check_k(cqb_ctx* ctx, int k) {
  if (k < 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "k must be >= 1");
  if (k > KMAX) return fail(ctx, CQB_ERR_UNSUPPORTED, "k = %d exceeds the device limit %d", k, KMAX);
  return CQB_OK;
}

// Raw mt19937_64 stream for init_centers (kmeans.hpp:56-65). The stream does
// not depend on N', so it is produced here and consumed on device.
int upload_draws(cqb_ctx* ctx, uint64_t seed, int ndraws) {
  if (ctx->draws_valid && ctx->draws_seed == seed && ctx->draws_n >= ndraws) return CQB_OK;
  if (ndraws > ctx->cap_draws) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_draws) cudaFreeHost(ctx->h_draws);
    ctx->h_draws = nullptr;
    CK(cudaMallocHost(&ctx->h_draws, sizeof(unsigned long long) * (size_t)ndraws));
    TRY(grow(ctx, &ctx->d_draws, (size_t)ndraws));
    ctx->cap_draws = ndraws;
  }
  CK(cudaEventSynchronize(ctx->ev[3]));  // previous upload finished reading h_draws
  std::mt19937_64 g(seed);
  for (int i = 0; i < ndraws; ++i) ctx->h_draws[i] = g();
  CK(cudaMemcpyAsync(ctx->d_draws, ctx->h_draws, sizeof(unsigned long long) * (size_t)ndraws, cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaEventRecord(ctx->ev[3], ctx->stream));
  ctx->draws_valid = true;
  ctx->draws_seed = seed;
  ctx->draws_n = ndraws;
  return CQB_OK;
}

int loop_grid(cqb_ctx* ctx) {
  int g = ctx->loop_blocks_max;
  if (ctx->grid_limit > 0) g = std::min(g, ctx->grid_limit);
  return std::max(1, std::min(g, MAXBLK));
}

// Zero the small per-run state (accumulators + scalars).
int reset_state(cqb_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->st->acc, 0, sizeof(ctx->st->acc), ctx->stream));
  CK(cudaMemsetAsync(&ctx->st->evals, 0,
                     sizeof(WsmState) - offsetof(WsmState, evals), ctx->stream));
  return CQB_OK;
}

// K2b: Morton-order samples from the bin table (also zeroes it). With
// `bitmap`, the bins hold ~first pixel index (K1) and K2b emits first indices
// + sets the first-occurrence bitmap; without, they hold ranks
// (k_bins_scatter).
int enqueue_morton(cqb_ctx* ctx, uint32_t* bitmap = nullptr, int first_mode = 0) {
  CK(cudaMemsetAsync(ctx->bin_tile_state, 0, sizeof(unsigned long long) * (N_BIN_TILES + 1), ctx->stream));
  k_bins_compact<<<N_BIN_TILES, BC_THREADS, 0, ctx->stream>>>(
      ctx->bins, ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->bin_tile_state,
      reinterpret_cast<unsigned int*>(ctx->bin_tile_state + N_BIN_TILES), ctx->d_n, bitmap,
      bitmap || first_mode ? 1 : 0);
  CKL();
  return CQB_OK;
}

// init_centers from first pixel indices (hist.cuh RS1-RS4): the samples carry
// their first pixel in d_mrank; center i = the chosen[i]-th smallest of them.
int enqueue_rank_select(cqb_ctx* ctx, const uint8_t* d_img, uint64_t P, int k, int ndraws) {
  const int cs = rank_select_shift(P);
  const int nc = (int)((P + (1ull << cs) - 1) >> cs);
  const int wps = 1 << (cs - 5);
  if ((size_t)KMAX * wps > ctx->cap_slot_bits) {
    TRY(grow(ctx, &ctx->rs_slot_bits, (size_t)KMAX * wps));
    ctx->cap_slot_bits = (size_t)KMAX * wps;
  }
  CK(cudaMemsetAsync(ctx->rs_coarse, 0, sizeof(uint32_t) * RS_NC, ctx->stream));
  k_first_coarse<<<ctx->num_sms, 1024, 0, ctx->stream>>>(ctx->d_mrank, ctx->d_n, cs, ctx->rs_coarse);
  CKL();
  k_init_select<<<1, RS_THREADS, 0, ctx->stream>>>(ctx->d_n, k, ctx->d_draws, ndraws, ctx->st, ctx->rs_coarse, nc,
                                                   ctx->rs_slot_of, ctx->rs_tgt, ctx->rs_tgt + KMAX,
                                                   ctx->rs_slot_bits, wps);
  CKL();
  k_first_mark<<<ctx->num_sms, 1024, 0, ctx->stream>>>(ctx->d_mrank, ctx->d_n, cs, ctx->rs_slot_of, wps,
                                                          ctx->rs_slot_bits);
  CKL();
  k_rank_pick<<<(k * 32 + 255) / 256, 256, 0, ctx->stream>>>(ctx->rs_slot_bits, wps, cs, ctx->rs_slot_of,
                                                              ctx->rs_tgt, ctx->rs_tgt + KMAX, d_img,
                                                              &ctx->st->status, k, ctx->st->C[0]);
  CKL();
  return CQB_OK;
}

// The whole unique-color reduction on ctx->stream over a device raster
// (16-B aligned), build_histogram (histogram.hpp:65-99):
//   K1   k_hist_count        2^24 Morton bins {count, ~first pixel}
//   K2b  k_bins_compact      Morton-order samples {key, count, first} (bins re-zeroed)
//                            + first-occurrence bitmap over the P pixels
//   K2c  k_bitmap_scan       per-word set-bit prefix
//   K2d  k_rank_from_bitmap  first-occurrence rank of every sample (and, for
//                            the build_histogram API, the histogram in
//                            first-occurrence order)
// Everything after K1 is N'-proportional; no pass re-reads the pixels.
// Images below this size compact the bin table through K1's occupancy map
// (their tables are sparse: cfg2's 0.37M colors touch 2% of the bins).
constexpr uint64_t OCC_MAX_PIXELS = 2u << 20;
constexpr size_t RES_DYN_MAX = (CQB_LOOP_MINB == 1 ? 160 : 40) * 1024;  // resident-sample loop: dynamic shared memory ceiling

bool sparse_path(const cqb_ctx* ctx, uint64_t P) { return P < OCC_MAX_PIXELS && !(ctx->debug_flags & 16); }
bool fused_prep(const cqb_ctx* ctx, uint64_t P) {
  return sparse_path(ctx, P) && ctx->prep_blocks > 0 && !(ctx->debug_flags & 32);
}

// zero_state (quantize path): the fused small-image kernel also zeroes the
// bitmap, the moment sums and the run scalars, replacing four host memsets.
int enqueue_histogram(cqb_ctx* ctx, const uint8_t* d_img, uint64_t P, bool stamps = false,
                      bool rank_order = false, int init_k = 0, int ndraws = 0, bool zero_state = false) {
  const uint64_t nchunk = (P + PX_PER_THREAD - 1) / PX_PER_THREAD;
  const uint32_t n_words = (uint32_t)((P + 31) / 32);
  const uint32_t ntiles = (n_words + BS_WORDS - 1) / BS_WORDS;
  const bool fused = fused_prep(ctx, P);
  // the dense quantize path (K2b without the bitmap + rank selection) uses
  // neither the first-occurrence bitmap nor the bitmap-scan look-back state
  const bool no_bitmap = !sparse_path(ctx, P) && !rank_order;
  if (!(fused && zero_state) && !no_bitmap)
    CK(cudaMemsetAsync(ctx->d_bitmap, 0, sizeof(uint32_t) * n_words, ctx->stream));
  if (!fused && !no_bitmap) CK(cudaMemsetAsync(ctx->tile_state, 0, sizeof(unsigned long long) * (ntiles + 1), ctx->stream));
  if (stamps && ctx->profiling) CK(cudaEventRecord(ctx->pev[1], ctx->stream));
  const int g1 = (int)std::min<uint64_t>((nchunk + HIST_THREADS - 1) / HIST_THREADS, (uint64_t)ctx->num_sms * CQB_K1_GRID);
  // Sparse tables (small images) are compacted through the occupancy map;
  // dense ones by scanning all 128 MiB (k_bins_compact), whose K1 runs in
  // 4 Morton slices so each pass's atomics stay in L2.
  const bool sparse = sparse_path(ctx, P);
  // fused: K1 runs inside k_prep_small; k1_done: cqb_quantize_ex ran it per H2D slice
  const int passes = fused || ctx->k1_done ? 0 : (P >= (4u << 20) ? ((ctx->debug_flags & DBG_K1_2PASS) ? 2 : (ctx->debug_flags & DBG_K1_1PASS) ? 1 : 4) : 1);
  for (int q = 0; q < passes; ++q) {
    const uint32_t span = (1u << 24) / passes;
    const uint32_t mlo = q * span, mhi = q + 1 == passes ? (1u << 24) : (q + 1) * span;
    if (passes <= 2 && !sparse)  // half-table passes: the raster streams (evict-first) so the slice stays in L2
      k_hist_count<true><<<std::max(g1, 1), HIST_THREADS, 0, ctx->stream>>>(d_img, P, ctx->bins, mlo, mhi,
                                                                           sparse ? ctx->d_occ : nullptr);
    else
      k_hist_count<<<std::max(g1, 1), HIST_THREADS, 0, ctx->stream>>>(d_img, P, ctx->bins, mlo, mhi,
                                                                      sparse ? ctx->d_occ : nullptr);
    CKL();
  }
  if (stamps && ctx->profiling) CK(cudaEventRecord(ctx->pev[2], ctx->stream));
  if (fused) {
    // compaction, first-occurrence ranks and init in one cooperative launch
    if (stamps && ctx->profiling) CK(cudaEventRecord(ctx->pev[3], ctx->stream));
    PrepParams Q{};
    Q.img = d_img;
    Q.P = P;
    Q.hist = 1;
    Q.occ = ctx->d_occ;
    Q.bins = ctx->bins;
    Q.m_keys = ctx->d_mkeys;
    Q.m_counts = ctx->d_mcounts;
    Q.m_rank = ctx->d_mrank;
    Q.n_unique = ctx->d_n;
    Q.bitmap = ctx->d_bitmap;
    Q.pre = ctx->d_bpre;
    Q.n_words = n_words;
    Q.block_counts = ctx->d_block_counts;
    Q.wofs = ctx->d_wofs;
    Q.units = ctx->d_units;
    Q.draws = ctx->d_draws;
    Q.ndraws = ndraws;
    Q.k = init_k;
    Q.st = ctx->st;
    Q.r_keys = rank_order ? ctx->d_keys : nullptr;
    Q.r_counts = ctx->d_counts;
    Q.r_first = ctx->d_first;
    Q.stamps = ctx->profiling ? ctx->d_block_times + 14 * MAXBLK : nullptr;
    Q.zero_state = zero_state ? 1 : 0;
    void* args[] = {&Q};
    // honour the lane's SM slice (cqb_quantize_batch) like the loop kernel
    const int pg = std::max(1, std::min(ctx->prep_blocks, ctx->grid_limit > 0 ? ctx->grid_limit : MAXBLK));
    CK(cudaLaunchCooperativeKernel((const void*)k_prep_small, dim3(pg),
                                   dim3(PREP_THREADS), args, 0, ctx->stream));
    CKL();
    return CQB_OK;
  }
  if (sparse) {
    CK(cudaMemsetAsync(ctx->bin_tile_state, 0, sizeof(unsigned long long) * (N_OCC_TILES + 1), ctx->stream));
    k_occ_compact<<<N_OCC_TILES, OC_THREADS, 0, ctx->stream>>>(
        ctx->d_occ, ctx->bins, ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->bin_tile_state,
        reinterpret_cast<unsigned int*>(ctx->bin_tile_state + N_OCC_TILES), ctx->d_n, ctx->d_bitmap);
    CKL();
  } else if (!rank_order) {
    // quantize path: samples keep their first pixel; init selects its ranks
    TRY(enqueue_morton(ctx, nullptr, 1));
    if (stamps && ctx->profiling) CK(cudaEventRecord(ctx->pev[3], ctx->stream));
    if (init_k > 0) TRY(enqueue_rank_select(ctx, d_img, P, init_k, ndraws));
    return CQB_OK;
  } else {
    TRY(enqueue_morton(ctx, ctx->d_bitmap));
  }
  if (init_k > 0) {  // init_centers needs only N': its chosen ranks, gathered by the rank pass
    if (stamps && ctx->profiling) CK(cudaEventRecord(ctx->pev[3], ctx->stream));
    k_init_centers<<<1, KMAX, 0, ctx->stream>>>(nullptr, ctx->d_n, init_k, ctx->d_draws, ndraws, ctx->st);
    CKL();
  }
  k_bitmap_scan<<<ntiles, BS_THREADS, 0, ctx->stream>>>(ctx->d_bitmap, n_words, ctx->d_bpre, ctx->tile_state,
                                                        reinterpret_cast<unsigned int*>(ctx->tile_state + ntiles));
  CKL();
  k_rank_from_bitmap<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(
      ctx->d_bitmap, ctx->d_bpre, ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->d_n,
      rank_order ? ctx->d_keys : nullptr, ctx->d_counts, ctx->d_first, init_k > 0 ? ctx->st->chosen : nullptr,
      &ctx->st->status, init_k, ctx->st->C[0]);
  CKL();
  return CQB_OK;
}

int launch_loop(cqb_ctx* ctx, int k, const cqb_termination* term, int dense_first, uint64_t total, double* traj,
                int traj_cap, uint64_t shard_lo = 0, uint64_t shard_hi = ~0ull, int moments_only = 0) {
  LoopParams L{};
  L.keys = ctx->d_mkeys;
  L.counts = ctx->d_mcounts;
  L.rank = ctx->d_mrank;
  L.labels = ctx->d_labels;
  L.n_ptr = ctx->d_n;
  L.shard_lo = shard_lo;
  L.shard_hi_or_max = shard_hi;
  L.moments_only = moments_only;
  L.total = total;
  L.k = k;
  L.mode = term->mode;
  L.max_iters = term->max_iters;
  L.eps = term->epsilon;
  L.cap = term->hard_cap;
  L.dense_first = dense_first;
  L.st = ctx->st;
  L.sse_hist = ctx->d_hist;
  L.hist_cap = ctx->cap_hist;
  L.traj = traj;
  L.traj_cap = traj_cap;
  L.timeline = ctx->profiling ? ctx->d_timeline : nullptr;
  L.block_times = ctx->profiling ? ctx->d_block_times : nullptr;
  L.stamp_iter = ctx->stamp_iter;
  L.debug_flags = ctx->debug_flags;
  ctx->coarse_built = false;
  if (ctx->fuse_map && !(ctx->debug_flags & 256)) {
    L.map_sortedDr = ctx->d_sortedDr;
    L.map_orderR = ctx->d_orderR;
    L.map_palkey = ctx->d_palkey;
    L.map_lut = ctx->lut;
    // large images: the coarse map table for k_map_pixels_coarse
    ctx->coarse_built = total >= OCC_MAX_PIXELS && !(ctx->debug_flags & DBG_NO_COARSE);
    if (ctx->coarse_built) {
      L.map_cellw = ctx->d_cellw;
      L.map_coarse = ctx->d_coarse;
    }
  }
  if (dense_first && !(ctx->debug_flags & 128)) {  // iteration 1 on per-cell candidate lists
    k_grid_cands<<<CAND_CELLS, KMAX, 0, ctx->stream>>>(ctx->st, k, ctx->d_cand, ctx->d_cand_n);
    CKL();
    L.cand = ctx->d_cand;
    L.cand_n = ctx->d_cand_n;
  }
  if (ctx->profiling)
    CK(cudaMemsetAsync(ctx->d_timeline, 0, sizeof(unsigned long long) * 8 * (size_t)ctx->cap_hist, ctx->stream));
  int X = 0;
  unsigned grid = (unsigned)loop_grid(ctx);
  if (ctx->xsharded) {
    X = ctx->xmode;
    L.xw = ctx->xw;
    L.xrank = X == 1 ? ctx->xrank : -1;
    L.xch_timeout_ns = ctx->xch_timeout_ns;
    for (int r = 0; r < ctx->xw; ++r) L.xbox[r] = ctx->xpeer[r];
    if (X == 1) L.labels = reinterpret_cast<uint8_t*>(ctx->xwin) + XB_LAB_OFF;
    if (X == 2) {
      L.xacc = ctx->xacc;
      grid = grid / (unsigned)ctx->xw * (unsigned)ctx->xw;  // equal block groups
      CK(cudaMemsetAsync(ctx->xacc, 0, sizeof(unsigned long long) * 5 * KMAX * ctx->xw, ctx->stream));
    }
  }
  void* args[] = {&L};
  // one point per lane per grab for small sample sets (N' <= P < 2M): finer
  // balance; two for large ones: more ILP (cfg2 +1.2%, cfg4 +8% respectively)
  const bool small = total < OCC_MAX_PIXELS;
  const void* kern = X == 1   ? (small ? (const void*)k_wsm_loop<1, 1> : (const void*)k_wsm_loop<CQB_PPT_LARGE, 1>)
                     : X == 2 ? (small ? (const void*)k_wsm_loop<1, 2> : (const void*)k_wsm_loop<CQB_PPT_LARGE, 2>)
                              : (small ? (const void*)k_wsm_loop<1, 0> : (const void*)k_wsm_loop<CQB_PPT_LARGE, 0>);
  size_t dyn = small ? LOOP_DYN_SMALL : LOOP_DYN_LARGE;
  if (X == 0 && small && !(ctx->debug_flags & 512)) {
    // resident samples when the block's share (bounded by P) fits in shared memory
    const uint64_t cap = ((total + 31) / 32 + grid - 1) / grid * 32;
    if (res_smem_bytes((int)std::min<uint64_t>(cap, 1u << 24)) <= RES_DYN_MAX) {
      L.res_cap = (int)cap;
      dyn = res_smem_bytes(L.res_cap);
      kern = (const void*)k_wsm_loop<1, 0, true>;
    }
  }
  CK(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(LOOP_THREADS), args, dyn, ctx->stream));
  CKL();
  return CQB_OK;
}

// The per-call results into the pinned staging block with one tiny kernel
// (zero-copy stores into mapped host memory) instead of six small D2H copies.
__global__ void k_publish(const WsmState* __restrict__ st, const unsigned long long* __restrict__ d_n,
                          const double* __restrict__ d_hist, int k, int hist_n, Staging* h, double* h_hist) {
  const int t = threadIdx.x;
  for (int i = t; i < 3 * k; i += blockDim.x) h->centers[i] = st->final_C[i];
  const int nh = min(hist_n, st->iterations);
  for (int i = t; i < nh; i += blockDim.x) h_hist[i] = d_hist[i];
  if (t == 0) {
    h->evals = st->evals;
    h->mse_err = st->mse_err;
    h->n_unique = *d_n;
    h->sse = st->sse;
    h->iterations = st->iterations;
    h->status = st->status;
    h->n_empty = st->n_empty_events;
  }
}

int stage_results(cqb_ctx* ctx, int k, int hist_n) {
  Staging* h = ctx->h_stage;
  WsmState* st = ctx->st;
  if (!(ctx->debug_flags & 65536)) {
    k_publish<<<1, 256, 0, ctx->stream>>>(st, ctx->d_n, ctx->d_hist, k, hist_n, h, ctx->h_hist);
    CKL();
    return CQB_OK;
  }
  CK(cudaMemcpyAsync(h->centers, st->final_C, sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&h->evals, &st->evals, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&h->mse_err, &st->mse_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&h->n_unique, ctx->d_n, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&h->sse, &st->sse, sizeof(double) + 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  if (hist_n > 0)
    CK(cudaMemcpyAsync(ctx->h_hist, ctx->d_hist, sizeof(double) * (size_t)hist_n, cudaMemcpyDeviceToHost, ctx->stream));
  return CQB_OK;
}

int check_status(cqb_ctx* ctx) {
  const int s = ctx->h_stage->status;
  if (s == ST_K_EXCEEDS_N)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "init_centers: k exceeds the number of candidate points");
  if (s == ST_DRAWS_EXHAUSTED) return fail(ctx, CQB_ERR_INTERNAL, "init_centers: raw draw buffer exhausted");
  if (s == ST_XCH_TIMEOUT) {
    // the ranks' exchange counters and flags no longer agree: the windows
    // must be set up again (cqb_xch_window + cqb_xch_open, or cqb_xch_emulate)
    // before the next sharded call
    ctx->xmode = 0;
    return fail(ctx, CQB_ERR_NCCL, "sharded loop: a peer rank did not answer within %.3g s; exchange reset",
                (double)ctx->xch_timeout_ns * 1e-9);
  }
  if (s != ST_OK) return fail(ctx, CQB_ERR_INTERNAL, "device status %d", s);
  return CQB_OK;
}

void fill_report(cqb_ctx* ctx, int k, uint64_t seed, uint64_t total, double* centers_out, double* sse_history,
                 int hist_cap, cqb_report* rep) {
  const Staging* h = ctx->h_stage;
  if (centers_out) memcpy(centers_out, h->centers, sizeof(double) * 3 * (size_t)k);
  if (sse_history)
    for (int i = 0; i < std::min(hist_cap, h->iterations); ++i) sse_history[i] = ctx->h_hist[i];
  if (rep) {
    rep->iterations = h->iterations;
    rep->k = k;
    rep->seed = seed;
    rep->sse = h->sse;
    rep->mse = total ? (double)h->mse_err / (double)total : 0.0;
    rep->dist_evals = h->evals;
    rep->n_unique = h->n_unique;
    rep->empty_events = h->n_empty;
    rep->gpu_launches = ctx->launches;
    float ms = 0.f;
    rep->elapsed_ms = cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]) == cudaSuccess ? ms : 0.0;
    rep->map_ms = cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]) == cudaSuccess ? ms : 0.0;
    cudaGetLastError();
  }
}

// The fused device pipeline: histogram -> init -> WSM loop -> map + MSE.
#define PROF(i)                                                   \
  do {                                                            \
    if (ctx->profiling) CK(cudaEventRecord(ctx->pev[i], ctx->stream)); \
  } while (0)

int enqueue_quantize(cqb_ctx* ctx, const uint8_t* d_img, uint64_t P, int k, const cqb_termination* term,
                     uint64_t seed, uint8_t* d_index, uint8_t* d_rgb_out, int ndraws) {
  ctx->launches = 0;
  TRY(ensure_samples(ctx, P));
  TRY(ensure_hist(ctx, term_iters(term)));
  TRY(upload_draws(ctx, seed, ndraws));
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  PROF(0);
  if (ctx->ext_samples) {  // the histogram came from the pixel-row shards (cqb_hist_rows / cqb_hist_merge)
    TRY(reset_state(ctx));
    const int gu = (int)std::min<uint64_t>((ctx->ext_n + 255) / 256, (uint64_t)ctx->num_sms * 8);
    k_unpack_triplets<<<std::max(gu, 1), 256, 0, ctx->stream>>>(ctx->ext_samples, ctx->ext_n, ctx->d_mkeys,
                                                                ctx->d_mcounts, ctx->d_mrank, ctx->d_n);
    CKL();
    PROF(1);
    PROF(2);
    PROF(3);
    TRY(enqueue_rank_select(ctx, d_img, P, k, ndraws));
  } else {
    const bool fused = fused_prep(ctx, P);
    if (!fused) TRY(reset_state(ctx));  // else zeroed inside k_prep_small
    TRY(enqueue_histogram(ctx, d_img, P, true, false, k, ndraws, fused));  // records PROF(1..3)
  }
  PROF(4);
  ctx->fuse_map = true;  // k_map_tables + k_map_unique run in the loop kernel's tail
  const int lrc = launch_loop(ctx, k, term, 1, P, nullptr, 0);
  const bool fused_map = !(ctx->debug_flags & 256);
  ctx->fuse_map = false;
  TRY(lrc);
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  PROF(5);
  if (!fused_map) {
    k_map_tables<<<k, 256, 0, ctx->stream>>>(ctx->st->final_C, k, ctx->d_sortedDr, ctx->d_orderR, ctx->d_palkey);
    CKL();
    const int gu = ctx->num_sms * 4;
    k_map_unique<<<gu, 256, 0, ctx->stream>>>(ctx->d_mkeys, ctx->d_mcounts, ctx->d_labels, ctx->d_n, k,
                                              ctx->d_sortedDr, ctx->d_orderR, ctx->d_palkey, ctx->lut,
                                              &ctx->st->mse_err);
    CKL();
  }
  PROF(6);
  uint8_t* d_err_out = ctx->err_target;
  // sharded: this rank maps its pixel range only (offsets are multiples of 16 pixels: aligned vectors)
  const uint64_t plo = ctx->xsharded ? ctx->px_lo : 0, pn = ctx->xsharded ? ctx->px_hi - ctx->px_lo : P;
  const bool d2h = ctx->h_index_dst || ctx->h_rgb_dst || ctx->h_err_dst;
  if ((d_index || d_rgb_out || d_err_out) && pn > 0) {
    // with host targets (cqb_quantize_ex): XFER_CHUNKS map launches, each
    // slice's D2H copies on ctx->xfer overlapping the next slice's map
    const uint64_t q16 = (pn + 15) / 16;
    const int nch = d2h ? XFER_CHUNKS : 1;
    for (int c = 0; c < nch; ++c) {
      const uint64_t a = plo + std::min(pn, q16 * c / nch * 16), b = plo + std::min(pn, q16 * (c + 1) / nch * 16);
      if (b <= a) continue;
      const uint64_t nchunk = (b - a + PX_PER_THREAD - 1) / PX_PER_THREAD;
      if (ctx->coarse_built && fused_map) {
        const int g = (int)std::min<uint64_t>((nchunk + MAPC_THREADS - 1) / MAPC_THREADS, (uint64_t)ctx->num_sms);
        k_map_pixels_coarse<<<std::max(g, 1), MAPC_THREADS, COARSE_BYTES, ctx->stream>>>(
            d_img + 3 * a, b - a, ctx->lut, ctx->d_coarse, ctx->d_palkey, k, d_index ? d_index + a : nullptr,
            d_rgb_out ? d_rgb_out + 3 * a : nullptr, d_err_out ? d_err_out + 3 * a : nullptr);
      } else {
        const int g = (int)std::min<uint64_t>((nchunk + HIST_THREADS - 1) / HIST_THREADS, (uint64_t)ctx->num_sms * 16);
        k_map_pixels<<<std::max(g, 1), HIST_THREADS, 0, ctx->stream>>>(
            d_img + 3 * a, b - a, ctx->lut, ctx->d_palkey, k, d_index ? d_index + a : nullptr,
            d_rgb_out ? d_rgb_out + 3 * a : nullptr, d_err_out ? d_err_out + 3 * a : nullptr);
      }
      CKL();
      if (d2h) {
        CK(cudaEventRecord(ctx->xev[XFER_CHUNKS + c], ctx->stream));
        CK(cudaStreamWaitEvent(ctx->xfer, ctx->xev[XFER_CHUNKS + c], 0));
        if (ctx->h_index_dst && d_index)
          CK(cudaMemcpyAsync(ctx->h_index_dst + a, d_index + a, b - a, cudaMemcpyDeviceToHost, ctx->xfer));
        if (ctx->h_rgb_dst && d_rgb_out)
          CK(cudaMemcpyAsync(ctx->h_rgb_dst + 3 * a, d_rgb_out + 3 * a, 3 * (b - a), cudaMemcpyDeviceToHost,
                             ctx->xfer));
        if (ctx->h_err_dst && d_err_out)
          CK(cudaMemcpyAsync(ctx->h_err_dst + 3 * a, d_err_out + 3 * a, 3 * (b - a), cudaMemcpyDeviceToHost,
                             ctx->xfer));
      }
    }
    if (d2h) {  // the caller's stream synchronisation covers the copies
      CK(cudaEventRecord(ctx->xev[2 * XFER_CHUNKS], ctx->xfer));
      CK(cudaStreamWaitEvent(ctx->stream, ctx->xev[2 * XFER_CHUNKS], 0));
    }
  }
  PROF(7);
  CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  TRY(stage_results(ctx, k, term_iters(term)));
  ctx->last_k = k;
  ctx->last_P = P;
  ctx->last_hist_cap = term_iters(term);
  return CQB_OK;
}

// The copy stream and its events (cqb_quantize_ex on large images).
int ensure_xfer(cqb_ctx* ctx) {
  if (ctx->xfer) return CQB_OK;
  CK(cudaStreamCreateWithFlags(&ctx->xfer, cudaStreamNonBlocking));
  for (auto& e : ctx->xev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return CQB_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Device view of a pinned, mapped host buffer (16-B aligned), else null.
// (allocated while this context's device was current: no cross-device mapping assumptions)
uint8_t* mapped_view(void* p, int device) {
  if (!p) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || a.device != device || !a.devicePointer || !aligned16(a.devicePointer))
    return nullptr;
  return static_cast<uint8_t*>(a.devicePointer);
}

}  // namespace

extern "C" {

int cqb_create(int device, cqb_ctx** out) {
  cqb_ctx* ctx = nullptr;
  if (!out) return CQB_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  ctx = new (std::nothrow) cqb_ctx();
  if (!ctx) return CQB_ERR_OOM;
  ctx->device = device;
  int rc = [&]() -> int {
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      return fail(ctx, CQB_ERR_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)", device,
                  prop.major, prop.minor);
    if (!prop.cooperativeLaunch) return fail(ctx, CQB_ERR_UNSUPPORTED, "cooperative launch unsupported");
    ctx->num_sms = prop.multiProcessorCount;
    int nb = 0;
    for (const void* f : {(const void*)k_wsm_loop<1, 0>, (const void*)k_wsm_loop<1, 1>, (const void*)k_wsm_loop<1, 2>})
      CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LOOP_DYN_SMALL));
    for (const void* f : {(const void*)k_wsm_loop<CQB_PPT_LARGE, 0>, (const void*)k_wsm_loop<CQB_PPT_LARGE, 1>,
                          (const void*)k_wsm_loop<CQB_PPT_LARGE, 2>})
      CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LOOP_DYN_LARGE));
    CK(cudaFuncSetAttribute((const void*)k_wsm_loop<1, 0, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RES_DYN_MAX));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wsm_loop<CQB_PPT_LARGE, 0>, LOOP_THREADS,
                                                     LOOP_DYN_LARGE));
    if (nb < 1) return fail(ctx, CQB_ERR_INTERNAL, "WSM loop kernel cannot be resident");
    ctx->loop_blocks_max = std::min(nb, CQB_LOOP_MINB) * ctx->num_sms;
    CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    CK(cudaMalloc(&ctx->bins, sizeof(uint2) << 24));
    CK(cudaMemset(ctx->bins, 0, sizeof(uint2) << 24));
    CK(cudaMalloc(&ctx->d_occ, sizeof(uint32_t) << 19));
    CK(cudaMalloc(&ctx->d_block_counts, sizeof(uint32_t) * 3 * MAXBLK));
    CK(cudaMalloc(&ctx->d_units, sizeof(uint32_t) * ((4u << 19) + 4 * MAXBLK)));
    CK(cudaMalloc(&ctx->d_cand, (size_t)CAND_CELLS * CAND_CAP));
    CK(cudaMalloc(&ctx->d_cand_n, sizeof(uint16_t) * CAND_CELLS));
    CK(cudaMalloc(&ctx->d_wofs, sizeof(uint32_t) << 19));
    CK(cudaMalloc(&ctx->rs_coarse, sizeof(uint32_t) * RS_NC));
    CK(cudaMalloc(&ctx->rs_slot_of, sizeof(uint16_t) * RS_NC));
    CK(cudaMalloc(&ctx->rs_tgt, sizeof(uint32_t) * 2 * KMAX));
    int pb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pb, k_prep_small, PREP_THREADS, 0));
    ctx->prep_blocks = std::min(std::max(pb, 0), 1) * ctx->num_sms;
    CK(cudaMemset(ctx->d_occ, 0, sizeof(uint32_t) << 19));
    CK(cudaMalloc(&ctx->lut, (size_t)1 << 24));
    CK(cudaMalloc(&ctx->d_cellw, sizeof(uint32_t) * COARSE_CELLS));
    CK(cudaMalloc(&ctx->d_coarse, COARSE_BYTES));
    CK(cudaFuncSetAttribute((const void*)k_map_pixels_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)COARSE_BYTES));
    CK(cudaMalloc(&ctx->bin_tile_state, sizeof(unsigned long long) * (N_BIN_TILES + 1)));
    CK(cudaMalloc(&ctx->st, sizeof(WsmState)));
    CK(cudaMemset(ctx->st, 0, sizeof(WsmState)));
    CK(cudaMalloc(&ctx->d_n, sizeof(unsigned long long)));
    CK(cudaMalloc(&ctx->d_centers_in, sizeof(double) * 3 * KMAX));
    CK(cudaMalloc(&ctx->d_block_times, sizeof(unsigned long long) * 16 * MAXBLK));
    CK(cudaMalloc(&ctx->d_mom, sizeof(unsigned long long) * 5 * KMAX));
    CK(cudaMallocHost(&ctx->h_mom, sizeof(unsigned long long) * (5 * KMAX + 1)));
    CK(cudaMalloc(&ctx->d_Cnew, sizeof(double) * 3 * KMAX));
    CK(cudaMalloc(&ctx->d_scal, sizeof(double) * 24));  // [0..7] sse + reseed, [8..16] cqb_hist_rows owner bounds
    CK(cudaMalloc(&ctx->d_ints, sizeof(int) * (KMAX + 8)));
    CK(cudaMalloc(&ctx->d_taken, sizeof(uint32_t) * KMAX));
    CK(cudaMalloc(&ctx->d_cand_d, sizeof(double) * MAXBLK));
    CK(cudaMalloc(&ctx->d_cand_r, sizeof(unsigned int) * MAXBLK));
    CK(cudaMalloc(&ctx->d_cand_k, sizeof(unsigned int) * MAXBLK));
    CK(cudaMalloc(&ctx->d_sortedDr, sizeof(int) * KMAX * KMAX));
    CK(cudaMalloc(&ctx->d_orderR, KMAX * KMAX));
    CK(cudaMalloc(&ctx->d_palkey, sizeof(uint32_t) * KMAX));
    CK(cudaMallocHost(&ctx->h_stage, sizeof(Staging)));
    CK(cudaMallocHost(&ctx->h_scalar, sizeof(unsigned long long) * 4));
    for (auto& e : ctx->ev) CK(cudaEventCreate(&e));
    for (auto& e : ctx->pev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ctx->ev[3], ctx->stream));
    CK(cudaDeviceSynchronize());
    return CQB_OK;
  }();
  if (rc != CQB_OK) {
    static thread_local std::string last;
    last = ctx->err;
    cqb_destroy(ctx);
    fprintf(stderr, "cqb_create: %s\n", last.c_str());
    return rc;
  }
  *out = ctx;
  return CQB_OK;
}

int cqb_destroy(cqb_ctx* ctx) {
  if (!ctx) return CQB_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  void* dev[] = {ctx->bins, ctx->lut, ctx->d_cellw, ctx->d_coarse, ctx->d_img, ctx->d_img2, ctx->d_index, ctx->d_rgb, ctx->d_err, ctx->tile_state,
                 ctx->d_keys, ctx->d_counts, ctx->d_first, ctx->d_bitmap, ctx->d_occ, ctx->d_block_counts, ctx->d_units, ctx->d_wofs, ctx->d_cand, ctx->d_cand_n, ctx->d_bpre, ctx->d_labels, ctx->d_lab_rank, ctx->d_mkeys,
                 ctx->d_mcounts, ctx->d_mrank, ctx->bin_tile_state, ctx->d_weights, ctx->d_n, ctx->st,
                 ctx->d_hist, ctx->d_timeline, ctx->d_block_times, ctx->d_mom, ctx->d_Cnew, ctx->d_scal,
                 ctx->d_ints, ctx->d_taken, ctx->d_cand_d, ctx->d_cand_r, ctx->d_cand_k, ctx->d_traj, ctx->d_centers_in, ctx->d_sortedDr, ctx->d_orderR, ctx->d_palkey,
                 ctx->d_draws, ctx->rs_coarse, ctx->rs_slot_of, ctx->rs_tgt, ctx->rs_slot_bits,
                 ctx->pts.X, ctx->pts.W, ctx->pts.m, ctx->pts.perm, ctx->pts.skip, ctx->pts.prevd,
                 ctx->pts.tcnt, ctx->pts.toff, ctx->pts.C, ctx->pts.next, ctx->pts.taken, ctx->pts.dists,
                 ctx->pts.order, ctx->pts.sortedD, ctx->pts.start, ctx->pts.empty, ctx->pts.part,
                 ctx->pts.cand_i, ctx->pts.scal, ctx->pts.evals, ctx->pts.chosen};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (ctx->h_draws) cudaFreeHost(ctx->h_draws);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->h_hist) cudaFreeHost(ctx->h_hist);
  if (ctx->h_scalar) cudaFreeHost(ctx->h_scalar);
  if (ctx->h_mom) cudaFreeHost(ctx->h_mom);
  if (ctx->xmode == 1)
    for (int r = 0; r < ctx->xw; ++r)
      if (r != ctx->xrank && ctx->xpeer[r]) cudaIpcCloseMemHandle(ctx->xpeer[r]);
  if (ctx->xwin) cudaFree(ctx->xwin);
  if (ctx->xacc) cudaFree(ctx->xacc);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->pev)
    if (e) cudaEventDestroy(e);
  if (ctx->xfer) cudaStreamSynchronize(ctx->xfer);
  for (auto& e : ctx->xev)
    if (e) cudaEventDestroy(e);
  if (ctx->xfer) cudaStreamDestroy(ctx->xfer);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  for (cqb_ctx* l : ctx->lanes) cqb_destroy(l);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->lane_done) cudaEventDestroy(ctx->lane_done);
  delete ctx;
  return CQB_OK;
}

const char* cqb_last_error(const cqb_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int cqb_set_stream(cqb_ctx* ctx, void* stream) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  ctx->draws_valid = false;
  CK(cudaEventRecord(ctx->ev[3], ctx->stream));
  return CQB_OK;
}

int cqb_set_grid_limit(cqb_ctx* ctx, int max_blocks) {
  if (!ctx || max_blocks < 0) return CQB_ERR_INVALID_ARGUMENT;
  ctx->grid_limit = max_blocks;
  return CQB_OK;
}

int cqb_set_profiling(cqb_ctx* ctx, int on) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  ctx->profiling = on != 0;
  if (on > 1) ctx->stamp_iter = on;  // on > 1: also selects the iteration for per-block stamps
  return CQB_OK;
}

int cqb_set_debug(cqb_ctx* ctx, int flags) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  ctx->debug_flags = flags;
  return CQB_OK;
}

int cqb_stage_times(cqb_ctx* ctx, float* ms, int n) {
  if (!ctx || !ms) return CQB_ERR_INVALID_ARGUMENT;
  if (!ctx->profiling) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "profiling is off");
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n && i < 7; ++i) CK(cudaEventElapsedTime(&ms[i], ctx->pev[i], ctx->pev[i + 1]));
  return CQB_OK;
}

int cqb_loop_timeline(cqb_ctx* ctx, unsigned long long* stamps, int n_iters) {
  if (!ctx || !stamps) return CQB_ERR_INVALID_ARGUMENT;
  if (!ctx->profiling) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "profiling is off");
  CK(cudaStreamSynchronize(ctx->stream));
  const int n = std::min(n_iters, ctx->cap_hist);
  CK(cudaMemcpy(stamps, ctx->d_timeline, sizeof(unsigned long long) * 8 * (size_t)n, cudaMemcpyDeviceToHost));
  return CQB_OK;
}

int cqb_block_times(cqb_ctx* ctx, unsigned long long* out, int n) {
  if (!ctx || !out) return CQB_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(out, ctx->d_block_times, sizeof(unsigned long long) * (size_t)std::min(n, 16 * MAXBLK),
                cudaMemcpyDeviceToHost));
  return CQB_OK;
}

int cqb_device_info(cqb_ctx* ctx, int* num_sms, int* loop_blocks) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (num_sms) *num_sms = ctx->num_sms;
  if (loop_blocks) *loop_blocks = loop_grid(ctx);
  return CQB_OK;
}

int cqb_build_histogram(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, uint32_t* keys, uint32_t* counts,
                        double* weights, uint32_t* first_index, uint64_t cap, uint64_t* n_unique) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (n_pixels == 0 || !rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "build_histogram: empty image");
  if (n_pixels >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  CK(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  TRY(ensure_pixels(ctx, n_pixels));
  TRY(ensure_samples(ctx, n_pixels));
  CK(cudaMemcpyAsync(ctx->d_img, rgb, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  TRY(enqueue_histogram(ctx, ctx->d_img, n_pixels, false, true));
  if (weights) {
    k_hist_weights<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->d_counts, ctx->d_n, n_pixels, ctx->d_weights);
    CKL();
  }
  CK(cudaMemcpyAsync(ctx->h_scalar, ctx->d_n, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const uint64_t nu = ctx->h_scalar[0];
  if (n_unique) *n_unique = nu;
  if (nu > cap) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "output capacity %llu < N' = %llu",
                            (unsigned long long)cap, (unsigned long long)nu);
  if (keys) CK(cudaMemcpyAsync(keys, ctx->d_keys, 4 * nu, cudaMemcpyDeviceToHost, ctx->stream));
  if (counts) CK(cudaMemcpyAsync(counts, ctx->d_counts, 4 * nu, cudaMemcpyDeviceToHost, ctx->stream));
  if (first_index) CK(cudaMemcpyAsync(first_index, ctx->d_first, 4 * nu, cudaMemcpyDeviceToHost, ctx->stream));
  if (weights) CK(cudaMemcpyAsync(weights, ctx->d_weights, 8 * nu, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return CQB_OK;
}

static int run_loop_common(cqb_ctx* ctx, const uint32_t* keys, const uint32_t* counts, uint64_t n, uint64_t total,
                           int k, const cqb_termination* term, int dense_first, const double* centers_in,
                           const uint8_t* labels_in, uint64_t seed, double* centers_out, double* sse_history,
                           int hist_cap, double* trajectory, int traj_cap, uint8_t* labels_out, cqb_report* report) {
  if (k < 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "init_centers: k must be >= 1");
  if (n == 0) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "empty histogram");
  if ((uint64_t)k > n) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "init_centers: k exceeds the number of candidate points");
  TRY(check_k(ctx, k));
  TRY(check_term(ctx, term));
  if (total == 0) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "total_pixels must be > 0");
  CK(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  TRY(ensure_samples(ctx, n));
  TRY(ensure_hist(ctx, term_iters(term)));
  const int tcap = trajectory ? std::min(traj_cap, term_iters(term)) : 0;
  if (tcap > 0 && (size_t)tcap * 3 * k > ctx->cap_traj) {
    TRY(grow(ctx, &ctx->d_traj, (size_t)tcap * 3 * k));
    ctx->cap_traj = (size_t)tcap * 3 * k;
  }
  CK(cudaMemcpyAsync(ctx->d_keys, keys, 4 * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_counts, counts, 4 * n, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h_scalar[1] = n;
  CK(cudaMemcpyAsync(ctx->d_n, &ctx->h_scalar[1], sizeof(unsigned long long), cudaMemcpyHostToDevice, ctx->stream));
  k_bins_scatter<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->d_keys, ctx->d_counts, ctx->d_n, ctx->bins);
  CKL();
  TRY(enqueue_morton(ctx));
  if (labels_in) {
    CK(cudaMemcpyAsync(ctx->d_lab_rank, labels_in, n, cudaMemcpyHostToDevice, ctx->stream));
    k_labels_gather<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->d_mrank, ctx->d_lab_rank, ctx->d_labels, ctx->d_n);
    CKL();
  } else {
    CK(cudaMemsetAsync(ctx->d_labels, 0, n, ctx->stream));
  }
  TRY(reset_state(ctx));
  const int ndraws = k + 64;
  if (centers_in) {
    CK(cudaMemcpyAsync(ctx->st->C[0], centers_in, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    TRY(upload_draws(ctx, seed, ndraws));
  }
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (!centers_in) {
    k_init_centers<<<1, KMAX, 0, ctx->stream>>>(ctx->d_keys, ctx->d_n, k, ctx->d_draws, ndraws, ctx->st);
    CKL();
  }
  TRY(launch_loop(ctx, k, term, dense_first, total, tcap ? ctx->d_traj : nullptr, tcap));
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  TRY(stage_results(ctx, k, term_iters(term)));
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(check_status(ctx));
  if (ctx->h_stage->n_unique != n)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "histogram keys must be distinct (%llu distinct of %llu)",
                (unsigned long long)ctx->h_stage->n_unique, (unsigned long long)n);
  const int iters = ctx->h_stage->iterations;
  if (tcap > 0)
    CK(cudaMemcpy(trajectory, ctx->d_traj, sizeof(double) * 3 * (size_t)k * (size_t)std::min(tcap, iters),
                  cudaMemcpyDeviceToHost));
  if (labels_out) {
    k_labels_scatter<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->d_mrank, ctx->d_labels, ctx->d_lab_rank, ctx->d_n);
    CKL();
    CK(cudaMemcpyAsync(labels_out, ctx->d_lab_rank, n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  fill_report(ctx, k, seed, 0, centers_out, sse_history, hist_cap, report);
  return CQB_OK;
}

int cqb_run_wsm(cqb_ctx* ctx, const uint32_t* keys, const uint32_t* counts, uint64_t n_unique, uint64_t total,
                int k, const cqb_termination* term, uint64_t seed, double* centers_out, double* sse_history,
                int hist_cap, double* trajectory, int traj_cap, uint8_t* labels_out, cqb_report* report) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  return run_loop_common(ctx, keys, counts, n_unique, total, k, term, 1, nullptr, nullptr, seed, centers_out,
                         sse_history, hist_cap, trajectory, traj_cap, labels_out, report);
}

int cqb_wsm_iterate(cqb_ctx* ctx, const uint32_t* keys, const uint32_t* counts, uint64_t n_unique, uint64_t total,
                    int k, const double* centers_in, uint8_t* labels_inout, int dense_first,
                    const cqb_termination* term, double* centers_out, double* sse_history, int hist_cap,
                    cqb_report* report) {
  if (!ctx || !centers_in || !labels_inout) return CQB_ERR_INVALID_ARGUMENT;
  return run_loop_common(ctx, keys, counts, n_unique, total, k, term, dense_first, centers_in, labels_inout, 0,
                         centers_out, sse_history, hist_cap, nullptr, 0, labels_inout, report);
}

int cqb_quantize_device(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int k, const cqb_termination* term,
                        uint64_t seed, uint8_t* d_index_out, uint8_t* d_rgb_out, int sync, double* centers_out,
                        double* sse_history, int hist_cap, cqb_report* report) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  TRY(check_k(ctx, k));
  TRY(check_term(ctx, term));
  if (n_pixels == 0 || !d_rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "quantize: empty image");
  if (n_pixels >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  CK(cudaSetDevice(ctx->device));
  TRY(ensure_pixels(ctx, n_pixels));
  const uint8_t* img = d_rgb;
  if (!aligned16(d_rgb)) {  // vector loads need a 16-B aligned raster
    CK(cudaMemcpyAsync(ctx->d_img2, d_rgb, 3 * n_pixels, cudaMemcpyDeviceToDevice, ctx->stream));
    img = ctx->d_img2;
  }
  uint8_t* idx_out = d_index_out;
  uint8_t* rgb_out = d_rgb_out;
  if (idx_out && !aligned16(idx_out)) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "index output must be 16-B aligned");
  if (rgb_out && !aligned16(rgb_out)) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "rgb output must be 16-B aligned");
  int ndraws = k + 64;
  for (int attempt = 0; attempt < 4; ++attempt) {
    TRY(enqueue_quantize(ctx, img, n_pixels, k, term, seed, idx_out, rgb_out, ndraws));
    if (!sync) return CQB_OK;
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_stage->status == ST_DRAWS_EXHAUSTED) {
      ndraws *= 4;
      continue;
    }
    break;
  }
  TRY(check_status(ctx));
  fill_report(ctx, k, seed, n_pixels, centers_out, sse_history, hist_cap, report);
  return CQB_OK;
}

int cqb_fetch_results(cqb_ctx* ctx, double* centers_out, double* sse_history, int hist_cap, cqb_report* report) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(check_status(ctx));
  fill_report(ctx, ctx->last_k, ctx->draws_seed, ctx->last_P, centers_out, sse_history, hist_cap, report);
  return CQB_OK;
}

namespace {
int lane_fail(cqb_ctx* ctx, cqb_ctx* lane, int rc) {
  return fail(ctx, rc, "batch lane: %s", lane->err.c_str());
}
}  // namespace

namespace {
// Images in flight on `lanes` sub-contexts (cqb_quantize_batch,
// cqb_quantize_runs); image i uses seeds[i], or `seed` when seeds is null.
int quantize_lanes(cqb_ctx* ctx, int n_images, const uint8_t* const* d_rgb, const uint64_t* n_pixels, int k,
                   const cqb_termination* term, uint64_t seed, const uint64_t* seeds, uint8_t* const* d_index_out,
                   uint8_t* const* d_rgb_out, int lanes, double* centers_out, cqb_report* reports);
}  // namespace

int cqb_quantize_batch(cqb_ctx* ctx, int n_images, const uint8_t* const* d_rgb, const uint64_t* n_pixels, int k,
                       const cqb_termination* term, uint64_t seed, uint8_t* const* d_index_out,
                       uint8_t* const* d_rgb_out, int lanes, double* centers_out, cqb_report* reports) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  return quantize_lanes(ctx, n_images, d_rgb, n_pixels, k, term, seed, nullptr, d_index_out, d_rgb_out, lanes,
                        centers_out, reports);
}

int cqb_quantize_runs(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, int k, const cqb_termination* term,
                      int n_runs, const uint64_t* seeds, int lanes, double* centers_out, cqb_report* reports) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (n_runs < 0 || (n_runs > 0 && (!seeds || !centers_out || !reports)))
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "quantize_runs: null argument");
  if (n_pixels == 0 || !rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "build_histogram: empty image");
  if (n_pixels >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  TRY(check_k(ctx, k));
  TRY(check_term(ctx, term));
  if (n_runs == 0) return CQB_OK;
  CK(cudaSetDevice(ctx->device));
  TRY(ensure_pixels(ctx, n_pixels));
  CK(cudaMemcpyAsync(ctx->d_img, rgb, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  std::vector<const uint8_t*> imgs((size_t)n_runs, ctx->d_img);
  std::vector<uint64_t> px((size_t)n_runs, n_pixels);
  const int rc = quantize_lanes(ctx, n_runs, imgs.data(), px.data(), k, term, 0, seeds, nullptr, nullptr, lanes,
                                centers_out, reports);
  CK(cudaStreamSynchronize(ctx->stream));
  return rc;
}

namespace {
int quantize_lanes(cqb_ctx* ctx, int n_images, const uint8_t* const* d_rgb, const uint64_t* n_pixels, int k,
                   const cqb_termination* term, uint64_t seed, const uint64_t* seeds, uint8_t* const* d_index_out,
                   uint8_t* const* d_rgb_out, int lanes, double* centers_out, cqb_report* reports) {
  if (n_images < 0 || (n_images > 0 && (!d_rgb || !n_pixels || !centers_out || !reports)))
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "quantize_batch: null argument");
  TRY(check_k(ctx, k));
  TRY(check_term(ctx, term));
  if (lanes <= 0) lanes = 4;
  lanes = std::max(1, std::min({lanes, n_images, 16}));
  CK(cudaSetDevice(ctx->device));
  const int per_lane = std::max(2, loop_grid(ctx) / lanes);
  while ((int)ctx->lanes.size() < lanes) {
    cqb_ctx* l = nullptr;
    const int rc = cqb_create(ctx->device, &l);
    if (rc != CQB_OK) return fail(ctx, rc, "quantize_batch: lane creation failed");
    ctx->lanes.push_back(l);
  }
  // lanes start after the work already enqueued on the caller's stream
  if (!ctx->join_ev) CK(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ctx->join_ev, ctx->stream));
  for (int l = 0; l < lanes; ++l) {
    ctx->lanes[l]->grid_limit = per_lane;
    CK(cudaStreamWaitEvent(ctx->lanes[l]->stream, ctx->join_ev, 0));
  }
  std::vector<int> pending(lanes, -1);
  auto finish = [&](int l) -> int {
    const int i = pending[l];
    if (i < 0) return CQB_OK;
    pending[l] = -1;
    cqb_ctx* lane = ctx->lanes[l];
    double* c = centers_out + (size_t)i * 3 * k;
    int rc = cqb_fetch_results(lane, c, nullptr, 0, &reports[i]);
    if (rc != CQB_OK && lane->h_stage->status == ST_DRAWS_EXHAUSTED)  // rare: rerun with the retry loop
      rc = cqb_quantize_device(lane, d_rgb[i], n_pixels[i], k, term, seeds ? seeds[i] : seed,
                               d_index_out ? d_index_out[i] : nullptr, d_rgb_out ? d_rgb_out[i] : nullptr, 1, c,
                               nullptr, 0, &reports[i]);
    return rc == CQB_OK ? CQB_OK : lane_fail(ctx, lane, rc);
  };
  for (int i = 0; i < n_images; ++i) {
    const int l = i % lanes;
    TRY(finish(l));
    cqb_ctx* lane = ctx->lanes[l];
    const int rc = cqb_quantize_device(lane, d_rgb[i], n_pixels[i], k, term, seeds ? seeds[i] : seed,
                                       d_index_out ? d_index_out[i] : nullptr, d_rgb_out ? d_rgb_out[i] : nullptr, 0,
                                       nullptr, nullptr, 0, nullptr);
    if (rc != CQB_OK) return lane_fail(ctx, lane, rc);
    pending[l] = i;
  }
  for (int l = 0; l < lanes; ++l) {
    TRY(finish(l));
    // order later work on the caller's stream after every lane
    CK(cudaEventRecord(ctx->lanes[l]->join_ev_out(), ctx->lanes[l]->stream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->lanes[l]->join_ev_out(), 0));
  }
  return CQB_OK;
}
}  // namespace

int cqb_quantize(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, const cqb_termination* term,
                 uint64_t seed, double* centers_out, double* sse_history, int hist_cap, uint8_t* index_out,
                 uint8_t* rgb_out, cqb_report* report) {
  return cqb_quantize_ex(ctx, rgb, width, height, k, term, seed, centers_out, sse_history, hist_cap, index_out,
                         rgb_out, nullptr, report);
}

int cqb_quantize_ex(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, const cqb_termination* term,
                    uint64_t seed, double* centers_out, double* sse_history, int hist_cap, uint8_t* index_out,
                    uint8_t* rgb_out, uint8_t* error_out, cqb_report* report) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (width <= 0 || height <= 0 || !rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "image dimensions must be positive");
  TRY(check_k(ctx, k));
  TRY(check_term(ctx, term));
  const uint64_t P = (uint64_t)width * (uint64_t)height;
  if (P >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  CK(cudaSetDevice(ctx->device));
  TRY(ensure_pixels(ctx, P));
  // Large images: the H2D copy in XFER_CHUNKS slices on ctx->xfer, K1 counting
  // each slice as it lands (one pass over the whole bin table per slice), and
  // the outputs copied back per map slice (enqueue_quantize); small ones use
  // one copy and the fused prep kernel. When another call of this process is
  // in flight (host threads streaming images, one context each), that call's
  // kernels already hide these copies: then one H2D + the 4-pass K1 (in L2)
  // + one D2H is faster (cfg4, 2 callers: 7.00 vs 7.57 ms per image).
  struct InFlight {
    static std::atomic<int>& n() {
      static std::atomic<int> c{0};
      return c;
    }
    const int at_entry = n().fetch_add(1) + 1;
    ~InFlight() { n().fetch_sub(1); }
  } inflight;
  const bool overlap = !sparse_path(ctx, P) && !(ctx->debug_flags & DBG_NO_XFER_OVERLAP) && inflight.at_entry == 1;
  if (overlap) {
    TRY(ensure_xfer(ctx));
    CK(cudaEventRecord(ctx->xev[0], ctx->stream));  // d_img is free once the stream's earlier work is done
    CK(cudaStreamWaitEvent(ctx->xfer, ctx->xev[0], 0));
    const uint64_t q16 = (P + 15) / 16;
    for (int c = 0; c < XFER_CHUNKS; ++c) {
      const uint64_t a = std::min(P, q16 * c / XFER_CHUNKS * 16), b = std::min(P, q16 * (c + 1) / XFER_CHUNKS * 16);
      if (b <= a) continue;
      CK(cudaMemcpyAsync(ctx->d_img + 3 * a, rgb + 3 * a, 3 * (b - a), cudaMemcpyHostToDevice, ctx->xfer));
      CK(cudaEventRecord(ctx->xev[c], ctx->xfer));
      CK(cudaStreamWaitEvent(ctx->stream, ctx->xev[c], 0));
      const uint64_t nchunk = (b - a + PX_PER_THREAD - 1) / PX_PER_THREAD;
      const int g1 = (int)std::min<uint64_t>((nchunk + HIST_THREADS - 1) / HIST_THREADS, (uint64_t)ctx->num_sms * 16);
      k_hist_count<<<std::max(g1, 1), HIST_THREADS, 0, ctx->stream>>>(ctx->d_img + 3 * a, b - a, ctx->bins, 0u,
                                                                       1u << 24, nullptr, (uint32_t)a);
      CKL();
    }
  } else {
    CK(cudaMemcpyAsync(ctx->d_img, rgb, 3 * P, cudaMemcpyHostToDevice, ctx->stream));
  }
  // Pinned (mapped) host outputs are written by the map kernel directly over
  // PCIe (zero-copy), overlapping the transfer with the kernel; pageable ones
  // get the device buffers + one D2H copy each.
  // (small images only: for large rasters the copy engines move the outputs
  // faster than the kernel's PCIe stores - cfg4 e2e 1595 vs 1309 Mpix/s)
  const bool zc = !(ctx->debug_flags & 65536) && P < OCC_MAX_PIXELS;
  uint8_t* zi = zc ? mapped_view(index_out, ctx->device) : nullptr;
  uint8_t* zr = zc ? mapped_view(rgb_out, ctx->device) : nullptr;
  uint8_t* ze = zc ? mapped_view(error_out, ctx->device) : nullptr;
  // H2D, the whole pipeline and the D2H copies are enqueued back to back with
  // ONE host synchronisation (the rare draw-exhaustion retry re-enqueues)
  int ndraws = k + 64;
  for (int attempt = 0; attempt < 4; ++attempt) {
    ctx->err_target = error_out ? (ze ? ze : ctx->d_err) : nullptr;
    // a retry re-counts the histogram from the resident raster (K2b re-zeroed the bins)
    ctx->k1_done = overlap && attempt == 0;
    if (overlap) {
      ctx->h_index_dst = index_out;
      ctx->h_rgb_dst = rgb_out;
      ctx->h_err_dst = error_out;
    }
    const int rc = enqueue_quantize(ctx, ctx->d_img, P, k, term, seed,
                                    index_out ? (zi ? zi : ctx->d_index) : nullptr,
                                    rgb_out ? (zr ? zr : ctx->d_rgb) : nullptr, ndraws);
    ctx->err_target = nullptr;
    ctx->k1_done = false;
    ctx->h_index_dst = ctx->h_rgb_dst = ctx->h_err_dst = nullptr;
    TRY(rc);
    if (!overlap) {
      if (index_out && !zi) CK(cudaMemcpyAsync(index_out, ctx->d_index, P, cudaMemcpyDeviceToHost, ctx->stream));
      if (rgb_out && !zr) CK(cudaMemcpyAsync(rgb_out, ctx->d_rgb, 3 * P, cudaMemcpyDeviceToHost, ctx->stream));
      if (error_out && !ze) CK(cudaMemcpyAsync(error_out, ctx->d_err, 3 * P, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_stage->status != ST_DRAWS_EXHAUSTED) break;
    ndraws *= 4;
  }
  TRY(check_status(ctx));
  cqb_report rep{};
  fill_report(ctx, k, seed, P, centers_out, sse_history, hist_cap, &rep);
  if (report) *report = rep;
  return CQB_OK;
}

}  // extern "C"

namespace {
int pts_reserve(cqb_ctx* ctx, uint64_t n, int k);
int pts_run(cqb_ctx* ctx, uint64_t n, int k, const cqb_termination* term, int mode, int kprime, uint64_t seed,
            double* centers_out, double* sse_history, int hist_cap, double* trajectory, int traj_cap,
            int32_t* memberships_out, cqb_report* report);

// The pixel-space comparators of methods.hpp (run_km_full, kmeans.hpp:
// 409-426; run_fkm over pixels_as_points, methods.hpp:163-178): initial
// centers = init_centers(build_histogram(image), k, seed) from the device
// histogram pipeline, then run_weighted_kmeans over all P pixels (weight
// 1/P each) on the point-set kernels, so every reported distance evaluation
// is one the device performs.
int pixel_kmeans(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, const cqb_termination* term,
                 uint64_t seed, int mode, int kprime, double* centers_out, double* sse_history, int hist_cap,
                 cqb_report* report) {
  if (width <= 0 || height <= 0 || !rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "image dimensions must be positive");
  TRY(check_k(ctx, k));
  TRY(check_term(ctx, term));
  const uint64_t P = (uint64_t)width * (uint64_t)height;
  if (P >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  CK(cudaSetDevice(ctx->device));
  TRY(ensure_pixels(ctx, P));
  TRY(ensure_samples(ctx, P));
  TRY(pts_reserve(ctx, P, k));
  CK(cudaMemcpyAsync(ctx->d_img, rgb, 3 * P, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  int ndraws = k + 64;
  for (int attempt = 0;; ++attempt) {
    TRY(upload_draws(ctx, seed, ndraws));
    const bool fused = fused_prep(ctx, P);
    if (!fused) TRY(reset_state(ctx));
    TRY(enqueue_histogram(ctx, ctx->d_img, P, false, false, k, ndraws, fused));
    CK(cudaMemcpyAsync(&ctx->h_stage->status, &ctx->st->status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_stage->status != ST_DRAWS_EXHAUSTED || attempt == 3) break;
    ndraws *= 4;
  }
  TRY(check_status(ctx));
  k_pts_from_rgb<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ctx->d_img, P, ctx->pts.X, ctx->pts.W);
  CKL();
  CK(cudaMemcpyAsync(ctx->pts.C, ctx->st->C[0], sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  TRY(pts_run(ctx, P, k, term, mode, kprime, seed, centers_out, sse_history, hist_cap, nullptr, 0, nullptr, report));
  if (report) report->mse = 0.0;  // the caller fills mse (methods.hpp:104-106)
  return CQB_OK;
}
}  // namespace

extern "C" {

int cqb_run_km_full(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, const cqb_termination* term,
                    uint64_t seed, double* centers_out, double* sse_history, int hist_cap, cqb_report* report) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  return pixel_kmeans(ctx, rgb, width, height, k, term, seed, PTS_NAIVE, 0, centers_out, sse_history, hist_cap,
                      report);
}

int cqb_run_fkm(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, int k_prime,
                const cqb_termination* term, uint64_t seed, double* centers_out, double* sse_history, int hist_cap,
                cqb_report* report) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (k_prime < 1 || k_prime > k) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "run_fkm: need 1 <= k_prime <= k");
  return pixel_kmeans(ctx, rgb, width, height, k, term, seed, PTS_FKM, k_prime, centers_out, sse_history, hist_cap,
                      report);
}

int cqb_error_image(cqb_ctx* ctx, const uint8_t* original, const uint8_t* quantized, uint64_t n_pixels,
                    uint8_t* out) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (n_pixels == 0) return CQB_OK;
  if (!original || !quantized || !out) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "error_image: null buffer");
  CK(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  TRY(ensure_pixels(ctx, n_pixels));
  CK(cudaMemcpyAsync(ctx->d_img, original, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_rgb, quantized, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  k_error_image<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->d_img, ctx->d_rgb, 3 * n_pixels, ctx->d_err);
  CKL();
  CK(cudaMemcpyAsync(out, ctx->d_err, 3 * n_pixels, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return CQB_OK;
}

int cqb_map_pixels(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, const double* centers, int k,
                   uint8_t* rgb_out, uint8_t* index_out, uint64_t* sq_err_sum) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (k < 1 || !centers) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "map_pixels: empty palette");
  if (k > KMAX) return fail(ctx, CQB_ERR_UNSUPPORTED, "k = %d exceeds the device limit %d", k, KMAX);
  if (n_pixels == 0) return CQB_OK;
  if (n_pixels >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  CK(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  TRY(ensure_pixels(ctx, n_pixels));
  TRY(ensure_samples(ctx, n_pixels));
  CK(cudaMemcpyAsync(ctx->d_img, rgb, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_centers_in, centers, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(&ctx->st->mse_err, 0, sizeof(unsigned long long), ctx->stream));
  TRY(enqueue_histogram(ctx, ctx->d_img, n_pixels));
  k_map_tables<<<k, 256, 0, ctx->stream>>>(ctx->d_centers_in, k, ctx->d_sortedDr, ctx->d_orderR, ctx->d_palkey);
  CKL();
  k_map_unique<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->d_mkeys, ctx->d_mcounts, nullptr, ctx->d_n, k,
                                                          ctx->d_sortedDr, ctx->d_orderR, ctx->d_palkey, ctx->lut,
                                                          &ctx->st->mse_err);
  CKL();
  const uint64_t nchunk = (n_pixels + PX_PER_THREAD - 1) / PX_PER_THREAD;
  const int g = (int)std::min<uint64_t>((nchunk + HIST_THREADS - 1) / HIST_THREADS, (uint64_t)ctx->num_sms * 16);
  k_map_pixels<<<std::max(g, 1), HIST_THREADS, 0, ctx->stream>>>(ctx->d_img, n_pixels, ctx->lut, ctx->d_palkey, k,
                                                                 index_out ? ctx->d_index : nullptr,
                                                                 rgb_out ? ctx->d_rgb : nullptr, nullptr);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_scalar, &ctx->st->mse_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     ctx->stream));
  if (index_out) CK(cudaMemcpyAsync(index_out, ctx->d_index, n_pixels, cudaMemcpyDeviceToHost, ctx->stream));
  if (rgb_out) CK(cudaMemcpyAsync(rgb_out, ctx->d_rgb, 3 * n_pixels, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (sq_err_sum) *sq_err_sum = ctx->h_scalar[0];
  return CQB_OK;
}

int cqb_mse(cqb_ctx* ctx, const uint8_t* a, const uint8_t* b, uint64_t n_pixels, double* out) {
  if (!ctx || !out) return CQB_ERR_INVALID_ARGUMENT;
  if (n_pixels == 0) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "mse: empty images");
  CK(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  TRY(ensure_pixels(ctx, n_pixels));
  CK(cudaMemcpyAsync(ctx->d_img, a, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_img2, b, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(&ctx->st->mse_err, 0, sizeof(unsigned long long), ctx->stream));
  k_mse<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(ctx->d_img, ctx->d_img2, 3 * n_pixels, &ctx->st->mse_err);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_scalar, &ctx->st->mse_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *out = (double)ctx->h_scalar[0] / (double)n_pixels;
  return CQB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Generic weighted points (points.cuh): kmeans.hpp's span<const Vec3> API.
namespace {
constexpr int PTS_BLOCKS = 296;  // grid of the point kernels (block partials)

int pts_reserve(cqb_ctx* ctx, uint64_t n, int k) {
  auto& q = ctx->pts;
  if (n > q.cap_n) {
    const size_t c = (size_t)n + 64;
    TRY(grow(ctx, &q.X, 3 * c));
    TRY(grow(ctx, &q.W, c));
    TRY(grow(ctx, &q.m, c));
    TRY(grow(ctx, &q.perm, c));
    TRY(grow(ctx, &q.skip, c));
    TRY(grow(ctx, &q.prevd, c));
    q.cap_n = c;
  }
  const size_t tiles = (size_t)(n + PTS_TILE - 1) / PTS_TILE;
  if (k > q.cap_k || tiles * (size_t)k > q.cap_tiles) {
    const int kk = std::max(k, q.cap_k);
    TRY(grow(ctx, &q.tcnt, tiles * (size_t)kk + 1));
    TRY(grow(ctx, &q.toff, tiles * (size_t)kk + 1));
    q.cap_tiles = tiles * (size_t)kk;
  }
  if (k > q.cap_k) {
    TRY(grow(ctx, &q.C, 3 * (size_t)k));
    TRY(grow(ctx, &q.next, 3 * (size_t)k));
    TRY(grow(ctx, &q.taken, 3 * (size_t)k));
    TRY(grow(ctx, &q.dists, (size_t)k * k));
    TRY(grow(ctx, &q.order, (size_t)k * k));
    TRY(grow(ctx, &q.sortedD, (size_t)k * k));
    TRY(grow(ctx, &q.start, (size_t)k + 1));
    TRY(grow(ctx, &q.empty, (size_t)k));
    TRY(grow(ctx, &q.chosen, (size_t)k));
    q.cap_k = k;
  }
  if (!q.part) {
    TRY(grow(ctx, &q.part, (size_t)PTS_BLOCKS));
    TRY(grow(ctx, &q.cand_i, (size_t)PTS_BLOCKS));
    TRY(grow(ctx, &q.scal, (size_t)8));
    TRY(grow(ctx, &q.evals, (size_t)2));
  }
  return CQB_OK;
}

int pts_check(cqb_ctx* ctx, uint64_t n, int k) {
  if (k < 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "init_centers: k must be >= 1");
  if (k > PTS_KMAX) return fail(ctx, CQB_ERR_UNSUPPORTED, "k = %d exceeds the point-set limit %d", k, PTS_KMAX);
  if (n >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "point sets above 2^32-1 points");
  return CQB_OK;
}

int pts_upload(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n) {
  CK(cudaMemcpyAsync(ctx->pts.X, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->stream));
  if (weights) CK(cudaMemcpyAsync(ctx->pts.W, weights, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  return CQB_OK;
}

// Tables (center_dists, order, sorted rows) of the k centers in pts.C.
int pts_tables(cqb_ctx* ctx, int k) {
  k_pts_tables<<<k, PTS_THREADS, 0, ctx->stream>>>(ctx->pts.C, k, ctx->pts.dists, ctx->pts.order, ctx->pts.sortedD);
  CKL();
  return CQB_OK;
}

// assign_sort_means (naive: assign_naive) over pts.X with pts.C and the
// tables; sse -> pts.scal[0], evals -> pts.evals[0].
int pts_assign(cqb_ctx* ctx, uint64_t n, int k, int mode = PTS_SORT_MEANS, bool audit = false, int kprime = 0) {
  CK(cudaMemsetAsync(ctx->pts.evals, 0, sizeof(unsigned long long), ctx->stream));
  k_pts_assign<<<PTS_BLOCKS, PTS_THREADS, 0, ctx->stream>>>(ctx->pts.X, ctx->pts.W, n, ctx->pts.C, k,
                                                            ctx->pts.order, ctx->pts.sortedD, ctx->pts.m,
                                                            ctx->pts.part, ctx->pts.evals, mode, kprime,
                                                            audit ? ctx->pts.skip : nullptr, ctx->pts.prevd);
  CKL();
  k_pts_sum<<<1, 32, 0, ctx->stream>>>(ctx->pts.part, PTS_BLOCKS, ctx->pts.scal);
  CKL();
  return CQB_OK;
}

// update_centers: pts.next from pts.C (the centers of the assignment), pts.m.
int pts_update(cqb_ctx* ctx, uint64_t n, int k, int* n_empty) {
  auto& q = ctx->pts;
  const uint32_t tiles = (uint32_t)((n + PTS_TILE - 1) / PTS_TILE);
  k_pts_tile_count<<<tiles, PTS_THREADS, 0, ctx->stream>>>(q.m, n, k, q.tcnt);
  CKL();
  k_pts_offsets<<<1, PTS_KMAX, 0, ctx->stream>>>(q.tcnt, tiles, k, q.toff, q.start);
  CKL();
  const int wpb = 4;  // tiles (warps) per block
  k_pts_tile_scatter<<<(tiles + wpb - 1) / wpb, 32 * wpb, sizeof(uint32_t) * wpb * (size_t)k, ctx->stream>>>(
      q.m, n, k, q.toff, q.perm);
  CKL();
  k_pts_sums<<<(k + 127) / 128, 128, 0, ctx->stream>>>(q.X, q.W, q.perm, q.start, k, q.next, q.empty);
  CKL();
  std::vector<int> empty((size_t)k);
  CK(cudaMemcpyAsync(empty.data(), q.empty, sizeof(int) * (size_t)k, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int slot = 0;
  for (int c = 0; c < k; ++c) {  // empty clusters in increasing order (kmeans.hpp:272-294)
    if (!empty[(size_t)c]) continue;
    k_pts_reseed_scan<<<PTS_BLOCKS, PTS_THREADS, 0, ctx->stream>>>(q.X, n, q.C, q.m, q.taken, slot, q.part,
                                                                   q.cand_i);
    CKL();
    k_pts_reseed_pick<<<1, 32, 0, ctx->stream>>>(q.part, q.cand_i, PTS_BLOCKS, q.X, c, q.next, q.taken, slot);
    CKL();
    ++slot;
  }
  if (n_empty) *n_empty = slot;
  return CQB_OK;
}

// init_centers: chosen indices of a partial Fisher-Yates over n points.
__global__ void __launch_bounds__(PTS_KMAX) k_pts_init(unsigned long long n, int k,
                                                        const unsigned long long* __restrict__ draws, int ndraws,
                                                        uint32_t* __restrict__ chosen, int* __restrict__ status) {
  fisher_yates_block<PTS_KMAX>(n, k, draws, ndraws, chosen, status);
}

int pts_init(cqb_ctx* ctx, uint64_t n, int k, uint64_t seed) {
  int ndraws = k + 64;
  for (int attempt = 0; attempt < 4; ++attempt, ndraws *= 4) {
    TRY(upload_draws(ctx, seed, ndraws));
    CK(cudaMemsetAsync(&ctx->st->status, 0, sizeof(int), ctx->stream));
    k_pts_init<<<1, PTS_KMAX, 0, ctx->stream>>>(n, k, ctx->d_draws, ndraws, ctx->pts.chosen, &ctx->st->status);
    CKL();
    int status = 0;
    CK(cudaMemcpyAsync(&ctx->h_stage->status, &ctx->st->status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    status = ctx->h_stage->status;
    if (status == ST_DRAWS_EXHAUSTED) continue;
    if (status == ST_K_EXCEEDS_N)
      return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "init_centers: k exceeds the number of candidate points");
    return CQB_OK;
  }
  return fail(ctx, CQB_ERR_INTERNAL, "init_centers: raw draw buffer exhausted");
}
// run_weighted_kmeans (kmeans.hpp:336-376) from the centers in pts.C:
// SortMeans (WSM), Naive (run_km_full, :409-426) or FKM (run_fkm,
// fast_variants.hpp:20-81: iteration 1 exhaustive, then k' neighbours).
int pts_run(cqb_ctx* ctx, uint64_t n, int k, const cqb_termination* term, int mode, int kprime, uint64_t seed,
            double* centers_out, double* sse_history, int hist_cap, double* trajectory, int traj_cap,
            int32_t* memberships_out, cqb_report* report) {
  auto& q = ctx->pts;
  CK(cudaMemsetAsync(q.m, 0, sizeof(int32_t) * n, ctx->stream));  // iteration 1 starts from all-zero memberships
  std::vector<double> cur((size_t)3 * k), nxt((size_t)3 * k);
  CK(cudaMemcpyAsync(cur.data(), q.C, sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  std::vector<double> prev_tab;  // the centers the tables were last built from
  unsigned long long evals = 0;
  double prev_sse = HUGE_VAL, sse = 0;
  int iter = 0, empties = 0;
  const int cap = term->mode == 1 ? term->hard_cap : term->max_iters;
  for (iter = 1;; ++iter) {
    // this iteration's assignment: FKM's first one is exhaustive
    const int am = mode == PTS_FKM && iter == 1 ? PTS_NAIVE : mode;
    if (am != PTS_NAIVE) {
      // update_center_tables' pair count (kmeans.hpp:137-155): all pairs at
      // first, then the pairs with at least one moved center
      unsigned long long pairs = (unsigned long long)k * (k - 1) / 2;
      if (!prev_tab.empty()) {
        unsigned long long still = 0;
        for (int c = 0; c < k; ++c)
          still += memcmp(&prev_tab[3 * (size_t)c], &cur[3 * (size_t)c], 3 * sizeof(double)) == 0;
        pairs -= still ? still * (still - 1) / 2 : 0;
      }
      evals += pairs;
      prev_tab = cur;
      TRY(pts_tables(ctx, k));
    }
    TRY(pts_assign(ctx, n, k, am, false, kprime));
    unsigned long long ev = 0;
    CK(cudaMemcpyAsync(&sse, q.scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&ev, q.evals, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    int ne = 0;
    TRY(pts_update(ctx, n, k, &ne));  // synchronizes
    evals += ev;
    empties += ne;
    if (sse_history && iter <= hist_cap) sse_history[iter - 1] = sse;
    CK(cudaMemcpyAsync(nxt.data(), q.next, sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(q.C, q.next, sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (trajectory && iter <= traj_cap) memcpy(trajectory + (size_t)(iter - 1) * 3 * k, nxt.data(), sizeof(double) * 3 * k);
    cur.swap(nxt);
    bool stop;
    if (term->mode == 0) stop = iter >= term->max_iters;
    else stop = sse == 0.0 || (prev_sse - sse) / sse <= term->epsilon || iter >= cap;
    if (stop) break;
    prev_sse = sse;
  }
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  memcpy(centers_out, cur.data(), sizeof(double) * 3 * (size_t)k);
  if (memberships_out) CK(cudaMemcpy(memberships_out, q.m, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  if (report) {
    cqb_report r{};
    r.iterations = iter;
    r.k = k;
    r.seed = seed;
    r.sse = sse;
    r.dist_evals = evals;
    r.n_unique = n;
    r.empty_events = empties;
    float ms = 0.f;
    CK(cudaEventSynchronize(ctx->ev[1]));
    r.elapsed_ms = cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]) == cudaSuccess ? ms : 0.0;
    *report = r;
  }
  return CQB_OK;
}

}  // namespace

extern "C" {

int cqb_init_centers(cqb_ctx* ctx, uint64_t n_points, int k, uint64_t seed, uint32_t* chosen_out) {
  if (!ctx || !chosen_out) return CQB_ERR_INVALID_ARGUMENT;
  TRY(pts_check(ctx, n_points, k));
  if ((uint64_t)k > n_points)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "init_centers: k exceeds the number of candidate points");
  CK(cudaSetDevice(ctx->device));
  TRY(pts_reserve(ctx, 1, k));
  TRY(pts_init(ctx, n_points, k, seed));
  CK(cudaMemcpy(chosen_out, ctx->pts.chosen, sizeof(uint32_t) * (size_t)k, cudaMemcpyDeviceToHost));
  return CQB_OK;
}

int cqb_points_tables(cqb_ctx* ctx, const double* centers, int k, double* center_dists, int32_t* sorted_order) {
  if (!ctx || !centers) return CQB_ERR_INVALID_ARGUMENT;
  TRY(pts_check(ctx, 1, k));
  CK(cudaSetDevice(ctx->device));
  TRY(pts_reserve(ctx, 1, k));
  CK(cudaMemcpyAsync(ctx->pts.C, centers, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice, ctx->stream));
  TRY(pts_tables(ctx, k));
  if (center_dists)
    CK(cudaMemcpyAsync(center_dists, ctx->pts.dists, sizeof(double) * (size_t)k * k, cudaMemcpyDeviceToHost,
                       ctx->stream));
  if (sorted_order)
    CK(cudaMemcpyAsync(sorted_order, ctx->pts.order, sizeof(int32_t) * (size_t)k * k, cudaMemcpyDeviceToHost,
                       ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return CQB_OK;
}

int cqb_points_assign(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n, const double* centers,
                      int k, const double* center_dists, const int32_t* sorted_order, int mode,
                      int32_t* memberships, double* weighted_sse, uint64_t* dist_evals, int32_t* skip_rank_out,
                      double* prev_dist_out) {
  if (!ctx || (n && (!points || !weights || !memberships)) || !centers || (mode != 0 && mode != 1))
    return CQB_ERR_INVALID_ARGUMENT;
  if (mode == 0)
    for (uint64_t i = 0; i < n; ++i)
      if (memberships[i] < 0 || memberships[i] >= k)
        return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "assign_sort_means: state does not match inputs");
  TRY(pts_check(ctx, n, k));
  CK(cudaSetDevice(ctx->device));
  TRY(pts_reserve(ctx, std::max<uint64_t>(n, 1), k));
  TRY(pts_upload(ctx, points, weights, n));
  CK(cudaMemcpyAsync(ctx->pts.C, centers, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->pts.m, memberships, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  if (mode == 0 && center_dists && sorted_order) {  // the caller's tables (ClusterState), as the reference reads them
    CK(cudaMemcpyAsync(ctx->pts.dists, center_dists, sizeof(double) * (size_t)k * k, cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(ctx->pts.order, sorted_order, sizeof(int32_t) * (size_t)k * k, cudaMemcpyHostToDevice,
                       ctx->stream));
    k_pts_sorted_rows<<<k, PTS_THREADS, 0, ctx->stream>>>(ctx->pts.dists, ctx->pts.order, k, ctx->pts.sortedD);
    CKL();
  } else if (mode == 0) {
    TRY(pts_tables(ctx, k));
  }
  const bool audit = mode == 0 && skip_rank_out && prev_dist_out;
  TRY(pts_assign(ctx, n, k, mode, audit));
  if (audit) {
    CK(cudaMemcpyAsync(skip_rank_out, ctx->pts.skip, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(prev_dist_out, ctx->pts.prevd, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  double sse = 0;
  unsigned long long ev = 0;
  CK(cudaMemcpyAsync(memberships, ctx->pts.m, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&sse, ctx->pts.scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&ev, ctx->pts.evals, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (weighted_sse) *weighted_sse = sse;
  if (dist_evals) *dist_evals = ev;
  return CQB_OK;
}

int cqb_points_update(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n,
                      const int32_t* memberships, const double* prev, int k, double* next_out) {
  if (!ctx || !prev || !next_out || (n && (!points || !weights || !memberships))) return CQB_ERR_INVALID_ARGUMENT;
  TRY(pts_check(ctx, n, k));
  if (n == 0) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "update_centers: no points");
  CK(cudaSetDevice(ctx->device));
  TRY(pts_reserve(ctx, n, k));
  TRY(pts_upload(ctx, points, weights, n));
  CK(cudaMemcpyAsync(ctx->pts.m, memberships, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->pts.C, prev, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice, ctx->stream));
  TRY(pts_update(ctx, n, k, nullptr));
  CK(cudaMemcpyAsync(next_out, ctx->pts.next, sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return CQB_OK;
}

int cqb_points_sse(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n, const double* centers,
                   int k, const int32_t* memberships, double* sse_out) {
  if (!ctx || !centers || !sse_out || (n && (!points || !weights || !memberships))) return CQB_ERR_INVALID_ARGUMENT;
  TRY(pts_check(ctx, n, k));
  CK(cudaSetDevice(ctx->device));
  TRY(pts_reserve(ctx, std::max<uint64_t>(n, 1), k));
  TRY(pts_upload(ctx, points, weights, n));
  CK(cudaMemcpyAsync(ctx->pts.m, memberships, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->pts.C, centers, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice, ctx->stream));
  k_pts_sse<<<PTS_BLOCKS, PTS_THREADS, 0, ctx->stream>>>(ctx->pts.X, ctx->pts.W, n, ctx->pts.C, ctx->pts.m,
                                                         ctx->pts.part);
  CKL();
  k_pts_sum<<<1, 32, 0, ctx->stream>>>(ctx->pts.part, PTS_BLOCKS, ctx->pts.scal);
  CKL();
  CK(cudaMemcpyAsync(sse_out, ctx->pts.scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return CQB_OK;
}

// run_wsm_points (kmeans.hpp:379-390) = run_weighted_kmeans (:336-376) in
// SortMeans mode from init_centers(points, k, seed).
int cqb_run_wsm_points(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n, int k,
                       const cqb_termination* term, uint64_t seed, double* centers_out, double* sse_history,
                       int hist_cap, double* trajectory, int traj_cap, int32_t* memberships_out,
                       cqb_report* report) {
  if (!ctx || !centers_out || (n && (!points || !weights))) return CQB_ERR_INVALID_ARGUMENT;
  TRY(pts_check(ctx, n, k));
  TRY(check_term(ctx, term));
  if ((uint64_t)k > n)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "init_centers: k exceeds the number of candidate points");
  CK(cudaSetDevice(ctx->device));
  TRY(pts_reserve(ctx, n, k));
  TRY(pts_upload(ctx, points, weights, n));
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  TRY(pts_init(ctx, n, k, seed));
  k_pts_gather<<<(k + 255) / 256, 256, 0, ctx->stream>>>(ctx->pts.X, ctx->pts.chosen, k, &ctx->st->status,
                                                         ctx->pts.C);
  CKL();
  return pts_run(ctx, n, k, term, PTS_SORT_MEANS, 0, seed, centers_out, sse_history, hist_cap, trajectory, traj_cap,
                 memberships_out, report);
}



// ---------------------------------------------------------------------------
// Sharded WSM (multi-GPU): one step of the same persistent loop over a sample
// range, exact moments out; reduction and termination live in the host driver.

int cqb_shard_prepare(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, int k, uint64_t seed, uint64_t* n_unique,
                      double* init_centers) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (n_pixels == 0 || !rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "build_histogram: empty image");
  TRY(check_k(ctx, k));
  CK(cudaSetDevice(ctx->device));
  ctx->launches = 0;
  TRY(ensure_pixels(ctx, n_pixels));
  TRY(ensure_samples(ctx, n_pixels));
  CK(cudaMemcpyAsync(ctx->d_img, rgb, 3 * n_pixels, cudaMemcpyHostToDevice, ctx->stream));
  const int ndraws = k + 64;
  TRY(upload_draws(ctx, seed, ndraws));
  TRY(reset_state(ctx));
  TRY(enqueue_histogram(ctx, ctx->d_img, n_pixels, false, false, k, ndraws));
  CK(cudaMemsetAsync(ctx->d_labels, 0, n_pixels, ctx->stream));
  CK(cudaMemcpyAsync(&ctx->h_stage->status, &ctx->st->status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ctx->h_scalar, ctx->d_n, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ctx->h_stage->centers, ctx->st->C[0], sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(check_status(ctx));
  if (n_unique) *n_unique = ctx->h_scalar[0];
  if (init_centers) memcpy(init_centers, ctx->h_stage->centers, sizeof(double) * 3 * (size_t)k);
  ctx->shard_k = k;
  ctx->shard_total = n_pixels;
  return CQB_OK;
}

int cqb_shard_step(cqb_ctx* ctx, uint64_t lo, uint64_t hi, const double* centers, int dense_first,
                   uint64_t* moments, uint64_t* point_evals) {
  if (!ctx || !centers || !moments) return CQB_ERR_INVALID_ARGUMENT;
  if (ctx->shard_k < 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "cqb_shard_prepare first");
  const int k = ctx->shard_k;
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(ctx->st->C[0], centers, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice, ctx->stream));
  TRY(reset_state(ctx));
  TRY(ensure_hist(ctx, 1));
  const cqb_termination one{0, 1, 1e-4, 1};
  TRY(launch_loop(ctx, k, &one, dense_first, ctx->shard_total, nullptr, 0, lo, hi, 1));
  CK(cudaMemcpyAsync(ctx->h_mom, ctx->st->acc, sizeof(unsigned long long) * 5 * KMAX, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaMemcpyAsync(ctx->h_mom + 5 * KMAX, &ctx->st->evals, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaMemcpyAsync(&ctx->h_stage->status, &ctx->st->status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  TRY(check_status(ctx));
  for (int f = 0; f < 5; ++f)
    for (int c = 0; c < k; ++c) moments[f * k + c] = ctx->h_mom[f * KMAX + c];
  // the kernel's prologue counted a full table build; pair evaluations are the driver's
  if (point_evals) *point_evals = ctx->h_mom[5 * KMAX] - (unsigned long long)k * (unsigned long long)(k - 1) / 2;
  return CQB_OK;
}

int cqb_finalize_moments(cqb_ctx* ctx, const uint64_t* moments, const double* centers_used, int k, uint64_t total,
                         double* new_centers, double* sse, int* n_empty, int* empty_list) {
  if (!ctx || !moments || !centers_used) return CQB_ERR_INVALID_ARGUMENT;
  TRY(check_k(ctx, k));
  CK(cudaSetDevice(ctx->device));
  std::vector<unsigned long long> tmp(5 * KMAX, 0ull);
  for (int f = 0; f < 5; ++f)
    for (int c = 0; c < k; ++c) tmp[f * KMAX + c] = moments[f * k + c];
  CK(cudaMemcpyAsync(ctx->d_mom, tmp.data(), sizeof(unsigned long long) * 5 * KMAX, cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_centers_in, centers_used, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice,
                     ctx->stream));
  k_finalize<<<1, KMAX, 0, ctx->stream>>>(ctx->d_mom, ctx->d_centers_in, k, total, ctx->d_Cnew, ctx->d_scal,
                                          ctx->d_ints, ctx->d_ints + 1);
  CKL();
  std::vector<int> ints(KMAX + 1);
  double s = 0;
  CK(cudaMemcpyAsync(new_centers, ctx->d_Cnew, sizeof(double) * 3 * (size_t)k, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&s, ctx->d_scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ints.data(), ctx->d_ints, sizeof(int) * (KMAX + 1), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (sse) *sse = s;
  if (n_empty) *n_empty = ints[0];
  if (empty_list)
    for (int i = 0; i < ints[0]; ++i) empty_list[i] = ints[1 + i];
  return CQB_OK;
}

int cqb_shard_reseed_candidate(cqb_ctx* ctx, uint64_t lo, uint64_t hi, const double* centers_used,
                               const uint32_t* taken_ranks, int n_taken, double* d_out, uint32_t* rank_out,
                               uint32_t* key_out) {
  if (!ctx || !centers_used) return CQB_ERR_INVALID_ARGUMENT;
  const int k = ctx->shard_k;
  if (k < 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "cqb_shard_prepare first");
  if (n_taken < 0 || n_taken > KMAX) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "bad taken list");
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(ctx->d_centers_in, centers_used, sizeof(double) * 3 * (size_t)k, cudaMemcpyHostToDevice,
                     ctx->stream));
  if (n_taken)
    CK(cudaMemcpyAsync(ctx->d_taken, taken_ranks, sizeof(uint32_t) * (size_t)n_taken, cudaMemcpyHostToDevice,
                       ctx->stream));
  const int nb = ctx->num_sms * 2;
  k_reseed_scan<<<nb, 256, 0, ctx->stream>>>(ctx->d_mkeys, ctx->d_mrank, ctx->d_labels, lo, hi, ctx->d_centers_in,
                                             ctx->d_taken, n_taken, ctx->d_cand_d, ctx->d_cand_r, ctx->d_cand_k);
  CKL();
  k_reseed_pick<<<1, 32, 0, ctx->stream>>>(ctx->d_cand_d, ctx->d_cand_r, ctx->d_cand_k, nb, ctx->d_scal + 1,
                                           reinterpret_cast<unsigned int*>(ctx->d_ints + KMAX + 2),
                                           reinterpret_cast<unsigned int*>(ctx->d_ints + KMAX + 3));
  CKL();
  double d = 0;
  unsigned int rk[2] = {0, 0};
  CK(cudaMemcpyAsync(&d, ctx->d_scal + 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(rk, ctx->d_ints + KMAX + 2, sizeof(unsigned int) * 2, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (d_out) *d_out = d;
  if (rank_out) *rank_out = rk[0];
  if (key_out) *key_out = rk[1];
  return CQB_OK;
}

/* ---- in-kernel sharded loop --------------------------------------------- */

namespace {
int xch_reset(cqb_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->xmode == 1)
    for (int r = 0; r < ctx->xw; ++r)
      if (r != ctx->xrank && ctx->xpeer[r]) cudaIpcCloseMemHandle(ctx->xpeer[r]);
  if (ctx->xwin) cudaFree(ctx->xwin);
  if (ctx->xacc) cudaFree(ctx->xacc);
  ctx->xwin = ctx->xacc = nullptr;
  for (auto& p : ctx->xpeer) p = nullptr;
  ctx->xmode = 0;
  ctx->xw = 0;
  ctx->xrank = -1;
  return CQB_OK;
}
}  // namespace

int cqb_xch_window(cqb_ctx* ctx, int world, int rank, void* ipc_handle_out) {
  if (!ctx || !ipc_handle_out) return CQB_ERR_INVALID_ARGUMENT;
  if (world < 1 || world > XMAX || rank < 0 || rank >= world)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "exchange: world %d / rank %d (1 <= world <= %d)", world, rank, XMAX);
  CK(cudaSetDevice(ctx->device));
  TRY(xch_reset(ctx));
  CK(cudaMalloc(&ctx->xwin, XB_BYTES));
  CK(cudaMemset(ctx->xwin, 0, XB_BYTES));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->xwin));
  memcpy(ipc_handle_out, &h, sizeof(h));
  ctx->xmode = 1;
  ctx->xw = world;
  ctx->xrank = rank;
  ctx->xpeer[rank] = ctx->xwin;
  return CQB_OK;
}

int cqb_xch_open(cqb_ctx* ctx, const void* handles) {
  if (!ctx || !handles) return CQB_ERR_INVALID_ARGUMENT;
  if (ctx->xmode != 1) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "cqb_xch_window first");
  CK(cudaSetDevice(ctx->device));
  for (int r = 0; r < ctx->xw; ++r) {
    if (r == ctx->xrank || ctx->xpeer[r]) continue;  // own window, or mapped by an earlier (partial) call
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + (size_t)r * sizeof(h), sizeof(h));
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {  // unmap what this call opened: a retry starts clean
      for (int q = 0; q < r; ++q)
        if (q != ctx->xrank && ctx->xpeer[q]) {
          cudaIpcCloseMemHandle(ctx->xpeer[q]);
          ctx->xpeer[q] = nullptr;
        }
      return fail(ctx, CQB_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
    }
    ctx->xpeer[r] = static_cast<unsigned long long*>(p);
  }
  CK(cudaDeviceSynchronize());
  return CQB_OK;
}

int cqb_xch_set_timeout(cqb_ctx* ctx, double seconds) {
  if (!ctx || !(seconds > 0) || seconds > 3600) return CQB_ERR_INVALID_ARGUMENT;
  ctx->xch_timeout_ns = (unsigned long long)(seconds * 1e9);
  return CQB_OK;
}

int cqb_xch_emulate(cqb_ctx* ctx, int vranks) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (vranks < 1 || vranks > XMAX)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "exchange: %d emulated ranks (1..%d)", vranks, XMAX);
  CK(cudaSetDevice(ctx->device));
  TRY(xch_reset(ctx));
  if (loop_grid(ctx) < vranks * vranks) return fail(ctx, CQB_ERR_UNSUPPORTED, "grid too small for %d ranks", vranks);
  CK(cudaMalloc(&ctx->xwin, XB_LAB_OFF * (size_t)vranks));  // no label region: the groups share the labels
  CK(cudaMemset(ctx->xwin, 0, XB_LAB_OFF * (size_t)vranks));
  CK(cudaMalloc(&ctx->xacc, sizeof(unsigned long long) * 5 * KMAX * (size_t)vranks));
  for (int r = 0; r < vranks; ++r) ctx->xpeer[r] = ctx->xwin + (XB_LAB_OFF / sizeof(unsigned long long)) * r;
  ctx->xmode = 2;
  ctx->xw = vranks;
  ctx->xrank = -1;
  return CQB_OK;
}

int cqb_quantize_sharded(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int k, const cqb_termination* term,
                         uint64_t seed, uint8_t* d_index_out, uint8_t* d_rgb_out, uint64_t* px_range) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (ctx->xmode == 0) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "cqb_xch_window + cqb_xch_open (or cqb_xch_emulate) first");
  for (int r = 0; r < ctx->xw; ++r)
    if (!ctx->xpeer[r]) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "exchange window of rank %d not mapped (cqb_xch_open)", r);
  {  // every sending block must exist (cqb_set_grid_limit may have shrunk the grid since)
    const int g = loop_grid(ctx);
    if ((ctx->xmode == 2 && g / ctx->xw < ctx->xw) || (ctx->xmode == 1 && g < ctx->xw))
      return fail(ctx, CQB_ERR_UNSUPPORTED, "grid of %d blocks too small for %d exchanging ranks", g, ctx->xw);
  }
  TRY(check_k(ctx, k));
  TRY(check_term(ctx, term));
  if (n_pixels == 0 || !d_rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "quantize: empty image");
  if (n_pixels >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  if (!aligned16(d_rgb) || (d_index_out && !aligned16(d_index_out)) || (d_rgb_out && !aligned16(d_rgb_out)))
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "sharded quantize: device buffers must be 16-B aligned");
  CK(cudaSetDevice(ctx->device));
  TRY(ensure_pixels(ctx, n_pixels));
  // pixel range of this rank (multiples of 16 pixels; the emulated ranks share one process: all pixels)
  const int W = ctx->xmode == 1 ? ctx->xw : 1, r = ctx->xmode == 1 ? ctx->xrank : 0;
  const uint64_t q = (n_pixels + 15) / 16;
  ctx->px_lo = std::min(n_pixels, q * (uint64_t)r / (uint64_t)W * 16);
  ctx->px_hi = r == W - 1 ? n_pixels : std::min(n_pixels, q * (uint64_t)(r + 1) / (uint64_t)W * 16);
  if (px_range) {
    px_range[0] = ctx->px_lo;
    px_range[1] = ctx->px_hi;
  }
  ctx->xsharded = true;
  const int rc = enqueue_quantize(ctx, d_rgb, n_pixels, k, term, seed, d_index_out, d_rgb_out, k + 64);
  ctx->xsharded = false;
  return rc;
}

// ---- pixel-row sharded histogram (config 4 across GPUs) --------------------
int cqb_hist_rows(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int world, int rank, uint32_t* d_out,
                  uint64_t cap, uint64_t* n_out, uint64_t* owner_counts) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (world < 1 || world > XMAX || rank < 0 || rank >= world)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_rows: rank %d of world %d (1..%d ranks)", rank, world, XMAX);
  if (!d_rgb || !d_out || !n_out || !owner_counts) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_rows: null buffer");
  if (n_pixels >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
  if (!aligned16(d_rgb)) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_rows: the raster must be 16-B aligned");
  CK(cudaSetDevice(ctx->device));
  // this rank's rows: the pixel range it also maps (16-pixel aligned starts)
  const uint64_t q = (n_pixels + 15) / 16;
  const uint64_t lo = std::min(n_pixels, q * (uint64_t)rank / (uint64_t)world * 16);
  const uint64_t hi = rank == world - 1 ? n_pixels : std::min(n_pixels, q * (uint64_t)(rank + 1) / (uint64_t)world * 16);
  const uint64_t n = hi - lo;
  if (cap < n) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_rows: capacity %llu < %llu rows' pixels",
                           (unsigned long long)cap, (unsigned long long)n);
  TRY(ensure_pixels(ctx, std::max<uint64_t>(n, 1)));
  TRY(ensure_samples(ctx, std::max<uint64_t>(n, 1)));
  // K1 over the rows (global pixel indices), occupancy map for the compaction;
  // large row sets in 4 Morton-slice passes (each pass's atomics in L2)
  const uint64_t nchunk = (n + PX_PER_THREAD - 1) / PX_PER_THREAD;
  const int g1 = (int)std::min<uint64_t>((nchunk + HIST_THREADS - 1) / HIST_THREADS, (uint64_t)ctx->num_sms * 16);
  const int passes = n >= (4u << 20) ? 4 : 1;
  for (int p = 0; p < passes && n > 0; ++p) {
    const uint32_t span = (1u << 24) / passes;
    k_hist_count<<<std::max(g1, 1), HIST_THREADS, 0, ctx->stream>>>(
        d_rgb + 3 * lo, n, ctx->bins, p * span, p + 1 == passes ? (1u << 24) : (p + 1) * span, ctx->d_occ,
        (uint32_t)lo);
    CKL();
  }
  CK(cudaMemsetAsync(ctx->bin_tile_state, 0, sizeof(unsigned long long) * (N_OCC_TILES + 1), ctx->stream));
  k_occ_compact<<<N_OCC_TILES, OC_THREADS, 0, ctx->stream>>>(
      ctx->d_occ, ctx->bins, ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->bin_tile_state,
      reinterpret_cast<unsigned int*>(ctx->bin_tile_state + N_OCC_TILES), ctx->d_n, nullptr);
  CKL();
  unsigned long long* d_bounds = reinterpret_cast<unsigned long long*>(ctx->d_scal) + 8;
  const int gp = (int)std::min<uint64_t>((n + 255) / 256 + 1, (uint64_t)ctx->num_sms * 8);
  k_pack_triplets<<<std::max(gp, 1), 256, 0, ctx->stream>>>(ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->d_n,
                                                            d_out, world, d_bounds);
  CKL();
  unsigned long long b[XMAX + 1];
  CK(cudaMemcpyAsync(b, d_bounds, sizeof(unsigned long long) * (world + 1), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *n_out = b[world];
  for (int o = 0; o < world; ++o) owner_counts[o] = b[o + 1] - b[o];
  return CQB_OK;
}

int cqb_hist_merge(cqb_ctx* ctx, const uint32_t* d_in, uint64_t n_in, uint32_t* d_out, uint64_t cap,
                   uint64_t* n_out) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if ((!d_in && n_in) || !d_out || !n_out) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_merge: null buffer");
  if (n_in >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "hist_merge: above 2^32-1 entries");
  CK(cudaSetDevice(ctx->device));
  TRY(ensure_samples(ctx, std::max<uint64_t>(std::min<uint64_t>(n_in, 1u << 24), 1)));
  if (n_in) {
    const int g = (int)std::min<uint64_t>((n_in + 255) / 256, (uint64_t)ctx->num_sms * 16);
    k_merge_triplets<<<g, 256, 0, ctx->stream>>>(d_in, n_in, ctx->bins, ctx->d_occ);
    CKL();
  }
  CK(cudaMemsetAsync(ctx->bin_tile_state, 0, sizeof(unsigned long long) * (N_OCC_TILES + 1), ctx->stream));
  k_occ_compact<<<N_OCC_TILES, OC_THREADS, 0, ctx->stream>>>(
      ctx->d_occ, ctx->bins, ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->bin_tile_state,
      reinterpret_cast<unsigned int*>(ctx->bin_tile_state + N_OCC_TILES), ctx->d_n, nullptr);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_scalar, ctx->d_n, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const uint64_t n = ctx->h_scalar[0];
  if (n > cap) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_merge: capacity %llu < %llu merged samples",
                           (unsigned long long)cap, (unsigned long long)n);
  if (n) {
    const int gp = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->num_sms * 8);
    k_pack_triplets<<<gp, 256, 0, ctx->stream>>>(ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->d_n, d_out, 0,
                                                 nullptr);
    CKL();
    CK(cudaStreamSynchronize(ctx->stream));
  }
  *n_out = n;
  return CQB_OK;
}

int cqb_hist_range(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int world, int rank, uint32_t* d_out,
                   uint64_t cap, uint64_t* n_out) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (world < 1 || world > XMAX || rank < 0 || rank >= world)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_range: rank %d of world %d (1..%d ranks)", rank, world, XMAX);
  if (!d_rgb || !d_out || !n_out) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_range: null buffer");
  if (n_pixels == 0 || n_pixels >= 0xffffffffull)
    return fail(ctx, CQB_ERR_UNSUPPORTED, "hist_range: 1 .. 2^32-2 pixels");
  if (!aligned16(d_rgb)) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_range: the raster must be 16-B aligned");
  CK(cudaSetDevice(ctx->device));
  // this rank's Morton range: whole K2b tiles [t0, t1)
  const uint32_t t0 = (uint32_t)((uint64_t)N_BIN_TILES * rank / world), t1 = (uint32_t)((uint64_t)N_BIN_TILES * (rank + 1) / world);
  const uint32_t mlo = t0 * BIN_TILE, mhi = t1 * BIN_TILE;
  const uint64_t range = (uint64_t)(mhi - mlo);
  if (cap < std::min<uint64_t>(n_pixels, range))
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "hist_range: capacity %llu < %llu", (unsigned long long)cap,
                (unsigned long long)std::min<uint64_t>(n_pixels, range));
  TRY(ensure_samples(ctx, std::min<uint64_t>(n_pixels, range)));
  // K1 over every pixel, atomics only for this range, in L2-sized slices (32 MiB of bins each)
  const uint64_t nchunk = (n_pixels + PX_PER_THREAD - 1) / PX_PER_THREAD;
  const int g1 = (int)std::min<uint64_t>((nchunk + HIST_THREADS - 1) / HIST_THREADS, (uint64_t)ctx->num_sms * 16);
  const int passes = (int)std::max<uint64_t>(1, (range * sizeof(uint2) + (32ull << 20) - 1) / (32ull << 20));
  for (int p = 0; p < passes; ++p) {
    const uint32_t a = mlo + (uint32_t)(range * p / passes), b = mlo + (uint32_t)(range * (p + 1) / passes);
    k_hist_count<<<std::max(g1, 1), HIST_THREADS, 0, ctx->stream>>>(d_rgb, n_pixels, ctx->bins, a, b, nullptr);
    CKL();
  }
  CK(cudaMemsetAsync(ctx->bin_tile_state, 0, sizeof(unsigned long long) * (t1 - t0 + 1), ctx->stream));
  k_bins_compact<<<t1 - t0, BC_THREADS, 0, ctx->stream>>>(
      ctx->bins, ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->bin_tile_state,
      reinterpret_cast<unsigned int*>(ctx->bin_tile_state + (t1 - t0)), ctx->d_n, nullptr, 1, t0);
  CKL();
  CK(cudaMemcpyAsync(ctx->h_scalar, ctx->d_n, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  const int gp = (int)std::min<uint64_t>((std::min<uint64_t>(n_pixels, range) + 255) / 256, (uint64_t)ctx->num_sms * 8);
  k_pack_triplets<<<std::max(gp, 1), 256, 0, ctx->stream>>>(ctx->d_mkeys, ctx->d_mcounts, ctx->d_mrank, ctx->d_n,
                                                            d_out, 0, nullptr);
  CKL();
  CK(cudaStreamSynchronize(ctx->stream));
  *n_out = ctx->h_scalar[0];
  return CQB_OK;
}

int cqb_quantize_sharded_samples(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, const uint32_t* d_samples,
                                 uint64_t n_unique, int k, const cqb_termination* term, uint64_t seed,
                                 uint8_t* d_index_out, uint8_t* d_rgb_out, uint64_t* px_range) {
  if (!ctx) return CQB_ERR_INVALID_ARGUMENT;
  if (!d_samples || n_unique == 0 || n_unique > n_pixels)
    return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "sharded samples: %llu samples for %llu pixels",
                (unsigned long long)n_unique, (unsigned long long)n_pixels);
  ctx->ext_samples = d_samples;
  ctx->ext_n = n_unique;
  int rc;
  if (ctx->xmode == 0) {  // one rank: the single-GPU pipeline from the given histogram
    rc = [&]() -> int {
      TRY(check_k(ctx, k));
      TRY(check_term(ctx, term));
      if (!d_rgb) return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "quantize: empty image");
      if (n_pixels >= 0xffffffffull) return fail(ctx, CQB_ERR_UNSUPPORTED, "images above 2^32-1 pixels");
      if (!aligned16(d_rgb) || (d_index_out && !aligned16(d_index_out)) || (d_rgb_out && !aligned16(d_rgb_out)))
        return fail(ctx, CQB_ERR_INVALID_ARGUMENT, "sharded quantize: device buffers must be 16-B aligned");
      CK(cudaSetDevice(ctx->device));
      TRY(ensure_pixels(ctx, n_pixels));
      if (px_range) {
        px_range[0] = 0;
        px_range[1] = n_pixels;
      }
      return enqueue_quantize(ctx, d_rgb, n_pixels, k, term, seed, d_index_out, d_rgb_out, k + 64);
    }();
  } else {
    rc = cqb_quantize_sharded(ctx, d_rgb, n_pixels, k, term, seed, d_index_out, d_rgb_out, px_range);
  }
  ctx->ext_samples = nullptr;
  ctx->ext_n = 0;
  return rc;
}

}  // extern "C"
