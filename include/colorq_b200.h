/*
 * colorq_b200 — C ABI of the B200-native WSM color-quantization hot path.
 *
 * Plain pointers and sizes only (no CUDA or torch types in the signatures;
 * streams are passed as void*). Every entry point returns a status code
 * (CQB_OK = 0) and leaves a message retrievable with cqb_last_error().
 *
 * Each entry point replaces one reference function of the colorq C++ API
 * (/root/reference/proj/include/colorq, header-only C++20); the drop-in C++
 * shim with the reference's own signatures is include/colorq_b200/colorq.hpp.
 *
 * Threading: one cqb_ctx per host thread (the shim keeps a thread_local one);
 * a context owns its CUDA stream and device arena, so concurrent calls on
 * distinct contexts are safe (bench.hpp:187-223).
 */
#ifndef COLORQ_B200_H
#define COLORQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The shim maps INVALID_ARGUMENT to std::invalid_argument
 * (the reference's error type; CLI exit code 4) and the rest to
 * std::runtime_error. */
#define CQB_OK 0
#define CQB_ERR_INVALID_ARGUMENT 1
#define CQB_ERR_UNSUPPORTED 2
#define CQB_ERR_CUDA 3
#define CQB_ERR_OOM 4
#define CQB_ERR_NCCL 5
#define CQB_ERR_INTERNAL 6

#define CQB_MAX_K 256

typedef struct cqb_ctx cqb_ctx;

/* Termination — replaces colorq::Termination (kmeans.hpp:25-38).
 * mode 0 = FixedIterations(max_iters); mode 1 = Convergent(epsilon, hard_cap). */
typedef struct {
  int mode;
  int max_iters;
  double epsilon;
  int hard_cap;
} cqb_termination;

/* Run report — the fields of colorq::RunReport (report.hpp:33-53) the WSM
 * path fills, plus device-side extras. */
typedef struct {
  int iterations;       /* number of assignment passes (kmeans.hpp:358) */
  int k;
  uint64_t seed;
  double sse;           /* weighted SSE at the last assignment (kmeans.hpp:373) */
  double mse;           /* full-image MSE of the mapped result (quantize only) */
  double elapsed_ms;    /* palette generation, device time (methods.hpp:111,195) */
  double map_ms;        /* map + mse, device time */
  uint64_t dist_evals;  /* point + pair distance evaluations (kmeans.hpp:353,356) */
  uint64_t n_unique;    /* N' */
  int empty_events;     /* clusters re-seeded (kmeans.hpp:272-294) */
  int gpu_launches;     /* kernels this call launched */
} cqb_report;

/* ---- context ---------------------------------------------------------- */
int cqb_create(int device, cqb_ctx** out);
int cqb_destroy(cqb_ctx* ctx);
const char* cqb_last_error(const cqb_ctx* ctx);
/* Use an external CUDA stream (cudaStream_t as void*); NULL restores the
 * context's own stream. */
int cqb_set_stream(cqb_ctx* ctx, void* stream);
/* Cap the persistent WSM grid (0 = one full wave: 148 SMs x occupancy), for
 * running several images concurrently on one GPU (config 5). */
int cqb_set_grid_limit(cqb_ctx* ctx, int max_blocks);
int cqb_device_info(cqb_ctx* ctx, int* num_sms, int* loop_blocks);
/* Per-stage CUDA-event timing of cqb_quantize* (off by default). Stages:
 * [0] state reset, [1] K1 histogram count, [2] K2 compaction, [3] init,
 * [4] WSM loop (tables+assign+update, all iterations), [5] map tables +
 * unique-color map + MSE, [6] per-pixel map. */
int cqb_set_profiling(cqb_ctx* ctx, int on);
/* Diagnostics only: disables parts of the assign phase (results become
 * WRONG); used by tools/ablate.py to attribute time. 0 = normal. */
int cqb_set_debug(cqb_ctx* ctx, int flags);
int cqb_stage_times(cqb_ctx* ctx, float* ms, int n);
/* With profiling on: %globaltimer stamps (ns) of block 0 per WSM iteration,
 * 8 per iteration: assign start, rows staged, points done, deltas flushed,
 * barrier passed, finalize done, tables done, (reserved). */
int cqb_loop_timeline(cqb_ctx* ctx, unsigned long long* stamps, int n_iters);
/* With profiling on: per-block finish stamps of the assign phase for the
 * first 8 iterations, [iteration][block] (load-balance diagnostics). */
int cqb_block_times(cqb_ctx* ctx, unsigned long long* out, int n);

/* ---- histogram ---------------------------------------------------------
 * Replaces build_histogram(const RgbImage&) (histogram.hpp:65-99,105-108).
 * rgb: n_pixels x {r,g,b} host bytes, row-major. Outputs (host, capacity
 * `cap` entries, entries in FIRST-OCCURRENCE order): packed keys
 * r<<16|g<<8|b, counts, optional weights = count*(1/P), optional first pixel
 * index. *n_unique = N'. Empty image -> CQB_ERR_INVALID_ARGUMENT (:66). */
int cqb_build_histogram(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, uint32_t* keys, uint32_t* counts,
                        double* weights, uint32_t* first_index, uint64_t cap, uint64_t* n_unique);

/* ---- clustering --------------------------------------------------------
 * Replaces run_wsm(const ColorHistogram&, k, Termination, seed, trajectory*)
 * (kmeans.hpp:394-404): init_centers (:53-74) + the sort-means loop
 * (:336-376) over a histogram given as packed keys + counts (total = P).
 * centers_out: k x 3 doubles (post-update palette of the last iteration).
 * sse_history: hist_cap doubles (one per iteration). trajectory (nullable):
 * traj_cap x k x 3 doubles, the palette after every update (:361).
 * labels_out (nullable): final memberships, u8. k in [1, 256]; k > N' ->
 * CQB_ERR_INVALID_ARGUMENT (:54-56). */
int cqb_run_wsm(cqb_ctx* ctx, const uint32_t* keys, const uint32_t* counts, uint64_t n_unique, uint64_t total,
                int k, const cqb_termination* term, uint64_t seed, double* centers_out, double* sse_history,
                int hist_cap, double* trajectory, int traj_cap, uint8_t* labels_out, cqb_report* report);

/* Teacher-forced iteration hook (parity tests): from the given centers and
 * memberships run `term` iterations of the same device loop (tables ->
 * assign_sort_means -> update_centers). dense_first = 1 only for the
 * reference's bootstrap pass (labels all 0, integer centers). Replaces one
 * update_center_tables + assign_sort_means + update_centers
 * (kmeans.hpp:132-296). labels_inout: u8 memberships in/out. */
int cqb_wsm_iterate(cqb_ctx* ctx, const uint32_t* keys, const uint32_t* counts, uint64_t n_unique, uint64_t total,
                    int k, const double* centers_in, uint8_t* labels_inout, int dense_first,
                    const cqb_termination* term, double* centers_out, double* sse_history, int hist_cap,
                    cqb_report* report);

/* ---- end to end --------------------------------------------------------
 * generate_palette's WSM / WSM-C branch (methods.hpp:182-189) + map_pixels
 * (image_ops.hpp:18-51) + mse (metrics.hpp:18-29) in one device pass.
 * rgb: width*height pixels (host). index_out (nullable): u8 palette index
 * per pixel (new output; the reference has none). rgb_out (nullable): the
 * mapped image. report->mse is filled. */
int cqb_quantize(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, const cqb_termination* term,
                 uint64_t seed, double* centers_out, double* sse_history, int hist_cap, uint8_t* index_out,
                 uint8_t* rgb_out, cqb_report* report);
/* cqb_quantize plus error_out (nullable): error_image(image, mapped)
 * (image_ops.hpp:55-71), fused into the map pass. This is the CLI quantize
 * command's outputs (tools/colorq.cpp:96-109) in one call. */
int cqb_quantize_ex(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, const cqb_termination* term,
                    uint64_t seed, double* centers_out, double* sse_history, int hist_cap, uint8_t* index_out,
                    uint8_t* rgb_out, uint8_t* error_out, cqb_report* report);
/* run_km_full (kmeans.hpp:409-426), the KM / KM-C branch of generate_palette
 * (methods.hpp:155-160): conventional k-means over
 * every pixel with the exhaustive assignment (assign_naive, kmeans.hpp:83-106),
 * initialized like run_wsm. Runs on the unique colors weighted by their
 * counts (the same memberships, sums and SSE); report->dist_evals is the
 * reference's P*k per iteration. report->mse is 0 (filled by the caller). */
int cqb_run_km_full(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, const cqb_termination* term,
                    uint64_t seed, double* centers_out, double* sse_history, int hist_cap, cqb_report* report);
/* run_fkm (fast_variants.hpp:20-81), the FKM / FKM-C branch of
 * generate_palette (methods.hpp:163-178): iteration 1
 * exhaustive, then each point searches only the k_prime centers nearest to
 * its previous one (the first k_prime entries of its sorted center row).
 * Initialized like run_wsm; report->dist_evals follows the reference
 * (P*k, then P*k' per iteration, plus the center-table pairs). */
int cqb_run_fkm(cqb_ctx* ctx, const uint8_t* rgb, int width, int height, int k, int k_prime,
                const cqb_termination* term, uint64_t seed, double* centers_out, double* sse_history, int hist_cap,
                cqb_report* report);
/* error_image(original, quantized) (image_ops.hpp:55-71): per channel
 * 255 - min(255, 4|o - q|). Host buffers of n_pixels u8x3 pixels. */
int cqb_error_image(cqb_ctx* ctx, const uint8_t* original, const uint8_t* quantized, uint64_t n_pixels,
                    uint8_t* out);

/* Same pipeline with DEVICE-resident image and outputs (all pointers are
 * device pointers on the context's device; outputs nullable). Enqueued on
 * the context stream; when `sync` is 0 the call returns without waiting and
 * report/centers/sse_history are NOT filled (use cqb_fetch_results). */
int cqb_quantize_device(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int k, const cqb_termination* term,
                        uint64_t seed, uint8_t* d_index_out, uint8_t* d_rgb_out, int sync, double* centers_out,
                        double* sse_history, int hist_cap, cqb_report* report);
/* Waits for the last enqueued quantize on this context and copies its results. */
int cqb_fetch_results(cqb_ctx* ctx, double* centers_out, double* sse_history, int hist_cap, cqb_report* report);

/* Config 5: n_images independent device-resident images,
 * each the generate_palette + map_pixels + mse of cqb_quantize_device, with
 * `lanes` images in flight on this GPU (0 = default 4). Each lane owns a
 * stream, a device arena and a 1/lanes slice of the SMs for its persistent
 * WSM kernel. Lanes wait for work already enqueued on the context's stream.
 * The call returns when every image is done.
 * d_rgb[i]: image i (u8x3, n_pixels[i] pixels). d_index_out / d_rgb_out:
 * arrays of n_images device pointers, or NULL; individual entries may be NULL.
 * centers_out: n_images x k x 3 doubles. reports: n_images entries. */
int cqb_quantize_batch(cqb_ctx* ctx, int n_images, const uint8_t* const* d_rgb, const uint64_t* n_pixels, int k,
                       const cqb_termination* term, uint64_t seed, uint8_t* const* d_index_out,
                       uint8_t* const* d_rgb_out, int lanes, double* centers_out, cqb_report* reports);

/* Many seeds of one image: the paper's repeated-run protocol (the
 * reference's run_bench calls generate_palette once per seed, bench.hpp:
 * 201-204). The host raster is uploaded once; run i uses seeds[i] and runs
 * the full device pipeline (histogram, WSM / WSM-C, map + MSE), `lanes` runs
 * in flight like cqb_quantize_batch. centers_out: n_runs x k x 3 doubles;
 * reports[i].mse is the run's exact MSE. No raster outputs. */
int cqb_quantize_runs(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, int k, const cqb_termination* term,
                      int n_runs, const uint64_t* seeds, int lanes, double* centers_out, cqb_report* reports);

/* ---- generic weighted points (kmeans.hpp's span<const Vec3> API) --------
 * points: n x 3 doubles (row-major), weights: n doubles, memberships: n
 * int32, centers: k x 3 doubles, 1 <= k <= 1024 (k > 1024 ->
 * CQB_ERR_UNSUPPORTED). Distances are FP64 without FMA and the tables are
 * sorted by (distance, index) with self first, as the reference builds them;
 * update_centers reproduces the reference's sequential per-cluster sums bit
 * for bit (stable sort by membership, one thread per cluster). */

/* Replaces init_centers(points, k, seed) (kmeans.hpp:53-70): the chosen point
 * indices of the partial Fisher-Yates (center i = points[chosen_out[i]]).
 * k < 1 or k > n -> CQB_ERR_INVALID_ARGUMENT (:54-56). */
int cqb_init_centers(cqb_ctx* ctx, uint64_t n_points, int k, uint64_t seed, uint32_t* chosen_out);

/* Replaces ClusterState::update_center_tables' full rebuild
 * (kmeans.hpp:132-184): center_dists k x k (symmetric, zero diagonal),
 * sorted_order k x k (row i = [i, others by (d, index)]). Outputs nullable. */
int cqb_points_tables(cqb_ctx* ctx, const double* centers, int k, double* center_dists, int32_t* sorted_order);

/* Replaces assign_sort_means(points, weights, palette, state, audit)
 * (kmeans.hpp:201-239; mode 0) and assign_naive(points, weights, palette, m)
 * (kmeans.hpp:83-106; mode 1, exhaustive, lowest index on ties).
 * memberships: in = previous (mode 0), out = new. With center_dists +
 * sorted_order (a ClusterState's tables) the scan reads them; with NULL the
 * tables of `centers` are built first. weighted_sse: fixed-order tree sum of
 * w * min distance; dist_evals: the reference's count. skip_rank_out /
 * prev_dist_out (nullable, mode 0): per point the row position where the scan
 * stopped early (-1 if it ran to the end) and its previous-center distance,
 * the arguments of the reference's SkipAudit callback. */
int cqb_points_assign(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n, const double* centers,
                      int k, const double* center_dists, const int32_t* sorted_order, int mode,
                      int32_t* memberships, double* weighted_sse, uint64_t* dist_evals, int32_t* skip_rank_out,
                      double* prev_dist_out);

/* Replaces update_centers(points, weights, memberships, prev)
 * (kmeans.hpp:245-296), the empty-cluster reseed included. */
int cqb_points_update(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n,
                      const int32_t* memberships, const double* prev, int k, double* next_out);

/* Replaces weighted_sse(points, weights, palette, memberships) (kmeans.hpp:306-317). */
int cqb_points_sse(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n, const double* centers,
                   int k, const int32_t* memberships, double* sse_out);

/* Replaces run_wsm_points(points, weights, k, term, seed, trajectory)
 * (kmeans.hpp:379-390); also the device path of run_wsm for histograms whose
 * colors or weights the integer histogram path cannot take. trajectory:
 * traj_cap x k x 3 doubles (the palette after every update), nullable;
 * memberships_out: n int32, nullable. */
int cqb_run_wsm_points(cqb_ctx* ctx, const double* points, const double* weights, uint64_t n, int k,
                       const cqb_termination* term, uint64_t seed, double* centers_out, double* sse_history,
                       int hist_cap, double* trajectory, int traj_cap, int32_t* memberships_out,
                       cqb_report* report);

/* ---- post-processing ---------------------------------------------------
 * Replaces map_pixels(img, palette) (image_ops.hpp:18-51): nearest ROUNDED
 * palette entry, lowest index on ties. centers: k x 3 doubles, k in [1,256];
 * k < 1 -> CQB_ERR_INVALID_ARGUMENT (:19). Outputs nullable; sq_err_sum
 * (nullable) = Σ squared error vs the input (mse numerator). */
int cqb_map_pixels(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, const double* centers, int k,
                   uint8_t* rgb_out, uint8_t* index_out, uint64_t* sq_err_sum);

/* Replaces mse(a, b) (metrics.hpp:18-29): exact u64 sum / P. */
int cqb_mse(cqb_ctx* ctx, const uint8_t* a, const uint8_t* b, uint64_t n_pixels, double* out);

/* ---- sharded WSM (multi-GPU, one process per GPU) ----------------------
 * The unique samples (Morton order) are split into contiguous ranges, one
 * per rank. Each WSM iteration: cqb_shard_step on the rank's range returns
 * the EXACT integer cluster moments (K x {Σc·r, Σc·g, Σc·b, Σc, Σc·|x|²},
 * row-major [5][k]); the host allreduces them (sum) and every rank runs
 * cqb_finalize_moments on the identical totals, so all ranks follow the
 * bit-identical trajectory of the single-GPU run. Driver:
 * paper_1011_0093_b200/distributed.py. */
int cqb_shard_prepare(cqb_ctx* ctx, const uint8_t* rgb, uint64_t n_pixels, int k, uint64_t seed, uint64_t* n_unique,
                      double* init_centers);
int cqb_shard_step(cqb_ctx* ctx, uint64_t lo, uint64_t hi, const double* centers, int dense_first,
                   uint64_t* moments, uint64_t* point_evals);
int cqb_finalize_moments(cqb_ctx* ctx, const uint64_t* moments, const double* centers_used, int k, uint64_t total,
                         double* new_centers, double* sse, int* n_empty, int* empty_list);
int cqb_shard_reseed_candidate(cqb_ctx* ctx, uint64_t lo, uint64_t hi, const double* centers_used,
                               const uint32_t* taken_ranks, int n_taken, double* d_out, uint32_t* rank_out,
                               uint32_t* key_out);

/* ---- sharded WSM with the exchange inside the persistent loop ------------
 * BASELINE config 4 at 1..8 GPUs, one process per GPU. Replaces the host
 * round trip per iteration of the cqb_shard_* path: every rank runs the whole
 * quantize (histogram of the full image, init, loop, map) on its own GPU; the
 * loop processes only the rank's contiguous range of the Morton-ordered
 * samples, and once per iteration each rank writes its exact K x 5 moment
 * sums into every peer's exchange window over NVLink (plain stores + a
 * sys-scope flag) and sums the world's contributions itself: no NCCL call and
 * no host involvement inside the loop. Empty-cluster reseed candidates use
 * the same mailboxes. At the end the label ranges are all-gathered into every
 * window, each rank builds the full key -> index table, and maps its own
 * pixel range. Integer moments make every rank's trajectory bit-identical to
 * the single-GPU run.
 *
 * Setup (collective): cqb_xch_window allocates this rank's window and returns
 * its cudaIpcMemHandle (CQB_IPC_HANDLE_BYTES bytes); the host all-gathers the
 * handles (torch.distributed) and passes all of them, in rank order, to
 * cqb_xch_open. cqb_xch_emulate(v) instead makes v block groups of the one
 * cooperative launch act as the ranks (single-GPU test of the protocol).
 *
 * cqb_quantize_sharded enqueues on the context stream (like
 * cqb_quantize_device with sync = 0); results via cqb_fetch_results. The
 * report is complete except dist_evals, which counts this rank's point
 * evaluations (+ the pair evaluations on rank 0): sum it over the ranks.
 * px_range (nullable, 2 values) receives the pixel range [lo, hi) this rank
 * wrote into d_index_out / d_rgb_out (full-image buffers). A peer that does
 * not answer within 5 s fails the call with CQB_ERR_NCCL instead of hanging. */
#define CQB_IPC_HANDLE_BYTES 64
int cqb_xch_window(cqb_ctx* ctx, int world, int rank, void* ipc_handle_out);
int cqb_xch_open(cqb_ctx* ctx, const void* handles);
/* Peer wait limit of the in-kernel exchange (default 5 s; the first exchange
 * of a launch waits 4x as long). On a timeout the call fails with
 * CQB_ERR_NCCL and the exchange is reset: every rank must call
 * cqb_xch_window + cqb_xch_open (or cqb_xch_emulate) again before the next
 * cqb_quantize_sharded. */
int cqb_xch_set_timeout(cqb_ctx* ctx, double seconds);

int cqb_xch_emulate(cqb_ctx* ctx, int vranks);
int cqb_quantize_sharded(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int k, const cqb_termination* term,
                         uint64_t seed, uint8_t* d_index_out, uint8_t* d_rgb_out, uint64_t* px_range);

/* ---- pixel-row sharded histogram (config 4 across GPUs) -----------------
 * build_histogram (histogram.hpp:65-99) split over the W ranks of
 * cqb_quantize_sharded, so no rank counts the whole image:
 *  1. cqb_hist_rows: rank r counts the pixel rows it maps (pixel_range: 16-
 *     pixel aligned, the last rank takes the tail; global pixel indices) into
 *     its own bin table and compacts the touched bins in Morton order into
 *     d_out as u32 triplets {key, count, first pixel} (cap >= its pixels).
 *     owner_counts[o] = how many of them fall in rank o's Morton range
 *     [o 2^24 / W, (o + 1) 2^24 / W); they are contiguous, in owner order.
 *  2. the host moves each run to its owner (all-to-all; NCCL over NVLink).
 *  3. cqb_hist_merge: the owner merges what it received (count sum, first
 *     pixel min) and compacts its range (Morton order) into d_out.
 *  4. the host all-gathers the owners' lists; concatenated in rank order they
 *     are the whole image's histogram in Morton order, which
 *     cqb_quantize_sharded_samples takes instead of counting the image
 *     (with no exchange set up: the single-GPU pipeline from that histogram).
 * The result is identical to the unsharded histogram, entry for entry. */
int cqb_hist_rows(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int world, int rank, uint32_t* d_out,
                  uint64_t cap, uint64_t* n_out, uint64_t* owner_counts);
int cqb_hist_merge(cqb_ctx* ctx, const uint32_t* d_in, uint64_t n_in, uint32_t* d_out, uint64_t cap,
                   uint64_t* n_out);
/* Morton-range sharded histogram (the cheaper split when every rank holds the
 * raster): rank r counts EVERY pixel but only into the bins of its Morton
 * range (whole compaction tiles: [r T / W, (r+1) T / W) of T = 2048 tiles of
 * 8192 bins), in L2-sized passes, and compacts that range into d_out
 * (triplets as above, cap >= min(n_pixels, range bins)). No exchange is
 * needed to finish the owners' lists; concatenated in rank order they are the
 * whole histogram. */
int cqb_hist_range(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, int world, int rank, uint32_t* d_out,
                   uint64_t cap, uint64_t* n_out);
int cqb_quantize_sharded_samples(cqb_ctx* ctx, const uint8_t* d_rgb, uint64_t n_pixels, const uint32_t* d_samples,
                                 uint64_t n_unique, int k, const cqb_termination* term, uint64_t seed,
                                 uint8_t* d_index_out, uint8_t* d_rgb_out, uint64_t* px_range);

#ifdef __cplusplus
}
#endif
#endif /* COLORQ_B200_H */
