// TEST INFRASTRUCTURE ONLY — C-ABI wrapper around the UNMODIFIED reference.
//
// Compiles the reference colorq headers where they lie
// (/root/reference/proj/include, passed with -I by oracle/Makefile; nothing is
// copied into this repo) and exposes the hot-path functions through extern "C"
// so tests can (1) pin the C restatement oracle/wsm_oracle.c and (2) generate
// the golden vectors under tests/golden/. The built library lands in
// oracle/_ref/ (git-ignored, travels to the GPU box) and also serves as the
// reference CPU arm of bench.py (`--impl reference`, cpu_baseline kind
// "reference"). The product library never links or calls it.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <sstream>
#include <thread>
#include <vector>

#include "colorq/bench.hpp"
#include "colorq/histogram.hpp"
#include "colorq/image_ops.hpp"
#include "colorq/kmeans.hpp"
#include "colorq/methods.hpp"
#include "colorq/metrics.hpp"
#include "colorq/palette.hpp"
#include "colorq/ppm.hpp"

using namespace colorq;

namespace {

RgbImage make_image(const std::uint8_t* rgb, std::uint64_t w, std::uint64_t h) {
  RgbImage img{int(w), int(h)};
  std::memcpy(img.pixels.data(), rgb, 3 * w * h);
  return img;
}

ColorHistogram make_hist(const std::uint32_t* keys, const std::uint32_t* counts, std::uint64_t n,
                         std::uint64_t total) {
  ColorHistogram h;
  h.total_pixels = total;
  h.colors.resize(n);
  h.counts.assign(counts, counts + n);
  h.weights.resize(n);
  const double inv_total = 1.0 / double(total);
  for (std::uint64_t i = 0; i < n; ++i) {
    h.colors[i] = to_vec3(unpack_rgb(keys[i]));
    h.weights[i] = double(counts[i]) * inv_total;  // histogram.hpp:95-97
  }
  return h;
}

Palette make_palette(const double* C, int k) {
  Palette p;
  p.centers.resize(std::size_t(k));
  for (int i = 0; i < k; ++i) p.centers[std::size_t(i)] = Vec3{C[3 * i], C[3 * i + 1], C[3 * i + 2]};
  return p;
}

void store_palette(const Palette& p, double* C) {
  for (std::size_t i = 0; i < p.size(); ++i)
    for (int d = 0; d < 3; ++d) C[3 * i + std::size_t(d)] = p[i][std::size_t(d)];
}

Termination make_term(int mode, int max_iters, double eps, int cap) {
  if (mode == 0) return Termination::fixed(max_iters);
  return Termination::convergent(eps, cap);
}

}  // namespace

extern "C" {

void ref_mt64_stream(std::uint64_t seed, std::uint64_t* out, int n) {
  std::mt19937_64 g(seed);
  for (int i = 0; i < n; ++i) out[i] = g();
}

std::uint64_t ref_next_prime(std::uint64_t n) { return next_prime(n); }

std::uint64_t ref_universal_hash(std::uint8_t r, std::uint8_t g, std::uint8_t b, std::uint64_t m,
                                 std::uint64_t a0, std::uint64_t a1, std::uint64_t a2) {
  UniversalHashParams p{m, {a0, a1, a2}};
  return universal_hash(RgbColor{r, g, b}, p);
}

// build_histogram(img) with the reference's default hash sizing
// (histogram.hpp:105-108), or explicit params when hash_expected > 0.
std::int64_t ref_build_histogram(const std::uint8_t* rgb, std::uint64_t n, std::uint32_t* keys,
                                 std::uint32_t* counts, double* weights, std::uint64_t hash_expected,
                                 std::uint64_t hash_seed) {
  try {
    const RgbImage img = make_image(rgb, n, 1);
    const ColorHistogram h = hash_expected ? build_histogram(img, make_hash_params(hash_expected, hash_seed))
                                           : build_histogram(img);
    for (std::size_t i = 0; i < h.size(); ++i) {
      keys[i] = pack_rgb(round_to_rgb(h.colors[i]));
      counts[i] = h.counts[i];
      if (weights) weights[i] = h.weights[i];
    }
    return std::int64_t(h.size());
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_init_centers(const std::uint32_t* keys, std::uint64_t n, int k, std::uint64_t seed, double* C) {
  try {
    std::vector<Vec3> pts(n);
    for (std::uint64_t i = 0; i < n; ++i) pts[i] = to_vec3(unpack_rgb(keys[i]));
    store_palette(init_centers(std::span<const Vec3>(pts), k, seed), C);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// One fresh update_center_tables + assign_sort_means (kmeans.hpp:132-239).
int ref_sort_means_step(const std::uint32_t* keys, const std::uint32_t* counts, std::uint64_t n,
                        std::uint64_t total, const double* C, int k, std::int32_t* labels,
                        double* sse, std::uint64_t* evals, double* D, std::int32_t* order) {
  try {
    const ColorHistogram h = make_hist(keys, counts, n, total);
    const Palette pal = make_palette(C, k);
    ClusterState st;
    st.memberships.assign(labels, labels + n);
    st.update_center_tables(pal);
    const AssignResult ar = assign_sort_means(h.colors, h.weights, pal, st);
    std::copy(st.memberships.begin(), st.memberships.end(), labels);
    *sse = ar.weighted_sse;
    *evals = ar.dist_evals;
    if (D) std::copy(st.center_dists.begin(), st.center_dists.end(), D);
    if (order) std::copy(st.sorted_order.begin(), st.sorted_order.end(), order);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_update_centers(const std::uint32_t* keys, const std::uint32_t* counts, std::uint64_t n,
                       std::uint64_t total, const std::int32_t* labels, const double* prev, int k,
                       double* next) {
  try {
    const ColorHistogram h = make_hist(keys, counts, n, total);
    Memberships m(labels, labels + n);
    store_palette(update_centers(h, m, make_palette(prev, k)), next);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// run_wsm (kmeans.hpp:394-404) with the trajectory hook. Returns iterations.
int ref_run_wsm(const std::uint32_t* keys, const std::uint32_t* counts, std::uint64_t n, std::uint64_t total,
                int k, int mode, int max_iters, double eps, int cap, std::uint64_t seed, double* C_out,
                double* sse_out, std::uint64_t* evals_out, double* sse_hist, int hist_cap, double* traj,
                int traj_cap) {
  try {
    const ColorHistogram h = make_hist(keys, counts, n, total);
    std::vector<Palette> trajectory;
    const KmRunResult r = run_wsm(h, k, make_term(mode, max_iters, eps, cap), seed, traj ? &trajectory : nullptr);
    store_palette(r.palette, C_out);
    *sse_out = r.report.sse;
    *evals_out = r.report.dist_evals;
    if (sse_hist)
      for (std::size_t i = 0; i < r.report.sse_history.size() && int(i) < hist_cap; ++i)
        sse_hist[i] = r.report.sse_history[i];
    if (traj)
      for (std::size_t t = 0; t < trajectory.size() && int(t) < traj_cap; ++t)
        store_palette(trajectory[t], traj + t * std::size_t(3 * k));
    return r.report.iterations;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_map_pixels(const std::uint8_t* rgb, std::uint64_t n, const double* C, int k, std::uint8_t* out_rgb) {
  try {
    const RgbImage out = map_pixels(make_image(rgb, n, 1), make_palette(C, k));
    std::memcpy(out_rgb, out.pixels.data(), 3 * n);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

double ref_mse(const std::uint8_t* a, const std::uint8_t* b, std::uint64_t n) {
  return mse(make_image(a, n, 1), make_image(b, n, 1));
}

// The reference hot path end to end as the CLI composes it
// (tools/colorq.cpp:96-102): generate_palette's WSM branch
// (methods.hpp:182-189: build_histogram + run_wsm) + map_pixels + mse.
// Termination is passed explicitly so BASELINE's convergent(1e-4, 100) is
// reachable (the CLI always uses cap 1000). Times in ms.
int ref_quantize(const std::uint8_t* rgb, int w, int h, int k, int mode, int max_iters, double eps, int cap,
                 std::uint64_t seed, double* C_out, int* iterations, double* sse, std::uint64_t* evals,
                 std::uint8_t* out_rgb, double* mse_out, double* palette_ms, double* map_ms) {
  try {
    const RgbImage img = make_image(rgb, std::uint64_t(w), std::uint64_t(h));
    StopWatch watch;
    const ColorHistogram hist = build_histogram(img);
    const KmRunResult r = run_wsm(hist, k, make_term(mode, max_iters, eps, cap), seed);
    if (palette_ms) *palette_ms = watch.elapsed_ms();
    StopWatch mwatch;
    const RgbImage mapped = map_pixels(img, r.palette);
    const double m = mse(img, mapped);
    if (map_ms) *map_ms = mwatch.elapsed_ms();
    store_palette(r.palette, C_out);
    *iterations = r.report.iterations;
    *sse = r.report.sse;
    *evals = r.report.dist_evals;
    *mse_out = m;
    if (out_rgb) std::memcpy(out_rgb, mapped.pixels.data(), 3 * std::size_t(w) * std::size_t(h));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Many independent images on a thread pool, one image per worker at a time
// (the bench.hpp:187-223 pattern). Returns wall ms for the whole batch.
double ref_quantize_many(const std::uint8_t* const* imgs, int count, int w, int h, int k, int mode,
                         int max_iters, double eps, int cap, std::uint64_t seed, int nthreads,
                         double* mse_out, int* iters_out) {
  std::atomic<int> next{0};
  auto worker = [&]() {
    for (;;) {
      const int i = next.fetch_add(1);
      if (i >= count) return;
      double C[3 * 256 * 16];
      std::vector<double> cbuf(std::size_t(3 * k));
      int it = 0;
      double s = 0, m = 0;
      std::uint64_t ev = 0;
      ref_quantize(imgs[i], w, h, k, mode, max_iters, eps, cap, seed, cbuf.data(), &it, &s, &ev, nullptr, &m,
                   nullptr, nullptr);
      (void)C;
      if (mse_out) mse_out[i] = m;
      if (iters_out) iters_out[i] = it;
    }
  };
  StopWatch watch;
  std::vector<std::thread> pool;
  const int nt = std::max(1, std::min(nthreads, count));
  for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  return watch.elapsed_ms();
}

// run_km_full (kmeans.hpp:409-426), §8(f) row f3: returns iterations or -1.
int ref_run_km_full(const std::uint8_t* rgb, int w, int h, int k, int mode, int max_iters, double eps, int cap,
                    std::uint64_t seed, double* C_out, double* sse, std::uint64_t* evals, double* hist, int hist_cap) {
  try {
    const RgbImage img = make_image(rgb, std::uint64_t(w), std::uint64_t(h));
    const KmRunResult r = run_km_full(img, k, make_term(mode, max_iters, eps, cap), seed);
    store_palette(r.palette, C_out);
    *sse = r.report.sse;
    *evals = r.report.dist_evals;
    for (int i = 0; i < std::min<int>(hist_cap, int(r.report.sse_history.size())); ++i) hist[i] = r.report.sse_history[i];
    return r.report.iterations;
  } catch (const std::exception&) {
    return -1;
  }
}

// run_fkm through generate_palette's FKM branch (methods.hpp:163-178), §8(f) row f4.
int ref_run_fkm(const std::uint8_t* rgb, int w, int h, int k, int k_prime, int mode, int max_iters, double eps,
                std::uint64_t seed, double* C_out, double* sse, std::uint64_t* evals, double* hist, int hist_cap) {
  try {
    const RgbImage img = make_image(rgb, std::uint64_t(w), std::uint64_t(h));
    MethodParams mp;
    mp.id = mode ? MethodId::FkmC : MethodId::Fkm;
    mp.iters = max_iters;
    mp.epsilon = eps;
    mp.k_prime = k_prime;
    const QuantizeOutcome r = generate_palette(img, mp, k, seed);
    store_palette(r.palette, C_out);
    *sse = r.report.sse;
    *evals = r.report.dist_evals;
    for (int i = 0; i < std::min<int>(hist_cap, int(r.report.sse_history.size())); ++i) hist[i] = r.report.sse_history[i];
    return r.report.iterations;
  } catch (const std::exception&) {
    return -1;
  }
}

// run_bench + write_bench_outputs (bench.hpp:160-313), §8(f) row f2: the
// config text as the CLI reads it; single-threaded. 0 ok, -1 error.
int ref_run_bench(const char* config_text, const char* prefix) {
  try {
    BenchConfig cfg;
    std::istringstream in(config_text);
    apply_config_text(cfg, in);
    cfg.output_prefix = prefix;
    cfg.threads = 1;
    write_bench_outputs(run_bench(cfg), cfg.output_prefix);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// ---- §8(f) row f1: file formats and error_image (ppm.hpp, palette.hpp,
// image_ops.hpp:55-71), for the CLI parity tests.

// write_ppm bytes of a w x h image; returns the byte count (or the needed
// capacity when cap is too small).
// ---- the span<const Vec3> point-set API (kmeans.hpp:53-74, 201-317, 379-390)
namespace {
std::vector<Vec3> make_points(const double* X, std::uint64_t n) {
  std::vector<Vec3> v(n);
  for (std::uint64_t i = 0; i < n; ++i) v[i] = Vec3{X[3 * i], X[3 * i + 1], X[3 * i + 2]};
  return v;
}
}  // namespace

int ref_init_centers_points(const double* X, std::uint64_t n, int k, std::uint64_t seed, double* C) {
  try {
    store_palette(init_centers(std::span<const Vec3>(make_points(X, n)), k, seed), C);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// One ClusterState step (update_center_tables + assign_sort_means, or
// assign_naive with naive = 1) from the given memberships.
int ref_points_assign(const double* X, const double* W, std::uint64_t n, const double* C, int k, int naive,
                      std::int32_t* m, double* sse, std::uint64_t* evals, std::uint64_t* audited) {
  try {
    const std::vector<Vec3> pts = make_points(X, n);
    const Palette pal = make_palette(C, k);
    AssignResult ar;
    if (naive) {
      Memberships mm;
      ar = assign_naive(pts, std::span<const double>(W, n), pal, mm);
      std::copy(mm.begin(), mm.end(), m);
    } else {
      ClusterState st;
      st.memberships.assign(m, m + n);
      st.update_center_tables(pal);
      std::uint64_t cnt = 0;
      const SkipAudit audit = [&](std::size_t, int, int, double) { ++cnt; };
      ar = assign_sort_means(pts, std::span<const double>(W, n), pal, st, &audit);
      std::copy(st.memberships.begin(), st.memberships.end(), m);
      if (audited) *audited = cnt;
    }
    *sse = ar.weighted_sse;
    *evals = ar.dist_evals;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_points_update(const double* X, const double* W, std::uint64_t n, const std::int32_t* m, const double* prev,
                      int k, double* out) {
  const std::vector<Vec3> pts = make_points(X, n);
  const Memberships mm(m, m + n);
  store_palette(update_centers(pts, std::span<const double>(W, n), mm, make_palette(prev, k)), out);
  return 0;
}

double ref_points_sse(const double* X, const double* W, std::uint64_t n, const double* C, int k,
                      const std::int32_t* m) {
  const std::vector<Vec3> pts = make_points(X, n);
  return weighted_sse(pts, std::span<const double>(W, n), make_palette(C, k), Memberships(m, m + n));
}

int ref_run_wsm_points(const double* X, const double* W, std::uint64_t n, int k, int mode, int max_iters,
                       double eps, int cap, std::uint64_t seed, double* C_out, double* sse, std::uint64_t* evals,
                       double* hist, int hist_cap) {
  try {
    const std::vector<Vec3> pts = make_points(X, n);
    const KmRunResult r =
        run_wsm_points(pts, std::span<const double>(W, n), k, make_term(mode, max_iters, eps, cap), seed);
    store_palette(r.palette, C_out);
    *sse = r.report.sse;
    *evals = r.report.dist_evals;
    for (int i = 0; i < std::min(hist_cap, r.report.iterations); ++i) hist[i] = r.report.sse_history[std::size_t(i)];
    return r.report.iterations;
  } catch (const std::exception&) {
    return -1;
  }
}

std::int64_t ref_write_ppm(const std::uint8_t* rgb, int w, int h, std::uint8_t* out, std::int64_t cap) {
  const std::vector<unsigned char> b = write_ppm(make_image(rgb, std::uint64_t(w), std::uint64_t(h)));
  if (std::int64_t(b.size()) <= cap) std::memcpy(out, b.data(), b.size());
  return std::int64_t(b.size());
}

// read_ppm: 0 ok (w, h, pixels into rgb_out if it fits), 1..4 = PpmError kind
// + 1 (BadMagic, BadHeader, BadMaxval, Truncated), -1 other error.
int ref_read_ppm(const std::uint8_t* bytes, std::int64_t n, std::uint8_t* rgb_out, std::int64_t cap, int* w,
                 int* h) {
  try {
    const RgbImage img = read_ppm(std::span<const unsigned char>(bytes, std::size_t(n)));
    *w = img.width;
    *h = img.height;
    if (std::int64_t(img.size()) * 3 <= cap) std::memcpy(rgb_out, img.pixels.data(), img.size() * 3);
    return 0;
  } catch (const PpmError& e) {
    return int(e.kind) + 1;
  } catch (const std::exception&) {
    return -1;
  }
}

std::int64_t ref_palette_text(const double* C, int k, char* out, std::int64_t cap) {
  const std::string t = palette_to_text(make_palette(C, k));
  if (std::int64_t(t.size()) <= cap) std::memcpy(out, t.data(), t.size());
  return std::int64_t(t.size());
}

void ref_error_image(const std::uint8_t* a, const std::uint8_t* b, std::uint64_t n, std::uint8_t* out) {
  const RgbImage e = error_image(make_image(a, n, 1), make_image(b, n, 1));
  std::memcpy(out, e.pixels.data(), 3 * n);
}

}  // extern "C"
