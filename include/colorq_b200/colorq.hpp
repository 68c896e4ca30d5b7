// colorq_b200/colorq.hpp — drop-in C++ front-end for the WSM hot path.
//
// Re-declares, in namespace colorq, the types and hot-path functions of the
// reference header-only library (/root/reference/proj/include/colorq) with
// the reference's signatures, and implements them over the C ABI
// (include/colorq_b200.h) of the sm_100a CUDA library. A caller of
//   build_histogram(const RgbImage&)                    histogram.hpp:105
//   run_wsm(const ColorHistogram&, k, Termination, seed, trajectory*)
//                                                       kmeans.hpp:394
//   generate_palette(const RgbImage&, MethodParams, k, seed)  [WSM/WSM-C]
//                                                       methods.hpp:107,182-189
//   map_pixels(const RgbImage&, const Palette&)         image_ops.hpp:18
//   mse(const RgbImage&, const RgbImage&)               metrics.hpp:18
// includes this header instead and links libcolorq_b200.so. Errors follow the
// reference: std::invalid_argument for argument errors (CLI exit code 4),
// std::runtime_error for device failures. Each host thread uses its own
// device context (thread_local), so concurrent calls are safe.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../colorq_b200.h"

namespace colorq {

using Vec3 = std::array<double, 3>;

struct RgbColor {
  std::uint8_t r = 0, g = 0, b = 0;
  friend bool operator==(const RgbColor&, const RgbColor&) = default;
};
static_assert(sizeof(RgbColor) == 3, "RgbColor must be packed u8x3");

constexpr std::uint32_t pack_rgb(RgbColor c) {
  return (std::uint32_t(c.r) << 16) | (std::uint32_t(c.g) << 8) | std::uint32_t(c.b);
}
constexpr RgbColor unpack_rgb(std::uint32_t k) {
  return RgbColor{std::uint8_t(k >> 16), std::uint8_t(k >> 8), std::uint8_t(k)};
}
inline Vec3 to_vec3(RgbColor c) { return Vec3{double(c.r), double(c.g), double(c.b)}; }

inline RgbColor round_to_rgb(const Vec3& v) {
  auto q = [](double x) {
    long r = std::lround(x);
    return std::uint8_t(r < 0 ? 0 : (r > 255 ? 255 : r));
  };
  return RgbColor{q(v[0]), q(v[1]), q(v[2])};
}

inline double dist2(const Vec3& a, const Vec3& b) {
  const double x = a[0] - b[0], y = a[1] - b[1], z = a[2] - b[2];
  return x * x + y * y + z * z;
}

struct RgbImage {
  int width = 0, height = 0;
  std::vector<RgbColor> pixels;
  RgbImage() = default;
  RgbImage(int w, int h, RgbColor fill = RgbColor{}) : width(w), height(h) {
    if (w <= 0 || h <= 0) throw std::invalid_argument("image dimensions must be positive");
    pixels.assign(std::size_t(w) * std::size_t(h), fill);
  }
  std::size_t size() const { return pixels.size(); }
  RgbColor& at(int x, int y) { return pixels[std::size_t(y) * std::size_t(width) + std::size_t(x)]; }
  const RgbColor& at(int x, int y) const { return pixels[std::size_t(y) * std::size_t(width) + std::size_t(x)]; }
  friend bool operator==(const RgbImage&, const RgbImage&) = default;
};

struct Palette {
  std::vector<Vec3> centers;
  Palette() = default;
  explicit Palette(std::vector<Vec3> c) : centers(std::move(c)) {}
  std::size_t size() const { return centers.size(); }
  bool empty() const { return centers.empty(); }
  Vec3& operator[](std::size_t i) { return centers[i]; }
  const Vec3& operator[](std::size_t i) const { return centers[i]; }
};

inline std::vector<RgbColor> round_palette(const Palette& p) {
  std::vector<RgbColor> out;
  out.reserve(p.size());
  for (const Vec3& c : p.centers) out.push_back(round_to_rgb(c));
  return out;
}

struct RunReport {
  std::string method;
  int k = 0;
  std::uint64_t seed = 0;
  int iterations = 0;
  double sse = 0.0;
  double mse = 0.0;
  double elapsed_ms = 0.0;
  std::uint64_t dist_evals = 0;
  std::vector<double> sse_history;

  // report.hpp:44-52: the runs CSV columns (6 significant digits for reals)
  static std::string csv_header() { return "method,k,seed,iterations,sse,mse,elapsed_ms,dist_evals"; }
  std::string csv_row() const {
    auto g6 = [](double v) {
      char b[40];
      std::snprintf(b, sizeof b, "%.6g", v);
      return std::string(b);
    };
    return method + "," + std::to_string(k) + "," + std::to_string(seed) + "," + std::to_string(iterations) + "," +
           g6(sse) + "," + g6(mse) + "," + g6(elapsed_ms) + "," + std::to_string(dist_evals);
  }
};

struct ColorHistogram {
  std::vector<Vec3> colors;
  std::vector<double> weights;
  std::vector<std::uint32_t> counts;
  std::uint64_t total_pixels = 0;
  std::size_t size() const { return colors.size(); }
};

struct Termination {
  enum class Mode { FixedIterations, Convergent };
  Mode mode = Mode::FixedIterations;
  int max_iters = 10;
  double epsilon = 1e-4;
  int hard_cap = 1000;
  static Termination fixed(int iters) { return Termination{Mode::FixedIterations, iters, 1e-4, 1000}; }
  static Termination convergent(double eps = 1e-4, int cap = 1000) {
    if (eps <= 0) throw std::invalid_argument("convergent termination requires epsilon > 0");
    return Termination{Mode::Convergent, 10, eps, cap};
  }
};

struct KmRunResult {
  Palette palette;
  RunReport report;
};

enum class MethodId { Mc, Wan, Wu, Mmm, Fcm, Pim, Km, KmC, Fkm, FkmC, Skm, Wsm, WsmC };

struct UnknownMethodError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// methods.hpp:71-85: every field of the reference, with its defaults. The
// SKM / FCM / PIM knobs (stable_iters, theta, q, delta, fuzzy_on_pixels)
// parameterize methods outside the B200 path; they are carried so callers
// that set them compile unchanged.
struct MethodParams {
  MethodId id = MethodId::Wsm;
  int iters = 10;                // fixed-iteration budget
  double epsilon = 1e-4;         // convergent threshold
  int k_prime = 8;               // fkm neighbour count
  int stable_iters = 10;         // skm warm-up iterations
  double theta = 1.0;            // skm stability threshold
  double q = 2.0;                // fcm / pim fuzziness
  double delta = 0.4;            // pim offset fraction
  bool fuzzy_on_pixels = false;  // fcm / pim on raw pixels
  Termination termination() const {
    return id == MethodId::WsmC || id == MethodId::KmC || id == MethodId::FkmC || id == MethodId::Skm
               ? Termination::convergent(epsilon)
               : Termination::fixed(iters);
  }
};

struct QuantizeOutcome {
  Palette palette;
  RunReport report;
};

namespace b200 {

struct CtxDeleter {
  void operator()(cqb_ctx* c) const { cqb_destroy(c); }
};

inline int& device_ordinal() {
  static int dev = 0;
  return dev;
}

inline cqb_ctx* context() {
  thread_local std::unique_ptr<cqb_ctx, CtxDeleter> ctx;
  if (!ctx) {
    cqb_ctx* raw = nullptr;
    const int rc = cqb_create(device_ordinal(), &raw);
    if (rc != CQB_OK) throw std::runtime_error("colorq_b200: cannot create a device context");
    ctx.reset(raw);
  }
  return ctx.get();
}

inline void check(int rc) {
  if (rc == CQB_OK) return;
  const std::string msg = cqb_last_error(context());
  if (rc == CQB_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error("colorq_b200: " + msg);
}

inline cqb_termination native(const Termination& t) {
  return cqb_termination{t.mode == Termination::Mode::Convergent ? 1 : 0, t.max_iters, t.epsilon, t.hard_cap};
}

inline int budget(const Termination& t) {
  return t.mode == Termination::Mode::Convergent ? t.hard_cap : t.max_iters;
}

inline Palette palette_from(const double* c, int k) {
  Palette p;
  p.centers.resize(std::size_t(k));
  for (int i = 0; i < k; ++i) p.centers[std::size_t(i)] = Vec3{c[3 * i], c[3 * i + 1], c[3 * i + 2]};
  return p;
}

inline const std::uint8_t* bytes(const RgbImage& img) {
  return reinterpret_cast<const std::uint8_t*>(img.pixels.data());
}

}  // namespace b200

// histogram.hpp:105-108
inline ColorHistogram build_histogram(const RgbImage& img) {
  if (img.size() == 0) throw std::invalid_argument("build_histogram: empty image");
  const std::uint64_t n = img.size();
  std::vector<std::uint32_t> keys(n), counts(n);
  std::vector<double> weights(n);
  std::uint64_t nu = 0;
  b200::check(cqb_build_histogram(b200::context(), b200::bytes(img), n, keys.data(), counts.data(), weights.data(),
                                  nullptr, n, &nu));
  ColorHistogram h;
  h.total_pixels = n;
  h.colors.resize(nu);
  for (std::uint64_t i = 0; i < nu; ++i) h.colors[i] = to_vec3(unpack_rgb(keys[i]));
  counts.resize(nu);
  weights.resize(nu);
  h.counts = std::move(counts);
  h.weights = std::move(weights);
  return h;
}

// ---------------------------------------------------------------- points
// kmeans.hpp's span<const Vec3> API over the device point-set kernels
// (cqb_init_centers / cqb_points_* / cqb_run_wsm_points), k <= 1024.
using Memberships = std::vector<std::int32_t>;

struct AssignResult {
  double weighted_sse = 0.0;
  std::uint64_t dist_evals = 0;
};

// kmeans.hpp:194-196: called for every point whose sorted scan stopped early.
using SkipAudit =
    std::function<void(std::size_t point, int prev_center, int first_skipped_rank, double prev_dist)>;

namespace b200 {
inline const double* flat(std::span<const Vec3> v) { return v.empty() ? nullptr : v.front().data(); }
inline std::vector<double> flat(const Palette& p) {
  std::vector<double> c(3 * p.size());
  for (std::size_t i = 0; i < p.size(); ++i)
    for (int d = 0; d < 3; ++d) c[3 * i + std::size_t(d)] = p[i][std::size_t(d)];
  return c;
}
}  // namespace b200

// kmeans.hpp:53-74
inline Palette init_centers(std::span<const Vec3> points, int k, std::uint64_t seed) {
  if (k < 1) throw std::invalid_argument("init_centers: k must be >= 1");
  if (std::size_t(k) > points.size())
    throw std::invalid_argument("init_centers: k exceeds the number of candidate points");
  std::vector<std::uint32_t> chosen(std::size_t(k), 0u);
  b200::check(cqb_init_centers(b200::context(), points.size(), k, seed, chosen.data()));
  Palette p;
  for (const std::uint32_t i : chosen) p.centers.push_back(points[i]);
  return p;
}
inline Palette init_centers(const ColorHistogram& hist, int k, std::uint64_t seed) {
  return init_centers(std::span<const Vec3>(hist.colors), k, seed);
}

// kmeans.hpp:86-113 (exhaustive; lowest index on ties)
inline AssignResult assign_naive(std::span<const Vec3> points, std::span<const double> weights,
                                 const Palette& palette, Memberships& out) {
  if (palette.empty()) throw std::invalid_argument("assign_naive: empty palette");
  out.assign(points.size(), 0);
  const std::vector<double> c = b200::flat(palette);
  AssignResult r;
  b200::check(cqb_points_assign(b200::context(), b200::flat(points), weights.data(), points.size(), c.data(),
                                int(palette.size()), nullptr, nullptr, 1, out.data(), &r.weighted_sse,
                                &r.dist_evals, nullptr, nullptr));
  return r;
}
inline Memberships assign_naive(const ColorHistogram& hist, const Palette& palette) {
  Memberships m;
  assign_naive(hist.colors, hist.weights, palette, m);
  return m;
}

// kmeans.hpp:118-189: previous memberships + the K x K center tables.
struct ClusterState {
  Memberships memberships;
  std::vector<double> center_dists;        // k*k, symmetric, zero diagonal
  std::vector<std::int32_t> sorted_order;  // k*k, row i = [i, others by (d, index)]
  int k = 0;

  double d(int i, int j) const { return center_dists[std::size_t(i) * std::size_t(k) + std::size_t(j)]; }
  const std::int32_t* order_row(int i) const { return &sorted_order[std::size_t(i) * std::size_t(k)]; }

  // Rebuilt on the device each call (a full rebuild equals the reference's
  // incremental one bit for bit); pair_evals counts the pairs the reference
  // recomputes: all of them first, then those with a moved center.
  void update_center_tables(const Palette& palette, std::uint64_t* pair_evals = nullptr) {
    const int nk = int(palette.size());
    const bool incremental = nk == k && prev_centers_.size() == std::size_t(nk);
    std::uint64_t still = 0;
    if (incremental)
      for (int i = 0; i < nk; ++i) still += palette[std::size_t(i)] == prev_centers_[std::size_t(i)];
    k = nk;
    center_dists.resize(std::size_t(k) * std::size_t(k));
    sorted_order.resize(std::size_t(k) * std::size_t(k));
    const std::vector<double> c = b200::flat(palette);
    b200::check(cqb_points_tables(b200::context(), c.data(), k, center_dists.data(), sorted_order.data()));
    if (pair_evals)
      *pair_evals += std::uint64_t(k) * std::uint64_t(k - 1) / 2 - (still ? still * (still - 1) / 2 : 0);
    prev_centers_ = palette.centers;
  }

 private:
  std::vector<Vec3> prev_centers_;
};

// kmeans.hpp:201-239
inline AssignResult assign_sort_means(std::span<const Vec3> points, std::span<const double> weights,
                                      const Palette& palette, ClusterState& state,
                                      const SkipAudit* audit = nullptr) {
  const int k = int(palette.size());
  if (state.k != k || state.memberships.size() != points.size())
    throw std::invalid_argument("assign_sort_means: state does not match inputs");
  const std::vector<double> c = b200::flat(palette);
  std::vector<std::int32_t> skip(audit ? points.size() : 0);
  std::vector<double> prev(audit ? points.size() : 0);
  const std::vector<std::int32_t> before = audit ? state.memberships : std::vector<std::int32_t>{};
  AssignResult r;
  b200::check(cqb_points_assign(b200::context(), b200::flat(points), weights.data(), points.size(), c.data(), k,
                                state.center_dists.data(), state.sorted_order.data(), 0, state.memberships.data(),
                                &r.weighted_sse, &r.dist_evals, audit ? skip.data() : nullptr,
                                audit ? prev.data() : nullptr));
  if (audit)
    for (std::size_t i = 0; i < points.size(); ++i)
      if (skip[i] >= 0) (*audit)(i, before[i], skip[i], prev[i]);
  return r;
}

// kmeans.hpp:245-302
inline Palette update_centers(std::span<const Vec3> points, std::span<const double> weights,
                              const Memberships& memberships, const Palette& prev) {
  const std::vector<double> c = b200::flat(prev);
  std::vector<double> next(c.size());
  b200::check(cqb_points_update(b200::context(), b200::flat(points), weights.data(), points.size(),
                                memberships.data(), c.data(), int(prev.size()), next.data()));
  return b200::palette_from(next.data(), int(prev.size()));
}
inline Palette update_centers(const ColorHistogram& hist, const Memberships& memberships, const Palette& prev) {
  return update_centers(std::span<const Vec3>(hist.colors), std::span<const double>(hist.weights), memberships, prev);
}

// kmeans.hpp:306-317
inline double weighted_sse(std::span<const Vec3> points, std::span<const double> weights, const Palette& palette,
                           const Memberships& memberships) {
  const std::vector<double> c = b200::flat(palette);
  double out = 0.0;
  b200::check(cqb_points_sse(b200::context(), b200::flat(points), weights.data(), points.size(), c.data(),
                             int(palette.size()), memberships.data(), &out));
  return out;
}
inline double weighted_sse(const ColorHistogram& hist, const Palette& palette, const Memberships& memberships) {
  return weighted_sse(hist.colors, hist.weights, palette, memberships);
}

namespace b200 {
inline KmRunResult run_points(std::span<const Vec3> points, std::span<const double> weights, int k,
                              const Termination& term, std::uint64_t seed, std::vector<Palette>* trajectory) {
  const auto t0 = std::chrono::steady_clock::now();
  if (k < 1) throw std::invalid_argument("init_centers: k must be >= 1");
  if (std::size_t(k) > points.size())
    throw std::invalid_argument("init_centers: k exceeds the number of candidate points");
  const cqb_termination t = native(term);
  const int cap = budget(term);
  std::vector<double> centers(3 * std::size_t(k)), hist_out(static_cast<std::size_t>(cap));
  std::vector<double> traj(trajectory ? std::size_t(cap) * 3 * std::size_t(k) : 0);
  cqb_report rep{};
  check(cqb_run_wsm_points(context(), flat(points), weights.data(), points.size(), k, &t, seed, centers.data(),
                           hist_out.data(), cap, trajectory ? traj.data() : nullptr, trajectory ? cap : 0, nullptr,
                           &rep));
  KmRunResult out;
  out.palette = palette_from(centers.data(), k);
  out.report.method = term.mode == Termination::Mode::Convergent ? "wsm-c" : "wsm";
  out.report.k = k;
  out.report.seed = seed;
  out.report.iterations = rep.iterations;
  out.report.sse = rep.sse;
  out.report.dist_evals = rep.dist_evals;
  out.report.sse_history.assign(hist_out.begin(), hist_out.begin() + rep.iterations);
  if (trajectory)
    for (int i = 0; i < rep.iterations; ++i) trajectory->push_back(palette_from(traj.data() + 3 * k * i, k));
  out.report.elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return out;
}
}  // namespace b200

// kmeans.hpp:379-390
inline KmRunResult run_wsm_points(std::span<const Vec3> points, std::span<const double> weights, int k,
                                  const Termination& term, std::uint64_t seed,
                                  std::vector<Palette>* trajectory = nullptr) {
  return b200::run_points(points, weights, k, term, seed, trajectory);
}

// kmeans.hpp:394-404. A histogram from build_histogram (8-bit colors, counts,
// weights = count * (1/total)) takes the integer path: exact u64 cluster sums
// in one persistent kernel, k <= 256. Any other histogram (real-valued
// colors or weights, k > 256) runs the point-set path over colors + weights.
inline KmRunResult run_wsm(const ColorHistogram& hist, int k, const Termination& term, std::uint64_t seed,
                           std::vector<Palette>* trajectory = nullptr) {
  const auto t0 = std::chrono::steady_clock::now();
  if (k < 1) throw std::invalid_argument("init_centers: k must be >= 1");
  if (std::size_t(k) > hist.size())
    throw std::invalid_argument("init_centers: k exceeds the number of candidate points");
  bool integer_path = k <= CQB_MAX_K && hist.counts.size() == hist.size() && hist.weights.size() == hist.size() &&
                      hist.total_pixels > 0;
  std::vector<std::uint32_t> keys(integer_path ? hist.size() : 0);
  const double inv_total = integer_path ? 1.0 / double(hist.total_pixels) : 0.0;
  for (std::size_t i = 0; integer_path && i < hist.size(); ++i) {
    const Vec3& c = hist.colors[i];
    for (double v : c) integer_path &= v >= 0 && v <= 255 && v == std::floor(v);
    integer_path &= hist.weights[i] == double(hist.counts[i]) * inv_total;  // histogram.hpp:94-97
    if (integer_path) keys[i] = pack_rgb(RgbColor{std::uint8_t(c[0]), std::uint8_t(c[1]), std::uint8_t(c[2])});
  }
  if (!integer_path) return b200::run_points(hist.colors, hist.weights, k, term, seed, trajectory);
  const cqb_termination t = b200::native(term);
  const int cap = b200::budget(term);
  std::vector<double> centers(3 * std::size_t(k)), hist_out(static_cast<std::size_t>(cap));
  std::vector<double> traj(trajectory ? std::size_t(cap) * 3 * std::size_t(k) : 0);
  cqb_report rep{};
  b200::check(cqb_run_wsm(b200::context(), keys.data(), hist.counts.data(), hist.size(), hist.total_pixels, k, &t,
                          seed, centers.data(), hist_out.data(), cap, trajectory ? traj.data() : nullptr,
                          trajectory ? cap : 0, nullptr, &rep));
  KmRunResult out;
  out.palette = b200::palette_from(centers.data(), k);
  out.report.method = term.mode == Termination::Mode::Convergent ? "wsm-c" : "wsm";
  out.report.k = k;
  out.report.seed = seed;
  out.report.iterations = rep.iterations;
  out.report.sse = rep.sse;
  out.report.dist_evals = rep.dist_evals;
  out.report.sse_history.assign(hist_out.begin(), hist_out.begin() + rep.iterations);
  if (trajectory)
    for (int i = 0; i < rep.iterations; ++i) trajectory->push_back(b200::palette_from(traj.data() + 3 * k * i, k));
  out.report.elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

// methods.hpp:107-197, WSM / WSM-C branch (:182-189). Other method ids are
// outside the B200 path and raise UnknownMethodError.
inline QuantizeOutcome generate_palette(const RgbImage& image, const MethodParams& mp, int k, std::uint64_t seed) {
  if (k < 1) throw std::invalid_argument("k must be >= 1");
  const bool km = mp.id == MethodId::Km || mp.id == MethodId::KmC;     // run_km_full, methods.hpp:155-160
  const bool fkm = mp.id == MethodId::Fkm || mp.id == MethodId::FkmC;  // run_fkm, methods.hpp:163-178
  if (mp.id != MethodId::Wsm && mp.id != MethodId::WsmC && !km && !fkm)
    throw UnknownMethodError("method not provided by the B200 path");
  if (image.size() == 0) throw std::invalid_argument("build_histogram: empty image");
  const auto t0 = std::chrono::steady_clock::now();
  const Termination term = mp.termination();
  const cqb_termination t = b200::native(term);
  const int cap = b200::budget(term);
  std::vector<double> centers(3 * std::size_t(k)), hist_out(static_cast<std::size_t>(cap));
  cqb_report rep{};
  if (km)
    b200::check(cqb_run_km_full(b200::context(), b200::bytes(image), image.width, image.height, k, &t, seed,
                                centers.data(), hist_out.data(), cap, &rep));
  else if (fkm)
    b200::check(cqb_run_fkm(b200::context(), b200::bytes(image), image.width, image.height, k, mp.k_prime, &t, seed,
                            centers.data(), hist_out.data(), cap, &rep));
  else
    b200::check(cqb_quantize(b200::context(), b200::bytes(image), image.width, image.height, k, &t, seed,
                             centers.data(), hist_out.data(), cap, nullptr, nullptr, &rep));
  QuantizeOutcome out;
  out.palette = b200::palette_from(centers.data(), k);
  out.report.method = km    ? (mp.id == MethodId::KmC ? "km-c" : "km")
                      : fkm ? (mp.id == MethodId::FkmC ? "fkm-c" : "fkm")
                            : (mp.id == MethodId::WsmC ? "wsm-c" : "wsm");
  out.report.k = k;
  out.report.seed = seed;
  out.report.iterations = rep.iterations;
  out.report.sse = rep.sse;
  out.report.dist_evals = rep.dist_evals;
  out.report.sse_history.assign(hist_out.begin(), hist_out.begin() + rep.iterations);
  out.report.elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

// image_ops.hpp:18-51
inline RgbImage map_pixels(const RgbImage& img, const Palette& palette) {
  if (palette.empty()) throw std::invalid_argument("map_pixels: empty palette");
  std::vector<double> c(3 * palette.size());
  for (std::size_t i = 0; i < palette.size(); ++i)
    for (int d = 0; d < 3; ++d) c[3 * i + std::size_t(d)] = palette[i][std::size_t(d)];
  RgbImage out(img.width, img.height);
  b200::check(cqb_map_pixels(b200::context(), b200::bytes(img), img.size(), c.data(), int(palette.size()),
                             reinterpret_cast<std::uint8_t*>(out.pixels.data()), nullptr, nullptr));
  return out;
}

// metrics.hpp:18-29
inline double mse(const RgbImage& a, const RgbImage& b) {
  if (a.width != b.width || a.height != b.height) throw std::invalid_argument("mse: dimension mismatch");
  double out = 0.0;
  b200::check(cqb_mse(b200::context(), b200::bytes(a), b200::bytes(b), a.size(), &out));
  return out;
}

// Fused quantize (the CLI's generate_palette + map_pixels + mse composition,
// tools/colorq.cpp:96-102) with the u8 index map as an extra output.
struct QuantizeResult {
  Palette palette;
  RunReport report;  // report.mse filled
  RgbImage mapped;
  std::vector<std::uint8_t> index_map;
};

inline QuantizeResult quantize(const RgbImage& image, int k, const Termination& term, std::uint64_t seed) {
  if (image.size() == 0) throw std::invalid_argument("build_histogram: empty image");
  const cqb_termination t = b200::native(term);
  const int cap = b200::budget(term);
  std::vector<double> centers(3 * std::size_t(std::max(k, 1))), hist_out(static_cast<std::size_t>(cap));
  QuantizeResult r;
  r.mapped = RgbImage(image.width, image.height);
  r.index_map.resize(image.size());
  cqb_report rep{};
  b200::check(cqb_quantize(b200::context(), b200::bytes(image), image.width, image.height, k, &t, seed,
                           centers.data(), hist_out.data(), cap, r.index_map.data(),
                           reinterpret_cast<std::uint8_t*>(r.mapped.pixels.data()), &rep));
  r.palette = b200::palette_from(centers.data(), k);
  r.report.method = term.mode == Termination::Mode::Convergent ? "wsm-c" : "wsm";
  r.report.k = k;
  r.report.seed = seed;
  r.report.iterations = rep.iterations;
  r.report.sse = rep.sse;
  r.report.mse = rep.mse;
  r.report.elapsed_ms = rep.elapsed_ms;
  r.report.dist_evals = rep.dist_evals;
  r.report.sse_history.assign(hist_out.begin(), hist_out.begin() + rep.iterations);
  return r;
}

}  // namespace colorq
