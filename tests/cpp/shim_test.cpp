// Drop-in shim test: the reference's own hot-path unit-test cases
// (histogram_test.cpp, kmeans_test.cpp, imageio_test.cpp, metrics_test.cpp,
// cli_test.cpp:142-151), restated against include/colorq_b200/colorq.hpp and
// therefore executed on the B200 through the C ABI. Prints one line per case;
// exit code = number of failures. Run by tests/test_gpu_parity.py.
#include <cmath>
#include <cstdio>
#include <map>
#include <random>
#include <set>

#include "colorq_b200/colorq.hpp"

using namespace colorq;

static int g_fail = 0;
#define REQUIRE(cond)                                                          \
  do {                                                                         \
    if (!(cond)) {                                                             \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
      ++g_fail;                                                                \
    }                                                                          \
  } while (0)
template <typename E, typename F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static RgbImage noise_image(int w, int h, int ncolors, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<RgbColor> table(static_cast<std::size_t>(ncolors));
  for (auto& c : table) c = RgbColor{std::uint8_t(rng()), std::uint8_t(rng()), std::uint8_t(rng())};
  RgbImage img(w, h);
  for (auto& px : img.pixels) px = table[rng() % table.size()];
  return img;
}

int main() {
  // histogram_test.cpp:46-61 — counts in scan order, weights 0.75 / 0.25
  {
    RgbImage one(1, 1, RgbColor{4, 5, 6});
    const ColorHistogram h1 = build_histogram(one);
    REQUIRE(h1.size() == 1 && h1.weights[0] == 1.0 && h1.counts[0] == 1);
    RgbImage img(2, 2);
    img.pixels = {RgbColor{0, 0, 0}, RgbColor{0, 0, 0}, RgbColor{255, 255, 255}, RgbColor{0, 0, 0}};
    const ColorHistogram h = build_histogram(img);
    REQUIRE(h.size() == 2);
    REQUIRE((h.colors[0] == Vec3{0, 0, 0}));
    REQUIRE(h.weights[0] == 0.75 && h.weights[1] == 0.25);
    REQUIRE(h.counts[0] + h.counts[1] == 4);
    std::printf("histogram known answers\n");
  }
  // histogram_test.cpp:63-97 — invariants; permutation keeps the multiset
  {
    RgbImage img = noise_image(40, 40, 60, 23);
    const ColorHistogram a = build_histogram(img);
    std::uint64_t total = 0;
    for (auto c : a.counts) total += c;
    REQUIRE(total == img.size());
    std::set<std::array<double, 3>> seen(a.colors.begin(), a.colors.end());
    REQUIRE(seen.size() == a.size());
    std::mt19937_64 rng(3);
    std::shuffle(img.pixels.begin(), img.pixels.end(), rng);
    const ColorHistogram b = build_histogram(img);
    std::map<std::array<double, 3>, std::uint32_t> ma, mb;
    for (std::size_t i = 0; i < a.size(); ++i) ma[a.colors[i]] = a.counts[i];
    for (std::size_t i = 0; i < b.size(); ++i) mb[b.colors[i]] = b.counts[i];
    REQUIRE(ma == mb);
    std::printf("histogram invariants\n");
  }
  // kmeans_test.cpp:242-248 — k = N' reaches zero SSE in one iteration
  {
    const RgbImage img = noise_image(16, 16, 12, 3);
    const ColorHistogram hist = build_histogram(img);
    const auto res = run_wsm(hist, int(hist.size()), Termination::convergent(), 1);
    REQUIRE(res.report.iterations == 1);
    REQUIRE(res.report.sse == 0.0);
    std::printf("k = N' converges in one iteration\n");
  }
  // kmeans_test.cpp:250-257 — SSE history nonincreasing, fixed budget honoured
  {
    const RgbImage img = noise_image(64, 64, 500, 15);
    const auto res = run_wsm(build_histogram(img), 16, Termination::fixed(12), 4);
    REQUIRE(res.report.iterations == 12);
    for (std::size_t i = 1; i < res.report.sse_history.size(); ++i)
      REQUIRE(res.report.sse_history[i] <= res.report.sse_history[i - 1] + 1e-9);
    std::printf("sse history nonincreasing\n");
  }
  // kmeans_test.cpp:102-111 analogue — k = 1: N' point evals, 0 pair evals per iteration
  {
    const RgbImage img = noise_image(8, 8, 40, 5);
    const ColorHistogram hist = build_histogram(img);
    const auto res = run_wsm(hist, 1, Termination::fixed(1), 1);
    REQUIRE(res.report.dist_evals == hist.size());
    std::printf("k = 1 evaluates each sample once\n");
  }
  // kmeans.hpp:54-56 / cli_test.cpp:142-151 — k > N' is an invalid argument
  {
    const RgbImage img = noise_image(4, 4, 3, 9);
    const ColorHistogram hist = build_histogram(img);
    REQUIRE(throws<std::invalid_argument>([&] { run_wsm(hist, int(hist.size()) + 1, Termination::fixed(3), 1); }));
    MethodParams mp;
    mp.id = MethodId::WsmC;
    REQUIRE(throws<std::invalid_argument>([&] { generate_palette(img, mp, 64, 1); }));
    REQUIRE(throws<std::invalid_argument>([&] { generate_palette(img, mp, 0, 1); }));
    REQUIRE(throws<std::invalid_argument>([&] { Termination::convergent(0.0); }));
    std::printf("argument errors\n");
  }
  // imageio_test.cpp:91-105,135-148 — map_pixels properties
  {
    const RgbImage img = noise_image(16, 16, 30, 3);
    Palette black;
    black.centers.push_back(Vec3{0, 0, 0});
    for (const auto& px : map_pixels(img, black).pixels) REQUIRE((px == RgbColor{0, 0, 0}));
    const RgbImage pal_img = noise_image(24, 24, 12, 5);
    Palette exact;
    exact.centers = build_histogram(pal_img).colors;
    REQUIRE(map_pixels(pal_img, exact) == pal_img);
    std::mt19937_64 rng(13);
    std::uniform_real_distribution<double> ch(0.0, 255.0);
    Palette p;
    for (int i = 0; i < 9; ++i) p.centers.push_back(Vec3{ch(rng), ch(rng), ch(rng)});
    const RgbImage once = map_pixels(img, p);
    REQUIRE(map_pixels(once, p) == once);
    REQUIRE(throws<std::invalid_argument>([&] { map_pixels(img, Palette{}); }));
    std::printf("map_pixels properties\n");
  }
  // metrics_test.cpp:14-24 — mse known answers
  {
    const RgbImage black(8, 8, RgbColor{0, 0, 0}), white(8, 8, RgbColor{255, 255, 255});
    REQUIRE(mse(black, white) == 195075.0);
    REQUIRE(mse(black, black) == 0.0);
    REQUIRE(throws<std::invalid_argument>([&] { mse(black, RgbImage(4, 4)); }));
    std::printf("mse known answers\n");
  }
  // cli_test.cpp:123-140 — deterministic; wsm-c MSE <= wsm MSE; quantize consistent
  {
    const RgbImage img = noise_image(64, 48, 2000, 77);
    MethodParams a;
    a.id = MethodId::Wsm;
    MethodParams c;
    c.id = MethodId::WsmC;
    const auto q1 = generate_palette(img, c, 16, 1), q2 = generate_palette(img, c, 16, 1);
    REQUIRE(q1.palette.centers == q2.palette.centers);
    const auto qa = generate_palette(img, a, 16, 1);
    REQUIRE(mse(img, map_pixels(img, q1.palette)) <= mse(img, map_pixels(img, qa.palette)));
    const auto fused = quantize(img, 16, c.termination(), 1);
    REQUIRE(fused.palette.centers == q1.palette.centers);
    REQUIRE(fused.mapped == map_pixels(img, q1.palette));
    REQUIRE(fused.report.mse == mse(img, fused.mapped));
    const auto rounded = round_palette(fused.palette);
    for (std::size_t i = 0; i < img.size(); ++i) REQUIRE(rounded[fused.index_map[i]] == fused.mapped.pixels[i]);
    std::printf("quantize determinism and fusion\n");
  }
  // ---- the point-set API (kmeans_test.cpp:24-240), real-valued points
  struct Pts {
    std::vector<Vec3> x;
    std::vector<double> w;
  };
  auto uniform_pts = [](std::size_t n, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 255.0), wd(0.05, 1.0);
    Pts p;
    double tot = 0;
    for (std::size_t i = 0; i < n; ++i) {
      p.x.push_back(Vec3{u(rng), u(rng), u(rng)});
      p.w.push_back(wd(rng));
      tot += p.w.back();
    }
    for (double& v : p.w) v /= tot;
    return p;
  };
  auto blob_pts = [](std::size_t n, int blobs, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(20.0, 235.0);
    std::normal_distribution<double> nd(0.0, 6.0);
    std::vector<Vec3> c;
    for (int b = 0; b < blobs; ++b) c.push_back(Vec3{u(rng), u(rng), u(rng)});
    Pts p;
    for (std::size_t i = 0; i < n; ++i) {
      const Vec3& m = c[rng() % c.size()];
      p.x.push_back(Vec3{m[0] + nd(rng), m[1] + nd(rng), m[2] + nd(rng)});
      p.w.push_back(1.0 / double(n));
    }
    return p;
  };
  {  // init_centers: k distinct input points, deterministic, k > n throws
    const Pts p = uniform_pts(10, 7);
    const Palette all = init_centers(p.x, 10, 123);
    std::set<Vec3> got(all.centers.begin(), all.centers.end()), src(p.x.begin(), p.x.end());
    REQUIRE(got.size() == 10 && got == src);
    REQUIRE(init_centers(p.x, 3, 99).centers == init_centers(p.x, 3, 99).centers);
    REQUIRE(throws<std::invalid_argument>([&] { init_centers(p.x, 11, 1); }));
    std::printf("init_centers (points)\n");
  }
  {  // assign_naive: one center; own centers; equidistant -> lowest index
    const Pts p = uniform_pts(50, 3);
    Palette single;
    single.centers.push_back(Vec3{1, 2, 3});
    Memberships m;
    assign_naive(p.x, p.w, single, m);
    for (auto v : m) REQUIRE(v == 0);
    Palette own;
    own.centers = {Vec3{0, 0, 0}, Vec3{100, 0, 0}, Vec3{0, 100, 0}};
    std::vector<double> w3(3, 1.0 / 3);
    assign_naive(own.centers, w3, own, m);
    REQUIRE((m == Memberships{0, 1, 2}));
    Palette six;
    for (int i = 0; i < 6; ++i) six.centers.push_back(Vec3{double(1000 + i * 1000), 0, 0});
    six.centers[2] = Vec3{10, 0, 0};
    six.centers[5] = Vec3{30, 0, 0};
    std::vector<Vec3> probe{Vec3{20, 0, 0}};
    std::vector<double> pw{1.0};
    assign_naive(probe, pw, six, m);
    REQUIRE(m[0] == 2);
    std::printf("assign_naive ties\n");
  }
  {  // sort-means: the break at d == 4 prev evaluates only prev; k = 1
    std::vector<Vec3> x{Vec3{1, 0, 0}};
    std::vector<double> w{1.0};
    Palette pal;
    pal.centers = {Vec3{0, 0, 0}, Vec3{2, 0, 0}};
    ClusterState st;
    st.memberships = {0};
    st.update_center_tables(pal);
    REQUIRE(st.d(0, 1) == 4.0);
    const AssignResult r = assign_sort_means(x, w, pal, st);
    REQUIRE(st.memberships[0] == 0 && r.dist_evals == 1 && r.weighted_sse == 1.0);
    const Pts p = uniform_pts(64, 5);
    Palette one;
    one.centers.push_back(Vec3{10, 20, 30});
    ClusterState s1;
    s1.memberships.assign(p.x.size(), 0);
    s1.update_center_tables(one);
    REQUIRE(assign_sort_means(p.x, p.w, one, s1).dist_evals == p.x.size());
    std::printf("sort-means boundary and k = 1\n");
  }
  {  // sort-means = exhaustive through 20 iterations; audited skips are valid
    const Pts p = blob_pts(1000, 10, 31);
    const int k = 16;
    Palette pal = init_centers(p.x, k, 77);
    ClusterState st;
    assign_naive(p.x, p.w, pal, st.memberships);
    std::uint64_t audited = 0;
    for (int iter = 0; iter < 20; ++iter) {
      pal = update_centers(p.x, p.w, st.memberships, pal);
      st.update_center_tables(pal);
      const SkipAudit audit = [&](std::size_t i, int prev_c, int first_rank, double prev_dist) {
        const auto* order = st.order_row(prev_c);
        for (int r = first_rank; r < k; ++r) {
          REQUIRE(dist2(p.x[i], pal[std::size_t(order[r])]) >= prev_dist * (1.0 - 1e-12));
          ++audited;
        }
      };
      const AssignResult fast = assign_sort_means(p.x, p.w, pal, st, &audit);
      Memberships ref;
      const AssignResult slow = assign_naive(p.x, p.w, pal, ref);
      REQUIRE(st.memberships == ref);
      REQUIRE(std::abs(fast.weighted_sse - slow.weighted_sse) <= 1e-12 * slow.weighted_sse);
      REQUIRE(fast.dist_evals <= slow.dist_evals);
      REQUIRE(std::abs(weighted_sse(p.x, p.w, pal, st.memberships) - slow.weighted_sse) <= 1e-12 * slow.weighted_sse);
    }
    REQUIRE(audited > 0);
    std::printf("sort-means equals exhaustive (20 iterations, audit)\n");
  }
  {  // center tables: symmetric, zero diagonal, self-first sorted permutation rows
    const Pts p = uniform_pts(40, 8);
    const Palette pal = init_centers(p.x, 12, 3);
    ClusterState st;
    std::uint64_t pairs = 0;
    st.update_center_tables(pal, &pairs);
    REQUIRE(pairs == 66);
    for (int i = 0; i < 12; ++i) {
      REQUIRE(st.d(i, i) == 0.0);
      for (int j = 0; j < 12; ++j) REQUIRE(st.d(i, j) == st.d(j, i));
      const auto* row = st.order_row(i);
      REQUIRE(row[0] == i);
      REQUIRE(std::set<int>(row, row + 12).size() == 12);
      for (int j = 2; j < 12; ++j) REQUIRE(st.d(i, row[j - 1]) <= st.d(i, row[j]));
    }
    Palette moved = pal;
    moved[3] = Vec3{1, 2, 3};
    st.update_center_tables(moved, &pairs);
    REQUIRE(pairs == 66 + 11);  // only the pairs of the moved center
    std::printf("center tables\n");
  }
  {  // update_centers: weighted means; an empty cluster re-seeded at the farthest point
    std::vector<Vec3> x{Vec3{0, 0, 0}, Vec3{255, 255, 255}};
    Palette prev;
    prev.centers.push_back(Vec3{1, 1, 1});
    Memberships m{0, 0};
    const Palette next = update_centers(x, std::vector<double>{0.75, 0.25}, m, prev);
    REQUIRE(std::abs(next[0][0] - 63.75) <= 1e-12 * 63.75);
    REQUIRE((update_centers(x, std::vector<double>{0.5, 0.5}, m, prev)[0] == Vec3{127.5, 127.5, 127.5}));
    std::vector<Vec3> y{Vec3{0, 0, 0}, Vec3{10, 0, 0}, Vec3{200, 0, 0}};
    Palette p2;
    p2.centers = {Vec3{5, 0, 0}, Vec3{999, 999, 999}};
    const Palette r2 = update_centers(y, std::vector<double>{0.3, 0.3, 0.4}, Memberships{0, 0, 0}, p2);
    REQUIRE((r2[1] == Vec3{200, 0, 0}));
    std::printf("update_centers means and reseed\n");
  }
  {  // run_wsm_points: deterministic, SSE nonincreasing; run_wsm on a
     // real-valued histogram takes the same point path
    const Pts p = blob_pts(3000, 12, 9);
    const auto a = run_wsm_points(p.x, p.w, 12, Termination::convergent(1e-4, 100), 5);
    const auto b = run_wsm_points(p.x, p.w, 12, Termination::convergent(1e-4, 100), 5);
    REQUIRE(a.palette.centers == b.palette.centers && a.report.iterations == b.report.iterations);
    for (std::size_t i = 1; i < a.report.sse_history.size(); ++i)
      REQUIRE(a.report.sse_history[i] <= a.report.sse_history[i - 1] * (1 + 1e-12));
    ColorHistogram h;
    h.colors = p.x;
    h.weights = p.w;
    h.total_pixels = p.x.size();
    const auto c = run_wsm(h, 12, Termination::convergent(1e-4, 100), 5);
    REQUIRE(c.palette.centers == a.palette.centers && c.report.dist_evals == a.report.dist_evals);
    const auto big = run_wsm_points(p.x, p.w, 300, Termination::fixed(3), 2);  // k > 256
    REQUIRE(big.palette.size() == 300 && big.report.iterations == 3);
    std::printf("run_wsm_points and the real-valued histogram path\n");
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAIL" : "PASS", g_fail);
  return g_fail;
}
