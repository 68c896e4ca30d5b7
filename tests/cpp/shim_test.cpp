// Drop-in shim test: the reference's own hot-path unit-test cases
// (histogram_test.cpp, kmeans_test.cpp, imageio_test.cpp, metrics_test.cpp,
// cli_test.cpp:142-151), restated against include/colorq_b200/colorq.hpp and
// therefore executed on the B200 through the C ABI. Prints one line per case;
// exit code = number of failures. Run by tests/test_gpu_parity.py.
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
  std::printf("%s (%d failures)\n", g_fail ? "FAIL" : "PASS", g_fail);
  return g_fail;
}
