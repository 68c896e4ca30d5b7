// colorq_b200: the `quantize` command of the reference CLI (tools/colorq.cpp:
// 71-119) on the B200 library — binary PPM in, quantized PPM out, optional
// palette text, error image and histogram CSV, one summary line on stdout.
//
//   colorq_b200 quantize INPUT.ppm -o OUT.ppm [-m wsm|wsm-c] [-k K] [-s SEED]
//               [--palette P.txt] [--error-image E.ppm] [--dump-histogram H.csv]
//               [--iters N] [--epsilon E]
//   colorq_b200 bench [-c CONFIG] [--images A,B] [--methods M1,M2] [--k-values K1,K2]
//               [--runs N] [--base-seed S] [--output PREFIX] [--threads T] [--serial-timing]
//   colorq_b200 scaling INPUT.ppm [-m METHOD] [--k-values K1,K2] [-s SEED] [-o OUT.csv]
//
// bench / scaling are tools/colorq.cpp:121-200 over include/colorq_b200/bench.hpp
// (SURVEY.md §8(f) row f2).
//
// Exit codes follow the reference (tools/colorq.cpp:21-43): 2 I/O or PPM
// error, 3 unknown / unsupported method, 4 invalid parameters. The WSM, KM and
// FKM methods are provided; the reference's other method names exit with 3.
// Argument parsing is hand-written (the reference uses CLI11).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "colorq_b200/bench.hpp"
#include "colorq_b200/colorq.hpp"
#include "colorq_b200/io.hpp"

namespace {

constexpr int kExitIo = 2;
constexpr int kExitBadMethod = 3;
constexpr int kExitBadParams = 4;

struct UsageError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

int usage(const char* msg) {
  std::cerr << "error: " << msg << "\n"
            << "usage: colorq_b200 quantize INPUT.ppm -o OUT.ppm [-m wsm|wsm-c] [-k K] [-s SEED]\n"
            << "                   [--palette P.txt] [--error-image E.ppm] [--dump-histogram H.csv]\n"
            << "                   [--iters N] [--epsilon E]\n"
            << "       colorq_b200 bench [-c CONFIG] [--images ...] [--methods ...] [--k-values ...] [--runs N]\n"
            << "                   [--base-seed S] [--output PREFIX] [--threads T] [--serial-timing]\n"
            << "       colorq_b200 scaling INPUT.ppm [-m METHOD] [--k-values ...] [-s SEED] [-o OUT.csv]\n";
  return 1;
}

struct Args {
  std::string input, output, method = "wsm", palette, error_image, hist_csv;
  int k = 256;
  std::uint64_t seed = 1;
  int iters = -1;
  double epsilon = -1;
};

template <typename F>
int guarded(F&& body) {
  try {
    return body();
  } catch (const colorq::PpmError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitIo;
  } catch (const colorq::UnknownMethodError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitBadMethod;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitBadParams;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitIo;
  }
}

int quantize(const Args& a) {
  return guarded([&]() {
    const auto id = colorq::parse_method(a.method);
    if (!id) throw colorq::UnknownMethodError("unknown method: " + a.method);
    colorq::MethodParams mp;
    mp.id = *id;
    if (a.iters > 0) mp.iters = a.iters;
    if (a.epsilon > 0) mp.epsilon = a.epsilon;
    const bool km = mp.id == colorq::MethodId::Km || mp.id == colorq::MethodId::KmC ||
                    mp.id == colorq::MethodId::Fkm || mp.id == colorq::MethodId::FkmC;
    if (mp.id != colorq::MethodId::Wsm && mp.id != colorq::MethodId::WsmC && !km)
      throw colorq::UnknownMethodError("method '" + a.method + "' is not provided by the B200 path");

    const colorq::RgbImage image = colorq::load_ppm(a.input);
    if (a.k < 1) throw std::invalid_argument("k must be >= 1");  // methods.hpp:109, after the load as in the reference
    if (km) {  // run_km_full / run_fkm, then map / mse / error image as the reference CLI composes them
      colorq::QuantizeOutcome qo = colorq::generate_palette(image, mp, a.k, a.seed);
      const colorq::RgbImage mapped = colorq::map_pixels(image, qo.palette);
      qo.report.mse = colorq::mse(image, mapped);
      colorq::save_ppm(mapped, a.output);
      if (!a.palette.empty()) colorq::save_palette(qo.palette, a.palette);
      if (!a.error_image.empty()) colorq::save_ppm(colorq::error_image(image, mapped), a.error_image);
      if (!a.hist_csv.empty()) {
        std::ofstream out(a.hist_csv);
        if (!out) throw std::runtime_error("cannot open " + a.hist_csv + " for writing");
        colorq::write_histogram_csv(out, colorq::build_histogram(image));
      }
      std::printf("method=%s k=%d seed=%llu iterations=%d mse=%s psnr=%s time_ms=%s\n", qo.report.method.c_str(),
                  a.k, (unsigned long long)a.seed, qo.report.iterations, colorq::fmt_g6(qo.report.mse).c_str(),
                  colorq::fmt_g6(colorq::psnr(qo.report.mse)).c_str(), colorq::fmt_g6(qo.report.elapsed_ms).c_str());
      return 0;
    }
    // generate_palette + map_pixels + mse + error_image in one device pass
    const colorq::Termination term = mp.termination();
    const cqb_termination t = colorq::b200::native(term);
    const int cap = colorq::b200::budget(term);
    std::vector<double> centers(3 * std::size_t(a.k)), hist(static_cast<std::size_t>(cap));
    colorq::RgbImage mapped(image.width, image.height);
    colorq::RgbImage err(image.width, image.height);
    cqb_report rep{};
    colorq::b200::check(cqb_quantize_ex(colorq::b200::context(), colorq::b200::bytes(image), image.width,
                                        image.height, a.k, &t, a.seed, centers.data(), hist.data(), cap, nullptr,
                                        reinterpret_cast<std::uint8_t*>(mapped.pixels.data()),
                                        a.error_image.empty() ? nullptr
                                                              : reinterpret_cast<std::uint8_t*>(err.pixels.data()),
                                        &rep));
    const colorq::Palette palette = colorq::b200::palette_from(centers.data(), a.k);

    colorq::save_ppm(mapped, a.output);
    if (!a.palette.empty()) colorq::save_palette(palette, a.palette);
    if (!a.error_image.empty()) colorq::save_ppm(err, a.error_image);
    if (!a.hist_csv.empty()) {
      std::ofstream out(a.hist_csv);
      if (!out) throw std::runtime_error("cannot open " + a.hist_csv + " for writing");
      colorq::write_histogram_csv(out, colorq::build_histogram(image));
    }
    std::printf("method=%s k=%d seed=%llu iterations=%d mse=%s psnr=%s time_ms=%s\n",
                mp.id == colorq::MethodId::WsmC ? "wsm-c" : "wsm", a.k, (unsigned long long)a.seed, rep.iterations,
                colorq::fmt_g6(rep.mse).c_str(), colorq::fmt_g6(colorq::psnr(rep.mse)).c_str(),
                colorq::fmt_g6(rep.elapsed_ms).c_str());  // palette generation, device time
    return 0;
  });
}

int env_threads() {
  if (const char* v = std::getenv("COLORQ_THREADS")) {
    const int n = std::atoi(v);
    if (n >= 1) return n;
  }
  return 1;
}

std::vector<int> parse_k_list(const std::string& s) {
  std::vector<int> ks;
  for (const std::string& t : colorq::bench::list_items(s)) ks.push_back(std::stoi(t));
  if (ks.empty()) throw std::invalid_argument("empty K list");
  return ks;
}

int bench_main(int argc, char** argv) {
  std::string config, images, methods, ks, output;
  int runs = -1, threads = -1;
  long long base_seed = -1;
  bool serial = false;
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string s = argv[i];
      auto value = [&](const char* name) -> std::string {
        if (i + 1 >= argc) throw UsageError(std::string("missing value for ") + name);
        return argv[++i];
      };
      if (s == "-c" || s == "--config") config = value("--config");
      else if (s == "--images") images = value("--images");
      else if (s == "--methods") methods = value("--methods");
      else if (s == "--k-values") ks = value("--k-values");
      else if (s == "--runs") runs = std::stoi(value("--runs"));
      else if (s == "--base-seed") base_seed = std::stoll(value("--base-seed"));
      else if (s == "--output") output = value("--output");
      else if (s == "--threads") threads = std::stoi(value("--threads"));
      else if (s == "--serial-timing") serial = true;
      else throw UsageError("unknown option " + s);
    }
  } catch (const std::exception& e) {
    return usage(e.what());
  }
  return guarded([&]() {
    colorq::bench::Plan plan;
    plan.threads = env_threads();
    if (!config.empty()) {
      std::ifstream in(config);
      if (!in) throw std::runtime_error("cannot open config file " + config);
      colorq::bench::read_plan(plan, in);
    }
    if (!images.empty()) plan.images = colorq::bench::list_items(images);
    if (!methods.empty()) {
      plan.methods.clear();
      for (const std::string& t : colorq::bench::list_items(methods))
        plan.methods.push_back(colorq::bench::parse_method_token(t));
    }
    if (!ks.empty()) plan.ks = parse_k_list(ks);
    if (runs > 0) plan.runs = runs;
    if (base_seed >= 0) plan.base_seed = std::uint64_t(base_seed);
    if (!output.empty()) plan.prefix = output;
    if (threads > 0) plan.threads = threads;
    plan.serial = serial;
    const colorq::bench::Results res = colorq::bench::run(plan);
    for (const auto& p : colorq::bench::write_outputs(res, plan.prefix)) std::cout << "wrote " << p.string() << "\n";
    std::cout << res.ranks_csv;
    return 0;
  });
}

int scaling_main(int argc, char** argv) {
  std::string input, method = "wsm-c", ks = "2,4,8,16,32,64,128,256", output;
  std::uint64_t seed = 1;
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string s = argv[i];
      auto value = [&](const char* name) -> std::string {
        if (i + 1 >= argc) throw UsageError(std::string("missing value for ") + name);
        return argv[++i];
      };
      if (s == "-m" || s == "--method") method = value("--method");
      else if (s == "--k-values") ks = value("--k-values");
      else if (s == "-s" || s == "--seed") seed = std::stoull(value("--seed"));
      else if (s == "-o" || s == "--output") output = value("--output");
      else if (!s.empty() && s[0] == '-') throw UsageError("unknown option " + s);
      else if (input.empty()) input = s;
      else throw UsageError("unexpected argument " + s);
    }
  } catch (const std::exception& e) {
    return usage(e.what());
  }
  if (input.empty()) return usage("missing INPUT");
  return guarded([&]() {
    const colorq::bench::Method spec = colorq::bench::parse_method_token(method);
    const std::vector<int> kv = parse_k_list(ks);
    const colorq::RgbImage image = colorq::load_ppm(input);
    std::string csv = "k,elapsed_ms,dist_evals\n";
    for (const int k : kv) {
      const colorq::QuantizeOutcome q = colorq::generate_palette(image, spec.params, k, seed);
      csv += std::to_string(k) + "," + colorq::fmt_g6(q.report.elapsed_ms) + "," + std::to_string(q.report.dist_evals) +
             "\n";
    }
    if (output.empty()) {
      std::cout << csv;
    } else {
      std::ofstream out(output);
      if (!out) throw std::runtime_error("cannot open " + output + " for writing");
      out << csv;
    }
    return 0;
  });
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && std::strcmp(argv[1], "bench") == 0) return bench_main(argc, argv);
  if (argc >= 2 && std::strcmp(argv[1], "scaling") == 0) return scaling_main(argc, argv);
  if (argc < 2 || std::strcmp(argv[1], "quantize") != 0) return usage("expected a subcommand: quantize, bench, scaling");
  Args a;
  bool have_out = false;
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string s = argv[i];
      auto value = [&](const char* name) -> std::string {
        if (i + 1 >= argc) throw UsageError(std::string("missing value for ") + name);
        return argv[++i];
      };
      if (s == "-o" || s == "--output") {
        a.output = value("--output");
        have_out = true;
      } else if (s == "-m" || s == "--method") {
        a.method = value("--method");
      } else if (s == "-k" || s == "--k") {
        a.k = std::stoi(value("--k"));
      } else if (s == "-s" || s == "--seed") {
        a.seed = std::stoull(value("--seed"));
      } else if (s == "--palette") {
        a.palette = value("--palette");
      } else if (s == "--error-image") {
        a.error_image = value("--error-image");
      } else if (s == "--dump-histogram") {
        a.hist_csv = value("--dump-histogram");
      } else if (s == "--iters") {
        a.iters = std::stoi(value("--iters"));
      } else if (s == "--epsilon") {
        a.epsilon = std::stod(value("--epsilon"));
      } else if (!s.empty() && s[0] == '-') {
        throw UsageError("unknown option " + s);
      } else if (a.input.empty()) {
        a.input = s;
      } else {
        throw UsageError("unexpected argument " + s);
      }
    }
  } catch (const std::exception& e) {
    return usage(e.what());
  }
  if (a.input.empty()) return usage("missing INPUT");
  if (!have_out) return usage("--output is required");
  return quantize(a);
}
