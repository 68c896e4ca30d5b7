// Host-side file formats and CLI helpers of the drop-in (SURVEY.md §8(f) row
// f1), written for this library. The behaviour and byte formats are those of
// the reference:
//   * binary PPM codec: ppm.hpp:89-149 (P6, maxval 255, '#' comments in the
//     header, one whitespace byte before the payload; errors typed BadMagic /
//     BadHeader / BadMaxval / Truncated);
//   * palette text: palette.hpp:37-74 ("%.10g %.10g %.10g\n" per center);
//   * error_image: image_ops.hpp:55-71, on the device (cqb_error_image);
//   * psnr: metrics.hpp:32-36; fmt_g6: report.hpp:13-17;
//   * write_histogram_csv: histogram.hpp:111-117; parse_method: methods.hpp:48-58.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <optional>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "colorq.hpp"

namespace colorq {

struct PpmError : std::runtime_error {
  enum class Kind { BadMagic, BadHeader, BadMaxval, Truncated };
  PpmError(Kind k, const std::string& msg) : std::runtime_error(msg), kind(k) {}
  Kind kind;
};

namespace io_detail {

inline bool ppm_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

// Header cursor: whitespace and '#'-to-end-of-line comments separate tokens.
struct HeaderCursor {
  std::span<const unsigned char> in;
  std::size_t at = 0;

  void skip() {
    for (;;) {
      while (at < in.size() && ppm_space(in[at])) ++at;
      if (at < in.size() && in[at] == '#') {
        while (at < in.size() && in[at] != '\n') ++at;
        continue;
      }
      return;
    }
  }
  std::string token() {
    skip();
    const std::size_t b = at;
    while (at < in.size() && !ppm_space(in[at])) ++at;
    if (at == b) throw PpmError(PpmError::Kind::BadHeader, "unexpected end of PPM header");
    return std::string(reinterpret_cast<const char*>(in.data() + b), at - b);
  }
  int positive(const char* field) {
    const std::string t = token();
    bool ok = !t.empty();
    long long v = 0;
    std::size_t i = 0;
    if (ok && (t[0] == '+' || t[0] == '-')) i = 1;
    ok = ok && i < t.size();
    for (; ok && i < t.size(); ++i) {
      if (t[i] < '0' || t[i] > '9') ok = false;
      else if ((v = v * 10 + (t[i] - '0')) > (1ll << 32)) ok = false;  // std::stoi would overflow
    }
    if (ok && t[0] == '-') v = -v;
    if (!ok || v <= 0 || v > std::numeric_limits<int>::max())
      throw PpmError(PpmError::Kind::BadHeader, std::string("invalid ") + field + " in PPM header: '" + t + "'");
    return int(v);
  }
};

}  // namespace io_detail

inline RgbImage read_ppm(std::span<const unsigned char> bytes) {
  io_detail::HeaderCursor cur{bytes};
  std::string magic;
  try {
    magic = cur.token();
  } catch (const PpmError&) {
    throw PpmError(PpmError::Kind::BadMagic, "not a PPM file: empty input");
  }
  if (magic != "P6")
    throw PpmError(PpmError::Kind::BadMagic, "not a binary PPM: expected magic 'P6', got '" + magic + "'");
  const int w = cur.positive("width");
  const int h = cur.positive("height");
  const int maxval = cur.positive("maxval");
  if (maxval != 255)
    throw PpmError(PpmError::Kind::BadMaxval, "unsupported maxval " + std::to_string(maxval) + " (only 255)");
  if (cur.at >= bytes.size() || !io_detail::ppm_space(bytes[cur.at]))
    throw PpmError(PpmError::Kind::BadHeader, "missing separator before PPM pixel data");
  ++cur.at;
  const std::size_t need = std::size_t(w) * std::size_t(h) * 3;
  const std::size_t have = bytes.size() - cur.at;
  if (have < need)
    throw PpmError(PpmError::Kind::Truncated, "truncated PPM pixel data: need " + std::to_string(need) +
                                                   " bytes, have " + std::to_string(have));
  RgbImage img(w, h);
  std::memcpy(img.pixels.data(), bytes.data() + cur.at, need);
  return img;
}

namespace io_detail {

// Whole-file reads and writes over C stdio (one fread / fwrite of the payload).
inline std::vector<unsigned char> slurp(const std::filesystem::path& path, const char* mode) {
  std::FILE* f = std::fopen(path.c_str(), mode);
  if (!f) throw std::runtime_error("cannot open " + path.string());
  std::vector<unsigned char> bytes;
  unsigned char chunk[1 << 16];
  for (std::size_t n; (n = std::fread(chunk, 1, sizeof chunk, f)) > 0;) bytes.insert(bytes.end(), chunk, chunk + n);
  std::fclose(f);
  return bytes;
}

inline void spill(const std::filesystem::path& path, const char* mode, const void* data, std::size_t n) {
  std::FILE* f = std::fopen(path.c_str(), mode);
  if (!f) throw std::runtime_error("cannot open " + path.string() + " for writing");
  const bool ok = std::fwrite(data, 1, n, f) == n;
  if (std::fclose(f) != 0 || !ok) throw std::runtime_error("write failed: " + path.string());
}

// One palette line: three stream-extracted doubles (the reference's reader accepts what
// operator>> accepts and ignores anything after the third value).
inline bool parse_center(std::string_view line, Vec3& c) {
  std::istringstream ls{std::string(line)};
  return bool(ls >> c[0] >> c[1] >> c[2]);
}

}  // namespace io_detail

// "P6\n<w> <h>\n255\n" then the raw RGB bytes.
inline std::vector<unsigned char> write_ppm(const RgbImage& img) {
  char head[64];
  const int hn = std::snprintf(head, sizeof head, "P6\n%d %d\n255\n", img.width, img.height);
  std::vector<unsigned char> out(std::size_t(hn) + img.size() * 3);
  std::memcpy(out.data(), head, std::size_t(hn));
  std::memcpy(out.data() + hn, img.pixels.data(), img.size() * 3);
  return out;
}

inline RgbImage load_ppm(const std::filesystem::path& path) { return read_ppm(io_detail::slurp(path, "rb")); }

inline void save_ppm(const RgbImage& img, const std::filesystem::path& path) {
  const std::vector<unsigned char> bytes = write_ppm(img);
  io_detail::spill(path, "wb", bytes.data(), bytes.size());
}

// One "%.10g %.10g %.10g" line per center, in palette-index order.
inline std::string palette_to_text(const Palette& p) {
  std::string s(p.centers.size() * 96, '\0');
  std::size_t at = 0;
  for (const Vec3& c : p.centers)
    at += std::size_t(std::snprintf(s.data() + at, 96, "%.10g %.10g %.10g\n", c[0], c[1], c[2]));
  s.resize(at);
  return s;
}

// Inverse of palette_to_text: newline-separated lines, empty lines skipped, a line
// without three numbers is an error.
inline Palette palette_from_text(const std::string& text) {
  Palette p;
  const std::string_view all(text);
  for (std::size_t b = 0; b < all.size();) {
    std::size_t e = all.find('\n', b);
    if (e == std::string_view::npos) e = all.size();
    const std::string_view line = all.substr(b, e - b);
    b = e + 1;
    if (line.empty()) continue;
    Vec3 c{};
    if (!io_detail::parse_center(line, c))
      throw std::runtime_error("malformed palette line: '" + std::string(line) + "'");
    p.centers.push_back(c);
  }
  return p;
}

inline void save_palette(const Palette& p, const std::filesystem::path& path) {
  const std::string text = palette_to_text(p);
  io_detail::spill(path, "w", text.data(), text.size());
}

inline Palette load_palette(const std::filesystem::path& path) {
  const std::vector<unsigned char> bytes = io_detail::slurp(path, "r");
  return palette_from_text(std::string(bytes.begin(), bytes.end()));
}

// 255 - min(255, 4|orig - quant|) per channel, computed on the device.
inline RgbImage error_image(const RgbImage& original, const RgbImage& quantized) {
  if (original.width != quantized.width || original.height != quantized.height)
    throw std::invalid_argument("error_image: dimension mismatch");
  RgbImage out(original.width, original.height);
  if (original.size() == 0) return out;
  b200::check(cqb_error_image(b200::context(), b200::bytes(original), b200::bytes(quantized), original.size(),
                              reinterpret_cast<std::uint8_t*>(out.pixels.data())));
  return out;
}

inline double psnr(double mse_value) {
  if (mse_value < 0) throw std::invalid_argument("psnr: negative MSE");
  if (mse_value == 0) return std::numeric_limits<double>::infinity();
  return 20.0 * std::log10(255.0 / std::sqrt(mse_value));
}

inline std::string fmt_g6(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.6g", v);
  return buf;
}

inline void write_histogram_csv(std::ostream& out, const ColorHistogram& h) {
  out << "r,g,b,count\n";
  for (std::size_t i = 0; i < h.counts.size(); ++i)
    out << int(h.colors[i][0]) << ',' << int(h.colors[i][1]) << ',' << int(h.colors[i][2]) << ',' << h.counts[i]
        << '\n';
}

// The reference's method names; only wsm / wsm-c are provided by this library
// (the others parse, and generate_palette raises UnknownMethodError for them).
inline std::optional<MethodId> parse_method(const std::string& s) {
  static const std::pair<const char*, MethodId> names[] = {
      {"mc", MethodId::Mc},     {"wan", MethodId::Wan}, {"wu", MethodId::Wu},     {"mmm", MethodId::Mmm},
      {"fcm", MethodId::Fcm},   {"pim", MethodId::Pim}, {"km", MethodId::Km},     {"km-c", MethodId::KmC},
      {"fkm", MethodId::Fkm},   {"fkm-c", MethodId::FkmC}, {"skm", MethodId::Skm}, {"wsm", MethodId::Wsm},
      {"wsm-c", MethodId::WsmC}};
  for (const auto& [n, id] : names)
    if (s == n) return id;
  return std::nullopt;
}

}  // namespace colorq
