// Host-only driver for the PPM / palette codecs of include/colorq_b200/io.hpp
// (tests/test_io_cpu.py compares its output with the reference's codecs):
//   io_test ppm IN OUT      read IN, write it back to OUT; prints "ok W H" or "err KIND message"
//   io_test palette IN OUT  parse palette text IN, print it back to OUT; "ok K" or "err runtime message"
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "colorq_b200/io.hpp"

int main(int argc, char** argv) {
  if (argc != 4) return 1;
  const std::string mode = argv[1];
  try {
    if (mode == "ppm") {
      const colorq::RgbImage img = colorq::load_ppm(argv[2]);
      colorq::save_ppm(img, argv[3]);
      std::printf("ok %d %d\n", img.width, img.height);
    } else if (mode == "palette") {
      const colorq::Palette p = colorq::load_palette(argv[2]);
      colorq::save_palette(p, argv[3]);
      std::printf("ok %zu\n", p.size());
    } else {
      return 1;
    }
  } catch (const colorq::PpmError& e) {
    static const char* kinds[] = {"BadMagic", "BadHeader", "BadMaxval", "Truncated"};
    std::printf("err %s %s\n", kinds[int(e.kind)], e.what());
  } catch (const std::exception& e) {
    std::printf("err runtime %s\n", e.what());
  }
  return 0;
}
