// gb_gen_bal — standalone writer of the synthetic BAL-shaped problems
// (synth.cpp) for the two bench arms.
//
// Both bench arms read the problem from this executable instead of
// generating it in-process, so the reference arm's python process loads only
// the oracle library (oracle/_ref/libgopt_ref.so) and never the product
// library. Host-only: no CUDA, no GPU.
//
//   gb_gen_bal NC NP NE [--seed S] [--stride K] [--zipf Z] [--text]
//
// Default output (stdout) is binary:
//   char[8] "GBBAL01\0"; uint64 nc, np, ne;
//   uint32 camera_index[ne]; uint32 point_index[ne]; double observed[2 ne];
//   double cameras[9 nc]; double points[3 np]            (little endian)
// --text writes the BAL text format with %.17g values exactly as the
// reference's serializer does (src/bal_problem.cpp:121-136), so the
// reference's own parse_bal_text (src/bal_problem.cpp:81-115) reads it back
// bit-identically.

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gb_bal.h"

namespace {

void put(const void* p, size_t bytes) {
  const char* c = static_cast<const char*>(p);
  while (bytes) {
    const size_t n = std::fwrite(c, 1, bytes, stdout);
    if (n == 0) {
      std::perror("gb_gen_bal: write");
      std::exit(3);
    }
    c += n;
    bytes -= n;
  }
}

int usage() {
  std::fprintf(stderr, "usage: gb_gen_bal NC NP NE [--seed S] [--stride K] [--zipf Z] [--text]\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) return usage();
  const uint64_t nc = std::strtoull(argv[1], nullptr, 10);
  const uint64_t np = std::strtoull(argv[2], nullptr, 10);
  const uint64_t ne = std::strtoull(argv[3], nullptr, 10);
  uint64_t seed = 42, stride = 0;
  double zipf = 0;
  bool text = false;
  for (int i = 4; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--text") {
      text = true;
    } else if (i + 1 < argc && a == "--seed") {
      seed = std::strtoull(argv[++i], nullptr, 10);
    } else if (i + 1 < argc && a == "--stride") {
      stride = std::strtoull(argv[++i], nullptr, 10);
    } else if (i + 1 < argc && a == "--zipf") {
      zipf = std::strtod(argv[++i], nullptr);
    } else {
      return usage();
    }
  }
  std::vector<uint32_t> cam(ne), pt(ne);
  std::vector<double> obs(2 * ne), cams(9 * nc), pts(3 * np);
  if (gb_synthetic_bal(nc, np, ne, seed, stride, zipf, cam.data(), pt.data(), obs.data(), cams.data(),
                       pts.data()) != GB_OK) {
    std::fprintf(stderr, "gb_gen_bal: invalid shape (need observations >= points and degree <= cameras)\n");
    return 1;
  }
  static char buf[1 << 20];
  std::setvbuf(stdout, buf, _IOFBF, sizeof(buf));
  if (text) {
    std::printf("%llu %llu %llu\n", static_cast<unsigned long long>(nc), static_cast<unsigned long long>(np),
                static_cast<unsigned long long>(ne));
    for (uint64_t i = 0; i < ne; ++i)
      std::printf("%u %u %.17g %.17g\n", cam[i], pt[i], obs[2 * i], obs[2 * i + 1]);
    for (double v : cams) std::printf("%.17g\n", v);
    for (double v : pts) std::printf("%.17g\n", v);
  } else {
    const char magic[8] = {'G', 'B', 'B', 'A', 'L', '0', '1', '\0'};
    const uint64_t hdr[3] = {nc, np, ne};
    put(magic, sizeof(magic));
    put(hdr, sizeof(hdr));
    put(cam.data(), ne * sizeof(uint32_t));
    put(pt.data(), ne * sizeof(uint32_t));
    put(obs.data(), obs.size() * sizeof(double));
    put(cams.data(), cams.size() * sizeof(double));
    put(pts.data(), pts.size() * sizeof(double));
  }
  if (std::fflush(stdout) != 0) return 3;
  return 0;
}
