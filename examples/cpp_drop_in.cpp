// examples/cpp_drop_in.cpp -- a reference-style C++ caller of the B200 path.
//
// Uses only include/lance/b200.hpp (the reference operator API by name) and
// the shared library; the only change from a reference caller
// (lance::lance_gemm, engines.hpp:492-536) is the namespace of the call.
//
//   g++ -std=c++20 -O2 -Iinclude examples/cpp_drop_in.cpp \
//       -Lpaper_2003_08646_b200/_build -llance_b200 -Wl,-rpath,$PWD/paper_2003_08646_b200/_build
//   ./cpp_drop_in N C H W K PAD SEED TILE_M
//
// Prints the reference CLI's line (lance_main.cpp:92-93):
//   output dims N OH OW K  checksum <fnv1a64 hex>
#include <cstdio>
#include <cstdlib>
#include <exception>

#include "lance/b200.hpp"

int main(int argc, char** argv) {
  if (argc != 9) {
    std::fprintf(stderr, "usage: %s N C H W K PAD SEED TILE_M\n", argv[0]);
    return 2;
  }
  lance::b200::ConvSpec spec;
  spec.n = std::atoi(argv[1]);
  spec.c = std::atoi(argv[2]);
  spec.h = std::atoi(argv[3]);
  spec.w = std::atoi(argv[4]);
  spec.k = std::atoi(argv[5]);
  spec.pad = std::atoi(argv[6]);
  const uint64_t seed = std::strtoull(argv[7], nullptr, 10);
  const int tile_m = std::atoi(argv[8]);
  lance::b200::LanceConfig cfg;
  cfg.bits_w = 8;
  cfg.bits_i = 8;
  cfg.granularity = lance::b200::Granularity::PerPosition;
  cfg.mode = lance::b200::LanceMode::Gemm;
  try {
    // x then w from one UniformSource stream (bench.hpp:129-133).
    lance::b200::Tensor4 x(spec.n, spec.h, spec.w, spec.c);
    lance::b200::FilterBank w(spec.k, 3, 3, spec.c);
    std::vector<float> s(x.data.size() + w.data.size());
    lance_uniform_fill(seed, s.data(), s.size());
    std::copy(s.begin(), s.begin() + x.data.size(), x.data.begin());
    std::copy(s.begin() + x.data.size(), s.end(), w.data.begin());
    const lance::b200::Tensor4 y = tile_m == 4 ? lance::b200::lance_gemm_f4(x, w, spec, cfg)
                                               : lance::b200::lance_gemm(x, w, spec, cfg);
    std::printf("output dims %d %d %d %d  checksum %llx\n", y.n, y.h, y.w, y.c,
                static_cast<unsigned long long>(lance_fnv1a64(y.data.data(), y.data.size())));
    return 0;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
