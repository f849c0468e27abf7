// oracle/ref_dropin_check.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The drop-in claim of include/lance/b200.hpp made concrete: one binary
// compiled against the UNMODIFIED reference headers (/root/reference/proj/
// include) that builds the reference's own lance::Tensor4 / lance::FilterBank /
// lance::ConvSpec / lance::LanceConfig, calls
//   lance::lance_gemm(x, w, spec, cfg)              (engines.hpp:492-536, CPU)
//   lance::b200::lance_gemm_any(x, w, spec, cfg)    (this repo, B200)
// on the same objects and compares the two lance::Tensor4 results byte for
// byte (Tensor4::operator==, tensor.hpp:55, plus a memcmp of the data).  The
// error path is compared too: for invalid specs / configs both sides must
// throw std::invalid_argument with the same message (engines.hpp:46-91,
// 496-499).
//
// Built by oracle/Makefile into oracle/_ref/ref_dropin_check (git-ignored,
// travels to the GPU box with the snapshot; /root/reference does not).
//   ref_dropin_check            run every case, exit 0 iff all match
//   ref_dropin_check --errors   only the validation cases (no device needed)
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "lance/engines.hpp"   // the reference (header-only; lance.hpp would pull in
                                // bench.hpp and its external json.hpp)
#include "lance/rng.hpp"
#include "lance/b200.hpp"      // this repo's host API over liblance_b200.so

namespace {

struct Case {
  int n, c, h, w, k, pad;
  int bits_w, bits_i;
  lance::Granularity gran;
  unsigned long long seed;
};

// Reference layer data exactly as bench.hpp:129-133 makes it.
void make_layer(const Case& cs, lance::Tensor4& x, lance::FilterBank& w) {
  x = lance::Tensor4(cs.n, cs.h, cs.w, cs.c);
  w = lance::FilterBank(cs.k, 3, 3, cs.c);
  lance::UniformSource src(cs.seed);
  src.fill(x.data);
  src.fill(w.data);
}

std::string what_of(auto&& fn) {
  try {
    fn();
  } catch (const std::invalid_argument& e) {
    return std::string("invalid_argument: ") + e.what();
  } catch (const std::exception& e) {
    return std::string("other: ") + e.what();
  }
  return "ok";
}

int run_errors() {
  int bad = 0;
  struct E {
    int n, c, h, w, k, pad, bw, bi;
    lance::Granularity g;
    lance::LanceMode mode;
  };
  const E es[] = {
      {1, 4, 8, 8, 4, 2, 8, 8, lance::Granularity::PerPosition, lance::LanceMode::Gemm},   // pad
      {1, 4, 1, 1, 4, 0, 8, 8, lance::Granularity::PerPosition, lance::LanceMode::Gemm},   // collapse
      {1, 4, 8, 8, 4, 1, 9, 8, lance::Granularity::PerPosition, lance::LanceMode::Gemm},   // bits
      {1, 4, 8, 8, 4, 1, 8, 8, lance::Granularity::PerTile, lance::LanceMode::Gemm},       // PerTile
      {1, 4, 8, 8, 4, 1, 32, 8, lance::Granularity::PerPosition, lance::LanceMode::Gemm},  // fp operand
      {1, 4, 8, 8, 4, 1, 8, 8, lance::Granularity::PerPosition, lance::LanceMode::Faithful},
  };
  for (const E& e : es) {
    lance::ConvSpec spec;
    spec.n = e.n, spec.c = e.c, spec.h = e.h, spec.w = e.w, spec.k = e.k, spec.pad = e.pad;
    lance::LanceConfig cfg;
    cfg.bits_w = e.bw, cfg.bits_i = e.bi, cfg.granularity = e.g, cfg.mode = e.mode;
    lance::Tensor4 x(e.n, e.h, e.w, e.c);
    lance::FilterBank w(e.k, 3, 3, e.c);
    const std::string r = what_of([&] { (void)lance::lance_gemm(x, w, spec, cfg); });
    const std::string b = what_of([&] { (void)lance::b200::lance_gemm_any(x, w, spec, cfg); });
    const bool same = r == b;
    bad += !same;
    std::printf("errors %s: reference \"%s\" / b200 \"%s\"\n", same ? "same" : "DIFFER", r.c_str(),
                b.c_str());
  }
  // Dims mismatch between tensor and spec (check_layer, engines.hpp:84-91).
  {
    lance::ConvSpec spec;
    spec.n = 1, spec.c = 4, spec.h = 8, spec.w = 8, spec.k = 4, spec.pad = 1;
    lance::LanceConfig cfg;
    cfg.granularity = lance::Granularity::PerPosition, cfg.mode = lance::LanceMode::Gemm;
    lance::Tensor4 x(1, 8, 8, 5);
    lance::FilterBank w(4, 3, 3, 4);
    const std::string r = what_of([&] { (void)lance::lance_gemm(x, w, spec, cfg); });
    const std::string b = what_of([&] { (void)lance::b200::lance_gemm_any(x, w, spec, cfg); });
    bad += r != b;
    std::printf("errors %s: reference \"%s\" / b200 \"%s\"\n", r == b ? "same" : "DIFFER", r.c_str(),
                b.c_str());
    lance::Tensor4 x2(1, 8, 8, 4);
    lance::FilterBank w2(4, 3, 3, 3);
    const std::string r2 = what_of([&] { (void)lance::lance_gemm(x2, w2, spec, cfg); });
    const std::string b2 = what_of([&] { (void)lance::b200::lance_gemm_any(x2, w2, spec, cfg); });
    bad += r2 != b2;
    std::printf("errors %s: reference \"%s\" / b200 \"%s\"\n", r2 == b2 ? "same" : "DIFFER", r2.c_str(),
                b2.c_str());
  }
  return bad;
}

int run_cases() {
  using G = lance::Granularity;
  const Case cases[] = {
      {1, 64, 32, 32, 64, 1, 8, 8, G::PerPosition, 42},     // BASELINE config 1
      {2, 3, 17, 13, 8, 1, 8, 8, G::PerPosition, 7},        // RGB, ragged
      {3, 16, 9, 9, 24, 0, 8, 8, G::PerPosition, 11},       // pad 0, odd output
      {2, 40, 12, 20, 33, 1, 6, 5, G::PerPosition, 13},     // odd K, 6/5-bit
      {2, 64, 16, 16, 32, 1, 8, 8, G::PerTensor, 17},       // PerTensor
      {2, 130, 10, 10, 48, 1, 7, 8, G::PerPosition, 19},    // C not a multiple of 32
      {8, 64, 56, 56, 64, 1, 8, 8, G::PerPosition, 42},     // ResNet-18 R64 (batch slice)
      {16, 128, 28, 28, 128, 1, 8, 8, G::PerPosition, 46},  // R128
      {16, 256, 14, 14, 256, 1, 8, 8, G::PerPosition, 49},  // R256
      {32, 512, 7, 7, 512, 1, 8, 8, G::PerPosition, 52},    // R512
  };
  int bad = 0;
  for (const Case& cs : cases) {
    lance::ConvSpec spec;
    spec.n = cs.n, spec.c = cs.c, spec.h = cs.h, spec.w = cs.w, spec.k = cs.k, spec.pad = cs.pad;
    lance::LanceConfig cfg;
    cfg.bits_w = cs.bits_w, cfg.bits_i = cs.bits_i, cfg.granularity = cs.gran;
    cfg.mode = lance::LanceMode::Gemm;
    lance::Tensor4 x;
    lance::FilterBank w;
    make_layer(cs, x, w);
    const lance::Tensor4 yr = lance::lance_gemm(x, w, spec, cfg);
    // Same reference objects, B200 path: the result type is lance::Tensor4.
    const lance::Tensor4 yb = lance::b200::lance_gemm_any(x, w, spec, cfg);
    std::size_t diff = 0;
    if (yr.data.size() == yb.data.size())
      for (std::size_t i = 0; i < yr.data.size(); ++i)
        diff += std::memcmp(&yr.data[i], &yb.data[i], sizeof(float)) != 0;
    const bool same = (yr == yb) && diff == 0 && yr.data.size() == yb.data.size() &&
                      yr.n == yb.n && yr.h == yb.h && yr.w == yb.w && yr.c == yb.c;
    bad += !same;
    std::printf("case n=%d c=%d h=%d w=%d k=%d pad=%d bits=%d/%d gran=%d: %zu outputs, %zu differ -> %s\n",
                cs.n, cs.c, cs.h, cs.w, cs.k, cs.pad, cs.bits_w, cs.bits_i, static_cast<int>(cs.gran),
                yr.data.size(), diff, same ? "bit-exact" : "MISMATCH");
  }
  return bad;
}

}  // namespace

int main(int argc, char** argv) {
  const bool errors_only = argc > 1 && std::strcmp(argv[1], "--errors") == 0;
  int bad = run_errors();
  if (!errors_only) {
    try {
      bad += run_cases();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
  }
  std::printf("%s\n", bad == 0 ? "ALL MATCH" : "FAILURES");
  return bad == 0 ? 0 : 3;
}
