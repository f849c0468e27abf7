// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference headers, compiled in place from
// /root/reference/proj/include by oracle/Makefile into oracle/_ref/ (never
// copied into this repo).  It lets the Python tests, the golden-fixture
// generator and bench.py's CPU baseline call the reference's own
// lance::lance_gemm (engines.hpp:492-536), its stage functions and its
// property suite (verify.hpp:611-651).  Built like the reference's CMake
// Release configuration: -O3 -DNDEBUG, no -march (no FMA contraction).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "lance/engines.hpp"
#include "lance/rng.hpp"
#include "lance/tensor_io.hpp"
#include "lance/verify.hpp"

namespace {
thread_local std::string g_err;

int fail_from(const std::exception& e) {
  g_err = e.what();
  return dynamic_cast<const std::invalid_argument*>(&e) ? 1 : 3;
}

lance::Granularity gran_of(int g) {
  return g == 0 ? lance::Granularity::PerTile
                : (g == 1 ? lance::Granularity::PerPosition : lance::Granularity::PerTensor);
}

lance::ConvSpec spec_of(int n, int c, int h, int w, int k, int pad) {
  lance::ConvSpec s;
  s.n = n; s.c = c; s.h = h; s.w = w; s.k = k; s.pad = pad;
  return s;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hardware_threads() { return int(std::thread::hardware_concurrency()); }

void ref_set_threads(int n) { lance::set_max_threads(n); }

// UniformSource (rng.hpp:27-47) stream: `count` draws from one seed.
void ref_uniform_fill(uint64_t seed, float* out, size_t count) {
  lance::UniformSource src(seed);
  src.fill(std::span<float>(out, count));
}

// lance::lance_gemm (engines.hpp:492-536).  mode_gemm=0 exercises the
// reference's own "cfg.mode must be Gemm" rejection.
int ref_lance_gemm(int n, int c, int h, int w, int k, int pad, int bits_w, int bits_i,
                   int gran, int mode_gemm, const float* x, const float* wt, float* y) {
  try {
    const lance::ConvSpec spec = spec_of(n, c, h, w, k, pad);
    lance::LanceConfig cfg;
    cfg.bits_w = bits_w;
    cfg.bits_i = bits_i;
    cfg.granularity = gran_of(gran);
    cfg.mode = mode_gemm ? lance::LanceMode::Gemm : lance::LanceMode::Faithful;
    // Tensor4 / FilterBank constructors validate their own dims (tensor.hpp:31-35).
    lance::Tensor4 xt(n, h, w, c, std::vector<float>(x, x + size_t(n) * h * w * c));
    lance::FilterBank wf(k, 3, 3, c, std::vector<float>(wt, wt + size_t(k) * 9 * c));
    const lance::Tensor4 out = lance::lance_gemm(xt, wf, spec, cfg);
    std::memcpy(y, out.data.data(), out.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

// lance::lance_faithful (engines.hpp:441-486), for mode-equivalence checks.
int ref_lance_faithful(int n, int c, int h, int w, int k, int pad, int bits_w, int bits_i,
                       int gran, const float* x, const float* wt, float* y) {
  try {
    const lance::ConvSpec spec = spec_of(n, c, h, w, k, pad);
    lance::LanceConfig cfg;
    cfg.bits_w = bits_w;
    cfg.bits_i = bits_i;
    cfg.granularity = gran_of(gran);
    cfg.mode = lance::LanceMode::Faithful;
    lance::Tensor4 xt(n, h, w, c, std::vector<float>(x, x + size_t(n) * h * w * c));
    lance::FilterBank wf(k, 3, 3, c, std::vector<float>(wt, wt + size_t(k) * 9 * c));
    const lance::Tensor4 out = lance::lance_faithful(xt, wf, spec, cfg);
    std::memcpy(y, out.data.data(), out.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

// Stage dump through the reference's own stage functions, in the same call
// sequence as lance_gemm (engines.hpp:501-525).  Any output may be NULL.
// v [16][M][C], u [16][C][K] fp32; codes_a [16][M][C], codes_w [16][C][K] u8;
// params [16] x {bits, t_min, t_max, scale}; acc [16][M][K]; rowsum [16][M];
// colsum [16][K].
int ref_stage_dump(int n, int c, int h, int w, int k, int pad, int bits_w, int bits_i,
                   int gran, const float* x, const float* wt, float* v_out, float* u_out,
                   uint8_t* codes_a, uint8_t* codes_w, float* params_a, float* params_w,
                   int32_t* acc, int32_t* rowsum, int32_t* colsum) {
  try {
    const lance::ConvSpec spec = spec_of(n, c, h, w, k, pad);
    lance::Tensor4 xt(n, h, w, c, std::vector<float>(x, x + size_t(n) * h * w * c));
    lance::FilterBank wf(k, 3, 3, c, std::vector<float>(wt, wt + size_t(k) * 9 * c));
    const lance::WinogradBasis& basis = lance::basis_f2x2_3x3();
    const lance::TileSet tiles = lance::extract_tiles(xt, basis.m, basis.r, spec.pad);
    const lance::DomainTensor v = lance::detail::domain_from_tiles(tiles, basis);
    const lance::DomainTensor u = lance::detail::domain_from_filters(wf, basis);
    const lance::QuantizedDomain vq = lance::quantize_domain(v, bits_i, gran_of(gran));
    const lance::QuantizedDomain uq = lance::quantize_domain(u, bits_w, gran_of(gran));
    if (v_out) std::memcpy(v_out, v.values.data(), v.values.size() * sizeof(float));
    if (u_out) std::memcpy(u_out, u.values.data(), u.values.size() * sizeof(float));
    if (codes_a) std::memcpy(codes_a, vq.codes.data(), vq.codes.size());
    if (codes_w) std::memcpy(codes_w, uq.codes.data(), uq.codes.size());
    for (int p = 0; p < 16; ++p) {
      const lance::QuantParams& pa = vq.param_at(p, 0, 0);
      const lance::QuantParams& pb = uq.param_at(p, 0, 0);
      if (params_a) {
        params_a[4 * p + 0] = float(pa.bits);
        params_a[4 * p + 1] = pa.t_min;
        params_a[4 * p + 2] = pa.t_max;
        params_a[4 * p + 3] = pa.scale;
      }
      if (params_w) {
        params_w[4 * p + 0] = float(pb.bits);
        params_w[4 * p + 1] = pb.t_min;
        params_w[4 * p + 2] = pb.t_max;
        params_w[4 * p + 3] = pb.scale;
      }
    }
    const std::size_t vslice = std::size_t(v.rows) * v.cols;
    const std::size_t uslice = std::size_t(u.rows) * u.cols;
    for (int p = 0; p < 16; ++p) {
      lance::CodeMatrix a;
      a.rows = v.rows;
      a.cols = v.cols;
      a.codes.assign(vq.codes.begin() + p * vslice, vq.codes.begin() + (p + 1) * vslice);
      lance::CodeMatrix b;
      b.rows = u.rows;
      b.cols = u.cols;
      b.codes.assign(uq.codes.begin() + p * uslice, uq.codes.begin() + (p + 1) * uslice);
      if (acc) {
        const lance::AccMatrix am = lance::gemm_codes(a, b);
        std::memcpy(acc + std::size_t(p) * am.sums.size(), am.sums.data(),
                    am.sums.size() * sizeof(int32_t));
      }
      if (rowsum)
        for (int i = 0; i < a.rows; ++i) {
          int32_t s = 0;
          for (int kk = 0; kk < a.cols; ++kk) s += a.at(i, kk);
          rowsum[std::size_t(p) * a.rows + i] = s;
        }
      if (colsum)
        for (int j = 0; j < b.cols; ++j) {
          int32_t s = 0;
          for (int kk = 0; kk < b.rows; ++kk) s += b.at(kk, j);
          colsum[std::size_t(p) * b.cols + j] = s;
        }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

// CPU baseline: the reference's own lance_gemm on `reps` timed repeats with
// the reference bench's method (median of steady_clock, bench.hpp:157-167).
// Inputs from UniformSource(seed), x then w from one stream (bench.hpp:129-133).
int ref_time_lance_gemm(int n, int c, int h, int w, int k, int pad, int threads, uint64_t seed,
                        int reps, double* median_ns, double* min_ns) {
  try {
    lance::set_max_threads(threads);
    const lance::ConvSpec spec = spec_of(n, c, h, w, k, pad);
    lance::LanceConfig cfg;
    cfg.granularity = lance::Granularity::PerPosition;
    cfg.mode = lance::LanceMode::Gemm;
    lance::Tensor4 xt(n, h, w, c);
    lance::FilterBank wf(k, 3, 3, c);
    lance::UniformSource src(seed);
    src.fill(xt.data);
    src.fill(wf.data);
    std::vector<double> ns;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const lance::Tensor4 y = lance::lance_gemm(xt, wf, spec, cfg);
      const auto t1 = std::chrono::steady_clock::now();
      ns.push_back(double(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count()));
      if (y.data.empty()) return 3;
    }
    std::sort(ns.begin(), ns.end());
    *median_ns = ns[ns.size() / 2];
    *min_ns = ns.front();
    return 0;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

// The reference property suite (verify.hpp:635-651): 17 named checks.
int ref_run_verify(char* report, size_t cap) {
  std::ostringstream os;
  const bool ok = lance::run_verify(os);
  const std::string s = os.str();
  if (report && cap) {
    const size_t nb = std::min(cap - 1, s.size());
    std::memcpy(report, s.data(), nb);
    report[nb] = 0;
  }
  return ok ? 0 : 1;
}

// tensor_io.hpp:94-150: the reference's own LTEN writer / reader (format pins
// for paper_2003_08646_b200/tensor_io.py).  ref_read_lten returns 0 and fills
// dims[4] (+ data when non-NULL and cap is enough), 2 on FormatError.
int ref_write_lten(const char* path, int n, int h, int w, int c, const float* data) {
  try {
    lance::Tensor4 t(n, h, w, c);
    std::memcpy(t.data.data(), data, sizeof(float) * t.data.size());
    lance::write_tensor_file(t, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

int ref_read_lten(const char* path, int* dims, float* data, size_t cap) {
  try {
    const lance::Tensor4 t = lance::read_tensor_file(path);
    dims[0] = t.n;
    dims[1] = t.h;
    dims[2] = t.w;
    dims[3] = t.c;
    if (data && cap >= t.data.size()) std::memcpy(data, t.data.data(), sizeof(float) * t.data.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"
