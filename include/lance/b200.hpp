// lance/b200.hpp -- C++ host API of the B200 lance_gemm path.
//
// Keeps the reference operator API (/root/reference/proj/include/lance/) by
// name and meaning and implements it over the C ABI in lance_b200.h:
//
//   ConvSpec      engines.hpp:33-54      LanceConfig  engines.hpp:60-80
//   QuantParams   quant.hpp:27-37        Granularity  quant.hpp:44
//   Tensor4       tensor.hpp:25-55       FilterBank   tensor.hpp:58-86
//   lance_gemm(x, w, spec, cfg) -> Tensor4            engines.hpp:492-536
//
// Errors are thrown exactly where the reference throws: std::invalid_argument
// with the reference's message for spec / config / shape violations and for
// NaN data (quant.hpp:62); std::runtime_error for CUDA failures (the reference
// has none).  The generic overload also accepts the reference's own
// lance::Tensor4 / lance::FilterBank / ConvSpec / LanceConfig objects, so a
// reference caller switches by changing the namespace of one call.
//
// Link: -L<repo>/paper_2003_08646_b200/_build -llance_b200
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../lance_b200.h"

namespace lance {
namespace b200 {

enum class Granularity { PerTile, PerPosition, PerTensor };
enum class LanceMode { Faithful, Gemm };

struct ConvSpec {
  int n = 1, c = 1, h = 1, w = 1;
  int k = 1;
  int pad = 0;
  static constexpr int r = 3, s = 3;
  static constexpr int stride = 1;
  int out_h() const { return h + 2 * pad - r + 1; }
  int out_w() const { return w + 2 * pad - s + 1; }
  int tiles_h() const { return (out_h() + 1) / 2; }
  int tiles_w() const { return (out_w() + 1) / 2; }
  int tiles_per_image() const { return tiles_h() * tiles_w(); }
};

struct LanceConfig {
  int bits_w = 8;
  int bits_i = 8;
  Granularity granularity = Granularity::PerTile;
  LanceMode mode = LanceMode::Faithful;
};

struct QuantParams {
  int bits = 8;
  float t_min = 0.0f, t_max = 0.0f, scale = 0.0f;
  int max_code() const { return (1 << bits) - 1; }
  bool operator==(const QuantParams&) const = default;
};

struct Tensor4 {
  int n = 0, h = 0, w = 0, c = 0;
  std::vector<float> data;
  Tensor4() = default;
  Tensor4(int n_, int h_, int w_, int c_) : n(n_), h(h_), w(w_), c(c_) {
    if (n < 1 || h < 1 || w < 1 || c < 1)
      throw std::invalid_argument("Tensor4: all dims must be >= 1");
    data.assign(std::size_t(n) * h * w * c, 0.0f);
  }
  std::size_t size() const { return data.size(); }
  std::size_t index(int ni, int hi, int wi, int ci) const {
    return ((std::size_t(ni) * h + hi) * w + wi) * c + ci;
  }
  float& at(int ni, int hi, int wi, int ci) { return data[index(ni, hi, wi, ci)]; }
  const float& at(int ni, int hi, int wi, int ci) const { return data[index(ni, hi, wi, ci)]; }
};

struct FilterBank {
  int k = 0, r = 0, s = 0, c = 0;
  std::vector<float> data;
  FilterBank() = default;
  FilterBank(int k_, int r_, int s_, int c_) : k(k_), r(r_), s(s_), c(c_) {
    if (k < 1 || r < 1 || s < 1 || c < 1)
      throw std::invalid_argument("FilterBank: all dims must be >= 1");
    data.assign(std::size_t(k) * r * s * c, 0.0f);
  }
  std::size_t size() const { return data.size(); }
};

namespace detail {

inline void throw_status(int rc) {
  if (rc == LANCE_OK) return;
  const std::string msg = lance_last_error();
  if (rc == LANCE_ERR_INVALID_ARGUMENT || rc == LANCE_ERR_NAN) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string(lance_status_string(rc)) + ": " + msg);
}

template <class Spec>
lance_conv_spec c_spec(const Spec& s) {
  return lance_conv_spec{s.n, s.c, s.h, s.w, s.k, s.pad};
}

template <class Cfg>
lance_config c_cfg(const Cfg& c) {
  return lance_config{c.bits_w, c.bits_i, static_cast<int>(c.granularity),
                      static_cast<int>(c.mode)};
}

}  // namespace detail

// lance_gemm for any types with the reference's members (this namespace's or
// the reference's own lance::Tensor4 / FilterBank / ConvSpec / LanceConfig).
// check_layer (engines.hpp:84-91) is reproduced before the ABI call.
// tile_m = 4 selects the F(4x4,3x3) extension (lance_gemm_host_tiled).
template <class T4, class FB, class Spec, class Cfg>
T4 lance_gemm_any(const T4& x, const FB& w, const Spec& spec, const Cfg& cfg, int tile_m = 2) {
  const lance_conv_spec cs = detail::c_spec(spec);
  const lance_config cc = detail::c_cfg(cfg);
  // ConvSpec::validate first, exactly as check_layer does.
  {
    lance_config probe{8, 8, LANCE_GRAN_PER_POSITION, LANCE_MODE_GEMM};
    detail::throw_status(lance_validate(&cs, &probe));
  }
  if (x.n != spec.n || x.h != spec.h || x.w != spec.w || x.c != spec.c)
    throw std::invalid_argument("input tensor dims do not match spec");
  if (w.k != spec.k || w.r != 3 || w.s != 3 || w.c != spec.c)
    throw std::invalid_argument("filter dims do not match spec");
  detail::throw_status(lance_validate(&cs, &cc));
  T4 y(spec.n, spec.out_h(), spec.out_w(), spec.k);
  detail::throw_status(
      lance_gemm_host_tiled(&cs, &cc, tile_m, x.data.data(), w.data.data(), y.data.data()));
  return y;
}

inline Tensor4 lance_gemm(const Tensor4& x, const FilterBank& w, const ConvSpec& spec,
                          const LanceConfig& cfg) {
  return lance_gemm_any(x, w, spec, cfg);
}

// F(4x4,3x3) extension: the same algorithm with 6x6 tiles at stride 4 and 36
// Winograd positions (not in the reference; SURVEY.md Appendix D basis).
inline Tensor4 lance_gemm_f4(const Tensor4& x, const FilterBank& w, const ConvSpec& spec,
                             const LanceConfig& cfg) {
  return lance_gemm_any(x, w, spec, cfg, 4);
}

// Device-resident layer: filters prepared once (K2), forward per batch.
class LanceConv {
 public:
  LanceConv(const ConvSpec& spec, const LanceConfig& cfg, int device = 0) : spec_(spec) {
    const lance_conv_spec cs = detail::c_spec(spec);
    const lance_config cc = detail::c_cfg(cfg);
    detail::throw_status(lance_plan_create(&cs, &cc, device, &plan_));
  }
  ~LanceConv() { lance_plan_destroy(plan_); }
  LanceConv(const LanceConv&) = delete;
  LanceConv& operator=(const LanceConv&) = delete;

  void set_filters(const float* w_dev, void* stream = nullptr) {
    detail::throw_status(lance_plan_set_filters(plan_, w_dev, stream));
  }
  void forward(const float* x_dev, float* y_dev, void* stream = nullptr) {
    detail::throw_status(lance_plan_forward(plan_, x_dev, y_dev, stream));
  }
  void forward_static(const QuantParams (&in)[16], const float* x_dev, float* y_dev,
                      void* stream = nullptr) {
    lance_qparams p[16];
    for (int i = 0; i < 16; ++i) p[i] = {in[i].bits, in[i].t_min, in[i].t_max, in[i].scale};
    detail::throw_status(lance_plan_forward_static(plan_, p, x_dev, y_dev, stream));
  }
  void set_epilogue(const float* bias_dev, bool relu) {
    detail::throw_status(lance_plan_set_epilogue(plan_, bias_dev, relu ? 1 : 0));
  }
  // Throws std::invalid_argument("fit_params: NaN in values") like the reference.
  void sync(void* stream = nullptr) { detail::throw_status(lance_plan_sync(plan_, stream)); }
  const ConvSpec& spec() const { return spec_; }
  lance_plan_t handle() const { return plan_; }

 private:
  ConvSpec spec_;
  lance_plan_t plan_ = nullptr;
};

}  // namespace b200
}  // namespace lance
