// lance_abi.cu -- host side of the B200 LANCE path behind the C ABI declared
// in include/lance_b200.h.  Owns validation (mirrors engines.hpp:46-91,
// 496-499 with the reference's messages), plan/workspace management, TMA
// tensor-map construction and the stream-ordered launch sequence
// K0 -> K1 -> K3/K4 (+ K2 once per layer).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <list>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/lance_b200.h"
#include "lance_kernels.cuh"

using namespace lance_dev;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(LANCE_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define LANCE_CUDA(call)                                         \
  do {                                                           \
    cudaError_t e_ = (call);                                     \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);          \
  } while (0)

}  // namespace

// Experiment / A-B switches (tools/*.sh): honoured only by LANCE_PROFILING
// builds; a release library ignores the environment and uses the defaults.
namespace lance_dev {
int lance_knob(const char* name, int def) {
#ifdef LANCE_PROFILING
  if (const char* e = std::getenv(name)) return std::atoi(e);
#else
  (void)name;
#endif
  return def;
}

cudaError_t ensure_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, fn}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e == cudaSuccess) have = bytes;
  return e;
}

bool pdl_enabled() {
  static const bool on = lance_knob("LANCE_PDL", 0) != 0;
  return on;
}

int current_sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  cache[dev] = sms;
  return sms;
}
}  // namespace lance_dev

namespace {

int out_h(const lance_conv_spec& s) { return s.h + 2 * s.pad - 3 + 1; }
int out_w(const lance_conv_spec& s) { return s.w + 2 * s.pad - 3 + 1; }
int round_up(int v, int m) { return (v + m - 1) / m * m; }

// ConvSpec::validate (engines.hpp:46-53), LanceConfig::validate (:66-79),
// lance_gemm's mode / depth checks (:496-499; lowpgemm.hpp:28).
int validate(const lance_conv_spec* s, const lance_config* c) {
  if (!s || !c) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance: null spec or config");
  if (s->n < 1 || s->c < 1 || s->h < 1 || s->w < 1 || s->k < 1)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "ConvSpec: all dims must be >= 1");
  if (s->pad != 0 && s->pad != 1)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "ConvSpec: pad must be 0 or 1");
  if (out_h(*s) < 1 || out_w(*s) < 1)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "ConvSpec: output dims collapse to zero");
  auto ok = [](int b) { return (b >= 2 && b <= 8) || b == 32; };
  if (!ok(c->bits_w) || !ok(c->bits_i))
    return fail(LANCE_ERR_INVALID_ARGUMENT, "LanceConfig: bits must be in [2, 8] or 32");
  if (c->mode == LANCE_MODE_GEMM) {
    if (c->granularity == LANCE_GRAN_PER_TILE)
      return fail(LANCE_ERR_INVALID_ARGUMENT,
                  "LanceConfig: Gemm mode cannot use PerTile granularity; integer "
                  "accumulation across channels needs one scale per position");
    if (c->bits_w == 32 || c->bits_i == 32)
      return fail(LANCE_ERR_INVALID_ARGUMENT,
                  "LanceConfig: Gemm mode requires quantized operands (bits <= 8)");
  }
  if (c->granularity != LANCE_GRAN_PER_TILE && c->granularity != LANCE_GRAN_PER_POSITION &&
      c->granularity != LANCE_GRAN_PER_TENSOR)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "LanceConfig: unknown granularity");
  if (c->mode != LANCE_MODE_GEMM)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_gemm: cfg.mode must be Gemm");
  if (s->c > 32768)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_gemm: channel count exceeds GEMM depth bound");
  return LANCE_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Row sums [16][rows] int32; box = 128 rows x 16 positions (OOB rows read 0).
int make_rowsum_map(CUtensorMap* map, void* base, long long rows, long long pitch) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(LANCE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), 16};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBM), 16};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LANCE_ERR_CUDA, "cuTensorMapEncodeTiled (row sums) failed: " + std::to_string(r));
  return LANCE_OK;
}

}  // namespace

struct lance_plan_s {
  int device = 0;
  int tm = 2;   // Winograd output tile side: 2 (reference F(2x2,3x3)) or 4 (F(4x4,3x3))
  int np = 16;  // positions (tm + 2)^2
  F4Geom f4{};
  lance_conv_spec spec{};
  lance_config cfg{};
  int OH = 0, OW = 0, TH = 0, TW = 0, P = 0;
  long long M = 0;
  int C_pad = 0, K_pad = 0, BK = 32, BN = 16;
  int sm_count = 148;
  int range_grid = 1, filter_grid = 1;
  InGeom in_geom{};
  int layout = LANCE_LAYOUT_NHWC;
  bool jsplit = false;      // GEMM j-split over 4 CTAs per tile (small M)
  float* tscratch = nullptr;
  int* tticket = nullptr;
  float* x_nhwc = nullptr;  // NCHW input: staging buffer of the transposed batch
  FilterGeom f_geom{};
  GemmGeom gemm_geom{};
  bool vec2 = false;
  bool small_acc = false;
  // device memory
  uint8_t* codes_a = nullptr;   // [16][M][C_pad]
  int32_t* rowsum = nullptr;    // [16][rs_pitch]
  long long rs_pitch = 0;       // M rounded up to 4
  uint8_t* codes_w = nullptr;   // [16][K_pad][C_pad]
  int32_t* colsum = nullptr;    // [16][K_pad]
  float* u_tmp = nullptr;       // [16][K][C]
  float* partials = nullptr;    // [max(range_grid, filter_grid)][32]
  LanceDevState* state = nullptr;
  size_t bytes = 0;
  CUtensorMap tmR{};
  bool filters_ready = false;
  int32_t* acc_dump = nullptr;
  const float* bias = nullptr;
  int relu = 0;
  int last_launches = 0;
  bool timing = false;
  std::vector<cudaEvent_t> events;  // 4 per recorded forward
  int recorded = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void free_plan(lance_plan_s* p) {
#ifdef LANCE_PROFILING
  if (p->gemm_geom.trace != nullptr) {
    if (const char* path = std::getenv("LANCE_GEMM_TRACE")) {
      std::vector<unsigned long long> h(800000);
      if (cudaMemcpy(h.data(), p->gemm_geom.trace, h.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
        const std::string f = std::string(path) + "_c" + std::to_string(p->spec.c) + "_h" +
                              std::to_string(p->spec.h) + ".bin";
        if (FILE* fp = std::fopen(f.c_str(), "wb")) {
          std::fwrite(h.data(), 8, h.size(), fp);
          std::fclose(fp);
        }
      }
    }
  }
#endif
  cudaFree(p->gemm_geom.trace);
  for (cudaEvent_t e : p->events) cudaEventDestroy(e);
  p->events.clear();
  cudaFree(p->x_nhwc);
  cudaFree(p->tscratch);
  cudaFree(p->tticket);
  cudaFree(p->codes_a);
  cudaFree(p->rowsum);
  cudaFree(p->codes_w);
  cudaFree(p->colsum);
  cudaFree(p->u_tmp);
  cudaFree(p->partials);
  cudaFree(p->state);
}

template <typename T>
int dev_alloc(lance_plan_s* p, T** ptr, size_t bytes) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), bytes < 16 ? 16 : bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  p->bytes += bytes;
  return LANCE_OK;
}

}  // namespace

extern "C" {

int lance_abi_version(void) { return LANCE_B200_ABI_VERSION; }

const char* lance_status_string(int s) {
  switch (s) {
    case LANCE_OK: return "ok";
    case LANCE_ERR_INVALID_ARGUMENT: return "invalid argument";
    case LANCE_ERR_NAN: return "NaN in data";
    case LANCE_ERR_CUDA: return "CUDA error";
    case LANCE_ERR_NO_DEVICE: return "no sm_100 device";
    default: return "unknown status";
  }
}

const char* lance_last_error(void) { return g_err.c_str(); }

int lance_validate(const lance_conv_spec* spec, const lance_config* cfg) {
  return validate(spec, cfg);
}

uint64_t lance_direct_multiply_count(const lance_conv_spec* s) {
  return uint64_t(s->n) * s->k * s->c * uint64_t(out_h(*s)) * out_w(*s) * 9u;
}

uint64_t lance_winograd_multiply_count(const lance_conv_spec* s) {
  const uint64_t tiles = uint64_t((out_h(*s) + 1) / 2) * ((out_w(*s) + 1) / 2);
  return 16u * tiles * s->n * s->c * uint64_t(s->k);
}

uint64_t lance_fnv1a64(const float* data, size_t count) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < count; ++i) {
    uint32_t bits;
    std::memcpy(&bits, data + i, 4);
    for (int b = 0; b < 4; ++b) {
      h ^= (bits >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

void lance_uniform_fill(uint64_t seed, float* out, size_t count) {
  std::mt19937_64 rng(seed);  // UniformSource (rng.hpp:27-47)
  for (size_t i = 0; i < count; ++i) {
    const auto top = static_cast<uint32_t>(rng() >> 40);
    out[i] = float(top) * (1.0f / 8388608.0f) - 1.0f;
  }
}

static int create_f4(lance_plan_s* p, const lance_conv_spec* spec, const lance_config* cfg);

int lance_plan_create(const lance_conv_spec* spec, const lance_config* cfg, int device,
                      lance_plan_t* out) {
  return lance_plan_create_tiled(spec, cfg, 2, device, out);
}

int lance_plan_create_tiled(const lance_conv_spec* spec, const lance_config* cfg, int tile_m,
                            int device, lance_plan_t* out) {
  if (!out) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_create: null output");
  *out = nullptr;
  if (tile_m != 2 && tile_m != 4)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_create: tile_m must be 2 or 4");
  int rc = validate(spec, cfg);
  if (rc) return rc;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(LANCE_ERR_NO_DEVICE,
                "no CUDA device: the B200 lance_gemm path has no CPU fallback");
  }
  if (device < 0 || device >= ndev) return fail(LANCE_ERR_INVALID_ARGUMENT, "bad device index");
  cudaDeviceProp prop;
  LANCE_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(LANCE_ERR_NO_DEVICE, std::string("device ") + prop.name +
                                         " is not sm_100 (this build targets sm_100a only)");
  DeviceGuard guard(device);

  auto* p = new lance_plan_s();
  p->device = device;
  p->spec = *spec;
  p->cfg = *cfg;
  p->sm_count = prop.multiProcessorCount;
  if (tile_m == 4) {
    if ((rc = create_f4(p, spec, cfg))) {
      free_plan(p);
      delete p;
      return rc;
    }
    *out = p;
    return LANCE_OK;
  }
  p->OH = out_h(*spec);
  p->OW = out_w(*spec);
  p->TH = (p->OH + 1) / 2;
  p->TW = (p->OW + 1) / 2;
  p->P = p->TH * p->TW;
  p->M = static_cast<long long>(spec->n) * p->P;
  p->C_pad = round_up(spec->c, 32);
  // GEMM tile width: 64 filters (two j-group accumulators of 4 x 64 TMEM
  // columns, 16 filters' S partials per epilogue thread) unless the layer has
  // fewer.  LANCE_GEMM_BN overrides.
  p->BN = spec->k > 32 ? 64 : (spec->k > 16 ? 32 : 16);
  // Small-M layers (64-filter tiles for at most half the SMs, e.g. VGG's
  // 4x4 / 2x2 maps, ResNet's 7x7 / 14x14 maps at per-GPU batches <= 32) get
  // twice the tiles at BN = 32.  Between half and all of the SMs, BN = 64 is
  // faster (R128 at batch 32: 19.7 vs 24.8 us; R256 at batch 64: 24.7 vs
  // 36.6 us, gpurun_out/gsmall).
  {
    const long long row_blocks = (static_cast<long long>(spec->n) * ((out_h(*spec) + 1) / 2) *
                                      ((out_w(*spec) + 1) / 2) + kBM - 1) / kBM;
    // j-split (JS): when even 4 CTAs per 64-filter tile fit in one wave, keep
    // BN = 64 and run each tile's 4 j-groups on 4 CTAs instead.
    p->jsplit = lance_knob("LANCE_GEMM_JSPLIT", 1) != 0 && p->BN == 64 &&
                4 * row_blocks * ((spec->k + 63) / 64) <= p->sm_count;
    if (p->BN == 64 && !p->jsplit && 2 * row_blocks * ((spec->k + 63) / 64) <= p->sm_count) p->BN = 32;
  }
  {
    const int v = lance_knob("LANCE_GEMM_BN", 0);
    if (v == 16 || v == 32 || v == 64) p->BN = v;
  }
  p->K_pad = round_up(spec->k, p->BN);
  p->BK = (p->C_pad % 128 == 0) ? 128 : (p->C_pad % 64 == 0 ? 64 : 32);
  p->vec2 = (spec->c % 2) == 0;

  if (static_cast<long long>(spec->n) * p->OH * p->OW >= (1LL << 27)) {
    delete p;
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_gemm: N * OH * OW exceeds 2^27 output pixels");
  }
  if (p->M >= (1LL << 31)) {
    delete p;
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_gemm: N * tiles exceeds 2^31 rows");
  }
  InGeom& g = p->in_geom;
  g.M = static_cast<int>(p->M);
  p->rs_pitch = (p->M + 3) / 4 * 4;
  g.rs_pitch = static_cast<int>(p->rs_pitch);
  g.P = p->P;
  g.TH = p->TH;
  g.TW = p->TW;
  g.H = spec->h;
  g.W = spec->w;
  g.C = spec->c;
  g.C_pad = p->C_pad;
  g.pad = spec->pad;
  g.nchunks = (p->C_pad + kChunk - 1) / kChunk;
  g.a_bk = p->BK;
  g.a_nk = p->C_pad / p->BK;
  // Warp strips: whole tile rows unless that leaves too few warps to fill
  // 148 SMs x 32 warps; then halve the strip length.  Long strips are also
  // halved down to 64 items per SM as long as they stay >= 7 tiles: K1 runs
  // one strip per warp in ~2.4 waves at 32 items per SM and ~4.8 at 64, so
  // its last partial wave shrinks (R64 K1 102.6 -> 99 us); shorter strips
  // than that cost more per-strip setup than they save (R256 / R512).
  g.seg_len = p->TW;
  for (;;) {
    g.nseg = (p->TW + g.seg_len - 1) / g.seg_len;
    g.num_items = static_cast<long long>(spec->n) * p->TH * g.nseg * g.nchunks;
    if (g.seg_len <= 2 || g.num_items >= 64LL * p->sm_count) break;
    if (g.num_items >= 32LL * p->sm_count && (g.seg_len + 1) / 2 < 7) break;
    g.seg_len = (g.seg_len + 1) / 2;
  }
  g.granularity = cfg->granularity;
  p->range_grid = input_range_grid(g, p->sm_count);
  p->small_acc = static_cast<double>(spec->c) * ((1 << cfg->bits_i) - 1) *
                     ((1 << cfg->bits_w) - 1) < 16777216.0;  // every accumulator < 2^24 (exact fp32 bit trick)

  FilterGeom& f = p->f_geom;
  f.K = spec->k;
  f.C = spec->c;
  f.K_pad = p->K_pad;
  f.C_pad = p->C_pad;
  f.granularity = cfg->granularity;
  f.bk = p->BK;
  f.bn = p->BN;
  f.nk = p->C_pad / p->BK;
  const long long kc = static_cast<long long>(spec->k) * spec->c;
  p->filter_grid = static_cast<int>(std::min<long long>((kc + 255) / 256, 2LL * p->sm_count));

  GemmGeom& gg = p->gemm_geom;
  gg.M = static_cast<int>(p->M);
  gg.K = spec->k;
  gg.C = spec->c;
  gg.P = p->P;
  gg.TW = p->TW;
  gg.OH = p->OH;
  gg.OW = p->OW;
  gg.num_kchunks = p->C_pad / p->BK;
  gg.num_n_tiles = p->K_pad / p->BN;
  gg.stages = 0;  // chosen by the launcher
  gg.exp = lance_knob("LANCE_GEMM_EXP", 0);
  gg.trace = nullptr;
  gg.b_resident = 0;
  gg.rs_pitch = static_cast<int>(p->rs_pitch);
  // Output staging + stage shape.  C >= 512 (BK = 128, 4 k chunks per
  // position): no y staging buffer, and stages of 2 k chunks (one 32 KB A
  // and one 16 KB B copy, 8 MMAs per producer / MMA handshake) -- measured
  // R512 GEMM 61 -> 49.5 us (gpurun_out/gsweep: only this combination helps;
  // more producer lanes, 4-chunk stages or unstaged y at C <= 256 do not).
  // LANCE_GEMM_STAGE / LANCE_GEMM_UNITS override.
  gg.stage_out = lance_knob("LANCE_GEMM_STAGE", p->C_pad >= 512 && p->BK == 128 ? 0 : 1) ? 1 : 0;
  // Row sums: in the GEMM's spare warps when its stages are 64-byte K chunks
  // (their shared-memory reads then cost the SS-UMMA little), else in K1.
  // LANCE_RS_GEMM overrides.
  gg.rs_warps = lance_knob("LANCE_RS_GEMM", p->BK <= 64 ? 1 : 0) ? 1 : 0;
  if (p->jsplit && gg.rs_warps) p->jsplit = false;  // JS reads K1's row sums (BK = 128 layers)
  gg.jsplit = p->jsplit ? 1 : 0;
  p->in_geom.rowsums = gg.rs_warps ? 0 : 1;
  {
    // 2 k chunks per stage also for 32-filter tiles with an even chunk count
    // (small-M layers: R256 at batch 32 22.7 -> 20.0 us, gpurun_out/gsmall).
    const int nk = p->C_pad / p->BK;
    const bool u2 = (p->C_pad >= 512 && p->BK == 128) || (p->BN == 32 && nk % 2 == 0);
    gg.units = lance_knob("LANCE_GEMM_UNITS", u2 ? 2 : 1);
  }
  p->in_geom.rev_items = lance_knob("LANCE_K1_REVERSE", 1) ? 1 : 0;

  // Operand images cover whole 128-row blocks; rows >= M stay code 0.
  const size_t codes_a_bytes = static_cast<size_t>(16) * ((p->M + kBM - 1) / kBM * kBM) * p->C_pad;
  const size_t codes_w_bytes = static_cast<size_t>(16) * p->K_pad * p->C_pad;
  const int part_rows = std::max(p->range_grid, p->filter_grid);
  if ((rc = dev_alloc(p, &p->codes_a, codes_a_bytes)) ||
      (rc = dev_alloc(p, &p->rowsum, sizeof(int32_t) * 16 * p->rs_pitch)) ||
      (rc = dev_alloc(p, &p->codes_w, codes_w_bytes)) ||
      (rc = dev_alloc(p, &p->colsum, sizeof(int32_t) * 16 * p->K_pad)) ||
      (rc = dev_alloc(p, &p->u_tmp, sizeof(float) * 16 * kc)) ||
      (rc = dev_alloc(p, &p->partials, sizeof(float) * 32 * part_rows)) ||
      (rc = dev_alloc(p, &p->state, sizeof(LanceDevState)))) {
    free_plan(p);
    delete p;
    return rc;
  }
  // K1's atomically accumulated row sums (several channel chunks per tile)
  // are cleared by K0 of the same forward.
  if (p->in_geom.nchunks > 1 && p->in_geom.rowsums) {
    p->in_geom.rs_zero = p->rowsum;
    p->in_geom.rs_zero_words = 16LL * p->rs_pitch;
  }
  // Channel / filter padding stays zero forever: both GEMM operands are padded
  // with code 0, which adds nothing to the accumulators.
  cudaError_t e = cudaMemset(p->codes_a, 0, codes_a_bytes);
  if (e == cudaSuccess) e = cudaMemset(p->codes_w, 0, codes_w_bytes);
  if (e == cudaSuccess) e = cudaMemset(p->colsum, 0, sizeof(int32_t) * 16 * p->K_pad);
  LanceDevState init{};
  init.bits_i = cfg->bits_i;
  init.bits_w = cfg->bits_w;
  if (e == cudaSuccess) e = cudaMemcpy(p->state, &init, sizeof init, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    free_plan(p);
    delete p;
    return cuda_fail(e, "plan init");
  }
#ifdef LANCE_PROFILING
  const bool want_trace = std::getenv("LANCE_GEMM_TRACE") != nullptr;  // value = dump path prefix
#else
  const bool want_trace = false;
#endif
  if (want_trace &&
      (rc = dev_alloc(p, &p->gemm_geom.trace, sizeof(unsigned long long) * 800000))) {
    free_plan(p);
    delete p;
    return rc;
  }
  if (p->jsplit) {
    const long long tiles = (p->M + kBM - 1) / kBM * (p->K_pad / p->BN);
    if ((rc = dev_alloc(p, &p->tscratch, sizeof(float) * tiles * 4 * 2 * kBM * p->BN)) ||
        (rc = dev_alloc(p, &p->tticket, sizeof(int) * tiles))) {
      free_plan(p);
      delete p;
      return rc;
    }
    if (cudaMemset(p->tticket, 0, sizeof(int) * tiles) != cudaSuccess) {
      free_plan(p);
      delete p;
      return cuda_fail(cudaGetLastError(), "plan init (j-split tickets)");
    }
    p->gemm_geom.tscratch = p->tscratch;
    p->gemm_geom.tticket = p->tticket;
  }
  if ((rc = make_rowsum_map(&p->tmR, p->rowsum, p->M, p->rs_pitch))) {
    free_plan(p);
    delete p;
    return rc;
  }
  *out = p;
  return LANCE_OK;
}

// F(4x4,3x3) plan (lance_f4.cu): 36 positions, BN = 16, B operand images
// of 16 filters, row sums written by the quantiser.
static int create_f4(lance_plan_s* p, const lance_conv_spec* spec, const lance_config* cfg) {
  p->tm = 4;
  p->np = 36;
  p->OH = out_h(*spec);
  p->OW = out_w(*spec);
  p->TH = (p->OH + 3) / 4;
  p->TW = (p->OW + 3) / 4;
  p->P = p->TH * p->TW;
  p->M = static_cast<long long>(spec->n) * p->P;
  if (static_cast<long long>(spec->n) * p->OH * p->OW >= (1LL << 27))
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_gemm: N * OH * OW exceeds 2^27 output pixels");
  p->C_pad = round_up(spec->c, 32);
  p->BK = (p->C_pad % 128 == 0) ? 128 : (p->C_pad % 64 == 0 ? 64 : 32);
  p->BN = 16;
  p->K_pad = round_up(spec->k, 16);
  p->rs_pitch = p->M;
  p->small_acc = static_cast<double>(spec->c) * ((1 << cfg->bits_i) - 1) *
                     ((1 << cfg->bits_w) - 1) < 16777216.0;
  F4Geom& g = p->f4;
  g.N = spec->n;
  g.H = spec->h;
  g.W = spec->w;
  g.C = spec->c;
  g.K = spec->k;
  g.pad = spec->pad;
  g.OH = p->OH;
  g.OW = p->OW;
  g.TH = p->TH;
  g.TW = p->TW;
  g.P = p->P;
  g.M = static_cast<int>(p->M);
  g.C_pad = p->C_pad;
  g.K_pad = p->K_pad;
  g.bk = p->BK;
  g.nk = p->C_pad / p->BK;
  g.rs_pitch = static_cast<int>(p->rs_pitch);
  g.granularity = cfg->granularity;
  g.num_n_tiles = p->K_pad / 16;
  g.stages = 0;
  g.units = 0;
  g.b_resident = 0;
  g.exp = lance_knob("LANCE_F4_EXP", 0);
  // Warp strips along tile rows: whole rows unless that leaves too few warps
  // to fill the SMs; then shorter strips.
  g.seg_len = p->TW;
  for (;;) {
    g.nseg = (p->TW + g.seg_len - 1) / g.seg_len;
    g.num_items = static_cast<long long>(spec->n) * p->TH * g.nseg * ((spec->c + 31) / 32);
    if (g.num_items >= 32LL * p->sm_count || g.seg_len <= 1) break;
    g.seg_len = (g.seg_len + 1) / 2;
  }
  p->range_grid = f4_range_grid(g, p->sm_count);
  const long long kc = static_cast<long long>(spec->k) * spec->c;
  p->filter_grid = static_cast<int>(std::min<long long>((kc + 255) / 256, 2LL * p->sm_count));
  const size_t codes_a_bytes = static_cast<size_t>(36) * ((p->M + kBM - 1) / kBM * kBM) * p->C_pad;
  const size_t codes_w_bytes = static_cast<size_t>(36) * p->K_pad * p->C_pad;
  const int part_rows = std::max(p->range_grid, p->filter_grid);
  int rc;
  if ((rc = dev_alloc(p, &p->codes_a, codes_a_bytes)) ||
      (rc = dev_alloc(p, &p->rowsum, sizeof(int32_t) * 36 * p->rs_pitch)) ||
      (rc = dev_alloc(p, &p->codes_w, codes_w_bytes)) ||
      (rc = dev_alloc(p, &p->colsum, sizeof(int32_t) * 36 * p->K_pad)) ||
      (rc = dev_alloc(p, &p->u_tmp, sizeof(float) * 36 * kc)) ||
      (rc = dev_alloc(p, &p->partials, sizeof(float) * 72 * part_rows)) ||
      (rc = dev_alloc(p, &p->state, sizeof(LanceDevState))))
    return rc;
  p->f4.rs_zero = p->rowsum;  // cleared by F0 of each forward that runs it
  p->f4.rs_zero_words = 36LL * p->rs_pitch;
  cudaError_t e = cudaMemset(p->codes_a, 0, codes_a_bytes);
  if (e == cudaSuccess) e = cudaMemset(p->codes_w, 0, codes_w_bytes);
  if (e == cudaSuccess) e = cudaMemset(p->colsum, 0, sizeof(int32_t) * 36 * p->K_pad);
  LanceDevState init{};
  init.bits_i = cfg->bits_i;
  init.bits_w = cfg->bits_w;
  if (e == cudaSuccess) e = cudaMemcpy(p->state, &init, sizeof init, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "plan init");
  return LANCE_OK;
}

int lance_plan_positions(lance_plan_t p) { return p ? p->np : 0; }

int lance_maxpool2x2_nhwc(const float* x_dev, float* y_dev, int n, int h, int w, int c,
                          void* stream) {
  if (!x_dev || !y_dev) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_maxpool2x2: null buffer");
  if (n < 1 || h < 2 || w < 2 || c < 1) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_maxpool2x2: bad dims");
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return fail(LANCE_ERR_NO_DEVICE, "no CUDA device");
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  LANCE_CUDA(launch_maxpool2x2(x_dev, y_dev, n, h, w, c, sms, static_cast<cudaStream_t>(stream)));
  return LANCE_OK;
}

uint64_t lance_winograd_multiply_count_tiled(const lance_conv_spec* s, int tile_m) {
  if (tile_m != 2 && tile_m != 4) return 0;
  const uint64_t tiles = uint64_t((out_h(*s) + tile_m - 1) / tile_m) * ((out_w(*s) + tile_m - 1) / tile_m);
  return uint64_t(tile_m + 2) * (tile_m + 2) * tiles * s->n * s->c * uint64_t(s->k);
}

int lance_plan_destroy(lance_plan_t p) {
  if (!p) return LANCE_OK;
  DeviceGuard guard(p->device);
  free_plan(p);
  delete p;
  return LANCE_OK;
}

size_t lance_plan_device_bytes(lance_plan_t p) { return p ? p->bytes : 0; }

int lance_plan_set_filters(lance_plan_t p, const float* w_dev, void* stream) {
  if (!p || !w_dev) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_set_filters: null argument");
  DeviceGuard guard(p->device);
  auto s = static_cast<cudaStream_t>(stream);
  if (p->tm == 4)
    LANCE_CUDA(launch_f4_filter_prepare(w_dev, p->u_tmp, p->partials, p->filter_grid, p->codes_w,
                                        p->colsum, p->state, p->f4, s));
  else
    LANCE_CUDA(launch_filter_prepare(w_dev, p->u_tmp, p->partials, p->filter_grid, p->codes_w,
                                     p->colsum, p->state, p->f_geom, s));
  p->filters_ready = true;
  return LANCE_OK;
}

// Input-parameter source of a forward: the batch's own range pass (K0), the
// caller's QuantParams, or device ranges already reduced across ranks.
static int run_forward(lance_plan_t p, const float* x_dev, float* y_dev, cudaStream_t s,
                       const lance_qparams* static_params, const float* minmax_dev = nullptr) {
  if (!p || !x_dev || !y_dev) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_forward: null argument");
  if (!p->filters_ready)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_forward: filters not set");
  DeviceGuard guard(p->device);
  int launches = 0;
  cudaEvent_t* ev = nullptr;
  if (p->timing && p->recorded < 4096) {
    while (p->events.size() < size_t(4) * (p->recorded + 1)) {
      cudaEvent_t e;
      LANCE_CUDA(cudaEventCreate(&e));
      p->events.push_back(e);
    }
    ev = &p->events[size_t(4) * p->recorded];
    ++p->recorded;
    LANCE_CUDA(cudaEventRecord(ev[0], s));
  }
  if (p->layout == LANCE_LAYOUT_NCHW) {  // staging transpose, then the NHWC kernels
    LANCE_CUDA(launch_nchw_to_nhwc(x_dev, p->x_nhwc, p->spec.n, p->spec.c, p->spec.h, p->spec.w, s));
    x_dev = p->x_nhwc;
    ++launches;
  }
  if (p->tm == 4) {
    if (static_params) {
      StaticParams prm{};
      prm.np = 36;
      for (int i = 0; i < 36; ++i) {
        if (static_params[i].bits != p->cfg.bits_i)
          return fail(LANCE_ERR_INVALID_ARGUMENT, "static params: bits differ from cfg.bits_i");
        prm.tmin[i] = static_params[i].t_min;
        prm.tmax[i] = static_params[i].t_max;
        prm.scale[i] = static_params[i].scale;
      }
      LANCE_CUDA(launch_static_params(p->state, prm, p->spec.c, s));
    } else if (minmax_dev) {
      LANCE_CUDA(launch_fit_minmax(p->state, minmax_dev, 36, p->cfg.granularity, p->spec.c, s));
    } else {
      LANCE_CUDA(launch_f4_range(x_dev, p->partials, p->range_grid, p->state, p->f4, s));
    }
    if (ev) LANCE_CUDA(cudaEventRecord(ev[1], s));
    LANCE_CUDA(launch_f4_quant(x_dev, p->codes_a, p->rowsum, p->state, p->f4, static_params != nullptr,
                               /*clear_rowsum=*/(static_params || minmax_dev) ? 1 : 0, p->sm_count, s));
    if (ev) LANCE_CUDA(cudaEventRecord(ev[2], s));
    LANCE_CUDA(launch_f4_gemm(p->codes_a, p->codes_w, p->rowsum, p->colsum, p->small_acc, p->state, y_dev,
                              p->acc_dump, p->bias, p->relu, p->f4, s));
    if (ev) LANCE_CUDA(cudaEventRecord(ev[3], s));
    p->last_launches = launches + 3;
    return LANCE_OK;
  }
  if (static_params) {
    StaticParams prm{};
    prm.np = 16;
    for (int i = 0; i < 16; ++i) {
      if (static_params[i].bits != p->cfg.bits_i)
        return fail(LANCE_ERR_INVALID_ARGUMENT, "static params: bits differ from cfg.bits_i");
      prm.tmin[i] = static_params[i].t_min;
      prm.tmax[i] = static_params[i].t_max;
      prm.scale[i] = static_params[i].scale;
    }
    LANCE_CUDA(launch_static_params(p->state, prm, p->spec.c, s));
  } else if (minmax_dev) {
    LANCE_CUDA(launch_fit_minmax(p->state, minmax_dev, 16, p->cfg.granularity, p->spec.c, s));
  } else {
    LANCE_CUDA(launch_input_range(x_dev, p->partials, p->range_grid, p->state, p->in_geom,
                                  p->vec2, s));
  }
  ++launches;
  if (ev) LANCE_CUDA(cudaEventRecord(ev[1], s));
  // K1 accumulates the row sums of multi-chunk layers atomically: K0 cleared
  // them above; the static / device-range modes run no K0, so clear here.
  if (p->in_geom.nchunks > 1 && p->in_geom.rowsums && (static_params || minmax_dev))
    LANCE_CUDA(cudaMemsetAsync(p->rowsum, 0, sizeof(int32_t) * 16 * p->rs_pitch, s));
  LANCE_CUDA(launch_input_quant(x_dev, p->codes_a, p->rowsum, p->state, p->in_geom, p->vec2,
                                static_params != nullptr, s));
  ++launches;
  if (ev) LANCE_CUDA(cudaEventRecord(ev[2], s));
  LANCE_CUDA(launch_gemm(p->codes_a, p->codes_w, &p->tmR, p->rowsum, p->BK, p->BN, p->small_acc, p->colsum, p->state, y_dev,
                         p->acc_dump, p->bias, p->relu, p->gemm_geom, s));
  ++launches;
  if (ev) LANCE_CUDA(cudaEventRecord(ev[3], s));
  p->last_launches = launches;
  return LANCE_OK;
}

int lance_plan_forward(lance_plan_t p, const float* x_dev, float* y_dev, void* stream) {
  return run_forward(p, x_dev, y_dev, static_cast<cudaStream_t>(stream), nullptr);
}

int lance_plan_forward_static(lance_plan_t p, const lance_qparams* in_params16,
                              const float* x_dev, float* y_dev, void* stream) {
  if (!in_params16) return fail(LANCE_ERR_INVALID_ARGUMENT, "static params: null");
  return run_forward(p, x_dev, y_dev, static_cast<cudaStream_t>(stream), in_params16);
}

int lance_plan_ranges(lance_plan_t p, const float* x_dev, float* minmax_dev, void* stream) {
  if (!p || !x_dev || !minmax_dev) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_ranges: null argument");
  DeviceGuard guard(p->device);
  auto s = static_cast<cudaStream_t>(stream);
  if (p->tm == 4)
    LANCE_CUDA(launch_f4_range(x_dev, p->partials, p->range_grid, p->state, p->f4, s));
  else {
    if (p->layout == LANCE_LAYOUT_NCHW) {
      LANCE_CUDA(launch_nchw_to_nhwc(x_dev, p->x_nhwc, p->spec.n, p->spec.c, p->spec.h, p->spec.w, s));
      x_dev = p->x_nhwc;
    }
    LANCE_CUDA(launch_input_range(x_dev, p->partials, p->range_grid, p->state, p->in_geom, p->vec2, s));
  }
  LANCE_CUDA(launch_export_minmax(p->state, minmax_dev, p->np, s));
  return LANCE_OK;
}

int lance_plan_forward_ranges(lance_plan_t p, const float* minmax_dev, const float* x_dev,
                              float* y_dev, void* stream) {
  if (!minmax_dev) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_forward_ranges: null ranges");
  return run_forward(p, x_dev, y_dev, static_cast<cudaStream_t>(stream), nullptr, minmax_dev);
}

int lance_plan_set_input_layout(lance_plan_t p, int layout) {
  if (!p) return fail(LANCE_ERR_INVALID_ARGUMENT, "null plan");
  if (layout != LANCE_LAYOUT_NHWC && layout != LANCE_LAYOUT_NCHW)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_set_input_layout: layout must be NHWC or NCHW");
  if (layout == LANCE_LAYOUT_NCHW && static_cast<long long>(p->spec.n) * p->spec.h >= 65536)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_set_input_layout: NCHW input needs N * H < 65536");
  if (layout == LANCE_LAYOUT_NCHW && !p->x_nhwc) {
    DeviceGuard guard(p->device);
    int rc = dev_alloc(p, &p->x_nhwc, sizeof(float) * size_t(p->spec.n) * p->spec.h * p->spec.w * p->spec.c);
    if (rc) return rc;
  }
  p->layout = layout;
  return LANCE_OK;
}

int lance_plan_input_layout(lance_plan_t p) { return p ? p->layout : -1; }

int lance_plan_set_epilogue_pool(lance_plan_t p, int pool) {
  if (!p) return fail(LANCE_ERR_INVALID_ARGUMENT, "null plan");
  if (pool != 0 && pool != 1) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_set_epilogue_pool: pool must be 0 or 1");
  if (pool && p->tm != 2)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_set_epilogue_pool: the fused pool needs tile_m = 2");
  if (pool && (p->OH < 2 || p->OW < 2))
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_plan_set_epilogue_pool: output smaller than 2x2");
  p->gemm_geom.pool = pool;
  p->gemm_geom.jsplit = (p->jsplit && !pool) ? 1 : 0;  // the fused pool needs the single-CTA fold
  return LANCE_OK;
}

int lance_plan_set_epilogue(lance_plan_t p, const float* bias_dev, int relu) {
  if (!p) return fail(LANCE_ERR_INVALID_ARGUMENT, "null plan");
  p->bias = bias_dev;
  p->relu = relu ? 1 : 0;
  return LANCE_OK;
}

int lance_plan_set_acc_dump(lance_plan_t p, int32_t* acc_dev) {
  if (!p) return fail(LANCE_ERR_INVALID_ARGUMENT, "null plan");
  p->acc_dump = acc_dev;
  return LANCE_OK;
}

int lance_plan_last_launch_count(lance_plan_t p) { return p ? p->last_launches : 0; }

int lance_plan_stage_timing(lance_plan_t p, int enable) {
  if (!p) return fail(LANCE_ERR_INVALID_ARGUMENT, "null plan");
  p->timing = enable != 0;
  p->recorded = 0;
  return LANCE_OK;
}

int lance_plan_read_stage_times(lance_plan_t p, double* sum_ms3, int* nforwards) {
  if (!p || !sum_ms3) return fail(LANCE_ERR_INVALID_ARGUMENT, "null argument");
  DeviceGuard guard(p->device);
  sum_ms3[0] = sum_ms3[1] = sum_ms3[2] = 0.0;
  for (int f = 0; f < p->recorded; ++f) {
    cudaEvent_t* ev = &p->events[size_t(4) * f];
    LANCE_CUDA(cudaEventSynchronize(ev[3]));
    for (int i = 0; i < 3; ++i) {
      float ms = 0.f;
      LANCE_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      sum_ms3[i] += ms;
    }
  }
  if (nforwards) *nforwards = p->recorded;
  p->recorded = 0;
  return LANCE_OK;
}

int lance_plan_sync(lance_plan_t p, void* stream) {
  if (!p) return fail(LANCE_ERR_INVALID_ARGUMENT, "null plan");
  DeviceGuard guard(p->device);
  LANCE_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  int flags[2];
  LANCE_CUDA(cudaMemcpy(flags, &p->state->nan_in, sizeof flags, cudaMemcpyDeviceToHost));
  if (flags[0] || flags[1]) return fail(LANCE_ERR_NAN, "fit_params: NaN in values");
  return LANCE_OK;
}

int lance_plan_get_params(lance_plan_t p, lance_qparams* in16, lance_qparams* w16) {
  if (!p) return fail(LANCE_ERR_INVALID_ARGUMENT, "null plan");
  DeviceGuard guard(p->device);
  LanceDevState st;
  LANCE_CUDA(cudaDeviceSynchronize());
  LANCE_CUDA(cudaMemcpy(&st, p->state, sizeof st, cudaMemcpyDeviceToHost));
  for (int i = 0; i < p->np; ++i) {
    if (in16) in16[i] = {p->cfg.bits_i, st.a_tmin[i], st.a_tmax[i], st.a_scale[i]};
    if (w16) w16[i] = {p->cfg.bits_w, st.w_tmin[i], st.w_tmax[i], st.w_scale[i]};
  }
  return LANCE_OK;
}

int lance_plan_debug_read(lance_plan_t p, int what, void* dst, size_t bytes) {
  if (!p || !dst) return fail(LANCE_ERR_INVALID_ARGUMENT, "null argument");
  DeviceGuard guard(p->device);
  LANCE_CUDA(cudaDeviceSynchronize());
  const long long M = p->M;
  const int C = p->spec.c, K = p->spec.k, np = p->np;
  switch (what) {
    case LANCE_DBG_CODES_A: {  // device UMMA images -> reference [np][M][C]
      if (bytes != size_t(np) * M * C) return fail(LANCE_ERR_INVALID_ARGUMENT, "bad size");
      std::string tmp(size_t(np) * ((M + kBM - 1) / kBM * kBM) * p->C_pad, '\0');
      LANCE_CUDA(cudaMemcpy(tmp.data(), p->codes_a, tmp.size(), cudaMemcpyDeviceToHost));
      auto* out = static_cast<uint8_t*>(dst);
      const int nk = p->C_pad / p->BK;
      for (int q = 0; q < np; ++q)
        for (long long m = 0; m < M; ++m)
          for (int c = 0; c < C; ++c)
            out[(size_t(q) * M + m) * C + c] = static_cast<uint8_t>(
                tmp[np == 16 ? umma_image_offset(m, c, q, kBM, p->BK, nk)
                             : umma_image_offset_np(m, c, f4_plane(q), kBM, p->BK, nk, np)]);
      return LANCE_OK;
    }
    case LANCE_DBG_ROWSUM: {
      if (bytes != sizeof(int32_t) * np * M) return fail(LANCE_ERR_INVALID_ARGUMENT, "bad size");
      LANCE_CUDA(cudaMemcpy2D(dst, sizeof(int32_t) * M, p->rowsum, sizeof(int32_t) * p->rs_pitch,
                              sizeof(int32_t) * M, np, cudaMemcpyDeviceToHost));
      return LANCE_OK;
    }
    case LANCE_DBG_CODES_W: {  // device UMMA images -> reference [np][C][K]
      if (bytes != size_t(np) * C * K) return fail(LANCE_ERR_INVALID_ARGUMENT, "bad size");
      std::string tmp(size_t(np) * p->K_pad * p->C_pad, '\0');
      LANCE_CUDA(cudaMemcpy(tmp.data(), p->codes_w, tmp.size(), cudaMemcpyDeviceToHost));
      auto* out = static_cast<uint8_t*>(dst);
      const int nk = p->C_pad / p->BK;
      for (int q = 0; q < np; ++q)
        for (int c = 0; c < C; ++c)
          for (int k = 0; k < K; ++k)
            out[(size_t(q) * C + c) * K + k] = static_cast<uint8_t>(
                tmp[np == 16 ? umma_image_offset(k, c, q, p->BN, p->BK, nk)
                             : umma_image_offset_np(k, c, f4_plane(q), p->BN, p->BK, nk, np)]);
      return LANCE_OK;
    }
    case LANCE_DBG_COLSUM: {
      if (bytes != sizeof(int32_t) * np * K) return fail(LANCE_ERR_INVALID_ARGUMENT, "bad size");
      LANCE_CUDA(cudaMemcpy2D(dst, sizeof(int32_t) * K, p->colsum, sizeof(int32_t) * p->K_pad,
                              sizeof(int32_t) * K, np, cudaMemcpyDeviceToHost));
      return LANCE_OK;
    }
    default:
      return fail(LANCE_ERR_INVALID_ARGUMENT, "unknown debug buffer");
  }
}

// --------------------------------------------------------------------------
// Host-buffer drop-in for lance::lance_gemm (engines.hpp:492-536).

namespace {
struct HostCtx {
  lance_plan_t plan = nullptr;
  float *x = nullptr, *w = nullptr, *y = nullptr;
  cudaStream_t stream = nullptr;
  size_t bytes = 0;  // plan + staging device bytes
};

void release(HostCtx& c) {
  if (c.stream) cudaStreamSynchronize(c.stream);
  lance_plan_destroy(c.plan);
  cudaFree(c.x);
  cudaFree(c.w);
  cudaFree(c.y);
  if (c.stream) cudaStreamDestroy(c.stream);
  c = HostCtx{};
}

using Key = std::tuple<int, int, int, int, int, int, int, int, int, int, int>;

// Per-thread LRU of host drop-in contexts (plan + staging buffers), bounded in
// entries and device bytes; the least recently used layers are released
// first and everything is freed when the thread exits.
struct HostCache {
  static constexpr size_t kMaxEntries = 16;
  static constexpr size_t kMaxBytes = size_t(8) << 30;
  std::list<std::pair<Key, HostCtx>> lru;  // front = most recent
  size_t bytes = 0;
  ~HostCache() { clear(); }
  void clear() {
    for (auto& kv : lru) release(kv.second);
    lru.clear();
    bytes = 0;
  }
  HostCtx* find(const Key& k) {
    for (auto it = lru.begin(); it != lru.end(); ++it)
      if (it->first == k) {
        lru.splice(lru.begin(), lru, it);
        return &lru.front().second;
      }
    return nullptr;
  }
  // Make room for an entry of `need` bytes.
  void evict_for(size_t need) {
    while (!lru.empty() && (lru.size() >= kMaxEntries || bytes + need > kMaxBytes)) {
      HostCtx& c = lru.back().second;
      bytes -= std::min(bytes, c.bytes);
      release(c);
      lru.pop_back();
    }
  }
};
thread_local HostCache g_host_cache;
}  // namespace

int lance_host_cache_clear(void) {
  g_host_cache.clear();
  return LANCE_OK;
}

int lance_gemm_host(const lance_conv_spec* spec, const lance_config* cfg, const float* x,
                    const float* w, float* y) {
  return lance_gemm_host_tiled(spec, cfg, 2, x, w, y);
}

int lance_gemm_host_tiled(const lance_conv_spec* spec, const lance_config* cfg, int tile_m,
                          const float* x, const float* w, float* y) {
  if (tile_m != 2 && tile_m != 4)
    return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_gemm: tile_m must be 2 or 4");
  int rc = validate(spec, cfg);
  if (rc) return rc;
  if (!x || !w || !y) return fail(LANCE_ERR_INVALID_ARGUMENT, "lance_gemm: null buffer");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return fail(LANCE_ERR_NO_DEVICE, "no CUDA device: the B200 lance_gemm path has no CPU fallback");
  }
  const Key key{dev, spec->n, spec->c, spec->h, spec->w, spec->k, spec->pad, cfg->bits_w,
                cfg->bits_i, cfg->granularity, tile_m};
  const size_t xb = sizeof(float) * size_t(spec->n) * spec->h * spec->w * spec->c;
  const size_t wb = sizeof(float) * size_t(spec->k) * 9 * spec->c;
  const size_t yb = sizeof(float) * size_t(spec->n) * out_h(*spec) * out_w(*spec) * spec->k;
  HostCtx* cp = g_host_cache.find(key);
  if (!cp) {
    g_host_cache.evict_for(xb + wb + yb);
    HostCtx c;
    if ((rc = lance_plan_create_tiled(spec, cfg, tile_m, dev, &c.plan))) return rc;
    cudaError_t e = cudaMalloc(&c.x, xb);
    if (e == cudaSuccess) e = cudaMalloc(&c.w, wb);
    if (e == cudaSuccess) e = cudaMalloc(&c.y, yb);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      release(c);
      return cuda_fail(e, "lance_gemm host staging");
    }
    c.bytes = lance_plan_device_bytes(c.plan) + xb + wb + yb;
    g_host_cache.lru.emplace_front(key, c);
    g_host_cache.bytes += c.bytes;
    cp = &g_host_cache.lru.front().second;
  }
  HostCtx& ctx = *cp;
  LANCE_CUDA(cudaMemcpyAsync(ctx.w, w, wb, cudaMemcpyHostToDevice, ctx.stream));
  LANCE_CUDA(cudaMemcpyAsync(ctx.x, x, xb, cudaMemcpyHostToDevice, ctx.stream));
  if ((rc = lance_plan_set_filters(ctx.plan, ctx.w, ctx.stream))) return rc;
  if ((rc = lance_plan_forward(ctx.plan, ctx.x, ctx.y, ctx.stream))) return rc;
  LANCE_CUDA(cudaMemcpyAsync(y, ctx.y, yb, cudaMemcpyDeviceToHost, ctx.stream));
  // One synchronisation per call; a NaN seen by the range passes is reported
  // like the reference's throw from fit_params (y is then unspecified).
  return lance_plan_sync(ctx.plan, ctx.stream);
}

}  // extern "C"
