/*
 * lance_b200.h -- C ABI of the B200-native LANCE int8 Winograd-domain
 * convolution (the reference's `lance_gemm` path).
 *
 * Reference: /root/reference/proj/include/lance/ (header-only C++20, no FFI).
 * Each entry point cites the reference interface it replaces.  The reference
 * has no C ABI; a C++ host above this ABI (include/lance/b200.hpp) keeps the
 * reference's operator API (ConvSpec / LanceConfig / QuantParams / Tensor4 /
 * FilterBank -> Tensor4) and its exception behaviour.
 *
 * Conventions: plain pointers and sizes; no exceptions cross the ABI; every
 * function returns a lance_status.  Device entry points are stream-ordered on
 * the caller's cudaStream_t (passed as void*).  x is NHWC fp32, w is KRSC fp32,
 * y is NHWC fp32 -- the reference layouts (tensor.hpp:24-86).
 */
#ifndef LANCE_B200_H
#define LANCE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LANCE_B200_ABI_VERSION 1

#if defined(__GNUC__)
#define LANCE_API __attribute__((visibility("default")))
#else
#define LANCE_API
#endif

/* lance::Granularity (quant.hpp:44), enum order kept. */
typedef enum {
  LANCE_GRAN_PER_TILE = 0,
  LANCE_GRAN_PER_POSITION = 1,
  LANCE_GRAN_PER_TENSOR = 2
} lance_granularity;

/* lance::LanceMode (engines.hpp:56). */
typedef enum { LANCE_MODE_FAITHFUL = 0, LANCE_MODE_GEMM = 1 } lance_mode;

/* lance::ConvSpec (engines.hpp:33-54).  r = s = 3 and stride = 1 are fixed. */
typedef struct {
  int n, c, h, w, k;
  int pad; /* 0 or 1 */
} lance_conv_spec;

/* lance::LanceConfig (engines.hpp:60-80). */
typedef struct {
  int bits_w;      /* 2..8 (32 = unquantized, rejected by the Gemm path) */
  int bits_i;      /* 2..8 */
  int granularity; /* lance_granularity */
  int mode;        /* lance_mode; must be LANCE_MODE_GEMM */
} lance_config;

/* lance::QuantParams (quant.hpp:27-37), bit-for-bit. */
typedef struct {
  int bits;
  float t_min, t_max, scale;
} lance_qparams;

typedef enum {
  LANCE_OK = 0,
  LANCE_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (engines.hpp:46-91,496-499) */
  LANCE_ERR_NAN = 2,              /* std::invalid_argument("fit_params: NaN in values"), quant.hpp:62 */
  LANCE_ERR_CUDA = 3,             /* CUDA runtime / launch failure */
  LANCE_ERR_NO_DEVICE = 4         /* no sm_100 device: the path has no CPU fallback */
} lance_status;

typedef struct lance_plan_s* lance_plan_t;

LANCE_API int lance_abi_version(void);
LANCE_API const char* lance_status_string(int status);
/* Message of the last failure on the calling thread (the what() text the
 * reference would have thrown). */
LANCE_API const char* lance_last_error(void);

/* Validation exactly as lance_gemm performs it before any work:
 * ConvSpec::validate (engines.hpp:46-53), LanceConfig::validate (:66-79),
 * the Gemm-mode and depth checks (:496-499). */
LANCE_API int lance_validate(const lance_conv_spec* spec, const lance_config* cfg);

/* Product-stage multiply counts (engines.hpp:568-575). */
LANCE_API uint64_t lance_winograd_multiply_count(const lance_conv_spec* spec);
LANCE_API uint64_t lance_direct_multiply_count(const lance_conv_spec* spec);

/* ---------------------------------------------------------------------------
 * Drop-in for lance::lance_gemm(x, w, spec, cfg) -> y (engines.hpp:492-536):
 * HOST buffers in and out, synchronous.  x [N][H][W][C], w [K][3][3][C],
 * y [N][OH][OW][K].  Internally caches one plan per (spec, cfg) per thread
 * (bounded LRU, see lance_host_cache_clear).
 * Pinned (page-locked) host buffers give full-bandwidth copies. */
LANCE_API int lance_gemm_host(const lance_conv_spec* spec, const lance_config* cfg, const float* x,
                    const float* w, float* y);
/* The host drop-in keeps a per-thread LRU of layer contexts (at most 16
 * layers / 8 GiB of device memory; freed at thread exit).  This releases the
 * calling thread's contexts now. */
LANCE_API int lance_host_cache_clear(void);

/* ---------------------------------------------------------------------------
 * Device API.  A plan owns the per-layer state: prepared filter codes (K2),
 * the int8 input-code workspace, per-position parameters and epilogue
 * constants.  One plan serves one stream at a time. */
LANCE_API int lance_plan_create(const lance_conv_spec* spec, const lance_config* cfg, int device,
                      lance_plan_t* plan);
LANCE_API int lance_plan_destroy(lance_plan_t plan);
LANCE_API size_t lance_plan_device_bytes(lance_plan_t plan);

/* K2: filter transform G g G^T + Winograd-domain quantization, once per layer
 * (domain_from_filters + quantize_domain(u), engines.hpp:215-233,140-183). */
LANCE_API int lance_plan_set_filters(lance_plan_t plan, const float* w_dev, void* stream);

/* K0 -> K1 -> K3/K4 on a device-resident batch: per-position input ranges
 * (quantize_domain(v) fit, engines.hpp:157-165), transform + quantize, and the
 * 16 u8 x u8 -> i32 GEMMs on tcgen05 with the fused affine de-quantization +
 * A^T m A + merge epilogue.  Asynchronous; NaN inputs are reported by
 * lance_plan_sync (the reference throws from fit_params). */
LANCE_API int lance_plan_forward(lance_plan_t plan, const float* x_dev, float* y_dev, void* stream);

/* Static-params variant: the caller supplies the 16 input QuantParams
 * (no range pass, no batch coupling; SURVEY.md section 8(e) mode 3). */
LANCE_API int lance_plan_forward_static(lance_plan_t plan, const lance_qparams* in_params16,
                              const float* x_dev, float* y_dev, void* stream);

/* Global-fit mode across batch shards (SURVEY.md section 8(e) mode 2): the
 * reference fits the PerPosition ranges over the WHOLE batch
 * (quantize_domain, engines.hpp:157-165; fit_params, quant.hpp:54-72), so a
 * batch split over G GPUs reproduces one full-batch lance_gemm call by
 *   1. lance_plan_ranges on every shard (K0 only): writes the shard's fitted
 *      ranges to minmax_dev as 2*P+1 floats [-t_min[0..P), t_max[0..P), nan];
 *   2. ONE element-wise MAX all-reduce of that buffer across ranks (e.g.
 *      ncclAllReduce(..., ncclFloat, ncclMax), 2*P+1 floats, on the stream);
 *   3. lance_plan_forward_ranges: re-fits the input QuantParams from the
 *      reduced ranges on the device, then K1 -> K3/K4.
 * Stream-ordered, no host synchronisation.  P = lance_plan_positions(plan).
 * A NaN anywhere in the global batch is reported by lance_plan_sync. */
LANCE_API int lance_plan_ranges(lance_plan_t plan, const float* x_dev, float* minmax_dev, void* stream);
LANCE_API int lance_plan_forward_ranges(lance_plan_t plan, const float* minmax_dev,
                                        const float* x_dev, float* y_dev, void* stream);

/* Input layout of subsequent forwards / range passes (north-star option; the
 * reference is NHWC-only, tensor.hpp:24-55).  LANCE_LAYOUT_NCHW reads x as
 * [N][C][H][W] fp32 (PyTorch's default): a shared-memory tiled transpose with
 * coalesced 128-bit channel-row loads stages it as NHWC in plan memory (one
 * extra launch, N*H*W*C*4 bytes), then the NHWC kernels run, so codes,
 * parameters and y (NHWC) are bit-identical to the NHWC path.  Needs
 * N * H < 65536. */
#define LANCE_LAYOUT_NHWC 0
#define LANCE_LAYOUT_NCHW 1
LANCE_API int lance_plan_set_input_layout(lance_plan_t plan, int layout);
LANCE_API int lance_plan_input_layout(lance_plan_t plan);

/* Optional fused bias + ReLU epilogue for subsequent forwards (north-star
 * extension; no reference oracle: equals relu(lance_gemm(x, w) + bias)).
 * bias_dev may be NULL (no bias).  relu is 0 or 1. */
LANCE_API int lance_plan_set_epilogue(lance_plan_t plan, const float* bias_dev, int relu);

/* Optional fused 2x2 / stride-2 max-pool after the (bias + ReLU) epilogue
 * (layer-stack option; no reference oracle:
 * equals lance_maxpool2x2_nhwc(relu(lance_gemm(x, w) + bias)), floor pooling).
 * With pool = 1, y is [N][OH/2][OW/2][K].  F(2x2) plans only. */
LANCE_API int lance_plan_set_epilogue_pool(lance_plan_t plan, int pool);

/* Synchronise `stream` and report a NaN seen by the range pass of the last
 * forward (LANCE_ERR_NAN) or any pending CUDA error. */
LANCE_API int lance_plan_sync(lance_plan_t plan, void* stream);

/* Parameters of the last forward / set_filters (synchronises the device). */
LANCE_API int lance_plan_get_params(lance_plan_t plan, lance_qparams* input16, lance_qparams* weight16);

/* Debug / parity access to intermediate stage buffers (synchronising copies to
 * host memory in the reference layouts):
 *   LANCE_DBG_CODES_A  u8  [16][M][C]   (vq.codes, engines.hpp:505)
 *   LANCE_DBG_ROWSUM   i32 [16][M]      (a_row_sum, lowpgemm.hpp:121-123)
 *   LANCE_DBG_CODES_W  u8  [16][C][K]   (uq.codes, engines.hpp:506)
 *   LANCE_DBG_COLSUM   i32 [16][K]      (b_col_sum, lowpgemm.hpp:124-126)
 * M = N * tiles_per_image.  `bytes` must equal the array size. */
enum { LANCE_DBG_CODES_A = 1, LANCE_DBG_ROWSUM = 2, LANCE_DBG_CODES_W = 3, LANCE_DBG_COLSUM = 4 };
LANCE_API int lance_plan_debug_read(lance_plan_t plan, int what, void* dst_host, size_t bytes);

/* When acc_dev is non-NULL, subsequent forwards also write the raw int32
 * accumulators [16][M][K] (gemm_codes per position, lowpgemm.hpp:76-100)
 * from the same GEMM kernel.  Pass NULL to disable. */
LANCE_API int lance_plan_set_acc_dump(lance_plan_t plan, int32_t* acc_dev);

/* Per-stage device timing (CUDA events recorded on the forward's stream
 * between the K0 / K1 / K3-K4 launches).  enable != 0 starts recording (up to
 * 4096 forwards); read_stage_times synchronises those events and returns the
 * summed milliseconds of {K0 range, K1 quantize, K3/K4 GEMM+epilogue} and the
 * number of forwards they cover, then clears the record. */
LANCE_API int lance_plan_stage_timing(lance_plan_t plan, int enable);
LANCE_API int lance_plan_read_stage_times(lance_plan_t plan, double* sum_ms3, int* nforwards);

/* Kernel launches issued by the most recent forward on this plan. */
LANCE_API int lance_plan_last_launch_count(lance_plan_t plan);

/* ---------------------------------------------------------------------------
 * F(4x4,3x3) extension (not in the reference,
 * whose extract_tiles rejects m != 2, tensor.hpp:117-118).  tile_m = 2 is
 * exactly lance_plan_create / lance_gemm_host; tile_m = 4 runs the same
 * algorithm with 6x6 tiles at stride 4 and 36 Winograd positions (SURVEY.md
 * Appendix D basis, reference matmul order).  On a tile_m = 4 plan every
 * per-position array of the API holds 36 entries instead of 16:
 * lance_plan_forward_static / lance_plan_get_params take 36 lance_qparams,
 * the debug buffers are [36][...] and the acc dump is [36][M][K], with
 * M = N * ceil(OH/4) * ceil(OW/4). */
LANCE_API int lance_plan_create_tiled(const lance_conv_spec* spec, const lance_config* cfg,
                                      int tile_m, int device, lance_plan_t* plan);
/* Winograd positions of the plan: 16 (tile_m 2) or 36 (tile_m 4). */
LANCE_API int lance_plan_positions(lance_plan_t plan);
LANCE_API int lance_gemm_host_tiled(const lance_conv_spec* spec, const lance_config* cfg,
                                    int tile_m, const float* x, const float* w, float* y);
/* (m+2)^2 * tiles * N * C * K for tile side m (engines.hpp:573-575 generalised). */
LANCE_API uint64_t lance_winograd_multiply_count_tiled(const lance_conv_spec* spec, int tile_m);

/* Layer-stack glue (not part of lance_gemm):
 * 2x2 / stride-2 max-pool of a device NHWC tensor, y [n][h/2][w/2][c], on
 * `stream` -- the pooling between VGG-16-CIFAR conv stages (BASELINE config 2). */
LANCE_API int lance_maxpool2x2_nhwc(const float* x_dev, float* y_dev, int n, int h, int w, int c,
                                    void* stream);

/* The CLI's output checksum (lance_main.cpp:41-51): FNV-1a 64 over the
 * little-endian bytes of `count` floats.  Host memory, no device needed. */
LANCE_API uint64_t lance_fnv1a64(const float* data, size_t count);

/* Synthetic-input fixture: lance::UniformSource(seed) stream (rng.hpp:27-47),
 * mt19937_64 top-24-bit -> U(-1,1).  Host memory. */
LANCE_API void lance_uniform_fill(uint64_t seed, float* out, size_t count);

#ifdef __cplusplus
}
#endif
#endif /* LANCE_B200_H */
