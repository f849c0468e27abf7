// lance_kernels.cuh -- device state, launch geometry and launchers of the B200
// LANCE path (reference: engines.hpp:492-536).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#ifndef LANCE_JMAJOR
#define LANCE_JMAJOR 0
#endif

namespace lance_dev {

constexpr int kPositions = 16;     // (m + r - 1)^2 for F(2x2,3x3)
constexpr int kMaxPositions = 36;  // F(4x4,3x3) extension (lance_f4.cu)
constexpr int kBM = 128;        // GEMM rows (Winograd tiles) per CTA = UMMA M
constexpr int kChunk = 64;      // channels per K0/K1 warp item (32 lanes x 2)

// Per-plan device state, written by the range / filter finalisers and read by
// the quantiser and the GEMM epilogue.  Mirrors QuantParams (quant.hpp:27-37)
// for both operands plus the hoisted affine constants of affine_term
// (lowpgemm.hpp:110-114): m = ((k1*dot + k2*sum_a) + k3*sum_b) + k4.
struct LanceDevState {
  float a_tmin[kMaxPositions], a_tmax[kMaxPositions], a_scale[kMaxPositions], a_rcp[kMaxPositions];
  float w_tmin[kMaxPositions], w_tmax[kMaxPositions], w_scale[kMaxPositions];
  float k1[kMaxPositions], k2[kMaxPositions], k3[kMaxPositions], k4[kMaxPositions];
  int bits_i, bits_w;
  int nan_in, nan_w;
  unsigned int ticket_in, ticket_w;
};

// Input-side geometry shared by the range pass (K0) and the quantiser (K1).
struct InGeom {
  int M;          // GEMM rows = N * P (< 2^31, checked at plan creation)
  int P, TH, TW;  // tiles per image, tile rows / columns per image
  int H, W, C;    // image dims, channels
  int C_pad;      // code row pitch (multiple of 32)
  int rs_pitch;   // row-sum plane pitch (M rounded up to 4: 16-byte TMA strides)
  int a_bk;       // GEMM K chunk (32, 64 or 128 channels): codes are stored as UMMA images
  int a_nk;       // C_pad / a_bk
  int rowsums;    // K1 fast path writes row sums (0 when the GEMM computes them)
  int rev_items;  // K1 walks its work items back to front (L2 reuse, LANCE_K1_REVERSE)
  int pad;
  int nchunks;    // ceil(C_pad / kChunk)
  int seg_len;    // tiles per warp strip (a tile row is split into nseg strips)
  int nseg;
  long long num_items;  // N * TH * nseg * nchunks warp items
  int granularity;  // 1 = PerPosition, 2 = PerTensor
  int32_t* rs_zero;       // K0 zeroes these words for K1's atomic row sums (nullptr: nothing)
  long long rs_zero_words;
};

struct FilterGeom {
  int K, C, K_pad, C_pad;
  int granularity;
  int bk, bn, nk;  // UMMA image geometry of the B operand (see umma_image_offset)
};

struct GemmGeom {
  int M;
  int K, C;
  int P, TW, OH, OW;
  int num_kchunks;  // C_pad / BK
  int num_n_tiles;  // K_pad / BN
  int stages;       // shared-memory ring depth (set by the launcher)
  int b_resident;   // B operand resident in shared memory (set by the launcher)
  int rs_pitch;     // row-sum plane pitch (acc-dump builds write the GEMM's row sums)
  int rs_warps;     // 1: the GEMM sums the A rows itself; 0: K1's row sums via TMA
  int units;        // k chunks per stage (0 = auto); the launcher settles it
  int exp;          // experiment switches (LANCE_GEMM_EXP, profiling only; 0 = normal)
  int pool;         // 1: fused 2x2 / stride-2 max-pool, y is [N][OH/2][OW/2][K]
  int jsplit;       // 1: a tile's 4 j-groups on 4 CTAs (small-M layers, BN = 64)
  float* tscratch;  // jsplit: [tiles][4 j][T0, T1][128 rows][BN] fp32
  int* tticket;     // jsplit: per-tile arrival counters (self-resetting)
  int stage_out;    // 1: y through the shared-memory staging buffer (128-byte lines); 0: from registers (BN = 64)
  unsigned long long* trace;  // CTA-0 event timestamps (LANCE_GEMM_TRACE, profiling only)
};

// Operand codes are stored in global memory exactly as the GEMM's shared-memory
// stages hold them, so one contiguous bulk copy fills a stage: the operand
// [rows][C_pad] u8 is cut into images of `rows_per_img` rows x bk channels
// (128 for A, BN for B), each image K-major with the UMMA / TMA swizzle of a
// bk-byte row (SWIZZLE_128B / 64B / 32B: 16-byte chunk c of row r sits at
// chunk c ^ f(r), i.e. byte bit 4+ ^= bits 7+), ordered
// [row block][j][a][k chunk][image] for position p = 4a + j (j-major: the
// GEMM consumes positions in j-groups, and a stage copies consecutive units).
// Plane order of the 16 positions inside a row block (kJMajorImages: j-major).
constexpr bool kJMajorImages = LANCE_JMAJOR;
__host__ __device__ __forceinline__ constexpr int image_plane(int p) {
  return kJMajorImages ? (p & 3) * 4 + (p >> 2) : p;
}
__host__ __device__ __forceinline__ uint32_t umma_swizzle(uint32_t lin, int bk) {
  const uint32_t mask = bk == 128 ? 7u : (bk == 64 ? 3u : 1u);
  return lin ^ (((lin >> 7) & mask) << 4);
}
__host__ __device__ __forceinline__ long long umma_image_offset(long long row, int c, int p,
                                                                 int rows_per_img, int bk,
                                                                 int nk) {
  const long long blk = row / rows_per_img;
  const int r = static_cast<int>(row - blk * rows_per_img);
  const int kc = c / bk, cb = c - kc * bk;
  const int pj = image_plane(p);
  return ((blk * 16 + pj) * nk + kc) * static_cast<long long>(rows_per_img * bk) +
         umma_swizzle(static_cast<uint32_t>(r * bk + cb), bk);
}

struct StaticParams {
  float tmin[kMaxPositions], tmax[kMaxPositions], scale[kMaxPositions];
  int np;  // positions in use (16, or 36 for F(4x4))
};

// F(4x4,3x3) geometry (lance_f4.cu): 6x6 input tiles at stride 4, 36
// positions, BN = 16 filters per GEMM tile.
struct F4Geom {
  int N, H, W, C, K, pad;
  int OH, OW, TH, TW, P;
  int M;             // N * P GEMM rows
  int C_pad, K_pad;  // C_pad = nk * bk, K_pad multiple of 16
  int bk, nk;        // UMMA image K chunk (32 / 64 / 128 channels) and chunks
  int rs_pitch;      // row-sum plane pitch
  int granularity;   // 1 PerPosition, 2 PerTensor
  int num_n_tiles;   // K_pad / 16
  int stages;        // GEMM ring depth (set by the launcher)
  int units;         // (position, k chunk) units per GEMM stage (divides 6 * nk; launcher)
  int b_resident;    // the CTA's filter tile stays in shared memory (launcher)
  int exp;           // experiment switches (LANCE_F4_EXP, profiling only; 0 = normal)
  int seg_len, nseg; // F0 / F1 strips: tiles per warp strip, strips per tile row
  long long num_items;  // N * TH * nseg * ceil(C / 32) warp strips
  int32_t* rs_zero;     // F0 zeroes the row sums F1 accumulates (nullptr: F1's launcher does)
  long long rs_zero_words;
};

// F(4x4) operand planes are j-major: position p = 6a + j is plane 6j + a, so
// the 6 positions of a GEMM j-group {6a + j} (and their k chunks) are one
// contiguous run and a stage can copy several units at once.
__host__ __device__ __forceinline__ constexpr int f4_plane(int p) { return (p % 6) * 6 + p / 6; }

// The operand image offset of umma_image_offset for np position planes; `p`
// is the PLANE index (F(4x4): f4_plane(position)).
__host__ __device__ __forceinline__ long long umma_image_offset_np(long long row, int c, int p,
                                                                    int rows_per_img, int bk,
                                                                    int nk, int np) {
  const long long blk = row / rows_per_img;
  const int r = static_cast<int>(row - blk * rows_per_img);
  const int kc = c / bk, cb = c - kc * bk;
  return ((blk * np + p) * nk + kc) * static_cast<long long>(rows_per_img * bk) +
         umma_swizzle(static_cast<uint32_t>(r * bk + cb), bk);
}

// Profiling-only kernel experiment switches (GemmGeom::exp / F4Geom::exp):
// compiled out of release builds, so their per-chunk tests cost nothing.
#ifdef LANCE_PROFILING
constexpr bool kExpSwitches = true;
#else
constexpr bool kExpSwitches = false;
#endif

// Experiment switches: the environment value in LANCE_PROFILING builds, else def.
int lance_knob(const char* name, int def);

// Thread-safe, per-device dynamic shared-memory opt-in: raises the attribute
// of kernel `fn` on the current device to at least `bytes` (cached per
// (device, kernel) behind a mutex; plans may be created from several host
// threads, one per GPU).
cudaError_t ensure_smem_attr(const void* fn, size_t bytes);
// Multiprocessor count of the current device (cached, thread-safe).
int current_sm_count();

// Programmatic dependent launch (kernels call pdl_entry() first).  Off by
// default: measured 1.2 % SLOWER on the ResNet-18 step (2.444 vs 2.416 ms,
// gpurun_out/pdl); LANCE_PDL=1 in profiling builds turns it on.
bool pdl_enabled();
#define LANCE_LAUNCH_CHECK(call)                  \
  do {                                            \
    const cudaError_t lance_e_ = (call);          \
    if (lance_e_ != cudaSuccess) return lance_e_; \
  } while (0)
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Host-side launchers.  All stream-ordered.
int input_range_grid(const InGeom& g, int sm_count);
cudaError_t launch_input_range(const float* x, float* partials, int grid, LanceDevState* st,
                               const InGeom& g, int vec2, cudaStream_t s);
cudaError_t launch_input_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                               const LanceDevState* st, const InGeom& g, int vec2,
                               int static_mode, cudaStream_t s);
// NCHW input: staging transpose x [N][C][H][W] -> xt [N][H][W][C] (then the
// NHWC K0 / K1).  grid.y = N * H must stay below 65536 (checked by the plan).
cudaError_t launch_nchw_to_nhwc(const float* x, float* xt, int N, int C, int H, int W, cudaStream_t s);
cudaError_t launch_static_params(LanceDevState* st, const StaticParams& prm, int C,
                                 cudaStream_t s);
// Global-fit mode: [-t_min[np], t_max[np], nan] export / re-fit on the device.
cudaError_t launch_export_minmax(const LanceDevState* st, float* minmax, int np, cudaStream_t s);
cudaError_t launch_fit_minmax(LanceDevState* st, const float* minmax, int np, int gran, int C,
                              cudaStream_t s);
cudaError_t launch_filter_prepare(const float* w, float* u_tmp, float* partials, int grid,
                                  uint8_t* codes_w, int32_t* colsum, LanceDevState* st,
                                  const FilterGeom& g, cudaStream_t s);
// bn: filters per GEMM tile (16, 32 or 64); TMEM holds two j-groups of 4 x bn columns.
cudaError_t launch_gemm(const uint8_t* codes_a, const uint8_t* codes_w, const CUtensorMap* tmR,
                        int32_t* rowsum_out,
                        int bk, int bn, int small_acc, const int32_t* colsum,
                        const LanceDevState* st, float* y, int32_t* acc_dump, const float* bias,
                        int relu, const GemmGeom& g, cudaStream_t s);

// Layer-stack glue (lance_stack.cu).
cudaError_t launch_maxpool2x2(const float* x, float* y, int N, int H, int W, int C, int sm_count,
                              cudaStream_t s);

// F(4x4,3x3) launchers (lance_f4.cu).
int f4_range_grid(const F4Geom& g, int sm_count);
cudaError_t launch_f4_range(const float* x, float* partials, int grid, LanceDevState* st,
                            const F4Geom& g, cudaStream_t s);
cudaError_t launch_f4_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                            const LanceDevState* st, const F4Geom& g, int static_mode,
                            int clear_rowsum, int sm_count, cudaStream_t s);
cudaError_t launch_f4_filter_prepare(const float* w, float* u_tmp, float* partials, int grid,
                                     uint8_t* codes_w, int32_t* colsum, LanceDevState* st,
                                     const F4Geom& g, cudaStream_t s);
cudaError_t launch_f4_gemm(const uint8_t* codes_a, const uint8_t* codes_w, const int32_t* rowsum,
                           const int32_t* colsum, int small_acc, const LanceDevState* st, float* y,
                           int32_t* acc_dump, const float* bias, int relu, const F4Geom& g,
                           cudaStream_t s);

}  // namespace lance_dev
