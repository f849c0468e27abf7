// lance_kernels.cuh -- device state, launch geometry and kernel entry points
// of the B200 LANCE path (reference: engines.hpp:492-536).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lance_dev {

constexpr int kPositions = 16;  // (m + r - 1)^2 for F(2x2,3x3)
constexpr int kBM = 128;        // GEMM rows (Winograd tiles) per CTA = UMMA M
constexpr int kBN = 32;         // filters per CTA: 16 positions x 32 = 512 TMEM columns
constexpr int kGemmThreads = 192;
constexpr int kStages = 8;

// Per-plan device state, written by the range / filter finalisers and read by
// the quantiser and the GEMM epilogue.  Mirrors QuantParams (quant.hpp:27-37)
// for both operands plus the hoisted affine constants of affine_term
// (lowpgemm.hpp:110-114): m = ((k1*dot + k2*sum_a) + k3*sum_b) + k4.
struct LanceDevState {
  float a_tmin[kPositions], a_tmax[kPositions], a_scale[kPositions];
  float w_tmin[kPositions], w_tmax[kPositions], w_scale[kPositions];
  float k1[kPositions], k2[kPositions], k3[kPositions], k4[kPositions];
  int bits_i, bits_w;
  int nan_in, nan_w;
  unsigned int ticket_in, ticket_w;
};

// Input-side geometry shared by the range pass (K0) and the quantiser (K1).
struct InGeom {
  long long M;         // GEMM rows = N * P
  int P, TW;           // tiles per image, tiles per image row
  int H, W, C, C4;     // image dims, channels, ceil(C / 4)
  int C_pad;           // code row pitch (multiple of 32)
  int pad;
  int G;               // threads per tile (power of two, <= 32)
  int TPB;             // tiles per 256-thread block
  long long num_tile_blocks;
  int granularity;     // 1 = PerPosition, 2 = PerTensor
};

struct FilterGeom {
  int K, C, K_pad, C_pad;
  int granularity;
};

struct GemmGeom {
  long long M;
  int K, C;
  int P, TW, OH, OW;
  int num_kchunks;  // C_pad / BK
  int num_n_tiles;  // K_pad / kBN
};

// Host-side launchers (lance_kernels.cu).  All stream-ordered.
cudaError_t launch_input_range(const float* x, float* partials, int grid, LanceDevState* st,
                               const InGeom& g, int vec4, cudaStream_t s);
cudaError_t launch_input_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                               const LanceDevState* st, const InGeom& g, int vec4,
                               cudaStream_t s);
struct StaticParams {
  float tmin[kPositions], tmax[kPositions], scale[kPositions];
};
cudaError_t launch_static_params(LanceDevState* st, const StaticParams& prm, int C,
                                 cudaStream_t s);
cudaError_t launch_filter_prepare(const float* w, float* u_tmp, float* partials, int grid,
                                  uint8_t* codes_w, int32_t* colsum, LanceDevState* st,
                                  const FilterGeom& g, cudaStream_t s);
cudaError_t launch_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, int bk,
                        const int32_t* rowsum, const int32_t* colsum, const LanceDevState* st,
                        float* y, int32_t* acc_dump, const float* bias, int relu,
                        const GemmGeom& g, cudaStream_t s);

}  // namespace lance_dev
