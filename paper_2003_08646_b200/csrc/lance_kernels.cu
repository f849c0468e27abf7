// lance_kernels.cu -- the four stages of the LANCE lance_gemm path on sm_100a.
//
//   K0  input_range_kernel    per-position (min, max) of B^T d B over the whole
//                             batch (quantize_domain/fit_params,
//                             engines.hpp:157-165, quant.hpp:54-72) + finaliser
//                             producing QuantParams[16] and the epilogue
//                             constants.
//   K1  input_quant_kernel    B^T d B recomputed and quantised to u8 codes
//                             (quant.hpp:77-84) + row sums (lowpgemm.hpp:121-123).
//   K2  filter_* kernels      G g G^T + per-position fit + codes + column sums
//                             (engines.hpp:215-233, lowpgemm.hpp:124-126).
//   K3/K4 gemm_epilogue_kernel  16 u8 x u8 -> s32 GEMMs on tcgen05 kind::i8
//                             (TMA-fed, accumulators in TMEM) with the fused
//                             affine de-quantisation (lowpgemm.hpp:110-114),
//                             A^T m A (winograd.hpp:80-84) and merge
//                             (tensor.hpp:157-182).
//
// Bit-exactness: every floating-point operation below is
// an explicit IEEE round-to-nearest intrinsic in the reference's association
// order; the file is compiled with -fmad=false and without fast-math.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "lance_kernels.cuh"
#include "lance_ptx.cuh"

namespace lance_dev {

// --------------------------------------------------------------------------
// Transforms (winograd.hpp:40-84 evaluated in matrix.hpp:75-84 order).  The
// products with zero basis entries only affect signed zeros; zero signs are
// canonicalised where they are observable (ranges and y).

// v = (B^T d) B for one channel; d, v indexed [a*4 + b].
__device__ __forceinline__ void input_transform(const float (&d)[16], float (&v)[16]) {
  float t[16];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    t[0 * 4 + b] = __fsub_rn(d[0 * 4 + b], d[2 * 4 + b]);
    t[1 * 4 + b] = __fadd_rn(d[1 * 4 + b], d[2 * 4 + b]);
    t[2 * 4 + b] = __fsub_rn(d[2 * 4 + b], d[1 * 4 + b]);
    t[3 * 4 + b] = __fsub_rn(d[1 * 4 + b], d[3 * 4 + b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    v[a * 4 + 0] = __fsub_rn(t[a * 4 + 0], t[a * 4 + 2]);
    v[a * 4 + 1] = __fadd_rn(t[a * 4 + 1], t[a * 4 + 2]);
    v[a * 4 + 2] = __fsub_rn(t[a * 4 + 2], t[a * 4 + 1]);
    v[a * 4 + 3] = __fsub_rn(t[a * 4 + 1], t[a * 4 + 3]);
  }
}

// u = (G g) G^T for one (k, c); g indexed [r*3 + s].
__device__ __forceinline__ void filter_transform(const float (&g)[9], float (&u)[16]) {
  float h[12];  // h[a*3 + s] = (G g)(a, s)
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const float g0 = g[0 * 3 + s], g1 = g[1 * 3 + s], g2 = g[2 * 3 + s];
    h[0 * 3 + s] = g0;
    h[1 * 3 + s] = __fadd_rn(__fadd_rn(__fmul_rn(0.5f, g0), __fmul_rn(0.5f, g1)),
                             __fmul_rn(0.5f, g2));
    h[2 * 3 + s] = __fadd_rn(__fsub_rn(__fmul_rn(0.5f, g0), __fmul_rn(0.5f, g1)),
                             __fmul_rn(0.5f, g2));
    h[3 * 3 + s] = g2;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float x0 = h[a * 3 + 0], x1 = h[a * 3 + 1], x2 = h[a * 3 + 2];
    u[a * 4 + 0] = x0;
    u[a * 4 + 1] = __fadd_rn(__fadd_rn(__fmul_rn(0.5f, x0), __fmul_rn(0.5f, x1)),
                             __fmul_rn(0.5f, x2));
    u[a * 4 + 2] = __fadd_rn(__fsub_rn(__fmul_rn(0.5f, x0), __fmul_rn(0.5f, x1)),
                             __fmul_rn(0.5f, x2));
    u[a * 4 + 3] = x2;
  }
}

// quantize (quant.hpp:77-84): scale == 0 -> 0; units = roundf((x - tmin) / scale)
// with IEEE division and half-away-from-zero rounding; clamp to [0, top].
// For q >= 0.5 (and q < 2^23) round-half-away(q) == floor(RN(q + 0.5)); every
// q < 0.5 (negatives, NaN) maps to 0; q >= 2^23 saturates to top either way.
__device__ __forceinline__ uint32_t quantize_code(float v, float tmin, float scale, float top) {
  const float d = __fsub_rn(v, tmin);
  const float q = __fdiv_rn(d, scale);
  const float r = floorf(__fadd_rn(q, 0.5f));
  const float c = (q >= 0.5f) ? fminf(r, top) : 0.0f;
  return (scale == 0.0f) ? 0u : static_cast<uint32_t>(c);
}

// --------------------------------------------------------------------------
// Tile gather: the 4x4 x 4-channel block of tile m starting at channel c0
// (extract_tiles, tensor.hpp:116-152: origin (2ti - pad, 2tj - pad), zero pad).
template <int VEC>
__device__ __forceinline__ void load_tile(const float* __restrict__ x, const InGeom& g,
                                          long long m, int c0, float (&d)[16][4]) {
  const long long img = m / g.P;
  const int t = static_cast<int>(m - img * g.P);
  const int ti = t / g.TW, tj = t - ti * g.TW;
  const int y0 = 2 * ti - g.pad, x0 = 2 * tj - g.pad;
  const float* base = x + img * static_cast<long long>(g.H) * g.W * g.C;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int yy = y0 + a;
    const bool rok = (yy >= 0) && (yy < g.H);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int xx = x0 + b;
      const bool ok = rok && (xx >= 0) && (xx < g.W);
      const float* px = base + (static_cast<long long>(yy) * g.W + xx) * g.C + c0;
      if (VEC == 4) {
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok) q = __ldg(reinterpret_cast<const float4*>(px));
        d[a * 4 + b][0] = q.x;
        d[a * 4 + b][1] = q.y;
        d[a * 4 + b][2] = q.z;
        d[a * 4 + b][3] = q.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          d[a * 4 + b][j] = (ok && c0 + j < g.C) ? __ldg(px + j) : 0.0f;
      }
    }
  }
}

// Block-wide (min, max) partials -> last block folds them into the 16
// QuantParams (fit_params semantics) and returns true in that block.
__device__ __forceinline__ bool block_minmax_and_ticket(float (&lo)[16], float (&hi)[16],
                                                        float* partials, unsigned int* ticket,
                                                        float* s_red /*[8][32]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int p = 0; p < 16; ++p) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      lo[p] = fmin_nan(lo[p], __shfl_xor_sync(0xffffffffu, lo[p], off));
      hi[p] = fmax_nan(hi[p], __shfl_xor_sync(0xffffffffu, hi[p], off));
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      s_red[warp * 32 + p] = lo[p];
      s_red[warp * 32 + 16 + p] = hi[p];
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int i = threadIdx.x;
    float r = s_red[i];
    const int nw = blockDim.x >> 5;
    for (int w = 1; w < nw; ++w) r = (i < 16) ? fmin_nan(r, s_red[w * 32 + i]) : fmax_nan(r, s_red[w * 32 + i]);
    partials[static_cast<long long>(blockIdx.x) * 32 + i] = r;
  }
  __threadfence();
  __syncthreads();
  __shared__ unsigned int s_last;
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  // Last block: reduce all partials. Thread t handles column t % 32.
  const int col = threadIdx.x & 31;
  float r = (col < 16) ? __int_as_float(0x7f800000) : __int_as_float(0xff800000);
  for (int b = threadIdx.x >> 5; b < static_cast<int>(gridDim.x); b += blockDim.x >> 5) {
    const float v = __ldcg(partials + static_cast<long long>(b) * 32 + col);
    r = (col < 16) ? fmin_nan(r, v) : fmax_nan(r, v);
  }
  __syncthreads();
  s_red[threadIdx.x] = r;  // blockDim.x == 256 -> [8][32]
  __syncthreads();
  if (threadIdx.x < 32) {
    float q = s_red[threadIdx.x];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      q = (threadIdx.x < 16) ? fmin_nan(q, s_red[w * 32 + threadIdx.x])
                             : fmax_nan(q, s_red[w * 32 + threadIdx.x]);
    s_red[threadIdx.x] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// fit_params for one operand from the reduced (lo[16], hi[16]) in s_red[0..31]
// (quant.hpp:54-72); PerTensor (engines.hpp:151-156) folds the 16 ranges and
// param_at() returns params[0] for every position (engines.hpp:131-136).
__device__ __forceinline__ void fit_from_ranges(const float* s_red, int gran, int bits,
                                                float* tmin, float* tmax, float* scale,
                                                int* nan_flag) {
  if (threadIdx.x < 16) {
    const int p = threadIdx.x;
    float lo = s_red[p], hi = s_red[16 + p];
    if (gran == 2) {
      lo = s_red[0];
      hi = s_red[16];
      for (int q = 1; q < 16; ++q) {
        lo = fmin_nan(lo, s_red[q]);
        hi = fmax_nan(hi, s_red[16 + q]);
      }
    }
    lo = __fadd_rn(lo, 0.0f);  // the reference never produces -0 (matrix.hpp:77-83)
    hi = __fadd_rn(hi, 0.0f);
    const bool bad = isnan(lo) || isnan(hi) || isinf(lo) || isinf(hi);
    tmin[p] = lo;
    tmax[p] = hi;
    scale[p] = __fdiv_rn(__fsub_rn(hi, lo), static_cast<float>((1 << bits) - 1));
    const unsigned anybad = __ballot_sync(0x0000ffffu, bad);
    if (p == 0) *nan_flag = anybad ? 1 : 0;
  }
}

// Epilogue constants of affine_term (lowpgemm.hpp:110-114), a = input, b = weight.
__device__ __forceinline__ void make_epilogue_consts(LanceDevState* st, int C) {
  if (threadIdx.x < 16) {
    const int p = threadIdx.x;
    const float sa = st->a_scale[p], oa = st->a_tmin[p];
    const float sb = st->w_scale[p], ob = st->w_tmin[p];
    st->k1[p] = __fmul_rn(sa, sb);
    st->k2[p] = __fmul_rn(sa, ob);
    st->k3[p] = __fmul_rn(sb, oa);
    st->k4[p] = __fmul_rn(__fmul_rn(static_cast<float>(C), oa), ob);
  }
}

// --------------------------------------------------------------------------
// K0: per-position range of v over the whole batch.
template <int VEC>
__global__ void __launch_bounds__(256) input_range_kernel(const float* __restrict__ x,
                                                          float* __restrict__ partials,
                                                          LanceDevState* __restrict__ st,
                                                          InGeom g) {
  __shared__ float s_red[256];
  float lo[16], hi[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const int tl = threadIdx.x / g.G, lg = threadIdx.x - tl * g.G;
  for (long long tb = blockIdx.x; tb < g.num_tile_blocks; tb += gridDim.x) {
    const long long m = tb * g.TPB + tl;
    if (m >= g.M) continue;
    for (int cg = lg; cg < g.C4; cg += g.G) {
      float d[16][4];
      load_tile<VEC>(x, g, m, cg * 4, d);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (VEC != 4 && cg * 4 + j >= g.C) break;
        float dj[16], v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) dj[i] = d[i][j];
        input_transform(dj, v);
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          lo[p] = fmin_nan(lo[p], v[p]);
          hi[p] = fmax_nan(hi[p], v[p]);
        }
      }
    }
  }
  if (block_minmax_and_ticket(lo, hi, partials, &st->ticket_in, s_red)) {
    fit_from_ranges(s_red, g.granularity, st->bits_i, st->a_tmin, st->a_tmax, st->a_scale,
                    &st->nan_in);
    __syncthreads();
    make_epilogue_consts(st, g.C);
  }
}

// K1: recompute v, quantise to u8 codes [16][M][C_pad], row sums [16][M].
template <int VEC>
__global__ void __launch_bounds__(256) input_quant_kernel(const float* __restrict__ x,
                                                          uint8_t* __restrict__ codes,
                                                          int32_t* __restrict__ rowsum,
                                                          const LanceDevState* __restrict__ st,
                                                          InGeom g) {
  __shared__ float s_tmin[16], s_scale[16];
  if (threadIdx.x < 16) {
    s_tmin[threadIdx.x] = st->a_tmin[threadIdx.x];
    s_scale[threadIdx.x] = st->a_scale[threadIdx.x];
  }
  const float top = static_cast<float>((1 << st->bits_i) - 1);
  __syncthreads();
  const int tl = threadIdx.x / g.G, lg = threadIdx.x - tl * g.G;
  const long long m = static_cast<long long>(blockIdx.x) * g.TPB + tl;
  const bool valid = m < g.M;
  uint32_t rs[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) rs[p] = 0u;
  if (valid) {
    for (int cg = lg; cg < g.C4; cg += g.G) {
      float d[16][4];
      load_tile<VEC>(x, g, m, cg * 4, d);
      uint32_t pack[16];
#pragma unroll
      for (int p = 0; p < 16; ++p) pack[p] = 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (VEC != 4 && cg * 4 + j >= g.C) break;
        float dj[16], v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) dj[i] = d[i][j];
        input_transform(dj, v);
#pragma unroll
        for (int p = 0; p < 16; ++p)
          pack[p] |= quantize_code(v[p], s_tmin[p], s_scale[p], top) << (8 * j);
      }
      uint8_t* dst = codes + static_cast<long long>(m) * g.C_pad + cg * 4;
      const long long pstride = g.M * static_cast<long long>(g.C_pad);
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        *reinterpret_cast<uint32_t*>(dst + p * pstride) = pack[p];
        rs[p] = __dp4a(pack[p], 0x01010101u, rs[p]);
      }
    }
  }
  // Sum the G partial row sums of this tile (lanes of one group differ only in
  // their low log2(G) bits).
  for (int off = g.G >> 1; off > 0; off >>= 1) {
#pragma unroll
    for (int p = 0; p < 16; ++p) rs[p] += __shfl_xor_sync(0xffffffffu, rs[p], off);
  }
  if (valid && lg == 0) {
#pragma unroll
    for (int p = 0; p < 16; ++p) rowsum[p * g.M + m] = static_cast<int32_t>(rs[p]);
  }
}

// Static-params mode: caller-supplied input QuantParams[16].
__global__ void static_params_kernel(LanceDevState* st, StaticParams prm, int C) {
  if (threadIdx.x < 16) {
    const int p = threadIdx.x;
    st->a_tmin[p] = prm.tmin[p];
    st->a_tmax[p] = prm.tmax[p];
    st->a_scale[p] = prm.scale[p];
    if (p == 0) st->nan_in = 0;
  }
  __syncwarp();
  make_epilogue_consts(st, C);
}

// --------------------------------------------------------------------------
// K2a: u = G g G^T for every (k, c); u_tmp [16][K][C]; per-position fit.
__global__ void __launch_bounds__(256) filter_transform_kernel(const float* __restrict__ w,
                                                               float* __restrict__ u_tmp,
                                                               float* __restrict__ partials,
                                                               LanceDevState* __restrict__ st,
                                                               FilterGeom g) {
  __shared__ float s_red[256];
  float lo[16], hi[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const long long total = static_cast<long long>(g.K) * g.C;
  const long long slice = total;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = i / g.C;
    const int c = static_cast<int>(i - k * g.C);
    float gg[9], u[16];
#pragma unroll
    for (int rs = 0; rs < 9; ++rs) gg[rs] = __ldg(w + (k * 9 + rs) * g.C + c);
    filter_transform(gg, u);
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      u_tmp[p * slice + i] = u[p];
      lo[p] = fmin_nan(lo[p], u[p]);
      hi[p] = fmax_nan(hi[p], u[p]);
    }
  }
  if (block_minmax_and_ticket(lo, hi, partials, &st->ticket_w, s_red)) {
    fit_from_ranges(s_red, g.granularity, st->bits_w, st->w_tmin, st->w_tmax, st->w_scale,
                    &st->nan_w);
  }
}

// K2b: codes_w [16][K_pad][C_pad] (K-major B operand) and column sums [16][K_pad].
__global__ void __launch_bounds__(128) filter_quant_kernel(const float* __restrict__ u_tmp,
                                                           uint8_t* __restrict__ codes_w,
                                                           int32_t* __restrict__ colsum,
                                                           const LanceDevState* __restrict__ st,
                                                           FilterGeom g) {
  __shared__ int s_sum[4];
  const int k = blockIdx.x;
  const float top = static_cast<float>((1 << st->bits_w) - 1);
  const long long slice = static_cast<long long>(g.K) * g.C;
  for (int p = 0; p < 16; ++p) {
    const float tmin = st->w_tmin[p], scale = st->w_scale[p];
    int sum = 0;
    for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
      const uint32_t code =
          quantize_code(u_tmp[p * slice + static_cast<long long>(k) * g.C + c], tmin, scale, top);
      codes_w[(static_cast<long long>(p) * g.K_pad + k) * g.C_pad + c] = static_cast<uint8_t>(code);
      sum += static_cast<int>(code);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) colsum[p * g.K_pad + k] = s_sum[0] + s_sum[1] + s_sum[2] + s_sum[3];
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// K3/K4: per CTA a 128-row x 32-filter tile of all 16 position GEMMs
// (16 x 32 = 512 TMEM columns of s32), then the fused epilogue.
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + UMMA issuer (one lane)
//   warps 2..5  epilogue: TMEM -> registers -> affine -> A^T m A -> y
template <int BK>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_epilogue_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB,
                         const int32_t* __restrict__ rowsum, const int32_t* __restrict__ colsum,
                         const LanceDevState* __restrict__ st, float* __restrict__ y,
                         int32_t* __restrict__ acc_dump, const float* __restrict__ bias,
                         int relu, GemmGeom g) {
  constexpr uint32_t kABytes = kBM * BK, kBBytes = kBN * BK, kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kLayout = (BK == 128) ? 2u : (BK == 64 ? 4u : 6u);
  constexpr uint32_t kIdesc = umma_idesc_u8(kBM, kBN);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* stage_base = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tmem_full_bar = empty_bar + kStages;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full_bar + 1);
  float* s_cterm = reinterpret_cast<float*>(tmem_holder + 4);  // [16][kBN]
  float* s_k1 = s_cterm + 16 * kBN;
  float* s_k4 = s_k1 + 16;
  float* s_bias = s_k4 + 16;  // [kBN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x % g.num_n_tiles;
  const long long m_tile = blockIdx.x / g.num_n_tiles;
  const long long m0 = m_tile * kBM;
  const int n0 = n_tile * kBN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(tmem_full_bar, 1);
    fence_barrier_init();
  }
  if (warp >= 2) {
    // Epilogue constants: c_p[n] = k3[p] * float(colsum[p][n]) (hoisted
    // third term of affine_term), k1, k4, bias.
    for (int i = threadIdx.x - 64; i < 16 * kBN; i += 128) {
      const int p = i / kBN, n = i % kBN;
      const int kf = n0 + n;
      const float cs = (kf < g.K) ? static_cast<float>(colsum[p * g.num_n_tiles * kBN + kf]) : 0.0f;
      s_cterm[i] = __fmul_rn(st->k3[p], cs);
    }
    if (threadIdx.x - 64 < 16) {
      s_k1[threadIdx.x - 64] = st->k1[threadIdx.x - 64];
      s_k4[threadIdx.x - 64] = st->k4[threadIdx.x - 64];
    }
    if (threadIdx.x - 64 < kBN) {
      const int kf = n0 + threadIdx.x - 64;
      s_bias[threadIdx.x - 64] = (bias != nullptr && kf < g.K) ? bias[kf] : 0.0f;
    }
  }
  __syncthreads();

  const int num_iters = g.num_kchunks * 16;
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      for (int it = 0; it < num_iters; ++it) {
        const int s = it % kStages;
        const uint32_t ph = static_cast<uint32_t>(it / kStages) & 1u;
        const int kc = it >> 4, p = it & 15;
        mbar_wait(&empty_bar[s], ph ^ 1u);
        uint8_t* sa = stage_base + s * kStageBytes;
        mbar_arrive_expect_tx(&full_bar[s], kStageBytes);
        tma_load_3d(sa, &tmA, kc * BK, static_cast<int>(m0), p, &full_bar[s]);
        tma_load_3d(sa + kABytes, &tmB, kc * BK, n0, p, &full_bar[s]);
      }
    }
  } else if (warp == 1) {
    tmem_alloc(tmem_holder, 512);
    tmem_relinquish();
    tc_fence_before();
    named_bar_sync(1, 160);
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    if (lane == 0) {
      for (int it = 0; it < num_iters; ++it) {
        const int s = it % kStages;
        const uint32_t ph = static_cast<uint32_t>(it / kStages) & 1u;
        const int kc = it >> 4, p = it & 15;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint32_t sa = smem_u32(stage_base + s * kStageBytes);
        const uint32_t sb = sa + kABytes;
#pragma unroll
        for (int kk = 0; kk < BK / 32; ++kk) {
          const uint64_t adesc = umma_smem_desc(sa + kk * 32, 8 * BK, kLayout);
          const uint64_t bdesc = umma_smem_desc(sb + kk * 32, 8 * BK, kLayout);
          umma_i8(tmem_base + static_cast<uint32_t>(p * kBN), adesc, bdesc, kIdesc,
                  (kc > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&empty_bar[s]);
      }
      umma_commit(tmem_full_bar);
    }
    __syncwarp();
  } else {
    // ---- epilogue warps ----
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int r = q * 32 + lane;
    const long long m = m0 + r;
    const bool row_ok = m < g.M;
    float rterm[16];
#pragma unroll
    for (int p = 0; p < 16; ++p)
      rterm[p] = row_ok ? __fmul_rn(st->k2[p], static_cast<float>(rowsum[p * g.M + m])) : 0.0f;
    long long img = 0;
    int ti = 0, tj = 0;
    if (row_ok) {
      img = m / g.P;
      const int t = static_cast<int>(m - img * g.P);
      ti = t / g.TW;
      tj = t - ti * g.TW;
    }
    named_bar_sync(1, 160);
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    mbar_wait(tmem_full_bar, 0);
    tc_fence_after();
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const bool vec_ok = (g.K & 3) == 0;
#pragma unroll 1
    for (int j = 0; j < kBN / 4; ++j) {
      uint32_t a[16][4];
#pragma unroll
      for (int p = 0; p < 16; ++p) tmem_ld_x4(lane_addr + p * kBN + j * 4, a[p]);
      tmem_ld_wait();
      const int kf0 = n0 + j * 4;
      if (acc_dump != nullptr && row_ok) {
#pragma unroll
        for (int p = 0; p < 16; ++p)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (kf0 + i < g.K)
              acc_dump[(static_cast<long long>(p) * g.M + m) * g.K + kf0 + i] =
                  static_cast<int32_t>(a[p][i]);
      }
      float out[4][4];  // [pixel a*2+b][filter i]
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float mv[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          // affine_term: ((k1*dot + k2*sum_a) + k3*sum_b) + k4 (lowpgemm.hpp:110-114)
          const float t1 = __fmul_rn(s_k1[p], __int2float_rn(static_cast<int>(a[p][i])));
          mv[p] = __fadd_rn(__fadd_rn(__fadd_rn(t1, rterm[p]), s_cterm[p * kBN + j * 4 + i]),
                            s_k4[p]);
        }
        // S = (A^T m) A (winograd.hpp:80-84 with matrix.hpp:75-84 order)
        float X0[4], X1[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          X0[c] = __fadd_rn(__fadd_rn(mv[c], mv[4 + c]), mv[8 + c]);
          X1[c] = __fsub_rn(__fsub_rn(mv[4 + c], mv[8 + c]), mv[12 + c]);
        }
        float s00 = __fadd_rn(__fadd_rn(X0[0], X0[1]), X0[2]);
        float s01 = __fsub_rn(__fsub_rn(X0[1], X0[2]), X0[3]);
        float s10 = __fadd_rn(__fadd_rn(X1[0], X1[1]), X1[2]);
        float s11 = __fsub_rn(__fsub_rn(X1[1], X1[2]), X1[3]);
        const float bb = s_bias[j * 4 + i];
        if (bias != nullptr) {
          s00 = __fadd_rn(s00, bb);
          s01 = __fadd_rn(s01, bb);
          s10 = __fadd_rn(s10, bb);
          s11 = __fadd_rn(s11, bb);
        }
        if (relu) {
          s00 = fmaxf(s00, 0.0f);
          s01 = fmaxf(s01, 0.0f);
          s10 = fmaxf(s10, 0.0f);
          s11 = fmaxf(s11, 0.0f);
        }
        out[0][i] = __fadd_rn(s00, 0.0f);  // +0.0f: the reference never yields -0
        out[1][i] = __fadd_rn(s01, 0.0f);
        out[2][i] = __fadd_rn(s10, 0.0f);
        out[3][i] = __fadd_rn(s11, 0.0f);
      }
      if (row_ok && kf0 < g.K) {
#pragma unroll
        for (int ab = 0; ab < 4; ++ab) {
          const int oy = 2 * ti + (ab >> 1), ox = 2 * tj + (ab & 1);
          if (oy >= g.OH || ox >= g.OW) continue;  // merge_tiles discard (tensor.hpp:172-175)
          float* dst = y + ((img * g.OH + oy) * static_cast<long long>(g.OW) + ox) * g.K + kf0;
          if (vec_ok) {
            *reinterpret_cast<float4*>(dst) = make_float4(out[ab][0], out[ab][1], out[ab][2], out[ab][3]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (kf0 + i < g.K) dst[i] = out[ab][i];
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(*tmem_holder, 512);
  }
}

// --------------------------------------------------------------------------
// Launchers

cudaError_t launch_input_range(const float* x, float* partials, int grid, LanceDevState* st,
                               const InGeom& g, int vec4, cudaStream_t s) {
  if (vec4)
    input_range_kernel<4><<<grid, 256, 0, s>>>(x, partials, st, g);
  else
    input_range_kernel<1><<<grid, 256, 0, s>>>(x, partials, st, g);
  return cudaGetLastError();
}

cudaError_t launch_input_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                               const LanceDevState* st, const InGeom& g, int vec4,
                               cudaStream_t s) {
  const long long grid = g.num_tile_blocks;
  if (vec4)
    input_quant_kernel<4><<<static_cast<unsigned>(grid), 256, 0, s>>>(x, codes, rowsum, st, g);
  else
    input_quant_kernel<1><<<static_cast<unsigned>(grid), 256, 0, s>>>(x, codes, rowsum, st, g);
  return cudaGetLastError();
}

cudaError_t launch_static_params(LanceDevState* st, const StaticParams& prm, int C,
                                 cudaStream_t s) {
  static_params_kernel<<<1, 32, 0, s>>>(st, prm, C);
  return cudaGetLastError();
}

cudaError_t launch_filter_prepare(const float* w, float* u_tmp, float* partials, int grid,
                                  uint8_t* codes_w, int32_t* colsum, LanceDevState* st,
                                  const FilterGeom& g, cudaStream_t s) {
  filter_transform_kernel<<<grid, 256, 0, s>>>(w, u_tmp, partials, st, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  filter_quant_kernel<<<g.K, 128, 0, s>>>(u_tmp, codes_w, colsum, st, g);
  return cudaGetLastError();
}

template <int BK>
static size_t gemm_smem_bytes() {
  return 1024 + kStages * static_cast<size_t>(kBM + kBN) * BK + (2 * kStages + 1) * 8 + 16 +
         (16 * kBN + 32 + kBN) * 4;
}

template <int BK>
static cudaError_t launch_gemm_bk(const CUtensorMap* tmA, const CUtensorMap* tmB,
                                  const int32_t* rowsum, const int32_t* colsum,
                                  const LanceDevState* st, float* y, int32_t* acc_dump,
                                  const float* bias, int relu, const GemmGeom& g,
                                  cudaStream_t s) {
  const size_t smem = gemm_smem_bytes<BK>();
  static bool configured[64] = {};  // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_epilogue_kernel<BK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev] = true;
  }
  const long long m_tiles = (g.M + kBM - 1) / kBM;
  const long long grid = m_tiles * g.num_n_tiles;
  gemm_epilogue_kernel<BK><<<static_cast<unsigned>(grid), kGemmThreads, smem, s>>>(
      *tmA, *tmB, rowsum, colsum, st, y, acc_dump, bias, relu, g);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, int bk,
                        const int32_t* rowsum, const int32_t* colsum, const LanceDevState* st,
                        float* y, int32_t* acc_dump, const float* bias, int relu,
                        const GemmGeom& g, cudaStream_t s) {
  switch (bk) {
    case 128:
      return launch_gemm_bk<128>(tmA, tmB, rowsum, colsum, st, y, acc_dump, bias, relu, g, s);
    case 64:
      return launch_gemm_bk<64>(tmA, tmB, rowsum, colsum, st, y, acc_dump, bias, relu, g, s);
    default:
      return launch_gemm_bk<32>(tmA, tmB, rowsum, colsum, st, y, acc_dump, bias, relu, g, s);
  }
}

}  // namespace lance_dev
