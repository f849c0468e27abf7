// lance_f4.cu -- the F(4x4,3x3) variant of the lance_gemm path (SURVEY.md
// section 8(f) row 1, BASELINE config 4).  Same algorithm as engines.hpp:492-536
// with alpha = 6 (36 Winograd positions, 6x6 input tiles at stride 4, 4x4
// output tiles) and the Appendix D basis; the checker is the oracle's
// lo_lance_gemm_tiled(tile_m = 4), which evaluates every transform as the
// reference's matmul (matrix.hpp:75-84: i-k-j, fp32, no FMA, from +0).
//
// Kernels:
//   F0  f4_range_kernel   B^T d B per (tile, channel) -> per-position min/max
//                         -> fit_params for 36 positions (+ affine constants)
//   F1  f4_quant_kernel   recompute v, quantise, write the A operand as UMMA
//                         images [row block][36][k chunk] + row sums [36][M]
//   F2  f4_filter_*       G g G^T, fit, B operand images + column sums
//   F3  f4_gemm_kernel    36 tcgen05 kind::i8 GEMMs (128 tiles x 16 filters per
//                         CTA tile) fused with affine_term and A^T m A
//
// Bit-exactness: the transforms below are the matmul folds with the zero basis
// entries skipped (a +-0 term only changes the sign of an all-zero sum, and
// every observable value is canonicalised with +0), products by +-1/2/4/8 are
// exact, products by 5, 1/6, 1/12, 1/24 are one __fmul_rn each; -fmad=false.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lance_common.cuh"

namespace lance_dev {

constexpr int kNP4 = 36;
constexpr float kC6 = 1.0f / 6.0f, kC12 = 1.0f / 12.0f, kC24 = 1.0f / 24.0f;

// y = B^T x for a 6-vector, rows of B^T = [4,0,-5,0,1,0], [0,-4,-4,1,1,0],
// [0,4,-4,-1,1,0], [0,-2,-1,2,1,0], [0,2,-1,-2,1,0], [0,4,0,-5,0,1]; terms
// added in k order (matrix.hpp:80-82).
__device__ __forceinline__ void bt6(const float (&x)[6], float (&y)[6]) {
  const float x1_4 = __fmul_rn(4.0f, x[1]), x1_2 = __fmul_rn(2.0f, x[1]);
  const float x2_4 = __fmul_rn(4.0f, x[2]);
  const float x3_2 = __fmul_rn(2.0f, x[3]);
  y[0] = __fadd_rn(__fsub_rn(__fmul_rn(4.0f, x[0]), __fmul_rn(5.0f, x[2])), x[4]);
  y[1] = __fadd_rn(__fadd_rn(__fsub_rn(-x1_4, x2_4), x[3]), x[4]);
  y[2] = __fadd_rn(__fsub_rn(__fsub_rn(x1_4, x2_4), x[3]), x[4]);
  y[3] = __fadd_rn(__fadd_rn(__fsub_rn(-x1_2, x[2]), x3_2), x[4]);
  y[4] = __fadd_rn(__fsub_rn(__fsub_rn(x1_2, x[2]), x3_2), x[4]);
  y[5] = __fadd_rn(__fsub_rn(x1_4, __fmul_rn(5.0f, x[3])), x[5]);
}

// y = G x for a 3-vector, G = [1/4,0,0], [-1/6,-1/6,-1/6], [-1/6,1/6,-1/6],
// [1/24,1/12,1/6], [1/24,-1/12,1/6], [0,0,1] (fp32 literals).
__device__ __forceinline__ void g6(const float (&x)[3], float (&y)[6]) {
  const float a6 = __fmul_rn(kC6, x[0]), b6 = __fmul_rn(kC6, x[1]), c6 = __fmul_rn(kC6, x[2]);
  const float a24 = __fmul_rn(kC24, x[0]), b12 = __fmul_rn(kC12, x[1]);
  y[0] = __fmul_rn(0.25f, x[0]);
  y[1] = __fsub_rn(__fsub_rn(-a6, b6), c6);
  y[2] = __fsub_rn(__fadd_rn(-a6, b6), c6);
  y[3] = __fadd_rn(__fadd_rn(a24, b12), c6);
  y[4] = __fadd_rn(__fsub_rn(a24, b12), c6);
  y[5] = x[2];
}

// T = A^T m for a 6-vector, A^T = [1,1,1,1,1,0], [0,1,-1,2,-2,0],
// [0,1,1,4,4,0], [0,1,-1,8,-8,1].
__device__ __forceinline__ void at6(const float (&m)[6], float (&t)[4]) {
  const float d12 = __fsub_rn(m[1], m[2]), s12 = __fadd_rn(m[1], m[2]);
  t[0] = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(m[0], m[1]), m[2]), m[3]), m[4]);
  t[1] = __fsub_rn(__fadd_rn(d12, __fmul_rn(2.0f, m[3])), __fmul_rn(2.0f, m[4]));
  t[2] = __fadd_rn(__fadd_rn(s12, __fmul_rn(4.0f, m[3])), __fmul_rn(4.0f, m[4]));
  t[3] = __fadd_rn(__fsub_rn(__fadd_rn(d12, __fmul_rn(8.0f, m[3])), __fmul_rn(8.0f, m[4])), m[5]);
}

// First pass of the input transform, fused with the loads: t = B^T d for the
// 6x6 tile of channel c (zero padded; tile origin (4ti-pad, 4tj-pad)),
// one column of d at a time.
__device__ __forceinline__ void load_bt_tile6(const float* __restrict__ x, const F4Geom& g, int img,
                                              int ti, int tj, int c, float (&t)[36]) {
  const int y0 = 4 * ti - g.pad, x0 = 4 * tj - g.pad;
  const float* base = x + (static_cast<long long>(img) * g.H * g.W) * g.C + c;
#pragma unroll
  for (int b = 0; b < 6; ++b) {
    const int xx = x0 + b;
    const bool cok = xx >= 0 && xx < g.W;
    float col[6], y6[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      const int yy = y0 + a;
      col[a] = (cok && yy >= 0 && yy < g.H)
                   ? __ldg(base + (static_cast<long long>(yy) * g.W + xx) * g.C)
                   : 0.0f;
    }
    bt6(col, y6);
#pragma unroll
    for (int a = 0; a < 6; ++a) t[a * 6 + b] = y6[a];
  }
}

// Second pass for row i: v[i][0..5] = (t B)[i][.].
__device__ __forceinline__ void bt_row6(const float (&t)[36], int i, float (&v)[6]) {
  float x[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) x[k] = t[i * 6 + k];
  bt6(x, v);
}

// --------------------------------------------------------------------------
// Block (min, max) of 36 positions -> partials; the last block folds them and
// returns true with the 72 results in s_fin (lo[36], hi[36]).
__device__ __forceinline__ bool block_minmax36(float (&lo)[kNP4], float (&hi)[kNP4],
                                               float* partials, unsigned int* ticket,
                                               float* s_red /*[8][72]*/, float* s_fin /*[72]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int p = 0; p < kNP4; ++p) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      lo[p] = fmin_nan(lo[p], __shfl_xor_sync(0xffffffffu, lo[p], off));
      hi[p] = fmax_nan(hi[p], __shfl_xor_sync(0xffffffffu, hi[p], off));
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int p = 0; p < kNP4; ++p) {
      s_red[warp * 72 + p] = lo[p];
      s_red[warp * 72 + 36 + p] = hi[p];
    }
  }
  __syncthreads();
  if (threadIdx.x < 72) {
    const int i = threadIdx.x;
    float r = s_red[i];
    for (int w = 1; w < nw; ++w) r = (i < 36) ? fmin_nan(r, s_red[w * 72 + i]) : fmax_nan(r, s_red[w * 72 + i]);
    partials[static_cast<long long>(blockIdx.x) * 72 + i] = r;
  }
  __threadfence();
  __syncthreads();
  __shared__ unsigned int s_last;
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  if (threadIdx.x < 72) {
    const int i = threadIdx.x;
    float r = (i < 36) ? __int_as_float(0x7f800000) : __int_as_float(0xff800000);
    for (int b = 0; b < static_cast<int>(gridDim.x); ++b) {
      const float v = __ldcg(partials + static_cast<long long>(b) * 72 + i);
      r = (i < 36) ? fmin_nan(r, v) : fmax_nan(r, v);
    }
    s_fin[i] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// fit_params (quant.hpp:54-72) for 36 positions from s_fin (PerTensor folds all
// 36, engines.hpp:151-156).  Called by the whole block.
__device__ __forceinline__ void fit36(const float* s_fin, int gran, int bits, float* tmin,
                                      float* tmax, float* scale, float* rcp, int* nan_flag) {
  bool bad = false;
  if (threadIdx.x < kNP4) {
    const int p = threadIdx.x;
    float lo = s_fin[p], hi = s_fin[36 + p];
    if (gran == 2) {
      lo = s_fin[0];
      hi = s_fin[36];
      for (int q = 1; q < kNP4; ++q) {
        lo = fmin_nan(lo, s_fin[q]);
        hi = fmax_nan(hi, s_fin[36 + q]);
      }
    }
    lo = __fadd_rn(lo, 0.0f);  // the reference never produces -0 (matrix.hpp:77-83)
    hi = __fadd_rn(hi, 0.0f);
    bad = isnan(lo) || isnan(hi) || isinf(lo) || isinf(hi);
    const float s = __fdiv_rn(__fsub_rn(hi, lo), static_cast<float>((1 << bits) - 1));
    tmin[p] = lo;
    tmax[p] = hi;
    scale[p] = s;
    if (rcp) rcp[p] = (s == 0.0f) ? 0.0f : __frcp_rn(s);
  }
  const int any = __syncthreads_or(bad ? 1 : 0);
  if (threadIdx.x == 0) *nan_flag = any ? 1 : 0;
}

// --------------------------------------------------------------------------
// F0: ranges.  One warp per Winograd tile, lanes over channels.
__global__ void __launch_bounds__(256, 2) f4_range_kernel(const float* __restrict__ x,
                                                          float* __restrict__ partials,
                                                          LanceDevState* __restrict__ st,
                                                          F4Geom g) {
  __shared__ float s_red[8 * 72];
  __shared__ float s_fin[72];
  float lo[kNP4], hi[kNP4];
#pragma unroll
  for (int p = 0; p < kNP4; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ntiles = static_cast<long long>(g.M);
  for (long long tile = static_cast<long long>(blockIdx.x) * 8 + warp; tile < ntiles;
       tile += static_cast<long long>(gridDim.x) * 8) {
    const int img = static_cast<int>(tile / g.P), t = static_cast<int>(tile - static_cast<long long>(img) * g.P);
    const int ti = t / g.TW, tj = t - ti * g.TW;
    for (int c = lane; c < g.C; c += 32) {
      float tb[36];  // B^T d of this channel
      load_bt_tile6(x, g, img, ti, tj, c, tb);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        float v[6];
        bt_row6(tb, i, v);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          lo[6 * i + k] = fmin_nan(lo[6 * i + k], v[k]);
          hi[6 * i + k] = fmax_nan(hi[6 * i + k], v[k]);
        }
      }
    }
  }
  if (block_minmax36(lo, hi, partials, &st->ticket_in, s_red, s_fin)) {
    fit36(s_fin, g.granularity, st->bits_i, st->a_tmin, st->a_tmax, st->a_scale, st->a_rcp,
          &st->nan_in);
    __syncthreads();
    make_epilogue_consts(st, g.C, kNP4);
  }
}

// F1: codes (A operand UMMA images) + row sums.  One warp per tile; lane l
// handles channels l, l + 32, ...; the warp's row sums are butterfly-reduced
// (no atomics, deterministic).
template <bool STATIC>
__global__ void __launch_bounds__(256, 2) f4_quant_kernel(const float* __restrict__ x,
                                                          uint8_t* __restrict__ codes,
                                                          int32_t* __restrict__ rowsum,
                                                          const LanceDevState* __restrict__ st,
                                                          F4Geom g) {
  __shared__ float s_tmin[kNP4], s_rcp[kNP4], s_scale[kNP4];
  if (threadIdx.x < kNP4) {
    s_tmin[threadIdx.x] = st->a_tmin[threadIdx.x];
    s_rcp[threadIdx.x] = st->a_rcp[threadIdx.x];
    s_scale[threadIdx.x] = st->a_scale[threadIdx.x];
  }
  __syncthreads();
  const float top = static_cast<float>((1 << st->bits_i) - 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long plane = static_cast<long long>(kBM) * g.bk;  // bytes of one image
  for (long long tile = static_cast<long long>(blockIdx.x) * 8 + warp; tile < g.M;
       tile += static_cast<long long>(gridDim.x) * 8) {
    const int img = static_cast<int>(tile / g.P), t = static_cast<int>(tile - static_cast<long long>(img) * g.P);
    const int ti = t / g.TW, tj = t - ti * g.TW;
    int rs[kNP4];
#pragma unroll
    for (int p = 0; p < kNP4; ++p) rs[p] = 0;
    const long long blk = tile / kBM;
    const int r = static_cast<int>(tile - blk * kBM);
    for (int c = lane; c < g.C; c += 32) {
      float tb[36];  // B^T d of this channel
      load_bt_tile6(x, g, img, ti, tj, c, tb);
      const int kc = c / g.bk, cb = c - kc * g.bk;
      uint8_t* dst = codes + ((blk * kNP4) * g.nk + kc) * plane +
                     umma_swizzle(static_cast<uint32_t>(r * g.bk + cb), g.bk);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        float v6[6];
        bt_row6(tb, i, v6);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const int p = 6 * i + k;
          uint32_t code;
          if (STATIC) {
            code = quantize_code(v6[k], s_tmin[p], s_scale[p], top);
          } else {
            const float dd = __fsub_rn(v6[k], s_tmin[p]);
            const float gq = __fmaf_rn(dd, s_rcp[p], kMagic);
            const float rr = __fmaf_rn(dd, s_rcp[p], __fsub_rn(kMagic, gq));
            code = (fabsf(rr) < kTieGuard) ? (__float_as_uint(gq) & 0xFFu)
                                           : exact_code_near_boundary(dd, s_scale[p], gq, rr, top);
          }
          dst[static_cast<long long>(p) * g.nk * plane] = static_cast<uint8_t>(code);
          rs[p] += static_cast<int>(code);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < kNP4; ++p) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) rs[p] += __shfl_xor_sync(0xffffffffu, rs[p], off);
    }
    int mine0 = 0, mine1 = 0;
#pragma unroll
    for (int p = 0; p < kNP4; ++p) {
      if (p == lane) mine0 = rs[p];
      if (p == lane + 32) mine1 = rs[p];
    }
    rowsum[static_cast<long long>(lane) * g.rs_pitch + tile] = mine0;
    if (lane + 32 < kNP4) rowsum[static_cast<long long>(lane + 32) * g.rs_pitch + tile] = mine1;
  }
}

// --------------------------------------------------------------------------
// F2: filters.  u_tmp [36][K][C]; per-position fit; B images + column sums.
__global__ void __launch_bounds__(256, 2) f4_filter_transform_kernel(const float* __restrict__ w,
                                                                     float* __restrict__ u_tmp,
                                                                     float* __restrict__ partials,
                                                                     LanceDevState* __restrict__ st,
                                                                     F4Geom g) {
  __shared__ float s_red[8 * 72];
  __shared__ float s_fin[72];
  float lo[kNP4], hi[kNP4];
#pragma unroll
  for (int p = 0; p < kNP4; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const long long total = static_cast<long long>(g.K) * g.C;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = i / g.C;
    const int c = static_cast<int>(i - k * g.C);
    float gg[9];
#pragma unroll
    for (int rs = 0; rs < 9; ++rs) gg[rs] = __ldg(w + (k * 9 + rs) * g.C + c);
    float h[18];  // (G g)[a][s]
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const float col[3] = {gg[s], gg[3 + s], gg[6 + s]};
      float y[6];
      g6(col, y);
#pragma unroll
      for (int a = 0; a < 6; ++a) h[a * 3 + s] = y[a];
    }
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      const float row[3] = {h[a * 3], h[a * 3 + 1], h[a * 3 + 2]};
      float y[6];
      g6(row, y);
#pragma unroll
      for (int b = 0; b < 6; ++b) {
        const int p = a * 6 + b;
        u_tmp[p * total + i] = y[b];
        lo[p] = fmin_nan(lo[p], y[b]);
        hi[p] = fmax_nan(hi[p], y[b]);
      }
    }
  }
  if (block_minmax36(lo, hi, partials, &st->ticket_w, s_red, s_fin))
    fit36(s_fin, g.granularity, st->bits_w, st->w_tmin, st->w_tmax, st->w_scale, nullptr,
          &st->nan_w);
}

__global__ void __launch_bounds__(128) f4_filter_quant_kernel(const float* __restrict__ u_tmp,
                                                              uint8_t* __restrict__ codes_w,
                                                              int32_t* __restrict__ colsum,
                                                              const LanceDevState* __restrict__ st,
                                                              F4Geom g) {
  __shared__ int s_sum[4];
  const int k = blockIdx.x;
  const float top = static_cast<float>((1 << st->bits_w) - 1);
  const long long total = static_cast<long long>(g.K) * g.C;
  for (int p = 0; p < kNP4; ++p) {
    const float tmin = st->w_tmin[p], scale = st->w_scale[p];
    int sum = 0;
    for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
      const uint32_t code = quantize_code(u_tmp[p * total + static_cast<long long>(k) * g.C + c], tmin, scale, top);
      codes_w[umma_image_offset_np(k, c, p, 16, g.bk, g.nk, kNP4)] = static_cast<uint8_t>(code);
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
// F3: GEMM + epilogue.  Persistent, one CTA per SM, tiles = 128 Winograd tiles
// x 16 filters, n-tile fastest.  Warps 0..15 epilogue (warp w: TMEM lane
// quadrant w % 4, filters 4 * (w / 4) .. +3 of the tile, one Winograd tile
// per thread), warp 16 bulk-copy producer, warp 17 TMEM + UMMA issuer.
// Positions are consumed in j-groups {6a + j : a = 0..5}: T_ij = (A^T m)_ij
// needs exactly that column, and S = T A is a left fold over j, so each
// thread keeps the 16 running S partials of its 4 filters (64 registers).
// A j-group is 6 x 16 TMEM columns; four are in flight.
constexpr int kF4EpiWarps = 16, kF4Threads = 640;
constexpr int kF4BN = 16;
constexpr int kF4GroupCols = 6 * kF4BN;
constexpr int kF4AccBufs = 4;

template <int BK>
struct F4Cfg {
  static constexpr uint32_t kABytes = kBM * BK;
  static constexpr uint32_t kBBytes = kF4BN * BK;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kLayout = (BK == 128) ? 2u : (BK == 64 ? 4u : 6u);
};

template <int BK, bool SMALL, bool DUMP>
__global__ void __launch_bounds__(kF4Threads, 1)
    f4_gemm_kernel(const uint8_t* __restrict__ codes_a, const uint8_t* __restrict__ codes_w,
                   const int32_t* __restrict__ rowsum, const int32_t* __restrict__ colsum,
                   const LanceDevState* __restrict__ st, float* __restrict__ y,
                   int32_t* __restrict__ acc_dump, const float* __restrict__ bias, int relu,
                   F4Geom g) {
  using Cfg = F4Cfg<BK>;
  constexpr uint32_t kIdesc = umma_idesc_u8(kBM, kF4BN);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ float s_k1[kNP4], s_k2[kNP4], s_k4[kNP4];
  __shared__ float s_ct[2][kNP4 * kF4BN];
  __shared__ uint64_t s_bars[2 * 16 + 2 * kF4AccBufs];
  __shared__ uint32_t s_tmem;
  __shared__ int s_fast;

  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stages = g.stages;
  const int nk = g.nk;
  uint64_t* full_bar = s_bars;
  uint64_t* empty_bar = s_bars + 16;
  uint64_t* acc_full = s_bars + 32;
  uint64_t* acc_empty = acc_full + kF4AccBufs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = g.num_n_tiles;
  const int num_tiles = ((g.M + kBM - 1) / kBM) * nt;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < kF4AccBufs; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kF4EpiWarps);
    }
    fence_barrier_init();
  }
  if (threadIdx.x < kNP4) {
    s_k1[threadIdx.x] = st->k1[threadIdx.x];
    s_k2[threadIdx.x] = st->k2[threadIdx.x];
    s_k4[threadIdx.x] = st->k4[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bool ok = SMALL;
    for (int p = 0; p < kNP4; ++p) {
      const float k1 = s_k1[p];
      ok = ok && (k1 == 0.0f || (k1 >= 9.860761315262648e-32f /*2^-103*/ && k1 < 4.0f));
    }
    s_fast = ok ? 1 : 0;
    if (ok)
      for (int p = 0; p < kNP4; ++p) s_k1[p] = __fmul_rn(s_k1[p], 8.507059173023462e37f /*2^126*/);
  }
  __syncthreads();

  if (warp >= kF4EpiWarps) {
    setmaxnreg_dec<32>();
    if (warp == kF4EpiWarps && lane == 0) {
      // ---------------- bulk-copy producer ----------------
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mt = t / nt, ntile = t - (t / nt) * nt;
        const uint8_t* a_tile = codes_a + static_cast<long long>(mt) * kNP4 * nk * Cfg::kABytes;
        const uint8_t* b_tile = codes_w + static_cast<long long>(ntile) * kNP4 * nk * Cfg::kBBytes;
        for (int j = 0; j < 6; ++j)
          for (int a = 0; a < 6; ++a) {
            const int u0 = (6 * a + j) * nk;
            for (int kc = 0; kc < nk; ++kc) {
              mbar_wait(&empty_bar[s], ph ^ 1u);
              uint8_t* sa = smem + static_cast<size_t>(s) * Cfg::kStageBytes;
              mbar_arrive_expect_tx(&full_bar[s], Cfg::kStageBytes);
              bulk_load(sa, a_tile + static_cast<long long>(u0 + kc) * Cfg::kABytes, Cfg::kABytes, &full_bar[s]);
              bulk_load(sa + Cfg::kABytes, b_tile + static_cast<long long>(u0 + kc) * Cfg::kBBytes,
                        Cfg::kBBytes, &full_bar[s]);
              if (++s == stages) {
                s = 0;
                ph ^= 1u;
              }
            }
          }
      }
    } else if (warp == kF4EpiWarps + 1) {
      // ---------------- TMEM + UMMA issuer ----------------
      tmem_alloc(&s_tmem, 512);
      tmem_relinquish();
      tc_fence_before();
      named_bar_sync(1, 32 + 32 * kF4EpiWarps);
      tc_fence_after();
      const uint32_t tmem_base = s_tmem;
      if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        uint32_t grp = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
          for (int j = 0; j < 6; ++j, ++grp) {
            const uint32_t buf = grp % kF4AccBufs;
            mbar_wait(&acc_empty[buf], (grp / kF4AccBufs) & 1u);
            tc_fence_after();
            const uint32_t d_base = tmem_base + buf * kF4GroupCols;
            for (int a = 0; a < 6; ++a) {
              for (int kc = 0; kc < nk; ++kc) {
                mbar_wait(&full_bar[s], ph);
                tc_fence_after();
                const uint32_t sa = smem_u32(smem + static_cast<size_t>(s) * Cfg::kStageBytes);
                const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
                for (int kk = 0; kk < BK / 32; ++kk) {
                  const uint64_t adesc = umma_smem_desc(sa + kk * 32, 8 * BK, Cfg::kLayout);
                  const uint64_t bdesc = umma_smem_desc(sb + kk * 32, 8 * BK, Cfg::kLayout);
                  umma_i8(d_base + static_cast<uint32_t>(a * kF4BN), adesc, bdesc, kIdesc,
                          (kc > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&empty_bar[s]);
                if (++s == stages) {
                  s = 0;
                  ph ^= 1u;
                }
              }
            }
            umma_commit(&acc_full[buf]);
          }
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue ----------------
    setmaxnreg_inc<112>();
    const int q = warp & 3;
    const int f0 = (warp >> 2) * 4;
    const int row = q * 32 + lane;
    named_bar_sync(1, 32 + 32 * kF4EpiWarps);
    tc_fence_after();
    const uint32_t lane_base = s_tmem + (static_cast<uint32_t>(q * 32) << 16);
    if (lane == 0)
      for (int b = 0; b < kF4AccBufs; ++b) mbar_arrive(&acc_empty[b]);
    const bool fast = s_fast != 0;
    const bool k4ok = (g.K & 3) == 0;
    uint32_t grp = 0, lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      const int m0 = (t / nt) * kBM, n0 = (t - (t / nt) * nt) * kF4BN;
      const int m = m0 + row;
      const bool row_ok = m < g.M;
      const int kf0 = n0 + f0;
      // k3[p] * float(colsum[p][k]) of the tile's 16 filters (double-buffered
      // by tile parity; one barrier per tile orders it against the readers).
      float* ct = s_ct[lt & 1u];
      for (int i = threadIdx.x; i < kNP4 * kF4BN; i += 32 * kF4EpiWarps) {
        const int p = i >> 4, kk = n0 + (i & 15);
        ct[i] = (kk < g.K) ? __fmul_rn(st->k3[p], static_cast<float>(colsum[p * g.K_pad + kk])) : 0.0f;
      }
      named_bar_sync(2, 32 * kF4EpiWarps);
      float S[16][4];  // S[4i + b][filter]
#pragma unroll
      for (int j = 0; j < 6; ++j, ++grp) {
        float rterm[6];
#pragma unroll
        for (int a = 0; a < 6; ++a) {
          const int p = 6 * a + j;
          const int rs = row_ok ? __ldg(rowsum + static_cast<long long>(p) * g.rs_pitch + m) : 0;
          rterm[a] = __fmul_rn(s_k2[p], static_cast<float>(rs));
        }
        const uint32_t buf = grp % kF4AccBufs;
        mbar_wait(&acc_full[buf], (grp / kF4AccBufs) & 1u);
        tc_fence_after();
        uint32_t ac[6][4];
#pragma unroll
        for (int a = 0; a < 6; ++a) tmem_ld_x4(lane_base + buf * kF4GroupCols + a * kF4BN + f0, ac[a]);
        tmem_ld_wait();
#pragma unroll
        for (int a = 0; a < 6; ++a) reg_fence(ac[a]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        if (DUMP && row_ok) {
#pragma unroll
          for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int f = 0; f < 4; ++f)
              if (kf0 + f < g.K)
                acc_dump[(static_cast<long long>(6 * a + j) * g.M + m) * g.K + kf0 + f] =
                    static_cast<int32_t>(ac[a][f]);
        }
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          float mm[6];
#pragma unroll
          for (int a = 0; a < 6; ++a) {
            const int p = 6 * a + j;
            float v;  // RN(RN(k1 * dot) + RN(k2 * sum_a))
            if (fast)
              v = __fmaf_rn(__fmul_rn(s_k1[p], __uint_as_float(ac[a][f])), 8388608.0f /*2^23*/, rterm[a]);
            else
              v = __fadd_rn(__fmul_rn(s_k1[p], __int2float_rn(static_cast<int>(ac[a][f]))), rterm[a]);
            // ((k1*dot + k2*sum_a) + k3*sum_b) + k4 (lowpgemm.hpp:110-114)
            mm[a] = __fadd_rn(__fadd_rn(v, ct[p * kF4BN + f0 + f]), s_k4[p]);
          }
          float T[4];
          at6(mm, T);
          // S_ib = sum_j T_ij * A^T[b][j], left fold over j (matrix.hpp:80-82).
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float tv = T[i];
            if (j == 0) {
              S[4 * i + 0][f] = tv;
            } else if (j == 1) {
              S[4 * i + 0][f] = __fadd_rn(S[4 * i + 0][f], tv);
              S[4 * i + 1][f] = tv;
              S[4 * i + 2][f] = tv;
              S[4 * i + 3][f] = tv;
            } else if (j == 2) {
              S[4 * i + 0][f] = __fadd_rn(S[4 * i + 0][f], tv);
              S[4 * i + 1][f] = __fsub_rn(S[4 * i + 1][f], tv);
              S[4 * i + 2][f] = __fadd_rn(S[4 * i + 2][f], tv);
              S[4 * i + 3][f] = __fsub_rn(S[4 * i + 3][f], tv);
            } else if (j == 3) {
              S[4 * i + 0][f] = __fadd_rn(S[4 * i + 0][f], tv);
              S[4 * i + 1][f] = __fadd_rn(S[4 * i + 1][f], __fmul_rn(2.0f, tv));
              S[4 * i + 2][f] = __fadd_rn(S[4 * i + 2][f], __fmul_rn(4.0f, tv));
              S[4 * i + 3][f] = __fadd_rn(S[4 * i + 3][f], __fmul_rn(8.0f, tv));
            } else if (j == 4) {
              S[4 * i + 0][f] = __fadd_rn(S[4 * i + 0][f], tv);
              S[4 * i + 1][f] = __fsub_rn(S[4 * i + 1][f], __fmul_rn(2.0f, tv));
              S[4 * i + 2][f] = __fadd_rn(S[4 * i + 2][f], __fmul_rn(4.0f, tv));
              S[4 * i + 3][f] = __fsub_rn(S[4 * i + 3][f], __fmul_rn(8.0f, tv));
            } else {
              S[4 * i + 3][f] = __fadd_rn(S[4 * i + 3][f], tv);
            }
          }
        }
      }
      // merge_tiles (tensor.hpp:157-182): output (4ti + i, 4tj + b), overhang
      // discarded; optional bias / ReLU; +0 canonicalisation.
      if (row_ok && kf0 < g.K) {
        const int img = m / g.P, tt = m - (m / g.P) * g.P;
        const int ti = tt / g.TW, tj = tt - ti * g.TW;
        float bv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (bias != nullptr)
#pragma unroll
          for (int f = 0; f < 4; ++f) bv[f] = (kf0 + f < g.K) ? __ldg(bias + kf0 + f) : 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int oh = 4 * ti + i;
          if (oh >= g.OH) break;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int ow = 4 * tj + b;
            if (ow >= g.OW) break;
            float o[4];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              float v = S[4 * i + b][f];
              if (bias != nullptr) v = __fadd_rn(v, bv[f]);
              if (relu) v = fmaxf(v, 0.0f);
              o[f] = __fadd_rn(v, 0.0f);
            }
            float* d = y + (static_cast<long long>(img * g.OH + oh) * g.OW + ow) * g.K + kf0;
            if (k4ok) {
              *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
              for (int f = 0; f < 4; ++f)
                if (kf0 + f < g.K) d[f] = o[f];
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == kF4EpiWarps + 1) {
    tc_fence_after();
    tmem_dealloc(s_tmem, 512);
  }
}

// --------------------------------------------------------------------------
int f4_range_grid(const F4Geom& g, int sm_count) {
  const long long blocks = (static_cast<long long>(g.M) + 7) / 8;
  const long long cap = 2LL * sm_count;
  return static_cast<int>(blocks < cap ? blocks : cap);
}

cudaError_t launch_f4_range(const float* x, float* partials, int grid, LanceDevState* st,
                            const F4Geom& g, cudaStream_t s) {
  f4_range_kernel<<<grid, 256, 0, s>>>(x, partials, st, g);
  return cudaGetLastError();
}

cudaError_t launch_f4_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                            const LanceDevState* st, const F4Geom& g, int static_mode,
                            int sm_count, cudaStream_t s) {
  const long long blocks = (static_cast<long long>(g.M) + 7) / 8;
  const int grid = static_cast<int>(blocks < 4LL * sm_count ? blocks : 4LL * sm_count);
  if (static_mode)
    f4_quant_kernel<true><<<grid, 256, 0, s>>>(x, codes, rowsum, st, g);
  else
    f4_quant_kernel<false><<<grid, 256, 0, s>>>(x, codes, rowsum, st, g);
  return cudaGetLastError();
}

cudaError_t launch_f4_filter_prepare(const float* w, float* u_tmp, float* partials, int grid,
                                     uint8_t* codes_w, int32_t* colsum, LanceDevState* st,
                                     const F4Geom& g, cudaStream_t s) {
  f4_filter_transform_kernel<<<grid, 256, 0, s>>>(w, u_tmp, partials, st, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  f4_filter_quant_kernel<<<g.K, 128, 0, s>>>(u_tmp, codes_w, colsum, st, g);
  return cudaGetLastError();
}

template <int BK, bool SMALL, bool DUMP>
static cudaError_t launch_f4_gemm_t(const uint8_t* codes_a, const uint8_t* codes_w,
                                    const int32_t* rowsum, const int32_t* colsum,
                                    const LanceDevState* st, float* y, int32_t* acc_dump,
                                    const float* bias, int relu, const F4Geom& g0, cudaStream_t s) {
  F4Geom g = g0;
  int stages = 16;
  const size_t kLimit = 200 * 1024;
  while (stages > 2 && 1024 + static_cast<size_t>(stages) * F4Cfg<BK>::kStageBytes > kLimit) --stages;
  g.stages = stages;
  const size_t smem = 1024 + static_cast<size_t>(stages) * F4Cfg<BK>::kStageBytes;
  static bool configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(f4_gemm_kernel<BK, SMALL, DUMP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kLimit));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev] = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = ((static_cast<long long>(g.M) + kBM - 1) / kBM) * g.num_n_tiles;
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  f4_gemm_kernel<BK, SMALL, DUMP><<<grid, kF4Threads, smem, s>>>(codes_a, codes_w, rowsum, colsum,
                                                                  st, y, acc_dump, bias, relu, g);
  return cudaGetLastError();
}

template <int BK>
static cudaError_t launch_f4_gemm_bk(const uint8_t* codes_a, const uint8_t* codes_w,
                                     const int32_t* rowsum, const int32_t* colsum, int small_acc,
                                     const LanceDevState* st, float* y, int32_t* acc_dump,
                                     const float* bias, int relu, const F4Geom& g, cudaStream_t s) {
  const bool dump = acc_dump != nullptr;
  if (small_acc)
    return dump ? launch_f4_gemm_t<BK, true, true>(codes_a, codes_w, rowsum, colsum, st, y, acc_dump, bias, relu, g, s)
                : launch_f4_gemm_t<BK, true, false>(codes_a, codes_w, rowsum, colsum, st, y, acc_dump, bias, relu, g, s);
  return dump ? launch_f4_gemm_t<BK, false, true>(codes_a, codes_w, rowsum, colsum, st, y, acc_dump, bias, relu, g, s)
              : launch_f4_gemm_t<BK, false, false>(codes_a, codes_w, rowsum, colsum, st, y, acc_dump, bias, relu, g, s);
}

cudaError_t launch_f4_gemm(const uint8_t* codes_a, const uint8_t* codes_w, const int32_t* rowsum,
                           const int32_t* colsum, int small_acc, const LanceDevState* st, float* y,
                           int32_t* acc_dump, const float* bias, int relu, const F4Geom& g,
                           cudaStream_t s) {
  switch (g.bk) {
    case 128: return launch_f4_gemm_bk<128>(codes_a, codes_w, rowsum, colsum, small_acc, st, y, acc_dump, bias, relu, g, s);
    case 64: return launch_f4_gemm_bk<64>(codes_a, codes_w, rowsum, colsum, small_acc, st, y, acc_dump, bias, relu, g, s);
    case 32: return launch_f4_gemm_bk<32>(codes_a, codes_w, rowsum, colsum, small_acc, st, y, acc_dump, bias, relu, g, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lance_dev
