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
#include <cstdlib>

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

// bt6 on two independent vectors at once (packed f32x2): products by 2 and 4
// by exact doubling, 5x as RN(4x + x) == RN(5x); negated leading terms are
// folded as RN(-a - b) = -RN(a + b), RN(-s + c) = RN(c - s) (same IEEE results).
__device__ __forceinline__ void bt6_2(const float2 (&x)[6], float2 (&y)[6]) {
  const float2 x0_2 = add2(x[0], x[0]), x0_4 = add2(x0_2, x0_2);
  const float2 x1_2 = add2(x[1], x[1]), x1_4 = add2(x1_2, x1_2);
  const float2 x2_2 = add2(x[2], x[2]), x2_4 = add2(x2_2, x2_2), x2_5 = add2(x2_4, x[2]);
  const float2 x3_2 = add2(x[3], x[3]), x3_4 = add2(x3_2, x3_2), x3_5 = add2(x3_4, x[3]);
  y[0] = add2(sub2(x0_4, x2_5), x[4]);
  y[1] = add2(sub2(x[3], add2(x1_4, x2_4)), x[4]);
  y[2] = add2(sub2(sub2(x1_4, x2_4), x[3]), x[4]);
  y[3] = add2(sub2(x3_2, add2(x1_2, x[2])), x[4]);
  y[4] = add2(sub2(sub2(x1_2, x[2]), x3_2), x[4]);
  y[5] = add2(sub2(x1_4, x3_5), x[5]);
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

// at6 on two filters at once (packed f32x2 adds; x2 / x4 / x8 by exact doubling).
__device__ __forceinline__ void at6_2(const float2 (&m)[6], float2 (&t)[4]) {
  const float2 d12 = sub2(m[1], m[2]), s12 = add2(m[1], m[2]);
  const float2 m3_2 = add2(m[3], m[3]), m4_2 = add2(m[4], m[4]);
  const float2 m3_4 = add2(m3_2, m3_2), m4_4 = add2(m4_2, m4_2);
  const float2 m3_8 = add2(m3_4, m3_4), m4_8 = add2(m4_4, m4_4);
  t[0] = add2(add2(add2(add2(m[0], m[1]), m[2]), m[3]), m[4]);
  t[1] = sub2(add2(d12, m3_2), m4_2);
  t[2] = add2(add2(s12, m3_4), m4_4);
  t[3] = add2(sub2(add2(d12, m3_8), m4_8), m[5]);
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
  {
    // Column i = threadIdx.x % 72 over the blocks b = threadIdx.x / 72 + k * (nthreads / 72),
    // eight independent loads in flight, then a shared-memory fold of the rows.
    const int rows = static_cast<int>(blockDim.x) / 72;
    const int i = threadIdx.x % 72, row0 = threadIdx.x / 72;
    float r = (i < 36) ? __int_as_float(0x7f800000) : __int_as_float(0xff800000);
    const int nb = static_cast<int>(gridDim.x);
    if (row0 < rows) {
      for (int b0 = row0; b0 < nb; b0 += 8 * rows) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = b0 + u * rows;
          v[u] = (b < nb) ? __ldcg(partials + static_cast<long long>(b) * 72 + i) : r;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) r = (i < 36) ? fmin_nan(r, v[u]) : fmax_nan(r, v[u]);
      }
    }
    __syncthreads();
    if (row0 < rows) s_red[row0 * 72 + i] = r;
    __syncthreads();
    if (threadIdx.x < 72) {
      float q = s_red[threadIdx.x];
      for (int w = 1; w < rows; ++w)
        q = (threadIdx.x < 36) ? fmin_nan(q, s_red[w * 72 + threadIdx.x]) : fmax_nan(q, s_red[w * 72 + threadIdx.x]);
      s_fin[threadIdx.x] = q;
    }
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
// F0 / F1 work decomposition: a warp walks a strip of tiles along one tile
// row (img, ti, tj0 .. tj1) for 32 channels (one per lane).  Adjacent tiles
// share two input columns, so each step loads the 4 new columns and carries
// the first-pass (B^T d) columns 4, 5 of the previous tile as columns 0, 1.
// The first pass is scalar per column; its outputs land directly in row-pair
// registers tp[r][k] = (t[r][k], t[r+3][k]) for the packed second pass.
struct F4Strip {
  int img, ti, tj0, tj1, c;
  bool cok;
  uint32_t rowmask;  // bit a: input row 4ti - pad + a inside the image
};

__device__ __forceinline__ F4Strip f4_strip(const F4Geom& g, long long item, int lane) {
  F4Strip st;
  const int ncg = (g.C + 31) >> 5;
  const int cg = static_cast<int>(item % ncg);
  long long rest = item / ncg;
  const int seg = static_cast<int>(rest % g.nseg);
  rest /= g.nseg;
  st.ti = static_cast<int>(rest % g.TH);
  st.img = static_cast<int>(rest / g.TH);
  st.tj0 = seg * g.seg_len;
  st.tj1 = min(st.tj0 + g.seg_len, g.TW);
  st.c = cg * 32 + lane;
  st.cok = st.c < g.C;
  const int y0 = 4 * st.ti - g.pad;
  st.rowmask = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
    if (y0 + a >= 0 && y0 + a < g.H) st.rowmask |= 1u << a;
  return st;
}

// First pass for input column xx of the strip's rows: t[.][b] into tp.
__device__ __forceinline__ void f4_col(const float* __restrict__ rowbase, long long rowstride,
                                       const F4Geom& g, const F4Strip& st, int xx, int b,
                                       float2 (&tp)[3][6]) {
  const bool colok = st.cok && xx >= 0 && xx < g.W;
  const float* p = rowbase + static_cast<long long>(xx) * g.C;
  float col[6], y6[6];
#pragma unroll
  for (int a = 0; a < 6; ++a)
    col[a] = (colok && ((st.rowmask >> a) & 1u)) ? __ldg(p + a * rowstride) : 0.0f;
  bt6(col, y6);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    tp[r][b].x = y6[r];
    tp[r][b].y = y6[r + 3];
  }
}

// Optional input staging (template D > 0): the 4 new input columns x 6 rows
// of the next D tiles are copied per lane with 4-byte cp.async (zero-fill
// outside the image) into a shared-memory ring; the first pass then reads them
// from the slot.  A lane only reads what it copied itself.
__device__ __forceinline__ void f4_cp_async4(float* sdst, const float* gsrc, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(gsrc), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void f4_cp_async4_sz(float* sdst, const float* gsrc, uint32_t src_bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void f4_cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void f4_cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int D>
__device__ __forceinline__ void f4_ring_issue(float* ring, int lane, const float* __restrict__ x,
                                              const float* __restrict__ rowbase, long long rowstride,
                                              const F4Geom& g, const F4Strip& sp, int t) {
  float* slot = ring + (t % D) * 24 * 32;
  if (t < sp.tj1) {
    // Zero-fill copies read nothing at size 0: the address is passed as is
    // and only the size is predicated (no pointer selects on the hot path).
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int xx = 4 * t - g.pad + 2 + cc;
      const uint32_t colsz = (sp.cok && static_cast<unsigned>(xx) < static_cast<unsigned>(g.W)) ? 4u : 0u;
      const float* p = rowbase + static_cast<long long>(xx) * g.C;
#pragma unroll
      for (int a = 0; a < 6; ++a)
        f4_cp_async4_sz(slot + (cc * 6 + a) * 32 + lane, p + a * rowstride,
                        ((sp.rowmask >> a) & 1u) ? colsz : 0u);
    }
  }
  f4_cp_commit();
}

// First pass for column b (2..5) of tile t from its staged slot.
template <int D>
__device__ __forceinline__ void f4_col_staged(const float* ring, int lane, int t, int b, float2 (&tp)[3][6]) {
  const float* slot = ring + (t % D) * 24 * 32 + (b - 2) * 6 * 32 + lane;
  float col[6], y6[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) col[a] = slot[a * 32];
  bt6(col, y6);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    tp[r][b].x = y6[r];
    tp[r][b].y = y6[r + 3];
  }
}

// F0: ranges.
template <int D>
__global__ void __launch_bounds__(256, 2) f4_range_kernel(const float* __restrict__ x,
                                                          float* __restrict__ partials,
                                                          LanceDevState* __restrict__ st,
                                                          F4Geom g) {
  pdl_entry();
  grid_zero_i32(g.rs_zero, g.rs_zero_words);  // F1's atomic row sums
  __shared__ float s_red[8 * 72];
  __shared__ float s_fin[72];
  float lo[kNP4], hi[kNP4];
#pragma unroll
  for (int p = 0; p < kNP4; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long rowstride = static_cast<long long>(g.W) * g.C;
  extern __shared__ float f4ring_all[];  // D > 0: [8 warps][D][24][32]
  float* f4ring = f4ring_all + static_cast<size_t>(warp) * (D > 0 ? D : 1) * 24 * 32;
  for (long long item = static_cast<long long>(blockIdx.x) * 8 + warp; item < g.num_items;
       item += static_cast<long long>(gridDim.x) * 8) {
    const F4Strip sp = f4_strip(g, item, lane);
    const float* rowbase = x + (static_cast<long long>(sp.img) * g.H + (4 * sp.ti - g.pad)) * rowstride + sp.c;
    float2 tp[3][6];
    f4_col(rowbase, rowstride, g, sp, 4 * sp.tj0 - g.pad, 0, tp);
    f4_col(rowbase, rowstride, g, sp, 4 * sp.tj0 - g.pad + 1, 1, tp);
    if (D > 0) {
#pragma unroll
      for (int q = 0; q < (D > 0 ? D : 1); ++q)
        f4_ring_issue<(D > 0 ? D : 1)>(f4ring, lane, x, rowbase, rowstride, g, sp, sp.tj0 + q);
    }
    for (int tj = sp.tj0; tj < sp.tj1; ++tj) {
      if (D > 0) {
        f4_cp_wait<(D > 0 ? D - 1 : 0)>();
#pragma unroll
        for (int b = 2; b < 6; ++b) f4_col_staged<(D > 0 ? D : 1)>(f4ring, lane, tj, b, tp);
        f4_ring_issue<(D > 0 ? D : 1)>(f4ring, lane, x, rowbase, rowstride, g, sp, tj + D);
      } else {
#pragma unroll
        for (int b = 2; b < 6; ++b) f4_col(rowbase, rowstride, g, sp, 4 * tj - g.pad + b, b, tp);
      }
      if (sp.cok) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          float2 v2[6];
          bt6_2(tp[r], v2);
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            lo[6 * r + k] = fmin_nan(lo[6 * r + k], v2[k].x);
            hi[6 * r + k] = fmax_nan(hi[6 * r + k], v2[k].x);
            lo[6 * r + 18 + k] = fmin_nan(lo[6 * r + 18 + k], v2[k].y);
            hi[6 * r + 18 + k] = fmax_nan(hi[6 * r + 18 + k], v2[k].y);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        tp[r][0] = tp[r][4];
        tp[r][1] = tp[r][5];
      }
    }
    if (D > 0) f4_cp_wait<0>();
  }
  if (block_minmax36(lo, hi, partials, &st->ticket_in, s_red, s_fin)) {
    fit36(s_fin, g.granularity, st->bits_i, st->a_tmin, st->a_tmax, st->a_scale, st->a_rcp,
          &st->nan_in);
    __syncthreads();
    make_epilogue_consts(st, g.C, kNP4);
  }
}

// F1: codes (A operand UMMA images, j-major planes) + row sums.  Positions
// (p, p + 18) are quantised as one packed pair; the warp's per-tile row sums
// are one REDUX per position, added into rowsum (zeroed by the launcher).
// BK / NK > 0: compile-time image geometry, so the 36 per-position store
// offsets are immediates; NK = 0: runtime geometry (any shape).  The tie
// check is one branch per row pair (12 codes), the rare fix-up recomputes
// that row's flagged codes exactly before they are stored.
// F1 CTA shape.  4-warp CTAs at 5 per SM (registers capped at 96, as the
// F(2x2) K1 runs) measured slower here: the F(4x4) tile state spills.
#ifndef LANCE_F4Q_THREADS
#define LANCE_F4Q_THREADS 256
#endif
#ifndef LANCE_F4Q_MINB
#define LANCE_F4Q_MINB 2
#endif
template <bool STATIC, int BK, int NK, int D = 0>
__global__ void __launch_bounds__(LANCE_F4Q_THREADS, LANCE_F4Q_MINB) f4_quant_kernel(const float* __restrict__ x,
                                                          uint8_t* __restrict__ codes,
                                                          int32_t* __restrict__ rowsum,
                                                          const LanceDevState* __restrict__ st,
                                                          F4Geom g) {
  pdl_entry();
  __shared__ float2 s_tmin2[18], s_rcp2[18], s_scale2[18];
  if (threadIdx.x < 18) {
    const int p = threadIdx.x;
    s_tmin2[p] = make_float2(st->a_tmin[p], st->a_tmin[p + 18]);
    s_rcp2[p] = make_float2(st->a_rcp[p], st->a_rcp[p + 18]);
    s_scale2[p] = make_float2(st->a_scale[p], st->a_scale[p + 18]);
  }
  __syncthreads();
  const float top = static_cast<float>((1 << st->bits_i) - 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long rowstride = static_cast<long long>(g.W) * g.C;
  const int bk = NK > 0 ? BK : g.bk;
  const int img_bytes = kBM * bk;                              // one UMMA image
  const int pstride = (NK > 0 ? NK : g.nk) * img_bytes;        // one position plane
  extern __shared__ float f4qring_all[];  // D > 0: [warps][D][24][32]
  float* f4ring = f4qring_all + static_cast<size_t>(warp) * (D > 0 ? D : 1) * 24 * 32;
  constexpr int kWarps = LANCE_F4Q_THREADS / 32;
  for (long long item = static_cast<long long>(blockIdx.x) * kWarps + warp; item < g.num_items;
       item += static_cast<long long>(gridDim.x) * kWarps) {
    const F4Strip sp = f4_strip(g, item, lane);
    const float* rowbase = x + (static_cast<long long>(sp.img) * g.H + (4 * sp.ti - g.pad)) * rowstride + sp.c;
    const int kc = sp.c / bk, cb = sp.c - kc * bk;
    float2 tp[3][6];
    f4_col(rowbase, rowstride, g, sp, 4 * sp.tj0 - g.pad, 0, tp);
    f4_col(rowbase, rowstride, g, sp, 4 * sp.tj0 - g.pad + 1, 1, tp);
    if (D > 0) {
#pragma unroll
      for (int q = 0; q < (D > 0 ? D : 1); ++q)
        f4_ring_issue<(D > 0 ? D : 1)>(f4ring, lane, x, rowbase, rowstride, g, sp, sp.tj0 + q);
    }
    for (int tj = sp.tj0; tj < sp.tj1; ++tj) {
      if (D > 0) {
        f4_cp_wait<(D > 0 ? D - 1 : 0)>();
#pragma unroll
        for (int b = 2; b < 6; ++b) f4_col_staged<(D > 0 ? D : 1)>(f4ring, lane, tj, b, tp);
        f4_ring_issue<(D > 0 ? D : 1)>(f4ring, lane, x, rowbase, rowstride, g, sp, tj + D);
      } else {
#pragma unroll
        for (int b = 2; b < 6; ++b) f4_col(rowbase, rowstride, g, sp, 4 * tj - g.pad + b, b, tp);
      }
      const long long tile = (static_cast<long long>(sp.img) * g.TH + sp.ti) * g.TW + tj;
      const long long blk = tile / kBM;
      const int r = static_cast<int>(tile - blk * kBM);
      uint8_t* dst = codes + (blk * kNP4) * static_cast<long long>(pstride) + kc * img_bytes +
                     umma_swizzle(static_cast<uint32_t>(r * bk + cb), bk);
      uint32_t mine0 = 0, mine1 = 0;  // row sums of positions lane, lane + 32
#pragma unroll
      for (int rr = 0; rr < 3; ++rr) {
        float2 v2[6];
        bt6_2(tp[rr], v2);
        uint32_t c0[6], c1[6];  // positions 6rr + k (.x) and 6rr + 18 + k (.y)
        if (STATIC) {
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const int p = 6 * rr + k;
            c0[k] = quantize_code(v2[k].x, s_tmin2[p].x, s_scale2[p].x, top);
            c1[k] = quantize_code(v2[k].y, s_tmin2[p].y, s_scale2[p].y, top);
          }
        } else {
          float rmax = 0.0f;
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const int p = 6 * rr + k;
            const float2 dd = sub2(v2[k], s_tmin2[p]);
            const float2 gq = fma2(dd, s_rcp2[p], bcast2(kMagic));
            const float2 rr2 = fma2(dd, s_rcp2[p], sub2(bcast2(kMagic), gq));
            c0[k] = __float_as_uint(gq.x) & 0xFFu;
            c1[k] = __float_as_uint(gq.y) & 0xFFu;
            rmax = fmax3_nan(rmax, fabsf(rr2.x), fabsf(rr2.y));
          }
          if (__builtin_expect(!(rmax < kTieGuard), 0)) {
            // Rare (~1e-4 per value): re-derive this row's flagged codes exactly.
#pragma unroll
            for (int k = 0; k < 6; ++k) {
              const int p = 6 * rr + k;
              const float2 dd = sub2(v2[k], s_tmin2[p]);
              const float2 gq = fma2(dd, s_rcp2[p], bcast2(kMagic));
              const float2 rr2 = fma2(dd, s_rcp2[p], sub2(bcast2(kMagic), gq));
              if (!(fabsf(rr2.x) < kTieGuard)) c0[k] = exact_code_near_boundary(dd.x, s_scale2[p].x, gq.x, rr2.x, top);
              if (!(fabsf(rr2.y) < kTieGuard)) c1[k] = exact_code_near_boundary(dd.y, s_scale2[p].y, gq.y, rr2.y, top);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const int p = 6 * rr + k;
          if (!sp.cok) c0[k] = c1[k] = 0u;
          else {
            dst[f4_plane(p) * pstride] = static_cast<uint8_t>(c0[k]);
            dst[f4_plane(p + 18) * pstride] = static_cast<uint8_t>(c1[k]);
          }
          const uint32_t s0 = __reduce_add_sync(0xffffffffu, c0[k]);
          const uint32_t s1 = __reduce_add_sync(0xffffffffu, c1[k]);
          if (lane == (p & 31)) {
            if (p < 32) mine0 = s0; else mine1 = s0;
          }
          if (lane == ((p + 18) & 31)) {
            if (p + 18 < 32) mine0 = s1; else mine1 = s1;
          }
        }
      }
      atomicAdd(rowsum + static_cast<long long>(lane) * g.rs_pitch + tile, static_cast<int>(mine0));
      if (lane + 32 < kNP4)
        atomicAdd(rowsum + static_cast<long long>(lane + 32) * g.rs_pitch + tile, static_cast<int>(mine1));
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        tp[q][0] = tp[q][4];
        tp[q][1] = tp[q][5];
      }
    }
    if (D > 0) f4_cp_wait<0>();
  }
}

// --------------------------------------------------------------------------
// F2: filters.  u_tmp [36][K][C]; per-position fit; B images + column sums.
__global__ void __launch_bounds__(256, 2) f4_filter_transform_kernel(const float* __restrict__ w,
                                                                     float* __restrict__ u_tmp,
                                                                     float* __restrict__ partials,
                                                                     LanceDevState* __restrict__ st,
                                                                     F4Geom g) {
  pdl_entry();
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
  pdl_entry();
  __shared__ int s_sum[4];
  const int k = blockIdx.x;
  const float top = static_cast<float>((1 << st->bits_w) - 1);
  const long long total = static_cast<long long>(g.K) * g.C;
  for (int p = 0; p < kNP4; ++p) {
    const float tmin = st->w_tmin[p], scale = st->w_scale[p];
    int sum = 0;
    for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
      const uint32_t code = quantize_code(u_tmp[p * total + static_cast<long long>(k) * g.C + c], tmin, scale, top);
      codes_w[umma_image_offset_np(k, c, f4_plane(p), 16, g.bk, g.nk, kNP4)] = static_cast<uint8_t>(code);
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
  __shared__ uint64_t s_bars[2 * 16 + 2 * kF4AccBufs + 1];
  __shared__ uint32_t s_tmem;
  __shared__ int s_fast;

  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stages = g.stages;
  const int nk = g.nk;
  const int U = g.units;  // (plane, k chunk) units per stage; divides 6 * nk
  const bool b_res = g.b_resident != 0;
  const uint32_t a_bytes = U * Cfg::kABytes, b_bytes = b_res ? 0u : U * Cfg::kBBytes;
  const uint32_t stage_bytes = a_bytes + b_bytes;
  uint8_t* b_base = smem + static_cast<size_t>(stages) * stage_bytes;  // resident B (b_res)
  float* s_out = reinterpret_cast<float*>(b_base + (b_res ? kNP4 * g.nk * Cfg::kBBytes : 0));  // [4][32][64]
  uint64_t* full_bar = s_bars;
  uint64_t* empty_bar = s_bars + 16;
  uint64_t* acc_full = s_bars + 32;
  uint64_t* acc_empty = acc_full + kF4AccBufs;
  uint64_t* b_full = acc_empty + kF4AccBufs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = g.num_n_tiles;
  const int num_tiles = ((g.M + kBM - 1) / kBM) * nt;
  const int grp_units = 6 * nk;  // units of one j-group (contiguous, j-major planes)

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < kF4AccBufs; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kF4EpiWarps);
    }
    mbar_init(b_full, 1);
    fence_barrier_init();
  }
  pdl_entry();  // barriers above are shared-memory only
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
    if (warp == kF4EpiWarps) {
      // ---------------- bulk-copy producer ----------------
      // A stage is U consecutive (plane, k chunk) units of the tile's j-major
      // operand images: one contiguous run per operand.  The whole warp runs
      // the uniform loop; one elected lane posts the bytes and issues the
      // copies.
      if (b_res && elect_one()) {  // the CTA's fixed filter tile (grid % nt == 0)
        const uint32_t bb = kNP4 * nk * Cfg::kBBytes;
        mbar_arrive_expect_tx(b_full, bb);
        bulk_load(b_base, codes_w + static_cast<long long>(blockIdx.x % nt) * bb, bb, b_full);
      }
      __syncwarp();
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mt = t / nt, ntile = t - (t / nt) * nt;
        const uint8_t* a_tile = codes_a + static_cast<long long>(mt) * kNP4 * nk * Cfg::kABytes;
        const uint8_t* b_tile = codes_w + static_cast<long long>(ntile) * kNP4 * nk * Cfg::kBBytes;
        for (int u = 0; u < kNP4 * nk; u += U) {
          mbar_wait(&empty_bar[s], ph ^ 1u);
          uint8_t* sa = smem + static_cast<size_t>(s) * stage_bytes;
          if (elect_one()) {
            mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
            bulk_load(sa, a_tile + static_cast<long long>(u) * Cfg::kABytes, a_bytes, &full_bar[s]);
            if (!b_res)
              bulk_load(sa + a_bytes, b_tile + static_cast<long long>(u) * Cfg::kBBytes, b_bytes, &full_bar[s]);
          }
          __syncwarp();
          if (++s == stages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    } else if (warp == kF4EpiWarps + 1) {
      // ---------------- TMEM + UMMA issuer ----------------
      // Warp-uniform loop (addresses / descriptors in uniform registers), one
      // elected lane issues each tcgen05.mma / commit; the (position, k chunk)
      // of a unit is tracked incrementally (no division on the issue path).
      tmem_alloc(&s_tmem, 512);
      tmem_relinquish();
      tc_fence_before();
      named_bar_sync(1, 32 + 32 * kF4EpiWarps);
      tc_fence_after();
      const uint32_t tmem_base = s_tmem;
      if (b_res) mbar_wait(b_full, 0);
      const uint32_t b_res_base = smem_u32(b_base);
      int s = 0;
      uint32_t ph = 0;
      uint32_t grp = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        for (int j = 0; j < 6; ++j, ++grp) {
          const uint32_t buf = grp % kF4AccBufs;
          mbar_wait(&acc_empty[buf], (grp / kF4AccBufs) & 1u);
          tc_fence_after();
          const uint32_t d_base = tmem_base + buf * kF4GroupCols;
          int a = 0, kc = 0;  // unit lu = a * nk + kc of the j-group
          for (int lu0 = 0; lu0 < grp_units; lu0 += U) {
            mbar_wait(&full_bar[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + static_cast<size_t>(s) * stage_bytes);
            for (int uu = 0; uu < U; ++uu) {
              const int lu = lu0 + uu;
              const uint32_t ua = sa + uu * Cfg::kABytes;
              const uint32_t ub = b_res ? b_res_base + (j * grp_units + lu) * Cfg::kBBytes
                                        : sa + a_bytes + uu * Cfg::kBBytes;
              const uint64_t adesc0 = umma_smem_desc(ua, 8 * BK, Cfg::kLayout);
              const uint64_t bdesc0 = umma_smem_desc(ub, 8 * BK, Cfg::kLayout);
              const uint32_t d_a = d_base + static_cast<uint32_t>(a * kF4BN);
#pragma unroll
              for (int kk = 0; kk < BK / 32; ++kk) {
                if (kExpSwitches && (g.exp & 2)) break;
                if (elect_one())
                  umma_i8(d_a, adesc0 + 2 * kk, bdesc0 + 2 * kk, kIdesc, (kc > 0 || kk > 0) ? 1u : 0u);
                __syncwarp();
              }
              if (++kc == nk) {
                kc = 0;
                ++a;
              }
            }
            if (elect_one()) umma_commit(&empty_bar[s]);
            __syncwarp();
            if (++s == stages) {
              s = 0;
              ph ^= 1u;
            }
          }
          if (elect_one()) umma_commit(&acc_full[buf]);
          __syncwarp();
        }
      }
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
    // k3[p] * float(colsum[p][k]) of a tile's 16 filters into s_ct[buf]; the
    // next tile's constants and first row sums are fetched one tile ahead so
    // their global-load latency hides behind the current tile.
    auto fill_ct = [&](int tt, uint32_t b) {
      if (tt >= num_tiles) return;
      const int nn0 = (tt - (tt / nt) * nt) * kF4BN;
      float* c = s_ct[b];
      for (int i = threadIdx.x; i < kNP4 * kF4BN; i += 32 * kF4EpiWarps) {
        const int p = i >> 4, kk = nn0 + (i & 15);
        c[i] = (kk < g.K) ? __fmul_rn(st->k3[p], static_cast<float>(colsum[p * g.K_pad + kk])) : 0.0f;
      }
    };
    auto row_sums_j0 = [&](int tt, int (&rs)[6]) {
      const int mm = (tt / nt) * kBM + row;
      const bool ok = tt < num_tiles && mm < g.M;
#pragma unroll
      for (int a = 0; a < 6; ++a) rs[a] = ok ? __ldg(rowsum + static_cast<long long>(6 * a) * g.rs_pitch + mm) : 0;
    };
    int rs_cur[6];
    fill_ct(blockIdx.x, 0);
    row_sums_j0(blockIdx.x, rs_cur);
    uint32_t grp = 0, lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      const int m0 = (t / nt) * kBM, n0 = (t - (t / nt) * nt) * kF4BN;
      const int m = m0 + row;
      const bool row_ok = m < g.M;
      const int kf0 = n0 + f0;
      // s_ct[lt & 1] was written during the previous tile (or the prologue);
      // after this barrier every thread is done with tile lt - 1, so the other
      // buffer can take the next tile's constants.
      named_bar_sync(2, 32 * kF4EpiWarps);
      float* ct = s_ct[lt & 1u];
      fill_ct(t + gridDim.x, (lt + 1) & 1u);
      float2 S[16][2];  // S[4i + b][filter pair]
#pragma unroll
      for (int j = 0; j < 6; ++j, ++grp) {
        float rterm[6];
#pragma unroll
        for (int a = 0; a < 6; ++a) rterm[a] = __fmul_rn(s_k2[6 * a + j], static_cast<float>(rs_cur[a]));
        if (j < 5) {  // prefetch the next j-group's row sums (hides the load behind this group)
#pragma unroll
          for (int a = 0; a < 6; ++a)
            rs_cur[a] = row_ok ? __ldg(rowsum + static_cast<long long>(6 * a + j + 1) * g.rs_pitch + m) : 0;
        } else {  // ... and across the tile boundary: the next tile's first j-group
          row_sums_j0(t + gridDim.x, rs_cur);
        }
        const uint32_t buf = grp % kF4AccBufs;
        mbar_wait(&acc_full[buf], (grp / kF4AccBufs) & 1u);
        tc_fence_after();
        // Two filters at a time (x2 loads keep 12 accumulators live, not 24);
        // the buffer is released once both halves are in registers.
#pragma unroll
        for (int fh = 0; fh < 2; ++fh) {
          uint32_t ac[6][2];
#pragma unroll
          for (int a = 0; a < 6; ++a)
            tmem_ld_x2(lane_base + buf * kF4GroupCols + a * kF4BN + f0 + 2 * fh, ac[a]);
          tmem_ld_wait();
#pragma unroll
          for (int a = 0; a < 6; ++a) reg_fence(ac[a]);
          if (fh == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
          }
          if (DUMP && row_ok) {
#pragma unroll
            for (int a = 0; a < 6; ++a)
#pragma unroll
              for (int f = 0; f < 2; ++f)
                if (kf0 + 2 * fh + f < g.K)
                  acc_dump[(static_cast<long long>(6 * a + j) * g.M + m) * g.K + kf0 + 2 * fh + f] =
                      static_cast<int32_t>(ac[a][f]);
          }
          if (kExpSwitches && (g.exp & 1)) continue;
          float2 mm[6];
#pragma unroll
          for (int a = 0; a < 6; ++a) {
            const int p = 6 * a + j;
            float2 v;  // RN(RN(k1 * dot) + RN(k2 * sum_a)), two filters
            if (fast) {
              const float2 u = fma2(bcast2(s_k1[p]),
                                    make_float2(__uint_as_float(ac[a][0]), __uint_as_float(ac[a][1])),
                                    bcast2(0.0f));
              v = fma2(u, bcast2(8388608.0f /*2^23*/), bcast2(rterm[a]));
            } else {
              v = add2(make_float2(__fmul_rn(s_k1[p], __int2float_rn(static_cast<int>(ac[a][0]))),
                                   __fmul_rn(s_k1[p], __int2float_rn(static_cast<int>(ac[a][1])))),
                       bcast2(rterm[a]));
            }
            // ((k1*dot + k2*sum_a) + k3*sum_b) + k4 (lowpgemm.hpp:110-114)
            const float2 c2 = *reinterpret_cast<const float2*>(ct + p * kF4BN + f0 + 2 * fh);
            mm[a] = add2(add2(v, c2), bcast2(s_k4[p]));
          }
          float2 T[4];
          at6_2(mm, T);
          // S_ib = sum_j T_ij * A^T[b][j], left fold over j (matrix.hpp:80-82).
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 tv = T[i];
            if (j == 0) {
              S[4 * i + 0][fh] = tv;
            } else if (j == 1) {
              S[4 * i + 0][fh] = add2(S[4 * i + 0][fh], tv);
              S[4 * i + 1][fh] = tv;
              S[4 * i + 2][fh] = tv;
              S[4 * i + 3][fh] = tv;
            } else if (j == 2) {
              S[4 * i + 0][fh] = add2(S[4 * i + 0][fh], tv);
              S[4 * i + 1][fh] = sub2(S[4 * i + 1][fh], tv);
              S[4 * i + 2][fh] = add2(S[4 * i + 2][fh], tv);
              S[4 * i + 3][fh] = sub2(S[4 * i + 3][fh], tv);
            } else if (j == 3 || j == 4) {
              const float2 t2 = add2(tv, tv), t4 = add2(t2, t2), t8 = add2(t4, t4);
              S[4 * i + 0][fh] = add2(S[4 * i + 0][fh], tv);
              S[4 * i + 1][fh] = (j == 3) ? add2(S[4 * i + 1][fh], t2) : sub2(S[4 * i + 1][fh], t2);
              S[4 * i + 2][fh] = add2(S[4 * i + 2][fh], t4);
              S[4 * i + 3][fh] = (j == 3) ? add2(S[4 * i + 3][fh], t8) : sub2(S[4 * i + 3][fh], t8);
            } else {
              S[4 * i + 3][fh] = add2(S[4 * i + 3][fh], tv);
            }
          }
        }
      }
      // merge_tiles (tensor.hpp:157-182): output (4ti + i, 4tj + b), overhang
      // discarded; optional bias / ReLU; +0 canonicalisation.  One output row
      // i at a time, each lane quadrant stages its 32 tiles x 4 pixels x 16
      // filters in shared memory (16-byte chunk c of a tile's 64-float row at
      // c ^ (tile & 7): conflict-free both ways), then its 4 warps write whole
      // 64-byte pixel segments (4 lanes per pixel) instead of one scattered
      // 16-byte piece per lane.
      if (kExpSwitches && (g.exp & 4)) continue;
      int pix0 = 0, vmask = 0;  // first output pixel of this lane's tile; bit 4i + b valid
      if (row_ok) {
        const int img = m / g.P, tt = m - (m / g.P) * g.P;
        const int ti = tt / g.TW, tj = tt - ti * g.TW;
        pix0 = (img * g.OH + 4 * ti) * g.OW + 4 * tj;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (4 * ti + i < g.OH && 4 * tj + b < g.OW) vmask |= 1 << (4 * i + b);
      }
      float2 bv[2] = {bcast2(0.0f), bcast2(0.0f)};
      if (bias != nullptr)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          bv[h] = make_float2(kf0 + 2 * h < g.K ? __ldg(bias + kf0 + 2 * h) : 0.0f,
                              kf0 + 2 * h + 1 < g.K ? __ldg(bias + kf0 + 2 * h + 1) : 0.0f);
      float* stg = s_out + q * (32 * 64);
      const int wq = warp >> 2;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          float2 o[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float2 v = S[4 * i + b][h];
            if (bias != nullptr) v = add2(v, bv[h]);
            if (relu) {
              v.x = fmaxf(v.x, 0.0f);
              v.y = fmaxf(v.y, 0.0f);
            }
            o[h] = add2(v, bcast2(0.0f));  // the reference never yields -0
          }
          const int chunk = (b * 4 + wq) ^ (lane & 7);
          *reinterpret_cast<float4*>(stg + lane * 64 + chunk * 4) = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
        }
        named_bar_sync(3 + q, 128);
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int k = wq * 32 + lane + 128 * it;  // chunk id: fq fastest, then b, then tile
          const int fq = k & 3, b = (k >> 2) & 3, tile = k >> 4;
          const int tpix = __shfl_sync(0xffffffffu, pix0, tile);
          const int tmask = __shfl_sync(0xffffffffu, vmask, tile);
          const float4 val = *reinterpret_cast<const float4*>(stg + tile * 64 + (((b * 4 + fq) ^ (tile & 7)) * 4));
          const int kf = n0 + 4 * fq;
          if (!((tmask >> (4 * i + b)) & 1) || kf >= g.K) continue;
          float* d = y + (static_cast<long long>(tpix) + i * g.OW + b) * g.K + kf;
          if (k4ok) {
            *reinterpret_cast<float4*>(d) = val;
          } else {
            const float e4[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (kf + e < g.K) d[e] = e4[e];
          }
        }
        named_bar_sync(3 + q, 128);  // staging buffer free again
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
  const long long blocks = (g.num_items + 7) / 8;
  const long long cap = 2LL * sm_count;
  return static_cast<int>(blocks < cap ? blocks : cap);
}

static int f4_async_depth() {
  static const int d = lance_knob("LANCE_F4_ASYNC", 2);  // measured: 2 beats 0 (no lookahead) and 4
  return d;
}

static int f4_quant_depth() {
  static const int d = lance_knob("LANCE_F4Q_ASYNC", 2);  // measured: -5 % on the 56x56 layer
  return d;
}

cudaError_t launch_f4_range(const float* x, float* partials, int grid, LanceDevState* st,
                            const F4Geom& g, cudaStream_t s) {
  const int d = f4_async_depth();
  if (d == 2 || d == 4) {
    const size_t smem = static_cast<size_t>(8) * d * 24 * 32 * sizeof(float);
    const cudaError_t e = d == 2 ? ensure_smem_attr(reinterpret_cast<const void*>(f4_range_kernel<2>), smem)
                                 : ensure_smem_attr(reinterpret_cast<const void*>(f4_range_kernel<4>), smem);
    if (e != cudaSuccess) return e;
    if (d == 2)
      LANCE_LAUNCH_CHECK(launch_k(f4_range_kernel<2>, grid, 256, smem, s, x, partials, st, g));
    else
      LANCE_LAUNCH_CHECK(launch_k(f4_range_kernel<4>, grid, 256, smem, s, x, partials, st, g));
  } else {
    LANCE_LAUNCH_CHECK(launch_k(f4_range_kernel<0>, grid, 256, 0, s, x, partials, st, g));
  }
  return cudaGetLastError();
}

cudaError_t launch_f4_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                            const LanceDevState* st, const F4Geom& g, int static_mode,
                            int clear_rowsum, int sm_count, cudaStream_t s) {
  constexpr int kWarps = LANCE_F4Q_THREADS / 32;
  const long long blocks = (g.num_items + kWarps - 1) / kWarps;
  const long long cap = (32LL / kWarps) * sm_count;  // grid-stride over 32 warps' worth per SM
  const int grid = static_cast<int>(blocks < cap ? blocks : cap);
  if (clear_rowsum) {  // else F0 of this forward cleared them
    const cudaError_t e = cudaMemsetAsync(rowsum, 0, sizeof(int32_t) * kNP4 * static_cast<size_t>(g.rs_pitch), s);
    if (e != cudaSuccess) return e;
  }
  const int qd = f4_quant_depth();
  const size_t qsmem = static_cast<size_t>(kWarps) * 2 * 24 * 32 * sizeof(float);
#define LANCE_F4Q(BKV, NKV)                                                                   \
  if ((NKV == 0) || (g.bk == BKV && g.nk == NKV)) {                                           \
    if (qd == 2) {                                                                            \
      const cudaError_t ea = static_mode                                                      \
          ? ensure_smem_attr(reinterpret_cast<const void*>(f4_quant_kernel<true, BKV, NKV, 2>), qsmem)  \
          : ensure_smem_attr(reinterpret_cast<const void*>(f4_quant_kernel<false, BKV, NKV, 2>), qsmem); \
      if (ea != cudaSuccess) return ea;                                                       \
      if (static_mode)                                                                        \
        LANCE_LAUNCH_CHECK(launch_k(f4_quant_kernel<true, BKV, NKV, 2>, grid, LANCE_F4Q_THREADS, qsmem, s, x, codes, rowsum, st, g)); \
      else                                                                                    \
        LANCE_LAUNCH_CHECK(launch_k(f4_quant_kernel<false, BKV, NKV, 2>, grid, LANCE_F4Q_THREADS, qsmem, s, x, codes, rowsum, st, g)); \
    } else if (static_mode) {                                                                 \
      LANCE_LAUNCH_CHECK(launch_k(f4_quant_kernel<true, BKV, NKV>, grid, LANCE_F4Q_THREADS, 0, s, x, codes, rowsum, st, g));          \
    } else {                                                                                  \
      LANCE_LAUNCH_CHECK(launch_k(f4_quant_kernel<false, BKV, NKV>, grid, LANCE_F4Q_THREADS, 0, s, x, codes, rowsum, st, g));         \
    }                                                                                         \
    return cudaGetLastError();                                                                \
  }
  LANCE_F4Q(64, 1)
  LANCE_F4Q(128, 1)
  LANCE_F4Q(128, 2)
  LANCE_F4Q(128, 4)
  LANCE_F4Q(32, 1)
  LANCE_F4Q(0, 0)
#undef LANCE_F4Q
  return cudaGetLastError();
}

cudaError_t launch_f4_filter_prepare(const float* w, float* u_tmp, float* partials, int grid,
                                     uint8_t* codes_w, int32_t* colsum, LanceDevState* st,
                                     const F4Geom& g, cudaStream_t s) {
  LANCE_LAUNCH_CHECK(launch_k(f4_filter_transform_kernel, grid, 256, 0, s, w, u_tmp, partials, st, g));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  LANCE_LAUNCH_CHECK(launch_k(f4_filter_quant_kernel, g.K, 128, 0, s, u_tmp, codes_w, colsum, st, g));
  return cudaGetLastError();
}

template <int BK, bool SMALL, bool DUMP>
static cudaError_t launch_f4_gemm_t(const uint8_t* codes_a, const uint8_t* codes_w,
                                    const int32_t* rowsum, const int32_t* colsum,
                                    const LanceDevState* st, float* y, int32_t* acc_dump,
                                    const float* bias, int relu, const F4Geom& g0, cudaStream_t s) {
  using Cfg = F4Cfg<BK>;
  F4Geom g = g0;
  const size_t kLimit = 220 * 1024;
  const int sms = current_sm_count();
  const int nt = g.num_n_tiles;
  const long long tiles = ((static_cast<long long>(g.M) + kBM - 1) / kBM) * nt;
  // Units per stage: the largest divisor of a j-group's 6 * nk units whose A
  // run stays within 32 KB (fewer, larger bulk copies).
  int U = 1;
  for (int u = 1; u <= 6 * g.nk; ++u)
    if ((6 * g.nk) % u == 0 && u * Cfg::kABytes <= 32 * 1024) U = u;
  {
    const int v = lance_knob("LANCE_F4_UNITS", 0);
    if (v >= 1 && (6 * g.nk) % v == 0) U = v;
  }
  g.units = U;
  // Resident B: the CTA keeps one filter tile (36 planes x nk chunks x 16 x BK)
  // when it fits beside a few stages; the grid is then a multiple of nt so each
  // CTA's tiles share one filter tile.
  const size_t b_bytes = static_cast<size_t>(kNP4) * g.nk * Cfg::kBBytes;
  const int res_grid = (sms / nt) * nt;
  g.b_resident = (b_bytes <= 80 * 1024 && res_grid >= 1) ? 1 : 0;
  g.b_resident = g.b_resident && lance_knob("LANCE_F4_BRES", 1) != 0;
  const size_t stage_bytes = static_cast<size_t>(U) * (Cfg::kABytes + (g.b_resident ? 0 : Cfg::kBBytes));
  const size_t fixed = 1024 + (g.b_resident ? b_bytes : 0) + 4 * 32 * 64 * sizeof(float);
  int stages = 16;
  while (stages > 2 && fixed + stages * stage_bytes > kLimit) --stages;
  g.stages = stages;
  const size_t smem = fixed + stages * stage_bytes;
  if (smem > kLimit) return cudaErrorInvalidValue;
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(f4_gemm_kernel<BK, SMALL, DUMP>), kLimit);
    if (e != cudaSuccess) return e;
  }
  const int cap = g.b_resident ? res_grid : sms;
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  LANCE_LAUNCH_CHECK(launch_k(f4_gemm_kernel<BK, SMALL, DUMP>, grid, kF4Threads, smem, s, codes_a, codes_w, rowsum, colsum,
                                                                  st, y, acc_dump, bias, relu, g));
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
