// lance_common.cuh -- device math shared by the LANCE kernels.
//
// Bit-exactness with the reference: every floating-point
// operation is an explicit IEEE round-to-nearest intrinsic (scalar or packed
// f32x2, which is two independent IEEE operations) in the reference's
// association order; the library is compiled with -fmad=false, no fast-math.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "lance_kernels.cuh"
#include "lance_ptx.cuh"

namespace lance_dev {

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: every forward-path kernel is launched with
// programmatic stream serialisation (launch_k), so it may become resident
// while its predecessor drains.  pdl_entry() first lets this grid's own
// dependent launch early, then blocks until the predecessor grid has completed
// and its memory is visible (griddepcontrol.wait): nothing before it may touch
// global memory.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// ---------------------------------------------------------------- packed f32x2
// sm_100a FADD2 / FMUL2 / FFMA2: two IEEE-RN operations per instruction.
#define LANCE_F2_BINOP(name, op)                                                             \
  __device__ __forceinline__ float2 name(float2 a, float2 b) {                               \
    float2 r;                                                                                \
    asm("{.reg .b64 a, b, d; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; " op                  \
        " d, a, b; mov.b64 {%0, %1}, d;}"                                                    \
        : "=f"(r.x), "=f"(r.y)                                                               \
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));                                           \
    return r;                                                                                \
  }
LANCE_F2_BINOP(add2, "add.rn.f32x2")
LANCE_F2_BINOP(sub2, "sub.rn.f32x2")
#undef LANCE_F2_BINOP
// NOTE: there is deliberately no packed multiply.  ptxas (CUDA 12.9) contracts
// mul.rn.f32x2 followed by add.rn.f32x2 into FFMA2 even with .rn and
// -fmad=false, which changes the rounding; products are issued as scalar
// __fmul_rn (never contracted) and only the adds are packed.
__device__ __forceinline__ float2 mul2_rn(float2 a, float2 b) {
  return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 a, b, c, d; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; mov.b64 c, {%6, %7}; "
      "fma.rn.f32x2 d, a, b, c; mov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

__device__ __forceinline__ float2 bcast2(float v) { return make_float2(v, v); }

// 3-input NaN-propagating min / max (FMNMX3.NAN).
__device__ __forceinline__ float fmin3_nan(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// ---------------------------------------------------------------- transforms
// winograd.hpp:40-84 evaluated in matrix.hpp:75-84 order (Bt d first combines
// the rows a of each column b).  Products with zero basis entries only affect
// signed zeros, which are canonicalised where observable (ranges, y).

// v = (B^T d) B, two channels at once; d, v indexed [a*4 + b].
__device__ __forceinline__ void input_transform2(const float2 (&d)[16], float2 (&v)[16]) {
  float2 t[16];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    t[0 * 4 + b] = sub2(d[0 * 4 + b], d[2 * 4 + b]);
    t[1 * 4 + b] = add2(d[1 * 4 + b], d[2 * 4 + b]);
    t[2 * 4 + b] = sub2(d[2 * 4 + b], d[1 * 4 + b]);
    t[3 * 4 + b] = sub2(d[1 * 4 + b], d[3 * 4 + b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    v[a * 4 + 0] = sub2(t[a * 4 + 0], t[a * 4 + 2]);
    v[a * 4 + 1] = add2(t[a * 4 + 1], t[a * 4 + 2]);
    v[a * 4 + 2] = sub2(t[a * 4 + 2], t[a * 4 + 1]);
    v[a * 4 + 3] = sub2(t[a * 4 + 1], t[a * 4 + 3]);
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

// ---------------------------------------------------------------- quantize
// Exact reference quantizer (quant.hpp:77-84): scale == 0 -> 0;
// units = roundf((x - tmin) / scale) with IEEE division, half away from zero;
// !(units > 0) -> 0; units >= top -> top.  For q >= 0.5 and q < 2^23,
// round-half-away(q) == floor(RN(q + 0.5)); every q < 0.5 (negatives, NaN)
// maps to 0; q >= 2^23 saturates to top either way.
__device__ __forceinline__ uint32_t quantize_code(float v, float tmin, float scale, float top) {
  const float d = __fsub_rn(v, tmin);
  const float q = __fdiv_rn(d, scale);
  const float r = floorf(__fadd_rn(q, 0.5f));
  const float c = (q >= 0.5f) ? fminf(r, top) : 0.0f;
  return (scale == 0.0f) ? 0u : static_cast<uint32_t>(c);
}

// Fast quantizer (division-free).  q0 = RN(d * RN(1/scale)) is within
// 1.5 * 2^-15 of q = RN(d / scale) whenever q <= 256 (relative error of the
// reciprocal <= 2^-24 plus one rounding of q0, ulp(q0) <= 2^-15).  The
// nearest integer n of q0 is taken with the 1.5 * 2^23 magic addend; if
// |q0 - n| < 0.5 - 2^-14 then |q - n| < 0.5, so the reference's
// round-half-away(q) is n exactly.  Values with |q0 - n| >= 0.5 - 2^-14 (or
// NaN) are flagged and re-quantised with quantize_code by the caller.
constexpr float kMagic = 12582912.0f;            // 1.5 * 2^23
constexpr float kTieGuard = 0.49993896484375f;   // 0.5 - 2^-14

// Exact reference code for a value whose fast-path residual flagged it as
// being near the rounding boundary h = n + 0.5*sign(r) (dynamic params: d >= 0,
// scale > 0 normal).  roundf(RN(d/s)) crosses to the upper code iff
// RN(d/s) >= h, i.e. iff d/s > mid(pred(h), h) (a float quotient is never a
// midpoint, so there is no tie), i.e. iff d - s*h > -s*delta with
// delta = (h - pred(h))/2.  d - s*h is exactly representable here
// (|d - s*h| <= s*2^-13, granularity ulp(s)/2), so one FFMA decides it.
__device__ __forceinline__ uint32_t exact_code_near_boundary(float d, float s, float gq, float r,
                                                             float top) {
  const float n = __fsub_rn(gq, kMagic);
  const float h = (r > 0.0f) ? __fadd_rn(n, 0.5f) : __fsub_rn(n, 0.5f);
  const float lower = (r > 0.0f) ? n : __fsub_rn(n, 1.0f);
  const float upper = __fadd_rn(lower, 1.0f);
  const float pred_h = __int_as_float(__float_as_int(h) - 1);
  const float delta = __fmul_rn(__fsub_rn(h, pred_h), 0.5f);
  const float e = __fmaf_rn(-s, h, d);
  float c = (e > -__fmul_rn(s, delta)) ? upper : lower;
  c = fminf(fmaxf(c, 0.0f), top);
  return static_cast<uint32_t>(c);
}

// ---------------------------------------------------------------- ranges
// Block-wide (min, max) of lo[16] / hi[16] -> this block's 32 partials.
__device__ __forceinline__ void block_minmax_to_partials(float (&lo)[16], float (&hi)[16],
                                                         float* partials, float* s_red /*[blockDim.x]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
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
    for (int w = 1; w < nw; ++w)
      r = (i < 16) ? fmin_nan(r, s_red[w * 32 + i]) : fmax_nan(r, s_red[w * 32 + i]);
    partials[static_cast<long long>(blockIdx.x) * 32 + i] = r;
  }
}

// Zero `words` int32 from every thread of the grid (16-byte stores, scalar
// tail); nullptr: nothing.  The range kernels clear the row-sum planes that
// the quantisers then accumulate atomically.
__device__ __forceinline__ void grid_zero_i32(int32_t* z, long long words) {
  if (z == nullptr) return;
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long nth = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long n4 = words >> 2;
  for (long long i = tid; i < n4; i += nth) reinterpret_cast<int4*>(z)[i] = make_int4(0, 0, 0, 0);
  for (long long i = 4 * n4 + tid; i < words; i += nth) z[i] = 0;
}

// Fold the 32-float partials of nb blocks -> s_red[0..31] (whole block).
__device__ __forceinline__ void fold_partials(const float* partials, int nb, float* s_red) {
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int col = threadIdx.x & 31;
  float r = (col < 16) ? __int_as_float(0x7f800000) : __int_as_float(0xff800000);
  // Eight independent partial loads in flight per thread (a serial chain of
  // dependent L2 round trips here cost tens of microseconds on small layers).
  for (int b0 = warp; b0 < nb; b0 += 8 * nw) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int b = b0 + u * nw;
      v[u] = (b < nb) ? __ldcg(partials + static_cast<long long>(b) * 32 + col) : r;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) r = (col < 16) ? fmin_nan(r, v[u]) : fmax_nan(r, v[u]);
  }
  __syncthreads();
  s_red[threadIdx.x] = r;
  __syncthreads();
  if (threadIdx.x < 32) {
    float q = s_red[threadIdx.x];
    for (int w = 1; w < nw; ++w)
      q = (threadIdx.x < 16) ? fmin_nan(q, s_red[w * 32 + threadIdx.x])
                             : fmax_nan(q, s_red[w * 32 + threadIdx.x]);
    s_red[threadIdx.x] = q;
  }
  __syncthreads();
}

// Block-wide (min, max) partials -> the last block to finish folds all
// partials; returns true in that block with the 32 results in s_red[0..31].
__device__ __forceinline__ bool block_minmax_and_ticket(float (&lo)[16], float (&hi)[16],
                                                        float* partials, unsigned int* ticket,
                                                        float* s_red /*[blockDim.x]*/) {
  block_minmax_to_partials(lo, hi, partials, s_red);
  __threadfence();
  __syncthreads();
  __shared__ unsigned int s_last;
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  fold_partials(partials, static_cast<int>(gridDim.x), s_red);
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// fit_params (quant.hpp:54-72) from the reduced (lo[16], hi[16]) in
// s_red[0..31].  PerTensor (engines.hpp:151-156) folds the 16 ranges; param_at
// then returns params[0] for every position (engines.hpp:131-136).  A NaN or
// non-finite range sets *nan_flag (the reference throws "fit_params: NaN in
// values"; any non-finite input makes its 0 * inf transform products NaN).
__device__ __forceinline__ void fit_from_ranges(const float* s_red, int gran, int bits,
                                                float* tmin, float* tmax, float* scale,
                                                float* rcp, int* nan_flag) {
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
    const float s = __fdiv_rn(__fsub_rn(hi, lo), static_cast<float>((1 << bits) - 1));
    tmin[p] = lo;
    tmax[p] = hi;
    scale[p] = s;
    if (rcp) rcp[p] = (s == 0.0f) ? 0.0f : __frcp_rn(s);
    const unsigned anybad = __ballot_sync(0x0000ffffu, bad);
    if (p == 0) *nan_flag = anybad ? 1 : 0;
  }
}

// Hoisted constants of affine_term (lowpgemm.hpp:110-114), a = input,
// b = weight:  m = ((k1*dot + k2*sum_a) + k3*sum_b) + k4.
__device__ __forceinline__ void make_epilogue_consts(LanceDevState* st, int C, int np = 16) {
  if (threadIdx.x < np) {
    const int p = threadIdx.x;
    const float sa = st->a_scale[p], oa = st->a_tmin[p];
    const float sb = st->w_scale[p], ob = st->w_tmin[p];
    st->k1[p] = __fmul_rn(sa, sb);
    st->k2[p] = __fmul_rn(sa, ob);
    st->k3[p] = __fmul_rn(sb, oa);
    st->k4[p] = __fmul_rn(__fmul_rn(static_cast<float>(C), oa), ob);
  }
}

}  // namespace lance_dev
