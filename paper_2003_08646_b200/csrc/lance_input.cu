// lance_input.cu -- input side of the LANCE path on sm_100a.
//
//   K0 input_range_kernel  per-position (min, max) of v = B^T d B over the whole
//                          batch (quantize_domain PerPosition / PerTensor fit,
//                          engines.hpp:151-165, fit_params quant.hpp:54-72);
//                          the last block folds the partials into
//                          QuantParams[16] and the epilogue constants.
//   K1 input_quant_kernel  v recomputed and quantised (quant.hpp:77-84) to u8
//                          codes [16][M][C_pad] (the K-major A operand of the
//                          position GEMMs) plus row sums [16][M]
//                          (lowpgemm.hpp:121-123).
//
// Mapping: one warp = one segment of a tile row (image img, tile row ti,
// tiles tj0..tj1) x 64 channels (2 per lane, float2 NHWC loads: 256
// contiguous bytes per pixel per warp).  The tile gather is extract_tiles
// (tensor.hpp:116-152): origin (2ti - pad, 2tj - pad), zero padding.
// Horizontally adjacent tiles share two pixel columns, so the warp slides along
// the row: per tile it loads 2 new columns (8 pixels) and reuses the first
// (column) pass of the transform for the 2 shared columns.  Transforms run on
// packed f32x2 (FADD2), ranges on 3-input FMNMX3.NAN.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "lance_common.cuh"

namespace lance_dev {

#ifndef LANCE_K1_INTERIOR
#define LANCE_K1_INTERIOR 1
#endif
constexpr bool K1_INTERIOR = LANCE_K1_INTERIOR != 0;
// K1 fast path: position pairs per tie vote.  2 (four positions, eight values
// per lane per __any_sync) measured 2.256 -> 2.190 ms on the step (K1 R64 121
// -> 113 us, R128 85 -> 77 us); 4 is no better and 1 was the round-1 form.
#ifndef LANCE_K1_KG
#define LANCE_K1_KG 2
#endif
constexpr int K1_KG = LANCE_K1_KG;
// K1 fast path CTA shape: 4-warp CTAs, 5 per SM (registers capped at 96,
// 20 warps per SM instead of 16).  Measured 2.180 -> 2.103 ms on the step,
// K1 R64 113 -> 103 us; 6 per SM (80 registers) spills and is slower.
#ifndef LANCE_K1_THREADS
#define LANCE_K1_THREADS 128
#endif
#ifndef LANCE_K1_MINB
#define LANCE_K1_MINB 5
#endif
constexpr int K1_THREADS = LANCE_K1_THREADS;
// K0 ring kernel CTA shape (the ring is per warp: 10 KB of shared memory
// each).  4-warp CTAs at 5 per SM (96 registers) measured slower than 8-warp
// CTAs at 2 per SM: R64 79 vs 70 us, R512 32 vs 25 us.
#ifndef LANCE_K0_THREADS
#define LANCE_K0_THREADS 256
#endif
#ifndef LANCE_K0_MINB
#define LANCE_K0_MINB 2
#endif
#ifndef LANCE_K0_DEPTH
#define LANCE_K0_DEPTH 4  // K0 ring: column pairs in flight per warp (2: +0.5 %, 6: +5 % step time)
#endif

// Warp work item: (img, ti, tile segment, channel chunk).
struct StripItem {
  int img, ti, tj0, tj1, ch;
};

__device__ __forceinline__ StripItem strip_item(const InGeom& g, long long item, int lane) {
  const int chunk = static_cast<int>(item % g.nchunks);
  long long r = item / g.nchunks;
  const int seg = static_cast<int>(r % g.nseg);
  r /= g.nseg;
  const int ti = static_cast<int>(r % g.TH);
  const int img = static_cast<int>(r / g.TH);
  const int tj0 = seg * g.seg_len;
  const int tj1 = min(tj0 + g.seg_len, g.TW);
  return {img, ti, tj0, tj1, chunk * kChunk + 2 * lane};
}

__device__ __forceinline__ void colpass(const float2 (&d)[4], float2 (&t)[4]);

// Row context of a strip: the 4 input rows of tile row ti for this lane's
// channel pair, with validity (zero padding above / below the image).
template <bool VEC2>
struct Strip {
  const float* row[4];
  bool rok[4];
  bool c0ok, c1ok;  // channel ch / ch + 1 < C
  int W, C;

  __device__ __forceinline__ Strip(const float* __restrict__ x, const InGeom& g,
                                   const StripItem& it) {
    W = g.W;
    C = g.C;
    c0ok = it.ch < g.C;
    c1ok = it.ch + 1 < g.C;
    const float* base = x + static_cast<long long>(it.img) * g.H * g.W * g.C + it.ch;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int yy = 2 * it.ti - g.pad + a;
      rok[a] = (yy >= 0) && (yy < g.H);
      row[a] = base + static_cast<long long>(rok[a] ? yy : 0) * g.W * g.C;
    }
  }

  // The 4 pixels (rows 0..3 of the strip) of input column xx, this lane's
  // channel pair; zero outside the image.
  __device__ __forceinline__ void load(int xx, float2 (&d)[4]) const {
    const bool cok = (xx >= 0) && (xx < W);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const float* px = row[a] + static_cast<long long>(cok ? xx : 0) * C;
      const bool ok = cok && rok[a];
      if (VEC2) {
        d[a] = (ok && c0ok) ? __ldg(reinterpret_cast<const float2*>(px)) : make_float2(0.f, 0.f);
      } else {
        d[a].x = (ok && c0ok) ? __ldg(px) : 0.f;
        d[a].y = (ok && c1ok) ? __ldg(px + 1) : 0.f;
      }
    }
  }

  // Unpredicated variant for columns inside the image with all 4 rows valid.
  __device__ __forceinline__ void load_in(int xx, float2 (&d)[4]) const {
#pragma unroll
    for (int a = 0; a < 4; ++a) d[a] = __ldg(reinterpret_cast<const float2*>(row[a] + static_cast<long long>(xx) * C));
  }
  __device__ __forceinline__ bool rows_ok() const { return rok[0] && rok[1] && rok[2] && rok[3] && c0ok; }

  // Column pass of B^T d for input column xx: t[a] = (B^T d)(a, col).
  __device__ __forceinline__ void column(int xx, float2 (&t)[4]) const {
    float2 d[4];
    load(xx, d);
    colpass(d, t);
  }
};

__device__ __forceinline__ void colpass(const float2 (&d)[4], float2 (&t)[4]) {
  t[0] = sub2(d[0], d[2]);
  t[1] = add2(d[1], d[2]);
  t[2] = sub2(d[2], d[1]);
  t[3] = sub2(d[1], d[3]);
}

// Second (row) pass: v[a*4+b] from the column-pass results of 4 columns.
__device__ __forceinline__ void row_pass(const float2 (&t0)[4], const float2 (&t1)[4],
                                         const float2 (&t2)[4], const float2 (&t3)[4],
                                         float2 (&v)[16]) {
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    v[a * 4 + 0] = sub2(t0[a], t2[a]);
    v[a * 4 + 1] = add2(t1[a], t2[a]);
    v[a * 4 + 2] = sub2(t2[a], t1[a]);
    v[a * 4 + 3] = sub2(t1[a], t3[a]);
  }
}

// --------------------------------------------------------------------------
// K0: per-position range of v over the whole batch (grid-stride over strips).
template <bool VEC2>
__global__ void __launch_bounds__(256, 2) input_range_kernel(const float* __restrict__ x,
                                                             float* __restrict__ partials,
                                                             LanceDevState* __restrict__ st,
                                                             InGeom g) {
  pdl_entry();
  grid_zero_i32(g.rs_zero, g.rs_zero_words);  // K1's atomic row sums (multi-chunk layers)
  __shared__ float s_red[256];
  float lo[16], hi[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const int lane = threadIdx.x & 31;
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long item = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       item < g.num_items; item += stride) {
    const StripItem it = strip_item(g, item, lane);
    if (it.ch >= g.C) continue;  // lane beyond C (only in the last channel chunk)
    const Strip<VEC2> sp(x, g, it);
    const bool two = it.ch + 1 < g.C;
    float2 ta[4], tb[4], tc[4], td[4], pc[4], pd[4];
    int xx = 2 * it.tj0 - g.pad;
    sp.column(xx, ta);
    sp.column(xx + 1, tb);
    sp.load(xx + 2, pc);
    sp.load(xx + 3, pd);
    for (int tj = it.tj0; tj < it.tj1; ++tj, xx += 2) {
      colpass(pc, tc);
      colpass(pd, td);
      if (tj + 1 < it.tj1) {  // software prefetch of the next tile's two new columns
        sp.load(xx + 4, pc);
        sp.load(xx + 5, pd);
      }
      float2 v[16];
      row_pass(ta, tb, tc, td, v);
      if (two) {
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          lo[p] = fmin3_nan(lo[p], v[p].x, v[p].y);
          hi[p] = fmax3_nan(hi[p], v[p].x, v[p].y);
        }
      } else {  // odd C: the lane's second channel is padding
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          lo[p] = fmin_nan(lo[p], v[p].x);
          hi[p] = fmax_nan(hi[p], v[p].x);
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ta[a] = tc[a];
        tb[a] = td[a];
      }
    }
  }
  if (block_minmax_and_ticket(lo, hi, partials, &st->ticket_in, s_red)) {
    fit_from_ranges(s_red, g.granularity, st->bits_i, st->a_tmin, st->a_tmax, st->a_scale,
                    st->a_rcp, &st->nan_in);
    __syncthreads();
    make_epilogue_consts(st, g.C);
  }
}

// Quantise one tile's v (this lane's channel pair) and store the codes into
// the A operand's UMMA images at dst (position planes pstride apart); returns
// this lane's row sum (lane p < 16: position p) of the warp's 64 channels.
// Generic over C (lane_on / two: the lane's channels exist).
template <bool STATIC>
__device__ __forceinline__ uint32_t quant_store_generic(const float2 (&v)[16], bool lane_on, bool two,
                                                        uint8_t* dst, long long pstride,
                                                        const float* s_tmin, const float* s_scale,
                                                        const float* s_rcp, float top, int lane) {
  uint32_t mine = 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint32_t pk[2] = {0u, 0u};
    if (lane_on) {
      float2 dd[2], gq[2], r[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * k + h;
        dd[h] = sub2(v[p], bcast2(s_tmin[p]));
        if (STATIC) {
          float2 q = mul2_rn(dd[h], bcast2(s_rcp[p]));
          q.x = fminf(fmaxf(q.x, 0.0f), top);  // NaN -> 0 like quant.hpp:81
          q.y = fminf(fmaxf(q.y, 0.0f), top);
          gq[h] = add2(q, bcast2(kMagic));
          r[h] = sub2(q, sub2(gq[h], bcast2(kMagic)));
        } else {
          gq[h] = fma2(dd[h], bcast2(s_rcp[p]), bcast2(kMagic));
          r[h] = fma2(dd[h], bcast2(s_rcp[p]),
                      make_float2(-__fsub_rn(gq[h].x, kMagic), -__fsub_rn(gq[h].y, kMagic)));
        }
        pk[h] = __byte_perm(__float_as_uint(gq[h].x), __float_as_uint(gq[h].y), 0x0040) & 0xFFFFu;
      }
      const float rmax = fmax3_nan(fmax3_nan(fabsf(r[0].x), fabsf(r[0].y), fabsf(r[1].x)),
                                   fabsf(r[1].y), 0.0f);
      if (!(rmax < kTieGuard)) {
        // Rare (~1e-4 per value): re-derive the flagged codes exactly.
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int p = 2 * k + h;
          uint32_t c0, c1;
          if (STATIC) {
            c0 = quantize_code(v[p].x, s_tmin[p], s_scale[p], top);
            c1 = quantize_code(v[p].y, s_tmin[p], s_scale[p], top);
          } else {
            c0 = (fabsf(r[h].x) < kTieGuard)
                     ? (pk[h] & 0xFFu)
                     : exact_code_near_boundary(dd[h].x, s_scale[p], gq[h].x, r[h].x, top);
            c1 = (fabsf(r[h].y) < kTieGuard)
                     ? (pk[h] >> 8)
                     : exact_code_near_boundary(dd[h].y, s_scale[p], gq[h].y, r[h].y, top);
          }
          pk[h] = c0 | (c1 << 8);
        }
      }
      if (!two) {  // odd C: padding channel code 0
        pk[0] &= 0x00FFu;
        pk[1] &= 0x00FFu;
      }
      // Codes: 64 contiguous bytes per warp per position (the A operand row).
      // position planes in j-major image order (umma_image_offset)
      const int p0 = 2 * k, p1 = 2 * k + 1;
      *reinterpret_cast<uint16_t*>(dst + image_plane(p0) * pstride) = static_cast<uint16_t>(pk[0]);
      *reinterpret_cast<uint16_t*>(dst + image_plane(p1) * pstride) = static_cast<uint16_t>(pk[1]);
    }
    // Row sums (lowpgemm.hpp:121-123): the lane's two codes of positions
    // (2k, 2k+1) as 16-bit halves, one warp reduction (REDUX) per pair.
    const uint32_t a = pk[0] | (pk[1] << 16);                          // [p.c0, p.c1, q.c0, q.c1]
    const uint32_t w = (a & 0x00FF00FFu) + ((a >> 8) & 0x00FF00FFu);  // [p sum | q sum]
    const uint32_t tot = __reduce_add_sync(0xffffffffu, w);
    if ((lane >> 1) == k) mine = (lane & 1) ? (tot >> 16) : (tot & 0xFFFFu);
  }
  return mine;
}

// --------------------------------------------------------------------------
// K1: codes + row sums, one strip per warp.
//
// Dynamic params (the reference's batch fit): d = v - tmin is in [0, range],
// so the exact product P = d * RN(1/scale) is within 2^-16 of d / scale <= 256.
// n = rint(P) comes from one FFMA2 with the 1.5 * 2^23 magic addend and
// r = RN(P - n) from another.  If |r| < 0.5 - 2^-14 then |RN(d / scale) - n|
// < 0.5, so the reference's roundf((x - t_min) / scale) equals n exactly
// (no clamp needed: 0 <= n <= top).  Otherwise (probability ~1e-4 per value)
// the lane re-quantises the flagged values with the IEEE formula.
// Static params (caller supplied): q may be anywhere, so it is formed with a
// scalar IEEE multiply, clamped to [0, top] and rounded with the magic addend.
template <bool VEC2, bool STATIC>
__global__ void __launch_bounds__(256, 2) input_quant_kernel(const float* __restrict__ x,
                                                             uint8_t* __restrict__ codes,
                                                             int32_t* __restrict__ rowsum,
                                                             const LanceDevState* __restrict__ st,
                                                             InGeom g) {
  pdl_entry();
  __shared__ float s_tmin[16], s_scale[16], s_rcp[16];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 16) {
    s_tmin[tid] = st->a_tmin[tid];
    s_scale[tid] = st->a_scale[tid];
    s_rcp[tid] = st->a_rcp[tid];
  }
  const float top = static_cast<float>((1 << st->bits_i) - 1);
  __syncthreads();
  // Reverse order: the range pass (K0) just streamed x front to back, so the
  // tail of x is still in L2 when this kernel starts; and the GEMM, which
  // reads the codes front to back, then finds the last-written rows in L2.
  const long long wi = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (tid >> 5);
  if (wi >= g.num_items) return;
  const long long item = g.rev_items ? g.num_items - 1 - wi : wi;
  const StripItem it = strip_item(g, item, lane);
  const bool lane_on = it.ch < g.C;
  const bool two = it.ch + 1 < g.C;
  const Strip<VEC2> sp(x, g, it);
  // Codes go to the A operand's UMMA images (lance_kernels.cuh): position
  // planes are nk images apart within a 128-row block.
  const long long pstride = static_cast<long long>(g.a_nk) * kBM * g.a_bk;
  float2 ta[4], tb[4], tc[4], td[4], pc[4], pd[4];
  int xx = 2 * it.tj0 - g.pad;
  if (lane_on) {
    sp.column(xx, ta);
    sp.column(xx + 1, tb);
    sp.load(xx + 2, pc);
    sp.load(xx + 3, pd);
  }
  int m = (it.img * g.TH + it.ti) * g.TW + it.tj0;
  for (int tj = it.tj0; tj < it.tj1; ++tj, xx += 2, ++m) {
    float2 v[16];
    if (lane_on) {
      colpass(pc, tc);
      colpass(pd, td);
      if (tj + 1 < it.tj1) {  // software prefetch of the next tile's two new columns
        sp.load(xx + 4, pc);
        sp.load(xx + 5, pd);
      }
      row_pass(ta, tb, tc, td, v);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ta[a] = tc[a];
        tb[a] = td[a];
      }
    }
    uint8_t* dst = codes + umma_image_offset(m, it.ch, 0, kBM, g.a_bk, g.a_nk);
    const uint32_t mine = quant_store_generic<STATIC>(v, lane_on, two, dst, pstride, s_tmin, s_scale,
                                                      s_rcp, top, lane);
    if (g.rowsums && lane < 16) {
      int32_t* rs = rowsum + static_cast<long long>(lane) * g.rs_pitch + m;
      if (g.nchunks == 1)
        *rs = static_cast<int32_t>(mine);
      else  // channel chunks of one tile run in different warps (rowsum pre-zeroed)
        atomicAdd(rs, static_cast<int32_t>(mine));
    }
  }
}

// K1 fast path: dynamic params, C % 64 == 0 (every lane owns two real
// channels), even C.  Same arithmetic as input_quant_kernel without the
// per-lane validity branches; BK is a template parameter so the UMMA-image
// address is a handful of shifts per tile, and the tie fix-up is one
// warp-uniform branch per position pair.
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8_sz(void* sdst, const void* gsrc, uint32_t src_bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// STATIC: caller-supplied params (values may lie outside [t_min, t_max]):
// q = RN(d * rcp) is clamped to [-1, top + 1] before the magic-number rounding
// and the code to [0, top]; far-out values then round to 0 / top exactly as the
// reference's clamps do, and near-ties (|residual| >= 0.5 - 2^-14, which
// includes the 0.5 and top + 0.5 boundaries) take the IEEE-division quantiser.
// v (row pass, winograd.hpp:40-84 order) is formed per position from the four
// column-pass results right where it is quantised, so at most one row of v is
// live at a time (the fast path then fits 96 registers).
__device__ __forceinline__ float2 row_pass_at(int p, const float2 (&t0)[4], const float2 (&t1)[4],
                                              const float2 (&t2)[4], const float2 (&t3)[4]) {
  const int a = p >> 2, b = p & 3;
  return b == 0 ? sub2(t0[a], t2[a]) : b == 1 ? add2(t1[a], t2[a]) : b == 2 ? sub2(t2[a], t1[a]) : sub2(t1[a], t3[a]);
}

// Quantise one tile's 16 positions (this lane's channel pair), store the
// codes into the UMMA images and (RS) the row sums of tile m.
template <int BK, int NK, bool RS, bool STATIC>
__device__ __forceinline__ void quant_fast_tile(const float2 (&t0)[4], const float2 (&t1)[4],
                                                const float2 (&t2)[4], const float2 (&t3)[4],
                                                int m, uint8_t* const cbase, int cb,
                                                int32_t* __restrict__ rowsum, const InGeom& g, int lane,
                                                const float* s_tmin, const float* s_scale,
                                                const float* s_rcp, float top, uint32_t* s_rsw) {
  constexpr int kImg = kBM * BK;                       // bytes of one image
  constexpr uint32_t kMask = BK == 128 ? 7u : (BK == 64 ? 3u : 1u);
  constexpr int pstride = NK * kImg;           // one position plane (compile-time: immediate offsets)
  constexpr long long blkstride = 16LL * pstride;  // one 128-row block
  const uint32_t lin = static_cast<uint32_t>((m & (kBM - 1)) * BK + cb);
  uint8_t* dst = cbase + (m >> 7) * blkstride + (lin ^ (((lin >> 7) & kMask) << 4));
  uint32_t tot[8];  // RS: warp sums of positions (2k, 2k + 1) as 16-bit halves (warp-uniform)
  // KG position pairs share one tie vote (KG = 2: 8 values per lane per vote).
#pragma unroll
  for (int kg = 0; kg < 8; kg += K1_KG) {
    float2 v[2 * K1_KG], dd[2 * K1_KG], gq[2 * K1_KG], r[2 * K1_KG];
#pragma unroll
    for (int h = 0; h < 2 * K1_KG; ++h) {
      const int p = 2 * kg + h;
      const float rcp = s_rcp[p];
      v[h] = row_pass_at(p, t0, t1, t2, t3);
      dd[h] = sub2(v[h], bcast2(s_tmin[p]));
      gq[h] = fma2(dd[h], bcast2(rcp), bcast2(kMagic));
      r[h] = fma2(dd[h], bcast2(rcp), sub2(bcast2(kMagic), gq[h]));
    }
    uint32_t pk[2 * K1_KG];
#pragma unroll
    for (int h = 0; h < 2 * K1_KG; ++h)
      pk[h] = __byte_perm(__float_as_uint(gq[h].x), __float_as_uint(gq[h].y), 0x0040);
    float rmax = 0.0f;
#pragma unroll
    for (int h = 0; h < 2 * K1_KG; h += 2)
      rmax = fmax3_nan(fmax3_nan(fabsf(r[h].x), fabsf(r[h].y), fabsf(r[h + 1].x)), fabsf(r[h + 1].y), rmax);
    if (STATIC) {
      // Caller params: a value whose rounded code falls outside [0, top]
      // (or whose product is too large for the magic-number rounding) joins
      // the exact path, which applies the reference's clamps.
      float glo = kMagic, ghi = kMagic;
#pragma unroll
      for (int h = 0; h < 2 * K1_KG; ++h) {
        glo = fmin3_nan(glo, gq[h].x, gq[h].y);
        ghi = fmax3_nan(ghi, gq[h].x, gq[h].y);
      }
      if (!(glo >= kMagic) || !(ghi <= __fadd_rn(kMagic, top))) rmax = 1.0f;
    }
    if (__builtin_expect(__any_sync(0xffffffffu, !(rmax < kTieGuard)), 0)) {
      // Rare (~1e-4 per value): re-derive flagged codes exactly.
      if (!(rmax < kTieGuard)) {
#pragma unroll
        for (int h = 0; h < 2 * K1_KG; ++h) {
          const int p = 2 * kg + h;
          const float sc = s_scale[p];
          uint32_t c[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float dv = e ? dd[h].y : dd[h].x, gv = e ? gq[h].y : gq[h].x, rv = e ? r[h].y : r[h].x;
            if (STATIC)
              c[e] = (fabsf(rv) < kTieGuard && gv >= kMagic && gv <= __fadd_rn(kMagic, top))
                         ? (__float_as_uint(gv) & 0xFFu)
                         : quantize_code(e ? v[h].y : v[h].x, s_tmin[p], sc, top);
            else
              c[e] = (fabsf(rv) < kTieGuard) ? (__float_as_uint(gv) & 0xFFu)
                                             : exact_code_near_boundary(dv, sc, gv, rv, top);
          }
          pk[h] = c[0] | (c[1] << 8);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2 * K1_KG; ++h)
      *reinterpret_cast<uint16_t*>(dst + image_plane(2 * kg + h) * pstride) = static_cast<uint16_t>(pk[h]);
    // Row sums (lowpgemm.hpp:121-123): positions (2k, 2k+1) as 16-bit halves
    // (RS = false: the GEMM sums the A rows from its stages instead).
    if constexpr (RS) {
#pragma unroll
      for (int kk = 0; kk < K1_KG; ++kk) {
        const uint32_t a = __byte_perm(pk[2 * kk], pk[2 * kk + 1], 0x5410);  // [p.c0, p.c1, q.c0, q.c1]
        const uint32_t hi = __byte_perm(a, 0u, 0x4341);                      // [p.c1, 0, q.c1, 0]
        tot[kg + kk] = __reduce_add_sync(0xffffffffu, a - 255u * hi);       // [p sum | q sum]
      }
    }
  }
  if constexpr (RS) {
    // Lane l < 16 takes position l's sum: the 16-bit half l of the eight
    // warp-uniform totals, through 32 bytes of per-warp shared scratch.
    reinterpret_cast<uint4*>(s_rsw)[0] = make_uint4(tot[0], tot[1], tot[2], tot[3]);
    reinterpret_cast<uint4*>(s_rsw)[1] = make_uint4(tot[4], tot[5], tot[6], tot[7]);
    __syncwarp();
    if (lane < 16) {
      const uint32_t mine = reinterpret_cast<const uint16_t*>(s_rsw)[lane];
      int32_t* rs = rowsum + static_cast<long long>(lane) * g.rs_pitch + m;
      if (g.nchunks == 1)
        *rs = static_cast<int32_t>(mine);
      else  // channel chunks of one tile run in different warps (rowsum pre-zeroed)
        atomicAdd(rs, static_cast<int32_t>(mine));
    }
    __syncwarp();
  }
}

// One K1 strip (item) of the fast path: v recomputed, quantised, codes +
// row sums written.
template <int BK, int NK, bool RS, bool STATIC>
__device__ __forceinline__ void quant_fast_item(const float* __restrict__ x, uint8_t* __restrict__ codes,
                                                int32_t* __restrict__ rowsum, const InGeom& g,
                                                long long item, int lane, const float* s_tmin,
                                                const float* s_scale, const float* s_rcp, float top,
                                                uint32_t* s_rsw) {
  const StripItem it = strip_item(g, item, lane);
  const Strip<true> sp(x, g, it);
  const bool rows_in = sp.rows_ok();
  constexpr int kImg = kBM * BK;
  const int kc = it.ch / BK, cb = it.ch % BK;
  uint8_t* const cbase = codes + static_cast<long long>(kc) * kImg;
  float2 ta[4], tb[4], tc[4], td[4], pc[4], pd[4];
  int xx = 2 * it.tj0 - g.pad;
  sp.column(xx, ta);
  sp.column(xx + 1, tb);
  sp.load(xx + 2, pc);
  sp.load(xx + 3, pd);
  int m = (it.img * g.TH + it.ti) * g.TW + it.tj0;
  for (int tj = it.tj0; tj < it.tj1; ++tj, xx += 2, ++m) {
    colpass(pc, tc);
    colpass(pd, td);
    if (tj + 1 < it.tj1) {  // software prefetch of the next tile's two new columns
      if (K1_INTERIOR && !RS && rows_in && xx + 4 >= 0 && xx + 5 < g.W) {  // warp-uniform; measured -3 % (RS variant: +1.5 %, so off there)
        sp.load_in(xx + 4, pc);
        sp.load_in(xx + 5, pd);
      } else {
        sp.load(xx + 4, pc);
        sp.load(xx + 5, pd);
      }
    }
    quant_fast_tile<BK, NK, RS, STATIC>(ta, tb, tc, td, m, cbase, cb, rowsum, g, lane, s_tmin, s_scale, s_rcp, top,
                                        s_rsw);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      ta[a] = tc[a];
      tb[a] = td[a];
    }
  }
}


template <int BK, int NK, bool RS, bool STATIC = false>
__global__ void __launch_bounds__(LANCE_K1_THREADS, LANCE_K1_MINB) input_quant_fast_kernel(const float* __restrict__ x,
                                                                  uint8_t* __restrict__ codes,
                                                                  int32_t* __restrict__ rowsum,
                                                                  const LanceDevState* __restrict__ st,
                                                                  InGeom g) {
  pdl_entry();
  __shared__ float s_tmin[16], s_scale[16], s_rcp[16];
  __shared__ __align__(16) uint32_t s_rsw[K1_THREADS / 32][8];  // RS: per-warp row-sum scratch
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 16) {
    s_tmin[tid] = st->a_tmin[tid];
    s_scale[tid] = st->a_scale[tid];
    s_rcp[tid] = st->a_rcp[tid];
  }
  const float top = static_cast<float>((1 << st->bits_i) - 1);
  __syncthreads();
  // Reverse order: the range pass (K0) just streamed x front to back, so the
  // tail of x is still in L2 when this kernel starts; and the GEMM, which
  // reads the codes front to back, then finds the last-written rows in L2.
  const long long wi = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (tid >> 5);
  if (wi >= g.num_items) return;
  const long long item = g.rev_items ? g.num_items - 1 - wi : wi;
  quant_fast_item<BK, NK, RS, STATIC>(x, codes, rowsum, g, item, lane, s_tmin, s_scale, s_rcp, top,
                                      s_rsw[tid >> 5]);
}

// Static-params mode: caller-supplied input QuantParams[16].
__global__ void static_params_kernel(LanceDevState* st, StaticParams prm, int C) {
  pdl_entry();
  if (threadIdx.x < prm.np) {
    const int p = threadIdx.x;
    const float s = prm.scale[p];
    st->a_tmin[p] = prm.tmin[p];
    st->a_tmax[p] = prm.tmax[p];
    st->a_scale[p] = s;
    st->a_rcp[p] = (s == 0.0f) ? 0.0f : __frcp_rn(s);
    if (p == 0) st->nan_in = 0;
  }
  __syncthreads();
  make_epilogue_consts(st, C, prm.np);
}

// --------------------------------------------------------------------------
// K0 (C % 64 == 0), lean ring version.  A warp walks a strip (img, tile row
// ti, tiles tj0..tj1, 64 channels = 2 per lane).  Pair q = input columns
// xx0 + 2q, xx0 + 2q + 1 (tile t of the strip uses pairs t and t + 1); every
// pair is staged per lane with eight 8-byte cp.async (zero fill for rows /
// columns outside the image = extract_tiles' zero padding, tensor.hpp:141-147)
// into a ring of D + 1 slots, D pairs ahead of the tile being transformed.
// Addressing is four 64-bit row pointers bumped by 2C per pair, with the
// pair's second column at an immediate offset when C is a template constant
// (CC > 0): no per-copy multiplies.  A lane only reads back the slots it
// copied itself, so per-thread cp.async groups are the only ordering needed.
// Transform and range arithmetic as input_range_kernel.
// The K0 strip loop (ring below) over this block's grid-stride items, folding
// every v into lo / hi.  s_ring: [warps][D + 1 slots][8][32] float2.
template <int D, int CC>
__device__ __forceinline__ void range_ring_phase(const float* __restrict__ x, const InGeom& g,
                                                 float (&lo)[16], float (&hi)[16], float2* s_ring) {
  constexpr int R = D + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int C = CC > 0 ? CC : g.C;
  const int W = g.W;
  float2* const ring = s_ring + static_cast<size_t>(warp) * R * 8 * 32 + lane;
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long item = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + warp;
       item < g.num_items; item += stride) {
    const StripItem it = strip_item(g, item, lane);
    const int xx0 = 2 * it.tj0 - g.pad;
    const float* img = x + static_cast<long long>(it.img) * g.H * W * C + it.ch;
    const float* cp[4];
    uint32_t rsz[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int yy = 2 * it.ti - g.pad + a;
      const bool ok = (yy >= 0) && (yy < g.H);
      cp[a] = img + (static_cast<long long>(ok ? yy : 0) * W + xx0) * C;
      rsz[a] = ok ? 8u : 0u;
    }
    const int n = it.tj1 - it.tj0;  // tiles; pairs 0..n
    int c0 = xx0;                   // first column of the next pair to issue
    int q_issue = 0;
    float2* wslot = ring;
    auto issue = [&]() {
      if (q_issue <= n) {
        if (c0 >= 0 && c0 + 1 < W) {  // interior pair (warp-uniform)
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            cp_async8_sz(wslot + a * 32, cp[a], rsz[a]);
            cp_async8_sz(wslot + (4 + a) * 32, cp[a] + C, rsz[a]);
          }
        } else {
          const uint32_t m0 = (static_cast<unsigned>(c0) < static_cast<unsigned>(W)) ? ~0u : 0u;
          const uint32_t m1 = (static_cast<unsigned>(c0 + 1) < static_cast<unsigned>(W)) ? ~0u : 0u;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            cp_async8_sz(wslot + a * 32, cp[a], rsz[a] & m0);
            cp_async8_sz(wslot + (4 + a) * 32, cp[a] + C, rsz[a] & m1);
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) cp[a] += 2 * C;
        c0 += 2;
      }
      cp_async_commit();  // one group per pair, empty past the strip end
      ++q_issue;
      wslot += 8 * 32;
      if (wslot == ring + R * 8 * 32) wslot = ring;
    };
#pragma unroll
    for (int q = 0; q < R; ++q) issue();  // pairs 0..D
    float2 ta[4], tb[4];
    const float2* rslot = ring;
    {
      cp_async_wait<D>();  // pair 0
      float2 d0[4], d1[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        d0[a] = rslot[a * 32];
        d1[a] = rslot[(4 + a) * 32];
      }
      colpass(d0, ta);
      colpass(d1, tb);
      rslot += 8 * 32;
    }
    for (int t = 0; t < n; ++t) {
      cp_async_wait<D - 1>();  // pair t + 1
      float2 pc[4], pd[4], tc[4], td[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        pc[a] = rslot[a * 32];
        pd[a] = rslot[(4 + a) * 32];
      }
      rslot += 8 * 32;
      if (rslot == ring + R * 8 * 32) rslot = ring;
      issue();  // pair t + 1 + D into the slot of pair t (consumed last iteration)
      colpass(pc, tc);
      colpass(pd, td);
      float2 v[16];
      row_pass(ta, tb, tc, td, v);
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        lo[p] = fmin3_nan(lo[p], v[p].x, v[p].y);
        hi[p] = fmax3_nan(hi[p], v[p].x, v[p].y);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ta[a] = tc[a];
        tb[a] = td[a];
      }
    }
  }
  cp_async_wait<0>();
}

template <int D, int CC>
__global__ void __launch_bounds__(LANCE_K0_THREADS, LANCE_K0_MINB) input_range_ring_kernel(const float* __restrict__ x,
                                                                  float* __restrict__ partials,
                                                                  LanceDevState* __restrict__ st,
                                                                  InGeom g) {
  pdl_entry();
  grid_zero_i32(g.rs_zero, g.rs_zero_words);  // K1's atomic row sums (multi-chunk layers)
  extern __shared__ float2 s_ring[];  // [warps][R slots][2 columns x 4 rows][32 lanes]
  __shared__ float s_red[LANCE_K0_THREADS];
  float lo[16], hi[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  range_ring_phase<D, CC>(x, g, lo, hi, s_ring);
  if (block_minmax_and_ticket(lo, hi, partials, &st->ticket_in, s_red)) {
    fit_from_ranges(s_red, g.granularity, st->bits_i, st->a_tmin, st->a_tmax, st->a_scale,
                    st->a_rcp, &st->nan_in);
    __syncthreads();
    make_epilogue_consts(st, g.C);
  }
}

// --------------------------------------------------------------------------
// NCHW input (north-star layout option; the reference itself is NHWC-only,
// tensor.hpp:24-55): a shared-memory tiled transpose NCHW -> NHWC into the
// plan's staging buffer, then the NHWC K0 / K1 unchanged, so codes,
// parameters and y are bit-identical to the NHWC path by construction.
// (Measured: K0 / K1 variants that stage 64-channel input windows per CTA and
// transpose them in shared memory ran 4-7x slower than the NHWC kernels --
// one 59 KB window per CTA leaves too few CTAs in flight to cover the load
// latency -- while this transpose is a pure HBM stream.)
//
// CTA = one (image, input row y, 32-pixel run x0.., 64-channel chunk c0..):
// load 64 channel rows x 32 pixels (one 128-byte run per channel row: a
// thread loads one 16-byte float4, 8 threads per row) into s[c][x] (row
// stride 33: conflict-free), then write 32 pixels x 64 channels (16 lanes x
// float4 = 256 contiguous bytes per pixel).  Ragged W / C (W % 4 or C % 4 !=
// 0, unaligned pointers) take predicated scalar accesses.
__global__ void __launch_bounds__(256) nchw_to_nhwc_kernel(const float* __restrict__ x,
                                                           float* __restrict__ xt, int N, int C,
                                                           int H, int W) {
  pdl_entry();
  __shared__ float s[64][33];
  const int tid = threadIdx.x;
  const int xb = blockIdx.x;             // 32-pixel run
  const int y = blockIdx.y % H, img = blockIdx.y / H;
  const int c0 = blockIdx.z * 64;
  const int x0 = xb * 32;
  const long long HW = static_cast<long long>(H) * W;
  const bool vec_in = ((W & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  {
    const int q = tid & 7;  // float4 quad within the 32-pixel run
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int cl = (tid >> 3) + 32 * k, c = c0 + cl;
      const int xx = x0 + 4 * q;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (c < C) {
        const float* src = x + (static_cast<long long>(img) * C + c) * HW + static_cast<long long>(y) * W;
        if (vec_in && xx + 3 < W) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(src + xx));
          v[0] = f.x, v[1] = f.y, v[2] = f.z, v[3] = f.w;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (xx + j < W) v[j] = __ldg(src + xx + j);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) s[cl][4 * q + j] = v[j];
    }
  }
  __syncthreads();
  const bool vec_out = ((C & 3) == 0) && ((reinterpret_cast<uintptr_t>(xt) & 15) == 0);
  const int cq = tid & 15;  // channel quad
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int xl = (tid >> 4) + 16 * k, xx = x0 + xl;
    const int c = c0 + 4 * cq;
    if (xx >= W || c >= C) continue;
    float* dst = xt + ((static_cast<long long>(img) * H + y) * W + xx) * C + c;
    const float4 f = make_float4(s[4 * cq][xl], s[4 * cq + 1][xl], s[4 * cq + 2][xl], s[4 * cq + 3][xl]);
    if (vec_out && c + 3 < C) {
      *reinterpret_cast<float4*>(dst) = f;
    } else {
      const float e[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c + j < C) dst[j] = e[j];
    }
  }
}

// --------------------------------------------------------------------------
// Small-C path (C < 32, e.g. the RGB first layer of VGG, C = 3): the strip
// kernels put channels on lanes, which would leave most lanes idle; here one
// thread owns one (tile, channel) and walks a grid-stride loop.  Same
// arithmetic as input_transform2 / the quantisers above, scalar.
__device__ __forceinline__ void smallc_tile(const float* __restrict__ x, const InGeom& g,
                                            long long i, float (&v)[16], long long& tile, int& c) {
  tile = i / g.C;
  c = static_cast<int>(i - tile * g.C);
  const int img = static_cast<int>(tile / g.P), t = static_cast<int>(tile - static_cast<long long>(img) * g.P);
  const int ti = t / g.TW, tj = t - ti * g.TW;
  const int y0 = 2 * ti - g.pad, x0 = 2 * tj - g.pad;
  const float* base = x + static_cast<long long>(img) * g.H * g.W * g.C + c;
  float d[16];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int yy = y0 + a, xx = x0 + b;
      d[a * 4 + b] = (yy >= 0 && yy < g.H && xx >= 0 && xx < g.W)
                         ? __ldg(base + (static_cast<long long>(yy) * g.W + xx) * g.C)
                         : 0.0f;
    }
  float t4[16];  // column pass first (B^T d), then rows
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    t4[0 * 4 + b] = __fsub_rn(d[0 * 4 + b], d[2 * 4 + b]);
    t4[1 * 4 + b] = __fadd_rn(d[1 * 4 + b], d[2 * 4 + b]);
    t4[2 * 4 + b] = __fsub_rn(d[2 * 4 + b], d[1 * 4 + b]);
    t4[3 * 4 + b] = __fsub_rn(d[1 * 4 + b], d[3 * 4 + b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    v[a * 4 + 0] = __fsub_rn(t4[a * 4 + 0], t4[a * 4 + 2]);
    v[a * 4 + 1] = __fadd_rn(t4[a * 4 + 1], t4[a * 4 + 2]);
    v[a * 4 + 2] = __fsub_rn(t4[a * 4 + 2], t4[a * 4 + 1]);
    v[a * 4 + 3] = __fsub_rn(t4[a * 4 + 1], t4[a * 4 + 3]);
  }
}

__global__ void __launch_bounds__(256) input_range_smallc_kernel(const float* __restrict__ x,
                                                                 float* __restrict__ partials,
                                                                 LanceDevState* __restrict__ st,
                                                                 InGeom g) {
  pdl_entry();
  grid_zero_i32(g.rs_zero, g.rs_zero_words);  // K1's atomic row sums (multi-chunk layers)
  __shared__ float s_red[256];
  float lo[16], hi[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const long long total = static_cast<long long>(g.M) * g.C;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float v[16];
    long long tile;
    int c;
    smallc_tile(x, g, i, v, tile, c);
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      lo[p] = fmin_nan(lo[p], v[p]);
      hi[p] = fmax_nan(hi[p], v[p]);
    }
  }
  if (block_minmax_and_ticket(lo, hi, partials, &st->ticket_in, s_red)) {
    fit_from_ranges(s_red, g.granularity, st->bits_i, st->a_tmin, st->a_tmax, st->a_scale,
                    st->a_rcp, &st->nan_in);
    __syncthreads();
    make_epilogue_consts(st, g.C);
  }
}

template <bool STATIC>
__global__ void __launch_bounds__(256) input_quant_smallc_kernel(const float* __restrict__ x,
                                                                 uint8_t* __restrict__ codes,
                                                                 int32_t* __restrict__ rowsum,
                                                                 const LanceDevState* __restrict__ st,
                                                                 InGeom g) {
  pdl_entry();
  __shared__ float s_tmin[16], s_scale[16], s_rcp[16];
  if (threadIdx.x < 16) {
    s_tmin[threadIdx.x] = st->a_tmin[threadIdx.x];
    s_scale[threadIdx.x] = st->a_scale[threadIdx.x];
    s_rcp[threadIdx.x] = st->a_rcp[threadIdx.x];
  }
  __syncthreads();
  const float top = static_cast<float>((1 << st->bits_i) - 1);
  const long long total = static_cast<long long>(g.M) * g.C;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float v[16];
    long long tile;
    int c;
    smallc_tile(x, g, i, v, tile, c);
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      uint32_t code;
      if (STATIC) {
        code = quantize_code(v[p], s_tmin[p], s_scale[p], top);
      } else {
        const float dd = __fsub_rn(v[p], s_tmin[p]);
        const float gq = __fmaf_rn(dd, s_rcp[p], kMagic);
        const float rr = __fmaf_rn(dd, s_rcp[p], __fsub_rn(kMagic, gq));
        code = (fabsf(rr) < kTieGuard) ? (__float_as_uint(gq) & 0xFFu)
                                       : exact_code_near_boundary(dd, s_scale[p], gq, rr, top);
      }
      codes[umma_image_offset(tile, c, p, kBM, g.a_bk, g.a_nk)] = static_cast<uint8_t>(code);
      if (g.rowsums) atomicAdd(rowsum + static_cast<long long>(p) * g.rs_pitch + tile, static_cast<int>(code));
    }
  }
}

// --------------------------------------------------------------------------
int input_range_grid(const InGeom& g, int sm_count) {
  if (g.C >= 32 && g.C % 64 == 0) {  // ring kernel: K0_MINB resident K0_THREADS-thread blocks per SM
    constexpr int wpb = LANCE_K0_THREADS / 32;
    const long long blocks = (g.num_items + wpb - 1) / wpb;
    const long long cap = static_cast<long long>(LANCE_K0_MINB) * sm_count;
    return static_cast<int>(blocks < cap ? blocks : cap);
  }
  const long long blocks = (g.num_items + 7) / 8;
  const long long cap = 2LL * sm_count;  // 2 resident 256-thread blocks per SM
  return static_cast<int>(blocks < cap ? blocks : cap);
}

cudaError_t launch_input_range(const float* x, float* partials, int grid, LanceDevState* st,
                               const InGeom& g, int vec2, cudaStream_t s) {
  // K0 input staging: cp.async ring of 4 tiles per warp (measured: 7-8 % faster
  // than register lookahead on the 56x56 / 28x28 layers; 8 halves residency).
  constexpr int kDepth = LANCE_K0_DEPTH;
  if (g.C < 32) {
    LANCE_LAUNCH_CHECK(launch_k(input_range_smallc_kernel, grid, 256, 0, s, x, partials, st, g));
  } else if (g.C % 64 == 0) {
    const size_t smem = static_cast<size_t>(LANCE_K0_THREADS / 32) * (kDepth + 1) * 8 * 32 * sizeof(float2);
#define LANCE_K0_RING(CCV)                                                                        \
    if (CCV == 0 || g.C == CCV) {                                                                \
      const cudaError_t attr =                                                                   \
          ensure_smem_attr(reinterpret_cast<const void*>(input_range_ring_kernel<kDepth, CCV>), smem); \
      if (attr != cudaSuccess) return attr;                                                      \
      LANCE_LAUNCH_CHECK(launch_k(input_range_ring_kernel<kDepth, CCV>, grid, LANCE_K0_THREADS, smem, s, x, partials, st, g));          \
      return cudaGetLastError();                                                                 \
    }
    LANCE_K0_RING(64)
    LANCE_K0_RING(128)
    LANCE_K0_RING(256)
    LANCE_K0_RING(512)
    LANCE_K0_RING(0)
#undef LANCE_K0_RING
  } else if (vec2) {
    LANCE_LAUNCH_CHECK(launch_k(input_range_kernel<true>, grid, 256, 0, s, x, partials, st, g));
  } else {
    LANCE_LAUNCH_CHECK(launch_k(input_range_kernel<false>, grid, 256, 0, s, x, partials, st, g));
  }
  return cudaGetLastError();
}

cudaError_t launch_input_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                               const LanceDevState* st, const InGeom& g, int vec2,
                               int static_mode, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((g.num_items + 7) / 8);
  if (g.C < 32) {
    const long long total = static_cast<long long>(g.M) * g.C;
    const unsigned sgrid = static_cast<unsigned>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    if (g.rowsums) {  // atomically accumulated here (normally the GEMM sums the rows at BK = 32)
      cudaError_t e = cudaMemsetAsync(rowsum, 0, sizeof(int32_t) * 16 * static_cast<size_t>(g.rs_pitch), s);
      if (e != cudaSuccess) return e;
    }
    if (static_mode)
      LANCE_LAUNCH_CHECK(launch_k(input_quant_smallc_kernel<true>, sgrid, 256, 0, s, x, codes, rowsum, st, g));
    else
      LANCE_LAUNCH_CHECK(launch_k(input_quant_smallc_kernel<false>, sgrid, 256, 0, s, x, codes, rowsum, st, g));
    return cudaGetLastError();
  }
  if (g.C % 64 == 0) {  // fast path: every lane owns two real channels
    const unsigned grid = static_cast<unsigned>((g.num_items + K1_THREADS / 32 - 1) / (K1_THREADS / 32));
#define LANCE_K1_FAST(BKV, NKV)                                                             \
  if (g.a_bk == BKV && g.a_nk == NKV) {                                                  \
    if (static_mode && g.rowsums)                                                        \
      LANCE_LAUNCH_CHECK(launch_k(input_quant_fast_kernel<BKV, NKV, true, true>, grid, K1_THREADS, 0, s, x, codes, rowsum, st, g)); \
    else if (static_mode)                                                                \
      LANCE_LAUNCH_CHECK(launch_k(input_quant_fast_kernel<BKV, NKV, false, true>, grid, K1_THREADS, 0, s, x, codes, rowsum, st, g)); \
    else if (g.rowsums)                                                                  \
      LANCE_LAUNCH_CHECK(launch_k(input_quant_fast_kernel<BKV, NKV, true>, grid, K1_THREADS, 0, s, x, codes, rowsum, st, g)); \
    else                                                                                 \
      LANCE_LAUNCH_CHECK(launch_k(input_quant_fast_kernel<BKV, NKV, false>, grid, K1_THREADS, 0, s, x, codes, rowsum, st, g)); \
    return cudaGetLastError();                                                           \
  }
    LANCE_K1_FAST(64, 1)
    LANCE_K1_FAST(128, 1)
    LANCE_K1_FAST(128, 2)
    LANCE_K1_FAST(128, 3)
    LANCE_K1_FAST(128, 4)
    LANCE_K1_FAST(64, 3)
    LANCE_K1_FAST(64, 5)
#undef LANCE_K1_FAST
  }
  if (vec2) {
    if (static_mode)
      LANCE_LAUNCH_CHECK(launch_k(input_quant_kernel<true, true>, grid, 256, 0, s, x, codes, rowsum, st, g));
    else
      LANCE_LAUNCH_CHECK(launch_k(input_quant_kernel<true, false>, grid, 256, 0, s, x, codes, rowsum, st, g));
  } else {
    if (static_mode)
      LANCE_LAUNCH_CHECK(launch_k(input_quant_kernel<false, true>, grid, 256, 0, s, x, codes, rowsum, st, g));
    else
      LANCE_LAUNCH_CHECK(launch_k(input_quant_kernel<false, false>, grid, 256, 0, s, x, codes, rowsum, st, g));
  }
  return cudaGetLastError();
}

// NCHW -> NHWC staging transpose (x [N][C][H][W] -> xt [N][H][W][C]).
cudaError_t launch_nchw_to_nhwc(const float* x, float* xt, int N, int C, int H, int W, cudaStream_t s) {
  const dim3 grid((W + 31) / 32, static_cast<unsigned>(N) * H, (C + 63) / 64);
  LANCE_LAUNCH_CHECK(launch_k(nchw_to_nhwc_kernel, grid, 256, 0, s, x, xt, N, C, H, W));
  return cudaSuccess;
}

// Global-fit mode (SURVEY 8(e) mode 2) on the device.  Export: the fitted
// per-position ranges of the last range pass as [-t_min[0..np), t_max[0..np),
// nan] -- the layout one element-wise MAX all-reduce combines across ranks
// (-(-x) is exact; a NaN flag rides along as 1.0 because fmax drops NaNs).
__global__ void export_minmax_kernel(const LanceDevState* st, float* minmax, int np) {
  pdl_entry();
  const int p = threadIdx.x;
  if (p < np) {
    minmax[p] = -st->a_tmin[p];
    minmax[np + p] = st->a_tmax[p];
  }
  if (p == 0) minmax[2 * np] = st->nan_in ? 1.0f : 0.0f;
}

// Import: fit_params (quant.hpp:54-72) on the reduced ranges -> the input
// QuantParams and affine constants of the plan (PerTensor folds, engines.hpp:151-156).
__global__ void fit_minmax_kernel(LanceDevState* st, const float* __restrict__ minmax, int np,
                                  int gran, int C) {
  pdl_entry();
  const int p = threadIdx.x;
  bool bad = false;
  if (p < np) {
    float lo = -minmax[p], hi = minmax[np + p];
    if (gran == 2) {
      lo = -minmax[0];
      hi = minmax[np];
      for (int q = 1; q < np; ++q) {
        lo = fmin_nan(lo, -minmax[q]);
        hi = fmax_nan(hi, minmax[np + q]);
      }
    }
    lo = __fadd_rn(lo, 0.0f);  // the reference never produces -0 (matrix.hpp:77-83)
    hi = __fadd_rn(hi, 0.0f);
    bad = isnan(lo) || isnan(hi) || isinf(lo) || isinf(hi);
    const float s = __fdiv_rn(__fsub_rn(hi, lo), static_cast<float>((1 << st->bits_i) - 1));
    st->a_tmin[p] = lo;
    st->a_tmax[p] = hi;
    st->a_scale[p] = s;
    st->a_rcp[p] = (s == 0.0f) ? 0.0f : __frcp_rn(s);
  }
  const int any = __syncthreads_or(bad ? 1 : 0);
  if (p == 0) st->nan_in = (any || minmax[2 * np] != 0.0f) ? 1 : 0;
  __syncthreads();
  make_epilogue_consts(st, C, np);
}

cudaError_t launch_export_minmax(const LanceDevState* st, float* minmax, int np, cudaStream_t s) {
  LANCE_LAUNCH_CHECK(launch_k(export_minmax_kernel, 1, 64, 0, s, st, minmax, np));
  return cudaGetLastError();
}

cudaError_t launch_fit_minmax(LanceDevState* st, const float* minmax, int np, int gran, int C,
                              cudaStream_t s) {
  LANCE_LAUNCH_CHECK(launch_k(fit_minmax_kernel, 1, 64, 0, s, st, minmax, np, gran, C));
  return cudaGetLastError();
}

cudaError_t launch_static_params(LanceDevState* st, const StaticParams& prm, int C,
                                 cudaStream_t s) {
  LANCE_LAUNCH_CHECK(launch_k(static_params_kernel, 1, 64, 0, s, st, prm, C));
  return cudaGetLastError();
}

}  // namespace lance_dev
