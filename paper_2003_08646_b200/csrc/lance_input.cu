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
// Mapping: one warp = one Winograd tile x 64 channels (2 per lane, float2
// NHWC loads: 256 contiguous bytes per pixel per warp); the tile gather is
// extract_tiles (tensor.hpp:116-152): origin (2ti - pad, 2tj - pad), zero pad.
// Transforms run on packed f32x2 (FADD2), ranges on 3-input FMNMX3.NAN.
#include <cuda_runtime.h>

#include <cstdint>

#include "lance_common.cuh"

namespace lance_dev {

struct TileOrigin {
  int img, y0, x0;
};

__device__ __forceinline__ TileOrigin tile_origin(const InGeom& g, int m) {
  const int img = m / g.P;
  const int t = m - img * g.P;
  const int ti = t / g.TW, tj = t - ti * g.TW;
  return {img, 2 * ti - g.pad, 2 * tj - g.pad};
}

// 16 pixels x channels (ch, ch + 1) of one tile; zero outside the image and
// for channels >= C.
template <bool VEC2>
__device__ __forceinline__ void load_tile2(const float* __restrict__ x, const InGeom& g,
                                           const TileOrigin& o, int ch, float2 (&d)[16]) {
  const float* base = x + static_cast<long long>(o.img) * g.H * g.W * g.C;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int yy = o.y0 + a;
    const bool rok = (yy >= 0) && (yy < g.H);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int xx = o.x0 + b;
      const bool ok = rok && (xx >= 0) && (xx < g.W);
      const float* px = base + (static_cast<long long>(yy) * g.W + xx) * g.C + ch;
      if (VEC2) {
        d[a * 4 + b] = (ok && ch < g.C) ? __ldg(reinterpret_cast<const float2*>(px))
                                        : make_float2(0.f, 0.f);
      } else {
        d[a * 4 + b].x = (ok && ch < g.C) ? __ldg(px) : 0.f;
        d[a * 4 + b].y = (ok && ch + 1 < g.C) ? __ldg(px + 1) : 0.f;
      }
    }
  }
}

// --------------------------------------------------------------------------
// K0: per-position range of v over the whole batch (grid-stride over
// (tile, 64-channel chunk) warp items).
template <bool VEC2>
__global__ void __launch_bounds__(256, 2) input_range_kernel(const float* __restrict__ x,
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
  const int lane = threadIdx.x & 31;
  const long long nitems = static_cast<long long>(g.M) * g.nchunks;
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long item = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       item < nitems; item += stride) {
    const int m = static_cast<int>(item / g.nchunks);
    const int ch = static_cast<int>(item - static_cast<long long>(m) * g.nchunks) * kChunk + 2 * lane;
    const TileOrigin o = tile_origin(g, m);
    float2 d[16], v[16];
    load_tile2<VEC2>(x, g, o, ch, d);
    input_transform2(d, v);
    if (ch + 1 < g.C) {
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        lo[p] = fmin3_nan(lo[p], v[p].x, v[p].y);
        hi[p] = fmax3_nan(hi[p], v[p].x, v[p].y);
      }
    } else if (ch < g.C) {  // odd C: last lane holds one real channel
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        lo[p] = fmin_nan(lo[p], v[p].x);
        hi[p] = fmax_nan(hi[p], v[p].x);
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

// --------------------------------------------------------------------------
// K1: codes + row sums.  Block = kTM tiles (one per warp); channels in chunks
// of 64; codes staged in shared memory and written with 16-byte stores.
template <bool VEC2, bool STATIC>
__global__ void __launch_bounds__(256, 2) input_quant_kernel(const float* __restrict__ x,
                                                             uint8_t* __restrict__ codes,
                                                             int32_t* __restrict__ rowsum,
                                                             const LanceDevState* __restrict__ st,
                                                             InGeom g) {
  __shared__ __align__(16) uint8_t s_codes[16][kTM][kChunk];
  __shared__ int s_rs[16][kTM];
  __shared__ float s_tmin[16], s_scale[16], s_rcp[16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 16) {
    s_tmin[tid] = st->a_tmin[tid];
    s_scale[tid] = st->a_scale[tid];
    s_rcp[tid] = st->a_rcp[tid];
  }
  if (tid < 16 * kTM) s_rs[tid / kTM][tid % kTM] = 0;
  const float top = static_cast<float>((1 << st->bits_i) - 1);
  __syncthreads();

  const int m0 = blockIdx.x * kTM;
  const int m = m0 + warp;
  const bool valid = m < g.M;
  const TileOrigin o = tile_origin(g, valid ? m : 0);

  for (int c0 = 0; c0 < g.C_pad; c0 += kChunk) {
    const int ch = c0 + 2 * lane;
    uint32_t pk[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) pk[p] = 0u;
    if (valid && ch < g.C) {
      float2 d[16], v[16];
      load_tile2<VEC2>(x, g, o, ch, d);
      input_transform2(d, v);
      float rmax = 0.0f;
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        float2 q = mul2(sub2(v[p], bcast2(s_tmin[p])), bcast2(s_rcp[p]));
        if (STATIC) {  // caller-supplied params: q may be anywhere (NaN -> 0)
          q.x = fminf(fmaxf(q.x, 0.0f), top);
          q.y = fminf(fmaxf(q.y, 0.0f), top);
        }
        const float2 gq = add2(q, bcast2(kMagic));
        const float2 r = sub2(q, sub2(gq, bcast2(kMagic)));
        rmax = fmax3_nan(rmax, fabsf(r.x), fabsf(r.y));
        pk[p] = __byte_perm(__float_as_uint(gq.x), __float_as_uint(gq.y), 0x0040) & 0xFFFFu;
      }
      if (!(rmax < kTieGuard)) {
        // Rare: some q0 lies within 2^-14 of a rounding boundary (or is NaN):
        // reload the tile and re-quantise exactly those values with the IEEE
        // reference formula (keeps v out of registers on the fast path).
        float2 d2[16], w2[16];
        load_tile2<VEC2>(x, g, o, ch, d2);
        input_transform2(d2, w2);
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const float2 q0 = mul2(sub2(w2[p], bcast2(s_tmin[p])), bcast2(s_rcp[p]));
          float qa = q0.x, qb = q0.y;
          if (STATIC) {
            qa = fminf(fmaxf(qa, 0.0f), top);
            qb = fminf(fmaxf(qb, 0.0f), top);
          }
          const float ra = __fsub_rn(qa, __fsub_rn(__fadd_rn(qa, kMagic), kMagic));
          const float rb = __fsub_rn(qb, __fsub_rn(__fadd_rn(qb, kMagic), kMagic));
          if (!(fabsf(ra) < kTieGuard))
            pk[p] = (pk[p] & 0xFF00u) | quantize_code(w2[p].x, s_tmin[p], s_scale[p], top);
          if (!(fabsf(rb) < kTieGuard))
            pk[p] = (pk[p] & 0x00FFu) | (quantize_code(w2[p].y, s_tmin[p], s_scale[p], top) << 8);
        }
      }
      if (ch + 1 >= g.C) {  // odd C: zero the padding channel's code
#pragma unroll
        for (int p = 0; p < 16; ++p) pk[p] &= 0x00FFu;
      }
    }
#pragma unroll
    for (int p = 0; p < 16; ++p)
      *reinterpret_cast<uint16_t*>(&s_codes[p][warp][2 * lane]) = static_cast<uint16_t>(pk[p]);
    __syncthreads();
    // Write-out: 16 positions x kTM tiles x 4 pieces of 16 codes.
#pragma unroll
    for (int k = 0; k < (16 * kTM * 4) / 256; ++k) {
      const int i = tid + 256 * k;
      const int p = i / (kTM * 4), t = (i / 4) % kTM, part = i % 4;
      const uint4 val = *reinterpret_cast<const uint4*>(&s_codes[p][t][part * 16]);
      uint32_t sum = __dp4a(val.x, 0x01010101u, 0u);
      sum = __dp4a(val.y, 0x01010101u, sum);
      sum = __dp4a(val.z, 0x01010101u, sum);
      sum = __dp4a(val.w, 0x01010101u, sum);
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      const int mt = m0 + t;
      if (mt < g.M && c0 + part * 16 < g.C_pad)
        *reinterpret_cast<uint4*>(codes + (static_cast<long long>(p) * g.M + mt) * g.C_pad + c0 +
                                  part * 16) = val;
      if (part == 0) s_rs[p][t] += static_cast<int>(sum);
    }
    __syncthreads();
  }
  if (tid < 16 * kTM) {
    const int p = tid / kTM, t = tid % kTM;
    if (m0 + t < g.M) rowsum[static_cast<long long>(p) * g.M + m0 + t] = s_rs[p][t];
  }
}

// Static-params mode: caller-supplied input QuantParams[16].
__global__ void static_params_kernel(LanceDevState* st, StaticParams prm, int C) {
  if (threadIdx.x < 16) {
    const int p = threadIdx.x;
    const float s = prm.scale[p];
    st->a_tmin[p] = prm.tmin[p];
    st->a_tmax[p] = prm.tmax[p];
    st->a_scale[p] = s;
    st->a_rcp[p] = (s == 0.0f) ? 0.0f : __frcp_rn(s);
    if (p == 0) st->nan_in = 0;
  }
  __syncwarp();
  make_epilogue_consts(st, C);
}

// --------------------------------------------------------------------------
int input_range_grid(const InGeom& g, int sm_count) {
  const long long warps = static_cast<long long>(g.M) * g.nchunks;
  const long long blocks = (warps + 7) / 8;
  const long long cap = 3LL * sm_count;  // 3 resident 256-thread blocks per SM
  return static_cast<int>(blocks < cap ? blocks : cap);
}

cudaError_t launch_input_range(const float* x, float* partials, int grid, LanceDevState* st,
                               const InGeom& g, int vec2, cudaStream_t s) {
  if (vec2)
    input_range_kernel<true><<<grid, 256, 0, s>>>(x, partials, st, g);
  else
    input_range_kernel<false><<<grid, 256, 0, s>>>(x, partials, st, g);
  return cudaGetLastError();
}

cudaError_t launch_input_quant(const float* x, uint8_t* codes, int32_t* rowsum,
                               const LanceDevState* st, const InGeom& g, int vec2,
                               int static_mode, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((g.M + kTM - 1) / kTM);
  if (vec2) {
    if (static_mode)
      input_quant_kernel<true, true><<<grid, 256, 0, s>>>(x, codes, rowsum, st, g);
    else
      input_quant_kernel<true, false><<<grid, 256, 0, s>>>(x, codes, rowsum, st, g);
  } else {
    if (static_mode)
      input_quant_kernel<false, true><<<grid, 256, 0, s>>>(x, codes, rowsum, st, g);
    else
      input_quant_kernel<false, false><<<grid, 256, 0, s>>>(x, codes, rowsum, st, g);
  }
  return cudaGetLastError();
}

cudaError_t launch_static_params(LanceDevState* st, const StaticParams& prm, int C,
                                 cudaStream_t s) {
  static_params_kernel<<<1, 32, 0, s>>>(st, prm, C);
  return cudaGetLastError();
}

}  // namespace lance_dev
