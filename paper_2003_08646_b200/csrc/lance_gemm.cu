// lance_gemm.cu -- K3/K4: the 16 per-position u8 x u8 -> s32 GEMMs of
// lance_gemm (gemm_codes x 16, lowpgemm.hpp:76-100, engines.hpp:510-525) on
// tcgen05 kind::i8 with TMA-fed operands and accumulators in TMEM, fused with
// the affine de-quantisation (affine_term, lowpgemm.hpp:110-114), the output
// transform A^T m A (winograd.hpp:80-84) and the merge with ragged-edge
// discard (tensor.hpp:157-182).
//
// Persistent kernel, one CTA per SM.  A tile = 128 Winograd tiles (UMMA M)
// x 16 filters (UMMA N) x all 16 positions = 16 x 16 s32 = 256 TMEM columns;
// TMEM holds two such accumulators, so the MMA of tile i+1 overlaps the
// epilogue of tile i, and the TMA producer runs ahead through an SMEM ring.
//   warp 0       TMA producer (one lane): per stage the A box
//                [128 rows x BK ch] and B box [16 filters x BK ch] of one
//                position
//   warp 1       TMEM allocator + UMMA issuer (one lane)
//   warps 2..9   epilogue: TMEM -> registers -> affine -> A^T m A -> y; warp
//                w drains TMEM lane quadrant w % 4, filters 8*((w-2)/4)..+8
// Tiles are assigned round-robin with the filter tile fastest, so the
// kBN-wide filter tiles of one row tile run concurrently on neighbouring SMs
// and share the A operand through L2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lance_common.cuh"

namespace lance_dev {

constexpr int kEpiWarps = 8;
constexpr int kGemmThreadsP = 64 + 32 * kEpiWarps;  // 320

template <int BK>
struct GemmCfg {
  static constexpr uint32_t kABytes = kBM * BK;
  static constexpr uint32_t kBBytes = kBN * BK;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr int kStagesRaw = (144 * 1024) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 16 ? 16 : kStagesRaw;
  static constexpr uint32_t kLayout = (BK == 128) ? 2u : (BK == 64 ? 4u : 6u);  // SW128/64/32
  static constexpr uint32_t kAccCols = 16 * kBN;                                // 256
  // + 16 * K_pad floats of per-filter constants, added at launch.
  static constexpr size_t kSmemBase = 1024 + static_cast<size_t>(kStages) * kStageBytes +
                                      (2 * kStages + 4) * 8 + 16;
};

constexpr size_t kSmemLimit = 227 * 1024 - 1024;  // leave room for static smem

// SMALL: C * top_a * top_b < 2^23, so every accumulator is below 2^23 and
// k1 * float(dot) is formed exactly by one FFMA (see below).
// EPI: fused bias + ReLU (north-star extension).
template <int BK, bool SMALL, bool EPI>
__global__ void __launch_bounds__(kGemmThreadsP, 1)
    gemm_epilogue_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB,
                         const int32_t* __restrict__ rowsum, const int32_t* __restrict__ colsum,
                         const LanceDevState* __restrict__ st, float* __restrict__ y,
                         int32_t* __restrict__ acc_dump, const float* __restrict__ bias,
                         int relu, GemmGeom g) {
  using Cfg = GemmCfg<BK>;
  constexpr int kStages = Cfg::kStages;
  constexpr uint32_t kIdesc = umma_idesc_u8(kBM, kBN);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ float s_k1[16], s_nk1m[16], s_k2[16], s_k4[16];

  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* stage_base = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* acc_full = empty_bar + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;        // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* s_cterm = reinterpret_cast<float*>(tmem_holder + 4);  // [16][K_pad]: k3[p]*colsum[p][k]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = g.num_n_tiles;
  const int K_pad = nt * kBN;
  const int num_tiles = ((g.M + kBM - 1) / kBM) * nt;
  const int num_iters = g.num_kchunks * 16;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp >= 2) {
    // Per-filter third term of affine_term for all filters of the layer.
    for (int i = threadIdx.x - 64; i < 16 * K_pad; i += 32 * kEpiWarps) {
      const int p = i / K_pad, kf = i - p * K_pad;
      const float cs = (kf < g.K) ? static_cast<float>(colsum[i]) : 0.0f;
      s_cterm[i] = __fmul_rn(st->k3[p], cs);
    }
    const int e = threadIdx.x - 64;
    if (e < 16) {
      const float k1 = st->k1[e];
      s_k1[e] = k1;
      s_nk1m[e] = __fmul_rn(k1, -8388608.0f);  // -k1 * 2^23, exact
      s_k2[e] = st->k2[e];
      s_k4[e] = st->k4[e];
    }
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / nt) * kBM, n0 = (tile % nt) * kBN;
        for (int it = 0; it < num_iters; ++it) {
          const int kc = it >> 4, p = it & 15;
          mbar_wait(&empty_bar[s], ph ^ 1u);
          uint8_t* sa = stage_base + s * Cfg::kStageBytes;
          mbar_arrive_expect_tx(&full_bar[s], Cfg::kStageBytes);
          tma_load_3d(sa, &tmA, kc * BK, m0, p, &full_bar[s]);
          tma_load_3d(sa + Cfg::kABytes, &tmB, kc * BK, n0, p, &full_bar[s]);
          if (++s == kStages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- TMEM + UMMA issuer ----------------
    tmem_alloc(tmem_holder, 2 * Cfg::kAccCols);
    tmem_relinquish();
    tc_fence_before();
    named_bar_sync(1, 32 + 32 * kEpiWarps);
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int buf = 0;
      uint32_t acc_ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&acc_empty[buf], acc_ph ^ 1u);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t d_base = tmem_base + static_cast<uint32_t>(buf) * Cfg::kAccCols;
        for (int it = 0; it < num_iters; ++it) {
          const int kc = it >> 4, p = it & 15;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(stage_base + s * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk) {
            const uint64_t adesc = umma_smem_desc(sa + kk * 32, 8 * BK, Cfg::kLayout);
            const uint64_t bdesc = umma_smem_desc(sb + kk * 32, 8 * BK, Cfg::kLayout);
            umma_i8(d_base + static_cast<uint32_t>(p * kBN), adesc, bdesc, kIdesc,
                    (kc > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[s]);
          if (++s == kStages) {
            s = 0;
            ph ^= 1u;
          }
        }
        umma_commit(&acc_full[buf]);
        if (++buf == 2) {
          buf = 0;
          acc_ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue ----------------
    const int ew = warp - 2;
    const int q = warp & 3;          // TMEM lane quadrant this warp may access
    const int f0 = (ew >> 2) * 8;    // this warp's 8 filters within the 16-filter tile
    named_bar_sync(1, 32 + 32 * kEpiWarps);
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const bool vec_ok = (g.K & 1) == 0;
    int buf = 0;
    uint32_t acc_ph = 0;
    // Row sums of the first tile (later tiles are prefetched one tile ahead).
    int32_t rs_next[16];
    {
      const int m = (blockIdx.x / nt) * kBM + q * 32 + lane;
#pragma unroll
      for (int p = 0; p < 16; ++p)
        rs_next[p] = (blockIdx.x < num_tiles && m < g.M)
                         ? __ldg(rowsum + static_cast<long long>(p) * g.M + m) : 0;
    }
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile / nt) * kBM, n0 = (tile % nt) * kBN;
      const int m = m0 + q * 32 + lane;
      const bool row_ok = m < g.M;
      float rterm[16];  // k2[p] * float(sum_a): second term of affine_term
#pragma unroll
      for (int p = 0; p < 16; ++p) rterm[p] = __fmul_rn(s_k2[p], static_cast<float>(rs_next[p]));
      {
        const int nxt = tile + gridDim.x;
        const int mn = (nxt / nt) * kBM + q * 32 + lane;
#pragma unroll
        for (int p = 0; p < 16; ++p)
          rs_next[p] = (nxt < num_tiles && mn < g.M)
                           ? __ldg(rowsum + static_cast<long long>(p) * g.M + mn) : 0;
      }
      // Output pixels of this tile: (2ti + a, 2tj + b); merge_tiles discards
      // the ceil-overhang (tensor.hpp:172-175).
      float* dst[4];
      bool ok[4];
      {
        const int mm = row_ok ? m : 0;
        const int img = mm / g.P;
        const int t = mm - img * g.P;
        const int ti = t / g.TW, tj = t - ti * g.TW;
#pragma unroll
        for (int ab = 0; ab < 4; ++ab) {
          const int oy = 2 * ti + (ab >> 1), ox = 2 * tj + (ab & 1);
          ok[ab] = row_ok && oy < g.OH && ox < g.OW;
          dst[ab] = y + ((static_cast<long long>(img) * g.OH + oy) * g.OW + ox) * g.K + n0 + f0;
        }
      }
      mbar_wait(&acc_full[buf], acc_ph);
      tc_fence_after();
      const uint32_t acc_addr = lane_base + static_cast<uint32_t>(buf) * Cfg::kAccCols + f0;
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {  // filter pairs of this warp's 8 filters
        uint32_t a[16][2];
#pragma unroll
        for (int p = 0; p < 16; ++p) tmem_ld_x2(acc_addr + p * kBN + j * 2, a[p]);
        tmem_ld_wait();
        if (j == 3) {
          // All of this warp's accumulators are in registers: hand the TMEM
          // buffer back to the MMA warp early.
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
        const int kf0 = n0 + f0 + j * 2;
        if (acc_dump != nullptr && row_ok) {
#pragma unroll
          for (int p = 0; p < 16; ++p)
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (kf0 + i < g.K)
                acc_dump[(static_cast<long long>(p) * g.M + m) * g.K + kf0 + i] =
                    static_cast<int32_t>(a[p][i]);
        }
        float2 mv[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const float2 c2 = *reinterpret_cast<const float2*>(&s_cterm[p * K_pad + kf0]);
          const float k1 = s_k1[p];
          float2 t1;
          if (SMALL) {
            // dot < 2^23: F = 2^23 + dot exactly, and fma(k1, F, -k1*2^23)
            // rounds once: RN(k1 * dot) = k1 * float(dot), bitwise.
            const float2 F = make_float2(__uint_as_float(a[p][0] | 0x4B000000u),
                                         __uint_as_float(a[p][1] | 0x4B000000u));
            t1 = fma2(bcast2(k1), F, bcast2(s_nk1m[p]));
          } else {
            t1 = make_float2(__fmul_rn(k1, __int2float_rn(static_cast<int>(a[p][0]))),
                             __fmul_rn(k1, __int2float_rn(static_cast<int>(a[p][1]))));
          }
          // ((k1*dot + k2*sum_a) + k3*sum_b) + k4, left to right.
          mv[p] = add2(add2(add2(t1, bcast2(rterm[p])), c2), bcast2(s_k4[p]));
        }
        // S = (A^T m) A (winograd.hpp:80-84 in matrix.hpp:75-84 order).
        float2 X0[4], X1[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          X0[c] = add2(add2(mv[c], mv[4 + c]), mv[8 + c]);
          X1[c] = sub2(sub2(mv[4 + c], mv[8 + c]), mv[12 + c]);
        }
        float2 s4[4];
        s4[0] = add2(add2(X0[0], X0[1]), X0[2]);
        s4[1] = sub2(sub2(X0[1], X0[2]), X0[3]);
        s4[2] = add2(add2(X1[0], X1[1]), X1[2]);
        s4[3] = sub2(sub2(X1[1], X1[2]), X1[3]);
        if (kf0 < g.K) {
#pragma unroll
          for (int ab = 0; ab < 4; ++ab) {
            float2 v = s4[ab];
            if (EPI) {
              if (bias != nullptr)
                v = add2(v, make_float2(bias[kf0], kf0 + 1 < g.K ? bias[kf0 + 1] : 0.0f));
              if (relu) {
                v.x = fmaxf(v.x, 0.0f);
                v.y = fmaxf(v.y, 0.0f);
              }
            }
            v = add2(v, bcast2(0.0f));  // the reference never yields -0
            if (!ok[ab]) continue;
            float* d = dst[ab] + j * 2;
            if (vec_ok)
              *reinterpret_cast<float2*>(d) = v;
            else {
              d[0] = v.x;
              if (kf0 + 1 < g.K) d[1] = v.y;
            }
          }
        }
      }
      if (++buf == 2) {
        buf = 0;
        acc_ph ^= 1u;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(*tmem_holder, 2 * Cfg::kAccCols);
  }
}

template <int BK, bool SMALL, bool EPI>
static cudaError_t launch_gemm_t(const CUtensorMap* tmA, const CUtensorMap* tmB,
                                 const int32_t* rowsum, const int32_t* colsum,
                                 const LanceDevState* st, float* y, int32_t* acc_dump,
                                 const float* bias, int relu, const GemmGeom& g, cudaStream_t s) {
  const size_t smem = GemmCfg<BK>::kSmemBase + static_cast<size_t>(16) * g.num_n_tiles * kBN * 4;
  if (smem > kSmemLimit) return cudaErrorInvalidValue;
  static size_t configured[64] = {};  // dynamic-smem attribute set so far, per device
  static int sm_count[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || configured[dev] < smem) {
    cudaError_t e = cudaFuncSetAttribute(gemm_epilogue_kernel<BK, SMALL, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) {
      configured[dev] = smem;
      sm_count[dev] = sms;
    }
  }
  const int sms = (dev >= 0 && dev < 64) ? sm_count[dev] : 148;
  const long long tiles = ((static_cast<long long>(g.M) + kBM - 1) / kBM) * g.num_n_tiles;
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  gemm_epilogue_kernel<BK, SMALL, EPI><<<grid, kGemmThreadsP, smem, s>>>(
      *tmA, *tmB, rowsum, colsum, st, y, acc_dump, bias, relu, g);
  return cudaGetLastError();
}

template <int BK>
static cudaError_t launch_gemm_bk(const CUtensorMap* tmA, const CUtensorMap* tmB, int small_acc,
                                  const int32_t* rowsum, const int32_t* colsum,
                                  const LanceDevState* st, float* y, int32_t* acc_dump,
                                  const float* bias, int relu, const GemmGeom& g, cudaStream_t s) {
  const bool epi = bias != nullptr || relu;
  if (small_acc)
    return epi ? launch_gemm_t<BK, true, true>(tmA, tmB, rowsum, colsum, st, y, acc_dump, bias,
                                               relu, g, s)
               : launch_gemm_t<BK, true, false>(tmA, tmB, rowsum, colsum, st, y, acc_dump, bias,
                                                relu, g, s);
  return epi ? launch_gemm_t<BK, false, true>(tmA, tmB, rowsum, colsum, st, y, acc_dump, bias,
                                              relu, g, s)
             : launch_gemm_t<BK, false, false>(tmA, tmB, rowsum, colsum, st, y, acc_dump, bias,
                                               relu, g, s);
}

cudaError_t launch_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, int bk, int small_acc,
                        const int32_t* rowsum, const int32_t* colsum, const LanceDevState* st,
                        float* y, int32_t* acc_dump, const float* bias, int relu,
                        const GemmGeom& g, cudaStream_t s) {
  switch (bk) {
    case 128:
      return launch_gemm_bk<128>(tmA, tmB, small_acc, rowsum, colsum, st, y, acc_dump, bias,
                                 relu, g, s);
    case 64:
      return launch_gemm_bk<64>(tmA, tmB, small_acc, rowsum, colsum, st, y, acc_dump, bias,
                                relu, g, s);
    case 32:
      return launch_gemm_bk<32>(tmA, tmB, small_acc, rowsum, colsum, st, y, acc_dump, bias,
                                relu, g, s);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace lance_dev
