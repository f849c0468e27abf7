// lance_gemm.cu -- K3/K4: the 16 per-position u8 x u8 -> s32 GEMMs of
// lance_gemm (gemm_codes x 16, lowpgemm.hpp:76-100, engines.hpp:510-525) on
// tcgen05 kind::i8 with TMA-fed operands and accumulators in TMEM, fused with
// the affine de-quantisation (affine_term, lowpgemm.hpp:110-114), the output
// transform A^T m A (winograd.hpp:80-84) and the merge with ragged-edge
// discard (tensor.hpp:157-182).
//
// Persistent kernel, one CTA per SM.  A tile = 128 Winograd tiles (UMMA M)
// x BN filters (UMMA N) x all 16 positions = 16*BN s32 TMEM columns; with
// BN = 16 TMEM holds two accumulators (the MMA of tile i+1 overlaps the
// epilogue of tile i), with BN = 32 one (twice the MMA work per A byte: a
// K=32 kind::i8 MMA with M=128 costs ~44 cycles for any N <= 32 because the
// 4 KB A operand is read from shared memory each time).  The TMA producer runs
// ahead of the MMA through a shared-memory ring.
//   warp 0       TMA producer (one lane): per stage the A box
//                [128 rows x BK ch] and the B box [BN filters x BK ch] of one
//                position
//   warp 1       TMEM allocator + UMMA issuer (one lane)
//   warps 2..9   epilogue: TMEM -> registers -> affine -> A^T m A -> shared
//                staging -> full-sector stores of y; warp w drains TMEM lane
//                quadrant w % 4 and filters (BN/2)*((w-2)/4) .. +BN/2
// CTAs form clusters of cs (1, 2 or 4) that work on the same row tile and on
// cs different filter tiles: each CTA loads 128/cs rows of the A box and
// multicasts them to the whole cluster (TMA .multicast::cluster), so the A
// operand is read from L2 once per cluster instead of once per filter tile;
// each CTA's MMA commit releases the stage in every CTA of the cluster.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lance_common.cuh"

namespace lance_dev {

constexpr int kEpiWarps = 8;
constexpr int kGemmThreadsP = 64 + 32 * kEpiWarps;  // 320
constexpr size_t kSmemLimit = 226 * 1024;           // dynamic part, leaves room for static smem

template <int BK, int BN>
struct GemmCfg {
  static constexpr int kBufs = (BN == 16) ? 2 : 1;
  static constexpr uint32_t kABytes = kBM * BK;
  static constexpr uint32_t kBBytes = BN * BK;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr int kStagesRaw = (128 * 1024) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 16 ? 16 : kStagesRaw;
  static constexpr uint32_t kLayout = (BK == 128) ? 2u : (BK == 64 ? 4u : 6u);  // SW128/64/32
  static constexpr uint32_t kAccCols = 16 * BN;
  static constexpr uint32_t kStagingBytes = kEpiWarps * 32 * 4 * 8 * 4;  // 8 filters x 4 px x 32 rows
  // + 16 * K_pad floats of per-filter constants, added at launch.
  static constexpr size_t kSmemBase = 1024 + static_cast<size_t>(kStages) * kStageBytes +
                                      kStagingBytes + (2 * kStages + 4) * 8 + 16;
};

// SMALL: C * top_a * top_b < 2^23, so every accumulator is below 2^23 and
// k1 * float(dot) is formed exactly by one FFMA (see below).
// EPI: fused bias + ReLU (north-star extension).
template <int BK, int BN, bool SMALL, bool EPI>
__global__ void __launch_bounds__(kGemmThreadsP, 1)
    gemm_epilogue_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB,
                         const int32_t* __restrict__ rowsum, const int32_t* __restrict__ colsum,
                         const LanceDevState* __restrict__ st, float* __restrict__ y,
                         int32_t* __restrict__ acc_dump, const float* __restrict__ bias,
                         int relu, GemmGeom g) {
  using Cfg = GemmCfg<BK, BN>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kBufs = Cfg::kBufs;
  constexpr uint32_t kIdesc = umma_idesc_u8(kBM, BN);
  constexpr int kWarpFilters = BN / 2;  // filters per epilogue warp

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ float s_k1[16], s_nk1m[16], s_k2[16], s_k4[16];

  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* stage_base = smem;
  float* staging = reinterpret_cast<float*>(smem + kStages * Cfg::kStageBytes);  // [8 warps][1024]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes +
                                                   Cfg::kStagingBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* acc_full = empty_bar + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;        // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* s_cterm = reinterpret_cast<float*>(tmem_holder + 4);  // [16][K_pad]: k3[p]*colsum[p][k]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = g.num_n_tiles;
  const int K_pad = nt * BN;
  const int cs = g.cluster;                       // CTAs per cluster (divides nt)
  const int rank = cs > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int cid = blockIdx.x / cs, ncl = gridDim.x / cs;
  const int ngrp = nt / cs;                       // filter-tile groups per row tile
  const int num_groups = ((g.M + kBM - 1) / kBM) * ngrp;
  const int num_iters = g.num_kchunks * 16;
  const uint16_t cl_mask = static_cast<uint16_t>((1u << cs) - 1u);
  const int a_rows = kBM / cs;                    // A rows this CTA loads and multicasts
  // Group index -> (row tile origin, this CTA's filter tile origin).
  auto tile_m0 = [&](int grp_i) { return (grp_i / ngrp) * kBM; };
  auto tile_n0 = [&](int grp_i) { return ((grp_i % ngrp) * cs + rank) * BN; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
#ifdef LANCE_DEBUG_HANG
      mbar_init(&empty_bar[s], g.dbg_mode >= 2 ? 1 : cs);
#else
      mbar_init(&empty_bar[s], cs);  // one MMA commit from every CTA of the cluster
#endif
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (cs > 1) cluster_sync();  // barrier inits visible cluster-wide before any multicast
#ifdef LANCE_DEBUG_HANG
  if (threadIdx.x == 0 && blockIdx.x < 2)
    printf("DBG block %d after cluster_sync: full0 0x%016llx empty0 0x%016llx stage_base 0x%x full_bar 0x%x holder 0x%x cterm 0x%x\n",
           blockIdx.x, (unsigned long long)*reinterpret_cast<volatile uint64_t*>(&full_bar[0]),
           (unsigned long long)*reinterpret_cast<volatile uint64_t*>(&empty_bar[0]), smem_u32(stage_base),
           smem_u32(full_bar), smem_u32(tmem_holder), smem_u32(s_cterm));
#endif
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
#ifdef LANCE_DEBUG_HANG
  if (threadIdx.x == 0 && blockIdx.x < 2)
    printf("DBG block %d after syncthreads: full0 0x%016llx empty0 0x%016llx\n", blockIdx.x,
           (unsigned long long)*reinterpret_cast<volatile uint64_t*>(&full_bar[0]),
           (unsigned long long)*reinterpret_cast<volatile uint64_t*>(&empty_bar[0]));
#endif

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int s = 0;
      uint32_t ph = 0;
      for (int grp_i = cid; grp_i < num_groups; grp_i += ncl) {
        const int m0 = tile_m0(grp_i), n0 = tile_n0(grp_i);
        for (int it = 0; it < num_iters; ++it) {
          const int kc = it >> 4, p = it & 15;
          mbar_wait(&empty_bar[s], ph ^ 1u, 1, grp_i, it);  // released by all cs consumers
          uint8_t* sa = stage_base + s * Cfg::kStageBytes;
          mbar_arrive_expect_tx(&full_bar[s], Cfg::kStageBytes);
#ifdef LANCE_DEBUG_HANG
          if (g.dbg_mode == 1 || g.dbg_mode == 3) {  // no multicast: local slices
            for (int rr = 0; rr < cs; ++rr)
              tma_load_3d(sa + rr * a_rows * BK, &tmA, kc * BK, m0 + rr * a_rows, p, &full_bar[s]);
          } else
#endif
          if (cs > 1)
            tma_load_3d_mc(sa + rank * a_rows * BK, &tmA, kc * BK, m0 + rank * a_rows, p,
                           &full_bar[s], cl_mask);
          else
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
    tmem_alloc(tmem_holder, 512);
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
      for (int grp_i = cid; grp_i < num_groups; grp_i += ncl) {
        mbar_wait(&acc_empty[buf], acc_ph ^ 1u, 2, grp_i, buf);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t d_base = tmem_base + static_cast<uint32_t>(buf) * Cfg::kAccCols;
        for (int it = 0; it < num_iters; ++it) {
          const int kc = it >> 4, p = it & 15;
          mbar_wait(&full_bar[s], ph, 3, grp_i, it);
          tc_fence_after();
          const uint32_t sa = smem_u32(stage_base + s * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk) {
            const uint64_t adesc = umma_smem_desc(sa + kk * 32, 8 * BK, Cfg::kLayout);
            const uint64_t bdesc = umma_smem_desc(sb + kk * 32, 8 * BK, Cfg::kLayout);
            umma_i8(d_base + static_cast<uint32_t>(p * BN), adesc, bdesc, kIdesc,
                    (kc > 0 || kk > 0) ? 1u : 0u);
          }
#ifdef LANCE_DEBUG_HANG
          if (g.dbg_mode >= 2) {  // per-CTA release only
            umma_commit(&empty_bar[s]);
          } else
#endif
          if (cs > 1)
            umma_commit_mc(&empty_bar[s], cl_mask);
          else
            umma_commit(&empty_bar[s]);
          if (++s == kStages) {
            s = 0;
            ph ^= 1u;
          }
        }
        umma_commit(&acc_full[buf]);
        if (++buf == kBufs) {
          buf = 0;
          acc_ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue ----------------
    const int ew = warp - 2;
    const int q = warp & 3;                   // TMEM lane quadrant this warp may access
    const int f0 = (ew >> 2) * kWarpFilters;  // this warp's filters within the tile
    float* stg = staging + ew * 1024;         // [32 rows][4 px][8 filters], 16-B chunks swizzled
    named_bar_sync(1, 32 + 32 * kEpiWarps);
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const bool k4ok = (g.K & 3) == 0;
    int buf = 0;
    uint32_t acc_ph = 0;
    // Row sums of the first tile (later tiles are prefetched one tile ahead).
    int32_t rs_next[16];
    {
      const int m = tile_m0(cid) + q * 32 + lane;
#pragma unroll
      for (int p = 0; p < 16; ++p)
        rs_next[p] = (cid < num_groups && m < g.M)
                         ? __ldg(rowsum + static_cast<long long>(p) * g.M + m) : 0;
    }
    for (int grp_i = cid; grp_i < num_groups; grp_i += ncl) {
      const int m0 = tile_m0(grp_i), n0 = tile_n0(grp_i);
      const int m = m0 + q * 32 + lane;
      const bool row_ok = m < g.M;
      float rterm[16];  // k2[p] * float(sum_a): second term of affine_term
#pragma unroll
      for (int p = 0; p < 16; ++p) rterm[p] = __fmul_rn(s_k2[p], static_cast<float>(rs_next[p]));
      {
        const int nxt = grp_i + ncl;
        const int mn = tile_m0(nxt) + q * 32 + lane;
#pragma unroll
        for (int p = 0; p < 16; ++p)
          rs_next[p] = (nxt < num_groups && mn < g.M)
                           ? __ldg(rowsum + static_cast<long long>(p) * g.M + mn) : 0;
      }
      // Output pixels of this lane's tile (2ti + a, 2tj + b) and their
      // validity (merge_tiles discards the ceil-overhang, tensor.hpp:172-175).
      // Packed (pixel index << 4 | validity mask): pixel counts < 2^27 are
      // checked at plan creation.
      int pixm;
      {
        const int mm = row_ok ? m : 0;
        const int img = mm / g.P;
        const int t = mm - img * g.P;
        const int ti = t / g.TW, tj = t - ti * g.TW;
        const int pix0 = (img * g.OH + 2 * ti) * g.OW + 2 * tj;
        const bool r1 = 2 * ti + 1 < g.OH, c1 = 2 * tj + 1 < g.OW;
        const int pmask = row_ok ? (1 | (c1 ? 2 : 0) | (r1 ? 4 : 0) | (r1 && c1 ? 8 : 0)) : 0;
        pixm = (pix0 << 4) | pmask;
      }
      mbar_wait(&acc_full[buf], acc_ph, 4, grp_i, warp);
      tc_fence_after();
      const uint32_t acc_addr = lane_base + static_cast<uint32_t>(buf) * Cfg::kAccCols + f0;
#pragma unroll 1
      for (int grp = 0; grp < kWarpFilters / 8; ++grp) {
#pragma unroll 1
        for (int jj = 0; jj < 4; ++jj) {  // filter pairs of this 8-filter group
          const int fl = grp * 8 + jj * 2;  // filter offset within the warp's range
          uint32_t a[16][2];
#pragma unroll
          for (int p = 0; p < 16; ++p) tmem_ld_x2(acc_addr + p * BN + fl, a[p]);
          tmem_ld_wait();
          if (grp == kWarpFilters / 8 - 1 && jj == 3) {
            // All of this warp's accumulators are in registers: hand the TMEM
            // buffer back to the MMA warp early.
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
          }
          const int kf0 = n0 + f0 + fl;
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
#pragma unroll
          for (int ab = 0; ab < 4; ++ab) {
            float2 v = s4[ab];
            if (EPI) {
              if (bias != nullptr)
                v = add2(v, make_float2(kf0 < g.K ? bias[kf0] : 0.0f,
                                        kf0 + 1 < g.K ? bias[kf0 + 1] : 0.0f));
              if (relu) {
                v.x = fmaxf(v.x, 0.0f);
                v.y = fmaxf(v.y, 0.0f);
              }
            }
            v = add2(v, bcast2(0.0f));  // the reference never yields -0
            // staging row = lane (tile), 16-B chunk (ab*2 + jj/2) ^ (lane & 7)
            const int chunk = (ab * 2 + (jj >> 1)) ^ (lane & 7);
            *reinterpret_cast<float2*>(&stg[lane * 32 + chunk * 4 + (jj & 1) * 2]) = v;
          }
        }
        __syncwarp();
        // Store phase: 32 rows x 4 pixels x 8 filters = 256 16-B chunks, two
        // lanes per 32-byte pixel segment (full sectors).
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = lane + 32 * i;
          const int r = c >> 3, ab = (c >> 1) & 3, half = c & 1;
          const int rp = __shfl_sync(0xffffffffu, pixm, r);  // row r's pixel base + mask
          const float4 val =
              *reinterpret_cast<const float4*>(&stg[r * 32 + (((ab * 2 + half) ^ (r & 7)) * 4)]);
          if (!((rp >> ab) & 1)) continue;
          const int kf = n0 + f0 + grp * 8 + half * 4;
          if (kf >= g.K) continue;
          const int pix = (rp >> 4) + (ab >> 1) * g.OW + (ab & 1);
          float* d = y + static_cast<long long>(pix) * g.K + kf;
          if (k4ok) {
            *reinterpret_cast<float4*>(d) = val;
          } else {
            const float v4[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (kf + e < g.K) d[e] = v4[e];
          }
        }
        __syncwarp();
      }
      if (++buf == kBufs) {
        buf = 0;
        acc_ph ^= 1u;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(*tmem_holder, 512);
  }
  if (cs > 1) cluster_sync();  // no CTA leaves while cluster peers may still signal it
}

template <int BK, int BN, bool SMALL, bool EPI>
static cudaError_t launch_gemm_t(const CUtensorMap* tmA, const CUtensorMap* tmB,
                                 const int32_t* rowsum, const int32_t* colsum,
                                 const LanceDevState* st, float* y, int32_t* acc_dump,
                                 const float* bias, int relu, const GemmGeom& g, cudaStream_t s) {
  const size_t smem =
      GemmCfg<BK, BN>::kSmemBase + static_cast<size_t>(16) * g.num_n_tiles * BN * 4;
  if (smem > kSmemLimit) return cudaErrorInvalidValue;
  static size_t configured[64] = {};  // dynamic-smem attribute set so far, per device
  static int sm_count[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || configured[dev] < smem) {
    cudaError_t e = cudaFuncSetAttribute(gemm_epilogue_kernel<BK, BN, SMALL, EPI>,
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
  const int cs = g.cluster;
  const long long groups =
      ((static_cast<long long>(g.M) + kBM - 1) / kBM) * (g.num_n_tiles / cs);
  const long long clusters = groups < sms / cs ? groups : sms / cs;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * cs));
  cfg.blockDim = dim3(kGemmThreadsP);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_epilogue_kernel<BK, BN, SMALL, EPI>, *tmA, *tmB, rowsum,
                            colsum, st, y, acc_dump, bias, relu, g);
}

template <int BK, int BN>
static cudaError_t launch_gemm_bk(const CUtensorMap* tmA, const CUtensorMap* tmB, int small_acc,
                                  const int32_t* rowsum, const int32_t* colsum,
                                  const LanceDevState* st, float* y, int32_t* acc_dump,
                                  const float* bias, int relu, const GemmGeom& g, cudaStream_t s) {
  const bool epi = bias != nullptr || relu;
  if (small_acc)
    return epi ? launch_gemm_t<BK, BN, true, true>(tmA, tmB, rowsum, colsum, st, y, acc_dump,
                                                   bias, relu, g, s)
               : launch_gemm_t<BK, BN, true, false>(tmA, tmB, rowsum, colsum, st, y, acc_dump,
                                                    bias, relu, g, s);
  return epi ? launch_gemm_t<BK, BN, false, true>(tmA, tmB, rowsum, colsum, st, y, acc_dump,
                                                  bias, relu, g, s)
             : launch_gemm_t<BK, BN, false, false>(tmA, tmB, rowsum, colsum, st, y, acc_dump,
                                                   bias, relu, g, s);
}

cudaError_t launch_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, int bk, int bn,
                        int small_acc, const int32_t* rowsum, const int32_t* colsum,
                        const LanceDevState* st, float* y, int32_t* acc_dump, const float* bias,
                        int relu, const GemmGeom& g, cudaStream_t s) {
#define LANCE_GEMM_CASE(BKV, BNV)                                                            \
  if (bk == BKV && bn == BNV)                                                                \
    return launch_gemm_bk<BKV, BNV>(tmA, tmB, small_acc, rowsum, colsum, st, y, acc_dump,    \
                                    bias, relu, g, s);
  LANCE_GEMM_CASE(128, 16)
  LANCE_GEMM_CASE(64, 16)
  LANCE_GEMM_CASE(32, 16)
  LANCE_GEMM_CASE(128, 32)
  LANCE_GEMM_CASE(64, 32)
  LANCE_GEMM_CASE(32, 32)
#undef LANCE_GEMM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace lance_dev
