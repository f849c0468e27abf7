// lance_gemm.cu -- K3/K4: the 16 per-position u8 x u8 -> s32 GEMMs of
// lance_gemm (gemm_codes x 16, lowpgemm.hpp:76-100, engines.hpp:510-525) on
// tcgen05 kind::i8 with TMA-fed operands and accumulators in TMEM, fused with
// the affine de-quantisation (affine_term, lowpgemm.hpp:110-114), the output
// transform A^T m A (winograd.hpp:80-84) and the merge with ragged-edge
// discard (tensor.hpp:157-182).
//
// Position order.  S = (A^T m) A is evaluated as in matrix.hpp:75-84:
//   T0j = (m_j + m_{4+j}) + m_{8+j},  T1j = (m_{4+j} - m_{8+j}) - m_{12+j}
//   S00 = (T00 + T01) + T02, S01 = (T01 - T02) - T03   (S1b likewise from T1j)
// Both folds are left folds, so the positions can be consumed in j-groups
// {j, 4+j, 8+j, 12+j}, j = 0..3, with four running partials S_ab per
// (tile, filter): bit-identical to the all-16-resident form.  A j-group
// needs 4 x BN TMEM columns, so TMEM (512 columns) double-buffers j-groups
// at BN = 64 filters per tile: a 128 x 64 x 32 kind::i8 UMMA runs at ~2/3 of
// the tensor peak where the 128 x 32 one needed for all-16-resident tiles
// runs at ~1/3 (A is re-read from shared memory by every MMA).
//
// Persistent kernel, one CTA per SM, tiles = 128 Winograd tiles (UMMA M) x
// BN filters, n-tile fastest so concurrent CTAs share the A rows in L2.
//   warps 0..15  epilogue: warp w drains TMEM lane quadrant w % 4 and
//                filters BN/4 * (w / 4) .. +BN/4 of the tile; each thread
//                owns one Winograd tile (row) and keeps the S partials of its
//                filters in registers; y leaves through a swizzled shared
//                staging buffer as whole 128-byte lines (or straight from
//                registers when the layer runs without staging).
//   warp 16      producer: per stage one bulk copy of U consecutive A images
//                [128 rows x BK ch] (and B images [BN filters x BK ch] unless
//                B is resident) of one position
//   warp 17      TMEM allocator + UMMA issuer
//   warps 18-19  row sums of the A stages (BK = 64 layers; else K1 writes them)
// The producer and the UMMA issuer run warp-uniform loops (addresses and
// descriptors in uniform registers) with one elect.sync lane issuing each
// copy / tcgen05.mma / commit: these two threads' per-stage latency is serial
// work, and the lane-0-only form cost up to 2x on the deep layers.
// JS (small M): a tile's 4 j-groups run on 4 CTAs (see the kernel comment).
// Exact int -> float epilogue without a conversion instruction (SMALL: every
// accumulator dot < 2^24, i.e. C * top_a * top_b < 2^24).  The int32 bits of
// dot read as an fp32 are the subnormal / first-binade float D = dot * 2^-149
// exactly, so with k1s = k1 * 2^126 (exact power-of-two scaling)
//   u = RN(k1s * D) = RN(k1 * dot) * 2^-23        (one FFMA2, exact scaling)
//   fma(u, 2^23, rterm) = RN(RN(k1 * dot) + rterm)  (one FFMA2)
// which is affine_term's first two terms bit for bit, provided k1 * dot stays
// a normal float (k1 == 0 or 2^-103 <= k1 < 4); other k1 fall back to I2F.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "lance_common.cuh"

namespace lance_dev {

constexpr int kEpiWarps = 16;                      // warps 0..15: epilogue (4 warpgroups)
constexpr int kProducerWarp = 16, kMmaWarp = 17;  // warpgroup 4: producer, MMA,
constexpr int kRowSumWarp0 = 18;                  // and two warps summing the A rows
constexpr int kGemmThreadsP = 32 * 20;            // 640
// Register split (setmaxnreg): the control warpgroup gives its registers to
// the epilogue warpgroups (S partials of 64-filter tiles live in registers).
constexpr int kCtrlRegs = 32, kEpiRegs = 112;
constexpr size_t kSmemLimit = 225 * 1024;           // dynamic part, leaves room for static smem
constexpr float kTwo23 = 8388608.0f;
constexpr float kTwo126 = 8.507059173023462e37f;   // 2^126

template <int BK, int BN>
struct GemmCfg {
  static constexpr uint32_t kABytes = kBM * BK;
  static constexpr uint32_t kBBytes = BN * BK;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kLayout = (BK == 128) ? 2u : (BK == 64 ? 4u : 6u);  // SW128/64/32
  static constexpr uint32_t kGroupCols = 4 * BN;  // one j-group: 4 positions x BN filters
  static constexpr int kAccBufs = (512 / kGroupCols) < 4 ? (512 / kGroupCols) : 4;
  static constexpr int kFPT = BN / 4;             // filters per epilogue thread
  static constexpr uint32_t kRsBytes = 16 * kBM * 4;  // row sums of one tile [16][128] i32
  // Output staging: per lane quadrant 32 tiles x 2 pixels x BN filters fp32.
  static constexpr uint32_t kOutBytes = 4 * 32 * 2 * BN * 4;
  // Third affine term k3[p] * colsum[p][k] of the tile's filters, two tile buffers.
  static constexpr uint32_t kCtBytes = 2 * 16 * BN * 4;
  static constexpr size_t kFixed =
      1024 /*align*/ + 2 * kRsBytes + kOutBytes + kCtBytes + 32 * 8 /*barriers, holder*/;
};

// STAGE = false: no output staging buffer (y written straight from registers,
// 64 contiguous bytes per thread and pixel); its 4 * 32 * 2 * BN * 4 bytes go
// to deeper operand stages instead.  Measured on the load-latency-bound deep
// layers (C >= 256) where bytes in flight per SM set the GEMM rate.
template <int BK, int BN>
__host__ __device__ constexpr size_t gemm_fixed_bytes(bool stage_out) {
  return GemmCfg<BK, BN>::kFixed - (stage_out ? 0 : GemmCfg<BK, BN>::kOutBytes);
}

// b_res: the whole B operand of the (single) filter tile stays resident in
// shared memory and stages carry only A.
// A stage holds `units` consecutive k chunks of one position (one bulk copy
// for A and one for B per stage: the images of a position are contiguous).
template <int BK, int BN>
__host__ __device__ constexpr size_t gemm_smem_bytes(int stages, int nk, int b_res, bool stage_out,
                                                     int units) {
  return gemm_fixed_bytes<BK, BN>(stage_out) +
         static_cast<size_t>(stages) * units *
             (b_res ? GemmCfg<BK, BN>::kABytes : GemmCfg<BK, BN>::kStageBytes) +
         (b_res ? static_cast<size_t>(16) * nk * GemmCfg<BK, BN>::kBBytes : 0) +
         static_cast<size_t>(stages) * 16;
}

// Epilogue of one j-group for 4 filters (one TMEM x4 load per position).
// acc[a][i]: accumulator of position p = 4a + j, filter f0 + 4c + i;
// k1s[a] = k1[p] * 2^126 (fast) or k1[p]; ct_j: the tile's cterm row of
// position j at this thread's 4 filters (rows of positions 4a + j are 4 * BN apart).
template <int BN>
__device__ __forceinline__ void affine_group4(const uint32_t (&acc)[4][4], bool fast,
                                              const float (&k1s)[4], const float (&k4)[4],
                                              const float (&rterm)[4], const float* ct_j,
                                              float2 (&T0)[2], float2 (&T1)[2]) {
  float2 m[4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float4 ct = *reinterpret_cast<const float4*>(ct_j + a * 4 * BN);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t d0 = acc[a][2 * h], d1 = acc[a][2 * h + 1];
      float2 v;  // RN(k1 * dot + k2 * sum_a), both products rounded first
      if (fast) {
        const float2 u = fma2(bcast2(k1s[a]), make_float2(__uint_as_float(d0), __uint_as_float(d1)),
                              bcast2(0.0f));
        v = fma2(u, bcast2(kTwo23), bcast2(rterm[a]));
      } else {
        v = add2(make_float2(__fmul_rn(k1s[a], __int2float_rn(static_cast<int>(d0))),
                             __fmul_rn(k1s[a], __int2float_rn(static_cast<int>(d1)))),
                 bcast2(rterm[a]));
      }
      const float2 c2 = h ? make_float2(ct.z, ct.w) : make_float2(ct.x, ct.y);
      // ((k1*dot + k2*sum_a) + k3*sum_b) + k4, left to right (lowpgemm.hpp:110-114).
      m[a][h] = add2(add2(v, c2), bcast2(k4[a]));
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    T0[h] = add2(add2(m[0][h], m[1][h]), m[2][h]);
    T1[h] = sub2(sub2(m[1][h], m[2][h]), m[3][h]);
  }
}

#ifndef LANCE_GEMM_TRACE_CTA
#define LANCE_GEMM_TRACE_CTA 0
#endif
// Profiling trace (LANCE_GEMM_TRACE): CTA LANCE_GEMM_TRACE_CTA records SM clocks, 8 slots x 100000
// events (buffer allocated by lance_abi.cu in LANCE_PROFILING builds).
__device__ __forceinline__ void trace_event(unsigned long long* tr, int slot, int i) {
#ifdef LANCE_GEMM_TRACE
  if (tr != nullptr && blockIdx.x == static_cast<unsigned>(LANCE_GEMM_TRACE_CTA) && i < 100000)
    tr[slot * 100000 + i] = clock64();
#else
  (void)tr;
  (void)slot;
  (void)i;
#endif
}

__device__ __forceinline__ void tmem_ld_group4(uint32_t addr, int bn, uint32_t (&acc)[4][4]) {
#pragma unroll
  for (int a = 0; a < 4; ++a) tmem_ld_x4(addr + a * bn, acc[a]);
}

// SMALL: see the file comment.  DUMP: also write the raw int32 accumulators
// (parity tests).  bias / relu: fused epilogue (north-star extension).
// JS (j-split, small-M layers): a tile's 4 j-groups run on 4 CTAs as separate
// work units (tile, j).  Each unit writes its T0j / T1j (the column folds of
// A^T m, exact fp32, matrix.hpp:75-84) to g.tscratch; the unit that finishes
// last (per-tile ticket) reads all four and completes the left fold
// S00 = (T00 + T01) + T02, S01 = (T01 - T02) - T03 (S1b likewise) in the
// reference order, so y is bit-identical to the single-CTA fold.
template <int BK, int BN, bool SMALL, bool DUMP, bool STAGE, bool JS>
__global__ void __launch_bounds__(kGemmThreadsP, 1)
    gemm_epilogue_kernel(const uint8_t* __restrict__ codes_a,
                         const uint8_t* __restrict__ codes_w,
                         const __grid_constant__ CUtensorMap tmR,
                         int32_t* __restrict__ rowsum_out,
                         const int32_t* __restrict__ colsum,
                         const LanceDevState* __restrict__ st, float* __restrict__ y,
                         int32_t* __restrict__ acc_dump, const float* __restrict__ bias,
                         int relu, GemmGeom g) {
  using Cfg = GemmCfg<BK, BN>;
  constexpr int FPT = Cfg::kFPT;
  constexpr int NCH = FPT / 4;  // 4-filter chunks per thread
  constexpr int NB = Cfg::kAccBufs;
  constexpr uint32_t kIdesc = umma_idesc_u8(kBM, BN);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ float s_k1[16], s_k2[16], s_k3[16], s_k4[16];
  __shared__ int s_fast;

  // 1024-byte aligned base (SWIZZLE_128B atoms), derived by offsetting the
  // __shared__ array so every access below stays in the shared window (LDS/STS,
  // not generic loads).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stages = g.stages;
  const int nk = g.num_kchunks;
  const bool b_res = g.b_resident != 0;
  const int U = g.units;  // k chunks per stage (divides nk)
  const uint32_t stage_bytes = U * (b_res ? Cfg::kABytes : Cfg::kStageBytes);
  uint8_t* stage_base = smem;
  uint8_t* b_base = smem + static_cast<size_t>(stages) * stage_bytes;  // resident B images
  int32_t* s_rs = reinterpret_cast<int32_t*>(b_base + (b_res ? 16 * nk * Cfg::kBBytes : 0));
  float* s_out = reinterpret_cast<float*>(s_rs + 2 * 16 * kBM);  // [4 quadrants][64 segs][BN]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(s_out + (STAGE ? Cfg::kOutBytes / 4 : 0));
  uint64_t* empty_bar = full_bar + stages;
  uint64_t* acc_full = empty_bar + stages;  // [4]
  uint64_t* acc_empty = acc_full + 4;       // [4]
  uint64_t* rs_ready = acc_empty + 4;       // [2 tile buffers][4 j-groups]
  uint64_t* rs_empty = rs_ready + 8;        // [2]
  uint64_t* b_full = rs_empty + 2;          // [1]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(b_full + 2);
  float* s_cterm = reinterpret_cast<float*>(tmem_holder + 4);  // [2 tiles][16][BN]: k3[p]*colsum[p][k]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = g.num_n_tiles;
  const int K_pad = nt * BN;
  const int num_tiles = ((g.M + kBM - 1) / kBM) * nt;
  // Work units: tiles, or (tile, j-group) pairs under JS (j fastest).
  const int num_work = JS ? 4 * num_tiles : num_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], g.rs_warps ? 3 : 1);  // MMA commit (+ the two row-sum warps)
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps);
    }
    // rs_warps: per (tile buffer, j-group), arrived by the two row-sum warps;
    // else one TMA of the tile's row sums (written by K1) completes [tb][0].
    for (int b = 0; b < 8; ++b) mbar_init(&rs_ready[b], g.rs_warps ? 2 : 1);
    for (int b = 0; b < 2; ++b) mbar_init(&rs_empty[b], kEpiWarps);
    mbar_init(b_full, 1);
    fence_barrier_init();
  }
  pdl_entry();  // barriers above are shared-memory only; st / codes / y below
  if (warp < kEpiWarps) {
    const int e = threadIdx.x;
    if (e < 32) {
      const float k1 = e < 16 ? st->k1[e] : 0.0f;
      const bool ok = k1 == 0.0f || (k1 >= 9.860761315262648e-32f /*2^-103*/ && k1 < 4.0f);
      const bool fast = SMALL && __all_sync(0xffffffffu, ok);
      if (e < 16) {
        s_k1[e] = fast ? __fmul_rn(k1, kTwo126) : k1;
        s_k2[e] = st->k2[e];
        s_k3[e] = st->k3[e];
        s_k4[e] = st->k4[e];
      }
      if (e == 0) s_fast = fast ? 1 : 0;
    }
  }
  __syncthreads();

  if (warp >= kEpiWarps) {
    setmaxnreg_dec<kCtrlRegs>();
    if (warp == kProducerWarp) {
      // ---------------- TMA producer ----------------
      // One bulk copy per operand per stage (U k chunks of one position).  As
      // for the MMA issuer, the whole warp runs the uniform loop and one
      // elected lane posts the expected bytes and issues the copies.
      if (b_res && elect_one()) {  // the single filter tile's B images, once
        mbar_arrive_expect_tx(b_full, 16 * nk * Cfg::kBBytes);
        bulk_load(b_base, codes_w, 16 * nk * Cfg::kBBytes, b_full);
      }
      __syncwarp();
      int s = 0;
      uint32_t ph = 0;
      uint32_t lt = 0;
      int tr_p = 0;
      for (int w = blockIdx.x; w < num_work; w += gridDim.x, ++lt) {
        const int t = JS ? w >> 2 : w;
        const int j_lo = JS ? (w & 3) : 0, j_hi = JS ? j_lo + 1 : 4;
        const int mt = t / nt, ntile = t % nt;
        const int m0 = mt * kBM;
        // Operand images of this tile (lance_kernels.cuh umma_image_offset).
        const uint8_t* a_tile = codes_a + static_cast<long long>(mt) * 16 * nk * Cfg::kABytes;
        const uint8_t* b_tile = codes_w + static_cast<long long>(ntile) * 16 * nk * Cfg::kBBytes;
        if (!g.rs_warps) {  // row sums of the tile's 128 rows, all 16 positions (OOB rows read 0)
          const uint32_t rb = lt & 1u;
          mbar_wait(&rs_empty[rb], ((lt >> 1) & 1u) ^ 1u);
          if (elect_one()) {
            mbar_arrive_expect_tx(&rs_ready[rb * 4], Cfg::kRsBytes);
            tma_load_2d(s_rs + rb * 16 * kBM, &tmR, m0, 0, &rs_ready[rb * 4]);
          }
          __syncwarp();
        }
        for (int j = j_lo; j < j_hi; ++j)
          for (int a = 0; a < 4; ++a) {
            const int u0 = image_plane(4 * a + j) * nk;
            for (int kc = 0; kc < nk; kc += U) {
              mbar_wait(&empty_bar[s], ph ^ 1u);
              if (lane == 0) trace_event(g.trace, 0, tr_p);
              ++tr_p;
              uint8_t* sa = stage_base + static_cast<size_t>(s) * stage_bytes;
              if (elect_one()) {
                mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
                bulk_load(sa, a_tile + (u0 + kc) * Cfg::kABytes, U * Cfg::kABytes, &full_bar[s]);
                if (!b_res)
                  bulk_load(sa + U * Cfg::kABytes, b_tile + (u0 + kc) * Cfg::kBBytes, U * Cfg::kBBytes,
                            &full_bar[s]);
              }
              __syncwarp();
              if (++s == stages) {
                s = 0;
                ph ^= 1u;
              }
            }
          }
      }
    } else if (warp == kMmaWarp) {
      // ---------------- TMEM + UMMA issuer ----------------
      // The whole warp runs the (warp-uniform) loop, so stage addresses and
      // descriptors live in uniform registers; one elected lane issues each
      // tcgen05.mma / commit.  This thread's per-stage instruction latency
      // bounds the shallow layers (16 one-position stages per tile on C = 64).
      tmem_alloc(tmem_holder, 512);
      tmem_relinquish();
      tc_fence_before();
      named_bar_sync(1, 32 + 32 * kEpiWarps);
      tc_fence_after();
      const uint32_t tmem_base = *tmem_holder;
      if (b_res) mbar_wait(b_full, 0);
      const uint32_t b_res_base = smem_u32(b_base);
      const uint32_t stage0 = smem_u32(stage_base);
      uint32_t sa0 = stage0;  // shared address of stage s
      int s = 0;
      uint32_t ph = 0;
      uint32_t grp = 0;
      int tr_m = 0;
      for (int w = blockIdx.x; w < num_work; w += gridDim.x) {
        const int j_lo = JS ? (w & 3) : 0, j_hi = JS ? j_lo + 1 : 4;
        for (int j = j_lo; j < j_hi; ++j, ++grp) {
          const uint32_t buf = grp % NB;
          mbar_wait(&acc_empty[buf], (grp / NB) & 1u);  // epilogue drained it
          if (lane == 0) trace_event(g.trace, 7, grp);
          tc_fence_after();
          const uint32_t d_base = tmem_base + buf * Cfg::kGroupCols;
          for (int a = 0; a < 4; ++a) {
            const int u0 = image_plane(4 * a + j) * nk;
            const uint32_t d_a = d_base + static_cast<uint32_t>(a * BN);
            for (int kc = 0; kc < nk; kc += U) {
              mbar_wait(&full_bar[s], ph);
              if (lane == 0) trace_event(g.trace, 1, tr_m);
              tc_fence_after();
              for (int u = 0; u < U; ++u) {
                const uint32_t sa = sa0 + u * Cfg::kABytes;
                const uint32_t sb = b_res ? b_res_base + (u0 + kc + u) * Cfg::kBBytes
                                          : sa0 + U * Cfg::kABytes + u * Cfg::kBBytes;
                const uint64_t adesc0 = umma_smem_desc(sa, 8 * BK, Cfg::kLayout);
                const uint64_t bdesc0 = umma_smem_desc(sb, 8 * BK, Cfg::kLayout);
#pragma unroll
                for (int kk = 0; kk < BK / 32; ++kk) {
                  if (kExpSwitches && (g.exp & 2)) break;
                  // +32 bytes along K = +2 in the descriptor's start-address field
                  if (elect_one())
                    umma_i8(d_a, adesc0 + 2 * kk, bdesc0 + 2 * kk, kIdesc, (kc + u > 0 || kk > 0) ? 1u : 0u);
                  __syncwarp();
                }
              }
              if (elect_one()) umma_commit(&empty_bar[s]);
              __syncwarp();
              if (lane == 0) trace_event(g.trace, 2, tr_m);
              ++tr_m;
              sa0 += stage_bytes;
              if (++s == stages) {
                s = 0;
                ph ^= 1u;
                sa0 = stage0;
              }
            }
          }
          if (elect_one()) umma_commit(&acc_full[buf]);
          __syncwarp();
        }
      }
    } else if (warp >= kRowSumWarp0 && g.rs_warps) {
      // ---------------- row sums (lowpgemm.hpp:121-123) ----------------
      // sum_c A[p][m][c] straight from every A stage: thread t owns rows t and
      // t + 64; 16-byte chunks are visited in a lane-rotated order (a row's
      // chunk order does not matter), which keeps the shared loads
      // conflict-free.  Ready per (tile, j-group) for the epilogue.
      constexpr int CPR = BK / 16;
      const int t = (warp - kRowSumWarp0) * 32 + lane;
      int s = 0;
      uint32_t ph = 0;
      uint32_t lt = 0;
      for (int t_i = blockIdx.x; t_i < num_tiles; t_i += gridDim.x, ++lt) {
        const int m0 = (t_i / nt) * kBM;
        const uint32_t tb = lt & 1u;
        mbar_wait(&rs_empty[tb], ((lt >> 1) & 1u) ^ 1u);  // epilogue done with this buffer
        int32_t* rs_t = s_rs + tb * 16 * kBM;
        for (int j = 0; j < 4; ++j) {
          for (int a = 0; a < 4; ++a) {
            const int p = 4 * a + j;
            uint32_t s0 = 0, s1 = 0;
            for (int kc = 0; kc < nk; ++kc) {
              mbar_wait(&full_bar[s], ph);
              const uint8_t* img = stage_base + static_cast<size_t>(s) * stage_bytes;
              const uint4* r0 = reinterpret_cast<const uint4*>(img + t * BK);
              const uint4* r1 = reinterpret_cast<const uint4*>(img + (t + 64) * BK);
#pragma unroll
              for (int c = 0; c < CPR; ++c) {
                const int cc = (c + lane) & (CPR - 1);
                const uint4 u = r0[cc], w = r1[cc];
                s0 = __dp4a(u.x, 0x01010101u, __dp4a(u.y, 0x01010101u, __dp4a(u.z, 0x01010101u, __dp4a(u.w, 0x01010101u, s0))));
                s1 = __dp4a(w.x, 0x01010101u, __dp4a(w.y, 0x01010101u, __dp4a(w.z, 0x01010101u, __dp4a(w.w, 0x01010101u, s1))));
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(&empty_bar[s]);
              if (++s == stages) {
                s = 0;
                ph ^= 1u;
              }
            }
            rs_t[p * kBM + t] = static_cast<int32_t>(s0);
            rs_t[p * kBM + t + 64] = static_cast<int32_t>(s1);
            if (DUMP) {
              if (m0 + t < g.M) rowsum_out[static_cast<long long>(p) * g.rs_pitch + m0 + t] = static_cast<int32_t>(s0);
              if (m0 + t + 64 < g.M)
                rowsum_out[static_cast<long long>(p) * g.rs_pitch + m0 + t + 64] = static_cast<int32_t>(s1);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&rs_ready[tb * 4 + j]);
        }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    setmaxnreg_inc<kEpiRegs>();
    const int ew = warp;
    const int q = warp & 3;          // TMEM lane quadrant this warp may access
    const int f0 = (ew >> 2) * FPT;  // this thread's filters within the tile
    const int row = q * 32 + lane;   // this thread's row (Winograd tile) within the tile
    named_bar_sync(1, 32 + 32 * kEpiWarps);
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const bool k4ok = (g.K & 3) == 0;
    // All j-group buffers start empty.
    if (lane == 0)
      for (int b = 0; b < NB; ++b) mbar_arrive(&acc_empty[b]);
    const bool fast = s_fast != 0;
    // Third affine term of a tile's filters, k3[p] * colsum[p][n0 + f]
    // (lowpgemm.hpp:110-114), into tile buffer b: 16 x BN values, 2 per thread.
    auto cterm_slice = [&](int t, uint32_t b) {
      const int n0 = (t % nt) * BN;
      for (int i = threadIdx.x; i < 16 * BN; i += 32 * kEpiWarps) {
        const int p = i / BN, kf = n0 + (i - p * BN);
        const float csum = (kf < g.K) ? static_cast<float>(__ldg(colsum + p * K_pad + kf)) : 0.0f;
        s_cterm[b * 16 * BN + i] = __fmul_rn(s_k3[p], csum);
      }
    };
    if (static_cast<int>(blockIdx.x) < num_work) cterm_slice(JS ? blockIdx.x >> 2 : blockIdx.x, 0);
    uint32_t grp = 0;
    uint32_t lt = 0;
    __shared__ int s_last;  // JS: this unit is its tile's last
    for (int w = blockIdx.x; w < num_work; w += gridDim.x, ++lt) {
      const int t = JS ? w >> 2 : w;
      // Slice lt is visible to every epilogue warp after this barrier, and
      // every warp is done with tile lt - 1, so its buffer takes tile lt + 1.
      named_bar_sync(6, 32 * kEpiWarps);
      if (w + static_cast<int>(gridDim.x) < num_work)
        cterm_slice(JS ? (w + gridDim.x) >> 2 : w + gridDim.x, (lt + 1) & 1u);
      const float* ct_tile = s_cterm + (lt & 1u) * 16 * BN;
      const int m0 = (t / nt) * kBM, n0 = (t % nt) * BN;
      const int m = m0 + row;
      const bool row_ok = m < g.M;
      const int kf0 = n0 + f0;
      // Output pixels of this lane's tile (2ti + a, 2tj + b) and their
      // validity (merge_tiles discards the ceil-overhang, tensor.hpp:172-175).
      int pix0, pmask, ppix;
      {
        const int mm = row_ok ? m : 0;
        const int img = mm / g.P;
        const int tt = mm - img * g.P;
        const int ti = tt / g.TW, tj = tt - ti * g.TW;
        pix0 = (img * g.OH + 2 * ti) * g.OW + 2 * tj;
        ppix = (img * (g.OH >> 1) + ti) * (g.OW >> 1) + tj;  // fused 2x2 max-pool output pixel
        const bool r1 = 2 * ti + 1 < g.OH, c1 = 2 * tj + 1 < g.OW;
        pmask = row_ok ? (1 | (c1 ? 2 : 0) | (r1 ? 4 : 0) | (r1 && c1 ? 8 : 0)) : 0;
      }
      // Output pixels (a = 0, b) and (a = 1, b) of the quadrant's 32 tiles:
      // each thread stages its FPT filters (bias / ReLU / +0 applied) into the
      // quadrant's swizzled buffer [64 segments = (tile, a)][BN filters], then
      // the quadrant's 4 warps write whole BN-filter segments (8 lanes per 128
      // bytes) instead of one scattered 16-byte piece per lane.
      auto store_col = [&](int b, float2 (&v0)[FPT / 2], float2 (&v1)[FPT / 2]) {
        constexpr int CPR = BN / 4;  // 16-byte chunks per segment
        float* stg = s_out + q * (64 * BN);
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          float2(&v)[FPT / 2] = a ? v1 : v0;
          if (bias != nullptr || relu) {  // fused epilogue (uniform branch)
#pragma unroll
            for (int i = 0; i < FPT / 2; ++i) {
              if (bias != nullptr)
                v[i] = add2(v[i], make_float2(kf0 + 2 * i < g.K ? __ldg(bias + kf0 + 2 * i) : 0.0f,
                                              kf0 + 2 * i + 1 < g.K ? __ldg(bias + kf0 + 2 * i + 1) : 0.0f));
              if (relu) {
                v[i].x = fmaxf(v[i].x, 0.0f);
                v[i].y = fmaxf(v[i].y, 0.0f);
              }
            }
          }
#pragma unroll
          for (int i = 0; i < FPT / 2; ++i) v[i] = add2(v[i], bcast2(0.0f));  // the reference never yields -0
          if (!STAGE) {  // straight from registers: this thread's FPT filters of pixel (a, b)
            if (!((pmask >> (2 * a + b)) & 1)) continue;
            float* d = y + static_cast<long long>(pix0 + a * g.OW + b) * g.K + kf0;
#pragma unroll
            for (int i = 0; i < FPT / 4; ++i) {
              const int kf = kf0 + 4 * i;
              if (k4ok && kf + 4 <= g.K) {
                *reinterpret_cast<float4*>(d + 4 * i) = make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
              } else {
                const float e4[4] = {v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (kf + e < g.K) d[4 * i + e] = e4[e];
              }
            }
            continue;
          }
          const int seg = 2 * lane + a;
#pragma unroll
          for (int i = 0; i < FPT / 4; ++i) {
            const int chunk = ((f0 >> 2) + i) ^ (lane & (CPR - 1));
            *reinterpret_cast<float4*>(stg + seg * BN + chunk * 4) =
                make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
          }
        }
        if (!STAGE) return;
        named_bar_sync(2 + q, 128);
        const int wq = ew >> 2;  // warp within the quadrant
        // Chunk id = wq * 32 + lane + 128 k: segment id / CPR, chunk id % CPR.
        const int cc = lane % CPR;
#pragma unroll
        for (int k = 0; k < (64 * CPR) / 128; ++k) {
          const int seg = (wq * 32 + lane + 128 * k) / CPR;
          const int tile = seg >> 1, a = seg & 1;
          const int tpix = __shfl_sync(0xffffffffu, pix0, tile);
          const int tmask = __shfl_sync(0xffffffffu, pmask, tile);
          const int kf = n0 + cc * 4;
          const float4 val = *reinterpret_cast<const float4*>(
              stg + seg * BN + ((cc ^ (tile & (CPR - 1))) * 4));
          if (!((tmask >> (2 * a + b)) & 1) || kf >= g.K) continue;
          float* d = y + static_cast<long long>(tpix + a * g.OW + b) * g.K + kf;
          if (k4ok && kf + 4 <= g.K) {
            *reinterpret_cast<float4*>(d) = val;
          } else {
            const float e4[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (kf + e < g.K) d[e] = e4[e];
          }
        }
        named_bar_sync(2 + q, 128);  // staging buffer free again
      };
      // Fused 2x2 / stride-2 max-pool (layer-stack option; floor pooling like
      // lance_maxpool2x2_nhwc): a tile's 4 output pixels are exactly one pool
      // window, so each thread folds its own S00, S01, S10, S11 -- after the
      // same bias / ReLU / +0 as the unpooled store -- in that kernel's order
      // max(max(y00, y01), max(y10, y11)) and writes one pooled pixel; tiles
      // that overhang the map (pmask != 15) have no pooled pixel.
      auto store_pool = [&](float2 (&s00)[FPT / 2], float2 (&s01)[FPT / 2], float2 (&s10)[FPT / 2],
                            float2 (&s11)[FPT / 2]) {
        if (pmask != 15) return;
        float* d = y + static_cast<long long>(ppix) * g.K + kf0;
        auto fin = [&](float2 v, int i) {
          if (bias != nullptr)
            v = add2(v, make_float2(kf0 + 2 * i < g.K ? __ldg(bias + kf0 + 2 * i) : 0.0f,
                                    kf0 + 2 * i + 1 < g.K ? __ldg(bias + kf0 + 2 * i + 1) : 0.0f));
          if (relu) {
            v.x = fmaxf(v.x, 0.0f);
            v.y = fmaxf(v.y, 0.0f);
          }
          return add2(v, bcast2(0.0f));
        };
#pragma unroll
        for (int i = 0; i < FPT / 2; i += 2) {
          float2 r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 a = fin(s00[i + h], i + h), b = fin(s01[i + h], i + h);
            const float2 c = fin(s10[i + h], i + h), e = fin(s11[i + h], i + h);
            r[h] = make_float2(fmaxf(fmaxf(a.x, b.x), fmaxf(c.x, e.x)), fmaxf(fmaxf(a.y, b.y), fmaxf(c.y, e.y)));
          }
          const int kf = kf0 + 2 * i;
          if (k4ok && kf + 4 <= g.K) {
            *reinterpret_cast<float4*>(d + 2 * i) = make_float4(r[0].x, r[0].y, r[1].x, r[1].y);
          } else {
            const float e4[4] = {r[0].x, r[0].y, r[1].x, r[1].y};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (kf + e < g.K) d[2 * i + e] = e4[e];
          }
        }
      };
      const uint32_t rb = lt & 1u;
      const int32_t* rs_tile = s_rs + rb * 16 * kBM + row;
      if constexpr (JS) {
        // ---- one j-group of the tile: T0j / T1j to the scratch, then the
        // tile's last unit folds all four and writes y.
        const int j = w & 3;
        const uint32_t buf = grp % NB;
        float rterm[4], k1s[4], k4[4];
        mbar_wait(&rs_ready[rb * 4], (lt >> 1) & 1u);
        if (ew == 0 && lane == 0) trace_event(g.trace, 6, grp);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          rterm[a] = __fmul_rn(s_k2[4 * a + j], static_cast<float>(rs_tile[(4 * a + j) * kBM]));
          k1s[a] = s_k1[4 * a + j];
          k4[a] = s_k4[4 * a + j];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rs_empty[rb]);
        mbar_wait(&acc_full[buf], (grp / NB) & 1u);
        if (ew == 0 && lane == 0) trace_event(g.trace, 3, grp);
        tc_fence_after();
        const uint32_t acc_addr = lane_base + buf * Cfg::kGroupCols + f0;
        // T scratch of this tile: [j][T0 / T1][BN / 4 filter quads][128 rows][4]
        // (a warp's 32 rows of one quad are 512 contiguous bytes).
        float* tsc = g.tscratch + static_cast<long long>(t) * 4 * 2 * kBM * BN;
        auto tptr = [&](int jj, int which, int quad) {
          return tsc + ((static_cast<long long>(jj * 2 + which) * (BN / 4) + quad) * kBM + row) * 4;
        };
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          uint32_t ac[4][4];
          tmem_ld_group4(acc_addr + 4 * c, BN, ac);
          tmem_ld_wait();
#pragma unroll
          for (int a = 0; a < 4; ++a) reg_fence(ac[a]);
          if (c == NCH - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
          }
          if (DUMP && row_ok) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (kf0 + 4 * c + i < g.K)
                  acc_dump[(static_cast<long long>(4 * a + j) * g.M + m) * g.K + kf0 + 4 * c + i] =
                      static_cast<int32_t>(ac[a][i]);
          }
          float2 T0[2], T1[2];
          affine_group4<BN>(ac, fast, k1s, k4, rterm, ct_tile + j * BN + f0 + 4 * c, T0, T1);
          __stcg(reinterpret_cast<float4*>(tptr(j, 0, f0 / 4 + c)), make_float4(T0[0].x, T0[0].y, T0[1].x, T0[1].y));
          __stcg(reinterpret_cast<float4*>(tptr(j, 1, f0 / 4 + c)), make_float4(T1[0].x, T1[0].y, T1[1].x, T1[1].y));
        }
        if (ew == 0 && lane == 0) trace_event(g.trace, 4, grp);
        ++grp;
        // Publish; the tile's fourth unit to arrive folds.
        __threadfence();
        named_bar_sync(7, 32 * kEpiWarps);
        if (threadIdx.x == 0) {
          const int old = atomicAdd(g.tticket + t, 1);
          s_last = old == 3;
          if (old == 3) g.tticket[t] = 0;  // reusable by the next launch
        }
        named_bar_sync(7, 32 * kEpiWarps);
        if (ew == 0 && lane == 0) trace_event(g.trace, 5, grp - 1);
#ifdef LANCE_GEMM_TRACE
        if (g.trace != nullptr && ew == 0 && lane == 0) g.trace[700000 + 4 * blockIdx.x + 2] = clock64();  // ticket done
#endif
        if (!s_last) continue;
#ifdef LANCE_GEMM_TRACE
        if (g.trace != nullptr && ew == 0 && lane == 0) g.trace[700000 + 4 * blockIdx.x] = clock64();  // fold start
#endif
        __threadfence();
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          float4 tv[4][2];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            tv[jj][0] = __ldcg(reinterpret_cast<const float4*>(tptr(jj, 0, f0 / 4 + c)));
            tv[jj][1] = __ldcg(reinterpret_cast<const float4*>(tptr(jj, 1, f0 / 4 + c)));
          }
          // pixel (a, b): S00, S10 (b = 0) and S01, S11 (b = 1), the fold of
          // the streaming path in the same order
          float2 px[4][2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            auto lo2 = [&](const float4& v) { return h ? make_float2(v.z, v.w) : make_float2(v.x, v.y); };
            const float2 t00 = lo2(tv[0][0]), t01 = lo2(tv[1][0]), t02 = lo2(tv[2][0]), t03 = lo2(tv[3][0]);
            const float2 t10 = lo2(tv[0][1]), t11 = lo2(tv[1][1]), t12 = lo2(tv[2][1]), t13 = lo2(tv[3][1]);
            px[0][h] = add2(add2(t00, t01), t02);  // S00: (a, b) = (0, 0)
            px[1][h] = add2(add2(t10, t11), t12);  // S10: (1, 0)
            px[2][h] = sub2(sub2(t01, t02), t03);  // S01: (0, 1)
            px[3][h] = sub2(sub2(t11, t12), t13);  // S11: (1, 1)
          }
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) {
            const int a = pp & 1, b = pp >> 1;
            if (!((pmask >> (2 * a + b)) & 1)) continue;
            const int kf = kf0 + 4 * c;
            float2 v[2] = {px[pp][0], px[pp][1]};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (bias != nullptr)
                v[h] = add2(v[h], make_float2(kf + 2 * h < g.K ? __ldg(bias + kf + 2 * h) : 0.0f,
                                              kf + 2 * h + 1 < g.K ? __ldg(bias + kf + 2 * h + 1) : 0.0f));
              if (relu) {
                v[h].x = fmaxf(v[h].x, 0.0f);
                v[h].y = fmaxf(v[h].y, 0.0f);
              }
              v[h] = add2(v[h], bcast2(0.0f));  // the reference never yields -0
            }
            float* d = y + static_cast<long long>(pix0 + a * g.OW + b) * g.K + kf;
            if (k4ok && kf + 4 <= g.K) {
              *reinterpret_cast<float4*>(d) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
            } else {
              const float e4[4] = {v[0].x, v[0].y, v[1].x, v[1].y};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (kf + e < g.K) d[e] = e4[e];
            }
          }
        }
#ifdef LANCE_GEMM_TRACE
        if (g.trace != nullptr && ew == 0 && lane == 0) g.trace[700000 + 4 * blockIdx.x + 1] = clock64();  // fold end
#endif
      } else {
      float2 S[4][FPT / 2];  // running S_ab partials, filter pairs
#pragma unroll
      for (int j = 0; j < 4; ++j, ++grp) {
        // Every tile has 4 j-groups and 4 % NB == 0, so the buffer is j % NB:
        // a compile-time constant once j is unrolled (TMEM / constant addresses
        // fold into immediates).  The phase parity still follows grp.
        static_assert(4 % NB == 0, "j-group buffers must divide the 4 j-groups of a tile");
        const uint32_t buf = static_cast<uint32_t>(j % NB);
        float rterm[4], k1s[4], k4[4];  // per position 4a + j of this j-group
        if (g.rs_warps || j == 0) mbar_wait(&rs_ready[rb * 4 + (g.rs_warps ? j : 0)], (lt >> 1) & 1u);
        if (ew == 0 && lane == 0) trace_event(g.trace, 6, grp);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          // k2[p] * float(sum_a): second term of affine_term
          rterm[a] = __fmul_rn(s_k2[4 * a + j], static_cast<float>(rs_tile[(4 * a + j) * kBM]));
          k1s[a] = s_k1[4 * a + j];
          k4[a] = s_k4[4 * a + j];
        }
        if (j == 3) {  // row sums of this tile fully read
          __syncwarp();
          if (lane == 0) mbar_arrive(&rs_empty[rb]);
        }
        mbar_wait(&acc_full[buf], (grp / NB) & 1u);
        if (ew == 0 && lane == 0) trace_event(g.trace, 3, grp);
        tc_fence_after();
        const uint32_t acc_addr = lane_base + buf * Cfg::kGroupCols + f0;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          uint32_t ac[4][4];
          tmem_ld_group4(acc_addr + 4 * c, BN, ac);
          tmem_ld_wait();
#pragma unroll
          for (int a = 0; a < 4; ++a) reg_fence(ac[a]);
          if (c == NCH - 1) {
            // Every accumulator of this warp is in registers: release the buffer.
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
            if (ew == 0 && lane == 0) trace_event(g.trace, 4, grp);
          }
          if (DUMP && row_ok) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (kf0 + 4 * c + i < g.K)
                  acc_dump[(static_cast<long long>(4 * a + j) * g.M + m) * g.K + kf0 + 4 * c + i] =
                      static_cast<int32_t>(ac[a][i]);
          }
          if (kExpSwitches && (g.exp & 1)) continue;
          float2 T0[2], T1[2];
          affine_group4<BN>(ac, fast, k1s, k4, rterm, ct_tile + j * BN + f0 + 4 * c, T0, T1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float2& s00 = S[0][2 * c + h];
            float2& s01 = S[1][2 * c + h];
            float2& s10 = S[2][2 * c + h];
            float2& s11 = S[3][2 * c + h];
            if (j == 0) {
              s00 = T0[h];
              s10 = T1[h];
            } else if (j == 1) {
              s00 = add2(s00, T0[h]);
              s01 = T0[h];
              s10 = add2(s10, T1[h]);
              s11 = T1[h];
            } else if (j == 2) {
              s00 = add2(s00, T0[h]);
              s01 = sub2(s01, T0[h]);
              s10 = add2(s10, T1[h]);
              s11 = sub2(s11, T1[h]);
            } else {
              s01 = sub2(s01, T0[h]);
              s11 = sub2(s11, T1[h]);
            }
          }
        }
        if (ew == 0 && lane == 0) trace_event(g.trace, 5, grp);
        if (kExpSwitches && (g.exp & 1)) continue;
        if (g.pool) {
          if (j == 3) store_pool(S[0], S[1], S[2], S[3]);
        } else if (j == 2) {
          store_col(0, S[0], S[2]);  // S00 and S10 are final after T_2
        } else if (j == 3) {
          store_col(1, S[1], S[3]);
        }
      }
      }  // !JS
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(*tmem_holder, 512);
  }
}

template <int BK, int BN, bool SMALL, bool DUMP, bool STAGE, bool JS>
static cudaError_t launch_gemm_t(const uint8_t* codes_a, const uint8_t* codes_w,
                                 const CUtensorMap* tmR, int32_t* rowsum_out, const int32_t* colsum,
                                 const LanceDevState* st, float* y, int32_t* acc_dump,
                                 const float* bias, int relu, const GemmGeom& g0, cudaStream_t s) {
  GemmGeom g = g0;
  const int nk = g.num_kchunks;
  // Resident B: one filter tile whose 16 positions x C_pad images fit in 64 KB.
  const int b_res = (g.num_n_tiles == 1 && 16 * nk * GemmCfg<BK, BN>::kBBytes <= 64 * 1024) ? 1 : 0;
  // Units per stage: g.units (0 = auto: 1) if it divides nk and leaves >= 3
  // stages; the row-sum warps read one image per stage, so U = 1 with them.
  int units = g.units > 0 ? g.units : 1;
  if (g.rs_warps || nk % units != 0 || gemm_smem_bytes<BK, BN>(3, nk, b_res, STAGE, units) > kSmemLimit)
    units = 1;
  int stages = 16;
  while (stages > 2 && gemm_smem_bytes<BK, BN>(stages, nk, b_res, STAGE, units) > kSmemLimit) --stages;
  const size_t smem = gemm_smem_bytes<BK, BN>(stages, nk, b_res, STAGE, units);
  if (smem > kSmemLimit) return cudaErrorInvalidValue;
  g.b_resident = b_res;
  g.stages = stages;
  g.units = units;
  const cudaError_t e =
      ensure_smem_attr(reinterpret_cast<const void*>(gemm_epilogue_kernel<BK, BN, SMALL, DUMP, STAGE, JS>), smem);
  if (e != cudaSuccess) return e;
  const int sms = current_sm_count();
  const long long tiles = ((static_cast<long long>(g.M) + kBM - 1) / kBM) * g.num_n_tiles * (JS ? 4 : 1);
  const int grid = static_cast<int>(tiles < sms ? tiles : sms);
  return launch_k(gemm_epilogue_kernel<BK, BN, SMALL, DUMP, STAGE, JS>, grid, kGemmThreadsP, smem, s, codes_a,
                  codes_w, *tmR, rowsum_out, colsum, st, y, acc_dump, bias, relu, g);
}

template <int BK, int BN, bool SMALL, bool DUMP>
static cudaError_t launch_gemm_s(const uint8_t* codes_a, const uint8_t* codes_w,
                                 const CUtensorMap* tmR, int32_t* rowsum_out, const int32_t* colsum,
                                 const LanceDevState* st, float* y, int32_t* acc_dump,
                                 const float* bias, int relu, const GemmGeom& g, cudaStream_t s) {
  if constexpr (BN == 64) {
    if (g.jsplit)  // y leaves from registers: no staging buffer, deeper operand stages
      return launch_gemm_t<BK, BN, SMALL, DUMP, false, true>(codes_a, codes_w, tmR, rowsum_out, colsum, st,
                                                             y, acc_dump, bias, relu, g, s);
    if (!g.stage_out)
      return launch_gemm_t<BK, BN, SMALL, DUMP, false, false>(codes_a, codes_w, tmR, rowsum_out, colsum, st,
                                                              y, acc_dump, bias, relu, g, s);
  }
  return launch_gemm_t<BK, BN, SMALL, DUMP, true, false>(codes_a, codes_w, tmR, rowsum_out, colsum, st, y,
                                                         acc_dump, bias, relu, g, s);
}

template <int BK, int BN>
static cudaError_t launch_gemm_bk(const uint8_t* codes_a, const uint8_t* codes_w, int small_acc,
                                  const CUtensorMap* tmR, int32_t* rowsum_out, const int32_t* colsum,
                                  const LanceDevState* st, float* y, int32_t* acc_dump,
                                  const float* bias, int relu, const GemmGeom& g, cudaStream_t s) {
  const bool dump = acc_dump != nullptr;
  if (small_acc)
    return dump ? launch_gemm_s<BK, BN, true, true>(codes_a, codes_w, tmR, rowsum_out, colsum, st, y, acc_dump,
                                                    bias, relu, g, s)
                : launch_gemm_s<BK, BN, true, false>(codes_a, codes_w, tmR, rowsum_out, colsum, st, y, acc_dump,
                                                     bias, relu, g, s);
  return dump ? launch_gemm_s<BK, BN, false, true>(codes_a, codes_w, tmR, rowsum_out, colsum, st, y, acc_dump,
                                                   bias, relu, g, s)
              : launch_gemm_s<BK, BN, false, false>(codes_a, codes_w, tmR, rowsum_out, colsum, st, y, acc_dump,
                                                    bias, relu, g, s);
}

cudaError_t launch_gemm(const uint8_t* codes_a, const uint8_t* codes_w, const CUtensorMap* tmR,
                        int32_t* rowsum_out,
                        int bk, int bn, int small_acc, const int32_t* colsum,
                        const LanceDevState* st, float* y, int32_t* acc_dump, const float* bias,
                        int relu, const GemmGeom& g, cudaStream_t s) {
#define LANCE_GEMM_CASE(BKV, BNV)                                                            \
  if (bk == BKV && bn == BNV)                                                                \
    return launch_gemm_bk<BKV, BNV>(codes_a, codes_w, small_acc, tmR, rowsum_out, colsum, st, y, acc_dump, \
                                    bias, relu, g, s);
  LANCE_GEMM_CASE(128, 64)
  LANCE_GEMM_CASE(64, 64)
  LANCE_GEMM_CASE(32, 64)
  LANCE_GEMM_CASE(128, 32)
  LANCE_GEMM_CASE(64, 32)
  LANCE_GEMM_CASE(32, 32)
  LANCE_GEMM_CASE(128, 16)
  LANCE_GEMM_CASE(64, 16)
  LANCE_GEMM_CASE(32, 16)
#undef LANCE_GEMM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace lance_dev
