// lance_band.cu -- input side of the LANCE path, v4 ("band" kernels).
//
//   K0 band_kernel<RANGE>  per-position (min, max) of v = B^T d B over the
//                          batch (quantize_domain PerPosition / PerTensor fit,
//                          engines.hpp:151-165, fit_params quant.hpp:54-72); the
//                          last CTA folds the partials into QuantParams[16].
//   K1 band_kernel<QUANT>  v recomputed and quantised (quant.hpp:77-84) into
//                          the A operand's UMMA images (lance_kernels.cuh),
//                          plus row sums [16][M] (lowpgemm.hpp:121-123).
//
// Work item = (image, channel band of chb channels, run of tile rows).  A CTA
// walks its tile rows top to bottom; the zero-padded input rows of the band
// (2*TW + 2 pixels from x = -pad, chb channels) arrive by 4-D TMA into a ring
// of shared-memory row slots -- the TMA's out-of-bounds zero fill is exactly
// extract_tiles' zero padding (tensor.hpp:141-147) -- and each row is loaded
// once per run (tile rows share two input rows).  Thread (tile tj, channel
// quad q) reads its 4 x 4 pixels with conflict-free 16-byte shared loads,
// transforms 4 channels with packed f32x2 adds in the reference order
// (column pass first, matrix.hpp:75-84) and, for K1, quantises them, packs
// the 4 codes of each position into one word and stages them in shared memory
// in the final UMMA-image byte order; one thread then writes each (position,
// k chunk) run of rows with a bulk copy.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lance_common.cuh"

namespace lance_dev {

constexpr int kBandThreads = 256;  // several CTAs per SM overlap their barrier phases
constexpr int kRangeMode = 0, kQuantMode = 1;

// ---------------------------------------------------------------- PTX bits
__device__ __forceinline__ void tma_load_4d(void* smem_dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(gdst)),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ float4 lds128(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

// ---------------------------------------------------------------- item decode
struct BandItem {
  int img, band, ti0, ti1, tj0, ntj;  // tile rows [ti0, ti1), tiles [tj0, tj0 + ntj)
};

__device__ __forceinline__ BandItem band_item(const BandGeom& b, const InGeom& g, long long it) {
  const int seg = static_cast<int>(it % b.nseg);
  long long r = it / b.nseg;
  const int cs = static_cast<int>(r % b.ncs);
  r /= b.ncs;
  const int band = static_cast<int>(r % b.nbc);
  const int img = static_cast<int>(r / b.nbc);
  const int ti0 = seg * b.trs;
  const int tj0 = cs * b.tws;
  return {img, band, ti0, min(ti0 + b.trs, g.TH), tj0, min(b.tws, g.TW - tj0)};
}

// Exact reference code for a value whose fast-path residual r flagged it as
// near a rounding boundary (see lance_input.cu exact_code_near_boundary).
__device__ __forceinline__ uint32_t band_exact_code(float d, float s, float gq, float r, float top) {
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

// Transform of one channel pair: d[a][b] (4 x 4 pixels) -> v (in place),
// column pass (over a) first, then the row pass (over b).
__device__ __forceinline__ void band_transform(float2 (&d)[4][4]) {
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const float2 d0 = d[0][b], d1 = d[1][b], d2 = d[2][b], d3 = d[3][b];
    d[0][b] = sub2(d0, d2);
    d[1][b] = add2(d1, d2);
    d[2][b] = sub2(d2, d1);
    d[3][b] = sub2(d1, d3);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float2 t0 = d[a][0], t1 = d[a][1], t2 = d[a][2], t3 = d[a][3];
    d[a][0] = sub2(t0, t2);
    d[a][1] = add2(t1, t2);
    d[a][2] = sub2(t2, t1);
    d[a][3] = sub2(t1, t3);
  }
}

// Profiling trace (built with -DLANCE_BAND_TRACE): CTA 0 clock64 stamps.
#ifdef LANCE_BAND_TRACE
__device__ unsigned long long g_band_trace[8 * 4096];
#endif
template <int MODE>
__device__ __forceinline__ void band_trace(int slot, int i) {
#ifdef LANCE_BAND_TRACE
  if (blockIdx.x == 0 && i < 4096) g_band_trace[(slot + 4 * MODE) * 4096 + i] = clock64();
#else
  (void)slot;
  (void)i;
#endif
}

// ---------------------------------------------------------------- kernel
// Warp-specialised: warps 0 .. NCW-1 compute (thread = tile x channel quad),
// the last warp's lane 0 streams input rows into the ring and writes staged
// codes back.  All hand-offs are mbarriers; there is no CTA-wide barrier in
// the loop:
//   row_full[slot]   TMA transaction barrier of a ring slot
//   stage_full[buf]  compute warps staged a tile row's codes (count NCW);
//                    also implies they are done with that tile row's rows
//   stage_empty[buf] the bulk stores of that staging buffer finished reading
template <int MODE, bool STATIC>
__global__ void __launch_bounds__(kBandThreads + 32, 2)
    band_kernel(const __grid_constant__ CUtensorMap tmX, uint8_t* __restrict__ codes,
                int32_t* __restrict__ rowsum, float* __restrict__ partials,
                LanceDevState* __restrict__ st, InGeom g, BandGeom b) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ float s_tmin[16], s_scale[16], s_rcp[16];
  __shared__ uint64_t row_full[16], stage_full[2], stage_empty[2], item_full[4], item_empty[4];
  __shared__ long long s_items[4];
  __shared__ float s_red[kBandThreads + 32];

  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* ring = reinterpret_cast<float*>(smem);                       // [ring][box_w][chb]
  uint8_t* stg = smem + static_cast<size_t>(b.ring) * b.slot_bytes;  // [2][16][nkb][tws][BK]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int QPT = b.chb >> 2;  // threads (channel quads) per tile
  constexpr int NCW = kBandThreads / 32;  // compute warps (all arrive on stage_full)
  const bool is_ctrl = warp == kBandThreads / 32;
  const int tj = tid / QPT, q = tid - tj * QPT;
  const int slot_floats = b.slot_bytes >> 2;

  if (tid < 16 && MODE == kQuantMode) {
    s_tmin[tid] = st->a_tmin[tid];
    s_scale[tid] = st->a_scale[tid];
    s_rcp[tid] = st->a_rcp[tid];
  }
  if (tid < (b.ring >> 1)) mbar_init(&row_full[tid], 1);
  if (tid < 2) {
    mbar_init(&stage_full[tid], NCW);
    mbar_init(&stage_empty[tid], 1);
  }
  if (tid < 4) {
    mbar_init(&item_full[tid], 1);
    mbar_init(&item_empty[tid], NCW);
  }
  fence_barrier_init();
  __syncthreads();
  const float top = static_cast<float>((1 << st->bits_i) - 1);

  float lo[16], hi[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }

  if (is_ctrl) {
    // ------------------------------------------------ loader / storer
    // Items are taken dynamically (one atomic counter per launch) and
    // published to the compute warps through a 4-slot item ring; row pairs are
    // streamed continuously across item boundaries (flat pair numbering).
    if (lane == 0) {
      const int npr = b.ring >> 1;  // pair slots
      struct QItem {
        BandItem it;
        int ntr;
        bool last;  // the sentinel
      };
      // Loader-private copies: the loader issues at most npr <= 8 pairs ahead
      // and every item has >= 2 pairs, so <= 5 items are in flight: 8 slots.
      QItem q[8];
      int k_pub = 0;                 // items published (incl. the final sentinel)
      bool exhausted = false;
      int ci_k = -1, ci_next = 0;    // item being issued (queue index), its next pair
      uint32_t flat_issued = 0;      // row pairs issued so far
      auto fetch_item = [&]() -> bool {
        const int slot = k_pub & 3;
        mbar_wait(&item_empty[slot], ((k_pub >> 2) & 1u) ^ 1u);
        long long idx = static_cast<long long>(atomicAdd(&st->band_ctr[MODE], 1u));
        if (idx >= b.items) idx = -1;
        s_items[slot] = idx;
        mbar_arrive(&item_full[slot]);
        QItem& qi = q[k_pub & 7];
        qi.last = idx < 0;
        if (idx < 0) {
          exhausted = true;
          ++k_pub;
          return false;
        }
        qi.it = band_item(b, g, idx);
        qi.ntr = qi.it.ti1 - qi.it.ti0;
        ci_k = k_pub++;
        ci_next = 0;
        return true;
      };
      auto issue_next_pair = [&]() -> bool {
        if (exhausted) return false;
        if (ci_k < 0 || ci_next == q[ci_k & 7].ntr + 1)
          if (!fetch_item()) return false;
        const BandItem& it = q[ci_k & 7].it;
        const int ps = static_cast<int>(flat_issued % npr);
        mbar_arrive_expect_tx(&row_full[ps], 2u * static_cast<uint32_t>(b.slot_bytes));
        for (int r = 0; r < 2; ++r)
          tma_load_4d(ring + static_cast<size_t>(2 * ps + r) * slot_floats, &tmX, it.band * b.chb,
                      2 * it.tj0 - g.pad, 2 * it.ti0 - g.pad + 2 * ci_next + r, it.img, &row_full[ps]);
        band_trace<MODE>(0, static_cast<int>(flat_issued));
        ++ci_next;
        ++flat_issued;
        return true;
      };
      while (flat_issued < static_cast<uint32_t>(npr) && issue_next_pair()) {
      }
      uint32_t freed = 0, iter = 0;
      for (int k_con = 0; k_con < k_pub; ++k_con) {
        if (q[k_con & 7].last) break;  // sentinel
        const BandItem it = q[k_con & 7].it;
        const int ntr = q[k_con & 7].ntr;
        for (int i = 0; i < ntr; ++i, ++iter) {
          const int ti = it.ti0 + i;
          const uint32_t buf = iter & 1u;
          mbar_wait(&stage_full[buf], (iter >> 1) & 1u);  // computed (and done reading rows)
          band_trace<MODE>(3, static_cast<int>(iter));
          if (MODE == kQuantMode) {
            // Codes: per (position plane, k chunk) the slice's ntj image rows
            // are contiguous in global memory, except across a 128-row edge.
            const uint8_t* sbuf = stg + buf * b.stg_bytes;
            const int m0 = (it.img * g.TH + ti) * g.TW + it.tj0;
            const int r0 = m0 & (kBM - 1);
            const int first = (kBM - r0) < it.ntj ? (kBM - r0) : it.ntj;
            const long long blk0 = m0 / kBM;
            for (int run = 0; run < 16 * b.nkb; ++run) {
              const int pj = run / b.nkb, kc = run - pj * b.nkb;
              const uint8_t* src = sbuf + run * b.run_bytes;
              const int kcg = kc + it.band * b.nkb;
              uint8_t* dst0 = codes + ((blk0 * 16 + pj) * g.a_nk + kcg) * static_cast<long long>(kBM * g.a_bk) +
                              r0 * g.a_bk;
              bulk_store(dst0, src, first * g.a_bk);
              if (first < it.ntj) {
                uint8_t* dst1 = codes + (((blk0 + 1) * 16 + pj) * g.a_nk + kcg) *
                                            static_cast<long long>(kBM * g.a_bk);
                bulk_store(dst1, src + first * g.a_bk, (it.ntj - first) * g.a_bk);
              }
            }
            bulk_commit();
            bulk_wait_read_all();  // this buffer may be refilled now
          }
          mbar_arrive(&stage_empty[buf]);
          // Tile row i frees pair i (and, being the item's last, pair i + 1).
          freed += (i == ntr - 1) ? 2u : 1u;
          while (flat_issued < freed + npr && issue_next_pair()) {
          }
        }
      }
      if (!exhausted) {  // publish the sentinel if the issue side never needed to
        while (issue_next_pair()) {
        }
      }
      if (MODE == kQuantMode) bulk_wait_all();
      // The last CTA to finish fetching resets the counter for the next launch.
      if (atomicAdd(&st->band_done[MODE], 1u) == gridDim.x - 1) {
        st->band_ctr[MODE] = 0u;
        st->band_done[MODE] = 0u;
        __threadfence();
      }
    }
  } else {
    // ------------------------------------------------ compute warps
    uint32_t kbase = 0, iter = 0;
    const int npr = b.ring >> 1;
    for (int k = 0;; ++k) {
      const int islot = k & 3;
      mbar_wait(&item_full[islot], (k >> 2) & 1u);
      const long long itn = s_items[islot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&item_empty[islot]);
      if (itn < 0) break;
      const BandItem it = band_item(b, g, itn);
      const int npairs = (it.ti1 - it.ti0) + 1;
      const int c0 = it.band * b.chb + 4 * q;  // this thread's first channel
      const bool active = tj < it.ntj;
      const bool cvalid = active && c0 < g.C;  // C % 4 == 0 on this path
      {
        const uint32_t kg = kbase;  // pair 0 of the item
        mbar_wait(&row_full[kg % npr], (kg / npr) & 1u);
      }
      for (int ti = it.ti0; ti < it.ti1; ++ti, ++iter) {
        const int i = ti - it.ti0;  // tile row i uses pairs i and i + 1
        const uint32_t kg1 = kbase + i + 1;
        mbar_wait(&row_full[kg1 % npr], (kg1 / npr) & 1u);
        if (tid == 0) band_trace<MODE>(1, static_cast<int>(kg1));
        float2 dA[4][4], dB[4][4];  // channels (c0, c0+1) and (c0+2, c0+3)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int slot = static_cast<int>((2 * ((kbase + i + (a >> 1)) % npr)) + (a & 1));
          const float* row = ring + static_cast<size_t>(slot) * slot_floats + (2 * tj) * b.chb + 4 * q;
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (active) v = lds128(row + bb * b.chb);
            dA[a][bb] = make_float2(v.x, v.y);
            dB[a][bb] = make_float2(v.z, v.w);
          }
        }
        band_transform(dA);
        band_transform(dB);
        const uint32_t buf = iter & 1u;
        // Both modes: at most two tile rows ahead of the loader, so the
        // stage_full phases it waits for can never alias.
        mbar_wait(&stage_empty[buf], ((iter >> 1) & 1u) ^ 1u);
        if (MODE == kRangeMode) {
          if (cvalid) {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int bb = 0; bb < 4; ++bb) {
                const int p = 4 * a + bb;
                lo[p] = fmin3_nan(fmin3_nan(lo[p], dA[a][bb].x, dA[a][bb].y), dB[a][bb].x, dB[a][bb].y);
                hi[p] = fmax3_nan(fmax3_nan(hi[p], dA[a][bb].x, dA[a][bb].y), dB[a][bb].x, dB[a][bb].y);
              }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&stage_full[buf]);  // rows of this tile row consumed
          if (tid == 0) band_trace<MODE>(2, static_cast<int>(iter));
        } else {
          // ---- quantise (quant.hpp:77-84) into the staging buffer ----
          uint8_t* sbuf = stg + buf * b.stg_bytes;
          const int m = (it.img * g.TH + ti) * g.TW + it.tj0 + tj;
          // Byte offset of (row m, channels c0..c0+3) inside a staged run of
          // the slice's image rows: row tj, 16-byte chunk swizzled with the
          // row's index inside its 128-row image (umma_swizzle keeps the row).
          const int rg = m & (kBM - 1);
          const int cb = (4 * q) & (g.a_bk - 1);
          const int stg_off = (4 * q / g.a_bk) * b.run_bytes + tj * g.a_bk +
                              static_cast<int>(umma_swizzle(static_cast<uint32_t>(rg * g.a_bk + cb), g.a_bk)) -
                              rg * g.a_bk;
          uint32_t* sdst = reinterpret_cast<uint32_t*>(sbuf + stg_off);
          const int pstride_w = (b.nkb * b.run_bytes) >> 2;  // one position plane, in words
          uint32_t rs_mine = 0;  // row sum of position (lane & 15), see below
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
              const int p = 4 * a + bb;
              const float tmin = s_tmin[p], rcp = s_rcp[p];
              const float2 v2[2] = {dA[a][bb], dB[a][bb]};
              float2 dd[2], gq[2], r[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                dd[h] = sub2(v2[h], bcast2(tmin));
                if (STATIC) {
                  float2 qq = mul2_rn(dd[h], bcast2(rcp));
                  qq.x = fminf(fmaxf(qq.x, 0.0f), top);  // NaN -> 0 like quant.hpp:81
                  qq.y = fminf(fmaxf(qq.y, 0.0f), top);
                  gq[h] = add2(qq, bcast2(kMagic));
                  r[h] = sub2(qq, sub2(gq[h], bcast2(kMagic)));
                } else {
                  // n = rint(d * rcp) via the magic addend, r = d * rcp - n
                  // exactly (one rounding); see input_quant_kernel.
                  gq[h] = fma2(dd[h], bcast2(rcp), bcast2(kMagic));
                  r[h] = fma2(dd[h], bcast2(rcp), sub2(bcast2(kMagic), gq[h]));
                }
              }
              const uint32_t w01 = __byte_perm(__float_as_uint(gq[0].x), __float_as_uint(gq[0].y), 0x0040);
              const uint32_t w23 = __byte_perm(__float_as_uint(gq[1].x), __float_as_uint(gq[1].y), 0x0040);
              uint32_t word = __byte_perm(w01, w23, 0x5410);
              const float rmax = fmax3_nan(fmax3_nan(fabsf(r[0].x), fabsf(r[0].y), fabsf(r[1].x)),
                                           fabsf(r[1].y), 0.0f);
              if (__builtin_expect(!(rmax < kTieGuard), 0)) {
                // Rare (~1e-4 per value): re-derive the 4 codes exactly.
                const float sc = s_scale[p];
                const float vv[4] = {v2[0].x, v2[0].y, v2[1].x, v2[1].y};
                const float dv[4] = {dd[0].x, dd[0].y, dd[1].x, dd[1].y};
                const float gv[4] = {gq[0].x, gq[0].y, gq[1].x, gq[1].y};
                const float rv[4] = {r[0].x, r[0].y, r[1].x, r[1].y};
                word = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  uint32_t c;
                  if (STATIC)
                    c = quantize_code(vv[e], tmin, sc, top);
                  else
                    c = (fabsf(rv[e]) < kTieGuard) ? (__float_as_uint(gv[e]) & 0xFFu)
                                                   : band_exact_code(dv[e], sc, gv[e], rv[e], top);
                  word |= c << (8 * e);
                }
              }
              word = cvalid ? word : 0u;
              if (active) sdst[image_plane(p) * pstride_w] = word;
              // Row sums (lowpgemm.hpp:121-123): the thread's 4 codes, then one
              // warp reduction; at QPT = 16 a warp holds two tiles (16-bit halves).
              uint32_t part = __dp4a(word, 0x01010101u, 0u);
              if (QPT == 16) part <<= 16 * ((lane >> 4) & 1);
              const uint32_t tot = __reduce_add_sync(0xffffffffu, part);
              if ((lane & 15) == p) rs_mine = tot;
            }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&stage_full[buf]);
          // Lane l writes the row sum of position l & 15 for its tile.
          {
            const int half = (lane >> 4) & 1;
            uint32_t val;
            int tl;
            if (QPT == 16) {
              val = (rs_mine >> (16 * half)) & 0xFFFFu;
              tl = (warp * 32 + half * 16) / QPT;
            } else {
              val = rs_mine;
              tl = (warp * 32) / QPT;
            }
            const bool writer = (QPT == 16) || lane < 16;
            if (writer && tl < it.ntj) {
              const int mm = (it.img * g.TH + ti) * g.TW + it.tj0 + tl;
              int32_t* dst = rowsum + static_cast<long long>(lane & 15) * g.rs_pitch + mm;
              if (b.nbc == 1 && QPT <= 32)
                *dst = static_cast<int32_t>(val);
              else
                atomicAdd(dst, static_cast<int32_t>(val));
            }
          }
        }
      }
      kbase += npairs;
    }
  }

  if (MODE == kRangeMode) {
    if (block_minmax_and_ticket(lo, hi, partials, &st->ticket_in, s_red)) {
      fit_from_ranges(s_red, g.granularity, st->bits_i, st->a_tmin, st->a_tmax, st->a_scale,
                      st->a_rcp, &st->nan_in);
      __syncthreads();
      make_epilogue_consts(st, g.C);
    }
  }
}

size_t band_smem_bytes(const BandGeom& b, int mode) {
  return 128 + static_cast<size_t>(b.ring) * b.slot_bytes +
         (mode == kQuantMode ? 2 * static_cast<size_t>(b.stg_bytes) : 0);
}

cudaError_t launch_band(const CUtensorMap* tmX, uint8_t* codes, int32_t* rowsum, float* partials,
                        LanceDevState* st, const InGeom& g, const BandGeom& b, int mode,
                        int static_mode, cudaStream_t s) {
  const size_t smem = band_smem_bytes(b, mode);
  static size_t configured[4] = {};
  auto fn = mode == kRangeMode ? band_kernel<kRangeMode, false>
                               : (static_mode ? band_kernel<kQuantMode, true> : band_kernel<kQuantMode, false>);
  const int fi = mode == kRangeMode ? 0 : (static_mode ? 1 : 2);
  if (configured[fi] < smem) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured[fi] = smem;
  }
  fn<<<b.grid, kBandThreads + 32, smem, s>>>(*tmX, codes, rowsum, partials, st, g, b);
  return cudaGetLastError();
}

}  // namespace lance_dev

#ifdef LANCE_BAND_TRACE
extern "C" __attribute__((visibility("default"))) int lance_debug_band_trace(void* host, size_t bytes) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, lance_dev::g_band_trace, bytes));
}
#endif
