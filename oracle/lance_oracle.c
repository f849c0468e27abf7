/*
 * oracle/lance_oracle.c -- TEST INFRASTRUCTURE ONLY (see lance_oracle.h).
 *
 * A plain-C restatement of the reference `lance_gemm` path.  Every function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/include/lance/).  Floating-point operations are issued
 * in the reference's order: the 4x4 transforms use the i-k-j `matmul`
 * accumulation from +0.0f of matrix.hpp:75-84, including the products with
 * zero basis entries, so the oracle reproduces the reference bitwise even for
 * signed zeros.  Build with -ffp-contract=off (oracle/Makefile): FMA
 * contraction would change the affine epilogue.
 */
#include "lance_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* lo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* rng.hpp:27-47.  std::mt19937_64 parameters (w=64, n=312, m=156, r=31).    */

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  static const uint64_t A = 0xB5026F5AA96619E9ULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= A;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* UniformSource::next (rng.hpp:31-34) */
void lo_uniform_fill(uint64_t seed, float* out, size_t count) {
  mt64* s = (mt64*)malloc(sizeof(mt64));
  mt64_seed(s, seed);
  for (size_t i = 0; i < count; ++i) {
    uint32_t top = (uint32_t)(mt64_next(s) >> 40);
    out[i] = (float)top * (1.0f / 8388608.0f) - 1.0f;
  }
  free(s);
}

/* ------------------------------------------------------------------------ */
/* engines.hpp:40-44 */
int lo_out_h(const lo_spec* s) { return s->h + 2 * s->pad - 3 + 1; }
int lo_out_w(const lo_spec* s) { return s->w + 2 * s->pad - 3 + 1; }
int lo_tiles_h(const lo_spec* s) { return (lo_out_h(s) + 1) / 2; }
int lo_tiles_w(const lo_spec* s) { return (lo_out_w(s) + 1) / 2; }
/* extract_tiles grid for tile side m (tensor.hpp:130-131). */
int lo_tiles_h_m(const lo_spec* s, int m) { return (lo_out_h(s) + m - 1) / m; }
int lo_tiles_w_m(const lo_spec* s, int m) { return (lo_out_w(s) + m - 1) / m; }

/* ------------------------------------------------------------------------ */
/* winograd.hpp:40-54: F(2x2,3x3) basis. */
static const float kG[4][3] = {{1.0f, 0.0f, 0.0f},
                               {0.5f, 0.5f, 0.5f},
                               {0.5f, -0.5f, 0.5f},
                               {0.0f, 0.0f, 1.0f}};
static const float kBt[4][4] = {{1.0f, 0.0f, -1.0f, 0.0f},
                                {0.0f, 1.0f, 1.0f, 0.0f},
                                {0.0f, -1.0f, 1.0f, 0.0f},
                                {0.0f, 1.0f, 0.0f, -1.0f}};
static const float kAt[2][4] = {{1.0f, 1.0f, 1.0f, 0.0f},
                                {0.0f, 1.0f, -1.0f, -1.0f}};

/* F(4x4,3x3): not in the reference (winograd.hpp:27 "Only F(2x2, 3x3) is
 * provided").  Builder-defined basis (Lavin & Gray),
 * evaluated through the same matmul/two_sided conventions as the reference's
 * F(2x2) basis; every entry is the fp32 value of the literal (1/6, 1/12, 1/24
 * rounded to nearest).  Parity of this extension is self-pinned (correlation
 * identity vs direct_conv, tests/test_f4.py). */
static const float kG4[6][3] = {{0.25f, 0.0f, 0.0f},
                                {-1.0f / 6.0f, -1.0f / 6.0f, -1.0f / 6.0f},
                                {-1.0f / 6.0f, 1.0f / 6.0f, -1.0f / 6.0f},
                                {1.0f / 24.0f, 1.0f / 12.0f, 1.0f / 6.0f},
                                {1.0f / 24.0f, -1.0f / 12.0f, 1.0f / 6.0f},
                                {0.0f, 0.0f, 1.0f}};
static const float kBt4[6][6] = {{4.0f, 0.0f, -5.0f, 0.0f, 1.0f, 0.0f},
                                 {0.0f, -4.0f, -4.0f, 1.0f, 1.0f, 0.0f},
                                 {0.0f, 4.0f, -4.0f, -1.0f, 1.0f, 0.0f},
                                 {0.0f, -2.0f, -1.0f, 2.0f, 1.0f, 0.0f},
                                 {0.0f, 2.0f, -1.0f, -2.0f, 1.0f, 0.0f},
                                 {0.0f, 4.0f, 0.0f, -5.0f, 0.0f, 1.0f}};
static const float kAt4[4][6] = {{1.0f, 1.0f, 1.0f, 1.0f, 1.0f, 0.0f},
                                 {0.0f, 1.0f, -1.0f, 2.0f, -2.0f, 0.0f},
                                 {0.0f, 1.0f, 1.0f, 4.0f, 4.0f, 0.0f},
                                 {0.0f, 1.0f, -1.0f, 8.0f, -8.0f, 1.0f}};

/* WinogradBasis (winograd.hpp:30-37) for m = 2 or 4. */
typedef struct {
  int m, alpha;
  const float *g, *bt, *at;
} lo_basis;

static lo_basis basis_for(int m) {
  lo_basis b;
  b.m = m;
  b.alpha = m + 2;
  b.g = (m == 4) ? &kG4[0][0] : &kG[0][0];
  b.bt = (m == 4) ? &kBt4[0][0] : &kBt[0][0];
  b.at = (m == 4) ? &kAt4[0][0] : &kAt[0][0];
  return b;
}

/* matrix.hpp:75-84: out = a*b, i-k-j order, accumulate from +0.0f. */
static void matmul(const float* a, int ar, int ac, const float* b, int bc, float* out) {
  for (int i = 0; i < ar * bc; ++i) out[i] = 0.0f;
  for (int i = 0; i < ar; ++i)
    for (int k = 0; k < ac; ++k) {
      const float av = a[i * ac + k];
      for (int j = 0; j < bc; ++j) out[i * bc + j] += av * b[k * bc + j];
    }
}

/* matrix.hpp:86-91 */
static void transpose(const float* a, int r, int c, float* out) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) out[j * r + i] = a[i * c + j];
}

/* winograd.hpp:59-61: two_sided(t, x) = (t x) t^T. t is tr x tc, x tc x tc. */
static void two_sided(const float* t, int tr, int tc, const float* x, float* out) {
  float tx[36], tt[36];
  matmul(t, tr, tc, x, tc, tx);
  transpose(t, tr, tc, tt);
  matmul(tx, tr, tc, tt, tr, out);
}

/* winograd.hpp:66-70 */
void lo_transform_input(const float d[16], float v[16]) { two_sided(&kBt[0][0], 4, 4, d, v); }
/* winograd.hpp:73-77 */
void lo_transform_filter(const float g[9], float u[16]) { two_sided(&kG[0][0], 4, 3, g, u); }
/* winograd.hpp:80-84 */
void lo_transform_output(const float m[16], float s[4]) { two_sided(&kAt[0][0], 2, 4, m, s); }
/* The same three transforms for F(4x4,3x3) (Appendix D basis). */
void lo_transform_input4(const float d[36], float v[36]) { two_sided(&kBt4[0][0], 6, 6, d, v); }
void lo_transform_filter4(const float g[9], float u[36]) { two_sided(&kG4[0][0], 6, 3, g, u); }
void lo_transform_output4(const float m[36], float s[16]) { two_sided(&kAt4[0][0], 4, 6, m, s); }

/* ------------------------------------------------------------------------ */
/* quant.hpp:54-72 */
int lo_fit_params(const float* values, size_t count, int bits, lo_qparams* out) {
  if (bits < 2 || bits > 8) return fail(LO_EINVAL, "fit_params: bits must be in [2, 8]");
  if (count == 0) return fail(LO_EINVAL, "fit_params: empty value set");
  float lo = values[0], hi = values[0];
  for (size_t i = 0; i < count; ++i) {
    const float v = values[i];
    if (isnan(v)) return fail(LO_ENAN, "fit_params: NaN in values");
    if (v < lo) lo = v;
    if (v > hi) hi = v;
  }
  out->bits = bits;
  out->t_min = lo;
  out->t_max = hi;
  out->scale = (hi - lo) / (float)((1 << bits) - 1);
  return LO_OK;
}

/* quant.hpp:77-84 (round = half away from zero) */
uint8_t lo_quantize(float x, const lo_qparams* p) {
  if (p->scale == 0.0f) return 0;
  const float units = roundf((x - p->t_min) / p->scale);
  const float top = (float)((1 << p->bits) - 1);
  if (!(units > 0.0f)) return 0;
  if (units >= top) return (uint8_t)top;
  return (uint8_t)units;
}

/* quant.hpp:86-91 */
float lo_dequantize(uint8_t code, const lo_qparams* p) {
  if (p->scale == 0.0f) return p->t_min;
  return (float)code * p->scale + p->t_min;
}

/* lowpgemm.hpp:110-114: left-to-right, every product rounded. */
float lo_affine_term(int32_t dot, int32_t a_sum, int32_t b_sum, int depth,
                     const lo_qparams* pa, const lo_qparams* pb) {
  return pa->scale * pb->scale * (float)dot + pa->scale * pb->t_min * (float)a_sum +
         pb->scale * pa->t_min * (float)b_sum + (float)depth * pa->t_min * pb->t_min;
}

/* ------------------------------------------------------------------------ */
/* engines.hpp:46-53 (ConvSpec::validate), 66-79 (LanceConfig::validate),
 * 496-499 (lance_gemm mode / depth checks), lowpgemm.hpp:28 (depth bound). */
int lo_validate(const lo_spec* s, int bits_w, int bits_i, int gran, int mode_gemm) {
  if (s->n < 1 || s->c < 1 || s->h < 1 || s->w < 1 || s->k < 1)
    return fail(LO_EINVAL, "ConvSpec: all dims must be >= 1");
  if (s->pad != 0 && s->pad != 1) return fail(LO_EINVAL, "ConvSpec: pad must be 0 or 1");
  if (lo_out_h(s) < 1 || lo_out_w(s) < 1)
    return fail(LO_EINVAL, "ConvSpec: output dims collapse to zero");
#define LO_BITS_OK(b) (((b) >= 2 && (b) <= 8) || (b) == 32)
  if (!LO_BITS_OK(bits_w) || !LO_BITS_OK(bits_i))
    return fail(LO_EINVAL, "LanceConfig: bits must be in [2, 8] or 32");
  if (mode_gemm) {
    if (gran == LO_PER_TILE)
      return fail(LO_EINVAL,
                  "LanceConfig: Gemm mode cannot use PerTile granularity; integer "
                  "accumulation across channels needs one scale per position");
    if (bits_w == 32 || bits_i == 32)
      return fail(LO_EINVAL, "LanceConfig: Gemm mode requires quantized operands (bits <= 8)");
  } else {
    return fail(LO_EINVAL, "lance_gemm: cfg.mode must be Gemm");
  }
  if (s->c > 32768) return fail(LO_EINVAL, "lance_gemm: channel count exceeds GEMM depth bound");
  return LO_OK;
}

/* ------------------------------------------------------------------------ */
/* quantize_domain (engines.hpp:140-183) for the PerPosition / PerTensor
 * cases lance_gemm admits.  values = [16][slice]. */
static int quantize_domain(const float* values, size_t slice, int np, int bits, int gran,
                           uint8_t* codes, lo_qparams* params) {
  int rc;
  if (gran == LO_PER_TENSOR) {
    rc = lo_fit_params(values, np * slice, bits, &params[0]);
    if (rc) return rc;
    for (int p = 1; p < np; ++p) params[p] = params[0]; /* param_at -> params[0] (:135) */
    for (size_t i = 0; i < np * slice; ++i) codes[i] = lo_quantize(values[i], &params[0]);
    return LO_OK;
  }
  for (int p = 0; p < np; ++p) {
    rc = lo_fit_params(values + (size_t)p * slice, slice, bits, &params[p]);
    if (rc) return rc;
    for (size_t i = 0; i < slice; ++i)
      codes[(size_t)p * slice + i] = lo_quantize(values[(size_t)p * slice + i], &params[p]);
  }
  return LO_OK;
}

/* lance_gemm (engines.hpp:492-536) for tile side m (2: the reference path;
 * 4: the F(4x4,3x3) extension, same algorithm with alpha = 6, 36 positions).
 * Every "16" / "2" / "4" literal of engines.hpp:240-255,510,531-532 and
 * extract_tiles (tensor.hpp:116-152) becomes np = alpha^2 / m / alpha. */
int lo_lance_gemm_tiled(const lo_spec* s, int tile_m, int bits_w, int bits_i, int gran,
                        const float* x, const float* w, float* y, const lo_qparams* in_params,
                        lo_dump* dump) {
  if (tile_m != 2 && tile_m != 4) return fail(LO_EINVAL, "lance_gemm: tile side must be 2 or 4");
  int rc = lo_validate(s, bits_w, bits_i, gran, 1);
  if (rc) return rc;
  const lo_basis bs = basis_for(tile_m);
  const int tm = bs.m, al = bs.alpha, np = al * al;
  const int N = s->n, C = s->c, H = s->h, W = s->w, K = s->k, pad = s->pad;
  const int OH = lo_out_h(s), OW = lo_out_w(s), PH = lo_tiles_h_m(s, tm), PW = lo_tiles_w_m(s, tm);
  const size_t P = (size_t)PH * PW, M = (size_t)N * P;

  float* v = (float*)malloc(sizeof(float) * np * M * C);
  float* u = (float*)malloc(sizeof(float) * np * (size_t)C * K);
  uint8_t* va = (uint8_t*)malloc(np * M * C);
  uint8_t* ub = (uint8_t*)malloc(np * (size_t)C * K);
  int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * M * K);
  float* mdom = (float*)malloc(sizeof(float) * np * M * K);
  int32_t* rsum = (int32_t*)malloc(sizeof(int32_t) * np * M);
  int32_t* csum = (int32_t*)malloc(sizeof(int32_t) * np * (size_t)K);
  lo_qparams pa[36], pb[36];
  if (!v || !u || !va || !ub || !acc || !mdom || !rsum || !csum) {
    rc = fail(LO_EINVAL, "oracle: out of memory");
    goto done;
  }

  /* extract_tiles (tensor.hpp:116-152) + domain_from_tiles (engines.hpp:189-211):
   * tile t = ti*PW + tj, row = img*P + t, origin (m*ti - pad, m*tj - pad), zero
   * padding, v[p][row][ch] with p = alpha*a + b. */
  for (int img = 0; img < N; ++img)
    for (int ti = 0; ti < PH; ++ti)
      for (int tj = 0; tj < PW; ++tj) {
        const size_t row = (size_t)img * P + (size_t)ti * PW + tj;
        for (int ch = 0; ch < C; ++ch) {
          float d[36], vv[36];
          for (int a = 0; a < al; ++a)
            for (int b = 0; b < al; ++b) {
              const int si = ti * tm - pad + a, sj = tj * tm - pad + b;
              d[a * al + b] = (si >= 0 && si < H && sj >= 0 && sj < W)
                                  ? x[(((size_t)img * H + si) * W + sj) * C + ch]
                                  : 0.0f;
            }
          two_sided(bs.bt, al, al, d, vv);
          for (int p = 0; p < np; ++p) v[((size_t)p * M + row) * C + ch] = vv[p];
        }
      }

  /* domain_from_filters (engines.hpp:215-233): g[a][b] = w.at(k,a,b,c), u[p][c][k]. */
  for (int ki = 0; ki < K; ++ki)
    for (int ci = 0; ci < C; ++ci) {
      float g[9], uu[36];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g[a * 3 + b] = w[(((size_t)ki * 3 + a) * 3 + b) * C + ci];
      two_sided(bs.g, al, 3, g, uu);
      for (int p = 0; p < np; ++p) u[((size_t)p * C + ci) * K + ki] = uu[p];
    }

  /* quantize_domain for v and u (engines.hpp:505-506). */
  if (in_params) {
    for (int p = 0; p < np; ++p) pa[p] = in_params[p];
    for (int p = 0; p < np; ++p)
      for (size_t i = 0; i < M * C; ++i) {
        const size_t idx = (size_t)p * M * C + i;
        va[idx] = lo_quantize(v[idx], &pa[p]);
      }
  } else {
    rc = quantize_domain(v, M * C, np, bits_i, gran, va, pa);
    if (rc) goto done;
  }
  rc = quantize_domain(u, (size_t)C * K, np, bits_w, gran, ub, pb);
  if (rc) goto done;

  /* np x affine_gemm (engines.hpp:510-525; lowpgemm.hpp:118-134). */
  for (int p = 0; p < np; ++p) {
    const uint8_t* A = va + (size_t)p * M * C;
    const uint8_t* B = ub + (size_t)p * C * K;
    memset(acc, 0, sizeof(int32_t) * M * K);
    for (size_t i = 0; i < M; ++i) { /* gemm_codes i-k-j (lowpgemm.hpp:87-97) */
      int32_t* orow = acc + i * K;
      for (int kk = 0; kk < C; ++kk) {
        const int32_t av = A[i * C + kk];
        const uint8_t* brow = B + (size_t)kk * K;
        for (int j = 0; j < K; ++j) orow[j] += av * (int32_t)brow[j];
      }
    }
    for (size_t i = 0; i < M; ++i) { /* a_row_sum (lowpgemm.hpp:121-123) */
      int32_t sum = 0;
      for (int kk = 0; kk < C; ++kk) sum += A[i * C + kk];
      rsum[(size_t)p * M + i] = sum;
    }
    for (int j = 0; j < K; ++j) { /* b_col_sum (lowpgemm.hpp:124-126) */
      int32_t sum = 0;
      for (int kk = 0; kk < C; ++kk) sum += B[(size_t)kk * K + j];
      csum[(size_t)p * K + j] = sum;
    }
    for (size_t i = 0; i < M; ++i) /* affine_term (lowpgemm.hpp:128-133) */
      for (int j = 0; j < K; ++j)
        mdom[((size_t)p * M + i) * K + j] =
            lo_affine_term(acc[i * K + j], rsum[(size_t)p * M + i], csum[(size_t)p * K + j],
                           C, &pa[p], &pb[p]);
    if (dump && dump->acc) memcpy(dump->acc + (size_t)p * M * K, acc, sizeof(int32_t) * M * K);
  }

  /* emit_output_tile + merge_tiles (engines.hpp:527-535, 247-256; tensor.hpp:157-182). */
  for (size_t row = 0; row < M; ++row) {
    const int img = (int)(row / P), t = (int)(row % P), ti = t / PW, tj = t % PW;
    for (int ki = 0; ki < K; ++ki) {
      float m[36], s2[16];
      for (int p = 0; p < np; ++p) m[p] = mdom[((size_t)p * M + row) * K + ki];
      two_sided(bs.at, tm, al, m, s2);
      for (int a = 0; a < tm; ++a) {
        const int oi = ti * tm + a;
        if (oi >= OH) break;
        for (int b = 0; b < tm; ++b) {
          const int oj = tj * tm + b;
          if (oj >= OW) break;
          y[(((size_t)img * OH + oi) * OW + oj) * K + ki] = s2[a * tm + b];
        }
      }
    }
  }

  if (dump) {
    if (dump->v) memcpy(dump->v, v, sizeof(float) * np * M * C);
    if (dump->u) memcpy(dump->u, u, sizeof(float) * np * (size_t)C * K);
    if (dump->codes_a) memcpy(dump->codes_a, va, np * M * C);
    if (dump->codes_w) memcpy(dump->codes_w, ub, np * (size_t)C * K);
    if (dump->rowsum) memcpy(dump->rowsum, rsum, sizeof(int32_t) * np * M);
    if (dump->colsum) memcpy(dump->colsum, csum, sizeof(int32_t) * np * (size_t)K);
    if (dump->params_a) memcpy(dump->params_a, pa, sizeof(lo_qparams) * np);
    if (dump->params_w) memcpy(dump->params_w, pb, sizeof(lo_qparams) * np);
  }
  rc = LO_OK;
done:
  free(v);
  free(u);
  free(va);
  free(ub);
  free(acc);
  free(mdom);
  free(rsum);
  free(csum);
  return rc;
}

int lo_lance_gemm(const lo_spec* s, int bits_w, int bits_i, int gran, const float* x,
                  const float* w, float* y, const lo_qparams* in_params, lo_dump* dump) {
  return lo_lance_gemm_tiled(s, 2, bits_w, bits_i, gran, x, w, y, in_params, dump);
}

/* direct_conv (engines.hpp:266-295): channels ascending, fp32 accumulation. */
int lo_direct_conv(const lo_spec* s, const float* x, const float* w, float* y) {
  const int OH = lo_out_h(s), OW = lo_out_w(s);
  for (int ni = 0; ni < s->n; ++ni)
    for (int ki = 0; ki < s->k; ++ki)
      for (int i = 0; i < OH; ++i)
        for (int j = 0; j < OW; ++j) {
          float acc = 0.0f;
          for (int ci = 0; ci < s->c; ++ci)
            for (int ri = 0; ri < 3; ++ri)
              for (int si = 0; si < 3; ++si) {
                const int xi = i + ri - s->pad, xj = j + si - s->pad;
                const float xv = (xi >= 0 && xi < s->h && xj >= 0 && xj < s->w)
                                     ? x[(((size_t)ni * s->h + xi) * s->w + xj) * s->c + ci]
                                     : 0.0f;
                acc += xv * w[(((size_t)ki * 3 + ri) * 3 + si) * s->c + ci];
              }
          y[(((size_t)ni * OH + i) * OW + j) * s->k + ki] = acc;
        }
  return LO_OK;
}
