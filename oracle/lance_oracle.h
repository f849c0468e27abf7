/*
 * oracle/lance_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference LANCE `lance_gemm` path
 * (/root/reference/proj/include/lance/engines.hpp:492-536) used as the parity
 * checker for the B200 path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library.  The product path never
 * links or calls it.
 *
 * Parity is PINNED: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference compiled in place (oracle/_ref, built by
 * oracle/Makefile from /root/reference headers) and against the committed
 * golden vectors in tests/golden/ (generated from the reference by
 * tests/golden/make_golden.py), plus the reference's own known-answer tests.
 */
#ifndef LANCE_ORACLE_H
#define LANCE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* engines.hpp:33-54 (r = s = 3, stride = 1 are constexpr there). */
typedef struct {
  int n, c, h, w, k, pad;
} lo_spec;

/* quant.hpp:27-37 */
typedef struct {
  int bits;
  float t_min, t_max, scale;
} lo_qparams;

/* quant.hpp:44 -- enum order kept. */
enum { LO_PER_TILE = 0, LO_PER_POSITION = 1, LO_PER_TENSOR = 2 };

/* Status codes. 1 = std::invalid_argument from a spec/config/shape check,
 * 2 = std::invalid_argument("fit_params: NaN in values") (quant.hpp:62). */
enum { LO_OK = 0, LO_EINVAL = 1, LO_ENAN = 2 };

/* Optional stage dumps (any pointer may be NULL).  Layouts follow the
 * reference containers: codes_a = vq.codes [16][M][C] (engines.hpp:118-138),
 * codes_w = uq.codes [16][C][K], acc = gemm_codes per position [16][M][K]
 * (lowpgemm.hpp:76-100), rowsum [16][M], colsum [16][K]
 * (lowpgemm.hpp:121-126), v [16][M][C] fp32, u [16][C][K] fp32. */
typedef struct {
  float* v;
  float* u;
  uint8_t* codes_a;
  uint8_t* codes_w;
  int32_t* rowsum;
  int32_t* colsum;
  int32_t* acc;
  lo_qparams* params_a; /* [16] ([36] for F(4x4)) */
  lo_qparams* params_w; /* [16] */
} lo_dump;

const char* lo_last_error(void);

/* rng.hpp:27-47: mt19937_64, top 24 bits -> U(-1,1) on a 2^-23 grid. */
void lo_uniform_fill(uint64_t seed, float* out, size_t count);

/* engines.hpp:40-44 */
int lo_out_h(const lo_spec* s);
int lo_out_w(const lo_spec* s);
int lo_tiles_h(const lo_spec* s);
int lo_tiles_w(const lo_spec* s);

/* winograd.hpp:66-84 evaluated with matrix.hpp:75-84 operation order. */
void lo_transform_input(const float d[16], float v[16]);
void lo_transform_filter(const float g[9], float u[16]);
void lo_transform_output(const float m[16], float s[4]);

/* F(4x4,3x3) extension (SURVEY.md Appendix D basis, not in the reference):
 * same matmul conventions, alpha = 6, 36 positions. */
void lo_transform_input4(const float d[36], float v[36]);
void lo_transform_filter4(const float g[9], float u[36]);
void lo_transform_output4(const float m[36], float s[16]);
int lo_tiles_h_m(const lo_spec* s, int m);
int lo_tiles_w_m(const lo_spec* s, int m);

/* quant.hpp:54-72 and 77-84. */
int lo_fit_params(const float* values, size_t count, int bits, lo_qparams* out);
uint8_t lo_quantize(float x, const lo_qparams* p);
float lo_dequantize(uint8_t code, const lo_qparams* p);
/* lowpgemm.hpp:110-114 */
float lo_affine_term(int32_t dot, int32_t a_sum, int32_t b_sum, int depth,
                     const lo_qparams* pa, const lo_qparams* pb);

/* Validation of engines.hpp:46-53, 66-79, 84-91, 496-499. */
int lo_validate(const lo_spec* s, int bits_w, int bits_i, int granularity, int mode_gemm);

/* lance_gemm (engines.hpp:492-536).  y = [N][OH][OW][K].  When in_params is
 * non-NULL the input-side parameters are taken from it instead of being fit
 * (static-params mode used to verify large shapes on batch slices). */
int lo_lance_gemm(const lo_spec* s, int bits_w, int bits_i, int granularity,
                  const float* x, const float* w, float* y,
                  const lo_qparams* in_params, lo_dump* dump);

/* lance_gemm for tile side m = 2 (== lo_lance_gemm) or 4 (F(4x4,3x3)
 * extension; dumps and in_params then hold 36 positions). */
int lo_lance_gemm_tiled(const lo_spec* s, int tile_m, int bits_w, int bits_i, int granularity,
                        const float* x, const float* w, float* y,
                        const lo_qparams* in_params, lo_dump* dump);

/* direct_conv (engines.hpp:266-295): fp32 reference used for error bounds. */
int lo_direct_conv(const lo_spec* s, const float* x, const float* w, float* y);

#ifdef __cplusplus
}
#endif
#endif
