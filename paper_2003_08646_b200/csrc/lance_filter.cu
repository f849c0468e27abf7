// lance_filter.cu -- K2: filter transform G g G^T + Winograd-domain
// quantisation, once per layer (domain_from_filters engines.hpp:215-233,
// quantize_domain(u) engines.hpp:140-183, b_col_sum lowpgemm.hpp:124-126).
#include <cuda_runtime.h>

#include <cstdint>

#include "lance_common.cuh"

namespace lance_dev {

// --------------------------------------------------------------------------
// K2a: u = G g G^T for every (k, c); u_tmp [16][K][C]; per-position fit.
__global__ void __launch_bounds__(256) filter_transform_kernel(const float* __restrict__ w,
                                                               float* __restrict__ u_tmp,
                                                               float* __restrict__ partials,
                                                               LanceDevState* __restrict__ st,
                                                               FilterGeom g) {
  pdl_entry();
  __shared__ float s_red[256];
  float lo[16], hi[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    lo[p] = __int_as_float(0x7f800000);
    hi[p] = __int_as_float(0xff800000);
  }
  const long long total = static_cast<long long>(g.K) * g.C;
  const long long slice = total;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = i / g.C;
    const int c = static_cast<int>(i - k * g.C);
    float gg[9], u[16];
#pragma unroll
    for (int rs = 0; rs < 9; ++rs) gg[rs] = __ldg(w + (k * 9 + rs) * g.C + c);
    filter_transform(gg, u);
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      u_tmp[p * slice + i] = u[p];
      lo[p] = fmin_nan(lo[p], u[p]);
      hi[p] = fmax_nan(hi[p], u[p]);
    }
  }
  if (block_minmax_and_ticket(lo, hi, partials, &st->ticket_w, s_red)) {
    fit_from_ranges(s_red, g.granularity, st->bits_w, st->w_tmin, st->w_tmax, st->w_scale,
                    nullptr, &st->nan_w);
  }
}

// K2b: codes_w as the B operand's UMMA images (lance_kernels.cuh) and column
// sums [16][K_pad].
__global__ void __launch_bounds__(128) filter_quant_kernel(const float* __restrict__ u_tmp,
                                                           uint8_t* __restrict__ codes_w,
                                                           int32_t* __restrict__ colsum,
                                                           const LanceDevState* __restrict__ st,
                                                           FilterGeom g) {
  pdl_entry();
  __shared__ int s_sum[4];
  const int k = blockIdx.x;
  const float top = static_cast<float>((1 << st->bits_w) - 1);
  const long long slice = static_cast<long long>(g.K) * g.C;
  for (int p = 0; p < 16; ++p) {
    const float tmin = st->w_tmin[p], scale = st->w_scale[p];
    int sum = 0;
    for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
      const uint32_t code =
          quantize_code(u_tmp[p * slice + static_cast<long long>(k) * g.C + c], tmin, scale, top);
      codes_w[umma_image_offset(k, c, p, g.bn, g.bk, g.nk)] = static_cast<uint8_t>(code);
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

cudaError_t launch_filter_prepare(const float* w, float* u_tmp, float* partials, int grid,
                                  uint8_t* codes_w, int32_t* colsum, LanceDevState* st,
                                  const FilterGeom& g, cudaStream_t s) {
  LANCE_LAUNCH_CHECK(launch_k(filter_transform_kernel, grid, 256, 0, s, w, u_tmp, partials, st, g));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  LANCE_LAUNCH_CHECK(launch_k(filter_quant_kernel, g.K, 128, 0, s, u_tmp, codes_w, colsum, st, g));
  return cudaGetLastError();
}

}  // namespace lance_dev
