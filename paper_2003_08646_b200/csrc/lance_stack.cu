// lance_stack.cu -- glue kernels of the layer-stack driver (SURVEY.md section
// 8(f) row 2; paper_2003_08646_b200/stack.py): the 2x2 / stride-2 max-pool
// between the VGG-16-CIFAR conv stages (BASELINE config 2).  Not part of the
// reference's lance_gemm path; it keeps chained activations on the device.
#include <cuda_runtime.h>

#include <cstdint>

#include "lance_common.cuh"

namespace lance_dev {

// y[n][h/2][w/2][c] = max of the 2x2 window (floor), NHWC, float4 over channels
// when C % 4 == 0.  Pure HBM streaming: reads x once, writes y once.
__global__ void __launch_bounds__(256) maxpool2x2_kernel(const float* __restrict__ x,
                                                         float* __restrict__ y, int N, int H,
                                                         int W, int C) {
  pdl_entry();
  const int OH = H / 2, OW = W / 2;
  const bool v4 = (C & 3) == 0;
  const int cw = v4 ? C / 4 : C;
  const long long total = static_cast<long long>(N) * OH * OW * cw;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cc = static_cast<int>(i % cw);
    long long r = i / cw;
    const int ow = static_cast<int>(r % OW);
    r /= OW;
    const int oh = static_cast<int>(r % OH);
    const long long n = r / OH;
    const long long base = ((n * H + 2 * oh) * W + 2 * ow) * C;
    const long long rowc = static_cast<long long>(W) * C;
    if (v4) {
      const float4* p = reinterpret_cast<const float4*>(x + base) + cc;
      const float4 a = __ldg(p), b = __ldg(p + C / 4), c = __ldg(p + rowc / 4), d = __ldg(p + rowc / 4 + C / 4);
      reinterpret_cast<float4*>(y)[i] =
          make_float4(fmaxf(fmaxf(a.x, b.x), fmaxf(c.x, d.x)), fmaxf(fmaxf(a.y, b.y), fmaxf(c.y, d.y)),
                      fmaxf(fmaxf(a.z, b.z), fmaxf(c.z, d.z)), fmaxf(fmaxf(a.w, b.w), fmaxf(c.w, d.w)));
    } else {
      const float* p = x + base + cc;
      y[i] = fmaxf(fmaxf(__ldg(p), __ldg(p + C)), fmaxf(__ldg(p + rowc), __ldg(p + rowc + C)));
    }
  }
}

cudaError_t launch_maxpool2x2(const float* x, float* y, int N, int H, int W, int C, int sm_count,
                              cudaStream_t s) {
  const long long total = static_cast<long long>(N) * (H / 2) * (W / 2) * (((C & 3) == 0) ? C / 4 : C);
  if (total == 0) return cudaSuccess;
  const long long blocks = (total + 255) / 256;
  const int grid = static_cast<int>(blocks < 8LL * sm_count ? blocks : 8LL * sm_count);
  LANCE_LAUNCH_CHECK(launch_k(maxpool2x2_kernel, grid, 256, 0, s, x, y, N, H, W, C));
  return cudaGetLastError();
}

}  // namespace lance_dev
