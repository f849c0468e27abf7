// Scratch microbenchmark (not product): 4-D tensor TMA loads of input rows
// (box = C channels x BW pixels x 1 row x 1 image from an NHWC fp32 tensor),
// as the band kernels issue them, vs 1-D bulk copies of the same bytes.
// Modes: 0 tensor box starting at x = 0, 1 tensor box starting at x = -1
// (one out-of-bounds pixel, zero fill), 2 bulk copy of the same byte count.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2003_08646_b200/csrc/lance_ptx.cuh"
using namespace lance_dev;

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
               :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap tm, const float* x, int N, int H, int W, int C,
                                         int BW, int depth, int mode, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)depth * BW * C * 4);
  const uint32_t bytes = BW * C * 4;
  if (threadIdx.x == 0) { for (int s = 0; s < depth; ++s) mbar_init(&full[s], 1); fence_barrier_init(); }
  __syncthreads();
  const long long rows = (long long)N * H;
  const int segs = W / BW;
  if (threadIdx.x == 0) {
    int s = 0; uint32_t ph = 0; long long issued = 0, done = 0;
    unsigned long long acc = 0;
    const long long total = (rows * segs + gridDim.x - 1 - blockIdx.x) / gridDim.x;
    while (done < total) {
      while (issued < total && issued - done < depth) {
        const long long it = blockIdx.x + issued * gridDim.x;
        const int seg = it % segs; const long long r = it / segs;
        const int img = r / H, y = r % H;
        const int slot = issued % depth;
        mbar_arrive_expect_tx(&full[slot], bytes);
        uint8_t* dst = smem + (size_t)slot * bytes;
        if (mode == 2) bulk_load(dst, x + ((r * W) + seg * BW) * C, bytes, &full[slot]);
        else tma4(dst, &tm, 0, seg * BW - (mode == 1 ? 1 : 0), y, img, &full[slot]);
        ++issued;
      }
      const int slot = done % depth;
      mbar_wait(&full[slot], (done / depth) & 1);
      acc += smem[(size_t)slot * bytes + 5];
      ++done;
    }
    sink[blockIdx.x] = acc;
  }
}

int main() {
  const int N = 256, H = 56, W = 56, C = 64;
  float* x; cudaMalloc(&x, sizeof(float) * N * H * W * C); cudaMemset(x, 0, sizeof(float) * N * H * W * C);
  unsigned long long* sink; cudaMalloc(&sink, 8 * 4096);
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fnp);
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int BW : {28, 56}) for (int depth : {4, 8, 16}) for (int mode = 0; mode < 3; ++mode) for (int per : {1, 2}) {
    CUtensorMap tm;
    const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    const cuuint64_t str[3] = {(cuuint64_t)C * 4, (cuuint64_t)C * 4 * W, (cuuint64_t)C * 4 * W * H};
    const cuuint32_t box[4] = {(cuuint32_t)C, (cuuint32_t)BW, 1, 1}, es[4] = {1, 1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = (size_t)depth * BW * C * 4 + 8 * depth + 64;
    if (smem > 200 * 1024 / per) continue;
    k<<<sms * per, 64, smem>>>(tm, x, N, H, W, C, BW, depth, mode, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) k<<<sms * per, 64, smem>>>(tm, x, N, H, W, C, BW, depth, mode, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("BW=%2d depth=%2d ctas/sm=%d %-10s : %6.0f GB/s (%s)\n", BW, depth, per,
           mode == 0 ? "tensor" : (mode == 1 ? "tensor-1" : "bulk"),
           3.0 * sizeof(float) * N * H * W * C / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
