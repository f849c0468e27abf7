// Scratch microbenchmark (not product): streaming global -> shared with 1-D
// bulk copies through an mbarrier ring, one producer lane + one consumer lane
// per CTA, one CTA per SM.  Reports achieved GB/s for stage sizes / depths,
// with the consumer releasing slots either directly (mbarrier arrive) or via
// an empty tcgen05.commit (as the GEMM's MMA thread does).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2003_08646_b200/csrc/lance_ptx.cuh"
using namespace lance_dev;

__global__ void __launch_bounds__(128, 1) stream_kernel(const uint8_t* src, size_t bytes, int stage_bytes,
                                                        int stages, int mode, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  if (warp == 1) { tmem_alloc(&holder, 32); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const size_t nchunks = bytes / stage_bytes;
  if (warp == 0 && lane == 0) {
    int s = 0; uint32_t ph = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      mbar_wait(&empty[s], ph ^ 1u);
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      bulk_load(smem + (size_t)s * stage_bytes, src + c * stage_bytes, stage_bytes, &full[s]);
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0; uint32_t ph = 0; unsigned long long acc = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      mbar_wait(&full[s], ph);
      acc += smem[(size_t)s * stage_bytes + (c & 1023)];
      if (mode == 1) { tc_fence_after(); umma_commit(&empty[s]); }
      else mbar_arrive(&empty[s]);
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
    sink[blockIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(holder, 32);
}

int main() {
  const size_t bytes = size_t(1) << 30;
  uint8_t* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  unsigned long long* sink; cudaMalloc(&sink, 8 * 1024);
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sizes[] = {8192, 16384, 32768};
  const int depths[] = {2, 4, 8, 16};
  for (int mode = 0; mode < 2; ++mode)
    for (int sb : sizes)
      for (int d : depths) {
        const size_t smem = (size_t)d * sb + 2 * d * 8 + 64;
        if (smem > 200 * 1024) continue;
        stream_kernel<<<sms, 128, smem>>>(src, bytes, sb, d, mode, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) stream_kernel<<<sms, 128, smem>>>(src, bytes, sb, d, mode, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("mode=%s stage=%6d depth=%2d : %7.0f GB/s  (%s)\n", mode ? "commit" : "arrive", sb, d,
               3.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
