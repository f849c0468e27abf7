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

__global__ void __launch_bounds__(640, 1) stream_kernel(const uint8_t* src, size_t bytes, int stage_bytes,
                                                        int stages, int mode, unsigned long long* sink,
                                                        size_t wrap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  __shared__ uint32_t holder;
  __shared__ uint64_t spin_bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&spin_bar, 1);
    done = 0;
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
      // mode 0: one copy; mode 1: 4/5 of the stage streamed + 1/5 from a shared
      // 64 KB region (all CTAs); mode 2: stage as 2 copies, both streamed.
      // wrap == 1: CTA-private contiguous regions (each CTA streams its own
      // slab) instead of the grid-interleaved sweep.
      const size_t nper = nchunks / gridDim.x;
      const size_t off = (wrap == 1) ? ((size_t)blockIdx.x * nper + (c / gridDim.x)) * stage_bytes
                                     : c * (size_t)stage_bytes;
      if (mode == 0) {
        bulk_load(smem + (size_t)s * stage_bytes, src + off, stage_bytes, &full[s]);
      } else if (mode == 1) {
        const int a = stage_bytes / 5 * 4 / 16 * 16, b = stage_bytes - a;
        bulk_load(smem + (size_t)s * stage_bytes, src + off, a, &full[s]);
        bulk_load(smem + (size_t)s * stage_bytes + a, src + (c * b) % 65536, b, &full[s]);
      } else {
        const int a = stage_bytes / 5 * 4 / 16 * 16, b = stage_bytes - a;
        bulk_load(smem + (size_t)s * stage_bytes, src + off, a, &full[s]);
        bulk_load(smem + (size_t)s * stage_bytes + a, src + off + a, b, &full[s]);
      }
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
    done = 1;
  } else if (warp >= 4 && mode == 7) {
    // mode 1/3: 16 warps spin on a barrier that completes only at the end.
    while (!mbar_try_wait(smem_u32(&spin_bar), 0u)) {
      if (done) break;
    }
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
  const int sizes[] = {8192, 16384};
  const int depths[] = {4, 8, 16};
  const size_t wraps[] = {bytes, 1};
  const char* names[] = {"one copy", "A+sharedB", "two copies"};
  for (size_t wrap : wraps)
  for (int mode = 0; mode < 1; ++mode)
    for (int sb : sizes)
      for (int d : depths) {
        const size_t smem = (size_t)d * sb + 2 * d * 8 + 64;
        if (smem > 200 * 1024) continue;
        (void)wrap;
        const int thr = 128;
        stream_kernel<<<sms, thr, smem>>>(src, bytes, sb, d, mode, sink, wrap);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) stream_kernel<<<sms, thr, smem>>>(src, bytes, sb, d, mode, sink, wrap);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%s %-14s stage=%6d depth=%2d : %7.0f GB/s  (%s)\n", wrap == bytes ? "interleaved" : "cta-slabs  ",
               names[mode], sb, d, 3.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
