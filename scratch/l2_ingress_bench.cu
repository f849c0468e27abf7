// Scratch microbenchmark (not product): per-SM L2 -> shared ingress with 1-D
// bulk copies from an L2-resident buffer (as the GEMM's A/B re-reads are), one
// CTA per SM, P producer lanes (each in its own warp with its own mbarrier
// ring) and one consumer lane per ring.  Reports aggregate GB/s and bytes per
// SM clock (clock64 span of the slowest CTA).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2003_08646_b200/csrc/lance_ptx.cuh"
using namespace lance_dev;

__global__ void __launch_bounds__(512, 1) ingress(const uint8_t* src, size_t src_bytes, int copy_bytes, int depth,
                                                  int producers, int copies_per_cta, unsigned long long* out, int same_warp) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)producers * depth * copy_bytes);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * producers * depth; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  const int per = copies_per_cta / producers;
  const size_t nsrc = src_bytes / copy_bytes;
  const int pid = same_warp ? lane : warp;
  if (same_warp ? (warp == 0 && lane < producers) : (warp < producers && lane == 0)) {
    uint64_t* full = bars + pid * depth * 2;
    uint64_t* empty = full + depth;
    uint8_t* ring = smem + (size_t)pid * depth * copy_bytes;
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < per; ++i) {
      mbar_wait(&empty[s], ph ^ 1u);
      mbar_arrive_expect_tx(&full[s], copy_bytes);
      const size_t idx = ((size_t)blockIdx.x * 7919 + (size_t)i * producers + pid) % nsrc;
      bulk_load(ring + (size_t)s * copy_bytes, src + idx * copy_bytes, copy_bytes, &full[s]);
      if (++s == depth) { s = 0; ph ^= 1u; }
    }
  } else if (warp >= 8 && warp < 8 + producers && lane == 0) {
    const int p = warp - 8;
    uint64_t* full = bars + p * depth * 2;
    uint64_t* empty = full + depth;
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < per; ++i) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == depth) { s = 0; ph ^= 1u; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t src_bytes_l2 = size_t(48) << 20;  // L2 resident
  const size_t src_bytes_hbm = size_t(2) << 30;
  uint8_t* src; cudaMalloc(&src, src_bytes_hbm); cudaMemset(src, 1, src_bytes_hbm);
  unsigned long long* out; cudaMalloc(&out, 8 * 4096);
  unsigned long long host[4096];
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int copies_total_bytes_per_cta = 8 << 20;
  for (int hbm : {0, 1})
  for (int sw : {0, 1})
  for (int cb : {4096, 8192, 16384, 32768})
    for (int p : {1, 2, 4, 8})
      for (int d : {2, 4}) {
        const size_t src_bytes = hbm ? src_bytes_hbm : src_bytes_l2;
        const size_t smem = (size_t)p * d * cb + 2 * p * d * 8 + 64;
        if (smem > 220 * 1024) continue;
        const int copies = copies_total_bytes_per_cta / cb;
        ingress<<<sms, 512, smem>>>(src, src_bytes, cb, d, p, copies, out, sw);
        cudaEventRecord(e0);
        ingress<<<sms, 512, smem>>>(src, src_bytes, cb, d, p, copies, out, sw);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(host, out, 8 * sms, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0; for (int i = 0; i < sms; ++i) mx = host[i] > mx ? host[i] : mx;
        const double per_cta = (double)(copies / p) * p * cb;
        printf("%s %s copy=%6d producers=%d depth=%d : %7.0f GB/s aggregate, %5.1f B/clk/SM (%s)\n", hbm ? "HBM" : "L2 ", sw ? "lanes" : "warps", cb, p, d,
               per_cta * sms / (ms * 1e-3) / 1e9, per_cta / mx, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
