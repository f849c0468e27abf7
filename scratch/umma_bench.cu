// Microbenchmark: tcgen05 kind::i8 SS-mode MMA throughput vs N (operands
// resident in SMEM, no loads), one CTA per SM.  Scratch tool, not product.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2003_08646_b200/csrc/lance_ptx.cuh"
using namespace lance_dev;

template <int N>
__global__ void __launch_bounds__(128, 1) umma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  // A: 128 rows x 128 B (SW128), B: N rows x 128 B, 4 K-steps of 32.
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) { tmem_alloc(&holder, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
    constexpr uint32_t idesc = umma_idesc_u8(128, N);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_i8(tmem + (it & 1) * 256, umma_smem_desc(sa + kk * 32, 1024, 2), umma_smem_desc(sb + kk * 32, 1024, 2), idesc, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8);
  const int smem = 1024 + (128 + N) * 128;
  cudaFuncSetAttribute(umma_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  umma_loop<N><<<148, 128, smem>>>(iters, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  umma_loop<N><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double macs = 148.0 * iters * 4 * 128.0 * N * 32;
  printf("N=%3d: %.1f cycles/MMA(K=32), %.0f TOPS (2*MAC/s over 148 SMs), err=%s\n", N,
         double(cyc) / (iters * 4), 2 * macs / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<16>(); run<32>(); run<64>(); run<128>(); run<256>();
  return 0;
}
