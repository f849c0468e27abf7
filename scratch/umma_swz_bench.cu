// Microbenchmark: tcgen05 kind::i8 SS-MMA throughput (M=128, N=64, K=32) vs the
// operand row width / swizzle (128 B rows SW128, 64 B rows SW64, 32 B rows
// SW32), operands resident in shared memory.  Scratch tool, not product.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2003_08646_b200/csrc/lance_ptx.cuh"
using namespace lance_dev;

template <int N, int RB>  // RB = row bytes (= BK)
__global__ void __launch_bounds__(128, 1) umma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  for (int i = threadIdx.x; i < (128 + N) * RB / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) { tmem_alloc(&holder, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = holder;
  constexpr uint32_t layout = RB == 128 ? 2u : (RB == 64 ? 4u : 6u);
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * RB;
    constexpr uint32_t idesc = umma_idesc_u8(128, N);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < RB / 32; ++kk)
        umma_i8(tmem + (it & 1) * 256, umma_smem_desc(sa + kk * 32, 8 * RB, layout),
                umma_smem_desc(sb + kk * 32, 8 * RB, layout), idesc, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, int RB>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8);
  const int smem = 1024 + (128 + N) * RB;
  cudaFuncSetAttribute(umma_loop<N, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  umma_loop<N, RB><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  umma_loop<N, RB><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d rowbytes=%3d: %.1f cycles/MMA(K=32) err=%s\n", N, RB, double(cyc) / (iters * (RB / 32)),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<64, 128>(); run<64, 64>(); run<64, 32>();
  run<32, 128>(); run<32, 64>(); run<128, 128>(); run<128, 64>();
  return 0;
}
