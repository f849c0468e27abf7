// Scratch: isolate TMA multicast within a cluster (not product code).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_2003_08646_b200/csrc/lance_ptx.cuh"
using namespace lance_dev;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// mode 0: each CTA loads rows [rank*R/cs, +R/cs) multicast; mode 1: rank 0 loads all rows multicast;
// mode 2: like 0 but expect_tx issued before a cluster barrier, then loads.
__global__ void mc_kernel(const __grid_constant__ CUtensorMap tm, int cs, int mode, int* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  uint8_t* buf = base + (mode >= 4 ? 0x20000 : 0);
  uint8_t* buf2 = buf + 128 * 64;
  uint64_t& bar = *reinterpret_cast<uint64_t*>(base + 0x27800);
  uint64_t& bar2 = *reinterpret_cast<uint64_t*>(base + 0x27808);
  uint64_t& bar3 = *reinterpret_cast<uint64_t*>(base + 0x27810);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, cs); mbar_init(&bar3, 1); fence_barrier_init(); }
  cluster_sync();
  const uint16_t mask = (1u << cs) - 1;
  const int rows = 128 / cs;
  if (threadIdx.x == 0) {
    if (mode == 2 && rank == 0) { long long t0 = clock64(); while (clock64() - t0 < 2000000) {} }
    mbar_arrive_expect_tx(&bar, 128 * 64 + (mode >= 3 ? 64 * rows : 0));
    if (mode >= 3) tma_load_3d(buf2, &tm, 0, 0, 0, &bar);
    if (mode == 1) {
      if (rank == 0) tma_load_3d_mc(buf, &tm, 0, 0, 0, &bar, mask);
    } else {
      tma_load_3d_mc(buf + rank * rows * 64, &tm, 0, rank * rows, 0, &bar, mask);
    }
  }
  if (threadIdx.x == 0) {
    long long spins = 0;
    while (!mbar_try_wait(smem_u32(&bar), 0)) if (++spins > (1ll << 24)) { printf("block %d rank %u timeout\n", blockIdx.x, rank); break; }
    int sum = 0;
    for (int i = 0; i < 128 * 64; ++i) sum += buf[i];
    out[blockIdx.x] = sum;
    if (mode >= 3) {
      umma_commit_mc(&bar2, mask);
      spins = 0;
      while (!mbar_try_wait(smem_u32(&bar2), 0)) if (++spins > (1ll << 24)) { printf("block %d rank %u commit-mc timeout bar2=0x%x bar3 state\n", blockIdx.x, rank, smem_u32(&bar2)); out[blockIdx.x] = -1; break; }
      if (mbar_try_wait(smem_u32(&bar3), 0)) printf("block %d rank %u: bar3 unexpectedly completed\n", blockIdx.x, rank);
    }
  }
  cluster_sync();
}

int main() {
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<EncodeTiledFn>(fnp);
  std::vector<uint8_t> h(128 * 64);
  long long expect = 0;
  for (int i = 0; i < 128 * 64; ++i) { h[i] = uint8_t(i * 7 + 3); expect += h[i]; }
  uint8_t* d; cudaMalloc(&d, h.size()); cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  int* out; cudaMalloc(&out, 64 * sizeof(int));
  for (int cs : {2, 4}) for (int mode : {0, 1, 2, 3, 4}) {
    CUtensorMap tm;
    const cuuint64_t dims[3] = {64, 128, 1};
    const cuuint64_t str[2] = {64, 128 * 64};
    const cuuint32_t box[3] = {64, (cuuint32_t)(mode == 1 ? 128 : 128 / cs), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemset(out, 0, 64 * sizeof(int));
    const int dsmem = 0x28000 + 2048;
    cudaFuncSetAttribute(mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(cs * 2); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = dsmem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, mc_kernel, tm, cs, mode, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    int ho[64]; cudaMemcpy(ho, out, sizeof ho, cudaMemcpyDeviceToHost);
    printf("cs=%d mode=%d encode=%d launch=%s sync=%s sums:", cs, mode, (int)r, cudaGetErrorString(e), cudaGetErrorString(e2));
    for (int i = 0; i < cs * 2; ++i) printf(" %d", ho[i]);
    printf(" (expect %lld)\n", expect);
  }
  return 0;
}
