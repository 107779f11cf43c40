// Microbenchmark: does a thread blocked in tcgen05.mma issue (tensor core busy) slow
// down the other warps of its SM sub-partition?  Warp 0 lane 0 issues M128 N128 K16
// MMAs back to back; warps 1..15 (SMSP = warp % 4) run an FFMA chain and report cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_02203_b200/csrc mma_issue_smsp.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ndf_tc_ptx.cuh"

using namespace ndf::tc;

template <bool MMA>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 16; i += blockDim.x) st_shared_v4(smem_u32(smem) + 16 * i, 0, 0, 0, 0);
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    if (MMA && tid == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      int n = 0;
      while (*(volatile int*)&done < 15) {
        const int kk = n++ & 7;
        mma_bf16(tm, smem_desc(a + kk * 256, 128, 2048), smem_desc(b + kk * 256, 128, 2048), idesc, 1u);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else {
    float x = 1.0f + tid * 1e-6f, y = 0.5f;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) x = fmaf(x, 0.9999f, y);
    }
    long long c1 = clock64();
    if ((tid & 31) == 0) {
      out[blockIdx.x * 16 + warp] = c1 - c0;
      atomicAdd(&done, 1);
    }
    if (x == 12345.f) out[0] = 1;
  }
  __syncthreads();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 16 * 8);
  const int iters = 4000;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int rep = 0; rep < 2; ++rep) kern<<<148, 16 * 32, 65536>>>(d, iters);
    cudaDeviceSynchronize();
    long long h[148 * 16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double sm0 = 0, oth = 0;
    int n0 = 0, n1 = 0;
    for (int b = 0; b < 148; ++b)
      for (int w = 1; w < 16; ++w) {
        if (w % 4 == 0) { sm0 += h[b * 16 + w]; ++n0; } else { oth += h[b * 16 + w]; ++n1; }
      }
    printf("%-16s FFMA-chain cycles/iter: SMSP0 warps %.1f, other SMSPs %.1f  (%s)\n", name,
           sm0 / n0 / iters, oth / n1 / iters, cudaGetErrorString(cudaGetLastError()));
  };
  run(k<false>, "no MMA");
  run(k<true>, "MMA issuing");
  return 0;
}
