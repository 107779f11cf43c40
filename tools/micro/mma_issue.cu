// Microbenchmark: issue cost and execution rate of tcgen05.mma kind::f16 M128 N128 K16
// with A from SMEM (SS) or TMEM (TS), one thread issuing, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_02203_b200/csrc mma_issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ndf_tc_ptx.cuh"

using namespace ndf::tc;

template <bool TS>
__global__ void k(long long* out, int n_mma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  // zero A/B operands (64 KB)
  for (int i = tid; i < 65536 / 16; i += blockDim.x) st_shared_v4(smem_u32(smem) + 16 * i, 0, 0, 0, 0);
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (tid == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int kk = i & 7;
      const uint64_t bd = smem_desc(b + kk * 256, 128, 2048);
      if (TS) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm),
            "r"(tm + 256 + 8 * kk), "l"(bd), "r"(idesc), "r"(1u));
      } else {
        mma_bf16(tm, smem_desc(a + kk * 256, 128, 2048), bd, idesc, 1u);
      }
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int ts = 0; ts < 2; ++ts) {
    for (int n : {1, 2, 4, 8, 16, 64, 256}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (ts) k<true><<<148, 128, 65536>>>(d, n);
        else k<false><<<148, 128, 65536>>>(d, n);
      }
      cudaDeviceSynchronize();
      long long h[296];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double is = 0, done = 0;
      for (int i = 0; i < 148; ++i) { is += h[2 * i]; done += h[2 * i + 1]; }
      printf("%s n=%3d  issue %7.1f cyc (%.1f/mma)  complete %7.1f cyc (%.1f/mma)\n",
             ts ? "TS" : "SS", n, is / 148, is / 148 / n, done / 148, done / 148 / n);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
