// Microbenchmark: tcgen05.mma (M128 N128 K16, TS form: A from TMEM) throughput with one
// vs two issuing threads (different warps, separate accumulators), streamed or in
// bursts of B MMAs each followed by commit + mbarrier wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_02203_b200/csrc mma_two_issuers.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ndf_tc_ptx.cuh"

using namespace ndf::tc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a),
               "l"(b), "r"(idesc));
}

// mode 0: commit + wait after each burst; 1: commit only (wait at the end);
// 2: TS form replaced by SS form (A from SMEM), commit + wait
__global__ void k(long long* out, int nissuers, int total, int burst, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 32768 / 16; i += blockDim.x) st_shared_v4(smem_u32(smem) + 16 * i, 0, 0, 0, 0);
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
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
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (warp < nissuers && (tid & 31) == 0) {
    const uint32_t d = tm + (uint32_t)(warp * 256);          // D in cols [256w, 256w+128)
    const uint32_t a = tm + (uint32_t)(warp * 256 + 128);   // A in the other 128 columns
    const uint32_t b = smem_u32(smem);
    const int mine = total / nissuers;
    uint32_t ph = 0;
    for (int i = 0; i < mine; ++i) {
      const int kk = i & 7;
      if (mode == 2)
        mma_bf16(d, smem_desc(b + 16384 + kk * 256, 128, 2048), smem_desc(b + kk * 256, 128, 2048),
                 idesc, 1u);
      else
        mma_ts(d, a + 16 * kk, smem_desc(b + kk * 256, 128, 2048), idesc);
      if (burst > 0 && (i % burst) == burst - 1) {
        mma_commit(&bar[warp]);
        if (mode != 1) {
          mbar_wait(&bar[warp], ph);
          ph ^= 1;
        }
      }
    }
    mma_commit(&bar[warp]);
    if (mode == 1) {                 // every commit arrived once: wait for the last phase
      const int commits = mine / (burst > 0 ? burst : mine + 1) + 1;
      for (int c = 0; c < commits; ++c) { mbar_wait(&bar[warp], ph); ph ^= 1; }
    } else {
      mbar_wait(&bar[warp], ph);
    }
  }
  tc_fence_before();
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int total = 1200;
  for (int mode : {0, 1, 2})
  for (int burst : {0, 25, 7}) {
    for (int nis : {1, 2}) {
      if (mode && burst == 0) continue;
      printf("mode %d ", mode);
      k<<<148, 128, 65536>>>(d, nis, total, burst, mode);
      k<<<148, 128, 65536>>>(d, nis, total, burst, mode);
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < 148; ++i) s += h[i];
      printf("issuers=%d burst=%3d  cycles per MMA (all issuers) = %6.1f\n", nis, burst,
             s / 148 / total);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
