// Microbenchmark: TMEM load/store rate of 16 epilogue-like warps with and without a
// concurrent MMA stream (one thread issuing M128 N128 K16 kind::f16 MMAs into the
// other half of TMEM), 1 CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_02203_b200/csrc tmem_contention.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ndf_tc_ptx.cuh"

using namespace ndf::tc;

template <bool MMA, bool STORE>
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
  if (warp == 16) {                       // MMA issuer: D in columns 256..383
    if (MMA && (tid & 31) == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      int n = 0;
      while (*(volatile int*)&done < 16) {
        const int kk = n++ & 7;
        mma_bf16(tm + 256, smem_desc(a + kk * 256, 128, 2048), smem_desc(b + kk * 256, 128, 2048),
                 idesc, 1u);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else {                                // 16 warps: LDTM x16 (+ STTM x8) on columns 0..255
    const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
    float acc = 0.f;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
          "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15])
          : "r"(base + (uint32_t)((it & 3) * 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (STORE) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                     ::"r"(base + 32u), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
                     "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
    }
    long long c1 = clock64();
    if ((tid & 31) == 0) {
      out[blockIdx.x * 16 + warp] = c1 - c0;
      atomicAdd(&done, 1);
    }
    if (tid == 0) out[148 * 16 + blockIdx.x] = (long long)acc;
  }
  __syncthreads();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, (148 * 17) * 8);
  const int iters = 2000;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int rep = 0; rep < 2; ++rep) kern<<<148, 17 * 32, 65536>>>(d, iters);
    cudaDeviceSynchronize();
    long long h[148 * 16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148 * 16; ++i) m += h[i];
    m /= 148 * 16;
    printf("%-28s cycles per LDTM.x16 iteration per warp = %6.1f   (%s)\n", name, m / iters,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(k<false, false>, "ld only");
  run(k<true, false>, "ld + concurrent MMA");
  run(k<false, true>, "ld + st");
  run(k<true, true>, "ld + st + concurrent MMA");
  return 0;
}
