// Microbenchmark: execution rate of a TS-form tcgen05.mma stream (M128 N128 K16, A and D
// in TMEM, like the query kernel's hidden layers) while 16 warps load (+ store) the
// other half of TMEM -- does epilogue TMEM traffic slow the tensor core down?
// Also: bursts of B MMAs separated by idle gaps (chunked issue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_02203_b200/csrc mma_under_load.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ndf_tc_ptx.cuh"

using namespace ndf::tc;

template <int LOAD, int BURST>   // LOAD: 0 none, 1 ld, 2 ld+st
__global__ void k(long long* out, int n_mma) {
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
  if (warp == 16) {
    if ((tid & 31) == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t b = smem_u32(smem + 32768);
      uint32_t ph = 0;
      long long t0 = clock64();
      for (int i = 0; i < n_mma; ++i) {
        const int kk = i & 7;
        const uint64_t bd = smem_desc(b + kk * 256, 128, 2048);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 256),
            "r"(tm + 384 + 16 * kk), "l"(bd), "r"(idesc), "r"(1u));
        if (BURST > 0 && (i + 1) % BURST == 0) {   // wait for the burst to complete
          mma_commit(&bar);
          mbar_wait(&bar, ph);
          ph ^= 1;
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
      atomicExch(&done, 1);
    }
  } else if (LOAD) {  // 16 warps: LDTM x16 (+ STTM x8) on columns 0..255
    const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
    float acc = 0.f;
    int it = 0;
    while (!*(volatile int*)&done) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
          "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15])
          : "r"(base + (uint32_t)((it & 3) * 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (LOAD == 2) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                     ::"r"(base + 32u), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
                     "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
      ++it;
    }
    if (acc == 1234.5f) out[148] = it;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 149 * 8);
  const int n = 512;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int rep = 0; rep < 2; ++rep) kern<<<148, 17 * 32, 65536>>>(d, n);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    printf("%-34s cycles per MMA = %6.1f   (%s)\n", name, m / n, cudaGetErrorString(cudaGetLastError()));
  };
  run(k<0, 0>, "stream, idle TMEM");
  run(k<1, 0>, "stream, 16 warps LDTM");
  run(k<2, 0>, "stream, 16 warps LDTM+STTM");
  run(k<0, 2>, "bursts of 2 (+commit wait), idle");
  run(k<2, 2>, "bursts of 2, LDTM+STTM");
  run(k<0, 9>, "bursts of 9, idle");
  run(k<2, 9>, "bursts of 9, LDTM+STTM");
  return 0;
}
