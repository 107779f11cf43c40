// Microbenchmark: M128 N128 K16 kind::f16 MMAs issued by one thread in bursts of B
// (accumulating into one TMEM accumulator, A from TMEM "TS" or SMEM "SS"), each burst
// followed by tcgen05.commit + mbarrier wait.  Reports cycles to issue a burst and to
// its completion.  TMEM and SMEM operands are zero-initialised.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_02203_b200/csrc mma_burst.cu
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

__device__ __forceinline__ uint32_t rnd_bf16x2(uint32_t& st) {
  // xorshift -> two bf16 values uniform in [-1, 1)
  st ^= st << 13; st ^= st >> 17; st ^= st << 5;
  const float a = (float)(st & 0xffff) / 32768.0f - 1.0f, b = (float)(st >> 16) / 32768.0f - 1.0f;
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void k(long long* out, int burst, int nburst, int ts, int random, int chains, int nhalf) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t st = 0x9E3779B9u * (tid + 1) + blockIdx.x;
  for (int i = tid; i < 65536 / 16; i += blockDim.x) {
    if (random)
      st_shared_v4(smem_u32(smem) + 16 * i, rnd_bf16x2(st), rnd_bf16x2(st), rnd_bf16x2(st),
                   rnd_bf16x2(st));
    else
      st_shared_v4(smem_u32(smem) + 16 * i, 0, 0, 0, 0);
  }
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
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
  {   // zero all 512 columns of the 128 lanes (warp w: lanes 32w..32w+31)
    uint32_t z[32] = {};
    for (int c = 0; c < 512; c += 32) {
      for (int j = 0; j < 32; ++j) z[j] = (random && c >= 128) ? rnd_bf16x2(st) : 0u;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
          "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
          "%28, %29, %30, %31, %32};" ::"r"(tm + ((uint32_t)(warp * 32) << 16) + c),
          "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]),
          "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]),
          "r"(z[15]), "r"(z[16]), "r"(z[17]), "r"(z[18]), "r"(z[19]), "r"(z[20]), "r"(z[21]),
          "r"(z[22]), "r"(z[23]), "r"(z[24]), "r"(z[25]), "r"(z[26]), "r"(z[27]), "r"(z[28]),
          "r"(z[29]), "r"(z[30]), "r"(z[31]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int N = nhalf ? 64 : 128;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  if (tid == 0) {
    const uint32_t b = smem_u32(smem);
    uint32_t ph = 0;
    long long issue = 0, total = 0;
    for (int r = 0; r < nburst; ++r) {
      const long long c0 = clock64();
      for (int i = 0; i < burst; ++i) {
        const int kk = i & 7;
        const int c = i % chains;
        // chains: accumulators at columns 0 / 256 (A at 128 + 16 kk);  nhalf: N=64 halves of
        // one accumulator at columns 0 / 64 (B rows 0-63 / 64-127: + 8 * 128 B core groups)
        const uint32_t dcol = nhalf ? (uint32_t)(64 * c) : (uint32_t)(256 * c);
        const uint32_t boff = nhalf ? (uint32_t)(c * 8 * 2048) : 0u;
        if (ts) mma_ts(tm + dcol, tm + 128 + 16 * kk, smem_desc(b + boff / 2 + kk * 256, 128, 2048), idesc);
        else mma_bf16(tm + dcol, smem_desc(b + 32768 + kk * 256, 128, 2048),
                      smem_desc(b + kk * 256, 128, 2048), idesc, 1u);
      }
      const long long c1 = clock64();
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      const long long c2 = clock64();
      if (r > 0) { issue += c1 - c0; total += c2 - c0; }
    }
    out[2 * blockIdx.x] = issue / (nburst - 1);
    out[2 * blockIdx.x + 1] = total / (nburst - 1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int cfg = 0; cfg < 3; ++cfg)
  for (int ts : {1})
    for (int burst : {7, 24, 64}) {
      const int nb = 4000 / burst + 2;
      const int chains = cfg == 0 ? 1 : 2, nhalf = cfg == 2;
      printf("%s ", cfg == 0 ? "1 chain N128    " : (cfg == 1 ? "2 chains N128   " : "2 N-halves N64  "));
      k<<<148, 128, 65536>>>(d, burst, nb, ts, 1, chains, nhalf);
      long long h[296];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double is = 0, tt = 0;
      for (int i = 0; i < 148; ++i) { is += h[2 * i]; tt += h[2 * i + 1]; }
      is /= 148; tt /= 148;
      printf("%s burst %3d: issue %7.0f cyc (%6.1f/mma)  complete %7.0f cyc (%6.1f/mma)\n",
             ts ? "TS" : "SS", burst, is, is / burst, tt, tt / burst);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
