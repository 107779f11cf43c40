// Microbenchmark: MMA stream rate from ONE warp issuing warp-collectively (elect.sync inside
// the asm, uniform operands -- the x3 kernel's issue form), kind::f16, A from TMEM (TS) or
// SMEM (SS), M128 x N{128,256} x K16, into one accumulator, random bf16 operands.  Reports
// cycles per MMA for a long stream (commit + wait at the end only) and, for comparison, two
// warps each streaming into their own accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_02203_b200/csrc mma_warp_issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "ndf_tc_ptx.cuh"

using namespace ndf::tc;

__device__ __forceinline__ uint32_t rnd_bf16x2(uint32_t& st) {
  st ^= st << 13; st ^= st >> 17; st ^= st << 5;
  const float a = (float)(st & 0xffff) / 32768.0f - 1.0f, b = (float)(st >> 16) / 32768.0f - 1.0f;
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void k(long long* out, int n_mma, int ts, int N, int issuers, int chains) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar[4];
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t st = 0x9E3779B9u * (tid + 1) + blockIdx.x;
  for (int i = tid; i < 98304 / 16; i += blockDim.x)
    st_shared_v4(smem_u32(smem) + 16 * i, rnd_bf16x2(st), rnd_bf16x2(st), rnd_bf16x2(st),
                 rnd_bf16x2(st));
  fence_proxy_async();
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(&bar[q], 1);
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
  if (warp < 4) {   // random A words in every column of the 128 lanes
    uint32_t z[32];
    for (int c = 0; c < 512; c += 32) {
      for (int j = 0; j < 32; ++j) z[j] = rnd_bf16x2(st);
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
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  if ((issuers >> warp) & 1) {
    const int ord = __popc(issuers & ((1 << warp) - 1));
    // issuer w: accumulator at column 256 w (N = 128) or 0 (N = 256, one issuer); A (TS) at
    // columns 128 + 16 kk of its own region; B: K-major N x 16 blocks, SBO 2048 B
    const uint32_t dcol = N == 256 ? 0u : (ts ? 256u * (uint32_t)ord : 128u * (uint32_t)ord);
    const uint32_t acol = N == 256 ? 256u : 256u * (uint32_t)ord + 128u;
    const uint32_t b = smem_u32(smem);
    tc_fence_after();
    const long long c0 = clock64();
    if (chains == 1) {
#pragma unroll 1
      for (int i = 0; i < n_mma; ++i) {
        const int kk = i & 7;
        if (ts) mma_ts_warp(tm + dcol, tm + acol + 16 * kk, smem_desc(b + kk * 256, 128, 2048), idesc, 1u);
        else mma_ss_warp(tm + dcol, smem_desc(b + 65536 + kk * 256, 128, 2048),
                         smem_desc(b + kk * 256, 128, 2048), idesc, 1u);
      }
    } else if (chains == 2) {   // two accumulators N apart (column halves when N = 64)
      const uint32_t bo = (uint32_t)(N * 256);
#pragma unroll 1
      for (int i = 0; i < n_mma; i += 2) {
        const int kk = (i >> 1) & 7;
        if (ts) {
          mma_ts_warp(tm + dcol, tm + acol + 16 * kk, smem_desc(b + kk * 256, 128, 2048), idesc, 1u);
          mma_ts_warp(tm + dcol + N, tm + acol + 16 * kk, smem_desc(b + bo + kk * 256, 128, 2048), idesc, 1u);
        } else {
          mma_ss_warp(tm + dcol, smem_desc(b + 65536 + kk * 256, 128, 2048),
                      smem_desc(b + kk * 256, 128, 2048), idesc, 1u);
          mma_ss_warp(tm + dcol + N, smem_desc(b + 65536 + kk * 256, 128, 2048),
                      smem_desc(b + bo + kk * 256, 128, 2048), idesc, 1u);
        }
      }
    } else if (chains >= 100) {   // two accumulators in bursts of (chains - 100) MMAs
      const int burst = chains - 100;
#pragma unroll 1
      for (int i = 0; i < n_mma; ++i) {
        const int kk = i & 7, c = (i / burst) & 1;
        mma_ts_warp(tm + dcol + (uint32_t)(c * N), tm + acol + 16 * kk,
                    smem_desc(b + kk * 256, 128, 2048), idesc, 1u);
      }
    } else {   // four accumulators N apart
      const uint32_t bo = (uint32_t)(N * 256);
#pragma unroll 1
      for (int i = 0; i < n_mma; i += 4) {
        const int kk = (i >> 2) & 7;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          mma_ts_warp(tm + dcol + c * N, tm + acol + 16 * kk,
                      smem_desc(b + c * bo + kk * 256, 128, 2048), idesc, 1u);
      }
    }
    const long long c1 = clock64();
    mma_commit_warp(&bar[ord]);
    mbar_wait(&bar[ord], 0);
    const long long c2 = clock64();
    if ((tid & 31) == 0) {
      out[8 * blockIdx.x + 2 * ord] = c1 - c0;
      out[8 * blockIdx.x + 2 * ord + 1] = c2 - c0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  const int n = 2000;
  // issuers: bitmask of warps (warp w runs on SMSP w % 4); chains 2: alternating accumulators
  struct C { int ts, N, mask, ch; const char* name; } cfgs[] = {
      {1, 128, 0x1, 1, "TS N128 1 chain                      "},
      {1, 128, 0x1, 2, "TS N128 2 accumulators, alternating  "},
      {1, 128, 0x1, 102, "TS N128 2 accumulators, bursts of 2  "},
      {1, 128, 0x1, 103, "TS N128 2 accumulators, bursts of 3  "},
      {1, 128, 0x1, 106, "TS N128 2 accumulators, bursts of 6  "},
      {1, 128, 0x1, 125, "TS N128 2 accumulators, bursts of 25 "}};
  for (auto c : cfgs) {
    k<<<148, 256, 98304>>>(d, n, c.ts, c.N, c.mask, c.ch);
    long long h[8 * 148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const int iss = __builtin_popcount(c.mask);
    double tot = 0;
    for (int i = 0; i < 148; ++i) {
      double t = 0;
      for (int w = 0; w < iss; ++w) t = t > h[8 * i + 2 * w + 1] ? t : h[8 * i + 2 * w + 1];
      tot += t;
    }
    tot /= 148;
    const double units = (double)n * iss * c.N / 128.0;
    printf("%s: %8.0f cycles, %d MMAs -> %6.1f cycles per N128 unit, %6.1f per instruction per issuer\n",
           c.name, tot, n * iss, tot / units, tot / n);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
