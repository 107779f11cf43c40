// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput on sm_100a, alone and
// interleaved with MUFU tanh work (the NDF epilogue's two co-bottlenecks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_rate tmem_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>   // 0: ld x32 + wait; 1: ld x32 + wait + 32 tanh; 2: 32 tanh only
__global__ void k(float* out, int iters, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32 % 512);
  float acc = 0.f;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    if (MODE != 2) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
          "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
            "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
            "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(base + (uint32_t)((it & 3) * 128)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(acc + i);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float x = __uint_as_float(r[i]) * 1e-3f;
      if (MODE >= 1) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(x));
      acc += x;
    }
  }
  long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"ld.x32+wait", "ld.x32+wait+32 tanh", "32 tanh only"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16}) {
      const int iters = 4000;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, warps * 32>>>(out, iters, cyc);
        else if (mode == 1) k<1><<<148, warps * 32>>>(out, iters, cyc);
        else k<2><<<148, warps * 32>>>(out, iters, cyc);
      }
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double mean = 0;
      for (int i = 0; i < 148; ++i) mean += h[i];
      mean /= 148;
      const double bytes = (double)warps * iters * 32 * 32 * 4;   // per SM
      printf("%-22s warps/SM=%2d  cycles/iter/warp=%7.1f  TMEM B/clk/SM=%6.1f\n", names[mode],
             warps, mean / iters, mode == 2 ? 0.0 : bytes / mean);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
