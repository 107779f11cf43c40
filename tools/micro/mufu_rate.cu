// Microbenchmark: issue rate of MUFU variants on sm_100a (cycles per warp-instruction
// per SM sub-partition).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = 0.001f * (threadIdx.x + i);
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      else if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      else if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      else if (OP == 3) { unsigned h = __float_as_uint(x[i]), r;
        asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h)); y = __uint_as_float(r); }
      else if (OP == 4) { unsigned h = __float_as_uint(x[i]), r;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h)); y = __uint_as_float(r); }
      else y = fmaf(x[i], 1.0001f, 0.5f);
      x[i] = y * 0.5f;
    }
  }
  long long c1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"tanh.f32", "ex2.f32", "rcp.f32", "tanh.f16x2", "ex2.f16x2", "ffma(+fmul)"};
  for (int op = 0; op < 6; ++op) {
    for (int warps : {4, 16}) {
      const int iters = 2000;
      auto launch = [&]() {
        switch (op) {
          case 0: k<0><<<148, warps * 32>>>(out, iters, cyc); break;
          case 1: k<1><<<148, warps * 32>>>(out, iters, cyc); break;
          case 2: k<2><<<148, warps * 32>>>(out, iters, cyc); break;
          case 3: k<3><<<148, warps * 32>>>(out, iters, cyc); break;
          case 4: k<4><<<148, warps * 32>>>(out, iters, cyc); break;
          default: k<5><<<148, warps * 32>>>(out, iters, cyc); break;
        }
      };
      launch(); cudaDeviceSynchronize();
      launch(); cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double c = h[0];
      // instructions of this op per SMSP: warps/4 * iters * 8
      double per_smsp = (double)warps / 4 * iters * 8;
      printf("%-12s warps/SM=%2d  cycles per warp-op per SMSP = %.2f  (ops/clk/SM = %.1f)\n",
             names[op], warps, c / per_smsp, 4 * 32 * per_smsp / c / 1.0);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
