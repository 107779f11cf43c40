// Microbenchmark: issue rate of the 16-bit pack conversion (F2FP) alone and mixed with
// MUFU tanh, 16 warps/SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 cvt_rate.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(unsigned* out, int iters, long long* cyc) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = 0.001f * (threadIdx.x + i);
  unsigned acc = 0;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float a = x[i], b = x[i + 1];
      if (OP == 1 || OP == 2) {
        asm volatile("tanh.approx.f32 %0, %0;" : "+f"(a));
        asm volatile("tanh.approx.f32 %0, %0;" : "+f"(b));
      }
      if (OP == 0 || OP == 2) {
        __half2 h = __floats2half2_rn(a, b);
        acc ^= *reinterpret_cast<unsigned*>(&h);
      } else {
        acc ^= __float_as_uint(a) ^ __float_as_uint(b);
      }
      x[i] += 1e-7f;
      x[i + 1] += 1e-7f;
    }
  }
  long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
}

int main() {
  unsigned* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"8 F2FP pack", "16 tanh", "16 tanh + 8 F2FP"};
  for (int op = 0; op < 3; ++op) {
    const int warps = 16, iters = 2000;
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) k<0><<<148, warps * 32>>>(out, iters, cyc);
      else if (op == 1) k<1><<<148, warps * 32>>>(out, iters, cyc);
      else k<2><<<148, warps * 32>>>(out, iters, cyc);
    }
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i];
    mean /= 148;
    printf("%-20s cycles per iteration per SMSP (4 warps) = %.1f\n", names[op], mean / iters);
  }
  return 0;
}
