// Shared device/host helpers for libndf_b200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/ndf_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libndf_b200 targets sm_100a only"
#endif

namespace ndf {

// ---- error plumbing (host) -------------------------------------------------
void set_error(const std::string& msg);
void count_launch(int n = 1);

#define NDF_REQUIRE(cond, code, msg)                 \
  do {                                               \
    if (!(cond)) {                                   \
      ::ndf::set_error(msg);                         \
      return (code);                                 \
    }                                                \
  } while (0)

#define NDF_CUDA_CHECK(expr)                                             \
  do {                                                                   \
    cudaError_t _e = (expr);                                             \
    if (_e != cudaSuccess) {                                             \
      ::ndf::set_error(std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
      return NDF_ERR_CUDA;                                               \
    }                                                                    \
  } while (0)

#define NDF_LAUNCH_CHECK()                                               \
  do {                                                                   \
    ::ndf::count_launch();                                               \
    cudaError_t _e = cudaGetLastError();                                 \
    if (_e != cudaSuccess) {                                             \
      ::ndf::set_error(std::string("kernel launch failed: ") + cudaGetErrorString(_e)); \
      return NDF_ERR_CUDA;                                               \
    }                                                                    \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();
// Per-device record of the dynamic-SMEM size a kernel's attribute has been raised to
// (cudaFuncSetAttribute is per device); thread-safe, devices 0..63.
struct SmemAttrCache {
  size_t bytes[64] = {};
  template <class K>
  cudaError_t ensure(K kernel, size_t smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (__atomic_load_n(&bytes[dev], __ATOMIC_ACQUIRE) >= smem) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) __atomic_store_n(&bytes[dev], smem, __ATOMIC_RELEASE);
    return e;
  }
};
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);
// Output buffers may be device memory or page-locked host memory (UVA-mapped):
// sets *dev to the pointer a kernel stores through; NDF_ERR_PARAMETER for pageable memory.
int resolve_output(void* p, void** dev);

// ---- exact IEEE fp64 helpers (no FMA contraction) ---------------------------
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }

// Output-grid node coordinate: measures.py:245-248 / ensemble.py:51-54
//   2.0 * i / (n - 1) - 1.0, and 0.0 for a single-node axis.
__device__ __forceinline__ double node_coord(int i, int n) {
  if (n == 1) return 0.0;
  return dsub(ddiv(2.0 * (double)i, (double)(n - 1)), 1.0);
}

}  // namespace ndf
