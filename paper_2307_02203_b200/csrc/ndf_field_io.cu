// Binary data plane of /api/reconstruct and /api/diff (service.py:392-416 of the reference):
// the response body is the field as little-endian fp32 values and its headers carry the
// value range (_field_headers, service.py:352-360).  One pass over the device field
// writes the body (optionally a - b, optionally clipped to [-1, 1] as reconstruct_field's
// clamp) straight into its destination -- page-locked host memory, so the stores go over
// PCIe as the kernel runs -- and reduces min / max on the way.
//
// Unit: one value, 4 B read (8 for a difference) + 4 B written; HBM / PCIe-write bound.
#include "ndf_common.cuh"
#include "ndf_query.cuh"

namespace ndf {

constexpr int kExportThreads = 256;

__device__ __forceinline__ float export_value(const float* __restrict__ a,
                                              const float* __restrict__ b, int64_t i, bool clamp) {
  float v = __ldg(a + i);
  if (b) v = __fsub_rn(v, __ldg(b + i));           // fa.values - fb.values (service.py:87-94)
  if (clamp && !(v != v)) v = fminf(fmaxf(v, -1.0f), 1.0f);   // np.clip keeps NaN
  return v;
}

__global__ void __launch_bounds__(kExportThreads)
field_export_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                    float* __restrict__ dst, uint32_t* __restrict__ stats, int clamp) {
  float lo = INFINITY, hi = -INFINITY;
  uint32_t nan = 0u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(dst) |
                     reinterpret_cast<uintptr_t>(b)) & 15u) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
    float4 v = __ldg(reinterpret_cast<const float4*>(a) + q);
    if (b) {
      const float4 w = __ldg(reinterpret_cast<const float4*>(b) + q);
      v.x = __fsub_rn(v.x, w.x); v.y = __fsub_rn(v.y, w.y);
      v.z = __fsub_rn(v.z, w.z); v.w = __fsub_rn(v.w, w.w);
    }
    float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (e[u] != e[u]) { nan = 1u; continue; }
      if (clamp) e[u] = fminf(fmaxf(e[u], -1.0f), 1.0f);
      lo = fminf(lo, e[u]);
      hi = fmaxf(hi, e[u]);
    }
    reinterpret_cast<float4*>(dst)[q] = make_float4(e[0], e[1], e[2], e[3]);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = export_value(a, b, i, clamp != 0);
    dst[i] = v;
    if (v != v) {
      nan = 1u;
    } else {
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
  }
  __shared__ float slo[kExportThreads / 32], shi[kExportThreads / 32];
  __shared__ uint32_t snan[kExportThreads / 32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { slo[w] = lo; shi[w] = hi; snan[w] = nan; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kExportThreads / 32; ++i) {
      lo = fminf(lo, slo[i]);
      hi = fmaxf(hi, shi[i]);
      nan |= snan[i];
    }
    if (lo <= hi) {                                 // this block saw a non-NaN value
      atomicMin(&stats[0], ordered_key(lo));
      atomicMax(&stats[1], ordered_key(hi));
    }
    if (nan) atomicOr(&stats[2], 1u);
  }
}

}  // namespace ndf

using namespace ndf;

extern "C" int ndf_field_export(const float* a, const float* b, int64_t n, float* dst,
                                uint32_t* stats, int32_t clamp, void* stream) {
  NDF_REQUIRE(n >= 0, NDF_ERR_PARAMETER, "negative length");
  NDF_REQUIRE(stats, NDF_ERR_PARAMETER, "null stats");
  cudaStream_t s = as_stream(stream);
  NDF_CUDA_CHECK(cudaMemsetAsync(stats, 0xff, sizeof(uint32_t), s));           // min key
  NDF_CUDA_CHECK(cudaMemsetAsync(stats + 1, 0, 2 * sizeof(uint32_t), s));      // max key, NaN
  if (n == 0) return NDF_OK;
  NDF_REQUIRE(a && dst, NDF_ERR_PARAMETER, "null pointer");
  const int64_t want = (n / 4 + kExportThreads - 1) / kExportThreads + 1;
  const int grid = (int)std::min<int64_t>(want, (int64_t)sm_count() * 8);
  field_export_kernel<<<grid, kExportThreads, 0, s>>>(a, b, n, dst, stats, clamp ? 1 : 0);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}
