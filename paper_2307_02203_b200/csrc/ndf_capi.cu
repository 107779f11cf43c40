// C-ABI plumbing: thread-local last error, launch counter, device queries.
#include <atomic>
#include <string>

#include "ndf_common.cuh"

namespace ndf {

static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) { g_launches += n; }

int sm_count() {
  static thread_local int cached_dev = -1;
  static thread_local int cached = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cached;
  if (dev != cached_dev) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    cached_dev = dev;
  }
  return cached;
}

// Stream-ordered scratch from the device's default memory pool.  The pool's release
// threshold is raised once per device so synchronising callers (one query per
// host round trip) do not pay an unmap / remap on every call.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured != dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    configured = dev;
  }
  return cudaMallocAsync(p, bytes, s);
}

int resolve_output(void* p, void** dev) {
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("output pointer: ") + cudaGetErrorString(e));
    return NDF_ERR_PARAMETER;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    *dev = p;
    return NDF_OK;
  }
  if (at.type == cudaMemoryTypeHost && at.devicePointer != nullptr) {
    *dev = at.devicePointer;   // page-locked host memory: the kernel writes it over PCIe
    return NDF_OK;
  }
  set_error("output must be device memory or page-locked (pinned) host memory");
  return NDF_ERR_PARAMETER;
}

}  // namespace ndf

extern "C" int32_t ndf_abi_version(void) { return NDF_ABI_VERSION; }

extern "C" const char* ndf_last_error(void) { return ndf::g_last_error.c_str(); }

extern "C" int32_t ndf_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

extern "C" int64_t ndf_launch_count(int32_t reset) {
  const int64_t n = ndf::g_launches;
  if (reset) ndf::g_launches = 0;
  return n;
}
