// Shared launch arguments of the two NDF query kernels.
#pragma once
#include "ndf_embed.cuh"

namespace ndf {

struct QueryArgs {
  ndf_model_desc m;
  EmbedGeom g;
  int mode;                 // 0 = output grid (ref vs all nodes), 1 = point pairs
  int ref_is_mu;            // ROLE_MU (service.py:63-80)
  double ref[3];
  int nx, ny, nz;
  int64_t v0, v1;
  const double* p_mu;       // points mode
  int64_t n_mu;
  const double* p_nu;
  float* out;
  int prec;                 // NDF_PREC_*
  uint32_t* stats;          // optional value range of the outputs (ndf_query_grid_stats)
};

// fp32 -> uint32 key whose unsigned order is the float order (NaN kept aside)
__device__ __forceinline__ uint32_t ordered_key(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Per-thread min / max / NaN of the values a thread stores; flush() folds a warp with
// redux.sync (any active mask) and one lane updates stats = {min key, max key, NaN}.
struct RangeAcc {
  float lo = INFINITY, hi = -INFINITY;
  uint32_t nan = 0u;
  __device__ __forceinline__ void add(float v) {
    if (v != v) {
      nan = 1u;
    } else {
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
  }
  __device__ __forceinline__ void flush(uint32_t* stats) const {
    const unsigned m = __activemask();
    const bool any = lo <= hi;
    const uint32_t kl = __reduce_min_sync(m, any ? ordered_key(lo) : 0xffffffffu);
    const uint32_t kh = __reduce_max_sync(m, any ? ordered_key(hi) : 0u);
    const uint32_t nn = __reduce_or_sync(m, nan);
    if ((int)(threadIdx.x & 31) == __ffs(m) - 1) {
      if (kl != 0xffffffffu) atomicMin(&stats[0], kl);
      if (kh != 0u) atomicMax(&stats[1], kh);
      if (nn) atomicOr(&stats[2], 1u);
    }
  }
};

// flat vertex (x fastest) -> node coordinates (measures.py:240-252)
__device__ __forceinline__ void vertex_position(const QueryArgs& a, int64_t v, double* p) {
  const int64_t plane = (int64_t)a.nx * a.ny;
  const int iz = (int)(v / plane);
  const int64_t r = v - (int64_t)iz * plane;
  const int iy = (int)(r / a.nx);
  const int ix = (int)(r - (int64_t)iy * a.nx);
  p[0] = node_coord(ix, a.nx);
  p[1] = node_coord(iy, a.ny);
  p[2] = node_coord(iz, a.nz);
}

int validate_model(const ndf_model_desc* m);
int launch_query_f32(const QueryArgs& a, cudaStream_t s);
int launch_query_tc(const QueryArgs& a, cudaStream_t s);

}  // namespace ndf
