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
