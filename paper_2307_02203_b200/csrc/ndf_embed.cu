// Positional encoder as a standalone kernel (K1): NdfModel.embed (model.py:169-177).
//
// The query kernels fuse the encoder (per-axis tables + the latent gather in the
// producer warps), so this entry point is the drop-in for callers that want the
// embedding itself -- the reference's forward_trace / training path and NdfModel.embed
// -- and the standalone measurement of the encoder's gather.  Same fp64 arithmetic as
// embed_point (ndf_embed.cuh), so every feature is bit-identical to the reference's
// fp64 -> fp32 embedding.
//
// Layout: one thread per point; the E features of the block's 128 points are staged in
// SMEM ([point][E + 1], odd stride against bank conflicts) and written back as one
// contiguous (128 x E) fp32 slab, so the stores are coalesced.
#include "ndf_query.cuh"

namespace ndf {

constexpr int kEmbThreads = 128;

// mode 0: grid nodes [v0, v0 + n) of an nx x ny x nz output grid (x fastest,
// node_coord positions, measures.py:240-252); mode 1: fp64 points pos[3 i ..].
__global__ void __launch_bounds__(kEmbThreads)
embed_kernel(const ndf_model_desc m, const EmbedGeom g, int branch, int mode, int nx, int ny,
             int nz, int64_t v0, const double* __restrict__ pos, int64_t n,
             float* __restrict__ out) {
  extern __shared__ float stage[];
  const int E = g.E;
  const int ld = E + 1;
  const float* grid = branch == 0 ? m.grid_mu : m.grid_nu;
  const int64_t base = (int64_t)blockIdx.x * kEmbThreads;
  const int64_t i = base + threadIdx.x;
  if (i < n) {
    double p[3];
    if (mode == 0) {
      const int64_t v = v0 + i;
      const int64_t plane = (int64_t)nx * ny;
      const int iz = (int)(v / plane);
      const int64_t r = v - (int64_t)iz * plane;
      const int iy = (int)(r / nx);
      const int ix = (int)(r - (int64_t)iy * nx);
      p[0] = node_coord(ix, nx);
      p[1] = node_coord(iy, ny);
      p[2] = node_coord(iz, nz);
    } else {
      p[0] = pos[3 * i];
      p[1] = pos[3 * i + 1];
      p[2] = pos[3 * i + 2];
    }
    float* row = stage + threadIdx.x * ld;
    embed_point(g, grid, p[0], p[1], p[2], [&](int k, float x) { row[k] = x; });
  }
  __syncthreads();
  const int64_t rows = min((int64_t)kEmbThreads, n - base);
  float* dst = out + base * E;
  for (int64_t k = threadIdx.x; k < rows * E; k += kEmbThreads) {
    const int r = (int)(k / E), c = (int)(k - (int64_t)r * E);
    dst[k] = stage[r * ld + c];
  }
}

static int launch_embed(const ndf_model_desc* m, int32_t branch, int mode, int nx, int ny, int nz,
                        int64_t v0, const double* pos, int64_t n, float* out, void* stream) {
  int st = validate_model(m);
  if (st) return st;
  NDF_REQUIRE(branch == 0 || branch == 1, NDF_ERR_PARAMETER, "branch must be 0 (mu) or 1 (nu)");
  NDF_REQUIRE(n >= 0, NDF_ERR_PARAMETER, "negative count");
  if (n == 0) return NDF_OK;
  NDF_REQUIRE(out != nullptr, NDF_ERR_PARAMETER, "null output");
  void* out_dev = nullptr;
  if ((st = resolve_output(out, &out_dev))) return st;
  const EmbedGeom g = make_geom(*m);
  const size_t smem = (size_t)kEmbThreads * (g.E + 1) * sizeof(float);
  static SmemAttrCache attr;
  NDF_CUDA_CHECK(attr.ensure(embed_kernel, (size_t)kEmbThreads * (kMaxEmbed + 1) * sizeof(float)));
  embed_kernel<<<(unsigned)((n + kEmbThreads - 1) / kEmbThreads), kEmbThreads, smem,
                 as_stream(stream)>>>(*m, g, branch, mode, nx, ny, nz, v0, pos, n,
                                      static_cast<float*>(out_dev));
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

}  // namespace ndf

using namespace ndf;

extern "C" int ndf_embed_nodes(const ndf_model_desc* m, int32_t branch, int32_t nx, int32_t ny,
                               int32_t nz, int64_t v0, int64_t v1, float* out, void* stream) {
  NDF_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, NDF_ERR_PARAMETER, "grid dims must be >= 1");
  const int64_t V = (int64_t)nx * ny * nz;
  NDF_REQUIRE(v0 >= 0 && v0 <= v1 && v1 <= V, NDF_ERR_PARAMETER, "vertex range out of bounds");
  NDF_REQUIRE((v1 - v0) < (1LL << 31) / 140, NDF_ERR_UNSUPPORTED, "too many nodes for one launch");
  return launch_embed(m, branch, 0, nx, ny, nz, v0, nullptr, v1 - v0, out, stream);
}

extern "C" int ndf_embed_points(const ndf_model_desc* m, int32_t branch, const double* pos,
                                int64_t n, float* out, void* stream) {
  NDF_REQUIRE(pos != nullptr || n == 0, NDF_ERR_PARAMETER, "null positions");
  NDF_REQUIRE(n < (1LL << 31) / 140, NDF_ERR_UNSUPPORTED, "too many points for one launch");
  return launch_embed(m, branch, 1, 1, 1, 1, 0, pos, n, out, stream);
}
