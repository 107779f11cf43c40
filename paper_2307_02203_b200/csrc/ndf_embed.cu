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
// contiguous (128 x E) fp32 slab, so the stores are coalesced.  Grid nodes of dense-latent
// models take the separable per-axis route (embed_nodes_kernel below).
#include <algorithm>

#include "ndf_query.cuh"

namespace ndf {

constexpr int kEmbThreads = 128;

// Coalesced store of the block's staged (rows x E) slab (SMEM row stride ld): flat
// element k = r * E + c; the row index comes from one float multiply (exact here:
// k < 128 * 140, so (k + 0.5) / E never lies within float error of an integer) instead
// of an integer division per element.
__device__ __forceinline__ void store_slab(const float* stage, int ld, int E, int rows,
                                           float* __restrict__ dst) {
  const float invE = 1.0f / (float)E;
  const int total = rows * E;
  auto at = [&](int k) {
    const int r = (int)(((float)k + 0.5f) * invE);
    return stage[r * ld + (k - r * E)];
  };
  // scalar head up to the first 16-byte boundary, 16-byte stores, scalar tail
  const int head = min(total, (int)(((16u - (reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u) >> 2));
  if ((int)threadIdx.x < head) dst[threadIdx.x] = at(threadIdx.x);
  const int t4 = (total - head) >> 2;
  float4* d4 = reinterpret_cast<float4*>(dst + head);
  for (int q = threadIdx.x; q < t4; q += kEmbThreads)
    d4[q] = make_float4(at(head + 4 * q), at(head + 4 * q + 1), at(head + 4 * q + 2),
                        at(head + 4 * q + 3));
  for (int k = head + 4 * t4 + threadIdx.x; k < total; k += kEmbThreads) dst[k] = at(k);
}

// Odd E (ld == E): the staged rows ARE the slab in order, so when the rows start at
// stage + slab_off(dst) the 16-byte stores read their 4 values with one aligned LDS.128
// (the generic store_slab's 4 scalar reads per float4 hit 4-way bank conflicts).
__device__ __forceinline__ int slab_head(const float* dst) {
  return (int)(((16u - (reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u) >> 2);
}
__device__ __forceinline__ int slab_off(const float* dst) { return (4 - slab_head(dst)) & 3; }
__device__ __forceinline__ void store_slab_lin(const float* lin, int total, float* __restrict__ dst) {
  const int head = min(total, slab_head(dst));
  if ((int)threadIdx.x < head) dst[threadIdx.x] = lin[threadIdx.x];
  const int t4 = (total - head) >> 2;
  const float4* s4 = reinterpret_cast<const float4*>(lin + head);
  float4* d4 = reinterpret_cast<float4*>(dst + head);
  for (int q = threadIdx.x; q < t4; q += kEmbThreads) d4[q] = s4[q];
  for (int k = head + 4 * t4 + threadIdx.x; k < total; k += kEmbThreads) dst[k] = lin[k];
}
// stage rows (ld floats apart) at stage_base(stage, ld, E, dst), then store_rows
__device__ __forceinline__ float* stage_base(float* stage, int ld, int E, const float* dst) {
  return ld == E ? stage + slab_off(dst) : stage;
}
__device__ __forceinline__ void store_rows(const float* base, int ld, int E, int rows,
                                           float* __restrict__ dst) {
  if (ld == E) store_slab_lin(base, rows * E, dst);
  else store_slab(base, ld, E, rows, dst);
}

// mode 0: grid nodes [v0, v0 + n) of an nx x ny x nz output grid (x fastest,
// node_coord positions, measures.py:240-252); mode 1: fp64 points pos[3 i ..].
__global__ void __launch_bounds__(kEmbThreads)
embed_kernel(const ndf_model_desc m, const EmbedGeom g, int branch, int mode, int nx, int ny,
             int nz, int64_t v0, const double* __restrict__ pos, int64_t n,
             float* __restrict__ out) {
  extern __shared__ float stage[];
  const int E = g.E;
  const int ld = E | 1;            // odd row stride: the per-thread row writes hit 32 banks
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
    float* row = stage_base(stage, ld, E, out + base * E) + threadIdx.x * ld;
    embed_point(g, grid, p[0], p[1], p[2], [&](int k, float x) { row[k] = x; });
  }
  __syncthreads();
  store_rows(stage_base(stage, ld, E, out + base * E), ld, E,
             (int)min((int64_t)kEmbThreads, n - base), out + base * E);
}

// ---- grid nodes of a dense-latent model: separable per axis ----------------------
// Every feature of a grid node except the latent channels depends on ONE axis node
// (raw p, Fourier sin / cos), and so do the latent cell (i0, t) per axis: an axis table
// computed once per launch (one fp64 sincos per node x octave, the same operations as
// embed_point -> the same bits) turns the node embedding into table reads plus the fp64
// eight-corner latent sum -- so the launch is bound by writing the (V, E) output.
constexpr int kAxisRowF = 32;       // [p | sin, cos x L (L <= 12) | pad | t (fp64) | i0]

__global__ void embed_axis_kernel(const EmbedGeom g, int nx, int ny, int nz, float* __restrict__ tab) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  const int nodes = nx + ny + nz;
  const int L = g.L;
  if (item >= nodes * (L + 1)) return;
  const int node = item / (L + 1), o = item % (L + 1);
  int i, n, res;
  if (node < nx) { i = node; n = nx; res = g.rx; }
  else if (node < nx + ny) { i = node - nx; n = ny; res = g.ry; }
  else { i = node - nx - ny; n = nz; res = g.rz; }
  const double p = fmin(fmax(node_coord(i, n), -1.0), 1.0);
  float* row = tab + (size_t)node * kAxisRowF;
  if (o == L) {                       // raw coordinate and the latent cell of this axis
    row[0] = (float)p;
    const AxisCoord c = level_coord(p, res);
    reinterpret_cast<double*>(row)[14] = c.t;      // floats 28-29
    reinterpret_cast<int*>(row)[30] = c.i0;
    return;
  }
  double scale = 3.141592653589793;
  for (int k = 0; k < o; ++k) scale = scale * 2.0;
  double sn, cs;
  sincos(dmul(scale, p), &sn, &cs);
  row[1 + 2 * o] = (float)sn;
  row[2 + 2 * o] = (float)cs;
}

#ifndef NDF_EMB_MINBLOCKS
#define NDF_EMB_MINBLOCKS 6      // 80 registers: 6 CTAs per SM (measured best of 1 / 6 / 8 / 12)
#endif
__global__ void __launch_bounds__(kEmbThreads, NDF_EMB_MINBLOCKS)
embed_nodes_kernel(const ndf_model_desc m, const EmbedGeom g, int branch, int nx, int ny, int nz,
                   int64_t v0, int64_t n, const float* __restrict__ tab, float* __restrict__ out) {
  extern __shared__ float stage[];
  const int E = g.E, L = g.L, C = g.C;
  const int ld = E | 1;            // odd row stride: the per-thread row writes hit 32 banks
  const float* grid = branch == 0 ? m.grid_mu : m.grid_nu;
  const int64_t base = (int64_t)blockIdx.x * kEmbThreads;
  const int64_t i = base + threadIdx.x;
  if (i < n) {
    const int64_t v = v0 + i;
    const int64_t plane = (int64_t)nx * ny;
    const int iz = (int)(v / plane);
    const int64_t r = v - (int64_t)iz * plane;
    const int iy = (int)(r / nx);
    const int ix = (int)(r - (int64_t)iy * nx);
    const float* rows[3] = {tab + (size_t)ix * kAxisRowF, tab + (size_t)(nx + iy) * kAxisRowF,
                            tab + (size_t)(nx + ny + iz) * kAxisRowF};
    float* dst = stage_base(stage, ld, E, out + base * E) + threadIdx.x * ld;
    // axis rows: [p | sin_0, cos_0, ..., sin_{L-1}, cos_{L-1} | ...], 128-byte aligned:
    // 16-byte loads of the first 4 (L + 1) / 4 quads, scattered into embed_point's order
    // [p_xyz | (sin, cos)_x, (sin, cos)_y, (sin, cos)_z per octave]
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const float4* r4 = reinterpret_cast<const float4*>(rows[ax]);
      for (int q = 0; 4 * q < 1 + 2 * L; ++q) {
        const float4 f = __ldg(r4 + q);
        const float e4[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;                  // position in the axis row
          if (j == 0) dst[ax] = e4[u];
          else if (j <= 2 * L) dst[3 + 6 * ((j - 1) >> 1) + 2 * ax + ((j - 1) & 1)] = e4[u];
        }
      }
    }
    // latent: embed_point's corner order, weights ((wx) * wy) * wz and fp64 sums
    double tt[3];
    int i0[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      tt[ax] = __ldg(reinterpret_cast<const double*>(rows[ax]) + 14);
      i0[ax] = __ldg(reinterpret_cast<const int*>(rows[ax]) + 30);
    }
    double w[8];
    int idx[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
      const double wx = dx ? tt[0] : dsub(1.0, tt[0]);
      const double wy = dy ? tt[1] : dsub(1.0, tt[1]);
      const double wz = dz ? tt[2] : dsub(1.0, tt[2]);
      w[c] = dmul(dmul(wx, wy), wz);
      idx[c] = (i0[0] + dx) + g.rx * ((i0[1] + dy) + g.ry * (i0[2] + dz));
    }
    const int lb = 3 + 6 * L;
    if (C == 16) {
      // corner-outer with 16-byte loads; per channel the corner order (and so the
      // fp64 rounding sequence) is embed_point's
      double acc[16];
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) acc[ch] = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4* rowp = reinterpret_cast<const float4*>(grid + (size_t)idx[c] * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 f = __ldg(rowp + q);
          acc[4 * q + 0] = dadd(acc[4 * q + 0], dmul(w[c], (double)f.x));
          acc[4 * q + 1] = dadd(acc[4 * q + 1], dmul(w[c], (double)f.y));
          acc[4 * q + 2] = dadd(acc[4 * q + 2], dmul(w[c], (double)f.z));
          acc[4 * q + 3] = dadd(acc[4 * q + 3], dmul(w[c], (double)f.w));
        }
      }
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) dst[lb + ch] = (float)acc[ch];
    } else {
      for (int ch = 0; ch < C; ++ch) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          acc = dadd(acc, dmul(w[c], (double)__ldg(grid + (size_t)idx[c] * C + ch)));
        dst[lb + ch] = (float)acc;
      }
    }
  }
  __syncthreads();
  store_rows(stage_base(stage, ld, E, out + base * E), ld, E,
             (int)min((int64_t)kEmbThreads, n - base), out + base * E);
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
  const size_t smem = ((size_t)kEmbThreads * (g.E + 1) + 4) * sizeof(float);
  if (mode == 0 && g.levels == 0) {
    // dense-latent model over grid nodes: per-axis tables, then table reads + latent sum
    static SmemAttrCache attr_n;
    NDF_CUDA_CHECK(attr_n.ensure(embed_nodes_kernel,
                                 ((size_t)kEmbThreads * (kMaxEmbed + 1) + 4) * sizeof(float)));
    const int nodes = nx + ny + nz;
    void* tab = nullptr;
    NDF_CUDA_CHECK(scratch_alloc(&tab, (size_t)nodes * kAxisRowF * sizeof(float),
                                 as_stream(stream)));
    const int items = nodes * (g.L + 1);
    embed_axis_kernel<<<(items + 127) / 128, 128, 0, as_stream(stream)>>>(g, nx, ny, nz,
                                                                          static_cast<float*>(tab));
    cudaError_t e = cudaGetLastError();
    count_launch();
    if (e == cudaSuccess) {
      embed_nodes_kernel<<<(unsigned)((n + kEmbThreads - 1) / kEmbThreads), kEmbThreads, smem,
                           as_stream(stream)>>>(*m, g, branch, nx, ny, nz, v0, n,
                                                static_cast<const float*>(tab),
                                                static_cast<float*>(out_dev));
      e = cudaGetLastError();
      count_launch();
    }
    cudaFreeAsync(tab, as_stream(stream));
    NDF_CUDA_CHECK(e);
    return NDF_OK;
  }
  static SmemAttrCache attr;
  NDF_CUDA_CHECK(attr.ensure(embed_kernel, ((size_t)kEmbThreads * (kMaxEmbed + 1) + 4) * sizeof(float)));
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
