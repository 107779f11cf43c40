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
// eight-corner latent sum.  The table is feature-major ([feature][axis node], then t and
// i0 per axis node), so a warp's 32 consecutive x-nodes read each feature as one
// coalesced 128-byte row instead of 32 scattered table rows.
struct AxisTab {
  const float* f;      // [1 + 2L][nodes]: p, (sin, cos) per octave
  const double* t;     // [nodes]
  const int* i0;       // [nodes]
  int nodes;
};

__host__ __device__ inline size_t axis_tab_bytes(int L, int nodes) {
  return (((size_t)(1 + 2 * L) * nodes * 4 + 15) & ~(size_t)15) + (size_t)nodes * 8 +
         (size_t)nodes * 4;
}
__host__ __device__ inline AxisTab axis_tab(void* base, int L, int nodes) {
  AxisTab T;
  uint8_t* p = static_cast<uint8_t*>(base);
  T.f = reinterpret_cast<const float*>(p);
  p += ((size_t)(1 + 2 * L) * nodes * 4 + 15) & ~(size_t)15;
  T.t = reinterpret_cast<const double*>(p);
  T.i0 = reinterpret_cast<const int*>(p + (size_t)nodes * 8);
  T.nodes = nodes;
  return T;
}

__global__ void embed_axis_kernel(const EmbedGeom g, int nx, int ny, int nz, AxisTab T) {
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
  float* f = const_cast<float*>(T.f);
  if (o == L) {                       // raw coordinate and the latent cell of this axis
    f[node] = (float)p;
    const AxisCoord c = level_coord(p, res);
    const_cast<double*>(T.t)[node] = c.t;
    const_cast<int*>(T.i0)[node] = c.i0;
    return;
  }
  double scale = 3.141592653589793;
  for (int k = 0; k < o; ++k) scale = scale * 2.0;
  double sn, cs;
  sincos(dmul(scale, p), &sn, &cs);
  f[(size_t)(1 + 2 * o) * nodes + node] = (float)sn;
  f[(size_t)(2 + 2 * o) * nodes + node] = (float)cs;
}

// Latent corners of a warp's 32 nodes: when they lie in one (y, z)-row, their x cells form
// a short run [c_lo, c_lo + S); the warp copies the 4 (dy, dz) x S x 16 corner values once,
// coalesced, into its own SMEM block (cell stride 20 floats: the lanes' 16-byte reads of
// different cells fall into different bank groups) and every lane reads its 8 corners
// from there -- instead of 32 scattered 16-byte global loads per node through L1, the
// kernel's bound before (L1 94% busy).  Warps that cross a row, or a run longer than
// kEmbCells, load their corners directly.
constexpr int kEmbCells = 12;
constexpr int kEmbCellStride = 20;
constexpr int kEmbWarpLat = 4 * kEmbCells * kEmbCellStride;     // floats per warp

#ifndef NDF_EMB_MINBLOCKS
#define NDF_EMB_MINBLOCKS 5
#endif
__global__ void __launch_bounds__(kEmbThreads, NDF_EMB_MINBLOCKS)
embed_nodes_kernel(const ndf_model_desc m, const EmbedGeom g, int branch, int nx, int ny, int nz,
                   int64_t v0, int64_t n, const AxisTab T, float* __restrict__ out) {
  extern __shared__ __align__(16) float stage[];
  const int E = g.E, L = g.L, C = g.C;
  const int ld = E | 1;            // odd row stride: the per-thread row writes hit 32 banks
  const float* grid = branch == 0 ? m.grid_mu : m.grid_nu;
  const int64_t base = (int64_t)blockIdx.x * kEmbThreads;
  const int64_t i = base + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* latw = stage + ((kEmbThreads * ld + 4 + 3) & ~3) + warp * kEmbWarpLat;
  const int64_t plane = (int64_t)nx * ny;
  const int64_t vi = v0 + min(i, n - 1);
  const int iz = (int)(vi / plane);
  const int64_t rr = vi - (int64_t)iz * plane;
  const int iy = (int)(rr / nx);
  const int ix = (int)(rr - (int64_t)iy * nx);
  const int nodes = T.nodes;
  // one (y, z)-row for the whole warp, every lane a node of the launch?
  const int64_t wlast = base + 32 * warp + 31;
  const bool full = wlast < n;
  const int row = iy + ny * iz;
  const bool one_row = full && __shfl_sync(0xffffffffu, row, 0) == __shfl_sync(0xffffffffu, row, 31);
  const int i0x = __ldg(T.i0 + ix);
  const int c_lo = __shfl_sync(0xffffffffu, i0x, 0);
  const int S = __shfl_sync(0xffffffffu, i0x, 31) + 2 - c_lo;
  const int i0y = __ldg(T.i0 + nx + iy), i0z = __ldg(T.i0 + nx + ny + iz);
  const bool staged = C == 16 && one_row && S <= kEmbCells;
  if (staged) {
    for (int it = lane; it < 16 * S; it += 32) {
      const int combo = it / (4 * S), rem = it - combo * 4 * S;
      const int cell = rem >> 2, q = rem & 3;
      const int idx = (c_lo + cell) + g.rx * ((i0y + (combo & 1)) + g.ry * (i0z + (combo >> 1)));
      const float4 f = __ldg(reinterpret_cast<const float4*>(grid + (size_t)idx * 16) + q);
      *reinterpret_cast<float4*>(latw + (combo * S + cell) * kEmbCellStride + 4 * q) = f;
    }
    __syncwarp();
  }
  float* const sbase = stage_base(stage, ld, E, out + base * E);
  if (i < n) {
    float* dst = sbase + threadIdx.x * ld;
    const int an[3] = {ix, nx + iy, nx + ny + iz};
    // [p_xyz | (sin, cos)_x, (sin, cos)_y, (sin, cos)_z per octave], feature-major reads
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      dst[ax] = __ldg(T.f + an[ax]);
      for (int o = 0; o < L; ++o) {
        dst[3 + 6 * o + 2 * ax] = __ldg(T.f + (size_t)(1 + 2 * o) * nodes + an[ax]);
        dst[3 + 6 * o + 2 * ax + 1] = __ldg(T.f + (size_t)(2 + 2 * o) * nodes + an[ax]);
      }
    }
    // latent: embed_point's corner order, weights ((wx) * wy) * wz and fp64 sums
    const double tt[3] = {__ldg(T.t + an[0]), __ldg(T.t + an[1]), __ldg(T.t + an[2])};
    double w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
      const double wx = dx ? tt[0] : dsub(1.0, tt[0]);
      const double wy = dy ? tt[1] : dsub(1.0, tt[1]);
      const double wz = dz ? tt[2] : dsub(1.0, tt[2]);
      w[c] = dmul(dmul(wx, wy), wz);
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
        const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
        const float4* rowp =
            staged ? reinterpret_cast<const float4*>(latw + ((c >> 1) * S + (i0x - c_lo + dx)) *
                                                                kEmbCellStride)
                   : reinterpret_cast<const float4*>(
                         grid + (size_t)((i0x + dx) + g.rx * ((i0y + dy) + g.ry * (i0z + dz))) * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 f = staged ? rowp[q] : __ldg(rowp + q);
          acc[4 * q + 0] = dadd(acc[4 * q + 0], dmul(w[c], (double)f.x));
          acc[4 * q + 1] = dadd(acc[4 * q + 1], dmul(w[c], (double)f.y));
          acc[4 * q + 2] = dadd(acc[4 * q + 2], dmul(w[c], (double)f.z));
          acc[4 * q + 3] = dadd(acc[4 * q + 3], dmul(w[c], (double)f.w));
        }
      }
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) dst[lb + ch] = (float)acc[ch];
    } else {
      int idx[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        idx[c] = (i0x + (c & 1)) + g.rx * ((i0y + ((c >> 1) & 1)) + g.ry * (i0z + (c >> 2)));
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
  store_rows(sbase, ld, E, (int)min((int64_t)kEmbThreads, n - base), out + base * E);
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
    const int nodes = nx + ny + nz;
    void* tab = nullptr;
    NDF_CUDA_CHECK(scratch_alloc(&tab, axis_tab_bytes(g.L, nodes), as_stream(stream)));
    const AxisTab T = axis_tab(tab, g.L, nodes);
    const int items = nodes * (g.L + 1);
    embed_axis_kernel<<<(items + 127) / 128, 128, 0, as_stream(stream)>>>(g, nx, ny, nz, T);
    cudaError_t e = cudaGetLastError();
    count_launch();
    const size_t smem_n = ((((size_t)kEmbThreads * (g.E | 1) + 4 + 3) & ~(size_t)3) +
                           (size_t)4 * kEmbWarpLat) * sizeof(float);
    if (e == cudaSuccess)
      e = attr_n.ensure(embed_nodes_kernel,
                        ((((size_t)kEmbThreads * (kMaxEmbed + 1) + 4 + 3) & ~(size_t)3) +
                         (size_t)4 * kEmbWarpLat) * sizeof(float));
    if (e == cudaSuccess) {
      embed_nodes_kernel<<<(unsigned)((n + kEmbThreads - 1) / kEmbThreads), kEmbThreads, smem_n,
                           as_stream(stream)>>>(*m, g, branch, nx, ny, nz, v0, n, T,
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
