// Positional encoder (K1): [raw xyz | Fourier(L) | dense latent grid(C)].
//
// Restates NdfModel.embed (model.py:169-177) for one dense latent level:
//   * clip to [-1, 1]                                   (model.py:174)
//   * fourier_encode: out[6i+2ax] = sin((2^i*pi)*p_ax), +1 = cos (encoding.py:37-51)
//   * latent lookup: per-axis _level_coords (encoding.py:105-113), corners in
//     _CORNER_OFFSETS order (encoding.py:116-118), weights ((1*wx)*wy)*wz
//     (encoding.py:156-160), fp64 corner sum in corner order (encoding.py:176)
//   * everything in fp64, cast once to fp32 (model.py:177).
// All fp64 basic ops use explicit _rn intrinsics, so the result is bit-identical
// to the NumPy reference wherever the reference is (sin/cos are libm-faithful
// and agree after the fp32 cast).
#pragma once
#include "ndf_common.cuh"

namespace ndf {

constexpr int kMaxEmbed = 3 + 6 * 12 + 64;   // L <= 12, latent (levels * C) <= 64

struct AxisCoord {
  int i0;
  double t;
};

// encoding.py:105-113: u = (clip(p)+1)*0.5*(res-1); i0 = clip(floor(u), 0, res-2);
// t = u - i0, snapped to {0, 1} within 1e-9.
__device__ __forceinline__ AxisCoord level_coord(double p, int res) {
  double pc = fmin(fmax(p, -1.0), 1.0);
  double u = dmul(dmul(dadd(pc, 1.0), 0.5), (double)(res - 1));
  double f = floor(u);
  int i0 = (int)f;
  if (i0 < 0) i0 = 0;
  if (i0 > res - 2) i0 = res - 2;
  double t = dsub(u, (double)i0);
  if (t < 1e-9) t = 0.0;
  if (t > 1.0 - 1e-9) t = 1.0;
  return {i0, t};
}

struct EmbedGeom {
  int L;         // Fourier octaves
  int C;         // latent channels (per level for HashGrids)
  int rx, ry, rz;
  int levels;    // 0: dense anisotropic level (rx, ry, rz); >= 1: HashGrid levels
  int log2T;     // HashGrid rows per level = 2^log2T
  int lres[NDF_MAX_LEVELS];
  int E;         // 3 + 6L + max(levels, 1) * C
};

__host__ __device__ inline EmbedGeom make_geom(const ndf_model_desc& m) {
  EmbedGeom g;
  g.L = m.fourier_octaves;
  g.C = m.grid_channels;
  g.rx = m.grid_res[0];
  g.ry = m.grid_res[1];
  g.rz = m.grid_res[2];
  g.levels = m.grid_levels;
  g.log2T = m.grid_log2_table;
  for (int l = 0; l < NDF_MAX_LEVELS; ++l) g.lres[l] = m.grid_level_res[l];
  g.E = 3 + 6 * g.L + (g.levels > 0 ? g.levels : 1) * g.C;
  return g;
}

// Table row of lattice corner (ix, iy, iz) on a HashGrid level of resolution res
// (encoding.py:90-102): dense when res^3 <= 2^T, else (ix*1 ^ iy*2654435761 ^
// iz*805459861) mod 2^T -- the low bits of the reference's uint64 products.
__device__ __forceinline__ int64_t hash_row(int res, int log2T, int ix, int iy, int iz) {
  const int64_t T = (int64_t)1 << log2T;
  if ((int64_t)res * res * res <= T) return (int64_t)ix + (int64_t)res * (iy + (int64_t)res * iz);
  const uint64_t h = (uint64_t)ix * 1ull ^ (uint64_t)iy * 2654435761ull ^ (uint64_t)iz * 805459861ull;
  return (int64_t)(h & (uint64_t)(T - 1));
}

// Write the fp32 embedding of position (px, py, pz) into out[0..E) via a
// functor store(idx, value) so callers can target registers, SMEM or global.
// `part` / `nparts` split the work of one point across cooperating threads (each
// writes a disjoint set of features, same arithmetic): part 0 does the raw and
// Fourier features, parts 1.. the latent levels round-robin.  part < 0: everything.
template <class Store>
__device__ __forceinline__ void embed_point(const EmbedGeom& g, const float* __restrict__ grid,
                                            double px, double py, double pz, Store store,
                                            int part = -1, int nparts = 1) {
  const double p[3] = {fmin(fmax(px, -1.0), 1.0), fmin(fmax(py, -1.0), 1.0),
                       fmin(fmax(pz, -1.0), 1.0)};
  const bool all = part < 0;
  if (all || part == 0) {
    store(0, (float)p[0]);
    store(1, (float)p[1]);
    store(2, (float)p[2]);
    double scale = 3.141592653589793;   // 2^i * pi, exact doubling
    for (int i = 0; i < g.L; ++i) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        double s, c;
        sincos(dmul(scale, p[ax]), &s, &c);
        store(3 + 6 * i + 2 * ax, (float)s);
        store(3 + 6 * i + 2 * ax + 1, (float)c);
      }
      scale = scale * 2.0;
    }
  }
  const int lstep = all ? 1 : (nparts > 1 ? nparts - 1 : 1);
  const int lfirst = all ? 0 : (nparts > 1 ? part - 1 : 0);
  if (!all && nparts > 1 && part == 0) return;
  if (g.levels > 0) {
    // HashGrid (encoding.py:149-178): per level, trilinear over the 8 corners in
    // _CORNER_OFFSETS order, weights ((1*wx)*wy)*wz and the corner sum in fp64,
    // output concatenated coarse to fine.
    const int64_t T = (int64_t)1 << g.log2T;
    for (int lv = lfirst; lv < g.levels; lv += lstep) {
      const int res = g.lres[lv];
      const AxisCoord cx = level_coord(p[0], res);
      const AxisCoord cy = level_coord(p[1], res);
      const AxisCoord cz = level_coord(p[2], res);
      double w[8];
      int64_t row[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
        const double wx = dx ? cx.t : dsub(1.0, cx.t);
        const double wy = dy ? cy.t : dsub(1.0, cy.t);
        const double wz = dz ? cz.t : dsub(1.0, cz.t);
        w[c] = dmul(dmul(wx, wy), wz);
        row[c] = hash_row(res, g.log2T, cx.i0 + dx, cy.i0 + dy, cz.i0 + dz);
      }
      const float* tab = grid + (size_t)lv * (size_t)T * g.C;
      const int base = 3 + 6 * g.L + lv * g.C;
      for (int ch = 0; ch < g.C; ++ch) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          acc = dadd(acc, dmul(w[c], (double)__ldg(tab + (size_t)row[c] * g.C + ch)));
        store(base + ch, (float)acc);
      }
    }
    return;
  }
  if (lfirst != 0) return;          // the single dense level belongs to part 1
  const AxisCoord cx = level_coord(p[0], g.rx);
  const AxisCoord cy = level_coord(p[1], g.ry);
  const AxisCoord cz = level_coord(p[2], g.rz);
  double w[8];
  int idx[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
    const double wx = dx ? cx.t : dsub(1.0, cx.t);
    const double wy = dy ? cy.t : dsub(1.0, cy.t);
    const double wz = dz ? cz.t : dsub(1.0, cz.t);
    w[c] = dmul(dmul(wx, wy), wz);
    idx[c] = (cx.i0 + dx) + g.rx * ((cy.i0 + dy) + g.ry * (cz.i0 + dz));
  }
  const int base = 3 + 6 * g.L;
  for (int ch = 0; ch < g.C; ++ch) {
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      acc = dadd(acc, dmul(w[c], (double)__ldg(grid + (size_t)idx[c] * g.C + ch)));
    store(base + ch, (float)acc);
  }
}

// Compile-time-shaped variant of embed_point (same operation order, so the
// same bits) whose output array stays in registers: e[0..3+6L+C).
template <int L, int C>
__device__ __forceinline__ void embed_point_t(int rx, int ry, int rz, const float* __restrict__ grid,
                                              double px, double py, double pz, float* e) {
  const double p[3] = {fmin(fmax(px, -1.0), 1.0), fmin(fmax(py, -1.0), 1.0),
                       fmin(fmax(pz, -1.0), 1.0)};
  e[0] = (float)p[0];
  e[1] = (float)p[1];
  e[2] = (float)p[2];
  double scale = 3.141592653589793;
#pragma unroll
  for (int i = 0; i < L; ++i) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      double s, c;
      sincos(dmul(scale, p[ax]), &s, &c);
      e[3 + 6 * i + 2 * ax] = (float)s;
      e[3 + 6 * i + 2 * ax + 1] = (float)c;
    }
    scale = scale * 2.0;
  }
  const AxisCoord cx = level_coord(p[0], rx);
  const AxisCoord cy = level_coord(p[1], ry);
  const AxisCoord cz = level_coord(p[2], rz);
  double acc[C];
#pragma unroll
  for (int ch = 0; ch < C; ++ch) acc[ch] = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
    const double wx = dx ? cx.t : dsub(1.0, cx.t);
    const double wy = dy ? cy.t : dsub(1.0, cy.t);
    const double wz = dz ? cz.t : dsub(1.0, cz.t);
    const double w = dmul(dmul(wx, wy), wz);
    const int idx = (cx.i0 + dx) + rx * ((cy.i0 + dy) + ry * (cz.i0 + dz));
    const float4* row = reinterpret_cast<const float4*>(grid + (size_t)idx * C);
#pragma unroll
    for (int q = 0; q < C / 4; ++q) {
      const float4 f = __ldg(row + q);
      acc[4 * q + 0] = dadd(acc[4 * q + 0], dmul(w, (double)f.x));
      acc[4 * q + 1] = dadd(acc[4 * q + 1], dmul(w, (double)f.y));
      acc[4 * q + 2] = dadd(acc[4 * q + 2], dmul(w, (double)f.z));
      acc[4 * q + 3] = dadd(acc[4 * q + 3], dmul(w, (double)f.w));
    }
  }
#pragma unroll
  for (int ch = 0; ch < C; ++ch) e[3 + 6 * L + ch] = (float)acc[ch];
}

// Combine (model.py:279-286 + sum_absdiff): writes merged input x[0..din).
template <class LoadA, class LoadB, class Store>
__device__ __forceinline__ void merge_into(int mode, int E, LoadA a, LoadB b, Store store) {
  for (int i = 0; i < E; ++i) {
    const float av = a(i), bv = b(i);
    switch (mode) {
      case NDF_MERGE_MULTIPLY: store(i, fmul(av, bv)); break;
      case NDF_MERGE_CONCAT: store(i, av); store(E + i, bv); break;
      case NDF_MERGE_ADD: store(i, fadd(av, bv)); break;
      case NDF_MERGE_ABSDIFF: store(i, fabsf(__fsub_rn(av, bv))); break;
      default: store(i, fadd(av, bv)); store(E + i, fabsf(__fsub_rn(av, bv))); break;
    }
  }
}

// Hidden activation in fp32 (nn.py:23-32 + SiLU), matching the oracle formulas.
__device__ __forceinline__ float act_exact(int kind, float x) {
  switch (kind) {
    case NDF_ACT_RELU: return fmaxf(x, 0.0f);
    case NDF_ACT_SNAKE: { float s = sinf(x); return fadd(x, fmul(s, s)); }
    case NDF_ACT_SNAKE_ALT: return fmul(0.5f, __fsub_rn(fadd(x, 1.0f), cosf(fmul(2.0f, x))));
    default: return __fdiv_rn(x, fadd(1.0f, expf(-x)));
  }
}

__device__ __forceinline__ float head_exact(int kind, float z) {
  switch (kind) {
    case NDF_HEAD_TANH: return tanhf(z);
    case NDF_HEAD_SOFTPLUS: return fadd(fmaxf(z, 0.0f), log1pf(expf(-fabsf(z))));
    default: return z;
  }
}

}  // namespace ndf
