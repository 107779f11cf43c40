// Fused NDF query on 5th-generation tensor cores (K1 + K2, sm_100a).
//
//   embed (fp64 -> fp32, bit-exact with model.py:169-177)
//   -> merge [e_r + e_q, |e_r - e_q|]                      (model.py:279-286 + BASELINE)
//   -> H x { tcgen05.mma 16-bit x 16-bit -> fp32 accumulator in TMEM ;
//            tcgen05.ld epilogue: bias + activation, packed back to SMEM as the
//            next layer's A operand }
//   -> output layer 128 -> 1 as a 16-column tcgen05.mma (zero-padded B) -> head.
//
// Layout / schedule (one persistent CTA per SM, NWG <= 4 warpgroups):
//   * the packed parameter blob (UMMA-canonical K-major 16-bit weights + fp32 bias
//     vectors) is fetched once per CTA by the bulk-copy engine (cp.async.bulk ->
//     mbarrier complete_tx) and stays resident in SMEM;
//   * each warpgroup owns a 128-row tile of query vertices, one 32 KB A buffer
//     (SWIZZLE_NONE canonical layout: 8x16 B core matrices, LBO = 128 B along K,
//     SBO = 2048 B along M) and 128 TMEM columns holding the fp32 accumulator
//     (row m of the tile = TMEM lane m = thread m of the warpgroup);
//   * one thread per warpgroup issues the K/16 tcgen05.mma steps of a layer and
//     commits them to the warpgroup's mbarrier; while one warpgroup runs its
//     epilogue, the other warpgroups' MMAs keep the tensor pipe busy -- a 4-way
//     ping-pong without any CTA-wide barrier.
//   * every accumulator is pre-loaded with its layer's bias (tcgen05.st while the
//     previous layer's values are drained), so the MMAs accumulate onto the bias
//     and the epilogue has no bias adds;
//   * SiLU layers are packed with W and b pre-scaled by 1/2 (exact in 16-bit), so
//     the accumulator holds x/2 and silu(x) = x/2 + (x/2)*tanh(x/2) is one
//     tanh.approx (MUFU) and one FMA per element, then a paired 16-bit pack.
//   * grid-mode Fourier features are per-axis: a prep kernel evaluates them once
//     per axis node (same fp64 sincos, so the same bits) and the query reads them.
//   * multi-reference queries (BASELINE config 3) embed each query vertex once and
//     reuse it for every reference (refs' embeddings come from the prep kernel).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "ndf_query.cuh"
#include "ndf_tc_ptx.cuh"

namespace ndf {
namespace tc {

constexpr int kHid = 128;           // hidden width (UMMA N)
constexpr int kTileM = 128;         // rows per tile (UMMA M)
constexpr int kABytes = kTileM * kHid * 2;     // 32 KB A buffer
constexpr int kSboA = (kHid / 8) * 128;        // 2048 B between 8-row groups
constexpr int kL = 6;               // Fourier octaves supported by the fused encoder
constexpr int kC = 16;              // latent channels supported by the fused encoder
constexpr int kE = 3 + 6 * kL + kC; // 55
constexpr int kERefStride = 64;     // floats per prepared reference embedding
constexpr int kOutN = 16;           // output-layer MMA width (column 0 is the result)
constexpr int kMaxSmem = 232448;    // 227 KB opt-in

struct Layout {
  int H;            // hidden layers (MMA stages before the output stage)
  int kin;          // padded layer-0 K (multiple of 16, <= 128)
  int w0_bytes;     // 128 x kin
  int wh_bytes;     // 128 x 128
  int wout_off;     // 16 x 128 output-layer B operand
  int vec_off;      // fp32: bias[H][128], b_out, pad
  int blob_bytes;   // multiple of 16
};

__host__ __device__ inline Layout make_layout(const ndf_model_desc& m) {
  Layout L;
  L.H = m.n_layers - 1;
  L.kin = (m.widths[0] + 15) / 16 * 16;
  L.w0_bytes = kHid * L.kin * 2;
  L.wh_bytes = kHid * kHid * 2;
  L.wout_off = L.w0_bytes + (L.H - 1) * L.wh_bytes;
  L.vec_off = L.wout_off + kOutN * kHid * 2;
  L.blob_bytes = L.vec_off + (L.H * kHid + 4) * 4;
  return L;
}

// byte offset of element (row r, k) inside a canonical K-major no-swizzle tile
__host__ __device__ __forceinline__ int canon_off(int r, int k, int sbo) {
  return (r >> 3) * sbo + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
      "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),
      "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
      "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// Write layer-0's bias (fp32, pre-scaled for SiLU) into this thread's accumulator row.
__device__ __forceinline__ void preload_bias(uint32_t tmem_row, const float* bias) {
  const float4* b4 = reinterpret_cast<const float4*>(bias);
#pragma unroll 1
  for (int c0 = 0; c0 < kHid; c0 += 32) {
    uint32_t nb[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = b4[(c0 >> 2) + q];
      nb[4 * q] = __float_as_uint(b.x); nb[4 * q + 1] = __float_as_uint(b.y);
      nb[4 * q + 2] = __float_as_uint(b.z); nb[4 * q + 3] = __float_as_uint(b.w);
    }
    tmem_st32(tmem_row + (uint32_t)c0, nb);
  }
}

// Generic (non-SiLU) hidden activations, fp32 fast forms (nn.py:23-32).
__device__ __forceinline__ float act_f32(int kind, float x) {
  switch (kind) {
    case NDF_ACT_RELU: return fmaxf(x, 0.0f);
    case NDF_ACT_SNAKE: { const float s = __sinf(x); return fmaf(s, s, x); }
    case NDF_ACT_SNAKE_ALT: return 0.5f * (x + 1.0f - __cosf(2.0f * x));
    default: { const float hx = 0.5f * x; return fmaf(hx, tanh_fast(hx), hx); }
  }
}

// Column of the tensor-core A operand that holds merged decoder input m.  For the
// two-block merges (sum_absdiff, concat) the blocks are interleaved -- A[2i] from
// e[i] of the first block, A[2i+1] of the second -- so each embedding element feeds
// one adjacent pair of columns and dies at once (no long register live ranges in
// the encoder); layer 0's weight rows are permuted identically at pack time.
__host__ __device__ __forceinline__ int a_column(int merge, int m, int E) {
  if (merge == NDF_MERGE_SUM_ABSDIFF || merge == NDF_MERGE_CONCAT)
    return m < E ? 2 * m : 2 * (m - E) + 1;
  return m;
}

// Value of A column c (model.py:279-286 + BASELINE's sum_absdiff), e_a = mu branch.
// MERGE >= 0 fixes the mode at compile time; -1 reads it at run time.
template <int MERGE, class FA, class FB>
__device__ __forceinline__ float merged_value(int merge_rt, int c, FA ea, FB eb) {
  const int merge = MERGE >= 0 ? MERGE : merge_rt;
  if (merge == NDF_MERGE_SUM_ABSDIFF || merge == NDF_MERGE_CONCAT) {
    const int i = c >> 1;
    if (i >= kE) return 0.0f;
    const float a = ea(i), b = eb(i);
    if (merge == NDF_MERGE_CONCAT) return (c & 1) ? b : a;
    return (c & 1) ? fabsf(a - b) : a + b;
  }
  if (c < kE) {
    const float a = ea(c), b = eb(c);
    switch (merge) {
      case NDF_MERGE_MULTIPLY: return a * b;
      case NDF_MERGE_ABSDIFF: return fabsf(a - b);
      default: return a + b;          // add
    }
  }
  return 0.0f;
}

template <bool F16, int MERGE, class FA, class FB>
__device__ __forceinline__ void write_input_row(uint32_t abase, int row, int merge, FA ea, FB eb,
                                                int kin) {
#pragma unroll
  for (int kg = 0; kg < 16; ++kg) {
    if (kg * 8 < kin) {
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = merged_value<MERGE>(merge, 8 * kg + j, ea, eb);
      st_shared_v4(abase + canon_off(row, kg * 8, kSboA), pack2<F16>(x[0], x[1]),
                   pack2<F16>(x[2], x[3]), pack2<F16>(x[4], x[5]), pack2<F16>(x[6], x[7]));
    }
  }
}

// Latent-grid trilinear lookup in fp32 (the 16-bit path rounds every merged input
// to 11/8 significant bits, so fp32 corner sums are exact enough by 2^-13 and keep
// the fp64 and conversion units free).  Same corner order and clamping rules as
// the reference (encoding.py:105-118).
__device__ __forceinline__ void latent_f32(const float* __restrict__ grid, int rx, int ry, int rz,
                                           double px, double py, double pz, float* out) {
  const AxisCoord cx = level_coord(px, rx);
  const AxisCoord cy = level_coord(py, ry);
  const AxisCoord cz = level_coord(pz, rz);
  const float tx = (float)cx.t, ty = (float)cy.t, tz = (float)cz.t;
  float acc[kC];
#pragma unroll
  for (int ch = 0; ch < kC; ++ch) acc[ch] = 0.0f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
    const float w = (dx ? tx : 1.0f - tx) * (dy ? ty : 1.0f - ty) * (dz ? tz : 1.0f - tz);
    const int idx = (cx.i0 + dx) + rx * ((cy.i0 + dy) + ry * (cz.i0 + dz));
    const float4* row = reinterpret_cast<const float4*>(grid + (size_t)idx * kC);
#pragma unroll
    for (int q = 0; q < kC / 4; ++q) {
      const float4 f = __ldg(row + q);
      acc[4 * q + 0] = fmaf(w, f.x, acc[4 * q + 0]);
      acc[4 * q + 1] = fmaf(w, f.y, acc[4 * q + 1]);
      acc[4 * q + 2] = fmaf(w, f.z, acc[4 * q + 2]);
      acc[4 * q + 3] = fmaf(w, f.w, acc[4 * q + 3]);
    }
  }
#pragma unroll
  for (int ch = 0; ch < kC; ++ch) out[ch] = acc[ch];
}

// Per-axis node table written by prep_kernel, one 64-byte row per axis node:
// [sin/cos of the L octaves (fp64 sincos, cast once) | p (fp32) | i0 | t (fp32) | pad].
constexpr int kAxisRow = 16;
static_assert(2 * kL + 4 == kAxisRow, "axis row layout");

// Node (ix, iy, iz) of row `row` of `tile` (x fastest): one 32-bit division pair for
// the tile's first vertex, then the row offset is carried along x.  Rows past the
// end of the range are clamped to the last vertex (their results are discarded).
__device__ __forceinline__ void tile_node(const QueryArgs& a, int64_t tile, int row, int& ix,
                                          int& iy, int& iz) {
  const int64_t n = a.v1 - a.v0;
  const int64_t vloc = min(tile * kTileM + row, n - 1);
  const int64_t vbase = tile * kTileM;
  const uint32_t vb = (uint32_t)(a.v0 + vbase);
  const uint32_t nxy = (uint32_t)a.nx * (uint32_t)a.ny;
  iz = (int)(vb / nxy);
  const uint32_t rem = vb - (uint32_t)iz * nxy;
  iy = (int)(rem / (uint32_t)a.nx);
  ix = (int)(rem - (uint32_t)iy * (uint32_t)a.nx) + (int)(vloc - vbase);
  while (ix >= a.nx) {
    ix -= a.nx;
    if (++iy == a.ny) { iy = 0; ++iz; }
  }
}

// Grid-mode embedding of node (ix, iy, iz) -- called by all 32 lanes of a warp
// (invalid lanes pass a clamped node).  Raw coords and the Fourier block come
// from the per-axis table; the latent cell is computed arithmetically
// (u = i * (r-1)/(n-1) in fp32) so the latent gathers do not wait for the table
// loads -- both go to L2 in one round trip (L1 is all SMEM here).
__device__ __forceinline__ void embed_grid_node(const QueryArgs& a, const float* __restrict__ grid,
                                                const float* __restrict__ ftab, int ix, int iy,
                                                int iz, const float* lscale, float* e) {
  const int idx3[3] = {ix, iy, iz};
  const int res[3] = {a.g.rx, a.g.ry, a.g.rz};
  const int nn[3] = {a.nx, a.ny, a.nz};
  int i0[3];
  float tt[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    // node i of an n-node axis sits at u = i*(r-1)/(n-1); a single-node axis at the
    // domain centre, u = (r-1)/2 (measures.py:245-247)
    const float u = nn[ax] > 1 ? (float)idx3[ax] * lscale[ax] : 0.5f * (float)(res[ax] - 1);
    i0[ax] = min((int)u, res[ax] - 2);
    tt[ax] = fminf(u - (float)i0[ax], 1.0f);
  }
  float acc[kC];
  // Warp-cooperative latent gather: the 32 lanes are consecutive x nodes, normally of
  // one (y, z) row, so they share the y/z cell and weights and touch only a few
  // x cells.  Lane L pre-interpolates column xmin+L over (y, z) (4 rows) and every lane
  // then lerps its two columns from registers via shuffles: ~6x fewer L2 requests.
  const unsigned full = 0xffffffffu;
  const int iy0 = __shfl_sync(full, i0[1], 0), iz0 = __shfl_sync(full, i0[2], 0);
  const float ty0 = __shfl_sync(full, tt[1], 0), tz0 = __shfl_sync(full, tt[2], 0);
  const int xmin = __reduce_min_sync(full, i0[0]);
  const int xmax = __reduce_max_sync(full, i0[0]);
  const bool coop = __all_sync(full, i0[1] == iy0 && i0[2] == iz0 && tt[1] == ty0 &&
                                         tt[2] == tz0) && (xmax - xmin + 2 <= 32);
  if (coop) {
    const int lane = threadIdx.x & 31;
    const int nc = xmax - xmin + 2;
    float g[kC];
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) g[ch] = 0.0f;
    if (lane < nc) {
      const int xl = xmin + lane;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int dy = c & 1, dz = c >> 1;
        const float w = (dy ? ty0 : 1.0f - ty0) * (dz ? tz0 : 1.0f - tz0);
        const int idx = xl + a.g.rx * ((iy0 + dy) + a.g.ry * (iz0 + dz));
        const float4* row = reinterpret_cast<const float4*>(grid + (size_t)idx * kC);
#pragma unroll
        for (int q = 0; q < kC / 4; ++q) {
          const float4 f = __ldg(row + q);
          g[4 * q + 0] = fmaf(w, f.x, g[4 * q + 0]);
          g[4 * q + 1] = fmaf(w, f.y, g[4 * q + 1]);
          g[4 * q + 2] = fmaf(w, f.z, g[4 * q + 2]);
          g[4 * q + 3] = fmaf(w, f.w, g[4 * q + 3]);
        }
      }
    }
    const int src = i0[0] - xmin;
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) {
      const float g0 = __shfl_sync(full, g[ch], src);
      const float g1 = __shfl_sync(full, g[ch], src + 1);
      acc[ch] = fmaf(tt[0], g1 - g0, g0);
    }
  } else {
    // same arithmetic per lane (columns x0 and x0+1 over (y, z), then the x lerp), so
    // a vertex's value does not depend on which path its warp took
    float g0[kC], g1[kC];
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) { g0[ch] = 0.0f; g1[ch] = 0.0f; }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int dy = c & 1, dz = c >> 1;
      const float w = (dy ? tt[1] : 1.0f - tt[1]) * (dz ? tt[2] : 1.0f - tt[2]);
      const int idx = i0[0] + a.g.rx * ((i0[1] + dy) + a.g.ry * (i0[2] + dz));
      const float4* r0 = reinterpret_cast<const float4*>(grid + (size_t)idx * kC);
      const float4* r1 = reinterpret_cast<const float4*>(grid + (size_t)(idx + 1) * kC);
#pragma unroll
      for (int q = 0; q < kC / 4; ++q) {
        const float4 f = __ldg(r0 + q), h = __ldg(r1 + q);
        g0[4 * q + 0] = fmaf(w, f.x, g0[4 * q + 0]); g1[4 * q + 0] = fmaf(w, h.x, g1[4 * q + 0]);
        g0[4 * q + 1] = fmaf(w, f.y, g0[4 * q + 1]); g1[4 * q + 1] = fmaf(w, h.y, g1[4 * q + 1]);
        g0[4 * q + 2] = fmaf(w, f.z, g0[4 * q + 2]); g1[4 * q + 2] = fmaf(w, h.z, g1[4 * q + 2]);
        g0[4 * q + 3] = fmaf(w, f.w, g0[4 * q + 3]); g1[4 * q + 3] = fmaf(w, h.w, g1[4 * q + 3]);
      }
    }
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) acc[ch] = fmaf(tt[0], g1[ch] - g0[ch], g0[ch]);
  }
  const int rows[3] = {ix, a.nx + iy, a.nx + a.ny + iz};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const float4* t = reinterpret_cast<const float4*>(ftab + (size_t)rows[ax] * kAxisRow);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 f = __ldg(t + q);
      const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = 4 * q + u;
        if (j < 2 * kL) e[3 + 6 * (j >> 1) + 2 * ax + (j & 1)] = fv[u];  // 2*octave + sin|cos
        else if (j == 2 * kL) e[ax] = fv[u];
      }
    }
  }
#pragma unroll
  for (int ch = 0; ch < kC; ++ch) e[3 + 6 * kL + ch] = acc[ch];
}

// Points-mode embedding (NdfModel.forward): fp64 sincos per point, fp32 latent.
__device__ __forceinline__ void embed_point_tc(const QueryArgs& a, const float* __restrict__ grid,
                                               const double* pos, float* e) {
  const double p[3] = {fmin(fmax(pos[0], -1.0), 1.0), fmin(fmax(pos[1], -1.0), 1.0),
                       fmin(fmax(pos[2], -1.0), 1.0)};
  e[0] = (float)p[0];
  e[1] = (float)p[1];
  e[2] = (float)p[2];
  double scale = 3.141592653589793;
#pragma unroll
  for (int i = 0; i < kL; ++i) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      double sn, cs;
      sincos(dmul(scale, p[ax]), &sn, &cs);
      e[3 + 6 * i + 2 * ax] = (float)sn;
      e[3 + 6 * i + 2 * ax + 1] = (float)cs;
    }
    scale = scale * 2.0;
  }
  latent_f32(grid, a.g.rx, a.g.ry, a.g.rz, p[0], p[1], p[2], e + 3 + 6 * kL);
}

struct TcArgs {
  QueryArgs q;
  const float* ftab;      // grid mode: (nx+ny+nz) x kAxisRow per-axis node table
  const float* erefs;     // grid mode: n_ref x kERefStride reference embeddings
  int n_ref;
  uint16_t* out16;        // multi-ref output (fp16), rows of ld_out
  int64_t ld_out;
  long long* trace;       // debug: per-phase clock64 stamps of CTA 0 (NULL = off)
  int stagger;            // cycles between warpgroup start times (de-phases the WGs)
  int tokens;             // max warpgroups in an epilogue at once (0 = unlimited)
};

// debug tracing of CTA 0's schedule: slot = (wg, tile#, event)
constexpr int kTraceTiles = 32, kTraceEvents = 12;
constexpr int kTraceBase = 6 * kTraceTiles * kTraceEvents;   // + 16 chunk stamps
#define NDF_TRACE_AT(slot_, ev)                                                          \
  do {                                                                                   \
    if (t.trace && blockIdx.x == 0 && wtid == 0 && (slot_) < kTraceTiles)                 \
      t.trace[(wg * kTraceTiles + (slot_)) * kTraceEvents + (ev)] = clock64();          \
  } while (0)
#define NDF_TRACE(ev)                                                                    \
  do {                                                                                   \
    if (t.trace && blockIdx.x == 0 && wtid == 0 && tcount < kTraceTiles)                  \
      t.trace[(wg * kTraceTiles + tcount) * kTraceEvents + (ev)] = clock64();           \
  } while (0)

// One MMA stage: K/16 tcgen05.mma steps into the warpgroup's accumulator, committed
// to its mbarrier.  Issued by one thread.
// acc_first = 1: the accumulator was pre-loaded (bias) and every step accumulates.
__device__ __forceinline__ void issue_stage(uint32_t d_tmem, uint32_t a_addr, uint32_t b_addr,
                                            int K, uint32_t sbo_b, uint32_t idesc, uint64_t* bar,
                                            uint32_t acc_first) {
  tc_fence_after();
  for (int kk = 0; kk < K / 16; ++kk) {
    const uint64_t ad = smem_desc(a_addr + kk * 256, 128, kSboA);
    const uint64_t bd = smem_desc(b_addr + kk * 256, 128, sbo_b);
    mma_bf16(d_tmem, ad, bd, idesc, kk > 0 ? 1u : acc_first);
  }
  mma_commit(bar);
}

// F16: fp16 (true) or bf16 operands.  SILU: SiLU-specialised epilogue (packed
// 16-bit tanh/fma) vs generic fp32 activation.  KIND: 0 = grid, one reference;
// 1 = grid, several references per query vertex (the query embedding stays live
// across them); 2 = paired points (NdfModel.forward).
constexpr int kGridSingle = 0, kGridMulti = 1, kPoints = 2;
template <bool F16, bool SILU, int KIND>
__global__ void __launch_bounds__(512, 1)
query_tc_kernel(const TcArgs t, const int nwg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const QueryArgs& a = t.q;
  const Layout lay = make_layout(a.m);
  uint8_t* wblob = smem;                                   // parameter blob
  uint8_t* abufs = smem + ((lay.blob_bytes + 1023) & ~1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(abufs + nwg * kABytes);   // [0] weights, [1+w]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  float* eref_s = reinterpret_cast<float*>(bars + 16);      // single-ref grid: e_ref in SMEM
  int* epi_tok = reinterpret_cast<int*>(bars + 64);          // epilogue admission counter

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int wg = warp >> 2;
  const int wtid = tid & 127;               // row of the tile owned by this thread
  const float* vecs = reinterpret_cast<const float*>(wblob + lay.vec_off);
  const uint32_t tmem_cols = nwg > 2 ? 512 : (nwg == 2 ? 256 : 128);

  if (tid == 0) {
    *epi_tok = 0;
    mbar_init(&bars[0], 1);
    for (int w = 0; w < nwg; ++w) mbar_init(&bars[1 + w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_expect_tx(&bars[0], (uint32_t)lay.blob_bytes);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.m.params_tc);
    for (int off = 0; off < lay.blob_bytes; off += 32768)
      bulk_g2s(wblob + off, src + off, (uint32_t)min(32768, lay.blob_bytes - off), &bars[0]);
  }
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t d_tmem = tmem_base + (uint32_t)(wg * kHid);       // column offset
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;    // TMEM lane quarter
  const uint32_t a_addr = smem_u32(abufs + wg * kABytes);
  const uint32_t tmem_row = tmem_base + lane_base + (uint32_t)(wg * kHid);  // this thread's lane
  const uint32_t w_addr = smem_u32(wblob);
  uint64_t* bar = &bars[1 + wg];
  // kind::f16 instruction descriptor: D fp32 (bit 4), A/B fp16 (0) or bf16 (1) at bits
  // 7-9 / 10-12, both K-major, N>>3 at bits 17-22, M>>4 at bits 24-28.
  const uint32_t ab_fmt = F16 ? 0u : 1u;
  const uint32_t idesc_base = (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) |
                              ((uint32_t)(kTileM >> 4) << 24);
  const uint32_t idesc = idesc_base | ((uint32_t)(kHid >> 3) << 17);
  const uint32_t idesc_out = idesc_base | ((uint32_t)(kOutN >> 3) << 17);
  const uint32_t sbo_w0 = (uint32_t)(lay.kin / 8) * 128;

  mbar_wait(&bars[0], 0);    // parameters resident
  const float bias_out = vecs[lay.H * kHid];

  const int64_t n = a.v1 - a.v0;
  const int64_t n_tiles = (n + kTileM - 1) / kTileM;
  const int64_t stride = (int64_t)gridDim.x * nwg;
  uint32_t phase = 0;
  const float* grid_q = a.ref_is_mu ? a.m.grid_nu : a.m.grid_mu;
  const int bar_id = 1 + wg;
  const int n_ref = KIND == kGridMulti ? t.n_ref : 1;
  if (KIND == kGridSingle) {
    if (tid < kERefStride) eref_s[tid] = t.erefs[tid];
    __syncthreads();
  }

  // De-phase the warpgroups so one WG's encoder / MMA waits overlap another's
  // MUFU-bound epilogue instead of all four contending for the same unit at once.
  if (t.stagger > 0) {
    const long long c0 = clock64();
    while (clock64() - c0 < (long long)wg * t.stagger) {
    }
  }
  const float lscale[3] = {a.nx > 1 ? (float)(a.g.rx - 1) / (float)(a.nx - 1) : 0.0f,
                           a.ny > 1 ? (float)(a.g.ry - 1) / (float)(a.ny - 1) : 0.0f,
                           a.nz > 1 ? (float)(a.g.rz - 1) / (float)(a.nz - 1) : 0.0f};
  int tcount = 0;
  for (int64_t tile = (int64_t)blockIdx.x * nwg + wg; tile < n_tiles; tile += stride, ++tcount) {
    NDF_TRACE(0);
    const int64_t vloc = tile * kTileM + wtid;   // local vertex index
    const bool valid = vloc < n;
    // ---- K1: embed the query vertex once -----------------------------------------
    float eq[kE];
    if (KIND != kPoints) {
      int ix, iy, iz;
      tile_node(a, tile, wtid, ix, iy, iz);
      embed_grid_node(a, grid_q, t.ftab, ix, iy, iz, lscale, eq);   // all lanes (shuffles)
      if (!valid) {
#pragma unroll
        for (int i = 0; i < kE; ++i) eq[i] = 0.0f;
      }
      NDF_TRACE(8);
    } else if (valid) {
      embed_point_tc(a, a.m.grid_nu, a.p_nu + 3 * (a.v0 + vloc), eq);
    } else {
#pragma unroll
      for (int i = 0; i < kE; ++i) eq[i] = 0.0f;
    }
    for (int r = 0; r < n_ref; ++r) {
      // ---- bias of layer 0 -> accumulator (tcgen05.st); the MMAs then accumulate ----
      preload_bias(tmem_row, vecs);
      NDF_TRACE(9);
      // ---- merge -> A ------------------------------------------------------------
      auto fq = [&](int i) { return eq[i]; };
      if constexpr (KIND != kPoints) {
        const float* er = t.erefs + (size_t)r * kERefStride;
        auto fr = [&](int i) { return KIND == kGridSingle ? eref_s[i] : __ldg(er + i); };
        if (a.m.merge == NDF_MERGE_SUM_ABSDIFF)      // symmetric: role does not matter
          write_input_row<F16, NDF_MERGE_SUM_ABSDIFF>(a_addr, wtid, 0, fr, fq, lay.kin);
        else if (a.ref_is_mu)
          write_input_row<F16, -1>(a_addr, wtid, a.m.merge, fr, fq, lay.kin);
        else
          write_input_row<F16, -1>(a_addr, wtid, a.m.merge, fq, fr, lay.kin);
      } else {
        float em[kE];
        if (valid) {
          const int64_t im = a.n_mu == 1 ? 0 : a.v0 + vloc;
          embed_point_tc(a, a.m.grid_mu, a.p_mu + 3 * im, em);
        } else {
#pragma unroll
          for (int i = 0; i < kE; ++i) em[i] = 0.0f;
        }
        auto fm = [&](int i) { return em[i]; };
        write_input_row<F16, -1>(a_addr, wtid, a.m.merge, fm, fq, lay.kin);
      }
      NDF_TRACE(11);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_proxy_async();
      tc_fence_before();
      named_bar(bar_id, 128);
      NDF_TRACE(1);
      // ---- K2: hidden layers on the tensor cores --------------------------------------
      for (int l = 0; l < lay.H; ++l) {
        if (wtid == 0) {
          const uint32_t wl = w_addr + (l == 0 ? 0 : lay.w0_bytes + (l - 1) * lay.wh_bytes);
          issue_stage(d_tmem, a_addr, wl, l == 0 ? lay.kin : kHid, l == 0 ? sbo_w0 : kSboA,
                      idesc, bar, 1u);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
        // Admission control: at most t.tokens warpgroups run the MUFU-bound epilogue at
        // a time, which keeps the others in their encoder / MMA phases and stops the
        // four warpgroups from phase-locking onto the same unit.
        if (t.tokens > 0) {
          if (wtid == 0) {
            while (atomicAdd(epi_tok, 1) >= t.tokens) {
              atomicSub(epi_tok, 1);
              __nanosleep(32);
            }
          }
          named_bar(bar_id, 128);
        }
        NDF_TRACE(2 + 2 * l);
        const bool next_hidden = l + 1 < lay.H;
        const float4* nbias4 = reinterpret_cast<const float4*>(vecs + (l + 1) * kHid);
#pragma unroll 1
        for (int c0 = 0; c0 < kHid; c0 += 32) {
          float v[32];
#define NDF_CHUNK_TRACE(e)                                                                   \
  if (t.trace && blockIdx.x == 0 && wg == 0 && wtid == 0 && tcount == 3 && l == 1)          \
    t.trace[kTraceBase + (c0 >> 5) * 4 + (e)] = clock64();
          NDF_CHUNK_TRACE(0);
          tmem_ld32(tmem_row + (uint32_t)c0, v);          // z (or z/2 for SiLU) incl. bias
          NDF_CHUNK_TRACE(1);
          if (next_hidden) {                               // next layer's bias -> same columns
            uint32_t nb[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 b4 = nbias4[(c0 >> 2) + q];
              nb[4 * q] = __float_as_uint(b4.x); nb[4 * q + 1] = __float_as_uint(b4.y);
              nb[4 * q + 2] = __float_as_uint(b4.z); nb[4 * q + 3] = __float_as_uint(b4.w);
            }
            tmem_st32(tmem_row + (uint32_t)c0, nb);
          }
          NDF_CHUNK_TRACE(2);
          float h[32];
          if constexpr (SILU) {
            // all 32 MUFU first (one in flight per scoreboard group), then the FMAs:
            // x = z/2, silu(z) = x + x*tanh(x)
#pragma unroll
            for (int i = 0; i < 32; ++i) h[i] = tanh_fast(v[i]);
#pragma unroll
            for (int i = 0; i < 32; ++i) h[i] = fmaf(v[i], h[i], v[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) h[i] = act_f32(a.m.activation, v[i]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            st_shared_v4(a_addr + canon_off(wtid, c0 + 8 * j, kSboA),
                         pack2<F16>(h[8 * j], h[8 * j + 1]), pack2<F16>(h[8 * j + 2], h[8 * j + 3]),
                         pack2<F16>(h[8 * j + 4], h[8 * j + 5]), pack2<F16>(h[8 * j + 6], h[8 * j + 7]));
          NDF_CHUNK_TRACE(3);
        }
        if (next_hidden) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async();
        tc_fence_before();
        named_bar(bar_id, 128);
        if (t.tokens > 0 && wtid == 0) atomicSub(epi_tok, 1);
        NDF_TRACE(3 + 2 * l);
      }
      // ---- output layer (128 -> 1) as a 16-column MMA ---------------------------------
      if (wtid == 0)
        issue_stage(d_tmem, a_addr, w_addr + lay.wout_off, kHid, kSboA, idesc_out, bar, 0u);
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_fence_after();
      NDF_TRACE(10);
      uint32_t zr;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                   : "=r"(zr) : "r"(tmem_row));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (valid) {
        const float z = head_exact(a.m.head, __uint_as_float(zr) + bias_out);
        if (t.out16) {
          const __half hz = __float2half_rn(z);
          t.out16[(size_t)r * t.ld_out + vloc] = *reinterpret_cast<const uint16_t*>(&hz);
        } else {
          a.out[vloc] = z;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
}

// ---------------------------------------------------------------------------
// Warp-specialised schedule (NDF_TC_SCHEDULE=ws; single-reference grid queries).
//   WG0..WG3 -- epilogue warpgroups, one TMEM-accumulator / A-buffer slot each:
//               drain the accumulator (tcgen05.ld pipelined one 32-column chunk
//               ahead), bias + activation, write the next A operand, issue the next
//               MMA, and finally read the output column and release the slot.
//   WG4, WG5 -- producer warpgroups: embed the next query tile and pack its merged
//               16-bit layer-0 rows in registers *before* the slot is released, then
//               only store them (14 x 16 B per row) and issue the layer-0 MMA, so
//               the L2-latency-bound encoder never sits on the epilogue warps' path.
// Synchronisation is mbarrier-only: acc_full[s] (tcgen05.commit after every MMA
// stage) and slot_free[s] (epilogue WG after reading the output column).
constexpr int kSlots = 4;
constexpr int kKinMax = 128;

template <bool F16, int MERGE, class FA, class FB>
__device__ __forceinline__ void pack_input_row(int merge, FA ea, FB eb, int kin, uint32_t* pk) {
#pragma unroll
  for (int kg = 0; kg < kKinMax / 8; ++kg) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i0 = 8 * kg + 2 * q;
      pk[4 * kg + q] = (8 * kg < kin)
          ? pack2<F16>(merged_value<MERGE>(merge, i0, ea, eb), merged_value<MERGE>(merge, i0 + 1, ea, eb))
          : 0u;
    }
  }
}

template <bool F16, bool SILU>
__device__ __forceinline__ void epilogue_chunk(const float* v, const float4* b4, int c0,
                                               int act, uint32_t a_addr, int row) {
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const float4 ba = b4[(c0 >> 2) + 2 * jj];
    const float4 bb = b4[(c0 >> 2) + 2 * jj + 1];
    const float x[8] = {v[8 * jj] + ba.x, v[8 * jj + 1] + ba.y, v[8 * jj + 2] + ba.z,
                        v[8 * jj + 3] + ba.w, v[8 * jj + 4] + bb.x, v[8 * jj + 5] + bb.y,
                        v[8 * jj + 6] + bb.z, v[8 * jj + 7] + bb.w};
    uint32_t p[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float x0 = x[2 * q], x1 = x[2 * q + 1];
      if constexpr (SILU)     // x = z/2 (weights pre-scaled): silu(z) = x + x*tanh(x)
        p[q] = pack2<F16>(fmaf(x0, tanh_fast(x0), x0), fmaf(x1, tanh_fast(x1), x1));
      else
        p[q] = pack2<F16>(act_f32(act, x0), act_f32(act, x1));
    }
    st_shared_v4(a_addr + canon_off(row, c0 + 8 * jj, kSboA), p[0], p[1], p[2], p[3]);
  }
}

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <bool F16, bool SILU, int KIND>
__global__ void __launch_bounds__(768, 1)
query_ws_kernel(const TcArgs t) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const QueryArgs& a = t.q;
  const Layout lay = make_layout(a.m);
  uint8_t* wblob = smem;
  uint8_t* abufs = smem + ((lay.blob_bytes + 1023) & ~1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(abufs + kSlots * kABytes);
  uint64_t* wbar = &bars[0];
  uint64_t* acc_full = &bars[1];            // [kSlots]
  uint64_t* slot_free = &bars[1 + kSlots];  // [kSlots]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  float* eref_s = reinterpret_cast<float*>(bars + 16);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int wg = warp >> 2;
  const int wtid = tid & 127;
  const float* vecs = reinterpret_cast<const float*>(wblob + lay.vec_off);

  if (tid == 0) {
    mbar_init(wbar, 1);
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&slot_free[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < kERefStride) eref_s[tid] = t.erefs[tid];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_expect_tx(wbar, (uint32_t)lay.blob_bytes);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.m.params_tc);
    for (int off = 0; off < lay.blob_bytes; off += 32768)
      bulk_g2s(wblob + off, src + off, (uint32_t)min(32768, lay.blob_bytes - off), wbar);
  }
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t w_addr = smem_u32(wblob);
  const uint32_t ab_fmt = F16 ? 0u : 1u;
  const uint32_t idesc_base = (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) |
                              ((uint32_t)(kTileM >> 4) << 24);
  const uint32_t idesc = idesc_base | ((uint32_t)(kHid >> 3) << 17);
  const uint32_t idesc_out = idesc_base | ((uint32_t)(kOutN >> 3) << 17);
  const uint32_t sbo_w0 = (uint32_t)(lay.kin / 8) * 128;

  const int64_t n = a.v1 - a.v0;
  const int64_t n_tiles = (n + kTileM - 1) / kTileM;
  const int64_t tile_stride = (int64_t)gridDim.x * kSlots;
  auto slot_tiles = [&](int s) -> int64_t {
    const int64_t first = (int64_t)blockIdx.x * kSlots + s;
    return first < n_tiles ? (n_tiles - first + tile_stride - 1) / tile_stride : 0;
  };
  const float* grid_q = a.ref_is_mu ? a.m.grid_nu : a.m.grid_mu;
  const int bar_id = 1 + wg;

  if (wg >= kSlots) {
    // ======================= producer warpgroups (WG4, WG5) =========================
    // WG4 fills slots 0 and 2, WG5 slots 1 and 3, alternating; the next tile's merged
    // 16-bit row is packed in registers before the slot is released.
    const int pslots[2] = {wg - kSlots, wg - kSlots + 2};
    const int64_t cnt[2] = {slot_tiles(pslots[0]), slot_tiles(pslots[1])};
    const float lscale[3] = {a.nx > 1 ? (float)(a.g.rx - 1) / (float)(a.nx - 1) : 0.0f,
                             a.ny > 1 ? (float)(a.g.ry - 1) / (float)(a.ny - 1) : 0.0f,
                             a.nz > 1 ? (float)(a.g.rz - 1) / (float)(a.nz - 1) : 0.0f};
    uint32_t free_ph[2] = {0u, 0u};
    bool weights_ready = false;
    const int64_t rounds = cnt[0] > cnt[1] ? cnt[0] : cnt[1];
    for (int64_t kk = 0; kk < rounds; ++kk) {
      for (int si = 0; si < 2; ++si) {
        if (kk >= cnt[si]) continue;
        const int s = pslots[si];
        const int64_t tile = (int64_t)blockIdx.x * kSlots + s + kk * tile_stride;
        const int64_t vloc = tile * kTileM + wtid;
        const int tslot = (int)(kk * 2 + si);
        NDF_TRACE_AT(tslot, 0);
        uint32_t pk[kKinMax / 2];
        {
          float eq[kE];
          {
            int ix, iy, iz;
            tile_node(a, tile, wtid, ix, iy, iz);
            embed_grid_node(a, grid_q, t.ftab, ix, iy, iz, lscale, eq);   // all lanes
            if (vloc >= n) {
#pragma unroll
              for (int i = 0; i < kE; ++i) eq[i] = 0.0f;
            }
          }
          auto fq = [&](int i) { return eq[i]; };
          auto fr = [&](int i) { return eref_s[i]; };
          if (a.m.merge == NDF_MERGE_SUM_ABSDIFF)
            pack_input_row<F16, NDF_MERGE_SUM_ABSDIFF>(0, fr, fq, lay.kin, pk);
          else if (a.ref_is_mu)
            pack_input_row<F16, -1>(a.m.merge, fr, fq, lay.kin, pk);
          else
            pack_input_row<F16, -1>(a.m.merge, fq, fr, lay.kin, pk);
        }
        NDF_TRACE_AT(tslot, 1);
        if (!weights_ready) {
          mbar_wait(wbar, 0);
          weights_ready = true;
        }
        if (kk >= 1) {                               // slot must be drained first
          mbar_wait(&slot_free[s], free_ph[si]);
          free_ph[si] ^= 1u;
        }
        NDF_TRACE_AT(tslot, 2);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(abufs + s * kABytes);
#pragma unroll
        for (int kg = 0; kg < kKinMax / 8; ++kg)
          if (8 * kg < lay.kin)
            st_shared_v4(a_addr + canon_off(wtid, 8 * kg, kSboA), pk[4 * kg], pk[4 * kg + 1],
                         pk[4 * kg + 2], pk[4 * kg + 3]);
        fence_proxy_async();
        tc_fence_before();
        named_bar(bar_id, 128);
        if (wtid == 0)
          issue_stage(tmem_base + (uint32_t)(s * kHid), a_addr, w_addr, lay.kin, sbo_w0, idesc,
                      &acc_full[s], 0u);
        NDF_TRACE_AT(tslot, 3);
      }
    }
  } else {
    // ======================= epilogue warpgroups (WG0..WG3, one slot each) ==========
    const int s = wg;
    const int64_t cnt = slot_tiles(s);
    mbar_wait(wbar, 0);
    const float bias_out = vecs[lay.H * kHid];
    const uint32_t tmem_row = tmem_base + lane_base + (uint32_t)(s * kHid);
    const uint32_t a_addr = smem_u32(abufs + s * kABytes);
    uint32_t acc_ph = 0u;
    for (int64_t kk = 0; kk < cnt; ++kk) {
      for (int st = 0; st < lay.H; ++st) {
        mbar_wait(&acc_full[s], acc_ph);
        acc_ph ^= 1u;
        tc_fence_after();
        NDF_TRACE_AT((int)kk, 2 * st);
        // ---- hidden layer st: drain (pipelined tcgen05.ld), bias + act, next A --------
        const float4* b4 = reinterpret_cast<const float4*>(vecs + st * kHid);
        float va[32], vb[32];
        tmem_ld32_nowait(tmem_row, va);
        tmem_wait_ld();
        tmem_ld32_nowait(tmem_row + 32u, vb);
        epilogue_chunk<F16, SILU>(va, b4, 0, a.m.activation, a_addr, wtid);
        tmem_wait_ld();
        tmem_ld32_nowait(tmem_row + 64u, va);
        epilogue_chunk<F16, SILU>(vb, b4, 32, a.m.activation, a_addr, wtid);
        tmem_wait_ld();
        tmem_ld32_nowait(tmem_row + 96u, vb);
        epilogue_chunk<F16, SILU>(va, b4, 64, a.m.activation, a_addr, wtid);
        tmem_wait_ld();
        epilogue_chunk<F16, SILU>(vb, b4, 96, a.m.activation, a_addr, wtid);
        fence_proxy_async();
        tc_fence_before();
        named_bar(bar_id, 128);
        NDF_TRACE_AT((int)kk, 2 * st + 1);
        if (wtid == 0) {
          if (st + 1 < lay.H)
            issue_stage(tmem_base + (uint32_t)(s * kHid), a_addr,
                        w_addr + lay.w0_bytes + st * lay.wh_bytes, kHid, kSboA, idesc,
                        &acc_full[s], 0u);
          else
            issue_stage(tmem_base + (uint32_t)(s * kHid), a_addr, w_addr + lay.wout_off, kHid,
                        kSboA, idesc_out, &acc_full[s], 0u);
        }
      }
      // ---- output column: head, store, release the slot -------------------------------
      mbar_wait(&acc_full[s], acc_ph);
      acc_ph ^= 1u;
      tc_fence_after();
      NDF_TRACE_AT((int)kk, 6);
      uint32_t zr;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(zr) : "r"(tmem_row));
      tmem_wait_ld();
      tc_fence_before();
      const int64_t vloc = ((int64_t)blockIdx.x * kSlots + s + kk * tile_stride) * kTileM + wtid;
      if (vloc < n) a.out[vloc] = head_exact(a.m.head, __uint_as_float(zr) + bias_out);
      named_bar(bar_id, 128);
      if (wtid == 0) mbar_arrive(&slot_free[s]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
}

// ---- per-query prep: per-axis Fourier table + reference embeddings ------------
__global__ void prep_kernel(const QueryArgs a, const double* refs, int n_ref, float* ftab,
                            float* erefs) {
  const int naxis = a.nx + a.ny + a.nz;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid < naxis) {
    int ax, i, n;
    if (tid < a.nx) { ax = 0; i = tid; n = a.nx; }
    else if (tid < a.nx + a.ny) { ax = 1; i = tid - a.nx; n = a.ny; }
    else { ax = 2; i = tid - a.nx - a.ny; n = a.nz; }
    const double p = fmin(fmax(node_coord(i, n), -1.0), 1.0);
    const int res = ax == 0 ? a.g.rx : (ax == 1 ? a.g.ry : a.g.rz);
    const AxisCoord lc = level_coord(p, res);
    float* row = ftab + (size_t)tid * kAxisRow;
    row[2 * kL] = (float)p;
    row[2 * kL + 1] = __int_as_float(lc.i0);
    row[2 * kL + 2] = (float)lc.t;
    row[2 * kL + 3] = 0.0f;
    double scale = 3.141592653589793;
    for (int o = 0; o < kL; ++o) {
      double s, c;
      sincos(dmul(scale, p), &s, &c);
      row[2 * o] = (float)s;
      row[2 * o + 1] = (float)c;
      scale = scale * 2.0;
    }
  } else if (tid < naxis + n_ref) {
    const int r = tid - naxis;
    const float* grid = a.ref_is_mu ? a.m.grid_mu : a.m.grid_nu;
    float e[kE];
    // refs == nullptr: the single reference travels by value in the kernel arguments
    const double rx = refs ? refs[3 * r] : a.ref[0];
    const double ry = refs ? refs[3 * r + 1] : a.ref[1];
    const double rz = refs ? refs[3 * r + 2] : a.ref[2];
    embed_point_t<kL, kC>(a.g.rx, a.g.ry, a.g.rz, grid, rx, ry, rz, e);
    for (int i = 0; i < kERefStride; ++i) erefs[(size_t)r * kERefStride + i] = i < kE ? e[i] : 0.f;
  }
}

// ---- parameter packing (device) ---------------------------------------------
__global__ void pack_zero_kernel(const ndf_model_desc m, uint8_t* blob) {
  const Layout lay = make_layout(m);
  const int64_t total = (int64_t)lay.blob_bytes / 4;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint32_t*>(blob)[w] = 0u;
}

__device__ __forceinline__ void store16(uint8_t* p, float v, bool f16) {
  if (f16) *reinterpret_cast<__half*>(p) = __float2half_rn(v);
  else *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
}

__global__ void pack_fill_kernel(const ndf_model_desc m, uint8_t* blob) {
  const Layout lay = make_layout(m);
  const bool f16 = m.tc_format == NDF_PREC_FP16;
  // SiLU layers are stored pre-scaled by 1/2 (exact): the accumulator holds x/2.
  const float hs = m.activation == NDF_ACT_SILU ? 0.5f : 1.0f;
  size_t off = 0;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  float* vecs = reinterpret_cast<float*>(blob + lay.vec_off);
  for (int l = 0; l < m.n_layers; ++l) {
    const int K = m.widths[l], N = m.widths[l + 1];
    const float* W = m.params_f32 + off;
    const float* b = W + (size_t)K * N;
    if (l < lay.H) {
      // layer l (K x N fp32 row-major, N = 128) -> canonical N x Kpad, K-major
      const int kpad = l == 0 ? lay.kin : kHid;
      const int sbo = (kpad / 8) * 128;
      uint8_t* dst = blob + (l == 0 ? 0 : lay.w0_bytes + (l - 1) * lay.wh_bytes);
      for (int64_t e = gtid; e < (int64_t)K * N; e += gsz) {
        const int k = (int)(e / N), nn = (int)(e % N);
        const int kc = l == 0 ? a_column(m.merge, k, kE) : k;   // layer-0 rows follow the A layout
        store16(dst + canon_off(nn, kc, sbo), hs * W[e], f16);
      }
      for (int64_t e = gtid; e < N; e += gsz) vecs[l * kHid + e] = hs * b[e];
    } else {
      // output layer (128 x 1) -> row 0 of a 16 x 128 canonical B operand
      for (int64_t e = gtid; e < K; e += gsz)
        store16(blob + lay.wout_off + canon_off(0, (int)e, kSboA), W[e], f16);
      if (gtid == 0) vecs[lay.H * kHid] = b[0];
    }
    off += (size_t)K * N + N;
  }
}

}  // namespace tc

static bool tc_supported(const ndf_model_desc& m, std::string* why) {
  auto fail = [&](const char* s) { if (why) *why = s; return false; };
  if (m.fourier_octaves != tc::kL || m.grid_channels != tc::kC)
    return fail("tcgen05 path needs fourier_octaves=6 and 16 latent channels");
  if (m.n_layers < 2) return fail("tcgen05 path needs >= 1 hidden layer");
  if (m.widths[0] > 128) return fail("tcgen05 path needs decoder input width <= 128");
  for (int i = 1; i < m.n_layers; ++i)
    if (m.widths[i] != tc::kHid) return fail("tcgen05 path needs hidden width 128");
  if (m.widths[m.n_layers] != 1) return fail("decoder must emit one scalar");
  const tc::Layout lay = tc::make_layout(m);
  if (((lay.blob_bytes + 1023) & ~1023) + tc::kABytes + 1024 > tc::kMaxSmem)
    return fail("too many hidden layers for the SMEM-resident weights");
  return true;
}

template <bool F16, bool SILU, int KIND>
static int launch_tc_t(const tc::TcArgs& t, int nwg, size_t smem, unsigned grid, cudaStream_t s) {
  static size_t attr = 0;
  if (attr < smem) {
    NDF_CUDA_CHECK(cudaFuncSetAttribute(tc::query_tc_kernel<F16, SILU, KIND>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NDF_CUDA_CHECK(cudaFuncSetAttribute(tc::query_ws_kernel<F16, SILU, KIND>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  // Schedule for single-reference grid queries: "ws" (default; 4 epilogue + 2
  // producer warpgroups) or "classic" (4 symmetric warpgroups doing everything;
  // also used for points and multi-reference queries).  Measured on B200 (c1):
  // ws 0.328 ms, classic 0.375 ms per query.
  static int classic = -1;
  if (classic < 0) {
    const char* e = getenv("NDF_TC_SCHEDULE");
    classic = (e && e[0] == 'c') ? 1 : 0;
  }
  if (classic || nwg != 4 || KIND != tc::kGridSingle) {
    tc::query_tc_kernel<F16, SILU, KIND><<<grid, nwg * 128, smem, s>>>(t, nwg);
  } else {
    // warp-specialised: 4 epilogue + 2 producer warpgroups per CTA, one CTA per SM
    const int64_t n = t.q.v1 - t.q.v0;
    const int64_t tiles = (n + tc::kTileM - 1) / tc::kTileM;
    const unsigned g2 = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((tiles + 3) / 4, sm_count()));
    tc::query_ws_kernel<F16, SILU, KIND><<<g2, 768, smem, s>>>(t);
  }
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

template <bool F16>
static int launch_tc_variant(const tc::TcArgs& t, int nwg, size_t smem, unsigned grid,
                             cudaStream_t s) {
  using namespace tc;
  const bool silu = t.q.m.activation == NDF_ACT_SILU;
  const int kind = t.q.mode == 1 ? kPoints : (t.n_ref > 1 ? kGridMulti : kGridSingle);
  if (silu) {
    if (kind == kGridSingle) return launch_tc_t<F16, true, kGridSingle>(t, nwg, smem, grid, s);
    if (kind == kGridMulti) return launch_tc_t<F16, true, kGridMulti>(t, nwg, smem, grid, s);
    return launch_tc_t<F16, true, kPoints>(t, nwg, smem, grid, s);
  }
  if (kind == kGridSingle) return launch_tc_t<F16, false, kGridSingle>(t, nwg, smem, grid, s);
  if (kind == kGridMulti) return launch_tc_t<F16, false, kGridMulti>(t, nwg, smem, grid, s);
  return launch_tc_t<F16, false, kPoints>(t, nwg, smem, grid, s);
}

// Grid / points query on the tensor cores; refs (device, n_ref x 3) and out16 are
// only used by the multi-reference entry point.
static long long* g_trace = nullptr;   // debug hook (ndf_debug_tc_trace)

static int run_tc(const QueryArgs& a, const double* refs_dev, int n_ref, uint16_t* out16,
                  int64_t ld_out, cudaStream_t s) {
  std::string why;
  NDF_REQUIRE(tc_supported(a.m, &why), NDF_ERR_UNSUPPORTED, why);
  NDF_REQUIRE(a.m.params_tc != nullptr, NDF_ERR_PARAMETER,
              "tensor-core query needs the packed parameter blob (ndf_tc_pack)");
  NDF_REQUIRE(a.m.tc_format == a.prec, NDF_ERR_PARAMETER,
              "packed blob element type does not match the requested precision");
  const tc::Layout lay = tc::make_layout(a.m);
  const int blob_al = (lay.blob_bytes + 1023) & ~1023;
  const int nwg = std::min((tc::kMaxSmem - blob_al - 1024) / tc::kABytes, 4);
  const size_t smem = (size_t)blob_al + (size_t)nwg * tc::kABytes + 1024;
  const int64_t n = a.v1 - a.v0;
  const int64_t tiles = (n + tc::kTileM - 1) / tc::kTileM;
  const int64_t ctas = std::min<int64_t>((tiles + nwg - 1) / nwg, sm_count());
  const unsigned grid = (unsigned)std::max<int64_t>(ctas, 1);

  tc::TcArgs t{};
  t.q = a;
  t.n_ref = n_ref;
  t.out16 = out16;
  t.ld_out = ld_out;
  t.trace = g_trace;
  {
    static int stagger = -1;
    if (stagger < 0) {
      const char* e = getenv("NDF_TC_STAGGER");
      stagger = e ? atoi(e) : 1500;
    }
    t.stagger = stagger;
    static int tokens = -1;
    if (tokens < 0) {
      const char* e = getenv("NDF_TC_TOKENS");
      tokens = e ? atoi(e) : 0;
    }
    t.tokens = tokens;
  }
  void* scratch = nullptr;
  if (a.mode == 0) {
    NDF_REQUIRE((int64_t)a.nx * a.ny * a.nz < (1LL << 32), NDF_ERR_UNSUPPORTED,
                "tensor-core grid query supports < 2^32 vertices");
    const int naxis = a.nx + a.ny + a.nz;
    const size_t fbytes = (size_t)naxis * tc::kAxisRow * sizeof(float);
    const size_t ebytes = (size_t)n_ref * tc::kERefStride * sizeof(float);
    NDF_CUDA_CHECK(scratch_alloc(&scratch, fbytes + ebytes + 64, s));
    t.ftab = reinterpret_cast<float*>(scratch);
    t.erefs = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(scratch) + fbytes);
    const double* refs = refs_dev;
    const int threads = 128;
    tc::prep_kernel<<<(naxis + n_ref + threads - 1) / threads, threads, 0, s>>>(
        a, refs, n_ref, const_cast<float*>(t.ftab), const_cast<float*>(t.erefs));
    NDF_LAUNCH_CHECK();
  }
  int st = a.prec == NDF_PREC_FP16 ? launch_tc_variant<true>(t, nwg, smem, grid, s)
                                   : launch_tc_variant<false>(t, nwg, smem, grid, s);
  if (scratch) cudaFreeAsync(scratch, s);
  return st;
}

int launch_query_tc(const QueryArgs& a, cudaStream_t s) { return run_tc(a, nullptr, 1, nullptr, 0, s); }

}  // namespace ndf

using namespace ndf;

// Debug only (not part of the C-ABI header): subsequent tensor-core queries record
// CTA 0's per-phase clock64() stamps into buf[6 * 32 * 12 + 16] (NULL disables).
extern "C" void ndf_debug_tc_trace(long long* buf) { ndf::g_trace = buf; }

extern "C" size_t ndf_tc_blob_bytes(const ndf_model_desc* m) {
  if (!m || !tc_supported(*m, nullptr)) return 0;
  return (size_t)tc::make_layout(*m).blob_bytes;
}

extern "C" int ndf_tc_pack(const ndf_model_desc* m, void* blob, size_t blob_bytes, void* stream) {
  NDF_REQUIRE(m && blob, NDF_ERR_PARAMETER, "null pointer");
  std::string why;
  NDF_REQUIRE(tc_supported(*m, &why), NDF_ERR_UNSUPPORTED, why);
  const tc::Layout lay = tc::make_layout(*m);
  NDF_REQUIRE(blob_bytes >= (size_t)lay.blob_bytes, NDF_ERR_PARAMETER, "blob too small");
  NDF_REQUIRE((reinterpret_cast<uintptr_t>(blob) & 15) == 0, NDF_ERR_PARAMETER,
              "blob must be 16-byte aligned");
  NDF_REQUIRE(m->params_f32 != nullptr, NDF_ERR_PARAMETER, "null params_f32");
  NDF_REQUIRE(m->tc_format == NDF_PREC_BF16 || m->tc_format == NDF_PREC_FP16, NDF_ERR_PARAMETER,
              "tc_format must be NDF_PREC_BF16 or NDF_PREC_FP16");
  tc::pack_zero_kernel<<<64, 256, 0, as_stream(stream)>>>(*m, (uint8_t*)blob);
  NDF_LAUNCH_CHECK();
  tc::pack_fill_kernel<<<64, 256, 0, as_stream(stream)>>>(*m, (uint8_t*)blob);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_query_grid_multi(const ndf_model_desc* m, const double* refs, int32_t n_ref,
                                    int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                                    int64_t v0, int64_t v1, uint16_t* out_f16, int64_t ld_out,
                                    void* stream) {
  int st = validate_model(m);
  if (st) return st;
  NDF_REQUIRE(n_ref >= 1 && refs != nullptr, NDF_ERR_PARAMETER, "need >= 1 reference");
  NDF_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, NDF_ERR_PARAMETER, "grid dims must be >= 1");
  const int64_t V = (int64_t)nx * ny * nz;
  NDF_REQUIRE(v0 >= 0 && v0 <= v1 && v1 <= V, NDF_ERR_PARAMETER, "vertex range out of bounds");
  NDF_REQUIRE(ld_out >= v1 - v0, NDF_ERR_PARAMETER, "ld_out smaller than the vertex range");
  NDF_REQUIRE(out_f16 != nullptr || v0 == v1, NDF_ERR_PARAMETER, "null output");
  NDF_REQUIRE(m->tc_format == NDF_PREC_BF16 || m->tc_format == NDF_PREC_FP16, NDF_ERR_PARAMETER,
              "multi-reference queries run on the tensor-core path only");
  if (v0 == v1) return NDF_OK;
  QueryArgs a{};
  a.m = *m;
  a.g = make_geom(*m);
  a.mode = 0;
  a.ref_is_mu = ref_is_mu ? 1 : 0;
  a.nx = nx; a.ny = ny; a.nz = nz;
  a.v0 = v0; a.v1 = v1;
  a.prec = m->tc_format;
  return run_tc(a, refs, n_ref, out_f16, ld_out, as_stream(stream));
}
