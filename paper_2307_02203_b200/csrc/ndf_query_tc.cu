// Fused NDF query on 5th-generation tensor cores (K1 + K2, sm_100a).
//
//   embed (fp64 -> fp32, bit-exact with model.py:169-177)
//   -> merge [e_r + e_q, |e_r - e_q|]                      (model.py:279-286 + BASELINE)
//   -> H x { tcgen05.mma 16-bit x 16-bit -> fp32 accumulator in TMEM ;
//            tcgen05.ld epilogue: activation, packed back as the next layer's A }
//   -> output layer 128 -> 1 -> head.
//
// Two schedules share the packed parameter blob (UMMA-canonical K-major 16-bit
// weights + fp32 bias vectors, fetched once per CTA by the bulk-copy engine and kept
// resident in SMEM) and the SiLU trick (W and b of SiLU layers pre-scaled by 1/2,
// exact in 16-bit, so silu(x) = y + y tanh(y) with y = x/2: one MUFU tanh and one
// FMA per element):
//
// * query_pp_kernel (default for grid queries with the sum_absdiff merge -- the
//   BASELINE hot path, single reference or multi-reference cube): per CTA two "slots"
//   of 128 query vertices, each with two TMEM accumulator
//   halves so layer l+1's MMAs run underneath layer l's epilogue, hidden-layer A
//   operands taken straight from TMEM, dedicated producer and MMA-issuer warps, and
//   the output layer as an fp32 dot product.  See the comment above the kernel.
//
// * query_tc_kernel ("classic"; paired/points forward and the reference's other
//   merges, single or multi-reference): one CTA per SM with up to 4 symmetric warpgroups,
//   each owning a 128-row tile, one 32 KB SMEM A buffer (SWIZZLE_NONE canonical:
//   8x16 B core matrices, LBO = 128 B along K, SBO = 2048 B along M) and 128 TMEM
//   columns (row m of the tile = TMEM lane m = thread m of the warpgroup); one thread
//   per warpgroup issues a layer's K/16 MMAs and commits them to the warpgroup's
//   mbarrier, so while one warpgroup runs its epilogue the others keep the tensor
//   pipe busy.  Accumulators are pre-loaded with the next layer's bias (tcgen05.st)
//   and the output layer is a 16-column tcgen05.mma (zero-padded B).  Multi-reference
//   queries (BASELINE config 3) embed each query vertex once and reuse it for every
//   reference.
//
// Grid-mode Fourier features are per-axis: prep kernels evaluate them once per axis
// node (the same fp64 sincos, so the same bits) and the queries read them.
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

// Layer-0 A operand layout for the two-block merges (sum_absdiff, concat): the
// blocks are interleaved -- 32-bit word w holds the 16-bit pair (first block,
// second block) of ONE embedding feature -- and the words are grouped by which
// grid axis the feature depends on, in 16-byte (4-word) groups:
//   words  0..11  (sin, cos) of octaves 0..5 along x               groups 0-2
//   words 12..35  (sin, cos) of octaves 0..5 along y, z (octave-major) groups 3-8
//   words 36..51  latent channels 0..15                             groups 9-12
//   words 52..54  raw x, y, z;  word 55 zero padding (K = 112)      group 13
// For a grid query the Fourier-x groups depend only on the vertex column ix and
// the Fourier-yz groups only on its row (iy, iz): they come pre-merged from small
// per-query tables (prep_ws_merge_kernel) straight into the A buffer by cp.async, and
// only the latent and raw words pass through registers.  Layer 0's weight rows
// are permuted identically at pack time.
constexpr int kWordFx = 0, kWordFyz = 12, kWordLat = 36, kWordRaw = 52;
constexpr int kXTabWords = 16;    // per ix: Fourier-x words 0..11, raw-x word at 12
constexpr int kYZTabWords = 32;   // per (iy, iz): Fourier-yz words 0..23, raw y, z at 24, 25

// embedding feature (model.py:169-177 order: raw 3 | Fourier 6L | latent C) -> word
__host__ __device__ __forceinline__ int word_of_feature(int f) {
  if (f < 3) return kWordRaw + f;
  if (f < 3 + 6 * kL) {
    const int j = f - 3, i = j / 6, ax = (j % 6) >> 1, sc = j & 1;
    return ax == 0 ? kWordFx + 2 * i + sc : kWordFyz + 4 * i + 2 * (ax - 1) + sc;
  }
  return kWordLat + (f - 3 - 6 * kL);
}
// inverse of word_of_feature; -1 for the padding word
__host__ __device__ __forceinline__ int feature_of_word(int w) {
  if (w < kWordFyz) return 3 + 6 * (w >> 1) + (w & 1);
  if (w < kWordLat) {
    const int j = w - kWordFyz, i = j >> 2, ax = 1 + ((j >> 1) & 1), sc = j & 1;
    return 3 + 6 * i + 2 * ax + sc;
  }
  if (w < kWordRaw) return 3 + 6 * kL + (w - kWordLat);
  return w < kWordRaw + 3 ? w - kWordRaw : -1;
}

// Column of the tensor-core A operand that holds merged decoder input m (row m of
// W0).  Single-block merges keep the natural order.
__host__ __device__ __forceinline__ int a_column(int merge, int m, int E) {
  if (merge == NDF_MERGE_SUM_ABSDIFF || merge == NDF_MERGE_CONCAT)
    return m < E ? 2 * word_of_feature(m) : 2 * word_of_feature(m - E) + 1;
  return m;
}

// Value of A column c (model.py:279-286 + BASELINE's sum_absdiff), e_a = mu branch.
// MERGE >= 0 fixes the mode at compile time; -1 reads it at run time.
template <int MERGE, class FA, class FB>
__device__ __forceinline__ float merged_value(int merge_rt, int c, FA ea, FB eb) {
  const int merge = MERGE >= 0 ? MERGE : merge_rt;
  if (merge == NDF_MERGE_SUM_ABSDIFF || merge == NDF_MERGE_CONCAT) {
    const int i = feature_of_word(c >> 1);
    if (i < 0) return 0.0f;
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

// Split an fp32 pair into bf16 hi / lo words: hi = bf16(x), lo = bf16(x - hi); the
// difference is exact in fp32 (at most 16 significant bits).
__device__ __forceinline__ void split_pair(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  hi = pack2<false>(x0, x1);
  const float h0 = __uint_as_float(hi << 16), h1 = __uint_as_float(hi & 0xffff0000u);
  float l0, l1;
  ffma2(l0, l1, h0, h1, -1.0f, -1.0f, x0, x1);       // x - hi, exact
  lo = pack2<false>(l0, l1);
}

// 8 consecutive K values of one row of a 16-bit A operand; bf16 (!F16) writes the hi
// plane at abase and the lo plane (x - bf16(x)) at abase + kABytes: the MMAs then run
// A_hi W + A_lo W.
template <bool F16>
__device__ __forceinline__ void store_a8(uint32_t abase, int row, int k, const float* x) {
  if constexpr (F16) {
    st_shared_v4(abase + canon_off(row, k, kSboA), pack2<true>(x[0], x[1]), pack2<true>(x[2], x[3]),
                 pack2<true>(x[4], x[5]), pack2<true>(x[6], x[7]));
  } else {
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_pair(x[2 * i], x[2 * i + 1], h[i], l[i]);
    st_shared_v4(abase + canon_off(row, k, kSboA), h[0], h[1], h[2], h[3]);
    st_shared_v4(abase + kABytes + canon_off(row, k, kSboA), l[0], l[1], l[2], l[3]);
  }
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
      store_a8<F16>(abase, row, kg * 8, x);
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

// Arithmetic latent cell of node i on an n-node axis with r latent nodes: node i sits
// at u = i*(r-1)/(n-1), a single-node axis at the domain centre u = (r-1)/2
// (measures.py:245-247); fp32, as embed_grid_node.
__device__ __forceinline__ void latent_cell(int i, int n, int r, int& i0, float& t) {
  const float ls = n > 1 ? (float)(r - 1) / (float)(n - 1) : 0.0f;
  const float u = n > 1 ? (float)i * ls : 0.5f * (float)(r - 1);
  i0 = min((int)u, r - 2);
  t = fminf(u - (float)i0, 1.0f);
}

// Latent channels of grid node (ix, iy, iz) from the per-query table that
// prep_ws_feat_kernel has already interpolated along z: lerp in y, then in x.
// Called by all 32 lanes; lanes of one (y, z) row share the row's few x cells
// through shuffles (each lane loads one x cell of the two y rows).
__device__ __forceinline__ void latent_yx_lerp(const float* __restrict__ lz, const QueryArgs& a,
                                               int ix, int iy, int iz, float* acc) {
  int x0, y0;
  float tx, ty;
  latent_cell(ix, a.nx, a.g.rx, x0, tx);
  latent_cell(iy, a.ny, a.g.ry, y0, ty);
  const unsigned full = 0xffffffffu;
  const int yz = iy + a.ny * iz;
  const int yz0 = __shfl_sync(full, yz, 0);
  const int xmin = __reduce_min_sync(full, x0);
  const int xmax = __reduce_max_sync(full, x0);
  const size_t rstride = (size_t)a.g.rx * kC;
  const float* r0 = lz + ((size_t)iz * a.g.ry + y0) * rstride;   // row (iz, y0); y0+1 follows
  if (__all_sync(full, yz == yz0) && xmax - xmin + 2 <= 32) {
    const int lane = threadIdx.x & 31;
    float g[kC];
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) g[ch] = 0.0f;
    if (lane < xmax - xmin + 2) {
      const float4* p0 = reinterpret_cast<const float4*>(r0 + (size_t)(xmin + lane) * kC);
      const float4* p1 = reinterpret_cast<const float4*>(r0 + rstride + (size_t)(xmin + lane) * kC);
#pragma unroll
      for (int q = 0; q < kC / 4; ++q) {
        const float4 f = __ldg(p0 + q), h = __ldg(p1 + q);
        g[4 * q + 0] = fmaf(ty, h.x - f.x, f.x);
        g[4 * q + 1] = fmaf(ty, h.y - f.y, f.y);
        g[4 * q + 2] = fmaf(ty, h.z - f.z, f.z);
        g[4 * q + 3] = fmaf(ty, h.w - f.w, f.w);
      }
    }
    const int src = x0 - xmin;
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) {
      const float g0 = __shfl_sync(full, g[ch], src);
      const float g1 = __shfl_sync(full, g[ch], src + 1);
      acc[ch] = fmaf(tx, g1 - g0, g0);
    }
  } else {
    // warp straddles (y, z) rows: same arithmetic per lane, one x cell at a time
    float g0[kC];
#pragma unroll 1
    for (int dx = 0; dx < 2; ++dx) {
      const float4* p0 = reinterpret_cast<const float4*>(r0 + (size_t)(x0 + dx) * kC);
      const float4* p1 = reinterpret_cast<const float4*>(r0 + rstride + (size_t)(x0 + dx) * kC);
#pragma unroll
      for (int q = 0; q < kC / 4; ++q) {
        const float4 f = __ldg(p0 + q), h = __ldg(p1 + q);
        const float gy[4] = {fmaf(ty, h.x - f.x, f.x), fmaf(ty, h.y - f.y, f.y),
                             fmaf(ty, h.z - f.z, f.z), fmaf(ty, h.w - f.w, f.w)};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (dx == 0) g0[4 * q + u] = gy[u];
          else acc[4 * q + u] = fmaf(tx, gy[u] - g0[4 * q + u], g0[4 * q + u]);
        }
      }
    }
  }
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
  const uint32_t* xtab;   // ws schedule: nx x kXTabWords pre-merged x words
  const uint32_t* yztab;  // ws schedule: (ny*nz) x kYZTabWords pre-merged (y, z) words
  const float* lz;        // ws schedule: nz x ry x rx x C latent rows interpolated in z
  int n_ref;
  uint16_t* out16;        // multi-ref output (fp16), rows of ld_out
  int64_t ld_out;
  long long* trace;       // debug: per-phase clock64 stamps of CTA 0 (NULL = off)
  int stagger;            // cycles between warpgroup start times (de-phases the WGs)
  int tokens;             // max warpgroups in an epilogue at once (0 = unlimited)
  const void* px;         // x3 schedule: per-reference PX / PYZ layer-0 tables
  const void* pyz;
  int ngx, ngyz;          //   4-node groups per reference in px / pyz
  int x3_wlo_mask;        //   bit l: hidden layer l runs the A_hi x W_lo term
  int x3_burst;           //   1: issue a hidden layer's MMAs after its whole epilogue
};

// debug tracing of CTA 0's schedule: slot = (wg, tile#, event)
constexpr int kTraceTiles = 32, kTraceEvents = 12;
constexpr int kTraceBase = 6 * kTraceTiles * kTraceEvents;   // + 16 chunk stamps
// Stamps are compiled only into trace builds (-DNDF_TRACE_BUILD, tools/trace_ws.py):
// the shipped library carries no clock reads or trace predicates in the hot loops.
#ifdef NDF_TRACE_BUILD
#define NDF_TRACE_ON(cond) (t.trace && (cond))
#else
#define NDF_TRACE_ON(cond) false
#endif
#define NDF_TRACE_AT(slot_, ev)                                                          \
  do {                                                                                   \
    if (NDF_TRACE_ON(blockIdx.x == 0 && wtid == 0 && (slot_) < kTraceTiles))              \
      t.trace[(wg * kTraceTiles + (slot_)) * kTraceEvents + (ev)] = clock64();          \
  } while (0)
// per-warp stamps of CTA 0, tile 3, layer 1 (tools/trace_ws.py)
#define NDF_TRACE_WARP(e)                                                                \
  do {                                                                                   \
    if (NDF_TRACE_ON(blockIdx.x == 0 && lane == 0 && kk == 3 && l == 1))                 \
      t.trace[kTraceBase + 16 + warp * 8 + (e)] = clock64();                             \
  } while (0)
#define NDF_TRACE(ev)                                                                    \
  do {                                                                                   \
    if (NDF_TRACE_ON(blockIdx.x == 0 && wtid == 0 && tcount < kTraceTiles))               \
      t.trace[(wg * kTraceTiles + tcount) * kTraceEvents + (ev)] = clock64();           \
  } while (0)

// One MMA stage: K/16 tcgen05.mma steps into the warpgroup's accumulator, committed
// to its mbarrier.  Issued by one thread.
// acc_first = 1: the accumulator was pre-loaded (bias) and every step accumulates.
// split: the A operand has a lo plane at a_addr + kABytes (bf16 path), issued as a
// second pass of K/16 steps against the same B.
__device__ __forceinline__ void issue_stage(uint32_t d_tmem, uint32_t a_addr, uint32_t b_addr,
                                            int K, uint32_t sbo_b, uint32_t idesc, uint64_t* bar,
                                            uint32_t acc_first, bool split = false) {
  tc_fence_after();
  for (int p = 0; p < (split ? 2 : 1); ++p) {
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t ad = smem_desc(a_addr + p * kABytes + kk * 256, 128, kSboA);
      const uint64_t bd = smem_desc(b_addr + kk * 256, 128, sbo_b);
      mma_bf16(d_tmem, ad, bd, idesc, (kk > 0 || p > 0) ? 1u : acc_first);
    }
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
  constexpr int kAPer = F16 ? kABytes : 2 * kABytes;   // bf16: hi and lo planes
  uint64_t* bars = reinterpret_cast<uint64_t*>(abufs + nwg * kAPer);     // [0] weights, [1+w]
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
  const uint32_t a_addr = smem_u32(abufs + wg * kAPer);
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
  RangeAcc rng;                                            // ndf_query_grid_stats only
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
                      idesc, bar, 1u, !F16);
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
  if (NDF_TRACE_ON(blockIdx.x == 0 && wg == 0 && wtid == 0 && tcount == 3 && l == 1))     \
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
            for (int i = 0; i < 32; i += 2)              // packed fma.rn.f32x2, same bits
              ffma2(h[i], h[i + 1], v[i], v[i + 1], h[i], h[i + 1], v[i], v[i + 1]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) h[i] = act_f32(a.m.activation, v[i]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) store_a8<F16>(a_addr, wtid, c0 + 8 * j, h + 8 * j);
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
      // bf16: column 3 of the output MMA is A . w_lo (packed into row 3 of the operand)
      if (wtid == 0)
        issue_stage(d_tmem, a_addr, w_addr + lay.wout_off, kHid, kSboA, idesc_out, bar, 0u, !F16);
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_fence_after();
      NDF_TRACE(10);
      uint32_t zr, z1, z2, z3;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(zr), "=r"(z1), "=r"(z2), "=r"(z3) : "r"(tmem_row));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      (void)z1; (void)z2;
      if (valid) {
        const float zo = F16 ? __uint_as_float(zr) : __uint_as_float(zr) + __uint_as_float(z3);
        const float z = head_exact(a.m.head, zo + bias_out);
        if (t.out16) {
          const __half hz = __float2half_rn(z);
          t.out16[(size_t)r * t.ld_out + vloc] = *reinterpret_cast<const uint16_t*>(&hz);
        } else {
          a.out[vloc] = z;
          if (a.stats) rng.add(z);
        }
      }
    }
  }
  if (a.stats) rng.flush(a.stats);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Issue K16 steps [k0, k0 + nsteps) of one layer into d_tmem (one thread).
__device__ __forceinline__ void issue_ksteps(uint32_t d_tmem, uint32_t a_addr, uint32_t b_addr,
                                             int k0, int nsteps, uint32_t sbo_b, uint32_t idesc,
                                             bool accumulate_first) {
  for (int kk = k0; kk < k0 + nsteps; ++kk) {
    const uint64_t ad = smem_desc(a_addr + kk * 256, 128, kSboA);
    const uint64_t bd = smem_desc(b_addr + kk * 256, 128, sbo_b);
    mma_bf16(d_tmem, ad, bd, idesc, (kk > k0 || accumulate_first) ? 1u : 0u);
  }
}
// A operand in TMEM ("TS" form): K16 steps [k0, k0 + nsteps), step kk's 8 columns at
// a_col(kk) = a_tmem + 16 kk (the epilogue packs each 16-column sub-chunk's 16-bit
// activations into the first 8 of its own, already drained, columns).
__device__ __forceinline__ void issue_ksteps_ts(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_addr,
                                                int k0, int nsteps, uint32_t sbo_b,
                                                uint32_t idesc, bool accumulate_first) {
  for (int kk = k0; kk < k0 + nsteps; ++kk) {
    const uint32_t ac = a_tmem + (uint32_t)(16 * kk);
    const uint64_t bd = smem_desc(b_addr + kk * 256, 128, sbo_b);
    const uint32_t acc = (kk > k0 || accumulate_first) ? 1u : 0u;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(ac), "l"(bd), "r"(idesc), "r"(acc));
  }
}
// warp-collective forms (whole warp, uniform operands, elect.sync inside; ndf_tc_ptx.cuh)
__device__ __forceinline__ void issue_ksteps_warp(uint32_t d_tmem, uint32_t a_addr, uint32_t b_addr,
                                                  int k0, int nsteps, uint32_t sbo_b, uint32_t idesc,
                                                  bool accumulate_first) {
#pragma unroll
  for (int kk = k0; kk < k0 + nsteps; ++kk)
    mma_ss_warp(d_tmem, smem_desc(a_addr + kk * 256, 128, kSboA), smem_desc(b_addr + kk * 256, 128, sbo_b),
                idesc, (kk > k0 || accumulate_first) ? 1u : 0u);
}
__device__ __forceinline__ void issue_ksteps_ts_warp(uint32_t d_tmem, uint32_t a_tmem,
                                                     uint32_t b_addr, int k0, int nsteps,
                                                     uint32_t sbo_b, uint32_t idesc,
                                                     bool accumulate_first) {
#pragma unroll
  for (int kk = k0; kk < k0 + nsteps; ++kk)
    mma_ts_warp(d_tmem, a_tmem + (uint32_t)(16 * kk), smem_desc(b_addr + kk * 256, 128, sbo_b),
                idesc, (kk > k0 || accumulate_first) ? 1u : 0u);
}
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// Timing experiment only (tools/ab_variants.sh): NDF_EXP_NOMUFU replaces tanh by an
// FMA-pipe stand-in (results are wrong).
#ifdef NDF_EXP_NOMUFU
#define NDF_EXP_TANH(x) ((x) * 0.25f)
#else
#define NDF_EXP_TANH(x) tanh_fast(x)
#endif

// SiLU of 16 pre-halved accumulators: h = y + y tanh(y) (weights and biases of SiLU
// layers are pre-scaled by 1/2), one MUFU tanh per element and packed fp32 FMAs
// (fma.rn.f32x2: same rounding as fmaf, half the issue slots).
// NDF_POLY_PAIRS pairs of the 16 (the last 2 * NDF_POLY_PAIRS columns of every sub-chunk)
// take tanh from tanh2_fma on the FMA pipe instead of MUFU (ndf_tc_ptx.cuh).  Measured on
// B200 and rejected (default 0): 1 / 2 / 3 pairs cost bf16 0.327 -> 0.352 / 0.361 / 0.395 ms
// and fp16 0.241 -> 0.250 / 0.287 / 0.308 ms -- the epilogue is bound by instruction issue
// and latency, not by MUFU throughput, so ~15 extra instructions per pair lose more than
// the freed MUFU slots gain.
#ifndef NDF_POLY_PAIRS
#define NDF_POLY_PAIRS 0
#endif
__device__ __forceinline__ void silu16(const float* x, float* h) {
  constexpr int kMufu = 16 - 2 * NDF_POLY_PAIRS;
#pragma unroll
  for (int i = 0; i < kMufu; ++i) h[i] = NDF_EXP_TANH(x[i]);
#pragma unroll
  for (int i = kMufu; i < 16; i += 2) tanh2_fma(x[i], x[i + 1], h[i], h[i + 1]);
#pragma unroll
  for (int i = 0; i < 16; i += 2)
    ffma2(h[i], h[i + 1], x[i], x[i + 1], h[i], h[i + 1], x[i], x[i + 1]);
}

// Hidden-layer epilogue of one 16-column sub-chunk (the bias is already in the
// accumulator): activation, 16-bit pack, and one tcgen05.st of the 8 packed words
// into TMEM, where the next layer's MMA reads its A operand (row = lane, K-pairs
// along the columns).
template <bool F16, bool SILU>
__device__ __forceinline__ void epilogue16(const float* x, int act, uint32_t a_taddr) {
  float h[16];
  if constexpr (SILU) {
    silu16(x, h);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = act_f32(act, x[i]);
  }
  uint32_t p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = pack2<F16>(h[2 * i], h[2 * i + 1]);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               ::"r"(a_taddr), "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]),
               "r"(p[6]), "r"(p[7]) : "memory");
}

// Last hidden layer, one 16-column sub-chunk (bias already in the accumulator):
// activation in fp32, then the output layer's partial dot product (fp32 weights in
// rows 1-2 of the packed N=16 output operand: k-group g's 8 weights are the 32
// bytes at g*128 + 16).
template <bool SILU>
__device__ __forceinline__ void dot16(const float* x, int c0, int act, uint32_t wout_addr,
                                      float* dots) {
  float w[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t wa = wout_addr + (uint32_t)(((c0 >> 3) + (q >> 1)) * 128 + 16 + 16 * (q & 1));
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(w[4 * q]), "=f"(w[4 * q + 1]), "=f"(w[4 * q + 2]), "=f"(w[4 * q + 3]) : "r"(wa));
  }
  float h[16];
  if constexpr (SILU) {
    silu16(x, h);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = act_f32(act, x[i]);
  }
  // dots[c] accumulates elements i = c (mod 4) in ascending i, two lanes per FFMA2
#pragma unroll
  for (int i = 0; i < 16; i += 2)
    ffma2(dots[i & 3], dots[(i & 3) + 1], h[i], h[i + 1], w[i], w[i + 1], dots[i & 3],
          dots[(i & 3) + 1]);
}

// Ping-pong schedule for grid queries with the sum_absdiff merge (the default --
// NDF_TC_SCHEDULE=classic selects query_tc_kernel instead).  A launch covers t.n_ref
// references: tile T is vertex tile T mod n_vt of reference T / n_vt, with that
// reference's x / (y, z) tables and latent channels; rows go to out (fp32, single
// reference) or out16 (fp16 cube rows of ld_out).
//   2 slots per CTA, each = 256 TMEM columns holding TWO accumulator halves plus a
//   32 KB SMEM buffer for layer 0's A operand.  Layer l of a slot accumulates into
//   half (l & 1) while the epilogue drains the other half, so the next layer's MMA
//   runs underneath the current epilogue (issued 32 K-columns at a time) instead of
//   after it.  Hidden layers take their A operand from TMEM ("TS" MMA): the epilogue
//   packs each 16-column sub-chunk's 16-bit activations into the first 8 of its own,
//   just drained, columns (K16 step k reads column 16k), so activations never touch
//   shared memory.
//   WG0-3 -- epilogue: WG 2s+c with the 4 TMEM lane quarters of slot s; column half c
//            drains sub-chunks c, c+2, c+4, c+6, so K-chunk i (sub-chunks 2i, 2i+1)
//            completes i-th.  Per sub-chunk: tcgen05.ld (one ahead), SiLU (MUFU tanh +
//            FFMA2), pack, tcgen05.st, bar.arrive on K-chunk barrier i.  The last
//            hidden layer feeds an fp32 dot product with the output weights instead
//            (the two column halves split at column 64, partials summed through SMEM)
//            and the head.
//   WG4, WG5 -- producer of slot 0 / 1: per query tile, the latent words (y/x lerp of
//            the prep kernel's z-interpolated rows, merged with the reference) and
//            raw-coordinate words in registers; once the previous layer-0 MMA has
//            consumed the SMEM A buffer, the pre-merged Fourier groups by cp.async
//            from the per-query x / (y, z) tables and the registers stored; the
//            layer-0 MMA is issued once the target accumulator half is drained.
//   WG6 -- warps 24 + s: the MMA issuer of slot s, blocked in bar.sync on the K-chunk
//            barriers; each passage issues that K-chunk's two K16 steps of the next
//            layer (the bias step first), tcgen05.commit after the fourth.  Issuing
//            blocks the issuing thread until the tensor core accepts the MMA, so a
//            warp of its own keeps that off the epilogue's critical path (as an
//            epilogue warp it made its lane quarter the straggler of every layer).
//   setmaxnreg rebalances the register file: launch 72, epilogue 80, producer 72
//   (64 spilled its per-tile state), issuer 24.
// Synchronisation: acc_full[s] (tcgen05.commit of each layer's MMAs), s_free[s]
// (layer 0's SMEM A consumed: the producer may write the next tile's), d_free[s] (the
// tile's last MMA has completed: the next tile's layer 0 may target the other D half)
// and named barriers 1 + 4s + i per K-chunk (8 epilogue warps arrive, the issuer syncs).
constexpr int kPPSlots = 2;
constexpr int kPPThreads = 896;
constexpr int kBiasBlk = 128 * 16 * 2;     // one 128 x 16 16-bit operand block

template <bool F16, bool SILU>
__global__ void __launch_bounds__(kPPThreads, 1)
query_pp_kernel(const TcArgs t) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const QueryArgs& a = t.q;
  const Layout lay = make_layout(a.m);
  uint8_t* wblob = smem;
  uint8_t* abufs = smem + ((lay.blob_bytes + 1023) & ~1023);
  // bias folding: a 128x16 "ones" A block (column 0 = 1) and per layer a 16x128 B block
  // whose k=0 row is the layer's bias, so one extra K16 MMA step initialises the
  // accumulator with the bias and the epilogue has no bias adds
  uint8_t* ones_blk = abufs + kPPSlots * kABytes;
  uint8_t* bias_blk = ones_blk + kBiasBlk;                    // [H] x kBiasBlk
  uint64_t* bars = reinterpret_cast<uint64_t*>(bias_blk + lay.H * kBiasBlk);
  uint64_t* wbar = &bars[0];
  uint64_t* acc_full = &bars[1];                  // [kPPSlots] a layer's MMAs completed
  uint64_t* s_free = &bars[1 + kPPSlots];         // [kPPSlots] layer-0 SMEM A consumed
  uint64_t* d_free = &bars[1 + 2 * kPPSlots];     // [kPPSlots] next tile's D half drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  float* eref_s = reinterpret_cast<float*>(bars + 16);      // reference latent channels
  float* dotx = reinterpret_cast<float*>(bars + 32);  // [2 tile parities][kPPSlots][128] partials

  const int tid = threadIdx.x;
  const int warp = warp_uniform(tid >> 5);
  const int lane = tid & 31;
  const int wg = warp >> 2;
  const int wq = warp & 3;                        // TMEM lane quarter
  const int wtid = tid & 127;                     // tile row
  const float* vecs = reinterpret_cast<const float*>(wblob + lay.vec_off);

  if (tid == 0) {
    mbar_init(wbar, 1);
    for (int s = 0; s < kPPSlots; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&s_free[s], 1);
      mbar_init(&d_free[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  {
    // ones / bias blocks (K-major canonical, SBO 256 B): row r, 8-element group g at
    // (r >> 3) * 256 + g * 128 + (r & 7) * 16; only element k = 0 of each row is nonzero
    const float* gvec = reinterpret_cast<const float*>(
        reinterpret_cast<const uint8_t*>(a.m.params_tc) + lay.vec_off);
    for (int i = tid; i < (1 + lay.H) * 256; i += blockDim.x) {
      const int blk = i >> 8, r = (i >> 1) & 127, g = i & 1;
      const float v0 = g ? 0.0f : (blk == 0 ? 1.0f : __ldg(gvec + (blk - 1) * kHid + r));
      st_shared_v4(smem_u32(ones_blk + blk * kBiasBlk) + (r >> 3) * 256 + g * 128 + (r & 7) * 16,
                   pack2<F16>(v0, 0.0f), 0u, 0u, 0u);
    }
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_expect_tx(wbar, (uint32_t)lay.blob_bytes);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.m.params_tc);
    for (int off = 0; off < lay.blob_bytes; off += 32768)
      bulk_g2s(wblob + off, src + off, (uint32_t)min(32768, lay.blob_bytes - off), wbar);
  }
  // Everything above only touches the model; launched with programmatic stream
  // serialisation, it overlaps the per-query prep kernels.  Their outputs are read
  // only after this wait.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tid < kC) eref_s[tid] = t.erefs[tid];
  __syncthreads();
  const uint32_t tmem_base = warp_uniform(*tmem_slot);
  const uint32_t w_addr = smem_u32(wblob);
  const uint32_t ab_fmt = F16 ? 0u : 1u;
  const uint32_t idesc = (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) |
                         ((uint32_t)(kHid >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);
  const uint32_t sbo_w0 = (uint32_t)(lay.kin / 8) * 128;
  const int H = lay.H;

  const int64_t n = a.v1 - a.v0;
  // multi-reference cubes: tile T covers vertex tile T % n_vt of reference T / n_vt, so
  // concurrently running tiles share one reference's tables in L2
  const int64_t n_vt = (n + kTileM - 1) / kTileM;
  const int64_t n_tiles = n_vt * t.n_ref;
  const int64_t tile_stride = (int64_t)gridDim.x * kPPSlots;
  const int s = wg < 4 ? (wg >> 1) : wg - 4;        // slot of this warpgroup
  const int64_t first = (int64_t)blockIdx.x * kPPSlots + s;
  const int64_t cnt = first < n_tiles ? (n_tiles - first + tile_stride - 1) / tile_stride : 0;
  const uint32_t a_addr = smem_u32(abufs + s * kABytes);
  const uint32_t d_slot = tmem_base + (uint32_t)(s * 2 * kHid);   // + kHid * half

  if (wg == 6) {
    // ======================== MMA issuer of slot warp - 24 ===========================
#ifndef NDF_PP_ISSUER_REGS
#define NDF_PP_ISSUER_REGS 24
#endif
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(NDF_PP_ISSUER_REGS));
    const int si = warp - 24;
    if (si < kPPSlots) {
      const int64_t fi = (int64_t)blockIdx.x * kPPSlots + si;
      const int64_t ci = fi < n_tiles ? (n_tiles - fi + tile_stride - 1) / tile_stride : 0;
      const uint32_t ds = tmem_base + (uint32_t)(si * 2 * kHid);
      mbar_wait(wbar, 0);
#pragma unroll 1
      for (int64_t kk = 0; kk < ci; ++kk) {
#pragma unroll 1
        for (int l = 0; l + 1 < H; ++l) {
          const uint32_t half = (uint32_t)((kk * H + l) & 1);
          const uint32_t d_next = ds + (half ^ 1u) * kHid;
          const uint32_t a_tm = ds + half * kHid;                      // A of layer l+1
          const uint32_t wl = w_addr + lay.w0_bytes + l * lay.wh_bytes;
#pragma unroll 1
          for (int k2 = 0; k2 < 4; ++k2) {
            named_bar(1 + 4 * si + k2, 288);
            NDF_TRACE_WARP(2 * k2);
            // whole issuer warp (elect.sync inside the MMA asm): uniform operands, the
            // MMAs go out back to back (x3 kernel: 0.41 -> 0.33 ms from this alone)
#ifdef NDF_PP_LANE0_ISSUER   // A/B: round-1 single-lane issue
            if (lane == 0) {
              tc_fence_after();
              if (k2 == 0)
                mma_bf16(d_next, smem_desc(smem_u32(ones_blk), 128, 256),
                         smem_desc(smem_u32(bias_blk + (l + 1) * kBiasBlk), 128, 256), idesc, 0u);
              issue_ksteps_ts(d_next, a_tm, wl, 2 * k2, 2, kSboA, idesc, true);
              if (k2 == 3) mma_commit(&acc_full[si]);
            }
#else
            tc_fence_after();
            if (k2 == 0)
              mma_ss_warp(d_next, smem_desc(smem_u32(ones_blk), 128, 256),      // D = bias
                          smem_desc(smem_u32(bias_blk + (l + 1) * kBiasBlk), 128, 256), idesc, 0u);
#ifndef NDF_EXP_NOKSTEP     // timing experiment: hidden-layer K16 steps skipped (wrong results)
            issue_ksteps_ts_warp(d_next, a_tm, wl, 2 * k2, 2, kSboA, idesc, true);
#else
            (void)a_tm; (void)wl;
#endif
            if (k2 == 3) mma_commit_warp(&acc_full[si]);
#endif
            NDF_TRACE_WARP(2 * k2 + 1);
          }
        }
      }
    }
  } else if (wg >= 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    // ============================ producer (slot s) ==================================
#pragma unroll 1
    for (int64_t kk = 0; kk < cnt; ++kk) {
      const int64_t tile_g = first + kk * tile_stride;
      const int r = t.n_ref == 1 ? 0 : (int)((uint32_t)tile_g / (uint32_t)n_vt);
      const int64_t tile = tile_g - (int64_t)r * n_vt;
      const uint32_t* xtab = t.xtab + (size_t)r * a.nx * kXTabWords;
      const uint32_t* yztab = t.yztab + (size_t)r * a.ny * a.nz * kYZTabWords;
      NDF_TRACE_AT((int)kk, 0);
      int ix, iy, iz;
      tile_node(a, tile, wtid, ix, iy, iz);
      const int yzrow = iy + a.ny * iz;
      uint32_t pv[20];    // words 36..55
      {
        float lat[kC];
#ifdef NDF_EXP_NOPROD    // timing experiment: no latent gather / Fourier copies (wrong results)
#pragma unroll
        for (int c = 0; c < kC; ++c) lat[c] = 0.0f;
#else
        latent_yx_lerp(t.lz, a, ix, iy, iz, lat);
#endif
#pragma unroll
        for (int q = 0; q < kC / 4; ++q) {
          const float4 r4 = t.n_ref == 1
              ? reinterpret_cast<const float4*>(eref_s)[q]
              : __ldg(reinterpret_cast<const float4*>(t.erefs + (size_t)r * kERefStride) + q);
          const float rv[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            pv[4 * q + u] = pack2<F16>(rv[u] + lat[4 * q + u], fabsf(rv[u] - lat[4 * q + u]));
        }
        pv[16] = __ldg(xtab + (size_t)ix * kXTabWords + 12);
        const uint2 ryz =
            __ldg(reinterpret_cast<const uint2*>(yztab + (size_t)yzrow * kYZTabWords + 24));
        pv[17] = ryz.x;
        pv[18] = ryz.y;
        pv[19] = 0u;
      }
      NDF_TRACE_AT((int)kk, 1);
      if (kk >= 1) mbar_wait(&s_free[s], (uint32_t)((kk - 1) & 1));   // previous layer 0 done
      NDF_TRACE_AT((int)kk, 2);
      {
        const uint32_t* xs = xtab + (size_t)ix * kXTabWords;
        const uint32_t* ys = yztab + (size_t)yzrow * kYZTabWords;
#ifndef NDF_EXP_NOPROD
#pragma unroll
        for (int g = 0; g < 3; ++g)
          cp_async16(a_addr + canon_off(wtid, 2 * kWordFx + 8 * g, kSboA), xs + 4 * g);
#pragma unroll
        for (int g = 0; g < 6; ++g)
          cp_async16(a_addr + canon_off(wtid, 2 * kWordFyz + 8 * g, kSboA), ys + 4 * g);
#else
        (void)xs; (void)ys;
#endif
        cp_async_commit();
      }
#pragma unroll
      for (int g = 0; g < 5; ++g)
        st_shared_v4(a_addr + canon_off(wtid, 2 * kWordLat + 8 * g, kSboA), pv[4 * g],
                     pv[4 * g + 1], pv[4 * g + 2], pv[4 * g + 3]);
      cp_async_wait_all();
      fence_proxy_async();
      named_bar(11 + s, 128);
#ifndef NDF_PP_WARP_PRODUCER
      // Layer 0 is issued by one producer thread.  A warp-collective producer issue (as
      // the issuer warps and the x3 kernel use) deadlocked this kernel within 50-800
      // back-to-back c1 queries on B200 (tools/stress_query.py; either change alone
      // passes 6,000 + 20,000, as does the x3 kernel with both: 35,000) -- root cause not
      // found, so the single-thread form stays here (it costs 0.006 ms).
      if (wtid == 0) {
        if (kk == 0) mbar_wait(wbar, 0);
        else mbar_wait(&d_free[s], (uint32_t)((kk - 1) & 1));
        tc_fence_after();
        const uint32_t half = (uint32_t)((kk * H) & 1);
        mma_bf16(d_slot + half * kHid, smem_desc(smem_u32(ones_blk), 128, 256),
                 smem_desc(smem_u32(bias_blk), 128, 256), idesc, 0u);
        issue_ksteps(d_slot + half * kHid, a_addr, w_addr, 0, lay.kin / 16, sbo_w0, idesc, true);
        mma_commit(&acc_full[s]);
      }
#else
      if (wq == 0) {                  // the producer's first warp issues layer 0 (elect.sync)
        if (kk == 0) mbar_wait(wbar, 0);
        else mbar_wait(&d_free[s], (uint32_t)((kk - 1) & 1));   // target D half drained
        tc_fence_after();
        const uint32_t half = (uint32_t)((kk * H) & 1);
        mma_ss_warp(d_slot + half * kHid, smem_desc(smem_u32(ones_blk), 128, 256),
                    smem_desc(smem_u32(bias_blk), 128, 256), idesc, 0u);       // D = b0
        issue_ksteps_warp(d_slot + half * kHid, a_addr, w_addr, 0, lay.kin / 16, sbo_w0, idesc,
                          true);
        mma_commit_warp(&acc_full[s]);
      }
#endif
      NDF_TRACE_AT((int)kk, 3);
    }
  } else {
    // ======================== epilogue (slot s, column half ch) ======================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 80;");
    const int ch = wg & 1;
    const bool lead = ch == 0 && wq == 0;           // arrives the s_free / d_free mbarriers
    // column half ch drains sub-chunks ch, ch+2, ch+4, ch+6 (16 columns each): K-chunk
    // barrier i completes sub-chunks 2i, 2i+1, so chunks complete in issue order and only
    // one K-chunk (two K16 steps) is left to issue when the epilogue ends
    const uint32_t first_col = 16u * (uint32_t)ch;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    mbar_wait(wbar, 0);
    const float bias_out = vecs[H * kHid];
    const uint32_t wout_addr = w_addr + lay.wout_off;
    uint32_t acc_ph = 0u;
    // a finished tile's output is written late, after the next tile's first epilogue (the
    // column-0 warps would wait on the layer-1 MMAs there anyway) -- as in query_x3_kernel
    float z_pend = 0.0f;
    int64_t kk_pend = -1;
    RangeAcc rng;                                   // ndf_query_grid_stats only
    auto flush = [&]() {
      if (kk_pend < 0) return;
      const int64_t tile_g = first + kk_pend * tile_stride;
      const int64_t r = t.n_ref == 1 ? 0 : (int64_t)((uint32_t)tile_g / (uint32_t)n_vt);
      const int64_t vloc = (tile_g - r * n_vt) * kTileM + wtid;
      if (vloc < n) {
        const float o = head_exact(a.m.head, z_pend);
        if (t.out16) {
          const __half ho = __float2half_rn(o);
          t.out16[r * t.ld_out + vloc] = *reinterpret_cast<const uint16_t*>(&ho);
        } else {
          a.out[vloc] = o;
          if (a.stats) rng.add(o);
        }
      }
      kk_pend = -1;
    };
#pragma unroll 1
    for (int64_t kk = 0; kk < cnt; ++kk) {
#pragma unroll 1
      for (int l = 0; l < H; ++l) {
        const uint32_t half = (uint32_t)((kk * H + l) & 1);
        const uint32_t d_base = d_slot + lane_base + half * kHid;   // this lane quarter
        mbar_wait(&acc_full[s], acc_ph);
        acc_ph ^= 1u;
        tc_fence_after();
        if (l == 0 && lead && lane == 0) mbar_arrive(&s_free[s]);   // SMEM A reusable
        NDF_TRACE_AT((int)kk, 2 * l);
        float va[16], vb[16];
        tmem_ld16_nowait(d_base + first_col, va);
        tmem_wait_ld();
        NDF_TRACE_WARP(0);
        if (l + 1 < H) {
          // ---- hidden layer l -> A of layer l+1: each sub-chunk's activations are packed
          // into the first 8 of its own, just drained, TMEM columns; the issuer warp sends
          // K-chunk i's two K16 steps of layer l+1 once barrier i completes ------------
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t col = first_col + 32u * (uint32_t)i;
            float* cur = (i & 1) ? vb : va;
            float* nxt = (i & 1) ? va : vb;
            if (i + 1 < 4) tmem_ld16_nowait(d_base + col + 32u, nxt);
            epilogue16<F16, SILU>(cur, a.m.activation, d_base + col);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            named_bar_arrive(1 + 4 * s + i, 288);     // 8 draining warps + the issuer
            NDF_TRACE_WARP(1 + i);
            if (i + 1 < 4) tmem_wait_ld();
          }
          NDF_TRACE_WARP(6);
          NDF_TRACE_AT((int)kk, 2 * l + 1);
          if (l == 0) flush();
        } else {
          // ---- last hidden layer: A is free for the producer; fp32 output dot ---------
          // layer H-1's MMA has completed, so the other D half (which held layer H-2 and
          // then A of layer H-1) is free for the next tile's layer 0
          if (lead && lane == 0) mbar_arrive(&d_free[s]);
          // the output dot product splits at column 64 for every lane quarter, so its fp32
          // summation order -- and the bits -- never depend on a vertex's row in the tile
          float dots[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          if (first_col != 64u * ch) tmem_ld16_nowait(d_base + 64u * ch, va);
          if (first_col != 64u * ch) tmem_wait_ld();
#pragma unroll 1
          for (int kc = 2 * ch; kc < 2 * ch + 2; ++kc) {
            const int col = 32 * kc;
            tmem_ld16_nowait(d_base + (uint32_t)(col + 16), vb);
            dot16<SILU>(va, col, a.m.activation, wout_addr, dots);
            tmem_wait_ld();
            if (kc + 1 < 2 * ch + 2) tmem_ld16_nowait(d_base + (uint32_t)(col + 32), va);
            dot16<SILU>(vb, col + 16, a.m.activation, wout_addr, dots);
            if (kc + 1 < 2 * ch + 2) tmem_wait_ld();
          }
          tc_fence_before();
          const float part = (dots[0] + dots[1]) + (dots[2] + dots[3]);
          float* dx = dotx + ((kk & 1) * kPPSlots + s) * kTileM;
          if (ch == 1) {
            dx[wtid] = part;
            named_bar_arrive(9 + s, 256);
          } else {
            named_bar(9 + s, 256);
            z_pend = part + dx[wtid] + bias_out;
            kk_pend = kk;
            if (H == 1) flush();
          }
          NDF_TRACE_AT((int)kk, 2 * l + 1);
          // no second barrier: dotx is double-buffered by tile parity (see x3)
          NDF_TRACE_AT((int)kk, 6);
        }
      }
    }
    flush();
    if (a.stats && ch == 0) rng.flush(a.stats);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
}

#include "ndf_query_x3.cuh"

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

// ---- per-query prep for the warp-specialised schedule (sum_absdiff merge) ----
// raw coordinate and (sin, cos) of the L octaves of one clipped axis coordinate:
// the same fp64 operations as embed_point_t, so the same bits.
__device__ __forceinline__ void axis_features(double p, float* f) {
  f[0] = (float)p;
  double scale = 3.141592653589793;
#pragma unroll
  for (int i = 0; i < kL; ++i) {
    double sn, cs;
    sincos(dmul(scale, p), &sn, &cs);
    f[1 + 2 * i] = (float)sn;
    f[2 + 2 * i] = (float)cs;
    scale = scale * 2.0;
  }
}

// Per-query prep, kernel 1 of 2 (one thread per item):
//   [0, F)    F = (nx+ny+nz+3)*L: one fp64 sincos each -> feat[node][1+2o, 2+2o]
//             (the octave-0 thread also writes the raw coordinate feat[node][0]);
//             nodes are the x, y, z axis nodes, then the reference's x, y, z
//   F         the reference's latent channels in fp64 (embed_point_t's latent part)
//   beyond    lz[iz][cy][cx][:] = latent grid interpolated along z at node iz
//             (fp32; the query branch's grid)
// Same fp64 operations as embed_point_t, so every feature has the same bits; one
// sincos per thread keeps the fp64 latency chain short.
// refs: n_ref x 3 fp64 device reference points (multi-reference cube), or NULL for
// the single reference in a.ref.  Nodes: nx + ny + nz query axis nodes, then 3 per
// reference; the reference latent channels go to eref_lat + r * kERefStride.
__global__ void prep_ws_feat_kernel(const QueryArgs a, const double* refs, int n_ref, float* feat,
                                    float* eref_lat, float* lz) {
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = a.nx + a.ny + a.nz;
  const int nnode = nq + 3 * n_ref;
  const int64_t F = (int64_t)nnode * kL;
  if (tid < F) {
    const int node = (int)(tid / kL), o = (int)(tid % kL);
    double p;
    if (node < a.nx) p = node_coord(node, a.nx);
    else if (node < a.nx + a.ny) p = node_coord(node - a.nx, a.ny);
    else if (node < nq) p = node_coord(node - a.nx - a.ny, a.nz);
    else p = refs ? refs[node - nq] : a.ref[node - nq];
    p = fmin(fmax(p, -1.0), 1.0);
    double scale = 3.141592653589793;
    for (int i = 0; i < o; ++i) scale = scale * 2.0;
    double sn, cs;
    sincos(dmul(scale, p), &sn, &cs);
    float* f = feat + (size_t)node * 16;
    f[1 + 2 * o] = (float)sn;
    f[2 + 2 * o] = (float)cs;
    if (o == 0) f[0] = (float)p;
  } else if (tid < F + n_ref) {
    const int r = (int)(tid - F);
    const double* rp = refs ? refs + 3 * r : a.ref;
    const float* grid = a.ref_is_mu ? a.m.grid_mu : a.m.grid_nu;
    const double p[3] = {fmin(fmax(rp[0], -1.0), 1.0), fmin(fmax(rp[1], -1.0), 1.0),
                         fmin(fmax(rp[2], -1.0), 1.0)};
    const AxisCoord cx = level_coord(p[0], a.g.rx);
    const AxisCoord cy = level_coord(p[1], a.g.ry);
    const AxisCoord cz = level_coord(p[2], a.g.rz);
    double acc[kC];
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) acc[ch] = 0.0;
    for (int c = 0; c < 8; ++c) {      // embed_point_t's corner order and rounding
      const int dx = c & 1, dy = (c >> 1) & 1, dz = c >> 2;
      const double wx = dx ? cx.t : dsub(1.0, cx.t);
      const double wy = dy ? cy.t : dsub(1.0, cy.t);
      const double wz = dz ? cz.t : dsub(1.0, cz.t);
      const double w = dmul(dmul(wx, wy), wz);
      const int idx = (cx.i0 + dx) + a.g.rx * ((cy.i0 + dy) + a.g.ry * (cz.i0 + dz));
#pragma unroll
      for (int ch = 0; ch < kC; ++ch)
        acc[ch] = dadd(acc[ch], dmul(w, (double)__ldg(grid + (size_t)idx * kC + ch)));
    }
    for (int ch = 0; ch < kC; ++ch) eref_lat[(size_t)r * kERefStride + ch] = (float)acc[ch];
  } else {
    const int64_t k = tid - F - n_ref;
    if (k >= (int64_t)a.nz * a.g.ry * a.g.rx) return;
    const int cx = (int)(k % a.g.rx), cy = (int)((k / a.g.rx) % a.g.ry);
    const int iz = (int)(k / ((int64_t)a.g.rx * a.g.ry));
    int z0;
    float tz;
    latent_cell(iz, a.nz, a.g.rz, z0, tz);
    const float* grid = a.ref_is_mu ? a.m.grid_nu : a.m.grid_mu;   // query branch
    const float4* p0 = reinterpret_cast<const float4*>(
        grid + ((size_t)(z0 * a.g.ry + cy) * a.g.rx + cx) * kC);
    const float4* p1 = p0 + (size_t)a.g.ry * a.g.rx * kC / 4;
    float4* dst = reinterpret_cast<float4*>(lz + (size_t)k * kC);
#pragma unroll
    for (int q = 0; q < kC / 4; ++q) {
      const float4 f = __ldg(p0 + q), h = __ldg(p1 + q);
      dst[q] = make_float4(fmaf(tz, h.x - f.x, f.x), fmaf(tz, h.y - f.y, f.y),
                           fmaf(tz, h.z - f.z, f.z), fmaf(tz, h.w - f.w, f.w));
    }
  }
}

// Per-query prep, kernel 2 of 2: merge the reference's and the query nodes' axis
// features into the 16-bit A words ([r + q, |r - q|], model.py:279-286 + BASELINE):
//   [0, nx)             xtab[ix]   = Fourier-x words 0..11, raw-x word at 12
//   [nx, nx + ny*nz)    yztab[row] = Fourier-(y, z) words in A order, raw y, z at 24, 25
template <bool F16>
// Per reference r: nx x-rows then ny*nz (y, z)-rows, tables of reference r at
// xtab + r * nx * kXTabWords and yztab + r * ny * nz * kYZTabWords.
__global__ void prep_ws_merge_kernel(const QueryArgs a, int n_ref, const float* __restrict__ feat,
                                     uint32_t* xtab, uint32_t* yztab) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");      // feat from prep_ws_feat_kernel
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nyz = a.ny * a.nz;
  const int64_t rows = (int64_t)a.nx + nyz;
  if (gtid >= rows * n_ref) return;
  const int r = (int)(gtid / rows);
  const int64_t tid = gtid - (int64_t)r * rows;
  const int nref = a.nx + a.ny + a.nz + 3 * r;  // first node of reference r
  xtab += (size_t)r * a.nx * kXTabWords;
  yztab += (size_t)r * nyz * kYZTabWords;
  auto merged = [](float r, float q) { return pack2<F16>(r + q, fabsf(r - q)); };
  if (tid < a.nx) {
    const float* r = feat + (size_t)nref * 16;
    const float* q = feat + (size_t)tid * 16;
    uint32_t* o = xtab + tid * kXTabWords;
#pragma unroll
    for (int j = 0; j < 2 * kL; ++j) o[j] = merged(r[1 + j], q[1 + j]);
    o[12] = merged(r[0], q[0]);
    o[13] = o[14] = o[15] = 0u;
  } else if (tid < a.nx + nyz) {
    const int row = (int)(tid - a.nx), iy = row % a.ny, iz = row / a.ny;
    const float* ry = feat + (size_t)(nref + 1) * 16;
    const float* rz = feat + (size_t)(nref + 2) * 16;
    const float* qy = feat + (size_t)(a.nx + iy) * 16;
    const float* qz = feat + (size_t)(a.nx + a.ny + iz) * 16;
    uint32_t* o = yztab + (size_t)row * kYZTabWords;
#pragma unroll
    for (int i = 0; i < kL; ++i) {       // words 12 + 4i + 2(ax-1) + sc
      o[4 * i + 0] = merged(ry[1 + 2 * i], qy[1 + 2 * i]);
      o[4 * i + 1] = merged(ry[2 + 2 * i], qy[2 + 2 * i]);
      o[4 * i + 2] = merged(rz[1 + 2 * i], qz[1 + 2 * i]);
      o[4 * i + 3] = merged(rz[2 + 2 * i], qz[2 + 2 * i]);
    }
    o[24] = merged(ry[0], qy[0]);
    o[25] = merged(rz[0], qz[0]);
#pragma unroll
    for (int j = 26; j < kYZTabWords; ++j) o[j] = 0u;
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
      for (int64_t e = gtid; e < K; e += gsz) {
        store16(blob + lay.wout_off + canon_off(0, (int)e, kSboA), W[e], f16);
        // fp32 copy in rows 1-2 (output columns 1..15 of the N=16 MMA are never read):
        // k-group g's 8 weights at g*128 + 16 (query_pp_kernel's output dot product)
        *reinterpret_cast<float*>(blob + lay.wout_off + (e >> 3) * 128 + 16 + (e & 7) * 4) = W[e];
        // bf16: lo part in row 3 (the classic kernel's output MMA reads column 3)
        if (!f16)
          store16(blob + lay.wout_off + canon_off(3, (int)e, kSboA),
                  W[e] - __bfloat162float(__float2bfloat16_rn(W[e])), false);
      }
      if (gtid == 0) vecs[lay.H * kHid] = b[0];
    }
    off += (size_t)K * N + N;
  }
}

}  // namespace tc

// Launch with programmatic stream serialisation (PDL): the kernel may start while the
// previous kernel on the stream is still running; it must execute griddepcontrol.wait
// before consuming that kernel's results.
template <class... KArgs, class... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

static bool tc_supported(const ndf_model_desc& m, std::string* why) {
  auto fail = [&](const char* s) { if (why) *why = s; return false; };
  if (m.grid_levels != 0 || m.enc_layers != 0)
    return fail("tcgen05 path needs one dense latent level and no encoder MLPs");
  if (m.fourier_octaves != tc::kL || m.grid_channels != tc::kC)
    return fail("tcgen05 path needs fourier_octaves=6 and 16 latent channels");
  if (m.n_layers < 2) return fail("tcgen05 path needs >= 1 hidden layer");
  if (m.widths[0] > 128) return fail("tcgen05 path needs decoder input width <= 128");
  for (int i = 1; i < m.n_layers; ++i)
    if (m.widths[i] != tc::kHid) return fail("tcgen05 path needs hidden width 128");
  if (m.widths[m.n_layers] != 1) return fail("decoder must emit one scalar");
  const tc::Layout lay = tc::make_layout(m);
  const int a_per_wg = m.tc_format == NDF_PREC_BF16 ? 2 * tc::kABytes : tc::kABytes;
  if (((lay.blob_bytes + 1023) & ~1023) + a_per_wg + 1024 > tc::kMaxSmem)
    return fail("too many hidden layers for the SMEM-resident weights");
  return true;
}

static bool tc_schedule_classic() {
  static int classic = -1;
  if (classic < 0) {
    const char* e = getenv("NDF_TC_SCHEDULE");
    classic = (e && e[0] == 'c') ? 1 : 0;
  }
  return classic == 1;
}

// Schedule for single-reference grid queries with the sum_absdiff merge: "ws"
// (default; 4 epilogue + 2 producer warpgroups fed by per-query x / (y, z) tables)
// or "classic" (4 symmetric warpgroups doing everything; also used for points,
// multi-reference queries and the other merges).  NDF_TC_SCHEDULE=classic forces it.
// fp16 only: bf16 grid queries of this family run the split-operand query_x3_kernel.
static bool use_ws(const QueryArgs& a, int n_ref, int nwg) {
  (void)n_ref;
  return !tc_schedule_classic() && a.prec == NDF_PREC_FP16 && nwg == 4 && a.mode == 0 &&
         a.m.merge == NDF_MERGE_SUM_ABSDIFF;
}

template <bool F16, bool SILU, int KIND>
static int launch_tc_t(const tc::TcArgs& t, int nwg, size_t smem, unsigned grid, cudaStream_t s) {
  static SmemAttrCache attr;
  NDF_CUDA_CHECK(attr.ensure(tc::query_tc_kernel<F16, SILU, KIND>, smem));
  tc::query_tc_kernel<F16, SILU, KIND><<<grid, nwg * 128, smem, s>>>(t, nwg);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

// ping-pong: 2 slots x (epilogue + producer warpgroup) per CTA, one CTA per SM;
// t.n_ref references (single query or multi-reference cube)
template <bool F16, bool SILU>
static int launch_pp_t(const tc::TcArgs& t, cudaStream_t s) {
  const int64_t n = t.q.v1 - t.q.v0;
  const int64_t tiles = (n + tc::kTileM - 1) / tc::kTileM * t.n_ref;
  const unsigned g2 = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((tiles + tc::kPPSlots - 1) / tc::kPPSlots, sm_count()));
  const tc::Layout lay = tc::make_layout(t.q.m);
  const size_t smem_pp = (size_t)((lay.blob_bytes + 1023) & ~1023) +
                         (size_t)tc::kPPSlots * tc::kABytes +
                         (size_t)(1 + lay.H) * tc::kBiasBlk + 2304;
  static SmemAttrCache attr;
  NDF_CUDA_CHECK(attr.ensure(tc::query_pp_kernel<F16, SILU>, smem_pp));
  NDF_CUDA_CHECK(launch_pdl(tc::query_pp_kernel<F16, SILU>, g2, tc::kPPThreads, smem_pp, s, t));
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

template <bool F16>
static int launch_tc_variant(const tc::TcArgs& t, int nwg, size_t smem, unsigned grid, bool ws,
                             cudaStream_t s) {
  using namespace tc;
  const bool silu = t.q.m.activation == NDF_ACT_SILU;
  const int kind = t.q.mode == 1 ? kPoints : (t.n_ref > 1 ? kGridMulti : kGridSingle);
  if constexpr (F16) {
    if (ws) return silu ? launch_pp_t<true, true>(t, s) : launch_pp_t<true, false>(t, s);
  }
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

// bf16 grid query on the split-operand kernel: prep_x3_kernel (PX / PYZ layer-0 tables per
// reference, z-interpolated latent rows, reference latent channels; one launch) ->
// query_x3_kernel (programmatic dependent launch: its prologue overlaps the prep).  NDF_X3_WLO (bitmask of hidden layers, default all) selects which hidden
// layers run the A_hi x W_lo term -- a timing / accuracy experiment knob.
static int run_x3(tc::TcArgs t, const double* refs_dev, int n_ref, cudaStream_t s) {
  const QueryArgs& a = t.q;
  static int wlo = -1;
  if (wlo < 0) {
    const char* e = getenv("NDF_X3_WLO");
    wlo = e ? (int)strtol(e, nullptr, 0) : 0xff;
  }
  t.x3_wlo_mask = wlo;
  static int burst = -1;
  if (burst < 0) {
    const char* e = getenv("NDF_X3_BURST");
    burst = e ? atoi(e) : 0;
  }
  t.x3_burst = burst;
  const int ngx = (a.nx + tc::kX3TX - 1) / tc::kX3TX * (tc::kX3TX / 4);
  const tc::X3Tiles tg = tc::x3_tiles(a.nx, a.v0, a.v1);
  const int64_t ngyz64 = tg.n_vt / (tg.n_xt) * (tc::kX3TY / 4);   // this launch's row-tiles
  NDF_REQUIRE(ngyz64 < (1LL << 30), NDF_ERR_UNSUPPORTED, "too many (y, z) rows for the bf16 path");
  const int ngyz = (int)ngyz64;
  NDF_REQUIRE((int64_t)n_ref * (ngx + ngyz) + (int64_t)a.nz * a.g.ry * a.g.rx / 128 + n_ref <
                  (1LL << 31), NDF_ERR_UNSUPPORTED,
              "too many reference x table groups for one bf16 launch");
  const size_t fb = 0;
  const size_t lb = ((size_t)a.nz * a.g.ry * a.g.rx * tc::kC * 4 + 255) & ~(size_t)255;
  const size_t eb = ((size_t)n_ref * tc::kERefStride * 4 + 255) & ~(size_t)255;
  const size_t xb = (size_t)n_ref * ngx * tc::kX3Blk;
  const size_t yb = (size_t)n_ref * ngyz * tc::kX3Blk;
  void* scratch = nullptr;
  NDF_CUDA_CHECK(scratch_alloc(&scratch, fb + lb + eb + xb + yb, s));
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  float* lt = reinterpret_cast<float*>(p + fb);
  float* et = reinterpret_cast<float*>(p + fb + lb);
  uint4* px = reinterpret_cast<uint4*>(p + fb + lb + eb);
  uint4* pyz = reinterpret_cast<uint4*>(p + fb + lb + eb + xb);
  t.lz = lt;
  t.erefs = et;
  t.px = px;
  t.pyz = pyz;
  t.ngx = ngx;
  t.ngyz = ngyz;
  int st = NDF_OK;
  do {
    // one prep launch (tables, z-interpolated latent rows, reference latent channels)
    const int64_t nT = (int64_t)n_ref * ((ngx + tc::kX3TabG - 1) / tc::kX3TabG +
                                         (ngyz + tc::kX3TabG - 1) / tc::kX3TabG);
    const int64_t nL = ((int64_t)a.nz * a.g.ry * a.g.rx + 127) / 128;
    const int64_t nR = (n_ref + 127) / 128;
    tc::prep_x3_kernel<<<(unsigned)(nT + nL + nR), 128, 0, s>>>(
        a, refs_dev, n_ref, ngx, ngyz, (int64_t)tg.ty0 * tc::kX3TY, px, pyz, et, lt);
    count_launch();
    cudaError_t e = cudaGetLastError();
    const int64_t tiles = tg.n_vt * n_ref;
    const unsigned g2 = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((tiles + tc::kPPSlots - 1) / tc::kPPSlots, sm_count()));
    const size_t smem = (size_t)tc::make_x3_layout(a.m).smem_total;
    const bool silu = a.m.activation == NDF_ACT_SILU;
    // the value-range variant only when ndf_query_grid_stats asked for it
    static int f8 = -1, shared_env = -2;
    if (f8 < 0) {
      const char* ev = getenv("NDF_X3_F8");
      f8 = ev ? atoi(ev) : 0;
      const char* es = getenv("NDF_X3_SHARED");
      shared_env = es ? atoi(es) : -1;
    }
    const bool shared = shared_env >= 0 ? shared_env != 0 : n_ref == 1;
    using K = void (*)(const tc::TcArgs);
#define NDF_X3_K(SH, F)                                                                         \
  tc::query_x3_kernel<false, false, F, SH>, tc::query_x3_kernel<false, true, F, SH>,           \
      tc::query_x3_kernel<true, false, F, SH>, tc::query_x3_kernel<true, true, F, SH>
    static const K kerns[16] = {NDF_X3_K(false, false), NDF_X3_K(false, true),
                                NDF_X3_K(true, false), NDF_X3_K(true, true)};
#undef NDF_X3_K
    const int ki = (shared ? 8 : 0) + (f8 ? 4 : 0) + (silu ? 2 : 0) + (a.stats ? 1 : 0);
    auto* kern = kerns[ki];
    static SmemAttrCache attr[16];
    if (e == cudaSuccess) e = attr[ki].ensure(kern, smem);
    if (e == cudaSuccess) e = launch_pdl(kern, g2, tc::kPPThreads, smem, s, t);
    count_launch();
    if (e != cudaSuccess) {
      set_error(std::string("bf16 query launch failed: ") + cudaGetErrorString(e));
      st = NDF_ERR_CUDA;
    }
  } while (0);
  cudaFreeAsync(scratch, s);
  return st;
}

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
  const int a_per_wg = a.prec == NDF_PREC_BF16 ? 2 * tc::kABytes : tc::kABytes;
  const int nwg = std::min((tc::kMaxSmem - blob_al - 1024) / a_per_wg, 4);
  const size_t smem = (size_t)blob_al + (size_t)nwg * a_per_wg + 1024;
  const int64_t n = a.v1 - a.v0;
  const int64_t tiles = (n + tc::kTileM - 1) / tc::kTileM;
  const int64_t ctas = std::min<int64_t>((tiles + nwg - 1) / nwg, sm_count());
  const unsigned grid = (unsigned)std::max<int64_t>(ctas, 1);
  const bool ws = use_ws(a, n_ref, nwg);

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
    if (!tc_schedule_classic() && tc::x3_supported(a.m)) return run_x3(t, refs_dev, n_ref, s);
    const int threads = 128;
    if (ws) {
      NDF_REQUIRE((a.v1 - a.v0 + tc::kTileM - 1) / tc::kTileM * n_ref < (1LL << 32),
                  NDF_ERR_UNSUPPORTED, "too many reference x vertex tiles for one launch");
      // per-query tables: axis features, x words and (y, z) words per reference,
      // z-interpolated latent rows, reference latent channels
      const int64_t nyz = (int64_t)a.ny * a.nz;
      const int nnode = a.nx + a.ny + a.nz + 3 * n_ref;
      const size_t fb = (size_t)nnode * 16 * 4;
      const size_t xb = (size_t)n_ref * a.nx * tc::kXTabWords * 4;
      const size_t yb = (size_t)n_ref * nyz * tc::kYZTabWords * 4;
      const size_t lb = (size_t)a.nz * a.g.ry * a.g.rx * tc::kC * 4;
      const size_t eb = (size_t)n_ref * tc::kERefStride * 4;
      NDF_CUDA_CHECK(scratch_alloc(&scratch, fb + xb + yb + lb + eb + 256, s));
      uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
      float* feat = reinterpret_cast<float*>(p);
      uint32_t* xt = reinterpret_cast<uint32_t*>(p + fb);
      uint32_t* yt = reinterpret_cast<uint32_t*>(p + fb + xb);
      float* lt = reinterpret_cast<float*>(p + fb + xb + yb);
      float* et = reinterpret_cast<float*>(p + fb + xb + yb + lb);
      t.xtab = xt;
      t.yztab = yt;
      t.lz = lt;
      t.erefs = et;
      const int64_t n1 = (int64_t)nnode * tc::kL + n_ref + (int64_t)a.nz * a.g.ry * a.g.rx;
      tc::prep_ws_feat_kernel<<<(unsigned)((n1 + 255) / 256), 256, 0, s>>>(
          a, refs_dev, n_ref, feat, et, lt);
      NDF_LAUNCH_CHECK();
      const unsigned b2 = (unsigned)(((a.nx + nyz) * n_ref + 255) / 256);
      const float* featc = feat;
      if (a.prec == NDF_PREC_FP16)
        NDF_CUDA_CHECK(launch_pdl(tc::prep_ws_merge_kernel<true>, b2, 256, 0, s, a, n_ref, featc,
                                  xt, yt));
      else
        NDF_CUDA_CHECK(launch_pdl(tc::prep_ws_merge_kernel<false>, b2, 256, 0, s, a, n_ref, featc,
                                  xt, yt));
      NDF_LAUNCH_CHECK();
    } else {
      const int naxis = a.nx + a.ny + a.nz;
      const size_t fbytes = (size_t)naxis * tc::kAxisRow * sizeof(float);
      const size_t ebytes = (size_t)n_ref * tc::kERefStride * sizeof(float);
      NDF_CUDA_CHECK(scratch_alloc(&scratch, fbytes + ebytes + 64, s));
      t.ftab = reinterpret_cast<float*>(scratch);
      t.erefs = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(scratch) + fbytes);
      tc::prep_kernel<<<(naxis + n_ref + threads - 1) / threads, threads, 0, s>>>(
          a, refs_dev, n_ref, const_cast<float*>(t.ftab), const_cast<float*>(t.erefs));
      NDF_LAUNCH_CHECK();
    }
  }
  int st = a.prec == NDF_PREC_FP16 ? launch_tc_variant<true>(t, nwg, smem, grid, ws, s)
                                   : launch_tc_variant<false>(t, nwg, smem, grid, ws, s);
  if (scratch) cudaFreeAsync(scratch, s);
  return st;
}

int launch_query_tc(const QueryArgs& a, cudaStream_t s) { return run_tc(a, nullptr, 1, nullptr, 0, s); }

}  // namespace ndf

using namespace ndf;

// Debug only (not part of the C-ABI header): subsequent tensor-core queries record
// CTA 0's per-phase clock64() stamps into buf[6 * 32 * 12 + 16 + 32 * 8] (NULL disables;
// trace builds only, -DNDF_TRACE_BUILD).
extern "C" void ndf_debug_tc_trace(long long* buf) { ndf::g_trace = buf; }

// bf16 blobs of the BASELINE family carry the split-operand extension (X3Layout).
static size_t tc_blob_total(const ndf_model_desc& m) {
  if (tc::x3_supported(m)) {
    const tc::X3Layout xl = tc::make_x3_layout(m);
    return (size_t)xl.ext_off + (size_t)xl.ext_global;
  }
  return (size_t)tc::make_layout(m).blob_bytes;
}

extern "C" size_t ndf_tc_blob_bytes(const ndf_model_desc* m) {
  if (!m || !tc_supported(*m, nullptr)) return 0;
  return tc_blob_total(*m);
}

extern "C" int ndf_tc_pack(const ndf_model_desc* m, void* blob, size_t blob_bytes, void* stream) {
  NDF_REQUIRE(m && blob, NDF_ERR_PARAMETER, "null pointer");
  std::string why;
  NDF_REQUIRE(tc_supported(*m, &why), NDF_ERR_UNSUPPORTED, why);
  NDF_REQUIRE(blob_bytes >= tc_blob_total(*m), NDF_ERR_PARAMETER, "blob too small");
  NDF_REQUIRE((reinterpret_cast<uintptr_t>(blob) & 15) == 0, NDF_ERR_PARAMETER,
              "blob must be 16-byte aligned");
  NDF_REQUIRE(m->params_f32 != nullptr, NDF_ERR_PARAMETER, "null params_f32");
  NDF_REQUIRE(m->tc_format == NDF_PREC_BF16 || m->tc_format == NDF_PREC_FP16, NDF_ERR_PARAMETER,
              "tc_format must be NDF_PREC_BF16 or NDF_PREC_FP16");
  tc::pack_zero_kernel<<<64, 256, 0, as_stream(stream)>>>(*m, (uint8_t*)blob);
  NDF_LAUNCH_CHECK();
  tc::pack_fill_kernel<<<64, 256, 0, as_stream(stream)>>>(*m, (uint8_t*)blob);
  NDF_LAUNCH_CHECK();
  if (tc::x3_supported(*m)) {
    tc::pack_x3_kernel<<<64, 256, 0, as_stream(stream)>>>(*m, (uint8_t*)blob);
    NDF_LAUNCH_CHECK();
  }
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
  // device memory or page-locked host memory (written over PCIe); pageable refused
  void* out_dev = nullptr;
  st = resolve_output(out_f16, &out_dev);
  if (st) return st;
  QueryArgs a{};
  a.m = *m;
  a.g = make_geom(*m);
  a.mode = 0;
  a.ref_is_mu = ref_is_mu ? 1 : 0;
  a.nx = nx; a.ny = ny; a.nz = nz;
  a.v0 = v0; a.v1 = v1;
  a.prec = m->tc_format;
  return run_tc(a, refs, n_ref, reinterpret_cast<uint16_t*>(out_dev), ld_out, as_stream(stream));
}
