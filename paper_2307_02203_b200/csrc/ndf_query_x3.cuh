// bf16 grid query with split ("bf16x3") operands -- included by ndf_query_tc.cu inside
// namespace ndf::tc (it reuses that file's helpers and the ping-pong warp roles).
//
// Why: plain bf16 operands (8 significant bits) put the decoder 1.2-1.4e-2 away from the
// fp32 reference on the BASELINE model at config-1 scale -- outside the north_star's 1e-2
// contract -- and NumPy simulation (tools/bf16_sim.py) shows the error is split between
// the layer-0 inputs, the hidden activations and the weights.  This kernel removes all
// three while every MMA stays a bf16 x bf16 -> fp32 tcgen05.mma:
//
// * Layer 0 is separable on the output grid: every embedding feature except the 16
//   latent channels depends on x alone (raw x, Fourier-x) or on the (y, z) row alone
//   (raw y/z, Fourier-y/z), so its pre-activation is
//       z0 = PX[ix] + PYZ[iy, iz] + W_lat^T [r + lat, |r - lat|]
//   with PX / PYZ (bias folded into PYZ) computed per query in fp64 by
//   prep_x3_kernel from the fp32 merged features and fp32 weights, stored as
//   bf16 hi + lo pairs (16 significant bits).  A tile is 16 x-nodes x 8 (y, z)-rows,
//   so PX and PYZ enter the accumulator through two constant one-hot selector blocks
//   (A = [1 1] in the columns of the row's node, B = the tile's 16 PX / 8 PYZ rows,
//   hi and lo): 3 K16 MMA steps, and each tile's B blocks are two contiguous bulk
//   copies (8 KB + 4 KB) from the tables (LBO = 2048 B along K, SBO = 128 B along N).
//   The latent words go hi/lo as well: A_hi W_hi + A_lo W_hi + A_hi W_lo (6 steps).
// * Hidden layers: the epilogue writes each 16-column sub-chunk's activations as 8 hi
//   words + 8 lo words (h - bf16(h) is exact in fp32) into the sub-chunk's own 16
//   drained TMEM columns, and the issuer runs A_hi W_hi + A_lo W_hi + A_hi W_lo per
//   K16 step (W_lo = bf16(w - bf16(w)) resident in SMEM).  The dropped A_lo W_lo term
//   is 2^-18 relative.
// * Biases of hidden layers: hi at k = 0, lo at k = 1 of the bias MMA step.
// * Output layer: fp32 dot product in the last epilogue (fp32 weights), as before.
// Remaining error: tanh.approx in SiLU and the 2^-17 representation error -- measured
// against the fp32 oracle in tests/test_gpu_query.py (TOL_BF16 = 1e-2).
//
// Warp roles, TMEM slots and barriers are those of query_pp_kernel (see there); the
// producer now only builds the 32 latent words, issues the two bulk copies and the 9
// layer-0 MMAs; the issuer sends 3 MMAs per K16 step.

// Tile = kX3TX x-nodes x kX3TY (y, z)-rows = 128 rows (row m: x offset m % TX, row
// offset m / TX).  16 x 8: the tile's outputs are 8 runs of 16 consecutive vertices
// (64 B stores -- the field goes straight to pinned host memory over PCIe, where 8 x 16
// tiles' 32 B runs measured slower end to end), and the selectors still take 3 K16 MMAs.
constexpr int kX3TX = 16;
constexpr int kX3TY = 8;
static_assert(kX3TX * kX3TY == 128 && kX3TX % 8 == 0 && kX3TY % 8 == 0, "x3 tile shape");
constexpr int kX3Blk = 128 * 16;          // one 8-K group of a 128-row operand (2 KB)
constexpr int kX3KX = 2 * kX3TX;          // selector K for PX: (node, hi/lo)
constexpr int kX3KYZ = 2 * kX3TY;         // selector K for PYZ
constexpr int kX3SelX = (kX3KX / 8) * kX3Blk;     // A selector for PX
constexpr int kX3SelYZ = (kX3KYZ / 8) * kX3Blk;   // A selector for PYZ
constexpr int kX3Bx = (kX3KX / 8) * kX3Blk;       // per slot: B = the tile's PX rows (hi, lo)
constexpr int kX3Byz = (kX3KYZ / 8) * kX3Blk;     // per slot: B = the tile's PYZ rows
constexpr int kX3ALat = 8 * kX3Blk;       // per slot: latent A, hi words K 0-31, lo 32-63
constexpr int kX3Slot = kX3Bx + kX3Byz + kX3ALat;
constexpr int kX3Lat = 3 + 6 * kL;        // first latent feature (39)
constexpr uint32_t kBf16One2 = 0x3F803F80u;   // (1.0, 1.0) in bf16

// NDF_X3_EARLY_BIAS: the issuer initialises each hidden layer's accumulator with its bias as
// soon as the previous layer's MMAs are done, instead of with the first K-chunk
#ifndef NDF_X3_EARLY_BIAS
#define NDF_X3_EARLY_BIAS 1
#endif

// SHARED (template): all 16 epilogue warps serve the two slots in turn (see the epilogue); the
// launcher takes it for single-reference queries (c1: 0.2994 vs 0.3022 ms) and the per-slot
// warps for multi-reference cubes (c3: 41.0 vs 43.2 ms); NDF_X3_SHARED=0/1 overrides

// Extension of the packed bf16 blob, after the standard layout (make_layout):
//   wlat_hi, wlat_lo: N=128 x K=32 (k = 2c + {0: sum, 1: absdiff} of latent channel c),
//                     canonical K-major, SBO 512 B
//   wh_lo[l-1]:       lo parts of hidden layers 1..H-1, same layout as their hi parts
//   wout32:           output weights, fp32
//   (SMEM-resident part ends here: ext_bytes)
//   wh_f8[l-1]:       fp8-corrected schedule (F8): per K32 step of hidden layer l, core
//                     matrix 0 = E5M2(w) and core matrix 1 = E5M2(w - bf16(w)) for the
//                     step's 16 K values; same bytes / layout as wh_lo, which it replaces
//                     in SMEM
struct X3Layout {
  int ext_off;
  int wlat_hi, wlat_lo, wh_lo, wout32, ext_bytes;
  int wh_f8, ext_global;   // global-only region, total extension bytes
  int smem_w;      // resident weights: hidden W_hi + extension, 1024-aligned
  int smem_total;  // dynamic SMEM of query_x3_kernel
};

__host__ __device__ inline X3Layout make_x3_layout(const ndf_model_desc& m) {
  const Layout lay = make_layout(m);
  X3Layout x;
  x.ext_off = (lay.blob_bytes + 1023) & ~1023;
  x.wlat_hi = 0;
  x.wlat_lo = 128 * 32 * 2;
  x.wh_lo = 2 * 128 * 32 * 2;
  x.wout32 = x.wh_lo + (lay.H - 1) * lay.wh_bytes;
  x.ext_bytes = x.wout32 + kHid * 4;
  x.wh_f8 = (x.ext_bytes + 1023) & ~1023;
  x.ext_global = x.wh_f8 + (lay.H - 1) * lay.wh_bytes;
  x.smem_w = ((lay.H - 1) * lay.wh_bytes + x.ext_bytes + 1023) & ~1023;
  x.smem_total = x.smem_w + (lay.H + 1) * kX3Blk + kX3SelX + kX3SelYZ + kPPSlots * kX3Slot + 2304 +
                 1024;   // + the shared epilogue's 3 dot partials per slot
  return x;
}

// The split path needs the BASELINE family (sum_absdiff, E = 55, hidden width 128) and
// SMEM for hi and lo weights of every hidden layer (H <= 3).
__host__ __device__ inline bool x3_supported(const ndf_model_desc& m) {
  if (m.tc_format != NDF_PREC_BF16 || m.merge != NDF_MERGE_SUM_ABSDIFF) return false;
  if (m.widths[0] != 2 * kE || m.n_layers < 2) return false;
  return make_x3_layout(m).smem_total <= kMaxSmem;
}

// fp32 value -> (hi, lo) bf16 pair in one word (hi in the low half: k = 2j + 0)
__device__ __forceinline__ uint32_t split_f32(float v) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
  return (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(lo) << 16);
}

constexpr int kX3TabG = 4;          // 4-node groups per prep block (16 nodes share each W load)

// PX / PYZ tables, per reference r: groups of 4 nodes, [n = 0..127][node][hi, lo] bf16 (16 B per
// (group, n)) at ((r * ng + g) * 128 + n) * 16; x-groups (PX: raw x and Fourier-x features) and
// (y, z)-row groups row0 + 4 g + j, row = iy + ny * iz (PYZ: raw y, z, Fourier-y, z, plus the
// bias), only the rows of the launch's row-tiles; nodes / rows past the grid are zero.  The
// merged values are formed in fp32 exactly as the reference merge (r + q, |r - q|,
// model.py:279-286 + BASELINE) and weighted with fp32 FMAs (pre-scaled by 1/2 for SiLU):
// their ~2^-21 relative error sits far below the 2^-17 of the hi + lo pair they are stored as.
//
// The whole per-query prep of the bf16 query in ONE launch (blocks of 128 threads):
//   [0, nT)            PX / PYZ table blocks: each computes the axis features it needs (one
//                      fp64 sincos per node x octave, the operations of prep_ws_feat_kernel /
//                      embed_point_t, so the same bits), stages the merged inputs of its 16
//                      nodes, and runs the weighted sums (see below)
//   [nT, nT + nL)      lz: the query grid's latent rows interpolated along z (fp32)
//   [nT + nL, ...)     the references' latent channels in fp64 (embed_point_t's corner order)
// One launch instead of two serialized ones (round 2: prep_ws_feat_kernel -> prep_x3_tab_kernel).
__device__ __forceinline__ double clamp1(double p) { return fmin(fmax(p, -1.0), 1.0); }

__global__ void __launch_bounds__(128)
prep_x3_kernel(const QueryArgs a, const double* refs, int n_ref, int ngx, int ngyz, int64_t row0,
               uint4* px, uint4* pyz, float* eref_lat, float* lz) {
  asm volatile("griddepcontrol.launch_dependents;");
  constexpr int kN = 4 * kX3TabG;   // nodes per table block
  constexpr int kF = 26;            // features per block: 13 (x blocks) or 26 (y / z blocks)
  constexpr int kSlots = 2 * kN + 2;   // node-feature slots: x: 16 nodes + ref x; yz: 16 y,
                                       // 16 z, ref y, ref z
  __shared__ float nf[kSlots][1 + 2 * kL];
  __shared__ __align__(16) float sm[kF][kN];
  __shared__ __align__(16) float dm[kF][kN];
  const int bx = (ngx + kX3TabG - 1) / kX3TabG, byz = (ngyz + kX3TabG - 1) / kX3TabG;
  const int per_ref = bx + byz;
  const int64_t nT = (int64_t)n_ref * per_ref;
  const int64_t nlz = (int64_t)a.nz * a.g.ry * a.g.rx;
  const int64_t nL = (nlz + 127) / 128;
  const int n = threadIdx.x;
  if ((int64_t)blockIdx.x >= nT) {
    const int64_t bb = (int64_t)blockIdx.x - nT;
    if (bb < nL) {                              // ---- lz rows (query branch grid) ----
      const int64_t k = bb * 128 + n;
      if (k >= nlz) return;
      const int cx = (int)(k % a.g.rx), cy = (int)((k / a.g.rx) % a.g.ry);
      const int iz = (int)(k / ((int64_t)a.g.rx * a.g.ry));
      int z0;
      float tz;
      latent_cell(iz, a.nz, a.g.rz, z0, tz);
      const float* grid = a.ref_is_mu ? a.m.grid_nu : a.m.grid_mu;
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
      return;
    }
    const int r = (int)((bb - nL) * 128 + n);   // ---- reference latent channels ----
    if (r >= n_ref) return;
    const double* rp = refs ? refs + 3 * r : a.ref;
    const float* grid = a.ref_is_mu ? a.m.grid_mu : a.m.grid_nu;
    const double p[3] = {clamp1(rp[0]), clamp1(rp[1]), clamp1(rp[2])};
    const AxisCoord cx = level_coord(p[0], a.g.rx);
    const AxisCoord cy = level_coord(p[1], a.g.ry);
    const AxisCoord cz = level_coord(p[2], a.g.rz);
    double acc[kC];
#pragma unroll
    for (int ch = 0; ch < kC; ++ch) acc[ch] = 0.0;
    for (int c = 0; c < 8; ++c) {
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
    return;
  }
  // ---- PX / PYZ table block ----
  const int r = blockIdx.x / per_ref, b = blockIdx.x - r * per_ref;
  const bool isx = b < bx;
  const int g0 = kX3TabG * (isx ? b : b - bx);
  const int ng = isx ? ngx : ngyz;
  const int nyz = a.ny * a.nz;
  const int nslot = isx ? kN + 1 : 2 * kN + 2;
  const double* rp = refs ? refs + 3 * r : a.ref;
  for (int item = n; item < nslot * (kL + 1); item += 128) {
    const int q = item / (kL + 1), o = item - q * (kL + 1);
    double p = 0.0;
    bool ok = true;
    if (isx) {
      if (q < kN) {
        const int ix = 4 * g0 + q;
        ok = ix < a.nx;
        p = ok ? node_coord(ix, a.nx) : 0.0;
      } else {
        p = rp[0];
      }
    } else if (q < 2 * kN) {
      const int64_t row = row0 + 4 * g0 + (q % kN);
      ok = row < nyz;
      if (ok) p = q < kN ? node_coord((int)(row % a.ny), a.ny) : node_coord((int)(row / a.ny), a.nz);
    } else {
      p = rp[1 + (q - 2 * kN)];
    }
    p = clamp1(p);
    if (o == kL) {
      nf[q][0] = ok ? (float)p : 0.0f;
    } else {
      double scale = 3.141592653589793;
      for (int i = 0; i < o; ++i) scale = scale * 2.0;
      double sn, cs;
      sincos(dmul(scale, p), &sn, &cs);
      nf[q][1 + 2 * o] = ok ? (float)sn : 0.0f;
      nf[q][2 + 2 * o] = ok ? (float)cs : 0.0f;
    }
  }
  __syncthreads();
  const int nfeat = isx ? 1 + 2 * kL : 2 + 4 * kL;
  for (int k = n; k < kN * kF; k += 128) {
    const int i = k / kN, j = k - i * kN;
    float sv = 0.0f, dv = 0.0f;
    if (i < nfeat) {
      int c, rslot, qslot;
      if (isx) {                         // raw x, then sin / cos per octave
        c = i; rslot = kN; qslot = j;
      } else if (i < 2) {                // raw y, raw z
        c = 0; rslot = 2 * kN + i; qslot = i * kN + j;
      } else {
        const int jj = i - 2, o = jj >> 2, ax = 1 + ((jj >> 1) & 1), sc = jj & 1;
        c = 1 + 2 * o + sc; rslot = 2 * kN + ax - 1; qslot = (ax - 1) * kN + j;
      }
      const float rv = nf[rslot][c], qv = nf[qslot][c];
      sv = rv + qv;
      dv = fabsf(rv - qv);
    }
    sm[i][j] = sv;
    dm[i][j] = dv;
  }
  __syncthreads();
  const float* W = a.m.params_f32;                 // W0: (2E x 128) row-major, then b0
  float v[kN];
  const float v0 = isx ? 0.0f : __ldg(W + (size_t)2 * kE * kHid + n);   // bias in PYZ
#pragma unroll
  for (int j = 0; j < kN; ++j) v[j] = v0;
  float ws[kF], wd[kF];
#pragma unroll
  for (int i = 0; i < kF; ++i) {
    const int f = isx ? (i == 0 ? 0 : 3 + 6 * ((i - 1) >> 1) + ((i - 1) & 1))
                      : (i < 2 ? 1 + i : 3 + 6 * ((i - 2) >> 2) + 2 * (1 + (((i - 2) >> 1) & 1)) + ((i - 2) & 1));
    ws[i] = i < nfeat ? __ldg(W + (size_t)f * kHid + n) : 0.0f;
    wd[i] = i < nfeat ? __ldg(W + (size_t)(kE + f) * kHid + n) : 0.0f;
  }
#pragma unroll
  for (int i = 0; i < kF; ++i) {
    if (i >= nfeat) break;
#pragma unroll
    for (int j = 0; j < kN; j += 2) {
      const float2 s2 = *reinterpret_cast<const float2*>(&sm[i][j]);
      const float2 d2 = *reinterpret_cast<const float2*>(&dm[i][j]);
      ffma2(v[j], v[j + 1], ws[i], ws[i], s2.x, s2.y, v[j], v[j + 1]);
      ffma2(v[j], v[j + 1], wd[i], wd[i], d2.x, d2.y, v[j], v[j + 1]);
    }
  }
  const float hs = a.m.activation == NDF_ACT_SILU ? 0.5f : 1.0f;
#pragma unroll
  for (int gi = 0; gi < kX3TabG; ++gi) {
    const int g = g0 + gi;
    if (g >= ng) break;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool valid = isx ? 4 * g + j < a.nx : row0 + 4 * g + j < nyz;
      w[j] = valid ? split_f32(v[4 * gi + j] * hs) : 0u;
    }
    uint4* dst = isx ? px + ((size_t)r * ngx + g) * kHid : pyz + ((size_t)r * ngyz + g) * kHid;
    dst[n] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Fill the blob extension (after pack_fill_kernel has written the standard layout).
__global__ void pack_x3_kernel(const ndf_model_desc m, uint8_t* blob) {
  const Layout lay = make_layout(m);
  const X3Layout xl = make_x3_layout(m);
  uint8_t* ext = blob + xl.ext_off;
  const float hs = m.activation == NDF_ACT_SILU ? 0.5f : 1.0f;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  const float* W0 = m.params_f32;
  // latent rows of W0: k = 2c + sd  <->  W0 row sd * E + 39 + c
  for (int64_t e = gtid; e < 32 * kHid; e += gsz) {
    const int k = (int)(e / kHid), nn = (int)(e % kHid);
    const int c = k >> 1, sd = k & 1;
    const float w = hs * W0[(size_t)(sd * kE + kX3Lat + c) * kHid + nn];
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    const __nv_bfloat16 lo = __float2bfloat16_rn(w - __bfloat162float(hi));
    *reinterpret_cast<__nv_bfloat16*>(ext + xl.wlat_hi + canon_off(nn, k, 512)) = hi;
    *reinterpret_cast<__nv_bfloat16*>(ext + xl.wlat_lo + canon_off(nn, k, 512)) = lo;
  }
  size_t off = (size_t)m.widths[0] * kHid + kHid;     // past W0, b0
  for (int l = 1; l < m.n_layers; ++l) {
    const int K = m.widths[l], N = m.widths[l + 1];
    const float* W = m.params_f32 + off;
    if (l < lay.H) {
      uint8_t* dst = ext + xl.wh_lo + (l - 1) * lay.wh_bytes;
      for (int64_t e = gtid; e < (int64_t)K * N; e += gsz) {
        const int k = (int)(e / N), nn = (int)(e % N);
        const float w = hs * W[e];
        const float hi = __bfloat162float(__float2bfloat16_rn(w));
        *reinterpret_cast<__nv_bfloat16*>(dst + canon_off(nn, k, kSboA)) = __float2bfloat16_rn(w - hi);
        // F8 pair: K32 step k >> 4, core matrix 0 = E5M2(w), 1 = E5M2(w - hi), 16 B per row
        uint8_t* d8 = ext + xl.wh_f8 + (l - 1) * lay.wh_bytes +
                      ((nn >> 3) * kSboA + (k >> 4) * 256 + (nn & 7) * 16 + (k & 15));
        d8[0] = (uint8_t)(pack4_e5m2(w, 0.0f, 0.0f, 0.0f) & 0xffu);
        d8[128] = (uint8_t)(pack4_e5m2(w - hi, 0.0f, 0.0f, 0.0f) & 0xffu);
      }
    } else {
      for (int64_t e = gtid; e < K; e += gsz)
        reinterpret_cast<float*>(ext + xl.wout32)[e] = W[e];
    }
    off += (size_t)K * N + N;
  }
}

// Latent channels of node (ix, iy, iz) from the z-interpolated table lz: lerp in y, then
// in x -- the arithmetic of latent_yx_lerp's per-lane branch (same bits).
__device__ __forceinline__ void latent_yx_direct(const float* __restrict__ lz, const QueryArgs& a,
                                                 int ix, int iy, int iz, float* acc) {
  int x0, y0;
  float tx, ty;
  latent_cell(ix, a.nx, a.g.rx, x0, tx);
  latent_cell(iy, a.ny, a.g.ry, y0, ty);
  const size_t rstride = (size_t)a.g.rx * kC;
  const float* r0 = lz + ((size_t)iz * a.g.ry + y0) * rstride;
  float g0[kC];
#pragma unroll
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

// Hidden-layer epilogue of one 16-column sub-chunk, split operands: activation in fp32,
// then 8 hi words into columns [0, 8) and 8 lo words into [8, 16) of the sub-chunk.
// F8 (fp8-corrected schedule): columns [0, 8) = bf16(h) words, [8, 12) = E5M2(h - bf16(h)),
// [12, 16) = E5M2(h) -- the K32 fp8 A operand of the correction MMA.
template <bool SILU, bool F8>
__device__ __forceinline__ void epilogue16_x3(const float* x, int act, uint32_t a_taddr) {
  float h[16];
  if constexpr (SILU) {
    silu16(x, h);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = act_f32(act, x[i]);
  }
  uint32_t p[16];
#ifndef NDF_EXP_X3_NOSPLIT   // timing experiment: lo words zero (wrong results)
  if constexpr (F8) {
    float l[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      p[i] = pack2<false>(h[2 * i], h[2 * i + 1]);
      ffma2(l[2 * i], l[2 * i + 1], __uint_as_float(p[i] << 16), __uint_as_float(p[i] & 0xffff0000u),
            -1.0f, -1.0f, h[2 * i], h[2 * i + 1]);          // h - hi, exact
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      p[8 + i] = pack4_e5m2(l[4 * i], l[4 * i + 1], l[4 * i + 2], l[4 * i + 3]);
      p[12 + i] = pack4_e5m2(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) split_pair(h[2 * i], h[2 * i + 1], p[i], p[8 + i]);
  }
#else
#pragma unroll
  for (int i = 0; i < 8; ++i) { p[i] = pack2<false>(h[2 * i], h[2 * i + 1]); p[8 + i] = 0u; }
#endif
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(a_taddr),
      "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]), "r"(p[6]), "r"(p[7]),
      "r"(p[8]), "r"(p[9]), "r"(p[10]), "r"(p[11]), "r"(p[12]), "r"(p[13]), "r"(p[14]), "r"(p[15])
      : "memory");
}

// Last hidden layer, one 16-column sub-chunk: activation, then the fp32 output dot with
// contiguous fp32 weights (same accumulation order as dot16).
template <bool SILU>
__device__ __forceinline__ void dot16_x3(const float* x, int c0, int act, uint32_t w32_addr,
                                         float* dots) {
  float w[16];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(w[4 * q]), "=f"(w[4 * q + 1]), "=f"(w[4 * q + 2]), "=f"(w[4 * q + 3])
        : "r"(w32_addr + (uint32_t)(4 * c0 + 16 * q)));
  float h[16];
  if constexpr (SILU) {
    silu16(x, h);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = act_f32(act, x[i]);
  }
#pragma unroll
  for (int i = 0; i < 16; i += 2)
    ffma2(dots[i & 3], dots[(i & 3) + 1], h[i], h[i + 1], w[i], w[i + 1], dots[i & 3],
          dots[(i & 3) + 1]);
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                       uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

// Tile geometry of a launch over flat vertices [v0, v1) of an nx x ny x nz grid: tiles of
// kX3TX x-nodes x kX3TY (y, z)-rows covering rows v0 / nx .. (v1 - 1) / nx; rows and nodes
// outside the range are computed and discarded.
struct X3Tiles {
  int n_xt;          // tiles along x
  int ty0;           // first row-tile
  int64_t n_vt;      // tiles per reference
};
__host__ __device__ inline X3Tiles x3_tiles(int nx, int64_t v0, int64_t v1) {
  X3Tiles t;
  t.n_xt = (nx + kX3TX - 1) / kX3TX;
  const int64_t row_lo = v0 / nx, row_hi = (v1 - 1) / nx;
  t.ty0 = (int)(row_lo / kX3TY);
  t.n_vt = (int64_t)t.n_xt * (row_hi / kX3TY - t.ty0 + 1);
  return t;
}

// schedule trace of CTA 0 (trace builds only, tools/trace_x3.py): t.trace[(slot * 32 + tile)
// * 24 + event]; producer 0-4, epilogue lead warp 5 + 2l (layer l's MMAs done) / 6 + 2l
// (its epilogue done), issuer 12 + 4l + k2 (K-chunk k2 of layer l + 1 issued)
// per-warp stamps (trace builds): layers 0 / 1 of tiles < 32, epilogue warp ch * 4 + wq
#define NDF_X3_TRACE_W(ev)                                                              \
  do {                                                                                  \
    if (NDF_TRACE_ON(blockIdx.x == 0 && kk < 32 && l < 2 && lane == 0))                  \
      t.trace[2 * 32 * 24 + 300 + ((((s * 32 + (int)kk) * 2 + l) * 8 + ch * 4 + wq) * 8) \
              + (ev)] = clock64();                                                      \
  } while (0)
#define NDF_X3_TRACE(slot_, kk_, ev)                                                    \
  do {                                                                                  \
    if (NDF_TRACE_ON(blockIdx.x == 0 && (kk_) < 32))                                     \
      t.trace[((slot_) * 32 + (kk_)) * 24 + (ev)] = clock64();                          \
  } while (0)

// RANGE: also reduce the outputs' min / max (ndf_query_grid_stats) -- a separate
// instantiation: the three extra live registers cost the plain query 5% (measured)
// F8: fp8-corrected hidden layers (one bf16 MMA + one K32 E5M2 correction MMA per K16 step)
template <bool SILU, bool RANGE, bool F8, bool SHARED>
__global__ void __launch_bounds__(kPPThreads, 1)
query_x3_kernel(const TcArgs t) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const QueryArgs& a = t.q;
  const Layout lay = make_layout(a.m);
  const X3Layout xl = make_x3_layout(a.m);
  const int H = lay.H;
  const int whb = (H - 1) * lay.wh_bytes;
  uint8_t* wh_s = smem;                           // hidden layers' hi weights
  uint8_t* ext_s = smem + whb;                    // blob extension (W_lat hi/lo, W_lo, wout32)
  uint8_t* bias_s = smem + xl.smem_w;             // [ones][bias 1..H-1][zero], 2 KB each
  uint8_t* selx = bias_s + (H + 1) * kX3Blk;
  uint8_t* selyz = selx + kX3SelX;
  uint8_t* slots = selyz + kX3SelYZ;              // per slot: Bx | Byz | A_lat
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kPPSlots * kX3Slot);
  uint64_t* wbar = &bars[0];
  uint64_t* acc_full = &bars[1];
  uint64_t* s_free = &bars[3];
  uint64_t* d_free = &bars[5];
  uint64_t* b_full = &bars[7];                    // [kPPSlots] the tile's PX / PYZ rows landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  uint64_t* e2_done = &bars[24];                  // [slot] last-layer TMEM reads of a tile done
  float* eref_s = reinterpret_cast<float*>(bars + 16);
  float* dotx = reinterpret_cast<float*>(bars + 32);     // [2 tile parities][kPPSlots][128]

  const int tid = threadIdx.x;
  const int warp = warp_uniform(tid >> 5);
  const int lane = tid & 31;
  const int wg = warp >> 2;
  const int wq = warp & 3;
  const int wtid = tid & 127;
  // trace builds: per-CTA globaltimer at entry / exit, CTA 0's clock64 (after the tiles)
#define NDF_X3_TRACE_CTA(k)                                                              \
  do {                                                                                  \
    if (NDF_TRACE_ON(tid == 0 && blockIdx.x < 148)) {                                   \
      uint64_t gt;                                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));                            \
      t.trace[2 * 32 * 24 + 2 * blockIdx.x + (k)] = (long long)gt;                      \
      if (blockIdx.x == 0) t.trace[2 * 32 * 24 + 296 + (k)] = clock64();                \
    }                                                                                   \
  } while (0)
  NDF_X3_TRACE_CTA(0);

  if (tid == 0) {
    mbar_init(wbar, 1);
    for (int s = 0; s < kPPSlots; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&s_free[s], 1);
      mbar_init(&d_free[s], 1);
      mbar_init(&b_full[s], 1);
      mbar_init(&e2_done[s], SHARED ? 16 : 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  {
    // constant operand blocks (K-major, 16 B per row of an 8-K group):
    //   bias region: block 0 = ones (A: k = 0, 1 -> 1), block l = bias of hidden layer l
    //   (B: k = 0 -> hi, k = 1 -> lo), block H = zeros (the k = 8..15 group of every one
    //   of them, reached through LBO);
    //   selx: row m -> 1 at k = 2 (m & 7), +1;  selyz: row m -> 1 at k = 2 (m >> 3), +1
    const float* gvec = reinterpret_cast<const float*>(
        reinterpret_cast<const uint8_t*>(a.m.params_tc) + lay.vec_off);
    for (int i = tid; i < (H + 1) * 128; i += blockDim.x) {
      const int blk = i >> 7, r = i & 127;
      uint32_t w0 = 0u;
      if (blk == 0) {
        w0 = kBf16One2;
      } else if (blk < H) {
        const float b = __ldg(gvec + blk * kHid + r);
        uint32_t lo;
        split_pair(b, 0.0f, w0, lo);               // w0 = (hi(b), 0), lo = (lo(b), 0)
        w0 = (w0 & 0xffffu) | (lo << 16);          // k = 0: hi, k = 1: lo
      }
      st_shared_v4(smem_u32(bias_s + blk * kX3Blk) + r * 16, w0, 0u, 0u, 0u);
    }
    constexpr int gx = kX3KX / 8, gyz = kX3KYZ / 8;     // 8-K groups of each selector
    for (int i = tid; i < 128 * (gx + gyz); i += blockDim.x) {
      const int r = i % 128, g = i / 128;
      uint32_t w[4];
      const int hot = g < gx ? (r % kX3TX) - 4 * g : (r / kX3TX) - 4 * (g - gx);
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = (u == hot) ? kBf16One2 : 0u;
      const uint32_t addr = g < gx ? smem_u32(selx) + canon_off(r, 8 * g, gx * 128)
                                   : smem_u32(selyz) + canon_off(r, 8 * (g - gx), gyz * 128);
      st_shared_v4(addr, w[0], w[1], w[2], w[3]);
    }
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_expect_tx(wbar, (uint32_t)(whb + xl.ext_bytes));
    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.m.params_tc);
    for (int off = 0; off < whb; off += 32768)
      bulk_g2s(wh_s + off, src + lay.w0_bytes + off, (uint32_t)min(32768, whb - off), wbar);
    if constexpr (F8) {   // W_lat + (fp8 pairs in place of W_lo) + wout32
      const int nlo = (H - 1) * lay.wh_bytes;
      bulk_g2s(ext_s, src + xl.ext_off, (uint32_t)xl.wh_lo, wbar);
      for (int off = 0; off < nlo; off += 32768)
        bulk_g2s(ext_s + xl.wh_lo + off, src + xl.ext_off + xl.wh_f8 + off,
                 (uint32_t)min(32768, nlo - off), wbar);
      bulk_g2s(ext_s + xl.wout32, src + xl.ext_off + xl.wout32, (uint32_t)(xl.ext_bytes - xl.wout32),
               wbar);
    } else {
      for (int off = 0; off < xl.ext_bytes; off += 32768)
        bulk_g2s(ext_s + off, src + xl.ext_off + off, (uint32_t)min(32768, xl.ext_bytes - off), wbar);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");   // prep tables ready
  if (tid < kC) eref_s[tid] = t.erefs[tid];
  __syncthreads();
  const uint32_t tmem_base = warp_uniform(*tmem_slot);
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kHid >> 3) << 17) |
                         ((uint32_t)(kTileM >> 4) << 24);

  const int64_t n = a.v1 - a.v0;
  const X3Tiles tg = x3_tiles(a.nx, a.v0, a.v1);
  const int64_t n_tiles = tg.n_vt * t.n_ref;
  const int64_t tile_stride = (int64_t)gridDim.x * kPPSlots;
  const int s = wg < 4 ? (wg >> 1) : wg - 4;
  const int64_t first = (int64_t)blockIdx.x * kPPSlots + s;
  const int64_t cnt = first < n_tiles ? (n_tiles - first + tile_stride - 1) / tile_stride : 0;
  const uint32_t d_slot = tmem_base + (uint32_t)(s * 2 * kHid);
  const int nyz = a.ny * a.nz;
  // tile -> (reference, x tile, row tile)
  auto decode = [&](int64_t tile_g, int& r, int& tx, int& ty) {
    r = t.n_ref == 1 ? 0 : (int)((uint64_t)tile_g / (uint64_t)tg.n_vt);
    const int64_t tl = tile_g - (int64_t)r * tg.n_vt;
    ty = tg.ty0 + (int)((uint64_t)tl / (uint32_t)tg.n_xt);
    tx = (int)(tl - (int64_t)(ty - tg.ty0) * tg.n_xt);
  };

  if (wg == 6) {
    // ======================== MMA issuer of slot warp - 24 ===========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");
    const int si = warp - 24;
    if (si < kPPSlots) {
      const int64_t fi = (int64_t)blockIdx.x * kPPSlots + si;
      const int64_t ci = fi < n_tiles ? (n_tiles - fi + tile_stride - 1) / tile_stride : 0;
      const uint32_t ds = tmem_base + (uint32_t)(si * 2 * kHid);
      const uint32_t wlo_mask = (uint32_t)t.x3_wlo_mask;
      mbar_wait(wbar, 0);
#pragma unroll 1
      for (int64_t kk = 0; kk < ci; ++kk) {
#pragma unroll 1
        for (int l = 0; l + 1 < H; ++l) {
          const uint32_t half = (uint32_t)((kk * H + l) & 1);
          const uint32_t d_next = ds + (half ^ 1u) * kHid;
          const uint32_t a_tm = ds + half * kHid;                      // A of layer l+1
          const uint32_t whi = smem_u32(wh_s) + (uint32_t)(l * lay.wh_bytes);
          const uint32_t wlo = smem_u32(ext_s) + (uint32_t)(xl.wh_lo + l * lay.wh_bytes);
          const bool use_lo = (wlo_mask >> (l + 1)) & 1u;
          // x3_burst: 0 = issue K-chunk by K-chunk as the epilogue completes them,
          // 1 = the whole layer after the epilogue, 2 = pairs of K-chunks
#if NDF_X3_EARLY_BIAS
          // layer l's MMAs are done (they read A_l from the half layer l + 1 accumulates
          // into): initialise that half with the bias now, ahead of the epilogue's K-chunks
          mbar_wait(&acc_full[si], (uint32_t)((kk * H + l) & 1));
          // l == 0: the target half held the previous tile's last layer -- wait until its
          // epilogue has read it
          if (l == 0 && kk > 0) mbar_wait(&e2_done[si], (uint32_t)((kk - 1) & 1));
          tc_fence_after();
          mma_ss_warp(d_next, smem_desc(smem_u32(bias_s), (uint32_t)(H * kX3Blk), 128),
                      smem_desc(smem_u32(bias_s) + (uint32_t)((l + 1) * kX3Blk),
                                (uint32_t)((H - l - 1) * kX3Blk), 128),
                      idesc, 0u);
#endif
          if (t.x3_burst == 1)
            for (int k2 = 0; k2 < 4; ++k2) named_bar(1 + 4 * si + k2, 288);
#pragma unroll 1
          for (int k2 = 0; k2 < 4; ++k2) {
            if (t.x3_burst == 0) named_bar(1 + 4 * si + k2, 288);
            if (t.x3_burst == 2 && (k2 & 1) == 0) {
              named_bar(1 + 4 * si + k2, 288);
              named_bar(1 + 4 * si + k2 + 1, 288);
            }
            // the whole issuer warp runs this (elect.sync inside the MMA asm): operands
            // stay in uniform registers, MMAs go out back to back
            tc_fence_after();
            if (k2 == 0 && !NDF_X3_EARLY_BIAS)
              mma_ss_warp(d_next, smem_desc(smem_u32(bias_s), (uint32_t)(H * kX3Blk), 128),
                          smem_desc(smem_u32(bias_s) + (uint32_t)((l + 1) * kX3Blk),
                                    (uint32_t)((H - l - 1) * kX3Blk), 128),
                          idesc, 0u);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int ks = 2 * k2 + j;
              const uint64_t bh = smem_desc(whi + ks * 256, 128, kSboA);
              mma_ts_warp(d_next, a_tm + (uint32_t)(16 * ks), bh, idesc, 1u);
#ifndef NDF_EXP_X3_ONEMMA    // timing experiment: hi x hi only (wrong results)
              if constexpr (F8) {   // [E5M2(h_lo) | E5M2(h)] . [E5M2(w) ; E5M2(w_lo)], K32
                mma_ts_f8_warp(d_next, a_tm + (uint32_t)(16 * ks + 8),
                               smem_desc(wlo + ks * 256, 128, kSboA), idesc, 1u);
                continue;
              }
              mma_ts_warp(d_next, a_tm + (uint32_t)(16 * ks + 8), bh, idesc, 1u);
              if (use_lo) mma_ts_warp(d_next, a_tm + (uint32_t)(16 * ks),
                                      smem_desc(wlo + ks * 256, 128, kSboA), idesc, 1u);
#else
              (void)use_lo; (void)wlo;
#endif
            }
            if (k2 == 3) mma_commit_warp(&acc_full[si]);
            if (lane == 0) NDF_X3_TRACE(si, (int)kk, 12 + 4 * l + k2);
          }
        }
      }
    }
  } else if (wg >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 80;");
    // ============================ producer (slot s) ==================================
    uint8_t* slot = slots + s * kX3Slot;
    const uint32_t bx_a = smem_u32(slot), byz_a = bx_a + kX3Bx, alat_a = byz_a + kX3Byz;
    const uint32_t wlat_hi = smem_u32(ext_s) + xl.wlat_hi, wlat_lo = smem_u32(ext_s) + xl.wlat_lo;
    const int j = wtid % kX3TX, q = wtid / kX3TX;
#pragma unroll 1
    for (int64_t kk = 0; kk < cnt; ++kk) {
      int r, tx, ty;
      if (wtid == 0) NDF_X3_TRACE(s, (int)kk, 0);
      decode(first + kk * tile_stride, r, tx, ty);
      const int ix = min(kX3TX * tx + j, a.nx - 1);
      const int row = min(kX3TY * ty + q, nyz - 1);
      const int iy = row % a.ny, iz = row / a.ny;
      uint32_t pv[32];    // latent words: hi 0..15, lo 16..31
      {
        float lat[kC];
        latent_yx_direct(t.lz, a, ix, iy, iz, lat);
#pragma unroll
        for (int c4 = 0; c4 < kC / 4; ++c4) {
          const float4 r4 = t.n_ref == 1
              ? reinterpret_cast<const float4*>(eref_s)[c4]
              : __ldg(reinterpret_cast<const float4*>(t.erefs + (size_t)r * kERefStride) + c4);
          const float rv[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = 4 * c4 + u;
            split_pair(rv[u] + lat[c], fabsf(rv[u] - lat[c]), pv[c], pv[16 + c]);
          }
        }
      }
      if (wtid == 0) NDF_X3_TRACE(s, (int)kk, 1);
      if (kk >= 1) mbar_wait(&s_free[s], (uint32_t)((kk - 1) & 1));   // previous layer 0 done
      if (wtid == 0) {
        NDF_X3_TRACE(s, (int)kk, 2);
        mbar_expect_tx(&b_full[s], (uint32_t)(kX3Bx + kX3Byz));
        bulk_g2s(slot, reinterpret_cast<const uint8_t*>(t.px) +
                           ((size_t)r * t.ngx + (kX3TX / 4) * tx) * (size_t)kX3Blk, kX3Bx,
                 &b_full[s]);
        bulk_g2s(slot + kX3Bx, reinterpret_cast<const uint8_t*>(t.pyz) +
                                   ((size_t)r * t.ngyz + (kX3TY / 4) * (ty - tg.ty0)) *
                                       (size_t)kX3Blk,
                 kX3Byz, &b_full[s]);
      }
#pragma unroll
      for (int g = 0; g < 8; ++g)
        st_shared_v4(alat_a + canon_off(wtid, 8 * g, 1024), pv[4 * g], pv[4 * g + 1],
                     pv[4 * g + 2], pv[4 * g + 3]);
      fence_proxy_async();
      named_bar(11 + s, 128);
      if (wq == 0) {                 // the producer's first warp issues layer 0 (elect.sync)
        if (kk == 0) mbar_wait(wbar, 0);
        else mbar_wait(&d_free[s], (uint32_t)((kk - 1) & 1));   // target D half drained
        if (lane == 0) NDF_X3_TRACE(s, (int)kk, 3);
        mbar_wait(&b_full[s], (uint32_t)(kk & 1));
        tc_fence_after();
        const uint32_t d0 = d_slot + (uint32_t)((kk * H) & 1) * kHid;
#pragma unroll
        for (int st = 0; st < kX3KX / 16; ++st)       // PX rows of the tile's x-nodes
          mma_ss_warp(d0, smem_desc(smem_u32(selx) + st * 256, 128, (kX3KX / 8) * 128),
                      smem_desc(bx_a + st * 4096, 2048, 128), idesc, st ? 1u : 0u);
#pragma unroll
        for (int st = 0; st < kX3KYZ / 16; ++st)      // PYZ rows of the tile's (y, z)-rows
          mma_ss_warp(d0, smem_desc(smem_u32(selyz) + st * 256, 128, (kX3KYZ / 8) * 128),
                      smem_desc(byz_a + st * 4096, 2048, 128), idesc, 1u);
#pragma unroll
        for (int st = 0; st < 2; ++st) {
          const uint64_t bh = smem_desc(wlat_hi + st * 256, 128, 512);
          mma_ss_warp(d0, smem_desc(alat_a + st * 256, 128, 1024), bh, idesc, 1u);         // hi x hi
          mma_ss_warp(d0, smem_desc(alat_a + (2 + st) * 256, 128, 1024), bh, idesc, 1u);   // lo x hi
          mma_ss_warp(d0, smem_desc(alat_a + st * 256, 128, 1024),
                      smem_desc(wlat_lo + st * 256, 128, 512), idesc, 1u);                 // hi x lo
        }
        mma_commit_warp(&acc_full[s]);
        if (lane == 0) NDF_X3_TRACE(s, (int)kk, 4);
      }
    }
  } else {
    if constexpr (SHARED) {
    // ============ epilogue: all 16 warps serve slot 0 and slot 1 in turn =============
    // Warp (j, wq): TMEM lane quarter wq, columns 64 it + 16 j (it = 0, 1) of every layer,
    // so K-chunk k2 = columns [32 k2, 32 k2 + 32) is finished by warps j = 2 (k2 & 1) + {0, 1}
    // at item k2 >> 1.  The slots' epilogues alternate (slot 0 layer l, slot 1 layer l,
    // slot 0 layer l + 1, ...): each runs on the whole SM's MUFU while the other slot's
    // layer MMAs run on the tensor pipe.
    asm volatile("setmaxnreg.inc.sync.aligned.u32 80;");
    const int j = wg;                                 // 0..3
    const bool lead = j == 0 && wq == 0;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    mbar_wait(wbar, 0);
    const float bias_out = __ldg(reinterpret_cast<const float*>(
        reinterpret_cast<const uint8_t*>(a.m.params_tc) + lay.vec_off) + H * kHid);
    const uint32_t w32_addr = smem_u32(ext_s) + xl.wout32;
    uint32_t acc_ph[kPPSlots] = {0u, 0u};
    int64_t cnt_s[kPPSlots];
#pragma unroll
    for (int q = 0; q < kPPSlots; ++q) {
      const int64_t f = (int64_t)blockIdx.x * kPPSlots + q;
      cnt_s[q] = f < n_tiles ? (n_tiles - f + tile_stride - 1) / tile_stride : 0;
    }
    float z_pend[kPPSlots] = {0.0f, 0.0f};
    int64_t kk_pend[kPPSlots] = {-1, -1};
    RangeAcc rng;                                   // ndf_query_grid_stats only
    auto flush = [&](int q) {
      if (kk_pend[q] < 0) return;
      int r, tx, ty;
      decode((int64_t)blockIdx.x * kPPSlots + q + kk_pend[q] * tile_stride, r, tx, ty);
      const int ix = kX3TX * tx + (wtid % kX3TX);
      const int row = kX3TY * ty + (wtid / kX3TX);
      const int64_t v = (int64_t)ix + (int64_t)a.nx * row;
      if (ix < a.nx && row < nyz && v >= a.v0 && v < a.v1) {
        const float o = head_exact(a.m.head, z_pend[q]);
        if (t.out16) {
          const __half ho = __float2half_rn(o);
          t.out16[(int64_t)r * t.ld_out + (v - a.v0)] = *reinterpret_cast<const uint16_t*>(&ho);
        } else {
          a.out[v - a.v0] = o;
          if constexpr (RANGE) rng.add(o);
        }
      }
      kk_pend[q] = -1;
    };
#pragma unroll 1
    for (int64_t kk = 0; kk < cnt_s[0]; ++kk) {
#pragma unroll 1
      for (int l = 0; l < H; ++l) {
#pragma unroll
        for (int q = 0; q < kPPSlots; ++q) {
          if (kk >= cnt_s[q]) continue;
          const uint32_t half = (uint32_t)((kk * H + l) & 1);
          const uint32_t d_base = tmem_base + (uint32_t)(q * 2 * kHid) + lane_base + half * kHid;
          mbar_wait(&acc_full[q], acc_ph[q]);
          acc_ph[q] ^= 1u;
          tc_fence_after();
          if (l == 0 && lead && lane == 0) mbar_arrive(&s_free[q]);   // slot SMEM reusable
          if (lead && lane == 0) NDF_X3_TRACE(q, (int)kk, 5 + 2 * l);
          float va[16], vb[16];
          tmem_ld16_nowait(d_base + 16u * (uint32_t)j, va);
          tmem_ld16_nowait(d_base + 64u + 16u * (uint32_t)j, vb);
          tmem_wait_ld();
          if (l + 1 < H) {
            epilogue16_x3<SILU, F8>(va, a.m.activation, d_base + 16u * (uint32_t)j);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            named_bar_arrive(1 + 4 * q + (j >> 1), 288);
            epilogue16_x3<SILU, F8>(vb, a.m.activation, d_base + 64u + 16u * (uint32_t)j);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            named_bar_arrive(1 + 4 * q + 2 + (j >> 1), 288);
            if (lead && lane == 0) NDF_X3_TRACE(q, (int)kk, 6 + 2 * l);
            if (l == 0 && j == 0) flush(q);
          } else {
            if (lead && lane == 0) mbar_arrive(&d_free[q]);
            tc_fence_before();
            if (lane == 0) mbar_arrive(&e2_done[q]);       // this warp's TMEM reads are done
            float dots[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            dot16_x3<SILU>(va, 16 * j, a.m.activation, w32_addr, dots);
            dot16_x3<SILU>(vb, 64 + 16 * j, a.m.activation, w32_addr, dots);
            tc_fence_before();
            const float part = (dots[0] + dots[1]) + (dots[2] + dots[3]);
            float* dx = dotx + q * 3 * kTileM;
            if (j > 0) {
              dx[(j - 1) * kTileM + wtid] = part;
              named_bar_arrive(9 + q, 512);
            } else {
              named_bar(9 + q, 512);
              z_pend[q] = ((part + dx[wtid]) + (dx[kTileM + wtid] + dx[2 * kTileM + wtid])) + bias_out;
              kk_pend[q] = kk;
              if (H == 1) flush(q);
            }
            if (lead && lane == 0) NDF_X3_TRACE(q, (int)kk, 6 + 2 * l);
          }
        }
      }
    }
    if (j == 0) {
      flush(0);
      flush(1);
    }
    if constexpr (RANGE) {
      if (j == 0) rng.flush(a.stats);
    }
    (void)rng;
    (void)n;
    (void)cnt;
    (void)first;
    (void)d_slot;
    } else {
    // ======================== epilogue (slot s, column half ch) ======================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 80;");
    const int ch = wg & 1;
    const bool lead = ch == 0 && wq == 0;
    const uint32_t first_col = 16u * (uint32_t)ch;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    mbar_wait(wbar, 0);
    const float bias_out = __ldg(reinterpret_cast<const float*>(
        reinterpret_cast<const uint8_t*>(a.m.params_tc) + lay.vec_off) + H * kHid);
    const uint32_t w32_addr = smem_u32(ext_s) + xl.wout32;
    uint32_t acc_ph = 0u;
    // Output of a finished tile, written late: the column-0 warps keep the row's pre-head
    // value and store it after the next tile's first epilogue (where they would otherwise
    // wait on the layer-1 MMAs), so decode / head / store stay off the critical chain.
    float z_pend = 0.0f;
    int64_t kk_pend = -1;
    RangeAcc rng;                                   // ndf_query_grid_stats only
    auto flush = [&]() {
      if (kk_pend < 0) return;
      int r, tx, ty;
      decode(first + kk_pend * tile_stride, r, tx, ty);
      const int ix = kX3TX * tx + (wtid % kX3TX);
      const int row = kX3TY * ty + (wtid / kX3TX);
      const int64_t v = (int64_t)ix + (int64_t)a.nx * row;
      if (ix < a.nx && row < nyz && v >= a.v0 && v < a.v1) {
        const float o = head_exact(a.m.head, z_pend);
        if (t.out16) {
          const __half ho = __float2half_rn(o);
          t.out16[(int64_t)r * t.ld_out + (v - a.v0)] = *reinterpret_cast<const uint16_t*>(&ho);
        } else {
          a.out[v - a.v0] = o;
          if constexpr (RANGE) rng.add(o);
        }
      }
      kk_pend = -1;
    };
#pragma unroll 1
    for (int64_t kk = 0; kk < cnt; ++kk) {
#pragma unroll 1
      for (int l = 0; l < H; ++l) {
        const uint32_t half = (uint32_t)((kk * H + l) & 1);
        const uint32_t d_base = d_slot + lane_base + half * kHid;
        mbar_wait(&acc_full[s], acc_ph);
        acc_ph ^= 1u;
        tc_fence_after();
        if (l == 0 && lead && lane == 0) mbar_arrive(&s_free[s]);   // slot SMEM reusable
        if (lead && lane == 0) NDF_X3_TRACE(s, (int)kk, 5 + 2 * l);
        NDF_X3_TRACE_W(0);
        float va[16], vb[16];
        tmem_ld16_nowait(d_base + first_col, va);
        tmem_wait_ld();
        NDF_X3_TRACE_W(1);
        if (l + 1 < H) {
#ifdef NDF_EXP_X3_NOEPI      // timing experiment: hidden epilogues only signal (wrong results)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            tc_fence_before();
            named_bar_arrive(1 + 4 * s + i, 288);
          }
          (void)vb;
#else
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t col = first_col + 32u * (uint32_t)i;
            float* cur = (i & 1) ? vb : va;
            float* nxt = (i & 1) ? va : vb;
            if (i + 1 < 4) tmem_ld16_nowait(d_base + col + 32u, nxt);
            epilogue16_x3<SILU, F8>(cur, a.m.activation, d_base + col);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            named_bar_arrive(1 + 4 * s + i, 288);
            NDF_X3_TRACE_W(2 + i);
            if (i + 1 < 4) tmem_wait_ld();
          }
#endif
          if (lead && lane == 0) NDF_X3_TRACE(s, (int)kk, 6 + 2 * l);
          if (l == 0) flush();
        } else {
          if (lead && lane == 0) mbar_arrive(&d_free[s]);
          // the shared epilogue's partials (column groups j = 2 ch, 2 ch + 1: columns 16 j and
          // 64 + 16 j, in that order) and its summation ((p0 + p1) + (p2 + p3)) + bias, so a
          // multi-reference cube row equals the single query bit for bit
          float dA[4] = {0.0f, 0.0f, 0.0f, 0.0f}, dB[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          const uint32_t cA = 32u * (uint32_t)ch, cB = cA + 16u;
          tmem_ld16_nowait(d_base + cA, va);
          tmem_ld16_nowait(d_base + cB, vb);
          tmem_wait_ld();
          dot16_x3<SILU>(va, (int)cA, a.m.activation, w32_addr, dA);
          dot16_x3<SILU>(vb, (int)cB, a.m.activation, w32_addr, dB);
          tmem_ld16_nowait(d_base + 64u + cA, va);
          tmem_ld16_nowait(d_base + 64u + cB, vb);
          tmem_wait_ld();
          tc_fence_before();
          if (lane == 0) mbar_arrive(&e2_done[s]);          // this warp's TMEM reads are done
          dot16_x3<SILU>(va, 64 + (int)cA, a.m.activation, w32_addr, dA);
          dot16_x3<SILU>(vb, 64 + (int)cB, a.m.activation, w32_addr, dB);
          const float part = ((dA[0] + dA[1]) + (dA[2] + dA[3])) + ((dB[0] + dB[1]) + (dB[2] + dB[3]));
          float* dx = dotx + ((kk & 1) * kPPSlots + s) * kTileM;
          if (wq == 0 && lane == 0) NDF_X3_TRACE(s, (int)kk, 20 + ch);
          if (ch == 1) {
            // dotx is double-buffered by tile parity: the column-1 warps run ahead into the
            // next tile (they cannot pass its hidden epilogues without the column-0 warps,
            // which read this buffer first)
            dx[wtid] = part;
            named_bar_arrive(9 + s, 256);
          } else {
            named_bar(9 + s, 256);
            z_pend = part + dx[wtid] + bias_out;
            kk_pend = kk;
            if (H == 1) flush();       // no later hidden epilogue to hide it behind
          }
          if (lead && lane == 0) NDF_X3_TRACE(s, (int)kk, 22);
          if (lead && lane == 0) NDF_X3_TRACE(s, (int)kk, 6 + 2 * l);
        }
      }
    }
    flush();
    if constexpr (RANGE) {
      if (ch == 0) rng.flush(a.stats);
    }
    (void)rng;
    (void)n;
    }
  }
  tc_fence_before();
  __syncthreads();
  NDF_X3_TRACE_CTA(1);
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
}
