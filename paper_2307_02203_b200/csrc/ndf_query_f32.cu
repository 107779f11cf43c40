// Exact fp32 NDF query (SIMT): embed -> [encoder MLP] -> merge -> decoder -> head.
//
// Every matmul restates matmul_exact (nn.py:18-20): z_j = sum_k h_k w_kj
// accumulated sequentially in ascending k with separately rounded multiply and
// add (no FMA contraction), bias added afterwards (nn.py:135) -- bit-identical
// to the reference's einsum.  Hidden activations / heads use libdevice fp32
// transcendentals (<= 2 ulp from NumPy's), so outputs agree to ~1e-7.
//
// Covers both latent-grid kinds (dense anisotropic level, reference HashGrid)
// and the reference's per-branch encoder MLPs (model.py:179-189), i.e. the
// reference default architecture as well as BASELINE config 0.
// Tile: 128 threads, 32 query vertices; activations staged k-major in SMEM so
// each k step reads the tile's 32 activations as 8 broadcast LDS.128.
#include <algorithm>

#include "ndf_query.cuh"

namespace ndf {

constexpr int kTV = 32;               // vertices per tile
constexpr int kTVP = kTV + 4;         // padded k-row stride (floats)
constexpr int kThreadsF32 = 128;

// Rows a tile buffer must hold for this model: the widest of the embedding, the
// encoder layers, the merged decoder input and the decoder layers.  SMEM is sized from
// it, so narrow models (the reference default: <= 51 rows) fit 4-6 CTAs per SM.
__host__ __device__ __forceinline__ int f32_buf_rows(const ndf_model_desc& m, int E) {
  int r = E;
  for (int i = 0; i <= m.enc_layers && m.enc_layers > 0; ++i) r = r > m.enc_widths[i] ? r : m.enc_widths[i];
  for (int i = 0; i < m.n_layers; ++i) r = r > m.widths[i] ? r : m.widths[i];
  return (r + 3) & ~3;
}

__device__ __forceinline__ int enc_out_dim(const ndf_model_desc& m, int E) {
  return m.enc_layers > 0 ? m.enc_widths[m.enc_layers] : E;
}

// One dense layer over the tile: Hout[j][v] = act(sum_k Hin[k][v] W[k][j] + b[j]) for
// j < N (sequential ascending k, unfused fp32 -- matmul_exact); `act` false = linear.
// Narrow layers split the tile's vertices across thread groups (VPT vertices per
// thread) so all 128 threads work; every output keeps the same arithmetic order.
template <int VPT>
__device__ __forceinline__ void tile_layer_v(const float* Hin, float* Hout, const float* W,
                                             const float* b, int K, int N, bool act, int kind) {
  constexpr int kGroups = kTV / VPT;
  constexpr int kJT = kThreadsF32 / kGroups;      // threads per vertex group
  const int grp = threadIdx.x / kJT;
  const int v0 = grp * VPT;
  for (int j = threadIdx.x % kJT; j < N; j += kJT) {
    float acc[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) acc[v] = 0.0f;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {          // unrolled: several weight loads in flight
      const float w = __ldg(W + (size_t)k * N + j);
      const float4* hr = reinterpret_cast<const float4*>(Hin + k * kTVP + v0);
#pragma unroll
      for (int q = 0; q < VPT / 4; ++q) {
        const float4 h = hr[q];
        acc[4 * q + 0] = fadd(acc[4 * q + 0], fmul(h.x, w));
        acc[4 * q + 1] = fadd(acc[4 * q + 1], fmul(h.y, w));
        acc[4 * q + 2] = fadd(acc[4 * q + 2], fmul(h.z, w));
        acc[4 * q + 3] = fadd(acc[4 * q + 3], fmul(h.w, w));
      }
    }
    const float bj = __ldg(b + j);
    float4* ho = reinterpret_cast<float4*>(Hout + j * kTVP + v0);
#pragma unroll
    for (int q = 0; q < VPT / 4; ++q) {
      float o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float z = fadd(acc[4 * q + u], bj);
        o[u] = act ? act_exact(kind, z) : z;
      }
      ho[q] = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void tile_layer(const float* Hin, float* Hout, const float* W,
                                           const float* b, int K, int N, bool act, int kind) {
  if (N <= kThreadsF32 / 4) tile_layer_v<kTV / 4>(Hin, Hout, W, b, K, N, act, kind);
  else if (N <= kThreadsF32 / 2) tile_layer_v<kTV / 2>(Hin, Hout, W, b, K, N, act, kind);
  else tile_layer_v<kTV>(Hin, Hout, W, b, K, N, act, kind);
}

// Encoder MLP over the tile (Mlp.forward, nn.py:124-137): activation on all layers
// but the last.  Input in *bufs[0]; returns the buffer holding the output.
__device__ __forceinline__ float* tile_encoder(const ndf_model_desc& m, const float* P,
                                               float* in, float* other) {
  size_t off = 0;
  float* hin = in;
  float* hout = other;
  for (int l = 0; l < m.enc_layers; ++l) {
    const int K = m.enc_widths[l], N = m.enc_widths[l + 1];
    const float* W = P + off;
    const float* b = W + (size_t)K * N;
    off += (size_t)K * N + N;
    tile_layer(hin, hout, W, b, K, N, l + 1 < m.enc_layers, m.activation);
    float* t = hin; hin = hout; hout = t;
  }
  return hin;
}

// Encoder MLP of ONE vector (the reference point): threads j < N, ping-pong in SMEM.
__device__ __forceinline__ float* vec_encoder(const ndf_model_desc& m, const float* P, float* x,
                                              float* y) {
  size_t off = 0;
  for (int l = 0; l < m.enc_layers; ++l) {
    const int K = m.enc_widths[l], N = m.enc_widths[l + 1];
    const float* W = P + off;
    const float* b = W + (size_t)K * N;
    off += (size_t)K * N + N;
    for (int j = threadIdx.x; j < N; j += kThreadsF32) {
      float acc = 0.0f;
      for (int k = 0; k < K; ++k) acc = fadd(acc, fmul(x[k], __ldg(W + (size_t)k * N + j)));
      const float z = fadd(acc, __ldg(b + j));
      y[j] = l + 1 < m.enc_layers ? act_exact(m.activation, z) : z;
    }
    __syncthreads();
    float* t = x; x = y; y = t;
  }
  return x;
}

// merge (model.py:279-286 + sum_absdiff) of branch values a (mu) and b (nu) into row
// i (and C + i for the two-block merges) of the decoder input
__device__ __forceinline__ void merge_store(int mode, int C, int i, int v, float av, float bv,
                                            float* D) {
  switch (mode) {
    case NDF_MERGE_MULTIPLY: D[i * kTVP + v] = fmul(av, bv); break;
    case NDF_MERGE_CONCAT: D[i * kTVP + v] = av; D[(C + i) * kTVP + v] = bv; break;
    case NDF_MERGE_ADD: D[i * kTVP + v] = fadd(av, bv); break;
    case NDF_MERGE_ABSDIFF: D[i * kTVP + v] = fabsf(__fsub_rn(av, bv)); break;
    default:
      D[i * kTVP + v] = fadd(av, bv);
      D[(C + i) * kTVP + v] = fabsf(__fsub_rn(av, bv));
      break;
  }
}

// SMEM: B0, B1 [rows][kTVP] (+ B2 for points mode: the mu branch; rows = f32_buf_rows),
// then two NDF_MAX_WIDTH vectors for the reference's embedding / encoding.
__global__ void __launch_bounds__(kThreadsF32)
query_f32_kernel(const QueryArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int buf_floats = f32_buf_rows(a.m, a.g.E) * kTVP;
  float* B0 = smem;
  float* B1 = B0 + buf_floats;
  float* B2 = B1 + buf_floats;                 // points mode only
  float* rv0 = a.mode == 1 ? B2 + buf_floats : B2;
  float* rv1 = rv0 + NDF_MAX_WIDTH;

  const int tid = threadIdx.x;
  const EmbedGeom& g = a.g;
  const int E = g.E;
  const int Cenc = enc_out_dim(a.m, E);
  const int64_t n_vert = a.v1 - a.v0;
  const float* P = a.m.params_f32;
  const float* enc_ref = a.ref_is_mu ? a.m.enc_mu : a.m.enc_nu;
  const float* enc_q = a.ref_is_mu ? a.m.enc_nu : a.m.enc_mu;

  // ---- reference branch (grid mode): embedded and encoded once per CTA ----------
  float* eref = rv0;
  if (a.mode == 0) {
    if (tid == 0) {
      const float* grid = a.ref_is_mu ? a.m.grid_mu : a.m.grid_nu;
      embed_point(g, grid, a.ref[0], a.ref[1], a.ref[2], [&](int i, float v) { rv0[i] = v; });
    }
    __syncthreads();
    if (a.m.enc_layers > 0) eref = vec_encoder(a.m, enc_ref, rv0, rv1);
  }

  RangeAcc rng;                                // ndf_query_grid_stats only
  for (int64_t tile = blockIdx.x; tile * kTV < n_vert; tile += gridDim.x) {
    const int64_t base = a.v0 + tile * kTV;
    const int nv = (int)min((int64_t)kTV, a.v1 - base);
    // ---- embed: 4 threads per vertex (Fourier | latent levels), k-major column v --
    {
      const int v = tid % kTV, part = tid / kTV;
      if (v < nv) {
        const int64_t gv = base + v;
        if (a.mode == 0) {
          double p[3];
          vertex_position(a, gv, p);
          const float* grid = a.ref_is_mu ? a.m.grid_nu : a.m.grid_mu;
          embed_point(g, grid, p[0], p[1], p[2], [&](int i, float x) { B0[i * kTVP + v] = x; },
                      part, kThreadsF32 / kTV);
        } else {
          const int64_t im = a.n_mu == 1 ? 0 : gv;
          embed_point(g, a.m.grid_mu, a.p_mu[3 * im], a.p_mu[3 * im + 1], a.p_mu[3 * im + 2],
                      [&](int i, float x) { B2[i * kTVP + v] = x; }, part, kThreadsF32 / kTV);
          embed_point(g, a.m.grid_nu, a.p_nu[3 * gv], a.p_nu[3 * gv + 1], a.p_nu[3 * gv + 2],
                      [&](int i, float x) { B0[i * kTVP + v] = x; }, part, kThreadsF32 / kTV);
        }
      } else if (part == 0) {
        for (int i = 0; i < E; ++i) {
          B0[i * kTVP + v] = 0.0f;
          if (a.mode == 1) B2[i * kTVP + v] = 0.0f;
        }
      }
    }
    __syncthreads();
    // ---- encoders (query branch; points mode: both branches) ---------------------
    float* q = B0;              // query / nu branch values, Cenc rows
    float* mu = B2;             // points mode: mu branch values
    float* free_buf = B1;
    if (a.m.enc_layers > 0) {
      q = tile_encoder(a.m, a.mode == 0 ? enc_q : a.m.enc_nu, B0, B1);
      free_buf = q == B0 ? B1 : B0;
      if (a.mode == 1) {
        mu = tile_encoder(a.m, a.m.enc_mu, B2, free_buf);
        if (mu != B2) {           // result landed in free_buf: B2 is free now
          float* t = free_buf; free_buf = B2; (void)t;
        }
      }
    }
    // ---- merge into the decoder input -----------------------------------------------
    float* D = free_buf;
    for (int e = tid; e < Cenc * kTV; e += kThreadsF32) {
      const int i = e / kTV, v = e % kTV;
      float av, bv;
      if (a.mode == 0) {
        const float r = eref[i], x = q[i * kTVP + v];
        av = a.ref_is_mu ? r : x;
        bv = a.ref_is_mu ? x : r;
      } else {
        av = mu[i * kTVP + v];
        bv = q[i * kTVP + v];
      }
      merge_store(a.m.merge, Cenc, i, v, av, bv, D);
    }
    __syncthreads();
    // ---- decoder ------------------------------------------------------------------
    float* Hin = D;
    float* Hout = D == B0 ? B1 : B0;
    size_t off = 0;
    const int L = a.m.n_layers;
    for (int l = 0; l < L; ++l) {
      const int K = a.m.widths[l];
      const int N = a.m.widths[l + 1];
      const float* W = P + off;
      const float* b = W + (size_t)K * N;
      off += (size_t)K * N + N;
      if (l == L - 1) {
        // output layer (N == 1): one thread per vertex
        if (tid < nv) {
          float acc = 0.0f;
          for (int k = 0; k < K; ++k) acc = fadd(acc, fmul(Hin[k * kTVP + tid], __ldg(W + k)));
          const float z = fadd(acc, __ldg(b));
          const float o = head_exact(a.m.head, z);
          a.out[base - a.v0 + tid] = o;
          if (a.stats) rng.add(o);
        }
        __syncthreads();
      } else {
        tile_layer(Hin, Hout, W, b, K, N, true, a.m.activation);
        float* t = Hin; Hin = Hout; Hout = t;
      }
    }
  }
  if (a.stats) rng.flush(a.stats);
}

size_t query_f32_smem_bytes(int mode, int rows = NDF_MAX_WIDTH) {
  return sizeof(float) * ((mode == 1 ? 3 : 2) * (size_t)rows * kTVP + 2 * NDF_MAX_WIDTH);
}

int validate_model(const ndf_model_desc* m) {
  NDF_REQUIRE(m != nullptr, NDF_ERR_PARAMETER, "null model descriptor");
  NDF_REQUIRE(m->fourier_octaves >= 0 && m->fourier_octaves <= 12, NDF_ERR_UNSUPPORTED,
              "fourier_octaves must be in [0, 12]");
  NDF_REQUIRE(m->grid_levels >= 0 && m->grid_levels <= NDF_MAX_LEVELS, NDF_ERR_UNSUPPORTED,
              "grid_levels must be in [0, 16]");
  const int nlev = m->grid_levels > 0 ? m->grid_levels : 1;
  NDF_REQUIRE(m->grid_channels >= 1 && nlev * m->grid_channels <= 64, NDF_ERR_UNSUPPORTED,
              "latent features (levels x channels) must be in [1, 64]");
  if (m->grid_levels == 0) {
    for (int i = 0; i < 3; ++i)
      NDF_REQUIRE(m->grid_res[i] >= 2, NDF_ERR_CONFIG, "latent resolution must be >= 2 per axis");
  } else {
    NDF_REQUIRE(m->grid_log2_table >= 1 && m->grid_log2_table < 31, NDF_ERR_CONFIG,
                "log2 table size must be in [1, 31)");
    for (int l = 0; l < m->grid_levels; ++l)
      NDF_REQUIRE(m->grid_level_res[l] >= 2, NDF_ERR_CONFIG, "level resolution must be >= 2");
  }
  const int E = 3 + 6 * m->fourier_octaves + nlev * m->grid_channels;
  NDF_REQUIRE(m->enc_layers >= 0 && m->enc_layers <= NDF_MAX_LAYERS, NDF_ERR_UNSUPPORTED,
              "encoder layer count out of range");
  int Cenc = E;
  if (m->enc_layers > 0) {
    NDF_REQUIRE(m->enc_widths[0] == E, NDF_ERR_SHAPE, "encoder input width != embedding width");
    for (int i = 0; i <= m->enc_layers; ++i)
      NDF_REQUIRE(m->enc_widths[i] >= 1 && m->enc_widths[i] <= NDF_MAX_WIDTH, NDF_ERR_UNSUPPORTED,
                  "encoder width out of range (1..256)");
    NDF_REQUIRE(m->enc_mu && m->enc_nu, NDF_ERR_PARAMETER, "null encoder parameters");
    Cenc = m->enc_widths[m->enc_layers];
  }
  NDF_REQUIRE(m->n_layers >= 1 && m->n_layers <= NDF_MAX_LAYERS, NDF_ERR_UNSUPPORTED,
              "decoder layer count out of range");
  const int din = (m->merge == NDF_MERGE_SUM_ABSDIFF || m->merge == NDF_MERGE_CONCAT) ? 2 * Cenc : Cenc;
  NDF_REQUIRE(m->widths[0] == din, NDF_ERR_SHAPE, "decoder input width does not match merge");
  NDF_REQUIRE(m->widths[m->n_layers] == 1, NDF_ERR_CONFIG, "decoder must emit one scalar");
  for (int i = 0; i <= m->n_layers; ++i)
    NDF_REQUIRE(m->widths[i] >= 1 && m->widths[i] <= NDF_MAX_WIDTH, NDF_ERR_UNSUPPORTED,
                "decoder width out of range (1..256)");
  NDF_REQUIRE(m->merge >= 0 && m->merge <= 4, NDF_ERR_CONFIG, "unknown merge mode");
  NDF_REQUIRE(m->activation >= 0 && m->activation <= 3, NDF_ERR_PARAMETER, "unknown activation");
  NDF_REQUIRE(m->head >= 0 && m->head <= 2, NDF_ERR_PARAMETER, "unknown head");
  NDF_REQUIRE(m->grid_mu && m->grid_nu && m->params_f32, NDF_ERR_PARAMETER,
              "null device pointer in model descriptor");
  return NDF_OK;
}

int launch_query_f32(const QueryArgs& a, cudaStream_t s) {
  static SmemAttrCache attr;
  const size_t smem = query_f32_smem_bytes(a.mode, f32_buf_rows(a.m, a.g.E));
  NDF_CUDA_CHECK(attr.ensure(query_f32_kernel, query_f32_smem_bytes(1)));
  // resident CTAs per SM for this SMEM size (registers cap it at 6), cached per size
  static thread_local size_t occ_smem = 0;
  static thread_local int occ_blocks = 1;
  if (occ_smem != smem) {
    int b = 0;
    NDF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, query_f32_kernel, kThreadsF32,
                                                                 smem));
    occ_blocks = std::max(b, 1);
    occ_smem = smem;
  }
  const int64_t n = a.v1 - a.v0;
  const int64_t tiles = (n + kTV - 1) / kTV;
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)sm_count() * occ_blocks);
  query_f32_kernel<<<(unsigned)std::max<int64_t>(grid, 1), kThreadsF32, smem, s>>>(a);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}


}  // namespace ndf

using namespace ndf;

static int query_grid(const ndf_model_desc* m, double rx, double ry, double rz,
                      int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz, int64_t v0,
                      int64_t v1, int32_t precision, float* out, uint32_t* stats,
                      void* stream) {
  int st = validate_model(m);
  if (st) return st;
  NDF_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, NDF_ERR_PARAMETER, "grid dims must be >= 1");
  const int64_t V = (int64_t)nx * ny * nz;
  NDF_REQUIRE(v0 >= 0 && v0 <= v1 && v1 <= V, NDF_ERR_PARAMETER, "vertex range out of bounds");
  NDF_REQUIRE(out != nullptr || v0 == v1, NDF_ERR_PARAMETER, "null output");
  if (v0 == v1) return NDF_OK;
  void* out_dev = nullptr;
  if ((st = resolve_output(out, &out_dev))) return st;
  QueryArgs a{};
  a.m = *m;
  a.g = make_geom(*m);
  a.mode = 0;
  a.ref_is_mu = ref_is_mu ? 1 : 0;
  a.ref[0] = rx; a.ref[1] = ry; a.ref[2] = rz;
  a.nx = nx; a.ny = ny; a.nz = nz;
  a.v0 = v0; a.v1 = v1;
  a.out = static_cast<float*>(out_dev);
  a.prec = precision;
  a.stats = stats;
  if (precision == NDF_PREC_BF16 || precision == NDF_PREC_FP16)
    return launch_query_tc(a, as_stream(stream));
  NDF_REQUIRE(precision == NDF_PREC_FP32, NDF_ERR_PARAMETER, "unknown precision");
  return launch_query_f32(a, as_stream(stream));
}

extern "C" int ndf_query_grid(const ndf_model_desc* m, double rx, double ry, double rz,
                              int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                              int64_t v0, int64_t v1, int32_t precision, float* out,
                              void* stream) {
  return query_grid(m, rx, ry, rz, ref_is_mu, nx, ny, nz, v0, v1, precision, out, nullptr,
                    stream);
}

extern "C" int ndf_query_grid_stats(const ndf_model_desc* m, double rx, double ry, double rz,
                                    int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                                    int64_t v0, int64_t v1, int32_t precision, float* out,
                                    uint32_t* stats, void* stream) {
  NDF_REQUIRE(stats, NDF_ERR_PARAMETER, "null stats");
  cudaStream_t s = as_stream(stream);
  NDF_CUDA_CHECK(cudaMemsetAsync(stats, 0xff, sizeof(uint32_t), s));           // min key
  NDF_CUDA_CHECK(cudaMemsetAsync(stats + 1, 0, 2 * sizeof(uint32_t), s));      // max key, NaN
  return query_grid(m, rx, ry, rz, ref_is_mu, nx, ny, nz, v0, v1, precision, out, stats,
                    stream);
}

extern "C" int ndf_query_points(const ndf_model_desc* m, const double* p_mu, int64_t n_mu,
                                const double* p_nu, int64_t n, int32_t precision, float* out,
                                void* stream) {
  int st = validate_model(m);
  if (st) return st;
  NDF_REQUIRE(n >= 0, NDF_ERR_PARAMETER, "negative batch");
  NDF_REQUIRE(n_mu == 1 || n_mu == n, NDF_ERR_SHAPE, "p_mu must have 1 or n rows");
  if (n == 0) return NDF_OK;
  NDF_REQUIRE(p_mu && p_nu && out, NDF_ERR_PARAMETER, "null pointer");
  void* out_dev = nullptr;
  if ((st = resolve_output(out, &out_dev))) return st;
  QueryArgs a{};
  a.m = *m;
  a.g = make_geom(*m);
  a.mode = 1;
  a.ref_is_mu = 1;
  a.v0 = 0; a.v1 = n;
  a.p_mu = p_mu; a.n_mu = n_mu; a.p_nu = p_nu;
  a.out = static_cast<float*>(out_dev);
  a.prec = precision;
  if (precision == NDF_PREC_BF16 || precision == NDF_PREC_FP16)
    return launch_query_tc(a, as_stream(stream));
  NDF_REQUIRE(precision == NDF_PREC_FP32, NDF_ERR_PARAMETER, "unknown precision");
  return launch_query_f32(a, as_stream(stream));
}
