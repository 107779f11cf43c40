// Exact fp32 NDF query (SIMT): embed -> merge -> decoder -> head.
//
// The decoder matmul restates matmul_exact (nn.py:18-20): z_j = sum_k h_k w_kj
// accumulated sequentially in ascending k with separately rounded multiply and
// add (no FMA contraction), bias added afterwards (nn.py:135) -- bit-identical
// to the reference's einsum.  Hidden activations / heads use libdevice fp32
// transcendentals (<= 2 ulp from NumPy's), so outputs agree to ~1e-7.
//
// Used for BASELINE config 0 (fp32) and as the exact mode of every query.
// Tile: 128 threads, 32 query vertices; activations staged k-major in SMEM so
// each k step reads the tile's 32 activations as 8 broadcast LDS.128.
#include <algorithm>

#include "ndf_query.cuh"

namespace ndf {

constexpr int kTV = 32;               // vertices per tile
constexpr int kTVP = kTV + 4;         // padded k-row stride (floats)
constexpr int kThreadsF32 = 128;

__global__ void __launch_bounds__(kThreadsF32)
query_f32_kernel(const QueryArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int Wmax = NDF_MAX_WIDTH;
  float* H0 = smem;                          // [Wmax][kTVP] k-major
  float* H1 = H0 + Wmax * kTVP;
  float* e_ref = H1 + Wmax * kTVP;           // [kMaxEmbed]
  float* e_q = e_ref + kMaxEmbed;            // [kTV][kMaxEmbed]

  const int tid = threadIdx.x;
  const EmbedGeom& g = a.g;
  const int E = g.E;
  const int64_t n_vert = a.v1 - a.v0;
  const float* P = a.m.params_f32;

  if (a.mode == 0 && tid == 0) {
    const float* grid = a.ref_is_mu ? a.m.grid_mu : a.m.grid_nu;
    embed_point(g, grid, a.ref[0], a.ref[1], a.ref[2], [&](int i, float v) { e_ref[i] = v; });
  }
  __syncthreads();

  for (int64_t tile = blockIdx.x; tile * kTV < n_vert; tile += gridDim.x) {
    const int64_t base = a.v0 + tile * kTV;
    const int nv = (int)min((int64_t)kTV, a.v1 - base);
    // ---- embed + merge: one thread per vertex ------------------------------
    if (tid < kTV) {
      const int v = tid;
      float* eq = e_q + v * kMaxEmbed;
      if (v < nv) {
        const int64_t gv = base + v;
        if (a.mode == 0) {
          double p[3];
          vertex_position(a, gv, p);
          const float* grid = a.ref_is_mu ? a.m.grid_nu : a.m.grid_mu;
          embed_point(g, grid, p[0], p[1], p[2], [&](int i, float x) { eq[i] = x; });
          auto ld_r = [&](int i) { return e_ref[i]; };
          auto ld_q = [&](int i) { return eq[i]; };
          auto st = [&](int i, float x) { H0[i * kTVP + v] = x; };
          if (a.ref_is_mu) merge_into(a.m.merge, E, ld_r, ld_q, st);
          else merge_into(a.m.merge, E, ld_q, ld_r, st);
        } else {
          const int64_t im = a.n_mu == 1 ? 0 : gv;
          float* em = eq;
          // mu embedding into e_q row, nu embedding into the H1 scratch column
          embed_point(g, a.m.grid_mu, a.p_mu[3 * im], a.p_mu[3 * im + 1], a.p_mu[3 * im + 2],
                      [&](int i, float x) { em[i] = x; });
          embed_point(g, a.m.grid_nu, a.p_nu[3 * gv], a.p_nu[3 * gv + 1], a.p_nu[3 * gv + 2],
                      [&](int i, float x) { H1[i * kTVP + v] = x; });
          auto ld_m = [&](int i) { return em[i]; };
          auto ld_n = [&](int i) { return H1[i * kTVP + v]; };
          auto st = [&](int i, float x) { H0[i * kTVP + v] = x; };
          merge_into(a.m.merge, E, ld_m, ld_n, st);
        }
      } else {
        const int din = a.m.widths[0];
        for (int i = 0; i < din; ++i) H0[i * kTVP + v] = 0.0f;
      }
    }
    __syncthreads();
    // ---- decoder ------------------------------------------------------------
    float* Hin = H0;
    float* Hout = H1;
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
          a.out[base - a.v0 + tid] = head_exact(a.m.head, z);
        }
      } else {
        for (int j = tid; j < N; j += kThreadsF32) {
          float acc[kTV];
#pragma unroll
          for (int v = 0; v < kTV; ++v) acc[v] = 0.0f;
          for (int k = 0; k < K; ++k) {
            const float w = __ldg(W + (size_t)k * N + j);
            const float4* hr = reinterpret_cast<const float4*>(Hin + k * kTVP);
#pragma unroll
            for (int q = 0; q < kTV / 4; ++q) {
              const float4 h = hr[q];
              acc[4 * q + 0] = fadd(acc[4 * q + 0], fmul(h.x, w));
              acc[4 * q + 1] = fadd(acc[4 * q + 1], fmul(h.y, w));
              acc[4 * q + 2] = fadd(acc[4 * q + 2], fmul(h.z, w));
              acc[4 * q + 3] = fadd(acc[4 * q + 3], fmul(h.w, w));
            }
          }
          const float bj = __ldg(b + j);
          float4* ho = reinterpret_cast<float4*>(Hout + j * kTVP);
#pragma unroll
          for (int q = 0; q < kTV / 4; ++q) {
            float4 o;
            o.x = act_exact(a.m.activation, fadd(acc[4 * q + 0], bj));
            o.y = act_exact(a.m.activation, fadd(acc[4 * q + 1], bj));
            o.z = act_exact(a.m.activation, fadd(acc[4 * q + 2], bj));
            o.w = act_exact(a.m.activation, fadd(acc[4 * q + 3], bj));
            ho[q] = o;
          }
        }
      }
      __syncthreads();
      float* t = Hin; Hin = Hout; Hout = t;
    }
  }
}

size_t query_f32_smem_bytes() {
  return sizeof(float) * (2 * NDF_MAX_WIDTH * kTVP + kMaxEmbed + kTV * kMaxEmbed);
}

int validate_model(const ndf_model_desc* m) {
  NDF_REQUIRE(m != nullptr, NDF_ERR_PARAMETER, "null model descriptor");
  NDF_REQUIRE(m->fourier_octaves >= 0 && m->fourier_octaves <= 12, NDF_ERR_UNSUPPORTED,
              "fourier_octaves must be in [0, 12]");
  NDF_REQUIRE(m->grid_channels >= 1 && m->grid_channels <= 64, NDF_ERR_UNSUPPORTED,
              "grid_channels must be in [1, 64]");
  for (int i = 0; i < 3; ++i)
    NDF_REQUIRE(m->grid_res[i] >= 2, NDF_ERR_CONFIG, "latent resolution must be >= 2 per axis");
  NDF_REQUIRE(m->n_layers >= 1 && m->n_layers <= NDF_MAX_LAYERS, NDF_ERR_UNSUPPORTED,
              "decoder layer count out of range");
  const int E = 3 + 6 * m->fourier_octaves + m->grid_channels;
  const int din = (m->merge == NDF_MERGE_SUM_ABSDIFF || m->merge == NDF_MERGE_CONCAT) ? 2 * E : E;
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
  static bool attr_set = false;
  const size_t smem = query_f32_smem_bytes();
  if (!attr_set) {
    NDF_CUDA_CHECK(cudaFuncSetAttribute(query_f32_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  const int64_t n = a.v1 - a.v0;
  const int64_t tiles = (n + kTV - 1) / kTV;
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)sm_count() * 3);
  query_f32_kernel<<<(unsigned)std::max<int64_t>(grid, 1), kThreadsF32, smem, s>>>(a);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}


}  // namespace ndf

using namespace ndf;

extern "C" int ndf_query_grid(const ndf_model_desc* m, double rx, double ry, double rz,
                              int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                              int64_t v0, int64_t v1, int32_t precision, float* out,
                              void* stream) {
  int st = validate_model(m);
  if (st) return st;
  NDF_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, NDF_ERR_PARAMETER, "grid dims must be >= 1");
  const int64_t V = (int64_t)nx * ny * nz;
  NDF_REQUIRE(v0 >= 0 && v0 <= v1 && v1 <= V, NDF_ERR_PARAMETER, "vertex range out of bounds");
  NDF_REQUIRE(out != nullptr || v0 == v1, NDF_ERR_PARAMETER, "null output");
  if (v0 == v1) return NDF_OK;
  QueryArgs a{};
  a.m = *m;
  a.g = make_geom(*m);
  a.mode = 0;
  a.ref_is_mu = ref_is_mu ? 1 : 0;
  a.ref[0] = rx; a.ref[1] = ry; a.ref[2] = rz;
  a.nx = nx; a.ny = ny; a.nz = nz;
  a.v0 = v0; a.v1 = v1;
  a.out = out;
  a.prec = precision;
  if (precision == NDF_PREC_BF16 || precision == NDF_PREC_FP16)
    return launch_query_tc(a, as_stream(stream));
  NDF_REQUIRE(precision == NDF_PREC_FP32, NDF_ERR_PARAMETER, "unknown precision");
  return launch_query_f32(a, as_stream(stream));
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
  QueryArgs a{};
  a.m = *m;
  a.g = make_geom(*m);
  a.mode = 1;
  a.ref_is_mu = 1;
  a.v0 = 0; a.v1 = n;
  a.p_mu = p_mu; a.n_mu = n_mu; a.p_nu = p_nu;
  a.out = out;
  a.prec = precision;
  if (precision == NDF_PREC_BF16 || precision == NDF_PREC_FP16)
    return launch_query_tc(a, as_stream(stream));
  NDF_REQUIRE(precision == NDF_PREC_FP32, NDF_ERR_PARAMETER, "unknown precision");
  return launch_query_f32(a, as_stream(stream));
}
