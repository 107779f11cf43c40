// Fused NDF query on 5th-generation tensor cores (K1 + K2, sm_100a).
//
//   embed (fp64 -> fp32, bit-exact with model.py:169-177)
//   -> merge [e_r + e_q, |e_r - e_q|]                      (model.py:279-286 + BASELINE)
//   -> H x { tcgen05.mma bf16 x bf16 -> fp32 (TMEM) ; bias + activation in the
//            tcgen05.ld epilogue ; bf16 back to SMEM as the next A operand }
//   -> output layer (128 -> 1) as an fp32 dot product in the last epilogue -> head.
//
// Layout / schedule (one persistent CTA per SM, NWG <= 4 warpgroups):
//   * the packed parameter blob (UMMA-canonical K-major bf16 weights + fp32 bias
//     vectors) is fetched once per CTA by the bulk-copy engine (cp.async.bulk ->
//     mbarrier complete_tx) and stays resident in SMEM;
//   * each warpgroup owns a 128-row tile of query vertices, one 32 KB A buffer
//     (SWIZZLE_NONE canonical layout: 8x16 B core matrices, LBO = 128 B along K,
//     SBO = 2048 B along M) and 128 TMEM columns holding the fp32 accumulator
//     (row m of the tile = TMEM lane m = thread m of the warpgroup);
//   * one thread per warpgroup issues the K/16 tcgen05.mma steps of a layer and
//     commits them to the warpgroup's mbarrier; while one warpgroup runs its
//     epilogue (MUFU/ALU-bound), the other warpgroups' MMAs keep the tensor pipe
//     busy -- a 4-way ping-pong without any CTA-wide barrier.
#include <algorithm>

#include "ndf_query.cuh"

namespace ndf {

namespace tc {

constexpr int kHid = 128;           // hidden width (UMMA N)
constexpr int kTileM = 128;         // rows per tile (UMMA M)
constexpr int kABytes = kTileM * kHid * 2;     // 32 KB A buffer
constexpr int kSboA = (kHid / 8) * 128;        // 2048 B between 8-row groups
constexpr int kL = 6;               // Fourier octaves supported by the fused encoder
constexpr int kC = 16;              // latent channels supported by the fused encoder
constexpr int kE = 3 + 6 * kL + kC; // 55
constexpr int kMaxSmem = 232448;    // 227 KB opt-in

struct Layout {
  int H;            // MMA layers (hidden layers)
  int kin;          // padded layer-0 K (multiple of 16, <= 128)
  int w0_bytes;     // 128 x kin bf16
  int wh_bytes;     // 128 x 128 bf16
  int vec_off;      // byte offset of fp32 vectors (biases, w_out, b_out)
  int blob_bytes;   // multiple of 16
};

__host__ __device__ inline Layout make_layout(const ndf_model_desc& m) {
  Layout L;
  L.H = m.n_layers - 1;
  L.kin = (m.widths[0] + 15) / 16 * 16;
  L.w0_bytes = kHid * L.kin * 2;
  L.wh_bytes = kHid * kHid * 2;
  L.vec_off = L.w0_bytes + (L.H - 1) * L.wh_bytes;
  const int vec_bytes = (L.H * kHid + kHid + 4) * 4;
  L.blob_bytes = L.vec_off + vec_bytes;
  return L;
}

// byte offset of element (row r, k) inside a canonical K-major no-swizzle tile
__host__ __device__ __forceinline__ int canon_off(int r, int k, int sbo) {
  return (r >> 3) * sbo + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

// ---------------------------------------------------------------------------
// PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  return d;                           // base_offset 0, lbo_mode 0, SWIZZLE_NONE
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
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
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <bool F16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (F16) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// Hidden activation for the bf16 path (fast forms; within the 1e-2 bf16 contract).
__device__ __forceinline__ float act_fast(int kind, float x) {
  switch (kind) {
    case NDF_ACT_SILU: {            // x*sigmoid(x) = hx + hx*tanh(hx), hx = x/2 (1 MUFU op)
      const float hx = 0.5f * x;
      return fmaf(hx, tanh_fast(hx), hx);
    }
    case NDF_ACT_RELU: return fmaxf(x, 0.0f);
    case NDF_ACT_SNAKE: { const float s = __sinf(x); return fmaf(s, s, x); }
    default: return 0.5f * (x + 1.0f - __cosf(2.0f * x));
  }
}

// Merged decoder-input element idx (model.py:279-286 + BASELINE's sum_absdiff),
// computed in fp32 from the two embeddings (ea = mu branch, eb = nu branch).
template <class FA, class FB>
__device__ __forceinline__ float merged_value(int merge, int idx, FA ea, FB eb) {
  if (idx < kE) {
    const float a = ea(idx), b = eb(idx);
    switch (merge) {
      case NDF_MERGE_MULTIPLY: return a * b;
      case NDF_MERGE_ABSDIFF: return fabsf(a - b);
      case NDF_MERGE_CONCAT: return a;
      default: return a + b;          // add, sum_absdiff
    }
  }
  if (idx < 2 * kE) {
    const float a = ea(idx - kE), b = eb(idx - kE);
    if (merge == NDF_MERGE_CONCAT) return b;
    if (merge == NDF_MERGE_SUM_ABSDIFF) return fabsf(a - b);
  }
  return 0.0f;
}

// Write one row of the layer-0 A operand (bf16, canonical layout).
template <bool F16, class FA, class FB>
__device__ __forceinline__ void write_input_row(uint32_t abase, int row, int merge, FA ea, FB eb,
                                                int kin) {
#pragma unroll
  for (int kg = 0; kg < 16; ++kg) {
    if (kg * 8 < kin) {
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = merged_value(merge, 8 * kg + j, ea, eb);
      st_shared_v4(abase + canon_off(row, kg * 8, kSboA), pack2<F16>(x[0], x[1]),
                   pack2<F16>(x[2], x[3]), pack2<F16>(x[4], x[5]), pack2<F16>(x[6], x[7]));
    }
  }
}

template <bool F16>
__global__ void __launch_bounds__(512, 1)
query_tc_kernel(const QueryArgs a, const int nwg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Layout lay = make_layout(a.m);
  uint8_t* wblob = smem;                                   // parameter blob
  uint8_t* abufs = smem + ((lay.blob_bytes + 1023) & ~1023);
  float* e_ref = reinterpret_cast<float*>(abufs + nwg * kABytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(e_ref + 64);   // [0] weights, [1+w] per WG
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int wg = warp >> 2;
  const int wtid = tid & 127;               // row of the tile owned by this thread
  const float* vecs = reinterpret_cast<const float*>(wblob + lay.vec_off);
  const uint32_t tmem_cols = nwg > 2 ? 512 : (nwg == 2 ? 256 : 128);

  if (tid == 0) {
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
  if (a.mode == 0 && tid == 32) {
    const float* grid = a.ref_is_mu ? a.m.grid_mu : a.m.grid_nu;
    embed_point(a.g, grid, a.ref[0], a.ref[1], a.ref[2], [&](int i, float v) { e_ref[i] = v; });
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
  uint8_t* abuf = abufs + wg * kABytes;
  const uint32_t a_addr = smem_u32(abuf);
  const uint32_t w_addr = smem_u32(wblob);
  uint64_t* bar = &bars[1 + wg];
  // kind::f16 instruction descriptor: D fp32, A/B bf16 (1) or fp16 (0), K-major both,
  // N = 128 (bits 17-22, N>>3), M = 128 (bits 24-28, M>>4)
  const uint32_t ab_fmt = F16 ? 0u : 1u;
  const uint32_t idesc = (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) |
                         ((uint32_t)(kHid >> 3) << 17) | ((uint32_t)(kTileM >> 4) << 24);
  const int sbo_w0 = (lay.kin / 8) * 128;

  mbar_wait(&bars[0], 0);    // parameters resident

  const int64_t n = a.v1 - a.v0;
  const int64_t n_tiles = (n + kTileM - 1) / kTileM;
  const int64_t stride = (int64_t)gridDim.x * nwg;
  uint32_t phase = 0;
  const float* grid_q = a.ref_is_mu ? a.m.grid_nu : a.m.grid_mu;
  const int bar_id = 1 + wg;

  for (int64_t tile = (int64_t)blockIdx.x * nwg + wg; tile < n_tiles; tile += stride) {
    const int64_t vloc = tile * kTileM + wtid;   // local vertex index
    const bool valid = vloc < n;
    // ---- K1: embed + merge -> A (bf16) ----------------------------------------
    if (valid) {
      const int64_t gv = a.v0 + vloc;
      float eq[kE];
      if (a.mode == 0) {
        double p[3];
        vertex_position(a, gv, p);
        embed_point_t<kL, kC>(a.g.rx, a.g.ry, a.g.rz, grid_q, p[0], p[1], p[2], eq);
        auto fq = [&](int i) { return eq[i]; };
        auto fr = [&](int i) { return e_ref[i]; };
        if (a.ref_is_mu) write_input_row<F16>(a_addr, wtid, a.m.merge, fr, fq, lay.kin);
        else write_input_row<F16>(a_addr, wtid, a.m.merge, fq, fr, lay.kin);
      } else {
        float em[kE];
        const int64_t im = a.n_mu == 1 ? 0 : gv;
        embed_point_t<kL, kC>(a.g.rx, a.g.ry, a.g.rz, a.m.grid_mu, a.p_mu[3 * im],
                              a.p_mu[3 * im + 1], a.p_mu[3 * im + 2], em);
        embed_point_t<kL, kC>(a.g.rx, a.g.ry, a.g.rz, a.m.grid_nu, a.p_nu[3 * gv],
                              a.p_nu[3 * gv + 1], a.p_nu[3 * gv + 2], eq);
        auto fm = [&](int i) { return em[i]; };
        auto fq = [&](int i) { return eq[i]; };
        write_input_row<F16>(a_addr, wtid, a.m.merge, fm, fq, lay.kin);
      }
    } else {
      auto fz = [](int) { return 0.0f; };
      write_input_row<F16>(a_addr, wtid, NDF_MERGE_ADD, fz, fz, lay.kin);
    }
    fence_proxy_async();
    tc_fence_before();
    named_bar(bar_id, 128);
    // ---- K2: H tensor-core layers -----------------------------------------------
    float out_acc = 0.0f;
    for (int l = 0; l < lay.H; ++l) {
      if (wtid == 0) {
        tc_fence_after();
        const int K = l == 0 ? lay.kin : kHid;
        const uint32_t wl = w_addr + (l == 0 ? 0 : lay.w0_bytes + (l - 1) * lay.wh_bytes);
        const uint32_t sbo_b = l == 0 ? sbo_w0 : kSboA;
        for (int kk = 0; kk < K / 16; ++kk) {
          const uint64_t ad = smem_desc(a_addr + kk * 256, 128, kSboA);
          const uint64_t bd = smem_desc(wl + kk * 256, 128, sbo_b);
          mma_bf16(d_tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_fence_after();
      const float* bias = vecs + l * kHid;
      const bool last = (l == lay.H - 1);
#pragma unroll 1
      for (int c0 = 0; c0 < kHid; c0 += 32) {
        float v[32];
        tmem_ld32(tmem_base + lane_base + (uint32_t)(wg * kHid + c0), v);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = act_fast(a.m.activation, v[i] + bias[c0 + i]);
        if (last) {
          const float* wo = vecs + lay.H * kHid;
#pragma unroll
          for (int i = 0; i < 32; ++i) out_acc = fmaf(v[i], wo[c0 + i], out_acc);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            st_shared_v4(a_addr + canon_off(wtid, c0 + 8 * j, kSboA),
                         pack2<F16>(v[8 * j], v[8 * j + 1]), pack2<F16>(v[8 * j + 2], v[8 * j + 3]),
                         pack2<F16>(v[8 * j + 4], v[8 * j + 5]), pack2<F16>(v[8 * j + 6], v[8 * j + 7]));
        }
      }
      if (!last) fence_proxy_async();
      tc_fence_before();
      named_bar(bar_id, 128);
    }
    if (valid) {
      const float z = out_acc + vecs[lay.H * kHid + kHid];
      a.out[vloc] = head_exact(a.m.head, z);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
}

// ---- parameter packing (device) ---------------------------------------------
__global__ void pack_kernel(const ndf_model_desc m, uint8_t* blob) {
  const Layout lay = make_layout(m);
  const int64_t total = (int64_t)lay.blob_bytes / 4;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint32_t*>(blob)[w] = 0u;
  __syncthreads();   // per-block only; a grid-wide order is provided by two launches
}

__global__ void pack_fill_kernel(const ndf_model_desc m, uint8_t* blob) {
  const Layout lay = make_layout(m);
  // weights: layer l (K x N fp32 row-major, N = 128) -> canonical N x Kpad bf16
  size_t off = 0;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  float* vecs = reinterpret_cast<float*>(blob + lay.vec_off);
  for (int l = 0; l < m.n_layers; ++l) {
    const int K = m.widths[l], N = m.widths[l + 1];
    const float* W = m.params_f32 + off;
    const float* b = W + (size_t)K * N;
    if (l < lay.H) {
      const int kpad = l == 0 ? lay.kin : kHid;
      const int sbo = (kpad / 8) * 128;
      uint8_t* dst = blob + (l == 0 ? 0 : lay.w0_bytes + (l - 1) * lay.wh_bytes);
      for (int64_t e = gtid; e < (int64_t)K * N; e += gsz) {
        const int k = (int)(e / N), nn = (int)(e % N);
        if (m.tc_format == NDF_PREC_FP16)
          *reinterpret_cast<__half*>(dst + canon_off(nn, k, sbo)) = __float2half_rn(W[e]);
        else
          *reinterpret_cast<__nv_bfloat16*>(dst + canon_off(nn, k, sbo)) = __float2bfloat16_rn(W[e]);
      }
      for (int64_t e = gtid; e < N; e += gsz) vecs[l * kHid + e] = b[e];
    } else {
      for (int64_t e = gtid; e < K; e += gsz) vecs[lay.H * kHid + e] = W[e];
      if (gtid == 0) vecs[lay.H * kHid + kHid] = b[0];
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

int launch_query_tc(const QueryArgs& a, cudaStream_t s) {
  std::string why;
  NDF_REQUIRE(tc_supported(a.m, &why), NDF_ERR_UNSUPPORTED, why);
  NDF_REQUIRE(a.m.params_tc != nullptr, NDF_ERR_PARAMETER,
              "tensor-core query needs the packed parameter blob (ndf_tc_pack)");
  NDF_REQUIRE(a.m.tc_format == a.prec, NDF_ERR_PARAMETER,
              "packed blob element type does not match the requested precision");
  const tc::Layout lay = tc::make_layout(a.m);
  const int blob_al = (lay.blob_bytes + 1023) & ~1023;
  int nwg = (tc::kMaxSmem - blob_al - 1024) / tc::kABytes;
  nwg = std::min(nwg, 4);
  const size_t smem = (size_t)blob_al + (size_t)nwg * tc::kABytes + 1024;
  static size_t attr_smem = 0;
  if (attr_smem < smem) {
    NDF_CUDA_CHECK(cudaFuncSetAttribute(tc::query_tc_kernel<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NDF_CUDA_CHECK(cudaFuncSetAttribute(tc::query_tc_kernel<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_smem = smem;
  }
  const int64_t n = a.v1 - a.v0;
  const int64_t tiles = (n + tc::kTileM - 1) / tc::kTileM;
  const int64_t ctas = std::min<int64_t>((tiles + nwg - 1) / nwg, sm_count());
  const unsigned grid = (unsigned)std::max<int64_t>(ctas, 1);
  if (a.prec == NDF_PREC_FP16)
    tc::query_tc_kernel<true><<<grid, nwg * 128, smem, s>>>(a, nwg);
  else
    tc::query_tc_kernel<false><<<grid, nwg * 128, smem, s>>>(a, nwg);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

}  // namespace ndf

using namespace ndf;

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
  tc::pack_kernel<<<64, 256, 0, as_stream(stream)>>>(*m, (uint8_t*)blob);
  NDF_LAUNCH_CHECK();
  tc::pack_fill_kernel<<<64, 256, 0, as_stream(stream)>>>(*m, (uint8_t*)blob);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_query_grid_multi(const ndf_model_desc* m, const double* refs, int32_t n_ref,
                                    int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                                    int64_t v0, int64_t v1, uint16_t* out_f16, int64_t ld_out,
                                    void* stream) {
  (void)m; (void)refs; (void)n_ref; (void)ref_is_mu; (void)nx; (void)ny; (void)nz;
  (void)v0; (void)v1; (void)out_f16; (void)ld_out; (void)stream;
  ndf::set_error("ndf_query_grid_multi: not implemented yet");
  return NDF_ERR_UNSUPPORTED;
}
