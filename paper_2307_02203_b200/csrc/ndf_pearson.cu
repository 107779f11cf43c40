// Ground-truth Pearson field (K3) + ensemble sampling / layout support (K5).
//
// Reference: measures.pearson_against (measures.py:84-108), pearson_rowwise
// (measures.py:111-133), ground_truth_field's Pearson branch (measures.py:286-295),
// sample_many (ensemble.py:130-167).
//
// Node-aligned fields use a one-time standardisation Z = (X - mean)/||X - mean||
// (fp64 statistics, fp32 storage) and then an HBM-streaming GEMV r = Z^T z_ref:
// each thread owns 4 consecutive vertices (one LDG.128 per member row, coalesced
// across the warp), partial sums are kept in fp32 for 32 members and folded into
// fp64 so the result stays within ~1e-7 of the reference's fp64 two-pass formula.
#include <algorithm>

#include "ndf_common.cuh"
#include "ndf_tc_ptx.cuh"


namespace ndf {

__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// ---- sample_many: ensemble.py:130-167 --------------------------------------
// out[b][m] = sum over (dz, dy, dx) of (wz*wy*wx) * X[m, iz+dz, iy+dy, ix+dx],
// accumulated from 0 in that loop order in fp64 (no FMA) -- bit-identical.
__device__ __forceinline__ void frac_index(double p, int n, int& i0, double& t) {
  double pc = fmin(fmax(p, -1.0), 1.0);
  double u = dmul(dmul(dadd(pc, 1.0), 0.5), (double)(n - 1));
  int i = (int)floor(u);
  if (i < 0) i = 0;
  if (i > n - 2) i = n - 2;
  t = dsub(u, (double)i);
  if (t < 1e-9) t = 0.0;
  if (t > 1.0 - 1e-9) t = 1.0;
  i0 = i;
}

// X holds node columns [col0, col0 + ld) of the member-major ensemble, member rows
// ld apart (ld = V, col0 = 0: the whole variable).
__global__ void sample_many_kernel(const float* __restrict__ X, int M, int64_t ld, int64_t col0,
                                   int nx, int ny, int nz, const double* __restrict__ pos,
                                   int64_t B, double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * (int64_t)M) return;
  const int64_t b = idx / M;
  const int m = (int)(idx - b * M);
  int ix, iy, iz;
  double tx, ty, tz;
  frac_index(pos[3 * b + 0], nx, ix, tx);
  frac_index(pos[3 * b + 1], ny, iy, ty);
  frac_index(pos[3 * b + 2], nz, iz, tz);
  const float* g = X + (int64_t)m * ld - col0;
  double acc = 0.0;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    const double wz = dz ? tz : dsub(1.0, tz);
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const double wy = dy ? ty : dsub(1.0, ty);
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const double wx = dx ? tx : dsub(1.0, tx);
        const double w = dmul(dmul(wz, wy), wx);
        const float c = g[(int64_t)(iz + dz) * ny * nx + (int64_t)(iy + dy) * nx + (ix + dx)];
        acc = dadd(acc, dmul(w, (double)c));
      }
    }
  }
  out[idx] = acc;
}

// Same samples from the vertex-major copy Xv (V, M): consecutive threads are consecutive
// members of one position, so each corner read is a contiguous row segment.
__global__ void sample_many_vm_kernel(const float* __restrict__ Xv, int M, int nx, int ny, int nz,
                                      const double* __restrict__ pos, int64_t B,
                                      double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * (int64_t)M) return;
  const int64_t b = idx / M;
  const int m = (int)(idx - b * M);
  int ix, iy, iz;
  double tx, ty, tz;
  frac_index(pos[3 * b + 0], nx, ix, tx);
  frac_index(pos[3 * b + 1], ny, iy, ty);
  frac_index(pos[3 * b + 2], nz, iz, tz);
  double acc = 0.0;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    const double wz = dz ? tz : dsub(1.0, tz);
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const double wy = dy ? ty : dsub(1.0, ty);
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const double wx = dx ? tx : dsub(1.0, tx);
        const double w = dmul(dmul(wz, wy), wx);
        const int64_t vtx = (int64_t)(iz + dz) * ny * nx + (int64_t)(iy + dy) * nx + (ix + dx);
        acc = dadd(acc, dmul(w, (double)__ldg(Xv + vtx * M + m)));
      }
    }
  }
  out[idx] = acc;
}

// ---- fused Pearson field: one streaming read of X ---------------------------
// r[v] = sum_m (x_mv - mu_v)(ref_m - mu_r) / sqrt(var_v * var_r), measures.py:84-108,
// computed per vertex in ONE pass over its member column: shifted fp64 moments
// (d = x - x_0v: sum d, sum d^2, sum d * rc_m with rc = ref - mean(ref) in fp64), so
// neither Z nor a second read exists -- the bytes are exactly the column reads of X.
// Rules of the reference: degenerate (var == 0 on either side) -> NaN (the field maps
// it to 0 with a warning, measures.py:291-295); a column equal to the reference member
// for member -> exactly 1.0 (measures.py:102-107); otherwise clipped to [-1, 1].
constexpr int kFieldMaxM = 8192;

struct RefStats {
  double var_ref;     // sum (ref - mean)^2, fp64 two-pass
  int exact32;        // every ref_m is an fp32 value (a node column can equal it)
};

// one block: rc_m = ref_m - mean(ref) (fp64, two-pass), r32 = (float)ref, var_ref
__global__ void __launch_bounds__(1024)
pearson_ref_kernel(const double* __restrict__ ref, int M, double* __restrict__ rc,
                   float* __restrict__ r32, RefStats* __restrict__ st) {
  __shared__ double red[32];
  __shared__ int ok32[32];
  auto block_sum = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
      t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    t = red[0];
    __syncthreads();
    return t;
  };
  double s = 0.0;
  int ex = 1;
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const double r = ref[m];
    s += r;
    ex &= ((double)(float)r == r);
  }
  const double mean = block_sum(s) / (double)M;
  ex = __all_sync(0xffffffffu, ex);
  if ((threadIdx.x & 31) == 0) ok32[threadIdx.x >> 5] = ex;
  double q = 0.0;
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const double c = ref[m] - mean;
    rc[m] = c;
    r32[m] = (float)ref[m];
    q += c * c;
  }
  const double var = block_sum(q);
  if (threadIdx.x == 0) {
    int all = 1;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) all &= ok32[w];
    st->var_ref = var;
    st->exact32 = all;
  }
}

template <bool kVec>
__global__ void __launch_bounds__(256)
pearson_field_kernel(const float* __restrict__ X, int M, int64_t ld, int64_t col0,
                     const double* __restrict__ rc_g, const float* __restrict__ r32_g,
                     const RefStats* __restrict__ st, int64_t v0, int64_t v1,
                     float* __restrict__ out) {
  extern __shared__ double rcs[];
  float* r32 = reinterpret_cast<float*>(rcs + M);
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    rcs[i] = rc_g[i];
    r32[i] = r32_g[i];
  }
  __syncthreads();
  const double var_ref = st->var_ref;
  const bool can_eq = st->exact32 != 0;
  const int64_t v = v0 + 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (v >= v1) return;
  const int nv = (int)min((int64_t)4, v1 - v);
  const float* col = X + (v - col0);
  double sd[4] = {0.0, 0.0, 0.0, 0.0}, sd2[4] = {0.0, 0.0, 0.0, 0.0}, sdr[4] = {0.0, 0.0, 0.0, 0.0};
  float x0[4];
  bool eq[4] = {can_eq, can_eq, can_eq, can_eq};
  if (kVec && nv == 4) {
    const float4 f = ld_stream4(col);
    x0[0] = f.x; x0[1] = f.y; x0[2] = f.z; x0[3] = f.w;
#pragma unroll 4
    for (int m = 0; m < M; ++m) {
      const float4 x4 = ld_stream4(col + (int64_t)m * ld);
      const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
      const double r = rcs[m];
      const float rr = r32[m];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double d = (double)xs[i] - (double)x0[i];
        sd[i] += d;
        sd2[i] = fma(d, d, sd2[i]);
        sdr[i] = fma(d, r, sdr[i]);
        eq[i] &= (xs[i] == rr);
      }
    }
  } else {
    for (int i = 0; i < nv; ++i) {
      x0[i] = __ldg(col + i);
      for (int m = 0; m < M; ++m) {
        const float x = __ldg(col + (int64_t)m * ld + i);
        const double d = (double)x - (double)x0[i];
        sd[i] += d;
        sd2[i] = fma(d, d, sd2[i]);
        sdr[i] = fma(d, rcs[m], sdr[i]);
        eq[i] &= (x == r32[m]);
      }
    }
  }
  for (int i = 0; i < nv; ++i) {
    const double var = sd2[i] - sd[i] * (sd[i] / (double)M);
    float r;
    if (!(var_ref > 0.0) || !(var > 0.0)) {
      r = __int_as_float(0x7fc00000);        // degenerate: NaN (measures.py:94-100)
    } else if (eq[i]) {
      r = 1.0f;                               // measures.py:102-107
    } else {
      r = (float)fmin(1.0, fmax(-1.0, sdr[i] / sqrt(var * var_ref)));
    }
    out[v + i - v0] = r;
  }
}

#ifndef NDF_ZS_COLS
#define NDF_ZS_COLS 64
#endif
#ifndef NDF_ZS_BATCH
#define NDF_ZS_BATCH 4
#endif
#ifndef NDF_ZS_HINT
#define NDF_ZS_HINT true
#endif
// ---- z-score prep: one DRAM read + one DRAM write -----------------------------
// Z[m, v] = (x_mv - mean_v) / ||x_v - mean_v||, fp64 statistics (moments shifted by
// x_0v), fp32 storage; norm[v] = ||x_v - mean_v|| (0 and a zero column: degenerate).
// A persistent grid (kZBlocksPerSM blocks per SM) walks groups of kZCols consecutive
// columns; a block streams its group's member rows twice -- pass 1 accumulates the
// moments per row lane, the lanes are folded in a fixed order (deterministic per column,
// independent of the launch range), pass 2 writes Z with streaming stores -- and the
// second read is served by L2 (the grid keeps <= sm_count x kZBlocksPerSM x kZCols x M x
// 4 B in flight: 38 MB at M = 1000, L2 126 MB), so DRAM sees one read and one write of
// the ensemble (round 1 read it twice from DRAM: 3 x 7.04 GB at config 1).  Loads go in
// batches of kZBatch rows, all issued before any is used: a plain unrolled loop with its
// exit test between iterations had left ONE load in flight per thread.
// The rows are read with L2 eviction-priority hints: evict_last in pass 1 (they must
// survive until pass 2), evict_first in pass 2 -- without them 5.4 GB of the second read
// still came from DRAM (the group footprint, 2 blocks x 148 SMs x 256 KB = 76 MB, shares
// L2 with the 7 GB of streamed Z stores).  Measured on B200 at config 1
// (tools/zscore_probe.py): 2.86 ms = 4.9 TB/s of algorithmic traffic, 0.75 of the copy
// peak (round 1: 4.2 ms; this kernel without the hints 3.50 ms).  Alternatives measured:
// 32 / 128 columns per group 4.5 / 3.2 ms, batches of 2 / 6 rows 3.26 / 2.85 ms, fp32
// partial moments 3.17 ms without hints (6x the Z error: kept fp64), a cluster of 8 CTAs
// sharing 512-column groups through DSMEM 9 ms, a cp.async ring of 16 copies per thread
// 5.4 ms, per-row 256 B bulk copies 11.6 ms.  The
// kernel stays latency-bound: 32 warps x 4 row loads in flight per SM (64 registers).
constexpr int kZCols = NDF_ZS_COLS;
constexpr int kZThreads = 512;
constexpr int kZLanes = kZThreads / (kZCols / 4);    // row lanes
constexpr int kZBlocksPerSM = 2;
constexpr int kZBatch = NDF_ZS_BATCH;

// 16-byte load with an L2 eviction-priority policy (createpolicy): pass 1 marks the
// group's rows evict_last so they survive until pass 2, which reads them evict_first
template <bool kLast>
__device__ __forceinline__ float4 ld_l2hint4(const float* p) {
  float4 r;
  if constexpr (kLast)
    asm volatile("{\n\t.reg .b64 pol;\n\t"
                 "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
                 "ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  else
    asm volatile("{\n\t.reg .b64 pol;\n\t"
                 "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
                 "ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w) : "memory");
}

__global__ void __launch_bounds__(kZThreads, kZBlocksPerSM)
zscore_kernel(const float* __restrict__ X, int M, int64_t V, int64_t v0, int64_t v1,
              float* __restrict__ Z, float* __restrict__ norm) {
  __shared__ double part[kZLanes][2][kZCols];
  __shared__ double stat[2][kZCols];              // mean, 1 / norm (0: degenerate)
  const int tid = threadIdx.x;
  const int t = tid % (kZCols / 4), lane = tid / (kZCols / 4);
  const int64_t ngroups = (v1 - v0 + kZCols - 1) / kZCols;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t c = v0 + g * kZCols + 4 * t;
    const bool live = c < v1;
    float K[4];
    double s1[4], s2[4];
    {
      const float4 f = live ? __ldg(reinterpret_cast<const float4*>(X + c)) : make_float4(0, 0, 0, 0);
      K[0] = f.x; K[1] = f.y; K[2] = f.z; K[3] = f.w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) { s1[i] = 0.0; s2[i] = 0.0; }
    if (live) {
      for (int mb = lane; mb < M; mb += kZBatch * kZLanes) {         // pass 1: moments
        float4 f[kZBatch];
#pragma unroll
        for (int u = 0; u < kZBatch; ++u) {
          const int m = mb + u * kZLanes;
          f[u] = m < M ? ld_l2hint4<NDF_ZS_HINT>(X + (int64_t)m * V + c)
                       : make_float4(K[0], K[1], K[2], K[3]);       // d = 0: no contribution
        }
#pragma unroll
        for (int u = 0; u < kZBatch; ++u) {
          const float x[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double d = (double)x[i] - (double)K[i];
            s1[i] += d;
            s2[i] = fma(d, d, s2[i]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      part[lane][0][4 * t + i] = s1[i];
      part[lane][1][4 * t + i] = s2[i];
    }
    __syncthreads();
    if (tid < kZCols) {                                 // fold the lanes in order
      double a = 0.0, b = 0.0;
      for (int l = 0; l < kZLanes; ++l) { a += part[l][0][tid]; b += part[l][1][tid]; }
      const int64_t v = v0 + g * kZCols + tid;
      const double Kc = v < v1 ? (double)__ldg(X + v) : 0.0;
      const double off = a / (double)M;
      const double var = b - a * off;
      const bool ok = var > 0.0;
      stat[0][tid] = Kc + off;
      stat[1][tid] = ok ? 1.0 / sqrt(var) : 0.0;
      if (norm && v < v1) norm[v] = ok ? (float)sqrt(var) : 0.0f;
    }
    __syncthreads();
    double mu[4], inv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { mu[i] = stat[0][4 * t + i]; inv[i] = stat[1][4 * t + i]; }
    __syncthreads();                                    // part / stat free for the next group
    if (live) {
      const bool whole = c + 4 <= v1;
      for (int mb = lane; mb < M; mb += kZBatch * kZLanes) {         // pass 2: Z (from L2)
        float4 f[kZBatch];
#pragma unroll
        for (int u = 0; u < kZBatch; ++u) {
          const int m = mb + u * kZLanes;
          f[u] = m < M ? ld_l2hint4<false>(X + (int64_t)m * V + c)
                       : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kZBatch; ++u) {
          const int m = mb + u * kZLanes;
          if (m >= M) break;
          const float x[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
          float z[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            z[i] = inv[i] != 0.0 ? (float)(((double)x[i] - mu[i]) * inv[i]) : 0.0f;
          const int64_t o = (int64_t)m * V + c;
          if (whole) {
            st_stream4(Z + o, make_float4(z[0], z[1], z[2], z[3]));
          } else {
            for (int i = 0; c + i < v1; ++i) Z[o + i] = z[i];
          }
        }
      }
    }
  }
}

// Other layouts (V or v0 not a multiple of 4, unaligned pointers): one thread per
// column, two passes, same statistics.
__global__ void zscore_lsu_kernel(const float* __restrict__ X, int M, int64_t V, int64_t v0,
                                  int64_t v1, float* __restrict__ Z, float* __restrict__ norm) {
  const int64_t v = v0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= v1) return;
  const float* col = X + v;
  const double K = (double)col[0];
  double s1 = 0.0, s2 = 0.0;
  for (int m = 0; m < M; ++m) {
    const double d = (double)__ldg(col + (int64_t)m * V) - K;
    s1 += d;
    s2 = fma(d, d, s2);
  }
  const double off = s1 / (double)M;
  const double var = s2 - s1 * off;
  const bool ok = var > 0.0;
  const double mu = K + off;
  const double inv = ok ? 1.0 / sqrt(var) : 0.0;
  for (int m = 0; m < M; ++m)
    Z[(int64_t)m * V + v] = ok ? (float)(((double)__ldg(col + (int64_t)m * V) - mu) * inv) : 0.0f;
  if (norm) norm[v] = ok ? (float)sqrt(var) : 0.0f;
}

// ---- Pearson GEMV over Z -----------------------------------------------------
template <bool kVec>
__global__ void __launch_bounds__(256)
gemv_kernel(const float* __restrict__ Z, const float* __restrict__ norm, int M, int64_t V,
            const float* __restrict__ zref, int ref_deg, int64_t v0, int64_t v1,
            float* __restrict__ out) {
  extern __shared__ float zr[];
  for (int i = threadIdx.x; i < M; i += blockDim.x) zr[i] = zref[i];
  __syncthreads();
  const int64_t v = v0 + 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (v >= v1) return;
  double tot[4] = {0.0, 0.0, 0.0, 0.0};
  bool eq[4] = {true, true, true, true};
  if (kVec) {
    const float* zp = Z + v;
    for (int m0 = 0; m0 < M; m0 += 32) {
      const int m1 = min(M, m0 + 32);
      float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll 8
      for (int m = m0; m < m1; ++m) {
        const float4 z = ld_stream4(zp + (int64_t)m * V);
        const float r = zr[m];
        p0 = fmaf(z.x, r, p0); p1 = fmaf(z.y, r, p1);
        p2 = fmaf(z.z, r, p2); p3 = fmaf(z.w, r, p3);
        eq[0] &= (z.x == r); eq[1] &= (z.y == r); eq[2] &= (z.z == r); eq[3] &= (z.w == r);
      }
      tot[0] += p0; tot[1] += p1; tot[2] += p2; tot[3] += p3;
    }
  } else {
    for (int i = 0; i < 4; ++i) {
      if (v + i >= v1) break;
      const float* zp = Z + v + i;
      for (int m0 = 0; m0 < M; m0 += 32) {
        const int m1 = min(M, m0 + 32);
        float p = 0.f;
        for (int m = m0; m < m1; ++m) {
          const float z = __ldg(zp + (int64_t)m * V);
          p = fmaf(z, zr[m], p);
          eq[i] &= (z == zr[m]);
        }
        tot[i] += p;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (v + i >= v1) break;
    float r;
    if (ref_deg || norm[v + i] == 0.0f) {
      r = __int_as_float(0x7fc00000);   // NaN: degenerate (measures.py:94-100)
    } else if (eq[i]) {
      r = 1.0f;                          // measures.py:102-107
    } else {
      r = (float)fmin(1.0, fmax(-1.0, tot[i]));
    }
    out[v + i - v0] = r;
  }
}

// ---- Pearson of fp64 rows (pearson_rowwise / pearson_against) ----------------
__global__ void pearson_rows_kernel(const double* __restrict__ a, int64_t a_stride,
                                    const double* __restrict__ b, int M, int64_t B,
                                    double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= B) return;
  const double* ar = a + row * a_stride;
  const double* br = b + row * (int64_t)M;
  double sa = 0.0, sb = 0.0;
  for (int m = lane; m < M; m += 32) { sa += ar[m]; sb += br[m]; }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  const double ma = sa / M, mb = sb / M;
  double saa = 0.0, sbb = 0.0, sab = 0.0;
  int eq = 1;
  for (int m = lane; m < M; m += 32) {
    const double x = ar[m] - ma, y = br[m] - mb;
    saa += x * x; sbb += y * y; sab += x * y;
    eq &= (ar[m] == br[m]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    saa += __shfl_xor_sync(0xffffffffu, saa, o);
    sbb += __shfl_xor_sync(0xffffffffu, sbb, o);
    sab += __shfl_xor_sync(0xffffffffu, sab, o);
  }
  eq = __all_sync(0xffffffffu, eq);
  if (lane == 0) {
    double r;
    if (!(saa > 0.0) || !(sbb > 0.0)) {
      r = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      r = sab / sqrt(saa * sbb);
      r = fmin(1.0, fmax(-1.0, r));
      if (eq && r > 1.0 - 1e-9) r = 1.0;
    }
    out[row] = r;
  }
}

// ---- Pearson of vertex pairs from the vertex-major copy ------------------------
__global__ void pearson_pairs_kernel(const float* __restrict__ Xv, int M,
                                     const int64_t* __restrict__ pa,
                                     const int64_t* __restrict__ pb, int64_t n,
                                     double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n) return;
  const float* ar = Xv + pa[p] * (int64_t)M;
  const float* br = Xv + pb[p] * (int64_t)M;
  double sa = 0.0, sb = 0.0;
  for (int m = lane; m < M; m += 32) { sa += ar[m]; sb += br[m]; }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  const double ma = sa / M, mb = sb / M;
  double saa = 0.0, sbb = 0.0, sab = 0.0;
  int eq = 1;
  for (int m = lane; m < M; m += 32) {
    const double x = (double)ar[m] - ma, y = (double)br[m] - mb;
    saa += x * x; sbb += y * y; sab += x * y;
    eq &= (ar[m] == br[m]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    saa += __shfl_xor_sync(0xffffffffu, saa, o);
    sbb += __shfl_xor_sync(0xffffffffu, sbb, o);
    sab += __shfl_xor_sync(0xffffffffu, sab, o);
  }
  eq = __all_sync(0xffffffffu, eq);
  if (lane == 0) {
    double r;
    if (!(saa > 0.0) || !(sbb > 0.0)) {
      r = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      r = fmin(1.0, fmax(-1.0, sab / sqrt(saa * sbb)));
      if (eq && r > 1.0 - 1e-9) r = 1.0;
    }
    out[p] = r;
  }
}

// Rows of M <= 128 * kPairNV members with M % 4 == 0: both rows are loaded ONCE into
// registers (up to 2 x kPairNV 16-byte loads in flight per lane, all issued before any
// is used) and both passes run from registers -- one read of 8 KB per pair at M = 1000
// (the scalar two-pass kernel above re-read the rows and kept one load in flight).
constexpr int kPairNV = 8;
__global__ void __launch_bounds__(256)
pearson_pairs_reg_kernel(const float* __restrict__ Xv, int M, const int64_t* __restrict__ pa,
                         const int64_t* __restrict__ pb, int64_t n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n) return;
  const float4* ar = reinterpret_cast<const float4*>(Xv + pa[p] * (int64_t)M);
  const float4* br = reinterpret_cast<const float4*>(Xv + pb[p] * (int64_t)M);
  const int n4 = M >> 2;
  float4 a[kPairNV], b[kPairNV];
#pragma unroll
  for (int u = 0; u < kPairNV; ++u) {
    const int i = lane + 32 * u;
    a[u] = i < n4 ? __ldg(ar + i) : make_float4(0, 0, 0, 0);
    b[u] = i < n4 ? __ldg(br + i) : make_float4(0, 0, 0, 0);
  }
  double sa = 0.0, sb = 0.0;
#pragma unroll
  for (int u = 0; u < kPairNV; ++u) {       // zero padding adds nothing
    sa += ((double)a[u].x + (double)a[u].y) + ((double)a[u].z + (double)a[u].w);
    sb += ((double)b[u].x + (double)b[u].y) + ((double)b[u].z + (double)b[u].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  const double ma = sa / M, mb = sb / M;
  double saa = 0.0, sbb = 0.0, sab = 0.0;
  int eq = 1;
#pragma unroll
  for (int u = 0; u < kPairNV; ++u) {
    if (lane + 32 * u >= n4) break;
    const float av[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
    const float bv[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double x = (double)av[q] - ma, y = (double)bv[q] - mb;
      saa = fma(x, x, saa);
      sbb = fma(y, y, sbb);
      sab = fma(x, y, sab);
      eq &= (av[q] == bv[q]);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    saa += __shfl_xor_sync(0xffffffffu, saa, o);
    sbb += __shfl_xor_sync(0xffffffffu, sbb, o);
    sab += __shfl_xor_sync(0xffffffffu, sab, o);
  }
  eq = __all_sync(0xffffffffu, eq);
  if (lane == 0) {
    double r;
    if (!(saa > 0.0) || !(sbb > 0.0)) {
      r = __longlong_as_double(0x7ff8000000000000ll);   // degenerate (measures.py:94-100)
    } else {
      r = fmin(1.0, fmax(-1.0, sab / sqrt(saa * sbb)));
      if (eq && r > 1.0 - 1e-9) r = 1.0;                // measures.py:128-131
    }
    out[p] = r;
  }
}

// ---- member-major -> vertex-major transpose (K5) -----------------------------
__global__ void transpose_kernel(const float* __restrict__ X, int M, int64_t V,
                                 float* __restrict__ Xv) {
  __shared__ float tile[32][33];
  const int64_t vb = (int64_t)blockIdx.x * 32;
  const int mb = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int m = mb + r;
    const int64_t v = vb + threadIdx.x;
    if (m < M && v < V) tile[r][threadIdx.x] = X[(int64_t)m * V + v];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t v = vb + r;
    const int m = mb + threadIdx.x;
    if (m < M && v < V) Xv[v * M + m] = tile[threadIdx.x][r];
  }
}

}  // namespace ndf

using namespace ndf;

extern "C" int ndf_sample_many_ld(const float* X, int32_t M, int64_t ld, int64_t col0, int32_t nx,
                                  int32_t ny, int32_t nz, const double* pos, int64_t B, double* out,
                                  void* stream) {
  NDF_REQUIRE(M >= 1 && nx >= 2 && ny >= 2 && nz >= 2, NDF_ERR_PARAMETER,
              "sample_many: need M >= 1 and >= 2 nodes per axis");
  NDF_REQUIRE(B >= 0, NDF_ERR_PARAMETER, "negative batch");
  NDF_REQUIRE(ld >= 1 && col0 >= 0, NDF_ERR_PARAMETER, "bad column window");
  if (B == 0) return NDF_OK;
  NDF_REQUIRE(X && pos && out, NDF_ERR_PARAMETER, "null pointer");
  const int64_t n = B * (int64_t)M;
  const int threads = 256;
  sample_many_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
      X, M, ld, col0, nx, ny, nz, pos, B, out);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_sample_many_vm(const float* Xv, int32_t M, int32_t nx, int32_t ny, int32_t nz,
                                  const double* pos, int64_t B, double* out, void* stream) {
  NDF_REQUIRE(M >= 1 && nx >= 2 && ny >= 2 && nz >= 2, NDF_ERR_PARAMETER,
              "sample_many: need M >= 1 and >= 2 nodes per axis");
  NDF_REQUIRE(B >= 0, NDF_ERR_PARAMETER, "negative batch");
  if (B == 0) return NDF_OK;
  NDF_REQUIRE(Xv && pos && out, NDF_ERR_PARAMETER, "null pointer");
  const int64_t n = B * (int64_t)M;
  const int threads = 256;
  sample_many_vm_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
      Xv, M, nx, ny, nz, pos, B, out);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_sample_many(const float* X, int32_t M, int32_t nx, int32_t ny, int32_t nz,
                               const double* pos, int64_t B, double* out, void* stream) {
  return ndf_sample_many_ld(X, M, (int64_t)nx * ny * nz, 0, nx, ny, nz, pos, B, out, stream);
}

extern "C" int ndf_pearson_field(const float* X, int32_t M, int64_t ld, int64_t col0,
                                 const double* ref_vec, int64_t v0, int64_t v1, float* out,
                                 void* stream) {
  NDF_REQUIRE(M >= 1 && M <= kFieldMaxM, NDF_ERR_UNSUPPORTED,
              "pearson_field: M must be in [1, 8192]");
  NDF_REQUIRE(ld >= 1 && col0 >= 0 && col0 <= v0 && v0 <= v1 && v1 <= col0 + ld,
              NDF_ERR_PARAMETER, "vertex range outside the ensemble's column window");
  if (v0 == v1) return NDF_OK;
  NDF_REQUIRE(X && ref_vec && out, NDF_ERR_PARAMETER, "null pointer");
  void* out_dev = nullptr;
  int st = resolve_output(out, &out_dev);
  if (st) return st;
  void* scratch = nullptr;
  NDF_CUDA_CHECK(scratch_alloc(&scratch, (size_t)M * 12 + 64, as_stream(stream)));
  RefStats* rs = reinterpret_cast<RefStats*>(scratch);
  double* rc = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(scratch) + 64);
  float* r32 = reinterpret_cast<float*>(rc + M);
  pearson_ref_kernel<<<1, 1024, 0, as_stream(stream)>>>(ref_vec, M, rc, r32, rs);
  cudaError_t e = cudaGetLastError();
  count_launch();
  if (e == cudaSuccess) {
    const int threads = 256;
    const int64_t nthreads = (v1 - v0 + 3) / 4;
    const unsigned blocks = (unsigned)((nthreads + threads - 1) / threads);
    const size_t smem = (size_t)M * 12;
    const bool vec = (ld % 4 == 0) && ((v0 - col0) % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    static SmemAttrCache attr;
    e = attr.ensure(pearson_field_kernel<true>, (size_t)kFieldMaxM * 12);
    if (e == cudaSuccess) e = attr.ensure(pearson_field_kernel<false>, (size_t)kFieldMaxM * 12);
    if (e == cudaSuccess) {
      if (vec)
        pearson_field_kernel<true><<<blocks, threads, smem, as_stream(stream)>>>(
            X, M, ld, col0, rc, r32, rs, v0, v1, static_cast<float*>(out_dev));
      else
        pearson_field_kernel<false><<<blocks, threads, smem, as_stream(stream)>>>(
            X, M, ld, col0, rc, r32, rs, v0, v1, static_cast<float*>(out_dev));
      e = cudaGetLastError();
      count_launch();
    }
  }
  cudaFreeAsync(scratch, as_stream(stream));
  NDF_CUDA_CHECK(e);
  return NDF_OK;
}

extern "C" int ndf_zscore(const float* X, int32_t M, int64_t V, int64_t v0, int64_t v1,
                          float* Z, float* norm, void* stream) {
  NDF_REQUIRE(M >= 1 && V >= 1, NDF_ERR_PARAMETER, "zscore: empty ensemble");
  NDF_REQUIRE(v0 >= 0 && v0 <= v1 && v1 <= V, NDF_ERR_PARAMETER, "vertex range out of bounds");
  if (v0 == v1) return NDF_OK;
  NDF_REQUIRE(X && Z, NDF_ERR_PARAMETER, "null pointer");
  const bool bulk = V % 4 == 0 && v0 % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(Z) & 15) == 0;
  if (bulk) {
    const int64_t groups = (v1 - v0 + kZCols - 1) / kZCols;
    const int64_t grid = std::min<int64_t>(groups, (int64_t)sm_count() * kZBlocksPerSM);
    zscore_kernel<<<(unsigned)grid, kZThreads, 0, as_stream(stream)>>>(X, M, V, v0, v1, Z, norm);
  } else {
    const int threads = 256;
    zscore_lsu_kernel<<<(unsigned)((v1 - v0 + threads - 1) / threads), threads, 0,
                        as_stream(stream)>>>(X, M, V, v0, v1, Z, norm);
  }
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_pearson_gemv(const float* Z, const float* norm, int32_t M, int64_t V,
                                const float* z_ref, int32_t ref_degenerate, int64_t v0,
                                int64_t v1, float* out, void* stream) {
  NDF_REQUIRE(M >= 1 && M <= 12288, NDF_ERR_UNSUPPORTED, "pearson_gemv: M must be in [1, 12288]");
  NDF_REQUIRE(v0 >= 0 && v0 <= v1 && v1 <= V, NDF_ERR_PARAMETER, "vertex range out of bounds");
  if (v0 == v1) return NDF_OK;
  NDF_REQUIRE(Z && norm && z_ref && out, NDF_ERR_PARAMETER, "null pointer");
  const int threads = 256;
  const int64_t nthreads = (v1 - v0 + 3) / 4;
  const unsigned blocks = (unsigned)((nthreads + threads - 1) / threads);
  const size_t smem = sizeof(float) * M;
  const bool vec = (V % 4 == 0) && (v0 % 4 == 0) && ((reinterpret_cast<uintptr_t>(Z) & 15) == 0);
  if (vec)
    gemv_kernel<true><<<blocks, threads, smem, as_stream(stream)>>>(Z, norm, M, V, z_ref,
                                                                    ref_degenerate, v0, v1, out);
  else
    gemv_kernel<false><<<blocks, threads, smem, as_stream(stream)>>>(Z, norm, M, V, z_ref,
                                                                     ref_degenerate, v0, v1, out);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_pearson_rows(const double* a, int64_t a_stride, const double* b, int32_t M,
                                int64_t B, double* out, void* stream) {
  NDF_REQUIRE(M >= 2, NDF_ERR_PARAMETER, "need at least two samples");
  NDF_REQUIRE(B >= 0, NDF_ERR_PARAMETER, "negative batch");
  if (B == 0) return NDF_OK;
  NDF_REQUIRE(a && b && out, NDF_ERR_PARAMETER, "null pointer");
  const int threads = 256;
  pearson_rows_kernel<<<(unsigned)((B * 32 + threads - 1) / threads), threads, 0,
                        as_stream(stream)>>>(a, a_stride, b, M, B, out);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_pearson_pairs(const float* Xv, int32_t M, int64_t V, const int64_t* pa,
                                 const int64_t* pb, int64_t n, double* out, void* stream) {
  NDF_REQUIRE(M >= 2, NDF_ERR_PARAMETER, "need at least two samples");
  NDF_REQUIRE(n >= 0 && V >= 1, NDF_ERR_PARAMETER, "bad sizes");
  if (n == 0) return NDF_OK;
  NDF_REQUIRE(Xv && pa && pb && out, NDF_ERR_PARAMETER, "null pointer");
  const int threads = 256;
  const unsigned blocks = (unsigned)((n * 32 + threads - 1) / threads);
  if (M % 4 == 0 && M <= 128 * kPairNV && (reinterpret_cast<uintptr_t>(Xv) & 15) == 0)
    pearson_pairs_reg_kernel<<<blocks, threads, 0, as_stream(stream)>>>(Xv, M, pa, pb, n, out);
  else
    pearson_pairs_kernel<<<blocks, threads, 0, as_stream(stream)>>>(Xv, M, pa, pb, n, out);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

extern "C" int ndf_vertex_major(const float* X, int32_t M, int64_t V, float* Xv, void* stream) {
  NDF_REQUIRE(M >= 1 && V >= 1, NDF_ERR_PARAMETER, "empty ensemble");
  NDF_REQUIRE(X && Xv, NDF_ERR_PARAMETER, "null pointer");
  NDF_REQUIRE(M <= 65535 * 32, NDF_ERR_UNSUPPORTED, "too many members");
  dim3 grid((unsigned)((V + 31) / 32), (unsigned)((M + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(X, M, V, Xv);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}
