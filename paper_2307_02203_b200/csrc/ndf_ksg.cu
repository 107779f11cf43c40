// KSG mutual information (K4), variant 1 with max-norm, bit-exact counts.
//
// Restates measures.ksg_mi (measures.py:173-203) per pair (a, b):
//   a' = a + r*(1e-10*ptp(a)), b' likewise, r = _tie_jitter(M)   (measures.py:190-192)
//   eps_i = (k+1)-th smallest max(|a'_i-a'_j|, |b'_i-b'_j|) over all j incl. self
//          == the cKDTree query of k+1 neighbours, p=inf       (measures.py:193-195)
//   n_x(i) = #{j : fl(a'_i - eps) < a'_j < fl(a'_i + eps)} - 1  (searchsorted, :196-201)
//   MI = (psi(k) + psi(M)) - mean(psi(n_x+1) + psi(n_y+1))      (:202-203)
// All fp64 basic ops are explicitly rounded (no FMA contraction) so distances,
// eps and the interval ends are the reference's bits; the k-th order statistic
// is taken by exact comparisons, so n_x / n_y are bit-exact.  psi comes from a
// host table built with the reference formula and the mean uses NumPy's
// pairwise summation order, so MI is reproduced bit for bit as well.
//
// One CTA per pair; the jittered vectors and their sorted copies live in SMEM;
// each thread keeps the running (k+1)-smallest distances of 4 points in
// registers while streaming all j from SMEM (broadcast reads).
#include <algorithm>

#include "ndf_common.cuh"

namespace ndf {

constexpr int kKsgThreads = 256;
constexpr int kKsgPts = 4;          // points per thread per sweep

struct KsgArgs {
  int mode;                   // 0 ref-vs-node-columns, 1 fp64 rows, 2 vertex-major pairs
  int M;
  int64_t V;
  const float* X;             // mode 0: member-major (M, V); mode 2: vertex-major (V, M)
  const double* ref;          // mode 0
  int64_t v0;                 // mode 0
  const double* A;            // mode 1
  int64_t a_stride;
  const double* B;
  const int64_t* pa;          // mode 2
  const int64_t* pb;
  int64_t n;                  // pairs
  int k;
  const double* jit;
  const double* psi;
  double psi_km;
  double* mi;
  float* mi_f32;
  int32_t* counts;
  int32_t* status;
  int P;                      // pow2 >= M (sort width)
};

// NumPy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum) -- the order np.mean uses on a contiguous fp64 array.
__device__ double pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = dadd(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], a[i + j]);
    }
    double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                      dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
    for (; i < n; ++i) res = dadd(res, a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return dadd(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

__device__ __forceinline__ int lower_bound_lt(const double* s, int P, double x) {
  // number of elements < x (searchsorted side="left")
  int lo = 0;
  for (int step = P >> 1; step > 0; step >>= 1)
    if (s[lo + step - 1] < x) lo += step;
  if (lo < P && s[lo] < x) ++lo;
  return lo;
}

__device__ __forceinline__ int upper_bound_le(const double* s, int P, double x) {
  // number of elements <= x (searchsorted side="right")
  int lo = 0;
  for (int step = P >> 1; step > 0; step >>= 1)
    if (s[lo + step - 1] <= x) lo += step;
  if (lo < P && s[lo] <= x) ++lo;
  return lo;
}

__device__ void bitonic_sort2(double* a, double* b, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        double x = a[lo], y = a[hi];
        if ((x > y) == up) { a[lo] = y; a[hi] = x; }
        x = b[lo]; y = b[hi];
        if ((x > y) == up) { b[lo] = y; b[hi] = x; }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ double block_reduce(double v, bool is_max, double* scratch) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : fmin(v, w);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? scratch[lane] : (is_max ? -INFINITY : INFINITY);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmax(v, w) : fmin(v, w);
    }
    if (lane == 0) scratch[0] = v;
  }
  __syncthreads();
  v = scratch[0];
  __syncthreads();
  return v;
}

template <int KP1>
__global__ void __launch_bounds__(kKsgThreads)
ksg_kernel(const KsgArgs g) {
  extern __shared__ __align__(16) double sm[];
  const int M = g.M, P = g.P;
  double* aj = sm;
  double* bj = aj + M;
  double* sa = bj + M;
  double* sb = sa + P;
  double* terms = sb + P;
  double* scratch = terms + M;      // 32 doubles
  __shared__ int bad_flag;

  for (int64_t p = blockIdx.x; p < g.n; p += gridDim.x) {
    // ---- load (fp32 node values are exact in fp64) --------------------------
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      double a, b;
      if (g.mode == 0) {
        a = g.ref[i];
        b = (double)__ldg(g.X + (int64_t)i * g.V + (g.v0 + p));
      } else if (g.mode == 1) {
        a = g.A[p * g.a_stride + i];
        b = g.B[p * (int64_t)M + i];
      } else {
        a = (double)__ldg(g.X + g.pa[p] * (int64_t)M + i);
        b = (double)__ldg(g.X + g.pb[p] * (int64_t)M + i);
      }
      aj[i] = a;
      bj[i] = b;
    }
    if (threadIdx.x == 0) bad_flag = 0;
    __syncthreads();
    // ---- ptp + jitter ----------------------------------------------------------
    double amin = INFINITY, amax = -INFINITY, bmin = INFINITY, bmax = -INFINITY;
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      amin = fmin(amin, aj[i]); amax = fmax(amax, aj[i]);
      bmin = fmin(bmin, bj[i]); bmax = fmax(bmax, bj[i]);
    }
    amin = block_reduce(amin, false, scratch);
    amax = block_reduce(amax, true, scratch);
    bmin = block_reduce(bmin, false, scratch);
    bmax = block_reduce(bmax, true, scratch);
    const double sca = dmul(1e-10, dsub(amax, amin));
    const double scb = dmul(1e-10, dsub(bmax, bmin));
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < M) {
        const double r = g.jit[i];
        const double x = dadd(aj[i], dmul(r, sca));
        const double y = dadd(bj[i], dmul(r, scb));
        aj[i] = x; bj[i] = y;
        sa[i] = x; sb[i] = y;
      } else {
        sa[i] = INFINITY; sb[i] = INFINITY;
      }
    }
    __syncthreads();
    bitonic_sort2(sa, sb, P);
    // ---- k-NN in max-norm: (k+1) smallest incl. self --------------------------
    for (int i0 = threadIdx.x; i0 < M; i0 += kKsgPts * blockDim.x) {
      double xi[kKsgPts], yi[kKsgPts], top[kKsgPts][KP1];
#pragma unroll
      for (int q = 0; q < kKsgPts; ++q) {
        const int i = i0 + q * blockDim.x;
        xi[q] = i < M ? aj[i] : 0.0;
        yi[q] = i < M ? bj[i] : 0.0;
#pragma unroll
        for (int s = 0; s < KP1; ++s) top[q][s] = INFINITY;
      }
      for (int j = 0; j < M; ++j) {
        const double xj = aj[j], yj = bj[j];
#pragma unroll
        for (int q = 0; q < kKsgPts; ++q) {
          const double d = fmax(fabs(dsub(xi[q], xj)), fabs(dsub(yi[q], yj)));
          if (d < top[q][KP1 - 1]) {
#pragma unroll
            for (int s = KP1 - 1; s > 0; --s)
              top[q][s] = d < top[q][s - 1] ? top[q][s - 1] : fmin(d, top[q][s]);
            top[q][0] = fmin(d, top[q][0]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kKsgPts; ++q) {
        const int i = i0 + q * blockDim.x;
        if (i >= M) continue;
        const double eps = top[q][KP1 - 1];
        const int nx = lower_bound_lt(sa, P, dadd(xi[q], eps)) -
                       upper_bound_le(sa, P, dsub(xi[q], eps)) - 1;
        const int ny = lower_bound_lt(sb, P, dadd(yi[q], eps)) -
                       upper_bound_le(sb, P, dsub(yi[q], eps)) - 1;
        if (g.counts) {
          g.counts[(p * 2) * (int64_t)M + i] = nx;
          g.counts[(p * 2 + 1) * (int64_t)M + i] = ny;
        }
        if (nx < 0 || ny < 0) {
          bad_flag = 1;
          terms[i] = __longlong_as_double(0x7ff8000000000000ll);
        } else {
          terms[i] = dadd(g.psi[nx], g.psi[ny]);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double mean = ddiv(pairwise_sum(terms, M), (double)M);
      const double mi = dsub(g.psi_km, mean);
      if (g.mi) g.mi[p] = mi;
      if (g.mi_f32) g.mi_f32[p] = (float)mi;
      if (bad_flag && g.status) atomicExch(g.status, 1);
    }
    __syncthreads();
  }
}

size_t ksg_smem_bytes(int M, int P) { return sizeof(double) * (3 * (size_t)M + 2 * P + 32); }

template <int KP1>
static int launch_ksg_t(const KsgArgs& g, cudaStream_t s) {
  const size_t smem = ksg_smem_bytes(g.M, g.P);
  NDF_CUDA_CHECK(cudaFuncSetAttribute(ksg_kernel<KP1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  NDF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ksg_kernel<KP1>,
                                                               kKsgThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(g.n, (int64_t)sm_count() * per_sm * 16);
  ksg_kernel<KP1><<<(unsigned)grid, kKsgThreads, smem, s>>>(g);
  NDF_LAUNCH_CHECK();
  return NDF_OK;
}

static int launch_ksg(KsgArgs g, cudaStream_t s) {
  NDF_REQUIRE(g.M >= 2, NDF_ERR_PARAMETER, "KSG needs at least two samples");
  NDF_REQUIRE(g.k >= 1 && g.k <= g.M - 1, NDF_ERR_PARAMETER, "need 1 <= k <= N-1");
  NDF_REQUIRE(g.k <= 16, NDF_ERR_UNSUPPORTED, "GPU KSG supports k <= 16");
  NDF_REQUIRE(g.M <= 4096, NDF_ERR_UNSUPPORTED, "GPU KSG supports M <= 4096 members");
  NDF_REQUIRE(g.jit && g.psi, NDF_ERR_PARAMETER, "null jitter / psi table");
  if (g.n == 0) return NDF_OK;
  int P = 1;
  while (P < g.M) P <<= 1;
  g.P = P;
  switch (g.k + 1) {
    case 2: return launch_ksg_t<2>(g, s);
    case 3: return launch_ksg_t<3>(g, s);
    case 4: return launch_ksg_t<4>(g, s);
    case 5: return launch_ksg_t<5>(g, s);
    case 6: return launch_ksg_t<6>(g, s);
    case 7: return launch_ksg_t<7>(g, s);
    case 8: return launch_ksg_t<8>(g, s);
    case 9: return launch_ksg_t<9>(g, s);
    case 10: return launch_ksg_t<10>(g, s);
    case 11: return launch_ksg_t<11>(g, s);
    case 12: return launch_ksg_t<12>(g, s);
    case 13: return launch_ksg_t<13>(g, s);
    case 14: return launch_ksg_t<14>(g, s);
    case 15: return launch_ksg_t<15>(g, s);
    case 16: return launch_ksg_t<16>(g, s);
    default: return launch_ksg_t<17>(g, s);
  }
}

}  // namespace ndf

using namespace ndf;

extern "C" int ndf_ksg_ref_nodes(const float* X, int32_t M, int64_t V, const double* ref_vec,
                                 int64_t v0, int64_t v1, int32_t k, const double* jitter_r,
                                 const double* psi_tab, double psi_km, double* mi, float* mi_f32,
                                 int32_t* counts, int32_t* status_out, void* stream) {
  NDF_REQUIRE(v0 >= 0 && v0 <= v1 && v1 <= V, NDF_ERR_PARAMETER, "vertex range out of bounds");
  NDF_REQUIRE(X && ref_vec, NDF_ERR_PARAMETER, "null pointer");
  KsgArgs g{};
  g.mode = 0; g.M = M; g.V = V; g.X = X; g.ref = ref_vec; g.v0 = v0; g.n = v1 - v0;
  g.k = k; g.jit = jitter_r; g.psi = psi_tab; g.psi_km = psi_km;
  g.mi = mi; g.mi_f32 = mi_f32; g.counts = counts; g.status = status_out;
  return launch_ksg(g, as_stream(stream));
}

extern "C" int ndf_ksg_rows(const double* a, int64_t a_stride, const double* b, int32_t M,
                            int64_t B, int32_t k, const double* jitter_r, const double* psi_tab,
                            double psi_km, double* mi, float* mi_f32, int32_t* counts,
                            int32_t* status_out, void* stream) {
  NDF_REQUIRE(B >= 0, NDF_ERR_PARAMETER, "negative batch");
  NDF_REQUIRE(B == 0 || (a && b), NDF_ERR_PARAMETER, "null pointer");
  KsgArgs g{};
  g.mode = 1; g.M = M; g.A = a; g.a_stride = a_stride; g.B = b; g.n = B;
  g.k = k; g.jit = jitter_r; g.psi = psi_tab; g.psi_km = psi_km;
  g.mi = mi; g.mi_f32 = mi_f32; g.counts = counts; g.status = status_out;
  return launch_ksg(g, as_stream(stream));
}

extern "C" int ndf_ksg_pairs(const float* Xv, int32_t M, int64_t V, const int64_t* pa,
                             const int64_t* pb, int64_t n, int32_t k, const double* jitter_r,
                             const double* psi_tab, double psi_km, double* mi, float* mi_f32,
                             int32_t* counts, int32_t* status_out, void* stream) {
  NDF_REQUIRE(n >= 0, NDF_ERR_PARAMETER, "negative batch");
  NDF_REQUIRE(n == 0 || (Xv && pa && pb), NDF_ERR_PARAMETER, "null pointer");
  KsgArgs g{};
  g.mode = 2; g.M = M; g.V = V; g.X = Xv; g.pa = pa; g.pb = pb; g.n = n;
  g.k = k; g.jit = jitter_r; g.psi = psi_tab; g.psi_km = psi_km;
  g.mi = mi; g.mi_f32 = mi_f32; g.counts = counts; g.status = status_out;
  return launch_ksg(g, as_stream(stream));
}
