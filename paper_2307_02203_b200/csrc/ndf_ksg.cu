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
// One CTA per pair.  The jittered vectors live in SMEM sorted by a' (with b' in the
// same order) and b' sorted on its own.  Each point's (k+1)-NN scan walks outward
// in a'-order from its own position and stops once |a'_i - a'_j| alone reaches the
// running (k+1)-th distance -- typically ~sqrt(kM) candidates instead of M -- and
// the marginal counts are two binary searches per axis.  For reference-vs-all
// fields the jittered reference is sorted once per query (ksg_prep_ref_kernel).
#include <algorithm>

#include "ndf_common.cuh"

namespace ndf {

#ifndef NDF_KSG_THREADS
#define NDF_KSG_THREADS 256
#endif
constexpr int kKsgThreads = NDF_KSG_THREADS;
#ifndef NDF_KSG_PNET
#define NDF_KSG_PNET 1           // compare-vector insertion network (knn_scan)
#endif
#ifndef NDF_KSG_DYN
#define NDF_KSG_DYN 1            // scans handed out per point from a CTA queue
#endif
#ifndef NDF_KSG_ONESCAN
#define NDF_KSG_ONESCAN 1        // one knn_scan call site for both scan axes
#endif

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
  const double* sa_ref;       // mode 0: jittered reference sorted (P, +inf padded)
  const int* perm_ref;        // mode 0: its argsort (P)
};

// NumPy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum) -- the order np.mean uses on a contiguous fp64 array.  Blocks of
// <= 128 are summed 8-way; larger ranges split at n/2 rounded down to a multiple of
// 8.  Evaluated with an explicit stack (no device recursion: a fixed, statically
// known stack frame whatever the register allocation).
__device__ double pairwise_leaf(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = dadd(r, a[i]);
    return r;
  }
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

__device__ double pairwise_sum(const double* a, int n) {
  int off[32], len[32];
  bool right[32];               // frame's left half is done, left[] holds its sum
  double left[32];
  int sp = 0;
  off[0] = 0; len[0] = n; right[0] = false;
  for (;;) {
    // descend along left halves to a leaf
    while (len[sp] > 128) {
      int n2 = len[sp] / 2;
      n2 -= n2 % 8;
      off[sp + 1] = off[sp]; len[sp + 1] = n2; right[sp + 1] = false;
      ++sp;
    }
    double ret = pairwise_leaf(a + off[sp], len[sp]);
    // return upwards: combine finished right halves, or switch to a pending right half
    for (;;) {
      if (sp == 0) return ret;
      --sp;
      if (!right[sp]) {
        left[sp] = ret;
        right[sp] = true;
        int n2 = len[sp] / 2;
        n2 -= n2 % 8;
        off[sp + 1] = off[sp] + n2; len[sp + 1] = len[sp] - n2; right[sp + 1] = false;
        ++sp;
        break;
      }
      ret = dadd(left[sp], ret);
    }
  }
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

// Bitonic sort of P = 2^m keys with an int payload (ascending by key), all in SMEM.
__device__ void bitonic_sort_kv_smem(double* key, int* val, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const double x = key[lo], y = key[hi];
        if ((x > y) == up) {
          key[lo] = y; key[hi] = x;
          const int v = val[lo]; val[lo] = val[hi]; val[hi] = v;
        }
      }
      __syncthreads();
    }
  }
}

// Compare-exchange of this lane's element (global index e, key k, payload v) with its
// partner at e ^ stride held by lane ^ stride (stride <= 16): keep the smaller key if
// the element is the lower of the pair in an ascending run, the larger otherwise.
// Equal keys never move, so the two lanes always keep complementary elements.
__device__ __forceinline__ void bitonic_lane_step(double& k, int& v, int e, int stride, int size) {
  const double pk = __shfl_xor_sync(0xffffffffu, k, stride);
  const int pv = __shfl_xor_sync(0xffffffffu, v, stride);
  const bool take_min = ((e & stride) == 0) == ((e & size) == 0);
  if (take_min ? pk < k : pk > k) { k = pk; v = pv; }
}

// Strides min(size/2, 32) .. 1 of bitonic merge stage(s) `size_lo..size_hi` on 64-element
// segments held in registers (lane holds elements lane and lane + 32 of its segment):
// the sub-64 strides need no shared-memory round trip and no block barrier.
__device__ __forceinline__ void bitonic_segment_phase(double* key, int* val, int P, int size_lo,
                                                      int size_hi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int seg = warp; seg < P / 64; seg += nw) {
    const int e0 = seg * 64 + lane, e1 = e0 + 32;
    double k0 = key[e0], k1 = key[e1];
    int v0 = val[e0], v1 = val[e1];
    for (int size = size_lo; size <= size_hi; size <<= 1) {
      for (int stride = min(size >> 1, 32); stride > 0; stride >>= 1) {
        if (stride == 32) {
          // pair (e0, e1) within the lane; e0 is the lower element
          if ((k0 > k1) == ((e0 & size) == 0)) {
            const double tk = k0; k0 = k1; k1 = tk;
            const int tv = v0; v0 = v1; v1 = tv;
          }
        } else {
          bitonic_lane_step(k0, v0, e0, stride, size);
          bitonic_lane_step(k1, v1, e1, stride, size);
        }
      }
    }
    key[e0] = k0; key[e1] = k1;
    val[e0] = v0; val[e1] = v1;
  }
}

// Same sort with every stride below 64 done in registers (warp shuffles): for P = 1024,
// 10 shared-memory compare-exchange stages and 15 block barriers instead of 55 of each.
// The sorted keys are the same; only the order of equal keys may differ, which no
// consumer observes (ranks, distances and counts depend on values alone).
__device__ void bitonic_sort_kv(double* key, int* val, int P) {
  if (P < 64) {
    bitonic_sort_kv_smem(key, val, P);
    return;
  }
  bitonic_segment_phase(key, val, P, 2, 64);       // sizes 2..64 entirely in registers
  __syncthreads();
  for (int size = 128; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride >= 64; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const double x = key[lo], y = key[hi];
        if ((x > y) == up) {
          key[lo] = y; key[hi] = x;
          const int v = val[lo]; val[lo] = val[hi]; val[hi] = v;
        }
      }
      __syncthreads();
    }
    bitonic_segment_phase(key, val, P, size, size);
    __syncthreads();
  }
}

// (k+1) smallest max-norm distances of point (xi, yi), found at sorted position q
// of an array sorted by x (sx) with the other coordinate in the same order (yx):
// scan outward in |x_i - x_j| order until that alone reaches the running (k+1)-th
// distance.  Every j with |dx| < eps is visited, so the result equals the
// brute-force order statistic.  Self is the 0 in top[0].
template <int KP1>
__device__ __forceinline__ double knn_scan(const double* __restrict__ sx,
                                           const double* __restrict__ yx, int M, int q) {
  const double xi = sx[q], yi = yx[q];
  double top[KP1];
  top[0] = 0.0;
#pragma unroll
  for (int s = 1; s < KP1; ++s) top[s] = INFINITY;
  int l = q - 1, r = q + 1;
  double dl = l >= 0 ? dsub(xi, sx[l]) : INFINITY;      // = |x_i - x_l| exactly
  double dr = r < M ? dsub(sx[r], xi) : INFINITY;
  for (;;) {
    const bool left = dl <= dr;
    const double dx = left ? dl : dr;
    if (!(dx < top[KP1 - 1])) break;
    const int j = left ? l : r;
    const double d = fmax(dx, fabs(dsub(yi, yx[j])));
#if NDF_KSG_PNET
    // sorted insert from the comparison vector p[s] = d < top[s] (monotone in s, as top
    // is sorted): slot s takes top[s-1] if d belongs below it, d if it belongs exactly
    // here; plain compares + selects (no fmin NaN canonicalisation), same values as the
    // fmin form for every non-NaN d, and a NaN d compares false and changes nothing
    bool pl[KP1];
#pragma unroll
    for (int s = 1; s < KP1; ++s) pl[s] = d < top[s];
#pragma unroll
    for (int s = KP1 - 1; s > 1; --s) top[s] = pl[s - 1] ? top[s - 1] : (pl[s] ? d : top[s]);
    top[1] = pl[1] ? d : top[1];
#else
    if (d < top[KP1 - 1]) {
      // sorted insert; top[0] is the point itself (distance 0 <= d) and never moves
#pragma unroll
      for (int s = KP1 - 1; s > 1; --s) top[s] = d < top[s - 1] ? top[s - 1] : fmin(d, top[s]);
      top[1] = fmin(d, top[1]);
    }
#endif
    if (left) { --l; dl = l >= 0 ? dsub(xi, sx[l]) : INFINITY; }
    else { ++r; dr = r < M ? dsub(sx[r], xi) : INFINITY; }
  }
  return top[KP1 - 1];
}

// Distance from sorted position q to its k-th nearest neighbour along one axis
// (a lower bound of the max-norm k-NN radius).
__device__ __forceinline__ double kth_gap_1d(const double* __restrict__ s, int M, int q, int k) {
  int l = q - 1, r = q + 1;
  double d = 0.0;
  for (int c = 0; c < k; ++c) {
    const double dl = l >= 0 ? dsub(s[q], s[l]) : INFINITY;
    const double dr = r < M ? dsub(s[r], s[q]) : INFINITY;
    if (dl <= dr) { d = dl; --l; } else { d = dr; ++r; }
  }
  return d;
}

__device__ __forceinline__ int lower_bound_lt(const double* s, int P, double x);
__device__ __forceinline__ int upper_bound_le(const double* s, int P, double x);

// Candidates a scan along an axis would visit at radius lb (points with |d| < lb).
__device__ __forceinline__ int strip_count(const double* s, int P, double c, double lb) {
  return lower_bound_lt(s, P, dadd(c, lb)) - upper_bound_le(s, P, dsub(c, lb));
}

// Reference mode prep: jitter + sort the fixed reference vector once per query.
__global__ void ksg_prep_ref_kernel(const double* __restrict__ ref, const double* __restrict__ jit,
                                    int M, int P, double* sa_out, int* perm_out) {
  extern __shared__ __align__(16) double sm[];
  double* key = sm;
  int* val = reinterpret_cast<int*>(key + P);
  double* scratch = reinterpret_cast<double*>(val + P + (P & 1));
  double amin = INFINITY, amax = -INFINITY;
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    amin = fmin(amin, ref[i]);
    amax = fmax(amax, ref[i]);
  }
  amin = block_reduce(amin, false, scratch);
  amax = block_reduce(amax, true, scratch);
  const double sc = dmul(1e-10, dsub(amax, amin));
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    key[i] = i < M ? dadd(ref[i], dmul(jit[i], sc)) : INFINITY;
    val[i] = i < M ? i : M;
  }
  __syncthreads();
  bitonic_sort_kv(key, val, P);
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    sa_out[i] = key[i];
    perm_out[i] = val[i];
  }
}

#ifndef NDF_KSG_MINBLOCKS
#define NDF_KSG_MINBLOCKS 4      // 4 CTAs (32 warps) per SM at M = 1000 (64 registers)
#endif
template <int KP1>
__global__ void __launch_bounds__(kKsgThreads, NDF_KSG_MINBLOCKS)
ksg_kernel(const KsgArgs g) {
  extern __shared__ __align__(16) double sm[];
  const int M = g.M, P = g.P;
  // 48 P + 8 M bytes (56 KB at M = 1000): 4 CTAs (32 warps) per SM
  double* sa = sm;                 // a' sorted ascending (P, +inf padded)
  double* bsa = sa + P;            // b' in a'-order
  double* sb = bsa + P;            // b' sorted ascending (P, +inf padded)
  double* asb = sb + P;            // a' in b'-order
  double* terms = asb + P;         // psi(n_x+1) + psi(n_y+1), original order (M)
  double* scratch = terms;         // block reductions (before terms is written)
  int* pa = reinterpret_cast<int*>(terms + M);      // a'-sorted position -> original index
  int* pb = pa + P;                                  // b'-sorted position -> original index
  int* posa = pb + P;                                // original index -> a'-sorted position
  int* posb = posa + P;                              // original index -> b'-sorted position
  __shared__ int bad_flag;
  __shared__ int work_next;                          // NDF_KSG_DYN scan queue
  const int k = KP1 - 1;

  for (int64_t p = blockIdx.x; p < g.n; p += gridDim.x) {
    // ---- load, original order (fp32 node values are exact in fp64) -------------------
    // mode 0: a' is the reference, already jittered and sorted (ksg_prep_ref_kernel)
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      if (g.mode == 0) {
        sa[i] = g.sa_ref[i];
        pa[i] = g.perm_ref[i];
      }
      if (i < M) {
        if (g.mode == 0) {
          sb[i] = (double)__ldg(g.X + (int64_t)i * g.V + (g.v0 + p));
        } else if (g.mode == 1) {
          sa[i] = g.A[p * g.a_stride + i];
          sb[i] = g.B[p * (int64_t)M + i];
        } else {
          sa[i] = (double)__ldg(g.X + g.pa[p] * (int64_t)M + i);
          sb[i] = (double)__ldg(g.X + g.pb[p] * (int64_t)M + i);
        }
      }
    }
    if (threadIdx.x == 0) bad_flag = 0;
    __syncthreads();
    // ---- ptp + jitter (measures.py:190-192) -------------------------------------
    double bmin = INFINITY, bmax = -INFINITY, amin = INFINITY, amax = -INFINITY;
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      bmin = fmin(bmin, sb[i]); bmax = fmax(bmax, sb[i]);
      if (g.mode != 0) { amin = fmin(amin, sa[i]); amax = fmax(amax, sa[i]); }
    }
    bmin = block_reduce(bmin, false, scratch);
    bmax = block_reduce(bmax, true, scratch);
    const double scb = dmul(1e-10, dsub(bmax, bmin));
    double sca = 0.0;
    if (g.mode != 0) {
      amin = block_reduce(amin, false, scratch);
      amax = block_reduce(amax, true, scratch);
      sca = dmul(1e-10, dsub(amax, amin));
    }
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < M) {
        sb[i] = dadd(sb[i], dmul(g.jit[i], scb));
        pb[i] = i;
        if (g.mode != 0) {
          sa[i] = dadd(sa[i], dmul(g.jit[i], sca));
          pa[i] = i;
        }
      } else {
        sb[i] = INFINITY;
        pb[i] = M;
        if (g.mode != 0) { sa[i] = INFINITY; pa[i] = M; }
      }
    }
    __syncthreads();
    if (g.mode != 0) bitonic_sort_kv(sa, pa, P);
    bitonic_sort_kv(sb, pb, P);      // ends with __syncthreads
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
      posa[pa[q]] = q;
      posb[pb[q]] = q;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < P; q += blockDim.x) {
      bsa[q] = q < M ? sb[posb[pa[q]]] : 0.0;
      asb[q] = q < M ? sa[posa[pb[q]]] : 0.0;
    }
    __syncthreads();
    // ---- k-NN (exact, scanned along the sparser axis) + marginal counts ------------
#if NDF_KSG_DYN
    // (a) per point: the scan axis (uniform work per point);
    //     posa is free now and holds (axis << 30 | sorted position) per a'-position q
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
      const int i = pa[q];
      const int qb = posb[i];
      const double xi = sa[q], yi = bsa[q];
#ifndef NDF_KSG_STRIPAXIS
      // the axis whose k-th 1-D gap is larger is locally sparser (fewer candidates per
      // unit of radius); any choice gives the same eps -- this only steers the work.
      // Measured +7% over counting both strips at the lower bound (4 binary searches).
      const double ga = kth_gap_1d(sa, M, q, k), gb = kth_gap_1d(sb, M, qb, k);
      const bool along_b = gb > ga;
      (void)xi; (void)yi;
#else
      const double lb = fmax(kth_gap_1d(sa, M, q, k), kth_gap_1d(sb, M, qb, k));
      const bool along_b = strip_count(sb, P, yi, lb) < strip_count(sa, P, xi, lb);
#endif
      posa[q] = along_b ? (qb | (1 << 30)) : q;
    }
    if (threadIdx.x == 0) work_next = 0;
    __syncthreads();
    // (b) the scans, points handed out one at a time from a CTA counter: a lane whose
    //     point is done takes the next one, so a warp's lanes stay busy instead of
    //     waiting for the longest of 32 fixed points; eps -> terms[q]
    {
      int q = atomicAdd(&work_next, 1);
      const double* sx = sa;
      const double* yx = bsa;
      double xi = 0.0, yi = 0.0, dl = INFINITY, dr = INFINITY;
      int l = 0, r = 0;
      double top[KP1];
      auto begin = [&]() {
        const int info = posa[q];
        const int pos = info & ((1 << 30) - 1);
        const bool ab = (info >> 30) != 0;
        sx = ab ? sb : sa;
        yx = ab ? asb : bsa;
        xi = sx[pos];
        yi = yx[pos];
        top[0] = 0.0;
#pragma unroll
        for (int t = 1; t < KP1; ++t) top[t] = INFINITY;
        l = pos - 1;
        r = pos + 1;
        dl = l >= 0 ? dsub(xi, sx[l]) : INFINITY;       // = |x_i - x_l| exactly
        dr = r < M ? dsub(sx[r], xi) : INFINITY;
      };
      if (q < M) begin();
      while (q < M) {
        const bool left = dl <= dr;
        const double dx = left ? dl : dr;
        if (!(dx < top[KP1 - 1])) {                      // every j with d < eps visited
          terms[q] = top[KP1 - 1];
          q = atomicAdd(&work_next, 1);
          if (q < M) begin();
          continue;
        }
        const int j = left ? l : r;
        const double d = fmax(dx, fabs(dsub(yi, yx[j])));
        bool pl[KP1];                                    // insertion network as knn_scan
#pragma unroll
        for (int t = 1; t < KP1; ++t) pl[t] = d < top[t];
#pragma unroll
        for (int t = KP1 - 1; t > 1; --t) top[t] = pl[t - 1] ? top[t - 1] : (pl[t] ? d : top[t]);
        top[1] = pl[1] ? d : top[1];
        if (left) { --l; dl = l >= 0 ? dsub(xi, sx[l]) : INFINITY; }
        else { ++r; dr = r < M ? dsub(sx[r], xi) : INFINITY; }
      }
    }
    __syncthreads();
    // (c) marginal counts per point; the psi terms go to ftm (posa / posb, free now) in
    //     original order for the pairwise mean
    double* ftm = reinterpret_cast<double*>(posa);
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
      const int i = pa[q];
      const double xi = sa[q], yi = bsa[q], eps = terms[q];
      const int nx = lower_bound_lt(sa, P, dadd(xi, eps)) - upper_bound_le(sa, P, dsub(xi, eps)) - 1;
      const int ny = lower_bound_lt(sb, P, dadd(yi, eps)) - upper_bound_le(sb, P, dsub(yi, eps)) - 1;
      if (g.counts) {
        g.counts[(p * 2) * (int64_t)M + i] = nx;
        g.counts[(p * 2 + 1) * (int64_t)M + i] = ny;
      }
      if (nx < 0 || ny < 0) {
        bad_flag = 1;
        ftm[i] = __longlong_as_double(0x7ff8000000000000ll);
      } else {
        ftm[i] = dadd(g.psi[nx], g.psi[ny]);
      }
    }
    __syncthreads();
    const double* tsum = ftm;
#else
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
      const int i = pa[q];
      const int qb = posb[i];
      const double xi = sa[q], yi = bsa[q];
      // lower bound of eps; scan the axis whose strip at that radius is thinner
      const double lb = fmax(kth_gap_1d(sa, M, q, k), kth_gap_1d(sb, M, qb, k));
      const bool along_b = strip_count(sb, P, yi, lb) < strip_count(sa, P, xi, lb);
#if NDF_KSG_ONESCAN
      // one scan loop for both axes (operands selected per lane): lanes of a warp that
      // chose different axes no longer run two loops one after the other
#ifdef NDF_EXP_KSG_NOSCAN   // timing experiment: eps = the lower bound (wrong results)
      const double eps = lb + 0.0 * (double)along_b;
#else
      const double eps = knn_scan<KP1>(along_b ? sb : sa, along_b ? asb : bsa, M,
                                       along_b ? qb : q);
#endif
#else
      const double eps = along_b ? knn_scan<KP1>(sb, asb, M, qb) : knn_scan<KP1>(sa, bsa, M, q);
#endif
      const int nx = lower_bound_lt(sa, P, dadd(xi, eps)) - upper_bound_le(sa, P, dsub(xi, eps)) - 1;
      const int ny = lower_bound_lt(sb, P, dadd(yi, eps)) - upper_bound_le(sb, P, dsub(yi, eps)) - 1;
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
    __syncthreads();
    const double* tsum = terms;
#endif
    if (threadIdx.x == 0) {
      const double mean = ddiv(pairwise_sum(tsum, M), (double)M);
      const double mi = dsub(g.psi_km, mean);
      if (g.mi) g.mi[p] = mi;
      if (g.mi_f32) g.mi_f32[p] = (float)mi;
      if (bad_flag && g.status) atomicExch(g.status, 1);
    }
    __syncthreads();
  }
}

size_t ksg_smem_bytes(int M, int P) {
  return sizeof(double) * (4 * (size_t)P + (size_t)std::max(M, 32)) + sizeof(int) * 4 * (size_t)P;
}

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

static int launch_ksg_body(KsgArgs g, cudaStream_t s);

static int launch_ksg(KsgArgs g, cudaStream_t s) {
  void* scratch = nullptr;
  int st = NDF_OK;
  if (g.mode == 0 && g.n > 0 && g.M >= 2 && g.M <= 4096) {
    int P = 1;
    while (P < g.M) P <<= 1;
    NDF_CUDA_CHECK(scratch_alloc(&scratch, (size_t)P * (sizeof(double) + sizeof(int)), s));
    g.sa_ref = reinterpret_cast<double*>(scratch);
    g.perm_ref = reinterpret_cast<int*>(reinterpret_cast<double*>(scratch) + P);
    const size_t smem = (size_t)P * (sizeof(double) + sizeof(int)) + 8 + 32 * sizeof(double);
    NDF_CUDA_CHECK(cudaFuncSetAttribute(ksg_prep_ref_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ksg_prep_ref_kernel<<<1, kKsgThreads, smem, s>>>(g.ref, g.jit, g.M, P,
                                                     const_cast<double*>(g.sa_ref),
                                                     const_cast<int*>(g.perm_ref));
    NDF_LAUNCH_CHECK();
  }
  st = launch_ksg_body(g, s);
  if (scratch) cudaFreeAsync(scratch, s);
  return st;
}

static int launch_ksg_body(KsgArgs g, cudaStream_t s) {
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
