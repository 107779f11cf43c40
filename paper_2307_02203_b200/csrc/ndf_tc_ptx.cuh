// Thin inline-PTX wrappers for sm_100a: mbarrier, bulk copy, tcgen05 (MMA, TMEM).
#pragma once
#include "ndf_common.cuh"

namespace ndf {
namespace tc {

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef NDF_MBAR_HINT
#define NDF_MBAR_HINT 1000000
#endif
#if NDF_MBAR_HINT > 0
// try_wait with a suspend-time hint (ns): the waiting warp sleeps (NANOSLEEP.SYNCS) until
// the phase completes instead of re-polling, leaving issue slots to the working warps
// (query_pp_kernel: 0.2998 -> 0.2977 ms; -DNDF_MBAR_HINT=0 restores the plain poll).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(NDF_MBAR_HINT)
      : "memory");
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif
// non-blocking: true once the phase with the given parity has completed
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
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
__device__ __forceinline__ void tcgen05_fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
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
// Warp-collective issue: the WHOLE (converged) warp executes these with warp-uniform
// operands and elect.sync picks the issuing lane inside the asm.  The compiler then keeps
// descriptors and TMEM addresses in uniform registers and emits back-to-back UTCHMMA,
// instead of wrapping every MMA issued under `if (lane == 0)` in an ELECT /
// R2UR.BROADCAST loop (divergent code with per-thread operands).
__device__ __forceinline__ void mma_ss_warp(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
// fp8 x fp8 -> fp32 (kind::f8f6f4; with a_format = b_format = 1 = E5M2 the instruction
// descriptor has the same bits as the bf16 one): one K32 step, A from TMEM (4 elements per
// 32-bit column, k ascending from the low byte)
__device__ __forceinline__ void mma_ts_f8_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
// four fp32 values -> four E5M2 bytes (round to nearest even, saturating), v0 in the low byte
__device__ __forceinline__ uint32_t pack4_e5m2(float v0, float v1, float v2, float v3) {
  uint32_t w;
  asm("{\n\t.reg .b16 l, h;\n\t"
      "cvt.rn.satfinite.e5m2x2.f32 l, %2, %1;\n\t"
      "cvt.rn.satfinite.e5m2x2.f32 h, %4, %3;\n\t"
      "mov.b32 %0, {l, h};\n}"
      : "=r"(w)
      : "f"(v0), "f"(v1), "f"(v2), "f"(v3));
  return w;
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ int warp_uniform(int v) { return __shfl_sync(0xffffffffu, v, 0); }
__device__ __forceinline__ uint32_t warp_uniform(uint32_t v) {
  return __shfl_sync(0xffffffffu, v, 0);
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
// Packed fp32 FMA (sm_100a FFMA2): (d0, d1) = (a0 * b0 + c0, a1 * b1 + c1), each
// rounded exactly like a scalar fmaf -- half the issue slots of two FFMAs.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0,
                                      float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
// Packed fp32 add / mul (sm_100a FADD2 / FMUL2).
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fmul2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// tanh of a pair on the FMA / integer pipes, no MUFU:
//   tanh|y| = 1 - 2 / (1 + 2^z),  z = 2 |y| log2(e) clamped to 64,
//   2^z = 2^n * p(f) (n = round(z) by the 1.5 * 2^23 trick, f in [-0.5, 0.5], p a degree-5
//   fit, 2.3e-7 relative in fp32 Horner), the reciprocal by a bit-trick seed and three
//   Newton steps (~4e-8); sign restored.  |error| <= ~3e-7, below what SiLU's fp32 output
//   resolves; NaN in -> NaN out through the caller's y + y * t.  Lets part of the epilogue's
//   tanh leave the (binding) MUFU pipe for the FMA pipe, which the epilogue leaves mostly idle.
__device__ __forceinline__ void tanh2_fma(float y0, float y1, float& t0, float& t1) {
  const float kM = 12582912.0f;   // 1.5 * 2^23: z + kM rounds z to an integer in the low bits
  float z0, z1;
  fmul2(z0, z1, fabsf(y0), fabsf(y1), 2.8853900817779268f, 2.8853900817779268f);
  z0 = fminf(z0, 64.0f);
  z1 = fminf(z1, 64.0f);
  float m0, m1, n0, n1, f0, f1;
  fadd2(m0, m1, z0, z1, kM, kM);
  fadd2(n0, n1, m0, m1, -kM, -kM);
  ffma2(f0, f1, n0, n1, -1.0f, -1.0f, z0, z1);                       // f = z - n
  float p0 = 0.0013267219765111804f, p1 = 0.0013267219765111804f;
  ffma2(p0, p1, p0, p1, f0, f1, 0.009675461798906326f, 0.009675461798906326f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.055507417768239975f, 0.055507417768239975f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.24022121727466583f, 0.24022121727466583f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.6931469440460205f, 0.6931469440460205f);
  ffma2(p0, p1, p0, p1, f0, f1, 1.0000001192092896f, 1.0000001192092896f);
  const int kMb = 0x4B400000;      // bits of kM
  const float e0 = __int_as_float(__float_as_int(p0) + ((__float_as_int(m0) - kMb) << 23));
  const float e1 = __int_as_float(__float_as_int(p1) + ((__float_as_int(m1) - kMb) << 23));
  float d0, d1;
  fadd2(d0, d1, e0, e1, 1.0f, 1.0f);
  float r0 = __int_as_float(0x7EF311C7 - __float_as_int(d0));
  float r1 = __int_as_float(0x7EF311C7 - __float_as_int(d1));
#pragma unroll
  for (int it = 0; it < 3; ++it) {
    float q0, q1;
    ffma2(q0, q1, -d0, -d1, r0, r1, 1.0f, 1.0f);
    ffma2(r0, r1, r0, r1, q0, q1, r0, r1);
  }
  ffma2(t0, t1, -2.0f, -2.0f, r0, r1, 1.0f, 1.0f);
  t0 = __int_as_float(__float_as_int(t0) | (__float_as_int(y0) & 0x80000000));
  t1 = __int_as_float(__float_as_int(t1) | (__float_as_int(y1) & 0x80000000));
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
// No "memory" clobber: the 16-bit operand tiles written with this are read only by
// the tensor cores (after fence.proxy.async, which clobbers memory), so ordinary
// loads may be scheduled across these stores.
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d));
}

// 16-byte global -> shared copy on the LSU async path (no registers); made visible
// to the tensor cores by cp_async_wait_all + fence.proxy.async
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace tc
}  // namespace ndf
