// gelu.cuh -- fp32 GELU (toydit.cpp:83, 0.5 x (1 + erf(x / sqrt2))) shared by
// the fused quantizer's prologue and the GEMM's activation epilogue.
#pragma once

#include <cuda_runtime.h>

namespace dtq_act {

// Packed fp32 GELU for the fast kernels: gelu(x) = x * Phi(x) (toydit.cpp:83)
// rewritten as max(x, 0) - |x| * E(z), z = |x| / sqrt(2), E = erfc(z) / 2 =
// exp(-z^2) * erfcx(z) / 2.  erfcx is entire and smooth on [0, 3.6], so a
// degree-11 polynomial in u = z / 1.8 - 1 (fp32 Horner; least squares in the
// Chebyshev basis weighted by the GELU error it causes, |x| exp(-z^2), with
// Lawson reweighting toward minimax) gives |gelu error| <= 4.9e-8 absolute
// -- below the fp32 rounding of the result for |gelu(x)| >= 1, so the codes
// downstream flip no more often than fp32 rounding alone makes them (the
// degree-8 fit of round 1 erred by 1.4e-5 and moved ~3e-4 of codes).  exp2
// on the MUFU, one per element; u is clamped at 1 (z = 3.6), where E < 2e-7
// and the clamp's overestimate costs < 5e-9.  Coefficients are -erfcx/2.
__device__ __forceinline__ float gelu_nerfcx_poly(float u) {
  // Horner with literal coefficients: FFMA's immediate form (twice the issue
  // rate of the 3-register form) and no coefficient registers
  float a = 3.810651368e-03f;
  a = fmaf(a, u, -1.157444203e-03f);
  a = fmaf(a, u, -2.343322383e-03f);
  a = fmaf(a, u, -7.673865184e-03f);
  a = fmaf(a, u, 1.215080731e-02f);
  a = fmaf(a, u, -1.378311217e-02f);
  a = fmaf(a, u, 2.538570575e-02f);
  a = fmaf(a, u, -4.080533609e-02f);
  a = fmaf(a, u, 6.018119678e-02f);
  a = fmaf(a, u, -8.510401100e-02f);
  a = fmaf(a, u, 1.130095497e-01f);
  return fmaf(a, u, -1.392800957e-01f);
}

// the same polynomial on two values at once: FFMA2 with a broadcast immediate
__device__ __forceinline__ float2 gelu_nerfcx_poly2(float2 u) {
  float2 a = make_float2(3.810651368e-03f, 3.810651368e-03f);
  a = __ffma2_rn(a, u, make_float2(-1.157444203e-03f, -1.157444203e-03f));
  a = __ffma2_rn(a, u, make_float2(-2.343322383e-03f, -2.343322383e-03f));
  a = __ffma2_rn(a, u, make_float2(-7.673865184e-03f, -7.673865184e-03f));
  a = __ffma2_rn(a, u, make_float2(1.215080731e-02f, 1.215080731e-02f));
  a = __ffma2_rn(a, u, make_float2(-1.378311217e-02f, -1.378311217e-02f));
  a = __ffma2_rn(a, u, make_float2(2.538570575e-02f, 2.538570575e-02f));
  a = __ffma2_rn(a, u, make_float2(-4.080533609e-02f, -4.080533609e-02f));
  a = __ffma2_rn(a, u, make_float2(6.018119678e-02f, 6.018119678e-02f));
  a = __ffma2_rn(a, u, make_float2(-8.510401100e-02f, -8.510401100e-02f));
  a = __ffma2_rn(a, u, make_float2(1.130095497e-01f, 1.130095497e-01f));
  return __ffma2_rn(a, u, make_float2(-1.392800957e-01f, -1.392800957e-01f));
}

__device__ __forceinline__ float gelu1(float x) {
  // z = |x| / sqrt(2) is folded into both constants: u = z * 5/9 - 1 and
  // exp(-z^2) = 2^(|x|^2 * -log2(e) / 2)
  const float ax = fabsf(x);
  const float u = fminf(fmaf(ax, 0.39283710065919303f, -1.f), 1.f);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(ax * ax * -0.72134752044448170f));
  return fmaf(ax, e * gelu_nerfcx_poly(u), fmaxf(x, 0.f));  // max(x,0) - |x| E
}

// Two values at once, packed (FFMA2 / FMUL2 with broadcast immediates: the
// polynomial is 11 instructions per pair instead of per value); every
// operation rounds exactly as in gelu1, so the results are identical.
__device__ __forceinline__ float2 gelu2(float2 x) {
  const float2 ax = make_float2(fabsf(x.x), fabsf(x.y));
  float2 u = __ffma2_rn(ax, make_float2(0.39283710065919303f, 0.39283710065919303f),
                        make_float2(-1.f, -1.f));
  u.x = fminf(u.x, 1.f);
  u.y = fminf(u.y, 1.f);
  const float2 arg = __fmul2_rn(__fmul2_rn(ax, ax),
                                make_float2(-0.72134752044448170f, -0.72134752044448170f));
  float2 e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(arg.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(arg.y));
  const float2 t = __fmul2_rn(e, gelu_nerfcx_poly2(u));
  return __ffma2_rn(ax, t, make_float2(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f)));
}

}  // namespace dtq_act
