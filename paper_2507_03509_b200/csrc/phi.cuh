// phi(x) = -ln(tanh(x/2)) for x >= 0, the magnitude map of the sum-product
// check update in the "phi domain":
//     |c2v_j| = phi( sum_{i != j} phi(|v2c_i|) ),   phi(phi(x)) = x,
// which is the reference's 2*atanh(prod tanh(m/2)) (decoder.cpp:86-95)
// rewritten so float32 never saturates: tanhf(|m|/2) rounds to 1.0 for
// |m| >= 20, inside the +-30 clamp, while phi keeps full relative precision
// (SURVEY Appendix C).  phi(0) = +inf and phi(+inf) = 0 reproduce the
// reference's tanh(0) = 0 product (punctured / zero messages) and its
// atanh(1) = inf -> clamp for degree-1 checks.
//
// Two branch-free pieces, selected per lane (no divergence):
//  x >= 1 : t = e^-x (MUFU.EX2), phi = 2*atanh(t) = 2t * (1 + w*A(w)), w = t^2
//  x <  1 : phi = -ln(x/2) + g(x),  g(x) = -ln(tanh(x/2)/(x/2)) = z*B(z),
//           z = x^2, and -ln(x/2) = (1 - log2 x) * ln 2 (MUFU.LG2)
// A and B are least-squares fits on Chebyshev nodes (fit error 1.3e-8 and
// 3.9e-9 absolute; script in tests/test_phi_numerics.py reproduces them).
#pragma once

namespace bpdec {
namespace dev {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 17 instructions, 2 MUFU: both pieces evaluated, selected per lane.
__device__ __forceinline__ float phi(float x) {
  // x >= 1: t = e^-x, phi = t * (2 + w*A2(w)), A2 = 2*A (coefficients doubled)
  const float t = ex2_approx(x * -1.4426950408889634f);
  const float w = t * t;
  float a = 2.0f * 0.14783698262526393f;
  a = fmaf(a, w, 2.0f * 0.1383879360711249f);
  a = fmaf(a, w, 2.0f * 0.2002081579507349f);
  a = fmaf(a, w, 2.0f * 0.3333303414682521f);
  const float hi = t * fmaf(a, w, 2.0f);
  // x < 1: phi = ln2 - ln2*log2(x) + z*B(z), z = x^2
  const float z = x * x;
  float b = -2.1672081029454006e-05f;
  b = fmaf(b, z, 0.0003380189508581495f);
  b = fmaf(b, z, -0.0048599077080608115f);
  b = fmaf(b, z, 0.08333320963387135f);
  const float lo = fmaf(lg2_approx(x), -0.6931471805599453f, fmaf(b, z, 0.6931471805599453f));
  return x < 1.0f ? lo : hi;
}

}  // namespace dev
}  // namespace bpdec
