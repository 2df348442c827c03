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

// ---------------------------------------------------------------------------
// The same check update in the "t domain": t(x) = e^-x, the ratio
// (1 - tanh(x/2)) / (1 + tanh(x/2)).  A product of tanh factors is, in t,
// the relativistic-velocity sum  a (+) b = (a + b) / (1 + a b)  (associative,
// commutative, 0 neutral, 1 absorbing), so
//     |c2v_j| = -ln( (+)_{i != j} t(|v2c_i|) ),
// the reference's 2*atanh(prod tanh(m/2)) without ever forming tanh: t keeps
// full relative precision where tanh rounds to 1 (large |m|, the saturation
// that rules out the float tanh form), and -ln T of a tiny T is as exact as
// phi of a small sum.  Only weak outputs (T near 1) lose relative precision:
// their absolute error stays ~1e-7, far below the float posterior rounding.
//
// Sums are kept as fractions n / d of non-negative terms (no cancellation,
// d >= 1, one MUFU.LG2 pair per output instead of two phi evaluations per
// edge):  inputs 1 MUFU (EX2) + 1 FMUL, each (+) 2 ops, outputs
// ln2 * |lg2 d - lg2 n| (2 MUFU + 2 ops) min clamp.
//
// Exact zeros: a zero input (t = 1) makes every other output exactly 0, as
// in the reference (tanh 0 = 0): every (+) below keeps n == d bitwise once
// one operand has n == d (fma / add commute), and lg2 d - lg2 n is then 0.
// An underflowed t (|m| >= ~87) is 0: the outputs of the others are their
// own -ln t, and an all-underflow sum gives n = 0 -> +inf -> clamp, the
// reference's atanh(1) = inf -> clamp.
namespace bpdec {
namespace dev {

struct TF {
  float n, d;  // T = n / d, 0 <= n <= d (up to rounding), d >= 1
};

__device__ __forceinline__ float tdom(float x) { return ex2_approx(x * -1.4426950408889634f); }

// raw (+) raw
__device__ __forceinline__ TF tf_pair(float a, float b) { return {a + b, fmaf(a, b, 1.0f)}; }
// fraction (+) raw
__device__ __forceinline__ TF tf_add(TF f, float t) { return {fmaf(t, f.d, f.n), fmaf(t, f.n, f.d)}; }
// fraction (+) fraction, rounded products then a commuting add (symmetric:
// n == d on either side gives n == d)
__device__ __forceinline__ TF tf_join(TF a, TF b) {
  return {__fadd_rn(__fmul_rn(a.n, b.d), __fmul_rn(a.d, b.n)), __fadd_rn(__fmul_rn(a.d, b.d), __fmul_rn(a.n, b.n))};
}
// |c2v| = min(-ln(n / d), clamp); |.| absorbs a rounding of n above d
__device__ __forceinline__ float tmag(TF f, float clamp) {
  return fminf(fabsf((lg2_approx(f.d) - lg2_approx(f.n)) * 0.6931471805599453f), clamp);
}

}  // namespace dev
}  // namespace bpdec
