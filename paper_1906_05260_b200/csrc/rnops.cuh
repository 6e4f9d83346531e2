// Several correctly rounded divisions by ONE divisor, branch-free, for the exact-order
// shape-matching chain (shape.cuh extract_rotation_exact): omega / (|d| + 1e-9), omega / angle
// and the four quaternion coefficients / |q| of Eigen's normalized().
//
// The compiler expands every a / b into its own reciprocal refinement followed by a slow-path
// branch on the quotient, so the divisions of one vector run one after another. Here the
// divisor's correctly rounded reciprocal y = RN(1/b) (__drcp_rn) is formed once and each
// quotient is q' = RN(q + (a - b q) y) with q = RN(a y) and the remainder exact (FMA) — Markstein's
// theorem makes q' = RN(a / b), the IEEE quotient the CPU computes. Operands outside the safe
// exponent range take the IEEE division instead (zero numerators give the IEEE signed zero directly), so the result equals a / b
// for every input; tools/ubench/exactops.cu checks this on 10^9 random and adversarial pairs.
#pragma once

namespace rn {

// |v| in [2^-480, 2^480): quotients and remainders stay normal. Integer test on the exponent
// field (the INT pipe, off the FP64 pipe the chain is bound by).
__device__ __forceinline__ bool safe(double v) {
  const unsigned e = (static_cast<unsigned>(__double2hiint(v)) >> 20) & 0x7ffu;
  return e - (1023u - 480u) < 960u;
}
__device__ __forceinline__ bool is_zero(double v) { return (static_cast<unsigned long long>(__double_as_longlong(v)) << 1) == 0ull; }

// q[i] = a[i] / b, correctly rounded, i < N.
template <int N>
__device__ __forceinline__ void div_by(const double (&a)[N], double b, double (&q)[N]) {
  const double y = __drcp_rn(b);
  bool ok = safe(b);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double q0 = a[i] * y;  // a zero numerator: +-0 * y is the IEEE signed zero quotient
    const double r = fma(-b, q0, a[i]);
    const bool z = is_zero(a[i]);
    q[i] = z ? q0 : fma(r, y, q0);
    ok = ok && (z || safe(a[i]));
  }
  if (!ok) {  // rare: tiny or huge operands
#pragma unroll
    for (int i = 0; i < N; ++i) q[i] = a[i] / b;
  }
}

}  // namespace rn
