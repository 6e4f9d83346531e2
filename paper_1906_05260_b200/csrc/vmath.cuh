// FP64 vector / quaternion / 3x3 helpers shared by the product's host setup code and its
// sm_100a kernels. Evaluation order follows the reference's Eigen expressions
// (proj/core/include/vrod/types.h:31-61 and their call sites): dot3 = (a0b0 + a1b1) + a2b2,
// quaternion squared norm over Eigen's (x,y,z,w) coefficient order = (x^2 + z^2) + (y^2 + w^2),
// Hamilton product and toRotationMatrix in Eigen's closed forms. Kernels compiled with
// --fmad=false therefore reproduce the reference bit for bit (the latency-tuned shape-matching
// chain in shape.cuh is the one place that uses explicit FMAs, within BASELINE.md's tolerance).
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define VHD __host__ __device__ __forceinline__
#else
#define VHD inline
#endif

namespace vm {

#ifndef __CUDACC__
using std::fabs;
using std::fmax;
using std::fmin;
using std::isfinite;
using std::isinf;
using std::sqrt;
#endif

struct V3 {
  double x, y, z;
};
struct Q4 {
  double w, x, y, z;
};

// a / b, IEEE. On the device a zero numerator is answered directly (+-0 with the quotient's
// sign): the compiler's div.rn.f64 expansion sends zero (and tiny) numerators down its slow-path
// subroutine call, and resting / straight rods divide exact zeros all the time.
VHD double qdiv(double a, double b) {
#ifdef __CUDA_ARCH__
  if (a == 0.0 && b != 0.0 && isfinite(b)) return a * copysign(1.0, b);
#endif
  return a / b;
}

// Division by a shared reciprocal, bit-identical to a / b (Markstein's theorem): y = RN(1/b),
// q = RN(a*y), e = a - b*q exactly (FMA), RN(q + e*y) == RN(a/b) whenever nothing under- or
// overflows on the way — guarded here to |a|, |b| in [2^-500, 2^500]; any other operand (zero,
// subnormal, huge, inf, nan) takes the IEEE division. Several quotients by one denominator then
// cost one correctly rounded reciprocal plus a multiply and two FMAs each, instead of one
// div.rn.f64 expansion each. tools/ubench/divcheck.cu: 8.6e9 random and adversarial operand
// pairs (all-ones / power-of-two / near-halfway mantissas, exponents -60..60), 0 mismatches on
// B200. Host code (no __drcp_rn) always divides.
struct Recip {
  double b, y;
  bool ok;
};
VHD Recip recip(double b) {
#ifdef __CUDA_ARCH__
  const double ab = fabs(b);
  const bool ok = ab >= 0x1p-500 && ab <= 0x1p500;
  return Recip{b, ok ? __drcp_rn(b) : 0.0, ok};
#else
  return Recip{b, 0.0, false};
#endif
}
// 1.0 / b (RN(1/b) is exactly the reciprocal recip() holds)
VHD double rinv(const Recip& r) { return r.ok ? r.y : 1.0 / r.b; }
#ifdef __CUDA_ARCH__
// the rare operands out of divr's range: one out-of-line IEEE division (keeps the inlined code small)
__device__ __noinline__ double div_slow(double a, double b) { return qdiv(a, b); }
#endif
VHD double divr(double a, const Recip& r) {
#ifdef __CUDA_ARCH__
  const double aa = fabs(a);
  if (r.ok && aa >= 0x1p-500 && aa <= 0x1p500) {
    const double q = a * r.y;
    const double e = fma(-r.b, q, a);
    return fma(e, r.y, q);
  }
  if (r.ok && a == 0.0) return a * copysign(1.0, r.b);  // exact zeros are common (qdiv's shortcut)
  return div_slow(a, r.b);
#else
  return qdiv(a, r.b);
#endif
}

VHD V3 v3(double x, double y, double z) { return V3{x, y, z}; }
VHD V3 operator+(const V3& a, const V3& b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
VHD V3 operator-(const V3& a, const V3& b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
VHD V3 operator-(const V3& a) { return V3{-a.x, -a.y, -a.z}; }
VHD V3 operator*(double s, const V3& a) { return V3{s * a.x, s * a.y, s * a.z}; }
VHD V3 operator/(const V3& a, double s) {
  const Recip r = recip(s);
  return V3{divr(a.x, r), divr(a.y, r), divr(a.z, r)};
}
VHD V3 cwmul(const V3& a, const V3& b) { return V3{a.x * b.x, a.y * b.y, a.z * b.z}; }
VHD double dot(const V3& a, const V3& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
VHD double sqnorm(const V3& a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
VHD double norm(const V3& a) { return sqrt(sqnorm(a)); }
VHD V3 cross(const V3& a, const V3& b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
VHD V3 normalized(const V3& a) {
  const double n = sqnorm(a);
  if (n <= 0.0) return a;
  return a / sqrt(n);
}
VHD bool finite3(const V3& a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }
VHD double comp(const V3& a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

VHD double qsqnorm(const Q4& q) { return (q.x * q.x + q.z * q.z) + (q.y * q.y + q.w * q.w); }
VHD double qnorm(const Q4& q) { return sqrt(qsqnorm(q)); }
VHD double qdot(const Q4& a, const Q4& b) { return (a.x * b.x + a.z * b.z) + (a.y * b.y + a.w * b.w); }
VHD Q4 qneg(const Q4& q) { return Q4{-q.w, -q.x, -q.y, -q.z}; }
VHD Q4 qconj(const Q4& q) { return Q4{q.w, -q.x, -q.y, -q.z}; }
VHD V3 qvec(const Q4& q) { return V3{q.x, q.y, q.z}; }
// Eigen normalized(): coefficient / sqrt(n) when n > 0.
VHD Q4 qnormalized(const Q4& q) {
  const double n = qsqnorm(q);
  if (n <= 0.0) return q;
  const Recip r = recip(sqrt(n));
  return Q4{divr(q.w, r), divr(q.x, r), divr(q.y, r), divr(q.z, r)};
}
VHD Q4 qmul(const Q4& a, const Q4& b) {
  return Q4{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
            a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z, a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x};
}
// Eigen _transformVector.
VHD V3 qrot(const Q4& q, const V3& v) {
  const V3 qv = qvec(q);
  V3 uv = cross(qv, v);
  uv = uv + uv;
  return (v + q.w * uv) + cross(qv, uv);
}
// small_rotation / apply_increment, types.h:31-42.
VHD Q4 apply_increment(const Q4& q, const V3& th) {
  const Q4 d = qnormalized(Q4{1.0, 0.5 * th.x, 0.5 * th.y, 0.5 * th.z});
  return qnormalized(qmul(q, d));
}
// relative_rotation, rod.cpp:151-155: conj(qa)*qb in the w >= 0 hemisphere.
VHD Q4 relative_rotation(const Q4& qa, const Q4& qb) {
  Q4 p = qmul(qconj(qa), qb);
  if (p.w < 0) p = qneg(p);
  return p;
}

struct M3 {
  double m[3][3];
};
// Eigen toRotationMatrix.
VHD M3 qmat(const Q4& q) {
  M3 r;
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  r.m[0][0] = 1.0 - (tyy + tzz);
  r.m[0][1] = txy - twz;
  r.m[0][2] = txz + twy;
  r.m[1][0] = txy + twz;
  r.m[1][1] = 1.0 - (txx + tzz);
  r.m[1][2] = tyz - twx;
  r.m[2][0] = txz - twy;
  r.m[2][1] = tyz + twx;
  r.m[2][2] = 1.0 - (txx + tyy);
  return r;
}
VHD V3 col(const M3& a, int j) { return V3{a.m[0][j], a.m[1][j], a.m[2][j]}; }
VHD M3 mmul(const M3& a, const M3& b) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.m[i][j] = (a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j]) + a.m[i][2] * b.m[2][j];
  return o;
}
VHD M3 mmul_bt(const M3& a, const M3& b) {  // a * b^T
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.m[i][j] = (a.m[i][0] * b.m[j][0] + a.m[i][1] * b.m[j][1]) + a.m[i][2] * b.m[j][2];
  return o;
}
VHD V3 mvmul(const M3& a, const V3& v) {
  return V3{(a.m[0][0] * v.x + a.m[0][1] * v.y) + a.m[0][2] * v.z,
            (a.m[1][0] * v.x + a.m[1][1] * v.y) + a.m[1][2] * v.z,
            (a.m[2][0] * v.x + a.m[2][1] * v.y) + a.m[2][2] * v.z};
}
// Eigen SSE2 redux order over 9 column-major coefficients.
VHD double sum9(const double* e) {
  const double l0 = (e[0] + e[2]) + (e[4] + e[6]);
  const double l1 = (e[1] + e[3]) + (e[5] + e[7]);
  return (l0 + l1) + e[8];
}
// Eigen Quaternion(Matrix3).
VHD Q4 qfrom_mat(const M3& a) {
  double c[4];  // x y z w
  double t = (a.m[0][0] + a.m[1][1]) + a.m[2][2];
  if (t > 0.0) {
    t = sqrt(t + 1.0);
    c[3] = 0.5 * t;
    t = 0.5 / t;
    c[0] = (a.m[2][1] - a.m[1][2]) * t;
    c[1] = (a.m[0][2] - a.m[2][0]) * t;
    c[2] = (a.m[1][0] - a.m[0][1]) * t;
  } else {
    int i = 0;
    if (a.m[1][1] > a.m[0][0]) i = 1;
    if (a.m[2][2] > a.m[i][i]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = sqrt(a.m[i][i] - a.m[j][j] - a.m[k][k] + 1.0);
    c[i] = 0.5 * t;
    t = 0.5 / t;
    c[3] = (a.m[k][j] - a.m[j][k]) * t;
    c[j] = (a.m[j][i] + a.m[i][j]) * t;
    c[k] = (a.m[k][i] + a.m[i][k]) * t;
  }
  return Q4{c[3], c[0], c[1], c[2]};
}
// Eigen setFromTwoVectors (antiparallel branch: axis from the least-aligned basis vector).
VHD Q4 qfrom_two_vectors(const V3& a, const V3& b) {
  const V3 v0 = normalized(a), v1 = normalized(b);
  double c = dot(v1, v0);
  if (c < -1.0 + 1e-12) {
    c = fmax(c, -1.0);
    int k = 0;
    if (fabs(v0.y) < fabs(comp(v0, k))) k = 1;
    if (fabs(v0.z) < fabs(comp(v0, k))) k = 2;
    const V3 e = V3{k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
    const V3 axis = normalized(cross(v0, e));
    const double w2 = (1.0 + c) * 0.5;
    const V3 v = sqrt(1.0 - w2) * axis;
    return Q4{sqrt(w2), v.x, v.y, v.z};
  }
  const V3 axis = cross(v0, v1);
  const double s = sqrt((1.0 + c) * 2.0);
  const double invs = 1.0 / s;
  return Q4{s * 0.5, axis.x * invs, axis.y * invs, axis.z * invs};
}

constexpr double kPi = 3.141592653589793;
constexpr double kMinScale = 1e-4;  // types.h:22

// inverse_stiffness, constraints.cpp:274-278.
VHD double inverse_stiffness(double k) {
  if (isinf(k)) return 0.0;
  if (k <= 0.0) return 1e30;
  return fmin(1.0 / k, 1e30);
}

// 3x3 solve of solve_block's dim-3 branch (constraints.cpp:446-454): singular test on Eigen's
// determinant, cofactor inverse, dlambda = beta * M^-1 * rhs.
VHD bool solve3(const double (&M)[3][3], const double (&rhs)[3], double beta, double (&dl)[3]) {
  // max |M_ij| as a tree (max is order-independent; fmax ignores NaN either way)
  const double m01 = fmax(fabs(M[0][0]), fabs(M[0][1])), m23 = fmax(fabs(M[0][2]), fabs(M[1][0]));
  const double m45 = fmax(fabs(M[1][1]), fabs(M[1][2])), m67 = fmax(fabs(M[2][0]), fabs(M[2][1]));
  double md = fmax(fmax(fmax(m01, m23), fmax(m45, m67)), fabs(M[2][2]));
  md = fmax(md, 1e-300);
  const double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                     M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                     M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
  if (fabs(det) <= 1e-14 * md * md * md) return false;
  const double c00 = M[1][1] * M[2][2] - M[1][2] * M[2][1];
  const double c10 = M[2][1] * M[0][2] - M[2][2] * M[0][1];
  const double c20 = M[0][1] * M[1][2] - M[0][2] * M[1][1];
  const double c01 = M[1][2] * M[2][0] - M[1][0] * M[2][2];
  const double c11 = M[2][2] * M[0][0] - M[2][0] * M[0][2];
  const double c21 = M[0][2] * M[1][0] - M[0][0] * M[1][2];
  const double c02 = M[1][0] * M[2][1] - M[1][1] * M[2][0];
  const double c12 = M[2][0] * M[0][1] - M[2][1] * M[0][0];
  const double c22 = M[0][0] * M[1][1] - M[0][1] * M[1][0];
  const double d = (c00 * M[0][0] + c10 * M[1][0]) + c20 * M[2][0];
  const double invdet = 1.0 / d;
  const double inv[3][3] = {{c00 * invdet, c10 * invdet, c20 * invdet},
                            {c01 * invdet, c11 * invdet, c21 * invdet},
                            {c02 * invdet, c12 * invdet, c22 * invdet}};
  for (int i = 0; i < 3; ++i)
    dl[i] = ((beta * inv[i][0]) * rhs[0] + (beta * inv[i][1]) * rhs[1]) + (beta * inv[i][2]) * rhs[2];
  return true;
}

}  // namespace vm
