// Small FP64 vector / quaternion / 3x3 helpers for the CPU restatement oracle.
// TEST INFRASTRUCTURE ONLY (see vrod_oracle.cpp).
//
// Every helper spells out its evaluation order so the restatement reproduces the arithmetic
// of the reference compiled against oracle/shim/Eigen (the oracle/_ref build) bit for bit:
//   dot3 / norm3: (a0*b0 + a1*b1) + a2*b2
//   quaternion squared norm (Eigen coeffs x,y,z,w): (x*x + z*z) + (y*y + w*w)
//   3x3 products: sum over k left to right
//   9-term sums (Frobenius norm, cwise sum): Eigen SSE2 packet order (see shim/Eigen/Dense)
#pragma once

#include <algorithm>
#include <cmath>

namespace vo {

struct V3 {
  double x = 0, y = 0, z = 0;
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline V3 mk(double x, double y, double z) { return V3{x, y, z}; }
inline V3 add(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 mul(double s, const V3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 divs(const V3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline V3 neg(const V3& a) { return {-a.x, -a.y, -a.z}; }
inline V3 cwmul(const V3& a, const V3& b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
inline double dot(const V3& a, const V3& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double sqnorm(const V3& a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
inline double norm(const V3& a) { return std::sqrt(sqnorm(a)); }
inline V3 normalized(const V3& a) {
  const double n = sqnorm(a);
  if (n <= 0.0) return a;
  const double s = std::sqrt(n);
  return divs(a, s);
}
inline V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline bool finite(const V3& a) { return std::isfinite(a.x) && std::isfinite(a.y) && std::isfinite(a.z); }
inline double maxc(const V3& a) { return std::max(std::max(a.x, a.y), a.z); }

struct Q {
  double w = 1, x = 0, y = 0, z = 0;
};
inline Q mkq(double w, double x, double y, double z) { return Q{w, x, y, z}; }
inline double qsqnorm(const Q& q) { return (q.x * q.x + q.z * q.z) + (q.y * q.y + q.w * q.w); }
inline double qnorm(const Q& q) { return std::sqrt(qsqnorm(q)); }
inline double qdot(const Q& a, const Q& b) { return (a.x * b.x + a.z * b.z) + (a.y * b.y + a.w * b.w); }
inline Q qnormalized(const Q& q) {  // Eigen normalized(): coefficient / sqrt(n), n > 0
  const double n = qsqnorm(q);
  if (n <= 0.0) return q;
  const double s = std::sqrt(n);
  return Q{q.w / s, q.x / s, q.y / s, q.z / s};
}
inline void qnormalize(Q& q) {  // Eigen normalize(): only when z > 0
  const double n = qsqnorm(q);
  if (n > 0.0) {
    const double s = std::sqrt(n);
    q = Q{q.w / s, q.x / s, q.y / s, q.z / s};
  }
}
inline Q qconj(const Q& q) { return Q{q.w, -q.x, -q.y, -q.z}; }
inline Q qmul(const Q& a, const Q& b) {
  return Q{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
           a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z, a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x};
}
inline V3 qvec(const Q& q) { return V3{q.x, q.y, q.z}; }
// Eigen _transformVector: uv = v x w-part ... v + w*uv + vec x uv.
inline V3 qrot(const Q& q, const V3& v) {
  const V3 qv = qvec(q);
  V3 uv = cross(qv, v);
  uv = add(uv, uv);
  return add(add(v, mul(q.w, uv)), cross(qv, uv));
}
// [theta/2, 1] renormalized (types.h:31-35).
inline Q small_rotation(const V3& th) {
  Q q{1.0, 0.5 * th.x, 0.5 * th.y, 0.5 * th.z};
  qnormalize(q);
  return q;
}
// q * small_rotation(theta), renormalized (types.h:38-42).
inline Q apply_increment(const Q& q, const V3& th) {
  Q out = qmul(q, small_rotation(th));
  qnormalize(out);
  return out;
}
inline bool is_unit(const Q& q, double tol = 1e-6) { return std::abs(qnorm(q) - 1.0) <= tol; }

struct M3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double& operator()(int i, int j) { return m[i][j]; }
  double operator()(int i, int j) const { return m[i][j]; }
  V3 col(int j) const { return V3{m[0][j], m[1][j], m[2][j]}; }
  V3 row(int i) const { return V3{m[i][0], m[i][1], m[i][2]}; }
};
inline M3 mmul(const M3& a, const M3& b) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o(i, j) = (a(i, 0) * b(0, j) + a(i, 1) * b(1, j)) + a(i, 2) * b(2, j);
  return o;
}
inline M3 mtrans(const M3& a) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o(i, j) = a(j, i);
  return o;
}
inline V3 mvmul(const M3& a, const V3& v) {
  return V3{(a(0, 0) * v.x + a(0, 1) * v.y) + a(0, 2) * v.z, (a(1, 0) * v.x + a(1, 1) * v.y) + a(1, 2) * v.z,
            (a(2, 0) * v.x + a(2, 1) * v.y) + a(2, 2) * v.z};
}
inline M3 mscale(double s, const M3& a) {
  M3 o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o(i, j) = s * a(i, j);
  return o;
}
inline void madd(M3& a, const M3& b) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a(i, j) = a(i, j) + b(i, j);
}
// Eigen SSE2 redux order over 9 column-major coefficients e[0..8].
inline double sum9(const double* e) {
  const double l0 = (e[0] + e[2]) + (e[4] + e[6]);
  const double l1 = (e[1] + e[3]) + (e[5] + e[7]);
  return (l0 + l1) + e[8];
}
inline double mfrob(const M3& a) {  // .norm()
  double e[9];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) e[i + 3 * j] = a(i, j) * a(i, j);
  return std::sqrt(sum9(e));
}
inline double mcwise_sum(const M3& a, const M3& b) {  // a.cwiseProduct(b).sum()
  double e[9];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) e[i + 3 * j] = a(i, j) * b(i, j);
  return sum9(e);
}

// Eigen toRotationMatrix.
inline M3 qmat(const Q& q) {
  M3 r;
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  r(0, 0) = 1.0 - (tyy + tzz);
  r(0, 1) = txy - twz;
  r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;
  r(1, 1) = 1.0 - (txx + tzz);
  r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;
  r(2, 1) = tyz + twx;
  r(2, 2) = 1.0 - (txx + tyy);
  return r;
}
// Eigen Quaternion(Matrix3).
inline Q qfrom_mat(const M3& m) {
  Q q;
  double c[4];  // x, y, z, w
  double t = (m(0, 0) + m(1, 1)) + m(2, 2);
  if (t > 0.0) {
    t = std::sqrt(t + 1.0);
    c[3] = 0.5 * t;
    t = 0.5 / t;
    c[0] = (m(2, 1) - m(1, 2)) * t;
    c[1] = (m(0, 2) - m(2, 0)) * t;
    c[2] = (m(1, 0) - m(0, 1)) * t;
  } else {
    int i = 0;
    if (m(1, 1) > m(0, 0)) i = 1;
    if (m(2, 2) > m(i, i)) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + 1.0);
    c[i] = 0.5 * t;
    t = 0.5 / t;
    c[3] = (m(k, j) - m(j, k)) * t;
    c[j] = (m(j, i) + m(i, j)) * t;
    c[k] = (m(k, i) + m(i, k)) * t;
  }
  q.x = c[0];
  q.y = c[1];
  q.z = c[2];
  q.w = c[3];
  return q;
}
// Eigen Quaternion(AngleAxis(angle, axis)).
inline Q qfrom_angle_axis(double angle, const V3& axis) {
  const double ha = 0.5 * angle;
  const V3 v = mul(std::sin(ha), axis);
  return Q{std::cos(ha), v.x, v.y, v.z};
}
// Eigen setFromTwoVectors (antiparallel branch: same deterministic axis as the shim).
inline Q qfrom_two_vectors(const V3& a, const V3& b) {
  const V3 v0 = normalized(a), v1 = normalized(b);
  double c = dot(v1, v0);
  if (c < -1.0 + 1e-12) {
    c = std::max(c, -1.0);
    int k = 0;
    if (std::abs(v0[1]) < std::abs(v0[k])) k = 1;
    if (std::abs(v0[2]) < std::abs(v0[k])) k = 2;
    V3 e{0, 0, 0};
    e[k] = 1.0;
    const V3 axis = normalized(cross(v0, e));
    const double w2 = (1.0 + c) * 0.5;
    const V3 v = mul(std::sqrt(1.0 - w2), axis);
    return Q{std::sqrt(w2), v.x, v.y, v.z};
  }
  const V3 axis = cross(v0, v1);
  const double s = std::sqrt((1.0 + c) * 2.0);
  const double invs = 1.0 / s;
  const V3 v{axis.x * invs, axis.y * invs, axis.z * invs};
  return Q{s * 0.5, v.x, v.y, v.z};
}
// Eigen slerp.
inline Q qslerp(const Q& a, double t, const Q& b) {
  const double one = 1.0 - 2.220446049250313e-16;
  const double d = qdot(a, b);
  const double absD = std::abs(d);
  double s0, s1;
  if (absD >= one) {
    s0 = 1.0 - t;
    s1 = t;
  } else {
    const double theta = std::acos(absD);
    const double sinTheta = std::sin(theta);
    s0 = std::sin((1.0 - t) * theta) / sinTheta;
    s1 = std::sin(t * theta) / sinTheta;
  }
  if (d < 0.0) s1 = -s1;
  return Q{s0 * a.w + s1 * b.w, s0 * a.x + s1 * b.x, s0 * a.y + s1 * b.y, s0 * a.z + s1 * b.z};
}

}  // namespace vo
