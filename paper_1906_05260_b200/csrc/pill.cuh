// Pill geometry shared by the collision kernels (collide.cu) and skin binding (skin.cu):
// the pill record and pill_project (collision.cpp:15-49) split into per-pill constants and the
// per-point projection — the same operations on the same inputs as the reference's single call.
#pragma once

#include "vmath.cuh"

namespace vdev {

using namespace vm;

struct PillV {
  V3 c0, c1;
  double r0, r1;
};

// Collide::pill is AoS, 8 doubles (64 B, two sectors) per pill: c0 xyz, c1 xyz, r0, r1 — a
// random pill costs two sectors instead of eight scattered SoA rows. (P kept for the callers.)
__device__ __forceinline__ PillV load_pill(const double* __restrict__ pill, int P, int i) {
  (void)P;
  const double2* q = reinterpret_cast<const double2*>(pill + 8ll * i);
  const double2 a = q[0], b = q[1], d = q[2], e = q[3];
  return PillV{V3{a.x, a.y, b.x}, V3{b.y, d.x, d.y}, e.x, e.y};
}

// pill_project (collision.cpp:15-49) with the per-pill constants (axis, length, unit axis,
// cone slope) computed once per query pill: same operations on the same inputs, so the
// results are identical to evaluating them inside every call.
struct PillPrep {
  V3 c0, c1;
  double r0, r1;
  bool degenerate;
  double l;
  Recip rl;  // 1 / l, shared by every projection's divisions (divr: the same bits as / l)
  V3 j;
  double tan_t;
};
__device__ __forceinline__ PillPrep prep_pill(const PillV& p) {
  PillPrep q;
  q.c0 = p.c0;
  q.c1 = p.c1;
  q.r0 = p.r0;
  q.r1 = p.r1;
  const V3 axis = p.c1 - p.c0;
  q.l = norm(axis);
  q.degenerate = q.l <= fabs(p.r0 - p.r1) || q.l < 1e-14;
  q.rl = recip(q.l);
  if (!q.degenerate) {
    q.j = V3{divr(axis.x, q.rl), divr(axis.y, q.rl), divr(axis.z, q.rl)};
    const double sin_t = divr(p.r1 - p.r0, q.rl);
    q.tan_t = sin_t / sqrt(fmax(1e-16, 1.0 - sin_t * sin_t));
  } else {
    q.j = V3{0, 0, 0};
    q.tan_t = 0;
  }
  return q;
}
__device__ __forceinline__ double project(const V3& x, const PillPrep& p, double& t_out, bool& deg) {
  if (p.degenerate) {
    const double d0 = norm(x - p.c0) - p.r0;
    const double d1 = norm(x - p.c1) - p.r1;
    deg = true;
    if (d0 <= d1) {
      t_out = 0.0;
      return d0;
    }
    t_out = 1.0;
    return d1;
  }
  deg = false;
  const V3 y = x - p.c0;
  const double a = dot(y, p.j);
  const double b = norm(y - a * p.j);
  double t = divr(a + b * p.tan_t, p.rl);
  t = fmin(fmax(t, 0.0), 1.0);
  t_out = t;
  const V3 c = (1.0 - t) * p.c0 + t * p.c1;  // pill_distance_at, collision.cpp:9-13
  const double r = (1.0 - t) * p.r0 + t * p.r1;
  return norm(x - c) - r;
}
}  // namespace vdev
