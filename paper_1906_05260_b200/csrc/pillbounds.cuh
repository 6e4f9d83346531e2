// A pill's bounding sphere and the broad phase's finiteness check, shared by the collision
// kernels (collide.cu) and the one-launch prediction (integrate.cu), which builds the rod pills
// of small worlds itself.
#pragma once

#include "kernels.cuh"
#include "pill.cuh"
#include "vmath.cuh"

namespace vdev {

// bounding_sphere, collision.cpp:137-153.
__device__ __forceinline__ void bounding_sphere(const PillV& p, V3& c, double& r) {
  const V3 axis = p.c1 - p.c0;
  const double l = norm(axis);
  if (l + p.r1 <= p.r0) {
    c = p.c0;
    r = p.r0;
    return;
  }
  if (l + p.r0 <= p.r1) {
    c = p.c1;
    r = p.r1;
    return;
  }
  const double u = 0.5 * (l + p.r1 - p.r0);
  c = p.c0 + (u / l) * axis;
  r = 0.5 * (l + p.r0 + p.r1);
}

// Pill i's bounding sphere into bsph, the finiteness check; returns its radius bits (0 if not finite).
__device__ __forceinline__ unsigned long long pill_bounds(const Collide& c, const PillV& p, int i, int substep,
                                                         unsigned long long* err) {
  V3 ctr;
  double r;
  bounding_sphere(p, ctr, r);
  c.bsph[i] = ctr.x;
  c.bsph[c.P + i] = ctr.y;
  c.bsph[2 * c.P + i] = ctr.z;
  c.bsph[3 * c.P + i] = r;
  if (!(finite3(ctr) && isfinite(r))) {
    if (c.P >= 2) atomicMin(err, err_code(substep, ERR_BROAD, 0, i));
    return 0;
  }
  return static_cast<unsigned long long>(__double_as_longlong(r));  // r >= 0: bit order == value order
}
}  // namespace vdev
