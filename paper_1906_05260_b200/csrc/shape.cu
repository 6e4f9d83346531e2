// Bundle shape matching (apply_shape_match / fit_similarity / extract_rotation,
// bundling.cpp:50-133), applied after every shape_match_period-th sweep (solver.cpp:336-338).
//
// One warp per group: member loads are strided over lanes, the centroid, the 3x3 covariance B
// and the scale numerator are warp tree reductions (fixed order, deterministic), the Müller
// rotation extraction (warm-started from the group's persistent rotation) runs redundantly in
// every lane, and lanes write their members back. The reference applies groups sequentially;
// groups are disjoint in vertices but may share a frame (vertices m-1 and m map to element
// m-1), so the host schedules groups into dependency levels (host_model.cpp) and each level is
// one launch: within a level no two groups touch the same frame, across levels the reference's
// order is kept.
#include "kernels.cuh"
#include "vmath.cuh"

namespace vdev {

using namespace vm;

namespace {

constexpr int kWarpsPerBlock = 4;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ V3 ldc(const double* X, int vp, int v) {
  return V3{X[CX * (long long)vp + v], X[CY * (long long)vp + v], X[CZ * (long long)vp + v]};
}
__device__ __forceinline__ Q4 ldq(const double* X, int vp, int v) {
  return Q4{X[QW * (long long)vp + v], X[QX * (long long)vp + v], X[QY * (long long)vp + v], X[QZ * (long long)vp + v]};
}

// extract_rotation, bundling.cpp:50-67: the same iteration (omega = sum R_a x B_a / (|sum
// R_a . B_a| + 1e-9), q <- AngleAxis(|omega|, omega^) q, normalize, stop at |omega| < 1e-9).
// The loop is one serial dependency chain (tens of iterations even warm-started), so it is
// written for latency. Warm-started steps are tiny: for half angles below 1e-2 the increment
// [cos(a/2), sin(a/2)/a * omega] comes from the Taylor series in a^2 (truncation < 1e-20
// relative) with no sqrt, division or sincos on the chain; larger steps take the general
// route. These change last-ulp rounding only; shape matching is tolerance-pinned.
__device__ Q4 extract_rotation(const M3& B, const Q4& guess) {
  Q4 q = qnormalized(guess);
  for (int it = 0; it < 100; ++it) {
    const M3 R = qmat(q);
    V3 omega{0, 0, 0};
    double d = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      omega = omega + cross(col(R, a), col(B, a));
      d += dot(col(R, a), col(B, a));
    }
    omega = (1.0 / (fabs(d) + 1e-9)) * omega;
    const double a2 = sqnorm(omega);
    if (a2 < 1e-18) break;  // |omega| < 1e-9
    const double x2 = 0.25 * a2;  // (angle / 2)^2
    double k, c;  // k = sin(angle/2) / angle, c = cos(angle/2)
    if (x2 < 1e-4) {
      k = 0.5 * (1.0 - x2 * (1.0 / 6) * (1.0 - x2 * (1.0 / 20) * (1.0 - x2 * (1.0 / 42) * (1.0 - x2 * (1.0 / 72)))));
      c = 1.0 - x2 * 0.5 *
                    (1.0 - x2 * (1.0 / 12) * (1.0 - x2 * (1.0 / 30) * (1.0 - x2 * (1.0 / 56) * (1.0 - x2 * (1.0 / 90)))));
    } else {
      const double angle = sqrt(a2);
      double s;
      sincos(0.5 * angle, &s, &c);
      k = s / angle;
    }
    const V3 v = k * omega;
    const Q4 p = qmul(Q4{c, v.x, v.y, v.z}, q);
    const double r = rsqrt(qsqnorm(p));
    q = Q4{p.w * r, p.x * r, p.y * r, p.z * r};
  }
  return q;
}

__global__ void k_shape_level(World w, Groups g, double* __restrict__ X, int gbeg, int gend, int pdl) {
  if (pdl) {
    pdl_wait();
    pdl_trigger();
  }
  const int lane = threadIdx.x & 31;
  const int gi = gbeg + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (gi >= gend) return;
  const int grp = g.level_groups[gi];
  const int m0 = g.off[grp], m1 = g.off[grp + 1];
  const int n = m1 - m0;
  const int vp = w.vpad;
  // centroid of the current member centers
  V3 sum{0, 0, 0};
  for (int i = m0 + lane; i < m1; i += 32) sum = sum + ldc(X, vp, g.mslot[i]);
  const V3 cent = V3{wsum(sum.x), wsum(sum.y), wsum(sum.z)} / static_cast<double>(n);
  // B = sum (s * sbar) R Rbar^T + (c - mu) cbar^T
  double Bp[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = m0 + lane; i < m1; i += 32) {
    const double* mr = g.mrest + 17ll * i;
    const int v = g.mslot[i];
    const V3 c = ldc(X, vp, v) - cent;
    const double s = X[S * (long long)vp + v];
    const M3 R = qmat(ldq(X, vp, g.meslot[i]));
    M3 rR;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) rR.m[a][b] = mr[4 + 3 * a + b];
    const double ss = s * mr[3];
    M3 A;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) A.m[a][b] = ss * R.m[a][b];
    const M3 P = mmul_bt(A, rR);
    const double cv[3] = {c.x, c.y, c.z};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) Bp[3 * a + b] += P.m[a][b] + cv[a] * mr[b];
  }
  M3 B;
  double sq[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      B.m[a][b] = wsum(Bp[3 * a + b]);
      sq[a + 3 * b] = B.m[a][b] * B.m[a][b];
    }
  const double* gr = g.grest + 4ll * grp;
  const double denom = gr[3];
  if (sqrt(sum9(sq)) < 1e-12 || denom < 1e-300) return;  // degenerate: no write (bundling.cpp:86-90)
  const double* wq = g.warm + 4ll * grp;
  const Q4 q = extract_rotation(B, Q4{wq[0], wq[1], wq[2], wq[3]});
  const M3 Rf = qmat(q);
  const V3 rcent{gr[0], gr[1], gr[2]};
  double numer = 0.0;
  for (int i = m0 + lane; i < m1; i += 32) {
    const double* mr = g.mrest + 17ll * i;
    const int v = g.mslot[i];
    const V3 c = ldc(X, vp, v) - cent;
    const double s = X[S * (long long)vp + v];
    const M3 R = qmat(ldq(X, vp, g.meslot[i]));
    M3 rR;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) rR.m[a][b] = mr[4 + 3 * a + b];
    const M3 RR = mmul(Rf, rR);
    double e[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) e[a + 3 * b] = RR.m[a][b] * R.m[a][b];
    numer += (s * mr[3]) * sum9(e);
    numer += dot(c, mvmul(Rf, V3{mr[0], mr[1], mr[2]}));
  }
  numer = wsum(numer);
  const double scale = fmax(numer / denom, kMinScale);
  const V3 t = cent - scale * mvmul(Rf, rcent);
  const Q4 qf = qfrom_mat(Rf);
  auto apply = [&](int i) {
    const double* mr = g.mrest + 17ll * i;
    const int v = g.mslot[i];
    if (!w.pinned[v]) {
      const V3 x = scale * mvmul(Rf, V3{mr[0], mr[1], mr[2]} + rcent) + t;
      X[CX * (long long)vp + v] = x.x;
      X[CY * (long long)vp + v] = x.y;
      X[CZ * (long long)vp + v] = x.z;
      const double sn = fmax(scale * mr[3], kMinScale);
      X[S * (long long)vp + v] = sn;
      double2* xr = reinterpret_cast<double2*>(w.xrec + 8ll * v);
      xr[0] = make_double2(x.x, x.y);
      xr[1] = make_double2(x.z, sn);
    }
    const Q4 fr = qnormalized(qmul(qf, Q4{mr[13], mr[14], mr[15], mr[16]}));
    const int e = g.meslot[i];
    X[QW * (long long)vp + e] = fr.w;
    X[QX * (long long)vp + e] = fr.x;
    X[QY * (long long)vp + e] = fr.y;
    X[QZ * (long long)vp + e] = fr.z;
  };
  __syncwarp();
  if (g.serial[grp]) {
    if (lane == 0)
      for (int i = m0; i < m1; ++i) apply(i);
  } else {
    for (int i = m0 + lane; i < m1; i += 32) apply(i);
  }
  if (lane == 0) {
    double* wo = g.warm + 4ll * grp;
    wo[0] = q.w;
    wo[1] = q.x;
    wo[2] = q.y;
    wo[3] = q.z;
  }
}

}  // namespace

void launch_shape_match(const World& w, const Groups& g, double* X, const int* level_off_host, bool pdl, cudaStream_t st) {
  for (int l = 0; l < g.levels; ++l) {
    const int gb = level_off_host[l], ge = level_off_host[l + 1];
    const int ng = ge - gb;
    if (ng <= 0) continue;
    const int blocks = (ng + kWarpsPerBlock - 1) / kWarpsPerBlock;
    launch_kernel(k_shape_level, blocks, 32 * kWarpsPerBlock, 0, st, pdl, w, g, X, gb, ge, pdl ? 1 : 0);
  }
}

}  // namespace vdev
