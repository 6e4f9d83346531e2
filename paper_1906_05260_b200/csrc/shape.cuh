// Bundle shape matching of one group (apply_shape_match / fit_similarity / extract_rotation,
// bundling.cpp:50-133) by one warp. Shared by the per-level kernel k_shape_level (shape.cu) and
// the persistent small-world iteration kernel (rodsweep.cu), so both paths give the same bits.
//
// Member loads are strided over lanes; the centroid, the 3x3 covariance B and the scale numerator
// are warp tree reductions (fixed order, deterministic); the Müller rotation extraction
// (warm-started from the group's persistent rotation) runs redundantly in every lane, and lanes
// write their members back. Shape matching is tolerance-pinned: the rotation
// chain uses explicit FMAs (both translation units compile with --fmad=false).
#pragma once

#include "crtrig.cuh"
#include "rnops.cuh"
#include "kernels.cuh"
#include "vmath.cuh"

namespace vdev {

__device__ __forceinline__ double shape_wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// General route of the rotation increment (half angle >= 1e-2: rare once warm-started); kept out
// of line so sincos's range reduction does not bloat the hot loop's code.
static __device__ __noinline__ double2 rotation_increment_general(double a2) {
  const double angle = sqrt(a2);
  double sn, cs;
  sincos(0.5 * angle, &sn, &cs);
  return make_double2(sn / angle, cs);  // (k, c), returned in registers
}

// 1 / |q| for a quaternion that is unit up to rounding: 1/sqrt(1+e) = 1 - e/2 + 3/8 e^2 (exact to
// 1e-30 for |e| < 1e-6; rsqrt otherwise).
__device__ __forceinline__ vm::Q4 qnormalized_fast(const vm::Q4& p) {
  const double e = fma(p.w, p.w, p.x * p.x) + fma(p.y, p.y, p.z * p.z) - 1.0;
  double r = fma(e, fma(e, 0.375, -0.5), 1.0);
  if (!(fabs(e) < 1e-6)) r = e > -1.0 ? rsqrt(e + 1.0) : 1.0;
  return vm::Q4{p.w * r, p.x * r, p.y * r, p.z * r};
}

// extract_rotation, bundling.cpp:50-67: the same iteration (omega = sum R_a x B_a / (|sum
// R_a . B_a| + 1e-9), q <- AngleAxis(|omega|, omega^) q, normalize, stop at |omega| < 1e-9).
// The loop is one serial dependency chain (~10 iterations warm-started at C3, up to ~20), so it
// is written for latency (shape matching is tolerance-pinned); per iteration the
// critical path is ~18 dependent FP64 operations + one MUFU (tools/ubench/rotbench.cu):
//  - R from q with FMA trees (depth 3); omega and the trace with FMA trees;
//  - a Newton reciprocal with one cubic step;
//  - the increment [cos(a/2), sin(a/2)/a * omega] from its Taylor series in x = (a/2)^2,
//    Estrin-evaluated (truncation < 1e-21 relative for x < 1e-4; larger steps take sincos);
//  - [c, k/d * omega] q = c q + (k/d) ([0, omega] q), the second product formed off the path;
//  - the stop test and the rare branches issued after the update, so nothing waits on them;
//  - the product of unit quaternions is unit to O(1e-16), so q is renormalised once at the end
//    (the 13-odd iterations drift |q| by ~1e-15, far below the 1e-9 stopping tolerance).
__device__ __forceinline__ vm::Q4 extract_rotation(const vm::M3& B, const vm::Q4& guess, int* iters = nullptr,
                                                   int max_iterations = 100, double tol2 = 1e-18) {
  using namespace vm;
  Q4 q = qnormalized_fast(guess);
  int it = 0;
#pragma unroll 1
  for (; it < max_iterations; ++it) {
    // R = toRotationMatrix(q)
    const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
    const double R[3][3] = {{fma(-ty, q.y, fma(-tz, q.z, 1.0)), fma(tx, q.y, -tz * q.w), fma(tx, q.z, ty * q.w)},
                            {fma(tx, q.y, tz * q.w), fma(-tx, q.x, fma(-tz, q.z, 1.0)), fma(ty, q.z, -tx * q.w)},
                            {fma(tx, q.z, -ty * q.w), fma(ty, q.z, tx * q.w), fma(-tx, q.x, fma(-ty, q.y, 1.0))}};
    // omega = sum_a col(R, a) x col(B, a); d = sum_a col(R, a) . col(B, a)
    double wx[3], wy[3], wz[3], dd[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double r0 = R[0][a], r1 = R[1][a], r2 = R[2][a];
      const double b0 = B.m[0][a], b1 = B.m[1][a], b2 = B.m[2][a];
      wx[a] = fma(r1, b2, -r2 * b1);
      wy[a] = fma(r2, b0, -r0 * b2);
      wz[a] = fma(r0, b1, -r1 * b0);
      dd[a] = fma(r0, b0, fma(r1, b1, r2 * b2));
    }
    const double ox = (wx[0] + wx[1]) + wx[2], oy = (wy[0] + wy[1]) + wy[2], oz = (wz[0] + wz[1]) + wz[2];
    const double den = fabs((dd[0] + dd[1]) + dd[2]) + 1e-9;
    // u = [0, omega] q: off the critical path (needs omega and q only)
    const double uw = -fma(ox, q.x, fma(oy, q.y, oz * q.z));
    const double ux = fma(ox, q.w, fma(oy, q.z, -oz * q.y));
    const double uy = fma(oy, q.w, fma(oz, q.x, -ox * q.z));
    const double uz = fma(oz, q.w, fma(ox, q.y, -oy * q.x));
    const double w2 = fma(ox, ox, fma(oy, oy, oz * oz));
    const double w2q = 0.25 * w2;
    // inv = 1 / den: MUFU seed (~2^-23) and one cubic Newton step (error ~2^-69)
    double inv;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(den));
    {
      const double e = fma(-den, inv, 1.0);
      inv = fma(inv, fma(e, e, e), inv);
    }
    const double x2 = (w2q * inv) * inv;  // (angle / 2)^2
    const double x4 = x2 * x2;
    // k = sin(angle/2) / angle, c = cos(angle/2)
    const double k = fma(x4, fma(x2, -1.0 / 10080, 1.0 / 240), fma(x2, -1.0 / 12, 0.5));
    const double c = fma(x4, fma(x2, -1.0 / 720, 1.0 / 24), fma(x2, -0.5, 1.0));
    const double ki = k * inv;
    Q4 p{fma(ki, uw, c * q.w), fma(ki, ux, c * q.x), fma(ki, uy, c * q.y), fma(ki, uz, c * q.z)};
    const bool stop = (w2 * inv) * inv < tol2;  // |omega| < tolerance (1e-9): keep q
    if (stop || !(x2 < 1e-4)) {  // one rare branch, at the end of the iteration
      if (stop) break;
      const double2 kc = rotation_increment_general(4.0 * x2);
      const double kg = kc.x * inv;
      p = Q4{fma(kg, uw, kc.y * q.w), fma(kg, ux, kc.y * q.x), fma(kg, uy, kc.y * q.y), fma(kg, uz, kc.y * q.z)};
    }
    q = p;
  }
  if (iters) *iters = it;
  return qnormalized_fast(q);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  return ns;
}

// Shared-memory copy of the static data of a few groups (the persistent kernel caches the groups
// of the chain its CTA runs, so a shape-matching pass loads only the members' state).
constexpr int kShapeCacheMembers = 64, kShapeCacheGroups = 4;
struct ShapeCache {
  int ng;
  int gid[kShapeCacheGroups], m0[kShapeCacheGroups], m1[kShapeCacheGroups], base[kShapeCacheGroups];
  int serial[kShapeCacheGroups];
  double grest[kShapeCacheGroups][4];
  int slot[kShapeCacheMembers], eslot[kShapeCacheMembers];
  uint8_t pinned[kShapeCacheMembers];
  double rest[kShapeCacheMembers][17];
};

// Fills `sc` with the groups k0 .. k1-1 of `list` while they fit (all threads of the CTA).
__device__ __forceinline__ void shape_cache_fill(ShapeCache& sc, const World& w, const Groups& g, const int* list, int k0,
                                                 int k1) {
  if (threadIdx.x == 0) {
    int ng = 0, nm = 0;
    for (int k = k0; k < k1 && ng < kShapeCacheGroups; ++k) {
      const int grp = list[k], m0 = g.off[grp], m1 = g.off[grp + 1];
      if (nm + (m1 - m0) > kShapeCacheMembers) break;
      sc.gid[ng] = grp;
      sc.m0[ng] = m0;
      sc.m1[ng] = m1;
      sc.base[ng] = nm;
      sc.serial[ng] = g.serial[grp];
      for (int a = 0; a < 4; ++a) sc.grest[ng][a] = g.grest[4ll * grp + a];
      nm += m1 - m0;
      ++ng;
    }
    sc.ng = ng;
  }
  __syncthreads();
  for (int c = 0; c < sc.ng; ++c)
    for (int i = threadIdx.x; i < sc.m1[c] - sc.m0[c]; i += blockDim.x) {
      const int m = sc.m0[c] + i, l = sc.base[c] + i;
      sc.slot[l] = g.mslot[m];
      sc.eslot[l] = g.meslot[m];
      sc.pinned[l] = w.pinned[g.mslot[m]];
      for (int a = 0; a < 17; ++a) sc.rest[l][a] = g.mrest[17ll * m + a];
    }
  __syncthreads();
}

// Per-warp state of one group fit between its phases: member range / cache mapping, the lane's
// first member (loaded once, reused), the centroid and the covariance.
struct ShapeState {
  int grp, m0, m1, ci, lb;
  vm::V3 cent, c0;
  double s0;
  vm::Q4 q0;
  vm::M3 B;
  bool degenerate;
};

// Member accessors of a group: the shared-memory cache when it holds the group, else global.
struct ShapeMembers {
  const Groups& g;
  const ShapeCache* sc;
  int ci, lb;
  __device__ __forceinline__ int slot(int i) const { return ci >= 0 ? sc->slot[i + lb] : g.mslot[i]; }
  __device__ __forceinline__ int eslot(int i) const { return ci >= 0 ? sc->eslot[i + lb] : g.meslot[i]; }
  __device__ __forceinline__ const double* rest(int i) const { return ci >= 0 ? &sc->rest[i + lb][0] : g.mrest + 17ll * i; }
};

// Phase 1 of fit_similarity (bundling.cpp:69-92): centroid and covariance
// B = sum (s * sbar) R Rbar^T + (c - mu) cbar^T (warp tree reductions), degenerate test.
__device__ __forceinline__ ShapeState shape_begin(const World& w, const Groups& g, const double* X, int grp, int lane,
                                                  const ShapeCache* sc, unsigned long long* tr) {
  using namespace vm;
  ShapeState st;
  st.grp = grp;
  st.ci = -1;
  if (sc)
    for (int k = 0; k < sc->ng; ++k)
      if (sc->gid[k] == grp) st.ci = k;
  const int ci = st.ci;
  st.m0 = ci >= 0 ? sc->m0[ci] : g.off[grp];
  st.m1 = ci >= 0 ? sc->m1[ci] : g.off[grp + 1];
  st.lb = ci >= 0 ? sc->base[ci] - st.m0 : 0;  // member m -> cache line m + lb
  const ShapeMembers M{g, sc, ci, st.lb};
  const int m0 = st.m0, m1 = st.m1;
  const int n = m1 - m0;
  const long long vp = w.vpad;
  auto ldc = [&](int v) { return V3{X[CX * vp + v], X[CY * vp + v], X[CZ * vp + v]}; };
  auto ldq = [&](int v) { return Q4{X[QW * vp + v], X[QX * vp + v], X[QY * vp + v], X[QZ * vp + v]}; };
  // The lane's first member's state is loaded once, all loads in flight together, and reused by
  // the three passes (members beyond 32 per group are reloaded).
  const int i0 = m0 + lane;
  st.c0 = V3{0, 0, 0};
  st.s0 = 0.0;
  st.q0 = Q4{1, 0, 0, 0};
  if (i0 < m1) {
    const int v = M.slot(i0), e = M.eslot(i0);
    st.c0 = ldc(v);
    st.s0 = X[S * vp + v];
    st.q0 = ldq(e);
  }
  // centroid of the current member centers
  V3 sum = st.c0;
  for (int i = i0 + 32; i < m1; i += 32) sum = sum + ldc(M.slot(i));
  st.cent = V3{shape_wsum(sum.x), shape_wsum(sum.y), shape_wsum(sum.z)} / static_cast<double>(n);
  if (tr && lane == 0) tr[1] = gtimer();
  double Bp[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = i0; i < m1; i += 32) {
    const double* mr = M.rest(i);
    const bool first = i == i0;
    const int v = first ? 0 : M.slot(i);
    const V3 c = (first ? st.c0 : ldc(v)) - st.cent;
    const double s = first ? st.s0 : X[S * vp + v];
    const M3 R = qmat(first ? st.q0 : ldq(M.eslot(i)));
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
  double sq[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      st.B.m[a][b] = shape_wsum(Bp[3 * a + b]);
      sq[a + 3 * b] = st.B.m[a][b] * st.B.m[a][b];
    }
  if (tr && lane == 0) tr[2] = gtimer();
  const double denom = ci >= 0 ? sc->grest[ci][3] : g.grest[4ll * grp + 3];
  st.degenerate = sqrt(sum9(sq)) < 1e-12 || denom < 1e-300;  // bundling.cpp:86-90
  return st;
}

// Phase 3 (bundling.cpp:94-133): scale numerator with the extracted rotation q, translation,
// projection of the members, warm rotation, optional fit record.
__device__ __forceinline__ void shape_end(const World& w, const Groups& g, double* X, double* xrec, const ShapeState& st,
                                          const vm::Q4& q, int lane, const ShapeCache* sc, unsigned long long* tr,
                                          double* fit) {
  using namespace vm;
  const ShapeMembers M{g, sc, st.ci, st.lb};
  const int m0 = st.m0, m1 = st.m1, grp = st.grp, i0 = m0 + lane;
  const long long vp = w.vpad;
  auto ldc = [&](int v) { return V3{X[CX * vp + v], X[CY * vp + v], X[CZ * vp + v]}; };
  auto ldq = [&](int v) { return Q4{X[QW * vp + v], X[QX * vp + v], X[QY * vp + v], X[QZ * vp + v]}; };
  const double* gr = st.ci >= 0 ? sc->grest[st.ci] : g.grest + 4ll * grp;
  const double denom = gr[3];
  const M3 Rf = qmat(q);
  const V3 rcent{gr[0], gr[1], gr[2]};
  double numer = 0.0;
  for (int i = i0; i < m1; i += 32) {
    const double* mr = M.rest(i);
    const bool first = i == i0;
    const int v = first ? 0 : M.slot(i);
    const V3 c = (first ? st.c0 : ldc(v)) - st.cent;
    const double s = first ? st.s0 : X[S * vp + v];
    const M3 R = qmat(first ? st.q0 : ldq(M.eslot(i)));
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
  numer = shape_wsum(numer);
  if (tr && lane == 0) tr[4] = gtimer();
  const double scale = fmax(numer / denom, kMinScale);
  const V3 t = st.cent - scale * mvmul(Rf, rcent);
  const Q4 qf = qfrom_mat(Rf);
  auto apply = [&](int i) {
    const double* mr = M.rest(i);
    const int v = M.slot(i);
    if (!(st.ci >= 0 ? sc->pinned[i + st.lb] : w.pinned[v])) {
      const V3 x = scale * mvmul(Rf, V3{mr[0], mr[1], mr[2]} + rcent) + t;
      X[CX * vp + v] = x.x;
      X[CY * vp + v] = x.y;
      X[CZ * vp + v] = x.z;
      const double sn = fmax(scale * mr[3], kMinScale);
      X[S * vp + v] = sn;
      double2* xr = reinterpret_cast<double2*>(xrec + 8ll * v);
      xr[0] = make_double2(x.x, x.y);
      xr[1] = make_double2(x.z, sn);
    }
    // product of unit quaternions: unit to O(1e-16), renormalised by the series (tolerance-pinned)
    const Q4 fr = qnormalized_fast(qmul(qf, Q4{mr[13], mr[14], mr[15], mr[16]}));
    const int e = M.eslot(i);
    X[QW * vp + e] = fr.w;
    X[QX * vp + e] = fr.x;
    X[QY * vp + e] = fr.y;
    X[QZ * vp + e] = fr.z;
  };
  __syncwarp();
  if (st.ci >= 0 ? sc->serial[st.ci] : g.serial[grp]) {
    if (lane == 0)
      for (int i = m0; i < m1; ++i) apply(i);
  } else {
    for (int i = m0 + lane; i < m1; i += 32) apply(i);
  }
  if (tr && lane == 0) tr[5] = gtimer();
  if (fit && lane == 0) {
    const double rec[14] = {scale, t.x, t.y, t.z, Rf.m[0][0], Rf.m[0][1], Rf.m[0][2], Rf.m[1][0], Rf.m[1][1],
                            Rf.m[1][2], Rf.m[2][0], Rf.m[2][1], Rf.m[2][2], 0.0};
    for (int k = 0; k < 14; ++k) fit[k] = rec[k];
  }
  if (lane == 0) {
    double* wo = g.warm + 4ll * grp;
    wo[0] = q.w;
    wo[1] = q.x;
    wo[2] = q.y;
    wo[3] = q.z;
  }
}

// The degenerate group's fit record (scale 1, identity, t = mu - mubar; bundling.cpp:86-90).
__device__ __forceinline__ void shape_degenerate_fit(const Groups& g, const ShapeCache* sc, const ShapeState& st,
                                                     int lane, double* fit) {
  if (!fit || lane != 0) return;
  const double* gr = st.ci >= 0 ? sc->grest[st.ci] : g.grest + 4ll * st.grp;
  const vm::V3 t = st.cent - vm::V3{gr[0], gr[1], gr[2]};
  const double rec[14] = {1.0, t.x, t.y, t.z, 1, 0, 0, 0, 1, 0, 0, 0, 1, 1.0};
  for (int k = 0; k < 14; ++k) fit[k] = rec[k];
}

// ---- exact-order variant (Groups::exact, VROD_SHAPE_EXACT) -----------------------------------
// The reference's arithmetic in the reference's order: every member sum is sequential in member
// order (all lanes run the same serial accumulation, reading member i's terms from lane i by
// shuffle), the rotation extraction is bundling.cpp:50-67 verbatim (division by |dot| + 1e-9,
// norm, Quaternion(AngleAxis) with correctly rounded sin / cos, crtrig.cuh, normalized()), and the
// projection uses the exact normalisation. Compiled --fmad=false like every kernel, so the result
// equals the reference bit for bit wherever glibc's sin / cos are correctly rounded.

// std::max(v, kMinScale) (NaN propagates, unlike fmax)
__device__ __forceinline__ double max_min_scale(double v) { return v < vm::kMinScale ? vm::kMinScale : v; }

// extract_rotation, bundling.cpp:50-67, in the reference's operation order (IEEE division and
// square root are correctly rounded, like the CPU's). kDevSin: CUDA's sincos instead of the
// correctly rounded one (diagnostics only: not the reference's bits).
template <bool kDevSin = false>
static __device__ __noinline__ vm::Q4 extract_rotation_exact(const vm::M3& B, const vm::Q4& guess, int* iters = nullptr,
                                                             int max_iterations = 100, double tolerance = 1e-9) {
  using namespace vm;
  // Eigen normalized(): coefficient / sqrt(squaredNorm) when it is > 0 (correctly rounded, rnops.cuh)
  auto normalized_rn = [](const Q4& p) {
    const double n = qsqnorm(p);
    if (n <= 0.0) return p;
    const double a[4] = {p.w, p.x, p.y, p.z};
    double o[4];
    rn::div_by(a, sqrt(n), o);
    return Q4{o[0], o[1], o[2], o[3]};
  };
  Q4 q = normalized_rn(guess);
  int it = 0;
#pragma unroll 1
  for (; it < max_iterations; ++it) {
    const M3 R = qmat(q);
    V3 omega{0, 0, 0};
    double d = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      omega = omega + cross(col(R, a), col(B, a));
      d += dot(col(R, a), col(B, a));
    }
    double w[3];
    rn::div_by({omega.x, omega.y, omega.z}, fabs(d) + 1e-9, w);
    const double angle = sqrt((w[0] * w[0] + w[1] * w[1]) + w[2] * w[2]);  // norm()
    if (angle < tolerance) break;
    double ax[3];
    rn::div_by(w, angle, ax);
    crt::DD sc;
    if (kDevSin)
      sincos(0.5 * angle, &sc.hi, &sc.lo);
    else
      sc = crt::sincos_rn(0.5 * angle);  // Quaternion(AngleAxisd(angle, axis)): (cos, sin * axis)
    q = normalized_rn(qmul(Q4{sc.lo, sc.hi * ax[0], sc.hi * ax[1], sc.hi * ax[2]}, q));
  }
  if (iters) *iters = it;
  return q;
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// Doubles of per-warp scratch the exact path uses for its ordered sums (32 members x 18 terms).
constexpr int kShapeScratch = 32 * 18;

// Ordered (member-sequential) accumulation of a 32-member chunk: lane j holds member j's N terms
// v[0..N); accumulator e (< E, held by lane e) adds, for j = 0 .. cnt-1 in order, the terms
// v_j[e], v_j[e + E], .. (K = N / E terms per member, in that order). With a scratch buffer the
// chunk is transposed through shared memory and the E serial chains run on E lanes side by side;
// without one, every lane runs every chain on shuffled values (same order, same bits, slower).
template <int N, int E>
__device__ __forceinline__ void ordered_accumulate(const double (&v)[N], int cnt, int lane, double* scratch,
                                                   double (&acc)[E]) {
  constexpr int K = N / E;
  if (scratch) {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < N; ++i) scratch[lane * N + i] = v[i];
    __syncwarp();
    if (lane < E) {
      double a = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e == lane) a = acc[e];
#pragma unroll 8
      for (int j = 0; j < cnt; ++j)
#pragma unroll
        for (int k = 0; k < K; ++k) a = a + scratch[j * N + lane + k * E];
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e == lane) acc[e] = a;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = shfl_d(acc[e], e);
  } else {
    for (int j = 0; j < cnt; ++j)
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = acc[e] + shfl_d(v[e + k * E], j);
  }
}

// One member's state and static data, loaded by the lane that owns it in a 32-member chunk.
struct ExactMember {
  vm::V3 c;   // current center (minus the centroid once known)
  double s;
  vm::M3 R;   // current frame as a matrix
  const double* mr;
};

__device__ __forceinline__ ExactMember exact_load(const ShapeMembers& M, const double* X, long long vp, int i) {
  using namespace vm;
  ExactMember e;
  const int v = M.slot(i), el = M.eslot(i);
  e.c = V3{X[CX * vp + v], X[CY * vp + v], X[CZ * vp + v]};
  e.s = X[S * vp + v];
  e.R = qmat(Q4{X[QW * vp + el], X[QX * vp + el], X[QY * vp + el], X[QZ * vp + el]});
  e.mr = M.rest(i);
  return e;
}

static __device__ __forceinline__ void shape_group_exact(const World& w, const Groups& g, double* X, double* xrec, int grp, int lane,
                                  const ShapeCache* sc, double* fit, unsigned long long* tr = nullptr,
                                  double* scratch = nullptr) {
  using namespace vm;
  if (tr && lane == 0) tr[0] = gtimer();
  int ci = -1;
  if (sc)
    for (int k = 0; k < sc->ng; ++k)
      if (sc->gid[k] == grp) ci = k;
  const int m0 = ci >= 0 ? sc->m0[ci] : g.off[grp], m1 = ci >= 0 ? sc->m1[ci] : g.off[grp + 1];
  const int lb = ci >= 0 ? sc->base[ci] - m0 : 0;
  const ShapeMembers M{g, sc, ci, lb};
  const long long vp = w.vpad;
  const int n = m1 - m0;
  const double* gr = ci >= 0 ? sc->grest[ci] : g.grest + 4ll * grp;
  const V3 rcent{gr[0], gr[1], gr[2]};
  const double denom = gr[3];
  // centroid (bundling.cpp:73-75): sequential sum, then division by n
  double cacc[3] = {0.0, 0.0, 0.0};
  for (int b = m0; b < m1; b += 32) {
    const int i = b + lane, cnt = min(32, m1 - b);
    double c[3] = {0.0, 0.0, 0.0};
    if (i < m1) {
      const int v = M.slot(i);
      c[0] = X[CX * vp + v];
      c[1] = X[CY * vp + v];
      c[2] = X[CZ * vp + v];
    }
    ordered_accumulate<3, 3>(c, cnt, lane, scratch, cacc);
  }
  const V3 cent = V3{cacc[0], cacc[1], cacc[2]} / static_cast<double>(n);
  if (tr && lane == 0) tr[1] = gtimer();
  // covariance (:77-85): B += (s * s_rest) R R_rest^T; B += c c_rest^T, member after member
  double bacc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = m0; b < m1; b += 32) {
    const int i = b + lane, cnt = min(32, m1 - b);
    double PO[18];  // the member's (s s_rest) R R_rest^T, then c c_rest^T, row-major
#pragma unroll
    for (int k = 0; k < 18; ++k) PO[k] = 0.0;
    if (i < m1) {
      const ExactMember e = exact_load(M, X, vp, i);
      const V3 c = e.c - cent;
      const double ss = e.s * e.mr[3];
      M3 A, rR;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          A.m[a][q] = ss * e.R.m[a][q];
          rR.m[a][q] = e.mr[4 + 3 * a + q];
        }
      const M3 Pm = mmul_bt(A, rR);
      const double cv[3] = {c.x, c.y, c.z};
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          PO[3 * a + q] = Pm.m[a][q];
          PO[9 + 3 * a + q] = cv[a] * e.mr[q];
        }
    }
    if (tr && lane == 0 && b == m0) tr[7] = gtimer();
    ordered_accumulate<18, 9>(PO, cnt, lane, scratch, bacc);
  }
  M3 B;
#pragma unroll
  for (int k = 0; k < 9; ++k) B.m[k / 3][k % 3] = bacc[k];
  double sq[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q) sq[a + 3 * q] = B.m[a][q] * B.m[a][q];
  if (sqrt(sum9(sq)) < 1e-12 || denom < 1e-300) {  // degenerate (:86-90): no write
    if (fit && lane == 0) {
      const V3 t = cent - rcent;
      const double rec[14] = {1.0, t.x, t.y, t.z, 1, 0, 0, 0, 1, 0, 0, 0, 1, 1.0};
      for (int k = 0; k < 14; ++k) fit[k] = rec[k];
    }
    return;
  }
  if (tr && lane == 0) tr[2] = gtimer();
  double* wq = g.warm + 4ll * grp;
  int nit = 0;
  const Q4 q = extract_rotation_exact(B, Q4{wq[0], wq[1], wq[2], wq[3]}, &nit);
  if (tr && lane == 0) {
    tr[3] = gtimer();
    tr[6] = nit;
  }
  const M3 Rf = qmat(q);
  // scale numerator (:97-108), sequential
  double nacc[1] = {0.0};
  for (int b = m0; b < m1; b += 32) {
    const int i = b + lane, cnt = min(32, m1 - b);
    double tt[2] = {0.0, 0.0};
    if (i < m1) {
      const ExactMember e = exact_load(M, X, vp, i);
      const V3 c = e.c - cent;
      M3 rR;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int r = 0; r < 3; ++r) rR.m[a][r] = e.mr[4 + 3 * a + r];
      const M3 RR = mmul(Rf, rR);
      double el[9];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int r = 0; r < 3; ++r) el[a + 3 * r] = RR.m[a][r] * e.R.m[a][r];
      tt[0] = (e.s * e.mr[3]) * sum9(el);
      tt[1] = dot(c, mvmul(Rf, V3{e.mr[0], e.mr[1], e.mr[2]}));
    }
    ordered_accumulate<2, 1>(tt, cnt, lane, scratch, nacc);
  }
  const double numer = nacc[0];
  if (tr && lane == 0) tr[4] = gtimer();
  const double scale = max_min_scale(numer / denom);
  const V3 t = cent - scale * mvmul(Rf, rcent);
  const Q4 qf = qfrom_mat(Rf);
  // projection (apply_shape_match, :116-133)
  auto apply = [&](int i) {
    const double* mr = M.rest(i);
    const int v = M.slot(i);
    if (!(ci >= 0 ? sc->pinned[i + lb] : w.pinned[v])) {
      const V3 x = scale * mvmul(Rf, V3{mr[0], mr[1], mr[2]} + rcent) + t;
      X[CX * vp + v] = x.x;
      X[CY * vp + v] = x.y;
      X[CZ * vp + v] = x.z;
      const double sn = max_min_scale(scale * mr[3]);
      X[S * vp + v] = sn;
      double2* xr = reinterpret_cast<double2*>(xrec + 8ll * v);
      xr[0] = make_double2(x.x, x.y);
      xr[1] = make_double2(x.z, sn);
    }
    const Q4 fr = qnormalized(qmul(qf, Q4{mr[13], mr[14], mr[15], mr[16]}));
    const int e = M.eslot(i);
    X[QW * vp + e] = fr.w;
    X[QX * vp + e] = fr.x;
    X[QY * vp + e] = fr.y;
    X[QZ * vp + e] = fr.z;
  };
  __syncwarp();
  if (ci >= 0 ? sc->serial[ci] : g.serial[grp]) {
    if (lane == 0)
      for (int i = m0; i < m1; ++i) apply(i);
  } else {
    for (int i = m0 + lane; i < m1; i += 32) apply(i);
  }
  if (tr && lane == 0) tr[5] = gtimer();
  if (fit && lane == 0) {
    const double rec[14] = {scale, t.x, t.y, t.z, Rf.m[0][0], Rf.m[0][1], Rf.m[0][2], Rf.m[1][0], Rf.m[1][1],
                            Rf.m[1][2], Rf.m[2][0], Rf.m[2][1], Rf.m[2][2], 0.0};
    for (int k = 0; k < 14; ++k) fit[k] = rec[k];
  }
  if (lane == 0) {
    wq[0] = q.w;
    wq[1] = q.x;
    wq[2] = q.y;
    wq[3] = q.z;
  }
}

// Fit and apply group `grp` (apply_shape_match, bundling.cpp:116-133) on the state rows X and
// the slot records xrec, all phases in one warp (the rotation extraction redundantly in every
// lane). tr: optional phase timestamps; sc: optional shared-memory copy of the group's statics;
// fit: optional SimilarityFit record (bundling.h:18-23), 14 doubles: scale, translation xyz,
// rotation (row-major 3x3), degenerate flag.
// kMode: 0 the latency-tuned path, 1 the exact-order path, -1 chosen by Groups::exact at run time.
template <int kMode = -1>
__device__ __forceinline__ void shape_group(const World& w, const Groups& g, double* X, double* xrec, int grp,
                                            int lane, unsigned long long* tr = nullptr, const ShapeCache* sc = nullptr,
                                            double* fit = nullptr, double* scratch = nullptr) {
  if (kMode == 1 || (kMode < 0 && g.exact)) {
    shape_group_exact(w, g, X, xrec, grp, lane, sc, fit, tr, scratch);
    return;
  }
  if (tr && lane == 0) tr[0] = gtimer();
  const ShapeState st = shape_begin(w, g, X, grp, lane, sc, tr);
  if (st.degenerate) {
    shape_degenerate_fit(g, sc, st, lane, fit);
    return;
  }
  const double* wq = g.warm + 4ll * grp;
  int nit = 0;
  const vm::Q4 q = extract_rotation(st.B, vm::Q4{wq[0], wq[1], wq[2], wq[3]}, &nit);
  if (tr && lane == 0) {
    tr[3] = gtimer();
    tr[6] = nit;
  }
  shape_end(w, g, X, xrec, st, q, lane, sc, tr, fit);
}

}  // namespace vdev
