// One external block (soft pin | pill contact | half-plane, the tail of the reference's block
// list, solver.cpp:324-328) evaluated and solved against a snapshot: residual + Jacobian
// (eval_constraint, constraints.cpp:215-267) and the generalized XPBD update (solve_block,
// :400-487). Shared by the per-block kernel k_ext_solve (sweep.cu), which writes every endpoint's
// correction into its slot-sorted incidence entry, and by the persistent small-world iteration
// kernel (rodsweep.cu), where each endpoint's gather re-solves the block itself and only the
// block's owner entry commits the multiplier.
#pragma once

#include "kernels.cuh"
#include "vmath.cuh"

namespace vdev {

struct ExtGeom {  // resolve_pill, constraints.cpp:76-97
  vm::V3 c0, c1;
  double r0, r1, rb0, rb1;
  int v0;
};

// Resolve from the 64-byte slot records (World::xrec): two records per rod pill.
__device__ __forceinline__ ExtGeom resolve_rec(const double* xrec, const Collide& c, int pill, int v, double (&ic)[2],
                                               double (&is)[2]) {
  ExtGeom g;
  if (v >= 0) {
    const double4* r0 = reinterpret_cast<const double4*>(xrec + 8ll * v);
    const double4 a = r0[0], b = r0[1], d = r0[2], e = r0[3];
    g.c0 = vm::V3{a.x, a.y, a.z};
    g.c1 = vm::V3{d.x, d.y, d.z};
    g.rb0 = b.x;
    g.rb1 = e.x;
    g.r0 = a.w * g.rb0;
    g.r1 = d.w * g.rb1;
    g.v0 = v;
    ic[0] = b.y;
    ic[1] = e.y;
    is[0] = b.z;
    is[1] = e.z;
  } else {
    g.c0 = vm::V3{c.pill[8ll * pill], c.pill[8ll * pill + 1], c.pill[8ll * pill + 2]};
    g.c1 = vm::V3{c.pill[8ll * pill + 3], c.pill[8ll * pill + 4], c.pill[8ll * pill + 5]};
    g.r0 = c.pill[8ll * pill + 6];
    g.r1 = c.pill[8ll * pill + 7];
    g.rb0 = g.rb1 = 0.0;
    g.v0 = -1;
    ic[0] = ic[1] = is[0] = is[1] = 0.0;
  }
  return g;
}

// Result of one external block: the multipliers after the block, whether it was singular
// (skipped) or produced a non-finite update. Every endpoint e that has an incidence entry
// (pins / half-planes: e = 0; contacts: 0,1 = pill A's slots, 2,3 = pill B's) is reported
// exactly once through emit(e, flag, dx, dy, dz, ds), flag 0 = no update, kExtCenter, or
// kExtCenter | kExtScale.
struct ExtResult {
  double lam[3];
  double rec[4];  // the block's record for Collide::ext_rec (see there)
  int nlam;
  int owner;  // endpoint whose entry commits the block (lowest existing endpoint)
  bool singular, bad;
};

// The per-substep constants of a contact block (solver.cpp:210-224): its pills, their first
// slots (-1: kinematic), the frozen alpha / beta.
struct ContactRef {
  int a, b, va, vb;
  double al, be;
};
__device__ __forceinline__ ContactRef contact_ref(const Collide& c, int k) {
  return ContactRef{c.ct_a[k], c.ct_b[k], c.ct_va[k], c.ct_vb[k], c.ct_alpha[k], c.ct_beta[k]};
}

__device__ __forceinline__ double xget(const double* X, int f, int vp, int v) { return X[static_cast<long long>(f) * vp + v]; }

// X: snapshot state rows (pins / half-planes); xrec: the matching slot records (contacts);
// lam: the multipliers before the sweep, SoA (component d of block b at lam[d * ls + b]);
// pre: the contact's constants if the caller has them at hand (else read from `c`); nct: the
// substep's contact count (c.scalars[SC_NCT], read once by the caller: a dependent load less).
template <class Emit>
__device__ __forceinline__ ExtResult ext_block(const World& w, const Collide& c, const double* X, const double* xrec,
                                               const double* lam, long long ls, int b, const SweepParams& sp,
                                               Emit&& emit, const ContactRef* pre, int nct) {
  using namespace vm;
  ExtResult r;
  r.singular = r.bad = false;
  r.owner = 0;
  r.rec[0] = r.rec[1] = r.rec[2] = r.rec[3] = ext_none();
  const int npins = sp.n_pins;
  const int vp = w.vpad;
  const double h2 = sp.h2;
  bool active = false, finite = true;
  if (b < npins) {  // kPin (constraints.cpp:261-267), dim 3
    r.nlam = 3;
    const int v = c.pin_slot[b];
    const double* pd = c.pin_data + 4 * b;
    const V3 x{xget(X, CX, vp, v), xget(X, CY, vp, v), xget(X, CZ, vp, v)};
    const double W[3] = {x.x - pd[0], x.y - pd[1], x.z - pd[2]};
    const double ic = xget(w.vstat, IC, vp, v);
    double M[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (ic != 0.0) {
      const double s = h2 * ic;
      M[0][0] = s;
      M[1][1] = s;
      M[2][2] = s;
    }
    const double kinv = inverse_stiffness(pd[3]);
    double rhs[3], dl[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      r.lam[d] = lam[d * ls + b];
      M[d][d] = M[d][d] + kinv;
      rhs[d] = W[d] - kinv * r.lam[d];
    }
    if (!solve3(M, rhs, sp.beta, dl)) {
      r.singular = true;
      emit(0, 0, 0.0, 0.0, 0.0, 0.0);
    } else {
      active = true;
      const double f = -h2 * ic;
      double o[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        r.lam[d] = r.lam[d] + dl[d];
        o[d] = f * dl[d];
        finite = finite && isfinite(dl[d]) && isfinite(o[d]);
        r.rec[d] = o[d];
      }
      emit(0, kExtCenter, o[0], o[1], o[2], 0.0);
    }
  } else if (b < npins + nct) {  // kContact (constraints.cpp:215-247), unilateral, dim 1
    r.nlam = 1;
    const int k = b - npins;
    // endpoint slots were stored by k_ext_count: the slot records are one dependent load away
    double icA[2], isA[2], icB[2], isB[2];
    const ContactRef cr = pre ? *pre : contact_ref(c, k);
    const ExtGeom A = resolve_rec(xrec, c, cr.a, cr.va, icA, isA);
    const ExtGeom B = resolve_rec(xrec, c, cr.b, cr.vb, icB, isB);
    const double al = cr.al, be = cr.be;
    const V3 ca = (1.0 - al) * A.c0 + al * A.c1;
    const V3 cb = (1.0 - be) * B.c0 + be * B.c1;
    const double ra = (1.0 - al) * A.r0 + al * A.r1;
    const double rb = (1.0 - be) * B.r0 + be * B.r1;
    V3 nrm = ca - cb;
    const double dist = norm(nrm);
    const bool live = dist >= 1e-12;
    double W = 0.0;
    if (live) {
      nrm = nrm / dist;
      W = dist - ra - rb;
    }
    bool wrote[4] = {false, false, false, false};
    r.owner = A.v0 >= 0 ? 0 : 2;
    const double icv[4] = {icA[0], icA[1], icB[0], icB[1]}, isv[4] = {isA[0], isA[1], isB[0], isB[1]};
    r.lam[0] = lam[b];
    if (!(W >= 0.0 && r.lam[0] == 0.0)) {
      const double coef[4] = {1.0 - al, al, -(1.0 - be), -be};
      const double sj[4] = {-(1.0 - al) * A.rb0, -al * A.rb1, -(1.0 - be) * B.rb0, -be * B.rb1};
      const bool has[4] = {live && A.v0 >= 0, live && A.v0 >= 0, live && B.v0 >= 0, live && B.v0 >= 0};
      double M = 0.0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // centers
        if (!has[e]) continue;
        const double ic = icv[e];
        if (ic == 0.0) continue;
        const double s = h2 * ic;
        const V3 j = coef[e] * nrm;
        M = M + (((s * j.x) * j.x + (s * j.y) * j.y) + (s * j.z) * j.z);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // scales
        if (!has[e]) continue;
        const double is = isv[e];
        if (is == 0.0) continue;
        M = M + (h2 * is * sj[e]) * sj[e];
      }
      const double kinv = sp.contact_kinv;
      M = M + kinv;
      const double rhs = W - kinv * r.lam[0];
      if (M <= 1e-250) {
        r.singular = true;
      } else {
        double dl = sp.beta * rhs / M;
        if (r.lam[0] + dl > 0.0) dl = -r.lam[0];
        active = true;
        r.lam[0] = r.lam[0] + dl;
        finite = isfinite(dl);
        if (live) {
          r.rec[0] = nrm.x;
          r.rec[1] = nrm.y;
          r.rec[2] = nrm.z;
          r.rec[3] = dl;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (!has[e]) continue;
          const V3 j = coef[e] * nrm;
          const double fc = -h2 * icv[e];
          const double ox = fc * (j.x * dl), oy = fc * (j.y * dl), oz = fc * (j.z * dl);
          const double os = -h2 * isv[e] * (sj[e] * dl);
          finite = finite && isfinite(ox) && isfinite(oy) && isfinite(oz) && isfinite(os);
          emit(e, kExtCenter | kExtScale, ox, oy, oz, os);
          wrote[e] = true;
        }
      }
    }
    const bool entry[4] = {A.v0 >= 0, A.v0 >= 0, B.v0 >= 0, B.v0 >= 0};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (entry[e] && !wrote[e]) emit(e, 0, 0.0, 0.0, 0.0, 0.0);
  } else {  // kHalfPlane (constraints.cpp:248-260), unilateral, dim 1
    r.nlam = 1;
    const int k = b - npins - nct;
    const int v = c.hp_slot[k];
    const double* pl = c.planes + 4 * c.hp_plane[k];
    const V3 n3{pl[0], pl[1], pl[2]};
    const double rbar = xget(w.vstat, RBAR, vp, v);
    const V3 x{xget(X, CX, vp, v), xget(X, CY, vp, v), xget(X, CZ, vp, v)};
    const double W = dot(n3, x) - pl[3] - xget(X, S, vp, v) * rbar;
    r.lam[0] = lam[b];
    if (!(W >= 0.0 && r.lam[0] == 0.0)) {
      const double ic = xget(w.vstat, IC, vp, v), is = xget(w.vstat, IS, vp, v);
      double M = 0.0;
      if (ic != 0.0) {
        const double s = h2 * ic;
        M = M + (((s * n3.x) * n3.x + (s * n3.y) * n3.y) + (s * n3.z) * n3.z);
      }
      if (is != 0.0) M = M + (h2 * is * -rbar) * -rbar;
      const double kinv = sp.contact_kinv;
      M = M + kinv;
      const double rhs = W - kinv * r.lam[0];
      if (M <= 1e-250) {
        r.singular = true;
      } else {
        double dl = sp.beta * rhs / M;
        if (r.lam[0] + dl > 0.0) dl = -r.lam[0];
        active = true;
        r.lam[0] = r.lam[0] + dl;
        const double fc = -h2 * ic;
        const double ox = fc * (n3.x * dl), oy = fc * (n3.y * dl), oz = fc * (n3.z * dl);
        const double os = -h2 * is * (-rbar * dl);
        finite = isfinite(dl) && isfinite(ox) && isfinite(oy) && isfinite(oz) && isfinite(os);
        r.rec[0] = ox;
        r.rec[1] = oy;
        r.rec[2] = oz;
        r.rec[3] = os;
        emit(0, kExtCenter | kExtScale, ox, oy, oz, os);
      }
    }
    if (!active) emit(0, 0, 0.0, 0.0, 0.0, 0.0);
  }
  r.bad = active && !finite;
  return r;
}

// Endpoint e's correction of a contact from its block record {n xyz, dl} (Collide::ext_rec): the
// expressions of ext_block's emission loop above, operand for operand, with the endpoint slot's
// own inverse weights and rest radius and the contact's alpha (e < 2) or beta (e >= 2).
__device__ __forceinline__ void contact_endpoint(int e, double ab, double nx, double ny, double nz, double dl, double h2,
                                                 double ic, double is, double rb, double (&o)[3], double& os) {
  const double coef = e == 0 ? 1.0 - ab : e == 1 ? ab : e == 2 ? -(1.0 - ab) : -ab;  // coef[e]
  const double sj = (e < 2 ? -coef : coef) * rb;                                      // sj[e]
  const double jx = coef * nx, jy = coef * ny, jz = coef * nz;
  const double fc = -h2 * ic;
  o[0] = fc * (jx * dl);
  o[1] = fc * (jy * dl);
  o[2] = fc * (jz * dl);
  os = -h2 * is * (sj * dl);
}

// Scene of external block b (batch only).
__device__ __forceinline__ int ext_scene(const World& w, const Collide& c, int b, int npins, int nct) {
  if (b < npins) return w.rod_scene[w.slot_rod[c.pin_slot[b]]];
  if (b < npins + nct) return c.pill_scene[c.ct_a[b - npins]];
  return c.plane_scene[c.hp_plane[b - npins - nct]];
}

}  // namespace vdev
