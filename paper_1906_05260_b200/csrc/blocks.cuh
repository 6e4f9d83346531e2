// The eight elastic block kinds of one rod position (eval_constraint, constraints.cpp:101-270, +
// solve_block, :400-487), each a pure function of its inputs: the tile sweep (rodsweep.cu
// solve_items, inputs from shared-memory rows) and the warp-per-rod sweep (rodwarp.cu, inputs in
// registers and from neighbouring lanes) call the same code, so both give the same bits. Every
// expression keeps the reference's operation order (compiled --fmad=false).
//
// Each solver returns true when the block was solved (active) and false when it was skipped as
// singular (the multipliers are then kept); `ok` is cleared when a result is non-finite (the
// reference's SimulationError "non-finite update from constraint ...", constraints.cpp:517-518).
#pragma once

#include "vmath.cuh"

namespace vdev {
namespace blk {

using namespace vm;

// StretchZ of element k (:106-119), dim 3. dt[2] is always 0.
__device__ __forceinline__ bool stretch_z(const V3& c0, const V3& c1, double ic0, double ic1, const V3& it, const Q4& q,
                                          double tbar, double l, double kinv, const double (&lam)[3], double h2,
                                          double beta, double (&dc0)[3], double (&dc1)[3], double (&dt)[3],
                                          double (&lam_out)[3], bool& ok) {
  const M3 Rm = qmat(q);
  const Recip rl = recip(l);
  const double inv_l = rinv(rl);
  const V3 d = c1 - c0;
  const V3 dzc{divr(d.x, rl), divr(d.y, rl), divr(d.z, rl)};
  const V3 wv = col(Rm, 2);
  const double W[3] = {dzc.x - tbar * wv.x, dzc.y - tbar * wv.y, dzc.z - tbar * wv.z};
  const double J0[3] = {tbar * Rm.m[0][1], tbar * Rm.m[1][1], tbar * Rm.m[2][1]};
  const double J1[3] = {-tbar * Rm.m[0][0], -tbar * Rm.m[1][0], -tbar * Rm.m[2][0]};
  double M[3][3];
  double cd = 0.0;
  if (ic0 != 0.0) cd = cd + (h2 * ic0 * inv_l) * inv_l;
  if (ic1 != 0.0) cd = cd + (h2 * ic1 * inv_l) * inv_l;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double b0 = (h2 * J0[a]) * it.x, b1 = (h2 * J1[a]) * it.y;
#pragma unroll
    for (int b = 0; b < 3; ++b) M[a][b] = (a == b ? cd : 0.0) + (b0 * J0[b] + b1 * J1[b]);
  }
  double rhs[3], dl[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    M[d][d] = M[d][d] + kinv;
    rhs[d] = W[d] - kinv * lam[d];
  }
  if (!solve3(M, rhs, beta, dl)) return false;
  const double f0 = -h2 * ic0, f1 = -h2 * ic1;
  bool fin = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    dc0[d] = f0 * (-inv_l * dl[d]);
    dc1[d] = f1 * (inv_l * dl[d]);
    fin = fin && isfinite(dl[d]) && isfinite(dc0[d]) && isfinite(dc1[d]);
  }
  const double jt0 = (J0[0] * dl[0] + J0[1] * dl[1]) + J0[2] * dl[2];
  const double jt1 = (J1[0] * dl[0] + J1[1] * dl[1]) + J1[2] * dl[2];
  dt[0] = -h2 * (it.x * jt0);
  dt[1] = -h2 * (it.y * jt1);
  dt[2] = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) lam_out[d] = lam[d] + dl[d];
  ok = fin && isfinite(dt[0]) && isfinite(dt[1]);
  return true;
}

// CrossSection of element k (:120-129), dim 1.
__device__ __forceinline__ bool cross_section(double s0, double s1, double sbar0, double sbar1, double is0, double is1,
                                              double kinv, double lam, double h2, double beta, double (&ds)[2],
                                              double& lam_out, bool& ok) {
  const double W = 0.5 * (s0 + s1) - 0.5 * (sbar0 + sbar1);
  double M = 0.0;
  if (is0 != 0.0) M = M + (h2 * is0 * 0.5) * 0.5;
  if (is1 != 0.0) M = M + (h2 * is1 * 0.5) * 0.5;
  M = M + kinv;
  if (!(M > 1e-250)) return false;
  const double dl = qdiv(beta * (W - kinv * lam), M);
  ds[0] = -h2 * is0 * (0.5 * dl);
  ds[1] = -h2 * is1 * (0.5 * dl);
  lam_out = lam + dl;
  ok = isfinite(dl) && isfinite(ds[0]) && isfinite(ds[1]);
  return true;
}

// SurfaceStretch of element k (:130-138), dim 1.
__device__ __forceinline__ bool surface_stretch(double s0, double s1, double l, double sgrad, double is0, double is1,
                                                double kinv, double lam, double h2, double beta, double (&ds)[2],
                                                double& lam_out, bool& ok) {
  const Recip rl = recip(l);
  const double W = divr(s1 - s0, rl) - sgrad;
  const double j1 = rinv(rl), j0 = -j1;  // -1.0 / l == -(1.0 / l) under round-to-nearest
  double M = 0.0;
  if (is0 != 0.0) M = M + (h2 * is0 * j0) * j0;
  if (is1 != 0.0) M = M + (h2 * is1 * j1) * j1;
  M = M + kinv;
  if (!(M > 1e-250)) return false;
  const double dl = qdiv(beta * (W - kinv * lam), M);
  ds[0] = -h2 * is0 * (j0 * dl);
  ds[1] = -h2 * is1 * (j1 * dl);
  lam_out = lam + dl;
  ok = isfinite(dl) && isfinite(ds[0]) && isfinite(ds[1]);
  return true;
}

// VolumeStretch of element k (:169-188), dim 3. dt[2] is always 0.
__device__ __forceinline__ bool volume_stretch(const V3& c0, const V3& c1, double s0, double s1, double sbar0,
                                               double sbar1, double ic0, double ic1, double is0, double is1,
                                               const V3& it, const Q4& q, double tbar, double l0, double kinv,
                                               const double (&lam)[3], double h2, double beta, double (&dc0)[3],
                                               double (&dc1)[3], double (&ds)[2], double (&dt)[3],
                                               double (&lam_out)[3], bool& ok) {
  const M3 Rm = qmat(q);
  const double smid = 0.5 * (s0 + s1);
  const double smr = 0.5 * (sbar0 + sbar1);
  const Recip rl0 = recip(l0);
  const V3 d = c1 - c0;
  const V3 dzc{divr(d.x, rl0), divr(d.y, rl0), divr(d.z, rl0)};
  const V3 wv = col(Rm, 2);
  const double ka = smid * smid, kb = smr * smr * tbar;
  const double W[3] = {ka * dzc.x - kb * wv.x, ka * dzc.y - kb * wv.y, ka * dzc.z - kb * wv.z};
  const double jc = divr(smid * smid, rl0);
  const double js[3] = {smid * dzc.x, smid * dzc.y, smid * dzc.z};
  const double fac = -smr * smr * tbar;
  const double J0[3] = {fac * -Rm.m[0][1], fac * -Rm.m[1][1], fac * -Rm.m[2][1]};
  const double J1[3] = {fac * Rm.m[0][0], fac * Rm.m[1][0], fac * Rm.m[2][0]};
  double M[3][3];
  double cd = 0.0;
  if (ic0 != 0.0) cd = cd + (h2 * ic0 * jc) * jc;
  if (ic1 != 0.0) cd = cd + (h2 * ic1 * jc) * jc;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double sa0 = h2 * is0 * js[a], sa1 = h2 * is1 * js[a];
    const double b0 = (h2 * J0[a]) * it.x, b1 = (h2 * J1[a]) * it.y;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double v = a == b ? cd : 0.0;
      if (is0 != 0.0) v = v + sa0 * js[b];
      if (is1 != 0.0) v = v + sa1 * js[b];
      M[a][b] = v + (b0 * J0[b] + b1 * J1[b]);
    }
  }
  double rhs[3], dl[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    M[d][d] = M[d][d] + kinv;
    rhs[d] = W[d] - kinv * lam[d];
  }
  if (!solve3(M, rhs, beta, dl)) return false;
  const double f0 = -h2 * ic0, f1 = -h2 * ic1;
  bool fin = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    dc0[d] = f0 * (-jc * dl[d]);
    dc1[d] = f1 * (jc * dl[d]);
    fin = fin && isfinite(dl[d]) && isfinite(dc0[d]) && isfinite(dc1[d]);
  }
  const double jd = (js[0] * dl[0] + js[1] * dl[1]) + js[2] * dl[2];
  ds[0] = -h2 * is0 * jd;
  ds[1] = -h2 * is1 * jd;
  const double jt0 = (J0[0] * dl[0] + J0[1] * dl[1]) + J0[2] * dl[2];
  const double jt1 = (J1[0] * dl[0] + J1[1] * dl[1]) + J1[2] * dl[2];
  dt[0] = -h2 * (it.x * jt0);
  dt[1] = -h2 * (it.y * jt1);
  dt[2] = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) lam_out[d] = lam[d] + dl[d];
  ok = fin && isfinite(ds[0]) && isfinite(ds[1]) && isfinite(dt[0]) && isfinite(dt[1]);
  return true;
}

// relative rotation p = canon(conj(qa) qb) of vertex k's two elements; the derivative blocks
// Da / Db = 0.5 (-+p.w I + [p_v]x) (constraints.cpp:50-51) are formed from it where they are used
// (each entry is one exact product, so recomputing costs nothing and keeps them out of registers).
struct VertexFrame {
  Q4 pr;
  __device__ __forceinline__ double Da(int a, int b) const {
    const double m[3][3] = {{-pr.w, -pr.z, pr.y}, {pr.z, -pr.w, -pr.x}, {-pr.y, pr.x, -pr.w}};
    return 0.5 * m[a][b];
  }
  __device__ __forceinline__ double Db(int a, int b) const {
    const double m[3][3] = {{pr.w, -pr.z, pr.y}, {pr.z, pr.w, -pr.x}, {-pr.y, pr.x, pr.w}};
    return 0.5 * m[a][b];
  }
};
__device__ __forceinline__ VertexFrame vertex_frame(const Q4& qa, const Q4& qb, bool need) {
  VertexFrame f;
  f.pr = Q4{1, 0, 0, 0};
  if (need) f.pr = relative_rotation(qa, qb);
  return f;
}

// BendTwist of interior vertex k (:139-155), dim 3. classic: the scale slot is omitted (ds = 0).
__device__ __forceinline__ bool bend_twist(const VertexFrame& vf, double s0, double sbar, double is0, const V3& ita,
                                           const V3& itb, double la, double lb, const V3& darb, double kinv0,
                                           double kinv2, const double (&lam)[3], int classic, double h2, double beta,
                                           double& ds, double (&dta)[3], double (&dtb)[3], double (&lam_out)[3],
                                           bool& ok) {
  const double inv_len = 4.0 / (la + lb);
  const V3 om = inv_len * qvec(vf.pr);
  const double s = classic ? sbar : s0;
  const double W[3] = {s * om.x - sbar * darb.x, s * om.y - sbar * darb.y, s * om.z - sbar * darb.z};
  const double fs = s * inv_len;
  double Ja[3][3], Jb[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      Ja[a][b] = fs * vf.Da(a, b);
      Jb[a][b] = fs * vf.Db(a, b);
    }
  const double omv[3] = {om.x, om.y, om.z};
  const bool sc_on = !classic && is0 != 0.0;
  double M[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double sa = h2 * is0 * omv[a];
    const double ba0 = (h2 * Ja[a][0]) * ita.x, ba1 = (h2 * Ja[a][1]) * ita.y, ba2 = (h2 * Ja[a][2]) * ita.z;
    const double bb0 = (h2 * Jb[a][0]) * itb.x, bb1 = (h2 * Jb[a][1]) * itb.y, bb2 = (h2 * Jb[a][2]) * itb.z;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double v = sc_on ? sa * omv[b] : 0.0;
      v = v + ((ba0 * Ja[b][0] + ba1 * Ja[b][1]) + ba2 * Ja[b][2]);
      v = v + ((bb0 * Jb[b][0] + bb1 * Jb[b][1]) + bb2 * Jb[b][2]);
      M[a][b] = v;
    }
  }
  const double kinv[3] = {kinv0, kinv0, kinv2};
  double rhs[3], dl[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    M[d][d] = M[d][d] + kinv[d];
    rhs[d] = W[d] - kinv[d] * lam[d];
  }
  if (!solve3(M, rhs, beta, dl)) return false;
  bool fin = isfinite(dl[0]) && isfinite(dl[1]) && isfinite(dl[2]);
  ds = 0.0;
  if (!classic) {
    ds = -h2 * is0 * ((omv[0] * dl[0] + omv[1] * dl[1]) + omv[2] * dl[2]);
    fin = fin && isfinite(ds);
  }
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    dta[b] = -h2 * (comp(ita, b) * ((Ja[0][b] * dl[0] + Ja[1][b] * dl[1]) + Ja[2][b] * dl[2]));
    dtb[b] = -h2 * (comp(itb, b) * ((Jb[0][b] * dl[0] + Jb[1][b] * dl[1]) + Jb[2][b] * dl[2]));
    fin = fin && isfinite(dta[b]) && isfinite(dtb[b]);
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) lam_out[d] = lam[d] + dl[d];
  ok = fin;
  return true;
}

// SurfaceBending of interior vertex k (:156-168), dim 1: ds of vertices k-1, k, k+1.
__device__ __forceinline__ bool surface_bending(double sm, double s0, double spp, double la, double lb, double slap,
                                                double ism, double is0, double isp, double kinv, double lam,
                                                double h2, double beta, double (&ds)[3], double& lam_out, bool& ok) {
  const Recip ra = recip(la), rb = recip(lb);
  const double lap = divr(spp - s0, rb) - divr(s0 - sm, ra);
  const double W = lap - slap;
  const double jm = rinv(ra), jp = rinv(rb), j0 = -jm - jp;  // (-1.0 / la) - 1.0 / lb
  double M = 0.0;
  if (ism != 0.0) M = M + (h2 * ism * jm) * jm;
  if (is0 != 0.0) M = M + (h2 * is0 * j0) * j0;
  if (isp != 0.0) M = M + (h2 * isp * jp) * jp;
  M = M + kinv;
  if (!(M > 1e-250)) return false;
  const double dl = qdiv(beta * (W - kinv * lam), M);
  ds[0] = -h2 * ism * (jm * dl);
  ds[1] = -h2 * is0 * (j0 * dl);
  ds[2] = -h2 * isp * (jp * dl);
  lam_out = lam + dl;
  ok = isfinite(dl) && isfinite(ds[0]) && isfinite(ds[1]) && isfinite(ds[2]);
  return true;
}

// VolumeBendU (cc = 0) / VolumeBendV (cc = 1) of interior vertex k (:189-214), dim 1.
__device__ __forceinline__ bool volume_bend(int cc, const VertexFrame& vf, double s0, double sbar, double is0,
                                            const V3& ita, const V3& itb, double la, double lb, double la0, double lb0,
                                            double darb_c, double kinv, double lam, double h2, double beta, double& ds,
                                            double (&dta)[3], double (&dtb)[3], double& lam_out, bool& ok) {
  const double inv_len0 = 4.0 / (la0 + lb0);
  const double om = inv_len0 * (cc == 0 ? vf.pr.x : vf.pr.y);
  const double rest_om = qdiv(darb_c * (la + lb), la0 + lb0);
  const double s = s0;
  const double W = s * s * s * om - sbar * sbar * sbar * rest_om;
  const double js = 3.0 * s * s * om;
  const double fs = s * s * s * inv_len0;
  const double ja[3] = {fs * vf.Da(cc, 0), fs * vf.Da(cc, 1), fs * vf.Da(cc, 2)};
  const double jb[3] = {fs * vf.Db(cc, 0), fs * vf.Db(cc, 1), fs * vf.Db(cc, 2)};
  double M = 0.0;
  if (is0 != 0.0) M = M + (h2 * is0 * js) * js;
  M = M + (((h2 * ja[0]) * ita.x * ja[0] + (h2 * ja[1]) * ita.y * ja[1]) + (h2 * ja[2]) * ita.z * ja[2]);
  M = M + (((h2 * jb[0]) * itb.x * jb[0] + (h2 * jb[1]) * itb.y * jb[1]) + (h2 * jb[2]) * itb.z * jb[2]);
  M = M + kinv;
  if (!(M > 1e-250)) return false;
  const double dl = qdiv(beta * (W - kinv * lam), M);
  ds = -h2 * is0 * (js * dl);
  bool fin = isfinite(dl) && isfinite(ds);
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    dta[b] = -h2 * (comp(ita, b) * (ja[b] * dl));
    dtb[b] = -h2 * (comp(itb, b) * (jb[b] * dl));
    fin = fin && isfinite(dta[b]) && isfinite(dtb[b]);
  }
  lam_out = lam + dl;
  ok = fin;
  return true;
}

}  // namespace blk
}  // namespace vdev
