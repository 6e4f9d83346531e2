// The averaged-Jacobi XPBD sweep (jacobi_sweep, constraints.cpp:491-556) on the GPU.
//
// One sweep = two kernels on the snapshot X, writing Y:
//   k_ext_solve   one thread per external block (soft pins | contacts | half-planes, the tail
//                 of the reference's block list, solver.cpp:324-328): residual + generalized
//                 XPBD update (solve_block, constraints.cpp:400-487), per-endpoint corrections.
//   k_rod_sweep   the rod stencil: CTA = 128 consecutive slots (126 owned + 1 halo each side).
//                 Each thread evaluates and solves the element-pass blocks of element k and the
//                 vertex-pass blocks of vertex k at its slot (eval_constraint :101-270),
//                 exchanges the neighbour contributions through shared memory, then GATHERS
//                 every correction touching its vertex / element in the reference's block order
//                 (elastic in assembly order, then external blocks through a slot-sorted
//                 incidence list), divides by the touch count of active blocks and applies
//                 (c += sum/n, s = max(s + sum/n, 1e-4), q <- q (x) [dtheta/2, 1]).
// No atomics on the data path: the reduction order is fixed, the result is bitwise
// deterministic run to run. There is no colouring — Jacobi snapshot semantics
// exactly as the reference (test_sweep.cpp:132-142).
#include "kernels.cuh"
#include "vmath.cuh"

namespace vdev {

using namespace vm;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double F(const double* a, int f, int vpad, int i) {
  return a[static_cast<long long>(f) * vpad + i];
}

// 3x3 solve of solve_block's dim-3 branch (constraints.cpp:446-454): singular test on Eigen's
// determinant, cofactor inverse, dlambda = beta * M^-1 * rhs.
__device__ __forceinline__ bool solve3(const double (&M)[3][3], const double (&rhs)[3], double beta, double (&dl)[3]) {
  double md = fabs(M[0][0]);
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int i = 0; i < 3; ++i) md = fmax(md, fabs(M[i][j]));
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
#pragma unroll
  for (int i = 0; i < 3; ++i)
    dl[i] = ((beta * inv[i][0]) * rhs[0] + (beta * inv[i][1]) * rhs[1]) + (beta * inv[i][2]) * rhs[2];
  return true;
}

__device__ __forceinline__ V3 ldc(const double* X, int vp, int v) { return V3{F(X, CX, vp, v), F(X, CY, vp, v), F(X, CZ, vp, v)}; }

// ---- external blocks ----------------------------------------------------------------------

struct ExtGeom {  // resolve_pill, constraints.cpp:76-97
  V3 c0, c1;
  double r0, r1, rb0, rb1;
  int v0;
};
__device__ __forceinline__ ExtGeom resolve(const World& w, const Collide& c, const double* X, int pill) {
  ExtGeom g;
  const int rod = c.pill_rod[pill];
  if (rod >= 0) {
    const int v = pill + rod;
    const int vp = w.vpad;
    g.c0 = ldc(X, vp, v);
    g.c1 = ldc(X, vp, v + 1);
    g.rb0 = F(w.vstat, RBAR, vp, v);
    g.rb1 = F(w.vstat, RBAR, vp, v + 1);
    g.r0 = F(X, S, vp, v) * g.rb0;
    g.r1 = F(X, S, vp, v + 1) * g.rb1;
    g.v0 = v;
  } else {
    const int P = c.P;
    g.c0 = V3{c.pill[pill], c.pill[P + pill], c.pill[2 * P + pill]};
    g.c1 = V3{c.pill[3 * P + pill], c.pill[4 * P + pill], c.pill[5 * P + pill]};
    g.r0 = c.pill[6 * P + pill];
    g.r1 = c.pill[7 * P + pill];
    g.rb0 = g.rb1 = 0.0;
    g.v0 = -1;
  }
  return g;
}

// Residual of an external block (contact / half-plane only), for the end-of-step penetration.
__device__ double ext_residual(const World& w, const Collide& c, const double* X, int b, int npins, int nct) {
  const int vp = w.vpad;
  if (b < npins + nct) {
    const int k = b - npins;
    const ExtGeom A = resolve(w, c, X, c.ct_a[k]);
    const ExtGeom B = resolve(w, c, X, c.ct_b[k]);
    const double al = c.ct_alpha[k], be = c.ct_beta[k];
    const V3 ca = (1.0 - al) * A.c0 + al * A.c1;
    const V3 cb = (1.0 - be) * B.c0 + be * B.c1;
    const double ra = (1.0 - al) * A.r0 + al * A.r1;
    const double rb = (1.0 - be) * B.r0 + be * B.r1;
    const double dist = norm(ca - cb);
    if (dist < 1e-12) return 0.0;
    return dist - ra - rb;
  }
  const int k = b - npins - nct;
  const int v = c.hp_slot[k];
  const double* pl = c.planes + 4 * c.hp_plane[k];
  return dot(V3{pl[0], pl[1], pl[2]}, ldc(X, vp, v)) - pl[3] - F(X, S, vp, v) * F(w.vstat, RBAR, vp, v);
}

__global__ void k_ext_solve(World w, Collide c, const double* __restrict__ X, SweepParams sp, int* singular,
                            unsigned long long* err) {
  const double contact_k = sp.contact_k;
  const int elastic_blocks = sp.elastic_blocks;
  const int npins = sp.n_pins;
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  const int vp = w.vpad;
  const double h2 = sp.h2;
  int nsing = 0;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    double* out = c.ext_out + 16ll * b;
    double* lam = c.ext_lam + 3ll * b;
    bool active = false, finite = true;
    if (b < npins) {  // kPin (constraints.cpp:261-267), dim 3
      const int v = c.pin_slot[b];
      const double* pd = c.pin_data + 4 * b;
      const V3 x = ldc(X, vp, v);
      const double W[3] = {x.x - pd[0], x.y - pd[1], x.z - pd[2]};
      const double ic = F(w.vstat, IC, vp, v);
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
        M[d][d] = M[d][d] + kinv;
        rhs[d] = W[d] - kinv * lam[d];
      }
      if (!solve3(M, rhs, sp.beta, dl)) {
        ++nsing;
      } else {
        active = true;
        const double f = -h2 * ic;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          lam[d] = lam[d] + dl[d];
          out[d] = f * dl[d];
          finite = finite && isfinite(dl[d]) && isfinite(out[d]);
        }
      }
    } else if (b < npins + nct) {  // kContact (constraints.cpp:215-247), unilateral, dim 1
      const int k = b - npins;
      const ExtGeom A = resolve(w, c, X, c.ct_a[k]);
      const ExtGeom B = resolve(w, c, X, c.ct_b[k]);
      const double al = c.ct_alpha[k], be = c.ct_beta[k];
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
      if (!(W >= 0.0 && lam[0] == 0.0)) {
        const double coef[4] = {1.0 - al, al, -(1.0 - be), -be};
        const double sj[4] = {-(1.0 - al) * A.rb0, -al * A.rb1, -(1.0 - be) * B.rb0, -be * B.rb1};
        const int slot[4] = {A.v0, A.v0 + 1, B.v0, B.v0 + 1};
        const bool has[4] = {live && A.v0 >= 0, live && A.v0 >= 0, live && B.v0 >= 0, live && B.v0 >= 0};
        double M = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // centers
          if (!has[e]) continue;
          const double ic = F(w.vstat, IC, vp, slot[e]);
          if (ic == 0.0) continue;
          const double s = h2 * ic;
          const V3 j = coef[e] * nrm;
          M = M + (((s * j.x) * j.x + (s * j.y) * j.y) + (s * j.z) * j.z);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // scales
          if (!has[e]) continue;
          const double is = F(w.vstat, IS, vp, slot[e]);
          if (is == 0.0) continue;
          M = M + (h2 * is * sj[e]) * sj[e];
        }
        const double kinv = inverse_stiffness(contact_k);
        M = M + kinv;
        const double rhs = W - kinv * lam[0];
        if (M <= 1e-250) {
          ++nsing;
        } else {
          double dl = sp.beta * rhs / M;
          if (lam[0] + dl > 0.0) dl = -lam[0];
          active = true;
          lam[0] = lam[0] + dl;
          finite = isfinite(dl);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (!has[e]) continue;
            const V3 j = coef[e] * nrm;
            const double fc = -h2 * F(w.vstat, IC, vp, slot[e]);
            out[3 * e] = fc * (j.x * dl);
            out[3 * e + 1] = fc * (j.y * dl);
            out[3 * e + 2] = fc * (j.z * dl);
            out[12 + e] = -h2 * F(w.vstat, IS, vp, slot[e]) * (sj[e] * dl);
            finite = finite && isfinite(out[3 * e]) && isfinite(out[3 * e + 1]) && isfinite(out[3 * e + 2]) &&
                     isfinite(out[12 + e]);
          }
        }
      }
    } else {  // kHalfPlane (constraints.cpp:248-260), unilateral, dim 1
      const int k = b - npins - nct;
      const int v = c.hp_slot[k];
      const double* pl = c.planes + 4 * c.hp_plane[k];
      const V3 n3{pl[0], pl[1], pl[2]};
      const double rbar = F(w.vstat, RBAR, vp, v);
      const double W = dot(n3, ldc(X, vp, v)) - pl[3] - F(X, S, vp, v) * rbar;
      if (!(W >= 0.0 && lam[0] == 0.0)) {
        const double ic = F(w.vstat, IC, vp, v), is = F(w.vstat, IS, vp, v);
        double M = 0.0;
        if (ic != 0.0) {
          const double s = h2 * ic;
          M = M + (((s * n3.x) * n3.x + (s * n3.y) * n3.y) + (s * n3.z) * n3.z);
        }
        if (is != 0.0) M = M + (h2 * is * -rbar) * -rbar;
        const double kinv = inverse_stiffness(contact_k);
        M = M + kinv;
        const double rhs = W - kinv * lam[0];
        if (M <= 1e-250) {
          ++nsing;
        } else {
          double dl = sp.beta * rhs / M;
          if (lam[0] + dl > 0.0) dl = -lam[0];
          active = true;
          lam[0] = lam[0] + dl;
          const double fc = -h2 * ic;
          out[0] = fc * (n3.x * dl);
          out[1] = fc * (n3.y * dl);
          out[2] = fc * (n3.z * dl);
          out[12] = -h2 * is * (-rbar * dl);
          finite = isfinite(dl) && isfinite(out[0]) && isfinite(out[1]) && isfinite(out[2]) && isfinite(out[12]);
        }
      }
    }
    c.ext_active[b] = active ? 1 : 0;
    if (active && !finite)
      atomicMin(err, err_code(sp.substep, ERR_SWEEP, sp.iter, static_cast<unsigned long long>(elastic_blocks) + b));
  }
  for (int o = 16; o > 0; o >>= 1) nsing += __shfl_down_sync(0xffffffffu, nsing, o);
  if ((threadIdx.x & 31) == 0 && nsing) atomicAdd(singular, nsing);
}

// ---- incidence list slot -> external blocks (built once per substep) ---------------------

__device__ __forceinline__ int ext_endpoints(const Collide& c, int b, int npins, int nct, int (&slots)[4]) {
  if (b < npins) {
    slots[0] = c.pin_slot[b];
    return 1;
  }
  if (b < npins + nct) {
    const int k = b - npins;
    int n = 0;
    const int a = c.ct_a[k], bb = c.ct_b[k];
    const int ra = c.pill_rod[a], rb = c.pill_rod[bb];
    slots[0] = slots[1] = slots[2] = slots[3] = -1;
    if (ra >= 0) {
      slots[0] = a + ra;
      slots[1] = a + ra + 1;
      n = 2;
    }
    if (rb >= 0) {
      slots[2] = bb + rb;
      slots[3] = bb + rb + 1;
      n = 4;
    }
    return n;
  }
  slots[0] = c.hp_slot[b - npins - nct];
  return 1;
}

__global__ void k_ext_count(Collide c, int npins) {
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    int slots[4];
    const int ne = ext_endpoints(c, b, npins, nct, slots);
    for (int e = 0; e < ne; ++e)
      if (slots[e] >= 0) atomicAdd(&c.ext_cnt[slots[e]], 1);
    c.ext_lam[3ll * b] = 0.0;
    c.ext_lam[3ll * b + 1] = 0.0;
    c.ext_lam[3ll * b + 2] = 0.0;
  }
}
__global__ void k_ext_fill(Collide c, int npins) {
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    int slots[4];
    const int ne = ext_endpoints(c, b, npins, nct, slots);
    for (int e = 0; e < ne; ++e) {
      if (slots[e] < 0) continue;
      const int pos = c.ext_off[slots[e]] + atomicAdd(&c.ext_cur[slots[e]], 1);
      c.ext_items[pos] = (b << 2) | e;
    }
  }
}
__global__ void k_ext_sort(Collide c, int V) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int s0 = c.ext_off[v], s1 = c.ext_off[v + 1];
  for (int a = s0 + 1; a < s1; ++a) {  // insertion sort: block order, then endpoint
    const int key = c.ext_items[a];
    int b = a - 1;
    while (b >= s0 && c.ext_items[b] > key) {
      c.ext_items[b + 1] = c.ext_items[b];
      --b;
    }
    c.ext_items[b + 1] = key;
  }
}

// ---- the rod stencil sweep ------------------------------------------------------------------

// Exchange records between neighbouring slots.
struct Fwd {  // element k / vertex k contributions consumed by slot k+1
  double sz_dc1[3], vs_dc1[3], cs_ds1, ss_ds1, vs_ds1, sb_dsp;
};
struct Bwd {  // vertex k contributions consumed by slot k-1
  double sb_dsm, bt_dta[3], vbu_dta[3], vbv_dta[3];
};
enum : int { F_SZ = 1, F_VS = 2, F_CS = 4, F_SS = 8, F_SB = 16 };
enum : int { B_SB = 1, B_BT = 2, B_VBU = 4, B_VBV = 8 };

__device__ __forceinline__ int rank_of(int kinds, int bit) { return __popc(kinds & (bit - 1)); }
__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }

__global__ void __launch_bounds__(kSweepThreads) k_rod_sweep(World w, Collide c, const double* __restrict__ X,
                                                             double* __restrict__ Y, SweepParams sp, int* singular,
                                                             unsigned long long* err, int has_ext) {
  constexpr int T = kSweepThreads;
  constexpr int NS = T + 2;
  __shared__ double sc[3][NS], ss[NS], sq[4][NS], ssb[NS], sic[NS], sis[NS], sit[3][NS];
  __shared__ Fwd fwd[T];
  __shared__ Bwd bwd[T];
  __shared__ int fflag[T], bflag[T];

  const int V = w.V, vp = w.vpad;
  const int start = blockIdx.x * (T - 2);
  const int tid = threadIdx.x;
  for (int i = tid; i < NS; i += T) {
    const int v = start - 2 + i;
    if (v >= 0 && v < V) {
      sc[0][i] = F(X, CX, vp, v);
      sc[1][i] = F(X, CY, vp, v);
      sc[2][i] = F(X, CZ, vp, v);
      ss[i] = F(X, S, vp, v);
      sq[0][i] = F(X, QW, vp, v);
      sq[1][i] = F(X, QX, vp, v);
      sq[2][i] = F(X, QY, vp, v);
      sq[3][i] = F(X, QZ, vp, v);
      ssb[i] = F(w.vstat, SBAR, vp, v);
      sic[i] = F(w.vstat, IC, vp, v);
      sis[i] = F(w.vstat, IS, vp, v);
      sit[0][i] = F(w.estat, ITX, vp, v);
      sit[1][i] = F(w.estat, ITY, vp, v);
      sit[2][i] = F(w.estat, ITZ, vp, v);
    }
  }
  __syncthreads();

  const int p = start - 1 + tid;
  const int li = tid + 1;
  const bool valid = p >= 0 && p < V;
  const bool owned = valid && tid >= 1 && tid <= T - 2;
  const double h2 = sp.h2, beta = sp.beta;

  int k = 0, m = 0, r = 0, ek = 0, vk = 0;
  if (valid) {
    k = w.slot_loc[p];
    m = w.slot_m[p];
    r = w.slot_rod[p];
    ek = w.rod_ekinds[r];
    vk = w.rod_vkinds[r];
  }
  const bool has_el = valid && k < m;
  const bool has_vx = valid && k >= 1 && k <= m - 1;

  // own contributions (kept in registers until the gather)
  V3 own_c0_sz{0, 0, 0}, own_c0_vs{0, 0, 0};
  double own_ds0_cs = 0, own_ds0_ss = 0, own_ds0_vs = 0, own_ds_bt = 0, own_ds_sb = 0, own_ds_vbu = 0, own_ds_vbv = 0;
  V3 th_sum{0, 0, 0};
  int th_cnt = 0;
  int own_flags = 0;  // bits: 1 SZ, 2 VS, 4 CS, 8 SS, 16 BT(ds), 32 SB, 64 VBU, 128 VBV
  int nsing = 0;
  Fwd f;
  Bwd bk;
  int ff = 0, bf = 0;
  unsigned long long bad = kNoError;
  const int ne = __popc(ek), nv = __popc(vk);
  const int bbase = valid ? w.rod_block_base[r] : 0;
  // Multipliers are ping-ponged like the state: every CTA reads lam_in (its halo blocks
  // included) and only the owner of a slot writes lam_out, so no CTA can observe another's
  // update within the sweep. A singular block keeps its multiplier (constraints.cpp:511-514).
  auto keep_lam = [&](int f0, int nf) {
    if (!owned) return;
    for (int f = f0; f < f0 + nf; ++f) sp.lam_out[f * (long long)vp + p] = sp.lam_in[f * (long long)vp + p];
  };

  if (has_el) {
    const V3 c0{sc[0][li], sc[1][li], sc[2][li]}, c1{sc[0][li + 1], sc[1][li + 1], sc[2][li + 1]};
    const double s0 = ss[li], s1 = ss[li + 1];
    const Q4 q{sq[0][li], sq[1][li], sq[2][li], sq[3][li]};
    const double ic0 = sic[li], ic1 = sic[li + 1], is0 = sis[li], is1 = sis[li + 1];
    const V3 it{sit[0][li], sit[1][li], sit[2][li]};
    const double tbar = F(w.estat, TDOT, vp, p);
    const int lbase = bbase + k * ne;
    M3 R;
    if (ek & (EK_SZ | EK_VS)) R = qmat(q);
    // --- StretchZ (constraints.cpp:106-119), dim 3
    if (ek & EK_SZ) {
      const double l = F(w.estat, LEN, vp, p);
      const double inv_l = 1.0 / l;
      const V3 dzc = (c1 - c0) / l;
      const V3 wv = col(R, 2);
      const double W[3] = {dzc.x - tbar * wv.x, dzc.y - tbar * wv.y, dzc.z - tbar * wv.z};
      const double J0[3] = {tbar * R.m[0][1], tbar * R.m[1][1], tbar * R.m[2][1]};
      const double J1[3] = {-tbar * R.m[0][0], -tbar * R.m[1][0], -tbar * R.m[2][0]};
      double M[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      double cd = 0.0;
      if (ic0 != 0.0) cd = cd + (h2 * ic0 * inv_l) * inv_l;
      if (ic1 != 0.0) cd = cd + (h2 * ic1 * inv_l) * inv_l;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double b0 = (h2 * J0[a]) * it.x, b1 = (h2 * J1[a]) * it.y;
#pragma unroll
        for (int b = 0; b < 3; ++b) M[a][b] = (a == b ? cd : 0.0) + (b0 * J0[b] + b1 * J1[b]);
      }
      const double kinv = inverse_stiffness(F(w.estat, KSZ, vp, p));
      double rhs[3], dl[3];
      const double lam[3] = {F(sp.lam_in, L_SZ0, vp, p), F(sp.lam_in, L_SZ1, vp, p), F(sp.lam_in, L_SZ2, vp, p)};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        M[d][d] = M[d][d] + kinv;
        rhs[d] = W[d] - kinv * lam[d];
      }
      if (solve3(M, rhs, beta, dl)) {
        const double f0 = -h2 * ic0, f1 = -h2 * ic1;
        own_c0_sz = V3{f0 * (-inv_l * dl[0]), f0 * (-inv_l * dl[1]), f0 * (-inv_l * dl[2])};
        f.sz_dc1[0] = f1 * (inv_l * dl[0]);
        f.sz_dc1[1] = f1 * (inv_l * dl[1]);
        f.sz_dc1[2] = f1 * (inv_l * dl[2]);
        const double jt0 = (J0[0] * dl[0] + J0[1] * dl[1]) + J0[2] * dl[2];
        const double jt1 = (J1[0] * dl[0] + J1[1] * dl[1]) + J1[2] * dl[2];
        const V3 dth{-h2 * (it.x * jt0), -h2 * (it.y * jt1), 0.0};
        th_sum = th_sum + dth;
        ++th_cnt;
        own_flags |= 1;
        ff |= F_SZ;
        if (owned) {
          double* L = sp.lam_out;
          L[L_SZ0 * (long long)vp + p] = lam[0] + dl[0];
          L[L_SZ1 * (long long)vp + p] = lam[1] + dl[1];
          L[L_SZ2 * (long long)vp + p] = lam[2] + dl[2];
          if (!(finite3(V3{dl[0], dl[1], dl[2]}) && finite3(own_c0_sz) && isfinite(f.sz_dc1[0]) &&
                isfinite(f.sz_dc1[1]) && isfinite(f.sz_dc1[2]) && finite3(dth)))
            bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, lbase + rank_of(ek, EK_SZ)));
        }
      } else {
        ++nsing;
        keep_lam(L_SZ0, 3);
      }
    }
    // --- CrossSection (:120-129) and SurfaceStretch (:130-138), dim 1
    if (ek & EK_CS) {
      const double W = 0.5 * (s0 + s1) - 0.5 * (ssb[li] + ssb[li + 1]);
      double M = 0.0;
      if (is0 != 0.0) M = M + (h2 * is0 * 0.5) * 0.5;
      if (is1 != 0.0) M = M + (h2 * is1 * 0.5) * 0.5;
      const double kinv = inverse_stiffness(F(w.estat, KCS, vp, p));
      const double lam = F(sp.lam_in, L_CS, vp, p);
      M = M + kinv;
      if (M > 1e-250) {
        const double dl = beta * (W - kinv * lam) / M;
        own_ds0_cs = -h2 * is0 * (0.5 * dl);
        f.cs_ds1 = -h2 * is1 * (0.5 * dl);
        own_flags |= 4;
        ff |= F_CS;
        if (owned) {
          sp.lam_out[L_CS * (long long)vp + p] = lam + dl;
          if (!(isfinite(dl) && isfinite(own_ds0_cs) && isfinite(f.cs_ds1)))
            bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, lbase + rank_of(ek, EK_CS)));
        }
      } else {
        ++nsing;
        keep_lam(L_CS, 1);
      }
    }
    if (ek & EK_SS) {
      const double l = F(w.estat, LEN, vp, p);
      const double W = (s1 - s0) / l - F(w.estat, SGRAD, vp, p);
      const double j0 = -1.0 / l, j1 = 1.0 / l;
      double M = 0.0;
      if (is0 != 0.0) M = M + (h2 * is0 * j0) * j0;
      if (is1 != 0.0) M = M + (h2 * is1 * j1) * j1;
      const double kinv = inverse_stiffness(F(w.estat, KSS, vp, p));
      const double lam = F(sp.lam_in, L_SS, vp, p);
      M = M + kinv;
      if (M > 1e-250) {
        const double dl = beta * (W - kinv * lam) / M;
        own_ds0_ss = -h2 * is0 * (j0 * dl);
        f.ss_ds1 = -h2 * is1 * (j1 * dl);
        own_flags |= 8;
        ff |= F_SS;
        if (owned) {
          sp.lam_out[L_SS * (long long)vp + p] = lam + dl;
          if (!(isfinite(dl) && isfinite(own_ds0_ss) && isfinite(f.ss_ds1)))
            bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, lbase + rank_of(ek, EK_SS)));
        }
      } else {
        ++nsing;
        keep_lam(L_SS, 1);
      }
    }
    // --- VolumeStretch (:169-188), dim 3
    if (ek & EK_VS) {
      const double l0 = F(w.estat, LEN0, vp, p);
      const double smid = 0.5 * (s0 + s1);
      const double smr = 0.5 * (ssb[li] + ssb[li + 1]);
      const V3 dzc = (c1 - c0) / l0;
      const V3 wv = col(R, 2);
      const double ka = smid * smid, kb = smr * smr * tbar;
      const double W[3] = {ka * dzc.x - kb * wv.x, ka * dzc.y - kb * wv.y, ka * dzc.z - kb * wv.z};
      const double jc = smid * smid / l0;
      const double js[3] = {smid * dzc.x, smid * dzc.y, smid * dzc.z};
      const double fac = -smr * smr * tbar;
      const double J0[3] = {fac * -R.m[0][1], fac * -R.m[1][1], fac * -R.m[2][1]};
      const double J1[3] = {fac * R.m[0][0], fac * R.m[1][0], fac * R.m[2][0]};
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
      const double kinv = inverse_stiffness(F(w.estat, KVS, vp, p));
      double rhs[3], dl[3];
      const double lam[3] = {F(sp.lam_in, L_VS0, vp, p), F(sp.lam_in, L_VS1, vp, p), F(sp.lam_in, L_VS2, vp, p)};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        M[d][d] = M[d][d] + kinv;
        rhs[d] = W[d] - kinv * lam[d];
      }
      if (solve3(M, rhs, beta, dl)) {
        const double f0 = -h2 * ic0, f1 = -h2 * ic1;
        own_c0_vs = V3{f0 * (-jc * dl[0]), f0 * (-jc * dl[1]), f0 * (-jc * dl[2])};
        f.vs_dc1[0] = f1 * (jc * dl[0]);
        f.vs_dc1[1] = f1 * (jc * dl[1]);
        f.vs_dc1[2] = f1 * (jc * dl[2]);
        const double jd = (js[0] * dl[0] + js[1] * dl[1]) + js[2] * dl[2];
        own_ds0_vs = -h2 * is0 * jd;
        f.vs_ds1 = -h2 * is1 * jd;
        const double jt0 = (J0[0] * dl[0] + J0[1] * dl[1]) + J0[2] * dl[2];
        const double jt1 = (J1[0] * dl[0] + J1[1] * dl[1]) + J1[2] * dl[2];
        const V3 dth{-h2 * (it.x * jt0), -h2 * (it.y * jt1), 0.0};
        th_sum = th_sum + dth;
        ++th_cnt;
        own_flags |= 2;
        ff |= F_VS;
        if (owned) {
          double* L = sp.lam_out;
          L[L_VS0 * (long long)vp + p] = lam[0] + dl[0];
          L[L_VS1 * (long long)vp + p] = lam[1] + dl[1];
          L[L_VS2 * (long long)vp + p] = lam[2] + dl[2];
          if (!(finite3(V3{dl[0], dl[1], dl[2]}) && finite3(own_c0_vs) && isfinite(f.vs_dc1[0]) &&
                isfinite(f.vs_dc1[1]) && isfinite(f.vs_dc1[2]) && isfinite(own_ds0_vs) && isfinite(f.vs_ds1) &&
                finite3(dth)))
            bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, lbase + rank_of(ek, EK_VS)));
        }
      } else {
        ++nsing;
        keep_lam(L_VS0, 3);
      }
    }
  }

  if (has_vx) {
    const Q4 qa{sq[0][li - 1], sq[1][li - 1], sq[2][li - 1], sq[3][li - 1]};
    const Q4 qb{sq[0][li], sq[1][li], sq[2][li], sq[3][li]};
    const double sm = ss[li - 1], s0 = ss[li], spp = ss[li + 1];
    const double is0 = sis[li];
    const V3 ita{sit[0][li - 1], sit[1][li - 1], sit[2][li - 1]};
    const V3 itb{sit[0][li], sit[1][li], sit[2][li]};
    const double sbar = ssb[li];
    const double la = F(w.estat, LEN, vp, p - 1), lb = F(w.estat, LEN, vp, p);
    const int lbase = bbase + m * ne + (k - 1) * nv;
    Q4 pr{1, 0, 0, 0};
    if (vk & (VK_BT | VK_VBU | VK_VBV)) pr = relative_rotation(qa, qb);
    // 0.5*(-+p.w I + [p_v]x) (constraints.cpp:50-51)
    const double Da[3][3] = {{0.5 * -pr.w, 0.5 * -pr.z, 0.5 * pr.y},
                             {0.5 * pr.z, 0.5 * -pr.w, 0.5 * -pr.x},
                             {0.5 * -pr.y, 0.5 * pr.x, 0.5 * -pr.w}};
    const double Db[3][3] = {{0.5 * pr.w, 0.5 * -pr.z, 0.5 * pr.y},
                             {0.5 * pr.z, 0.5 * pr.w, 0.5 * -pr.x},
                             {0.5 * -pr.y, 0.5 * pr.x, 0.5 * pr.w}};
    // --- BendTwist (:139-155), dim 3
    if (vk & VK_BT) {
      const double inv_len = 4.0 / (la + lb);
      const V3 om = inv_len * qvec(pr);
      const double s = sp.classic ? sbar : s0;
      const V3 darb{F(w.estat, DARBX, vp, p - 1), F(w.estat, DARBY, vp, p - 1), F(w.estat, DARBZ, vp, p - 1)};
      const double W[3] = {s * om.x - sbar * darb.x, s * om.y - sbar * darb.y, s * om.z - sbar * darb.z};
      const double fs = s * inv_len;
      double Ja[3][3], Jb[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          Ja[a][b] = fs * Da[a][b];
          Jb[a][b] = fs * Db[a][b];
        }
      const double omv[3] = {om.x, om.y, om.z};
      const bool sc_on = !sp.classic && is0 != 0.0;
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
      const double kinv[3] = {inverse_stiffness(F(w.estat, KBT0, vp, p)), inverse_stiffness(F(w.estat, KBT1, vp, p)),
                              inverse_stiffness(F(w.estat, KBT2, vp, p))};
      const double lam[3] = {F(sp.lam_in, L_BT0, vp, p), F(sp.lam_in, L_BT1, vp, p), F(sp.lam_in, L_BT2, vp, p)};
      double rhs[3], dl[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        M[d][d] = M[d][d] + kinv[d];
        rhs[d] = W[d] - kinv[d] * lam[d];
      }
      if (solve3(M, rhs, beta, dl)) {
        bool ok = finite3(V3{dl[0], dl[1], dl[2]});
        if (!sp.classic) {
          own_ds_bt = -h2 * is0 * ((omv[0] * dl[0] + omv[1] * dl[1]) + omv[2] * dl[2]);
          own_flags |= 16;
          ok = ok && isfinite(own_ds_bt);
        }
        V3 ta, tb;
        ta.x = -h2 * (ita.x * ((Ja[0][0] * dl[0] + Ja[1][0] * dl[1]) + Ja[2][0] * dl[2]));
        ta.y = -h2 * (ita.y * ((Ja[0][1] * dl[0] + Ja[1][1] * dl[1]) + Ja[2][1] * dl[2]));
        ta.z = -h2 * (ita.z * ((Ja[0][2] * dl[0] + Ja[1][2] * dl[1]) + Ja[2][2] * dl[2]));
        tb.x = -h2 * (itb.x * ((Jb[0][0] * dl[0] + Jb[1][0] * dl[1]) + Jb[2][0] * dl[2]));
        tb.y = -h2 * (itb.y * ((Jb[0][1] * dl[0] + Jb[1][1] * dl[1]) + Jb[2][1] * dl[2]));
        tb.z = -h2 * (itb.z * ((Jb[0][2] * dl[0] + Jb[1][2] * dl[1]) + Jb[2][2] * dl[2]));
        bk.bt_dta[0] = ta.x;
        bk.bt_dta[1] = ta.y;
        bk.bt_dta[2] = ta.z;
        bf |= B_BT;
        th_sum = th_sum + tb;
        ++th_cnt;
        if (owned) {
          double* L = sp.lam_out;
          L[L_BT0 * (long long)vp + p] = lam[0] + dl[0];
          L[L_BT1 * (long long)vp + p] = lam[1] + dl[1];
          L[L_BT2 * (long long)vp + p] = lam[2] + dl[2];
          if (!(ok && finite3(ta) && finite3(tb)))
            bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, lbase + rank_of(vk, VK_BT)));
        }
      } else {
        ++nsing;
        keep_lam(L_BT0, 3);
      }
    }
    // --- SurfaceBending (:156-168), dim 1
    if (vk & VK_SB) {
      const double lap = (spp - s0) / lb - (s0 - sm) / la;
      const double W = lap - F(w.estat, SLAP, vp, p - 1);
      const double jm = 1.0 / la, j0 = -1.0 / la - 1.0 / lb, jp = 1.0 / lb;
      const double ism = sis[li - 1], isp = sis[li + 1];
      double M = 0.0;
      if (ism != 0.0) M = M + (h2 * ism * jm) * jm;
      if (is0 != 0.0) M = M + (h2 * is0 * j0) * j0;
      if (isp != 0.0) M = M + (h2 * isp * jp) * jp;
      const double kinv = inverse_stiffness(F(w.estat, KSB, vp, p));
      const double lam = F(sp.lam_in, L_SB, vp, p);
      M = M + kinv;
      if (M > 1e-250) {
        const double dl = beta * (W - kinv * lam) / M;
        bk.sb_dsm = -h2 * ism * (jm * dl);
        own_ds_sb = -h2 * is0 * (j0 * dl);
        f.sb_dsp = -h2 * isp * (jp * dl);
        bf |= B_SB;
        ff |= F_SB;
        own_flags |= 32;
        if (owned) {
          sp.lam_out[L_SB * (long long)vp + p] = lam + dl;
          if (!(isfinite(dl) && isfinite(bk.sb_dsm) && isfinite(own_ds_sb) && isfinite(f.sb_dsp)))
            bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, lbase + rank_of(vk, VK_SB)));
        }
      } else {
        ++nsing;
        keep_lam(L_SB, 1);
      }
    }
    // --- VolumeBendU / V (:189-214), dim 1
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int bit = cc == 0 ? VK_VBU : VK_VBV;
      if (!(vk & bit)) continue;
      const double la0 = F(w.estat, LEN0, vp, p - 1), lb0 = F(w.estat, LEN0, vp, p);
      const double inv_len0 = 4.0 / (la0 + lb0);
      const double om = inv_len0 * (cc == 0 ? pr.x : pr.y);
      const double darb = F(w.estat, cc == 0 ? DARBX : DARBY, vp, p - 1);
      const double rest_om = darb * (la + lb) / (la0 + lb0);
      const double s = s0;
      const double W = s * s * s * om - sbar * sbar * sbar * rest_om;
      const double js = 3.0 * s * s * om;
      const double fs = s * s * s * inv_len0;
      const double ja[3] = {fs * Da[cc][0], fs * Da[cc][1], fs * Da[cc][2]};
      const double jb[3] = {fs * Db[cc][0], fs * Db[cc][1], fs * Db[cc][2]};
      double M = 0.0;
      if (is0 != 0.0) M = M + (h2 * is0 * js) * js;
      M = M + (((h2 * ja[0]) * ita.x * ja[0] + (h2 * ja[1]) * ita.y * ja[1]) + (h2 * ja[2]) * ita.z * ja[2]);
      M = M + (((h2 * jb[0]) * itb.x * jb[0] + (h2 * jb[1]) * itb.y * jb[1]) + (h2 * jb[2]) * itb.z * jb[2]);
      const double kinv = inverse_stiffness(F(w.estat, KVB, vp, p));
      const int lf = cc == 0 ? L_VBU : L_VBV;
      const double lam = F(sp.lam_in, lf, vp, p);
      M = M + kinv;
      if (M > 1e-250) {
        const double dl = beta * (W - kinv * lam) / M;
        const double ds = -h2 * is0 * (js * dl);
        const V3 ta{-h2 * (ita.x * (ja[0] * dl)), -h2 * (ita.y * (ja[1] * dl)), -h2 * (ita.z * (ja[2] * dl))};
        const V3 tb{-h2 * (itb.x * (jb[0] * dl)), -h2 * (itb.y * (jb[1] * dl)), -h2 * (itb.z * (jb[2] * dl))};
        if (cc == 0) {
          own_ds_vbu = ds;
          own_flags |= 64;
          bk.vbu_dta[0] = ta.x;
          bk.vbu_dta[1] = ta.y;
          bk.vbu_dta[2] = ta.z;
          bf |= B_VBU;
        } else {
          own_ds_vbv = ds;
          own_flags |= 128;
          bk.vbv_dta[0] = ta.x;
          bk.vbv_dta[1] = ta.y;
          bk.vbv_dta[2] = ta.z;
          bf |= B_VBV;
        }
        th_sum = th_sum + tb;
        ++th_cnt;
        if (owned) {
          sp.lam_out[lf * (long long)vp + p] = lam + dl;
          if (!(isfinite(dl) && isfinite(ds) && finite3(ta) && finite3(tb)))
            bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, lbase + rank_of(vk, bit)));
        }
      } else {
        ++nsing;
        keep_lam(lf, 1);
      }
    }
  }

  fwd[tid] = f;
  bwd[tid] = bk;
  fflag[tid] = ff;
  bflag[tid] = bf;
  __syncthreads();

  if (owned) {
    if (nsing) atomicAdd(singular, nsing);
    if (bad != kNoError) atomicMin(err, bad);
    // ---- gather in block order (constraints.cpp:509-534) and apply (:537-554)
    const int pf = fflag[tid - 1];
    const int nb = bflag[tid + 1];
    const Fwd& F1 = fwd[tid - 1];
    const Bwd& B1 = bwd[tid + 1];
    const bool prev_el = k >= 1;         // element k-1 exists
    const bool prev_vx = k - 1 >= 1;     // vertex k-1 interior
    const bool next_vx = k + 1 <= m - 1; // vertex k+1 interior
    V3 csum{0, 0, 0};
    int ccnt = 0;
    double ssum = 0.0;
    int scnt = 0;
    if (prev_el) {
      if (pf & F_SZ) {
        csum = csum + V3{F1.sz_dc1[0], F1.sz_dc1[1], F1.sz_dc1[2]};
        ++ccnt;
      }
      if (pf & F_CS) {
        ssum += F1.cs_ds1;
        ++scnt;
      }
      if (pf & F_SS) {
        ssum += F1.ss_ds1;
        ++scnt;
      }
      if (pf & F_VS) {
        csum = csum + V3{F1.vs_dc1[0], F1.vs_dc1[1], F1.vs_dc1[2]};
        ++ccnt;
        ssum += F1.vs_ds1;
        ++scnt;
      }
    }
    if (has_el) {
      if (own_flags & 1) {
        csum = csum + own_c0_sz;
        ++ccnt;
      }
      if (own_flags & 4) {
        ssum += own_ds0_cs;
        ++scnt;
      }
      if (own_flags & 8) {
        ssum += own_ds0_ss;
        ++scnt;
      }
      if (own_flags & 2) {
        csum = csum + own_c0_vs;
        ++ccnt;
        ssum += own_ds0_vs;
        ++scnt;
      }
    }
    if (prev_vx && (pf & F_SB)) {
      ssum += F1.sb_dsp;
      ++scnt;
    }
    if (has_vx) {
      if (own_flags & 16) {
        ssum += own_ds_bt;
        ++scnt;
      }
      if (own_flags & 32) {
        ssum += own_ds_sb;
        ++scnt;
      }
      if (own_flags & 64) {
        ssum += own_ds_vbu;
        ++scnt;
      }
      if (own_flags & 128) {
        ssum += own_ds_vbv;
        ++scnt;
      }
    }
    if (next_vx) {
      if (nb & B_SB) {
        ssum += B1.sb_dsm;
        ++scnt;
      }
      if (has_el) {
        if (nb & B_BT) {
          th_sum = th_sum + V3{B1.bt_dta[0], B1.bt_dta[1], B1.bt_dta[2]};
          ++th_cnt;
        }
        if (nb & B_VBU) {
          th_sum = th_sum + V3{B1.vbu_dta[0], B1.vbu_dta[1], B1.vbu_dta[2]};
          ++th_cnt;
        }
        if (nb & B_VBV) {
          th_sum = th_sum + V3{B1.vbv_dta[0], B1.vbv_dta[1], B1.vbv_dta[2]};
          ++th_cnt;
        }
      }
    }
    if (has_ext) {  // external blocks touching this vertex, in block order
      const int e0 = c.ext_off[p], e1 = c.ext_off[p + 1];
      for (int q = e0; q < e1; ++q) {
        const int item = c.ext_items[q];
        const int b = item >> 2, ep = item & 3;
        if (!c.ext_active[b]) continue;
        const double* o = c.ext_out + 16ll * b;
        csum = csum + V3{o[3 * ep], o[3 * ep + 1], o[3 * ep + 2]};
        ++ccnt;
        if (b >= sp.n_pins) {
          ssum += o[12 + ep];
          ++scnt;
        }
      }
    }
    V3 cn{sc[0][li], sc[1][li], sc[2][li]};
    if (ccnt > 0) cn = cn + csum / static_cast<double>(ccnt);
    double sn = ss[li];
    if (scnt > 0) sn = fmax(sn + ssum / static_cast<double>(scnt), kMinScale);
    Q4 qn{sq[0][li], sq[1][li], sq[2][li], sq[3][li]};
    if (has_el && th_cnt > 0) qn = apply_increment(qn, th_sum / static_cast<double>(th_cnt));
    Y[CX * (long long)vp + p] = cn.x;
    Y[CY * (long long)vp + p] = cn.y;
    Y[CZ * (long long)vp + p] = cn.z;
    Y[S * (long long)vp + p] = sn;
    Y[QW * (long long)vp + p] = qn.w;
    Y[QX * (long long)vp + p] = qn.x;
    Y[QY * (long long)vp + p] = qn.y;
    Y[QZ * (long long)vp + p] = qn.z;
  }
}

// ---- end-of-substep report (elastic_residual_norms, constraints.cpp:558-596, and
//      end_of_step_penetration, solver.cpp:291-299) ----------------------------------------

constexpr int kRepThreads = 256;

__global__ void k_report_partial(World w, const double* __restrict__ X, int classic, double* partials) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  if (v < w.V) {
    const int vp = w.vpad;
    const int k = w.slot_loc[v], m = w.slot_m[v], r = w.slot_rod[v];
    const int ek = w.rod_ekinds[r], vk = w.rod_vkinds[r];
    if (k < m) {
      const V3 c0 = ldc(X, vp, v), c1 = ldc(X, vp, v + 1);
      const double s0 = F(X, S, vp, v), s1 = F(X, S, vp, v + 1);
      const double sb0 = F(w.vstat, SBAR, vp, v), sb1 = F(w.vstat, SBAR, vp, v + 1);
      const double l = F(w.estat, LEN, vp, v), l0 = F(w.estat, LEN0, vp, v), tbar = F(w.estat, TDOT, vp, v);
      const M3 R = qmat(Q4{F(X, QW, vp, v), F(X, QX, vp, v), F(X, QY, vp, v), F(X, QZ, vp, v)});
      const V3 wv = col(R, 2);
      if (ek & EK_SZ) {
        const V3 W = (c1 - c0) / l - tbar * wv;
        acc[0] += l * sqnorm(W);
        acc[8] += l;
      }
      if (ek & EK_CS) {
        const double W = 0.5 * (s0 + s1) - 0.5 * (sb0 + sb1);
        acc[1] += l * (W * W);
        acc[9] += l;
      }
      if (ek & EK_SS) {
        const double W = (s1 - s0) / l - F(w.estat, SGRAD, vp, v);
        acc[2] += l * (W * W);
        acc[10] += l;
      }
      if (ek & EK_VS) {
        const double smid = 0.5 * (s0 + s1), smr = 0.5 * (sb0 + sb1);
        const V3 W = (smid * smid) * ((c1 - c0) / l0) - (smr * smr * tbar) * wv;
        acc[5] += l0 * sqnorm(W);
        acc[13] += l0;
      }
    }
    if (k >= 1 && k <= m - 1) {
      const double la = F(w.estat, LEN, vp, v - 1), lb = F(w.estat, LEN, vp, v);
      const double la0 = F(w.estat, LEN0, vp, v - 1), lb0 = F(w.estat, LEN0, vp, v);
      const Q4 qa{F(X, QW, vp, v - 1), F(X, QX, vp, v - 1), F(X, QY, vp, v - 1), F(X, QZ, vp, v - 1)};
      const Q4 qb{F(X, QW, vp, v), F(X, QX, vp, v), F(X, QY, vp, v), F(X, QZ, vp, v)};
      const Q4 pr = relative_rotation(qa, qb);
      const double s0 = F(X, S, vp, v), sbar = F(w.vstat, SBAR, vp, v);
      const V3 darb{F(w.estat, DARBX, vp, v - 1), F(w.estat, DARBY, vp, v - 1), F(w.estat, DARBZ, vp, v - 1)};
      if (vk & VK_BT) {
        const V3 om = (4.0 / (la + lb)) * qvec(pr);
        const double s = classic ? sbar : s0;
        const V3 W = s * om - sbar * darb;
        const double lw = 0.5 * (la + lb);
        acc[3] += lw * sqnorm(W);
        acc[11] += lw;
      }
      if (vk & VK_SB) {
        const double sm = F(X, S, vp, v - 1), spp = F(X, S, vp, v + 1);
        const double W = ((spp - s0) / lb - (s0 - sm) / la) - F(w.estat, SLAP, vp, v - 1);
        const double lw = 0.5 * (la + lb);
        acc[4] += lw * (W * W);
        acc[12] += lw;
      }
      const double inv_len0 = 4.0 / (la0 + lb0);
      const double lw0 = 0.5 * (la0 + lb0);
      for (int cc = 0; cc < 2; ++cc) {
        if (!(vk & (cc == 0 ? VK_VBU : VK_VBV))) continue;
        const double om = inv_len0 * (cc == 0 ? pr.x : pr.y);
        const double rest_om = (cc == 0 ? darb.x : darb.y) * (la + lb) / (la0 + lb0);
        const double W = s0 * s0 * s0 * om - sbar * sbar * sbar * rest_om;
        acc[6 + cc] += lw0 * (W * W);
        acc[14 + cc] += lw0;
      }
    }
  }
  // fixed-order block tree reduction
  __shared__ double red[kRepThreads];
  for (int q = 0; q < 16; ++q) {
    red[threadIdx.x] = acc[q];
    __syncthreads();
    for (int s = kRepThreads / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) partials[16ll * blockIdx.x + q] = red[0];
    __syncthreads();
  }
}

__global__ void k_report_final(const double* partials, int parts, double* out8) {
  const int q = threadIdx.x;
  if (q >= 8) return;
  double num = 0.0, den = 0.0;
  for (int b = 0; b < parts; ++b) {
    num += partials[16ll * b + q];
    den += partials[16ll * b + 8 + q];
  }
  out8[q] = den > 0 ? sqrt(num / den) : 0.0;
}

__global__ void k_penetration(World w, Collide c, const double* __restrict__ X, StepAccum* acc) {
  const int npins = c.n_pins;
  const int nct = c.scalars[SC_NCT];
  const int n = nct + c.scalars[SC_NHP];
  double deepest = 0.0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const double pen = -ext_residual(w, c, X, npins + q, npins, nct);
    if (pen > deepest) deepest = pen;
  }
  for (int o = 16; o > 0; o >>= 1) deepest = fmax(deepest, __shfl_down_sync(0xffffffffu, deepest, o));
  if ((threadIdx.x & 31) == 0 && deepest > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(&acc->max_penetration),
              static_cast<unsigned long long>(__double_as_longlong(deepest)));
}

int grid_for(long long n) {
  const long long b = (n + kThreads - 1) / kThreads;
  return static_cast<int>(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

int report_parts(int V) { return (V + kRepThreads - 1) / kRepThreads; }

void launch_ext_setup(const World& w, Collide& c, cudaStream_t st) {
  cudaMemsetAsync(c.ext_cnt, 0, sizeof(int) * (w.V + 1), st);
  cudaMemsetAsync(c.ext_cur, 0, sizeof(int) * w.V, st);
  const int g = grid_for(c.ext_cap);
  k_ext_count<<<g, kThreads, 0, st>>>(c, c.n_pins);
  scan_exclusive(c.ext_cnt, c.ext_off, w.V, nullptr, c.scan_tmp, c.scan_parts, st);
  k_ext_fill<<<g, kThreads, 0, st>>>(c, c.n_pins);
  k_ext_sort<<<(w.V + kThreads - 1) / kThreads, kThreads, 0, st>>>(c, w.V);
}

void launch_ext_solve(const World& w, Collide& c, const double* X, const SweepParams& sp, int* singular_counter,
                      unsigned long long* err, cudaStream_t st) {
  if (c.ext_cap > 0) k_ext_solve<<<grid_for(c.ext_cap), kThreads, 0, st>>>(w, c, X, sp, singular_counter, err);
}

void launch_rod_sweep(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp,
                      int* singular_counter, unsigned long long* err, cudaStream_t st) {
  const int has_ext = c.ext_cap > 0 ? 1 : 0;
  const int blocks = (w.V + (kSweepThreads - 2) - 1) / (kSweepThreads - 2);
  k_rod_sweep<<<blocks, kSweepThreads, 0, st>>>(w, c, X, Y, sp, singular_counter, err, has_ext);
}

void launch_iteration(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp,
                      int* singular_counter, unsigned long long* err, cudaStream_t st) {
  launch_ext_solve(w, c, X, sp, singular_counter, err, st);
  launch_rod_sweep(w, c, X, Y, sp, singular_counter, err, st);
}

void launch_residuals(const World& w, const double* X, int classic, double* partials, int parts, double* out8,
                      cudaStream_t st) {
  k_report_partial<<<parts, kRepThreads, 0, st>>>(w, X, classic, partials);
  k_report_final<<<1, 32, 0, st>>>(partials, parts, out8);
}

void launch_penetration(const World& w, Collide& c, const double* X, StepAccum* acc, cudaStream_t st) {
  k_penetration<<<grid_for(c.contact_cap + c.hp_cap), kThreads, 0, st>>>(w, c, X, acc);
}

}  // namespace vdev
