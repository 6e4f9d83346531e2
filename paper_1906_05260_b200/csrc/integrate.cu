// Integration kernels: animate (Solver::animate, solver.cpp:138-154), prediction
// (predict_rod + warm_start_lbs + refresh_orientation_inertia, solver.cpp:21-100,156-183,
// layout.cpp:76-93) and finalization (post_step_scales + finalize_velocities,
// solver.cpp:253-289). Compiled with --fmad=false: every expression keeps the reference's
// operation order, so these kernels reproduce the oracle bit for bit.
#include "kernels.cuh"
#include "pillbounds.cuh"
#include "vmath.cuh"

namespace vdev {

using namespace vm;

namespace {

__device__ __forceinline__ double F(const double* a, int f, int vpad, int i) { return a[static_cast<long long>(f) * vpad + i]; }
__device__ __forceinline__ double& Fr(double* a, int f, int vpad, int i) { return a[static_cast<long long>(f) * vpad + i]; }

__global__ void k_pin_motions(World w, const double* __restrict__ anim, AnimLayout al, const int* __restrict__ pm_slot) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= al.n_pm) return;
  const int v = pm_slot[i];
  const double* p = anim + al.off_pm + 3 * i;
  Fr(w.X, CX, w.vpad, v) = p[0];
  Fr(w.X, CY, w.vpad, v) = p[1];
  Fr(w.X, CZ, w.vpad, v) = p[2];
}

// One CTA per rod carrying activations: apply_activation (rod.cpp:164-176) for every activation
// whose amount changed, then refresh_length_derived (rod.cpp:42-56) and refresh_stiffness
// (constraints.cpp:331-372) for the rod.
struct ActArgs {
  const int* rod_off;
  const int* list;
  double* applied;
  const int* rods;
  const double* stat;
  int n_rods;
};
__device__ __forceinline__ void activation_block(const World& w, const double* __restrict__ anim, const AnimLayout& al,
                                                 const ActArgs& aa, int blk) {
  const int* __restrict__ rod_off = aa.rod_off;
  const int* __restrict__ act_list = aa.list;
  double* applied = aa.applied;
  const double* __restrict__ act_static = aa.stat;
  const int r = aa.rods[blk];
  const int v0 = w.rod_vbase[r];
  const int n = w.rod_n[r];
  const int m = n - 1;
  __shared__ int changed;
  if (threadIdx.x == 0) changed = 0;
  __syncthreads();
  for (int k = rod_off[blk]; k < rod_off[blk + 1]; ++k) {  // activation order
    const int a_id = act_list[k];
    const double a = anim[al.off_act + a_id];
    const double prev = applied[a_id];
    __syncthreads();
    if (a == prev) continue;
    const double factor = act_static[3 * a_id];
    const int first = static_cast<int>(act_static[3 * a_id + 1]);
    int last = static_cast<int>(act_static[3 * a_id + 2]);
    if (last < 0) last = m - 1;
    const double scale = 1.0 - a * factor;
    for (int e = first + threadIdx.x; e <= last; e += blockDim.x)
      Fr(w.estat, LEN, w.vpad, v0 + e) = F(w.estat, LEN0, w.vpad, v0 + e) * scale;
    if (threadIdx.x == 0) {
      applied[a_id] = a;
      changed = 1;
    }
    __syncthreads();
  }
  __syncthreads();
  if (!changed) return;
  const int vp = w.vpad;
  const double* mat = w.mat + 8 * w.rod_material[r];
  const double kxy = mat[0] + mat[1];
  for (int e = threadIdx.x; e < m; e += blockDim.x) {
    const int s = v0 + e;
    const double len = F(w.estat, LEN, vp, s);
    Fr(w.estat, SGRAD, vp, s) = (F(w.vstat, SBAR, vp, s + 1) - F(w.vstat, SBAR, vp, s)) / len;
    // element-pass stiffness (StretchZ, CrossSection, SurfaceStretch), stored inverted (K rows)
    Fr(w.estat, KSZ, vp, s) = inverse_stiffness(F(w.estat, A2E, vp, s) * mat[2] * len);
    Fr(w.estat, KCS, vp, s) = inverse_stiffness(F(w.estat, A2E, vp, s) * kxy * len);
    Fr(w.estat, KSS, vp, s) = inverse_stiffness(F(w.estat, A4EP, vp, s) * kxy * len);
    if (e >= 1) {  // interior vertex j = e: Darboux, laplacian, BendTwist / SurfaceBending stiffness
      const int j = s;
      const double la = F(w.estat, LEN, vp, j - 1);
      const double lb = len;
      const Q4 qa{F(w.estat, RQW, vp, j - 1), F(w.estat, RQX, vp, j - 1), F(w.estat, RQY, vp, j - 1),
                  F(w.estat, RQZ, vp, j - 1)};
      const Q4 qb{F(w.estat, RQW, vp, j), F(w.estat, RQX, vp, j), F(w.estat, RQY, vp, j), F(w.estat, RQZ, vp, j)};
      const V3 d = (4.0 / (la + lb)) * qvec(relative_rotation(qa, qb));
      Fr(w.estat, DARBX, vp, j - 1) = d.x;
      Fr(w.estat, DARBY, vp, j - 1) = d.y;
      Fr(w.estat, DARBZ, vp, j - 1) = d.z;
      const double sm = F(w.vstat, SBAR, vp, j - 1), s0 = F(w.vstat, SBAR, vp, j), sp = F(w.vstat, SBAR, vp, j + 1);
      Fr(w.estat, SLAP, vp, j - 1) = (sp - s0) / lb - (s0 - sm) / la;
      const double a4 = F(w.estat, A4VP, vp, j);
      const double lw = 0.5 * (la + lb);
      Fr(w.estat, KBT0, vp, j) = inverse_stiffness(a4 * mat[2] * lw);
      Fr(w.estat, KBT1, vp, j) = inverse_stiffness(a4 * mat[2] * lw);
      Fr(w.estat, KBT2, vp, j) = inverse_stiffness(a4 * kxy * lw);
      Fr(w.estat, KSB, vp, j) = inverse_stiffness(a4 * (mat[3] + mat[4]) * lw);
    }
  }
}
__global__ void k_activation(World w, const double* __restrict__ anim, AnimLayout al, ActArgs aa) {
  pdl_wait();
  pdl_trigger();
  activation_block(w, anim, al, aa, blockIdx.x);
}

// The predicted scale of vertex v (predict_rod, solver.cpp:41-50): s + h * sdot plus the radial
// load term, floored; unchanged for pinned vertices. gamma_bad: the load term is not finite.
__device__ __forceinline__ double predicted_scale(const World& w, double h, int v, bool& gamma_bad) {
  const int vp = w.vpad;
  double s = F(w.X, S, vp, v);
  gamma_bad = false;
  if (w.pinned[v]) return s;
  const int r = w.slot_rod[v];
  const int k = w.slot_loc[v];
  const int m = w.slot_m[v];
  const uint8_t lf = w.has_loads ? w.load_flags[r] : 0;
  double ds = h * F(w.vel, VS, vp, v);
  if ((lf & 4) && !w.classic) {
    const double rho = w.mat[8 * w.rod_material[r] + 7];
    double gamma = 0.0;
    int count = 0;
    if (k > 0) {
      gamma += F(w.loads, 6, vp, v - 1);
      ++count;
    }
    if (k < m) {
      gamma += F(w.loads, 6, vp, v);
      ++count;
    }
    gamma /= count;
    gamma_bad = !isfinite(gamma);
    const double rr = F(w.vstat, RBAR, vp, v);
    const double h2 = h * h;
    ds += 2.0 * h2 * gamma / (kPi * rr * rr * rr * rr * rho);
  }
  return fmax(s + ds, kMinScale);
}

// predict_rod vertex loop (solver.cpp:29-58) + warm_start_lbs (:75-100) + the non-finite
// prediction check (:179-181). Also takes the pre-predict snapshot (solver.cpp:311-316).
// Returns the predicted scale.
__device__ __forceinline__ double predict_vertex(const World& w, const double* __restrict__ anim, const AnimLayout& al,
                                                 const V3& g, double h, int substep, unsigned long long* err, int v,
                                                 V3* c_out = nullptr) {
  const int vp = w.vpad;
  const int r = w.slot_rod[v];
  const int k = w.slot_loc[v];
  V3 c{F(w.X, CX, vp, v), F(w.X, CY, vp, v), F(w.X, CZ, vp, v)};
  Fr(w.prev, CX, vp, v) = c.x;
  Fr(w.prev, CY, vp, v) = c.y;
  Fr(w.prev, CZ, vp, v) = c.z;
  Fr(w.prev, S, vp, v) = F(w.X, S, vp, v);
  const double h2 = h * h;
  const uint8_t lf = w.has_loads ? w.load_flags[r] : 0;
  bool gamma_bad;
  const double s = predicted_scale(w, h, v, gamma_bad);
  if (!w.pinned[v]) {
    const double rho = w.mat[8 * w.rod_material[r] + 7];
    V3 accel = g;
    if (lf & 1) {
      const V3 fd{F(w.loads, 0, vp, v), F(w.loads, 1, vp, v), F(w.loads, 2, vp, v)};
      if (!finite3(fd)) atomicMin(err, err_code(substep, ERR_PREDICT, r, 2ull * k));
      accel = accel + fd / rho;
    }
    const V3 vel{F(w.vel, VX, vp, v), F(w.vel, VY, vp, v), F(w.vel, VZ, vp, v)};
    c = c + (h * vel + h2 * accel);
    if (gamma_bad) atomicMin(err, err_code(substep, ERR_PREDICT, r, 2ull * k + 1));
    if (w.has_bones) {
      const int b0 = w.rod_bone_off[r], b1 = w.rod_bone_off[r + 1];
      if (b1 > b0) {  // warm_start_lbs
        V3 blended{0, 0, 0};
        const double* bw = w.bone_w + w.slot_bw_off[v];
        for (int b = b0; b < b1; ++b) {
          const double* bt = anim + al.off_bone + 14 * w.rod_bones[b];
          const Q4 rp{bt[0], bt[1], bt[2], bt[3]}, rn{bt[4], bt[5], bt[6], bt[7]};
          const V3 pp{bt[8], bt[9], bt[10]}, pn{bt[11], bt[12], bt[13]};
          const Q4 delta = qmul(rn, qconj(rp));
          blended = blended + bw[b - b0] * (qrot(delta, c - pp) + pn);
        }
        c = blended;
      }
    }
  }
  if (w.classic) Fr(w.vel, VS, vp, v) = 0.0;
  if (!finite3(c)) atomicMin(err, err_code(substep, ERR_PREDICT, r, 0xfffffffeull));
  Fr(w.X, CX, vp, v) = c.x;
  Fr(w.X, CY, vp, v) = c.y;
  Fr(w.X, CZ, vp, v) = c.z;
  Fr(w.X, S, vp, v) = s;
  double2* xr = reinterpret_cast<double2*>(w.xrec + 8ll * v);
  xr[0] = make_double2(c.x, c.y);
  xr[1] = make_double2(c.z, s);
  if (c_out) *c_out = c;
  return s;
}

// predict_rod element loop (solver.cpp:60-72) + refresh_orientation_inertia (layout.cpp:76-93)
// from the predicted scales s0, s1 of the element's vertices.
__device__ __forceinline__ void predict_element(const World& w, double h, int substep, unsigned long long* err, int v,
                                                double s0, double s1) {
  const int m = w.slot_m[v];
  const int vp = w.vpad;
  const int r = w.slot_rod[v];
  const int k = w.slot_loc[v];
  Q4 q{F(w.X, QW, vp, v), F(w.X, QX, vp, v), F(w.X, QY, vp, v), F(w.X, QZ, vp, v)};
  Fr(w.prev, QW, vp, v) = q.w;
  Fr(w.prev, QX, vp, v) = q.x;
  Fr(w.prev, QY, vp, v) = q.y;
  Fr(w.prev, QZ, vp, v) = q.z;
  const double h2 = h * h;
  const double rho = w.mat[8 * w.rod_material[r] + 7];
  V3 dth = h * V3{F(w.vel, WX, vp, v), F(w.vel, WY, vp, v), F(w.vel, WZ, vp, v)};
  if (w.has_loads && (w.load_flags[r] & 2)) {
    const V3 tq{F(w.loads, 3, vp, v), F(w.loads, 4, vp, v), F(w.loads, 5, vp, v)};
    if (!finite3(tq)) atomicMin(err, err_code(substep, ERR_PREDICT, r, 2ull * (m + 1) + k));
    const double smid = 0.5 * (s0 + s1);
    const double rmid = 0.5 * (F(w.vstat, RBAR, vp, v) + F(w.vstat, RBAR, vp, v + 1));
    const double r4 = rmid * rmid * rmid * rmid;
    const V3 bt = qrot(qconj(q), tq);
    const V3 ii{4.0 / (kPi * r4), 4.0 / (kPi * r4), 2.0 / (kPi * r4)};
    dth = dth + (h2 / (smid * smid * rho)) * cwmul(ii, bt);
  }
  q = apply_increment(q, dth);
  Fr(w.X, QW, vp, v) = q.w;
  Fr(w.X, QX, vp, v) = q.x;
  Fr(w.X, QY, vp, v) = q.y;
  Fr(w.X, QZ, vp, v) = q.z;
  // refresh_orientation_inertia with the predicted midpoint scale
  const double rbar = 0.5 * (F(w.vstat, RBAR, vp, v) + F(w.vstat, RBAR, vp, v + 1));
  const double smid = 0.5 * (s0 + s1);
  const double r4 = kPi * rbar * rbar * rbar * rbar;
  const double base = rho * smid * smid * r4 * F(w.estat, LEN0, vp, v);
  Fr(w.estat, TWB, vp, v) = base;
  Fr(w.estat, ITX, vp, v) = 1.0 / (0.25 * base);
  Fr(w.estat, ITY, vp, v) = 1.0 / (0.25 * base);
  Fr(w.estat, ITZ, vp, v) = 1.0 / (0.5 * base);
}

__global__ void k_predict_vertices(World w, const double* __restrict__ anim, AnimLayout al, V3 g, double h,
                                   int substep, unsigned long long* err) {
  pdl_wait();
  pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < w.V) predict_vertex(w, anim, al, g, h, substep, err, v);
}
__global__ void k_predict_elements(World w, double h, int substep, unsigned long long* err) {
  pdl_wait();
  pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= w.V || w.slot_loc[v] >= w.slot_m[v]) return;
  predict_element(w, h, substep, err, v, F(w.X, S, w.vpad, v), F(w.X, S, w.vpad, v + 1));
}

// Worlds whose rods all have <= 32 vertices: the whole prediction in one launch, one warp per
// rod (lane k = slot k): vertex k, then element k with the predicted scale of vertex k + 1 from
// the next lane. A rod never spans two warps, so no lane reads a scale another warp rewrites.
// With activations, their rods' CTAs come first in the same launch (activation_block: disjoint
// fields — LEN and the length-derived statics — from the ones the prediction reads and writes).
constexpr int kPredictRodsPerCta = 4;
// pills != 0 (single-scene worlds without kinematic pills; the broad phase's resets already ran):
// also the rod pills of the predicted state with their bounding spheres and the max radius
// (k_build_pills' work: the same values from the same operands, one launch less).
__global__ void __launch_bounds__(32 * kPredictRodsPerCta) k_predict_rods(World w, const double* __restrict__ anim,
                                                                         AnimLayout al, V3 g, double h, int substep,
                                                                         unsigned long long* err, ActArgs aa,
                                                                         Collide cl, int pills) {
  pdl_wait();
  pdl_trigger();
  if (static_cast<int>(blockIdx.x) < aa.n_rods) {
    activation_block(w, anim, al, aa, blockIdx.x);
    return;
  }
  const int r = (blockIdx.x - aa.n_rods) * kPredictRodsPerCta + (threadIdx.x >> 5);
  if (r >= w.R) return;  // whole warps
  const int k = threadIdx.x & 31, n = w.rod_n[r], v = w.rod_vbase[r] + k;
  double s0 = 0.0;
  V3 c0{0, 0, 0};
  if (k < n) s0 = predict_vertex(w, anim, al, g, h, substep, err, v, &c0);
  const double s1 = __shfl_down_sync(0xffffffffu, s0, 1);
  if (pills) {  // rod_pills (collision.cpp:275-296) + bounding spheres
    const V3 c1{__shfl_down_sync(0xffffffffu, c0.x, 1), __shfl_down_sync(0xffffffffu, c0.y, 1),
                __shfl_down_sync(0xffffffffu, c0.z, 1)};
    unsigned long long bits = 0;
    if (k < n - 1) {
      const int vp = w.vpad;
      const PillV p{c0, c1, s0 * w.vstat[RBAR * vp + v], s1 * w.vstat[RBAR * vp + v + 1]};
      const int i = v - r;
      double2* o = reinterpret_cast<double2*>(cl.pill + 8ll * i);
      o[0] = make_double2(p.c0.x, p.c0.y);
      o[1] = make_double2(p.c0.z, p.c1.x);
      o[2] = make_double2(p.c1.y, p.c1.z);
      o[3] = make_double2(p.r0, p.r1);
      bits = pill_bounds(cl, p, i, substep, err);
    }
    for (int o = 16; o > 0; o >>= 1) {  // warp max, one atomic per warp
      const unsigned long long x = __shfl_down_sync(0xffffffffu, bits, o);
      bits = x > bits ? x : bits;
    }
    if (k == 0 && bits) atomicMax(cl.maxr_bits, bits);
  }
  if (k < n - 1) predict_element(w, h, substep, err, v, s0, s1);
}

// post_step_scales (classic mode, solver.cpp:253-271) + finalize_velocities (:273-289).
// Reads the final sweep buffer `src`, writes the canonical state X and the velocities.
__global__ void k_finalize(World w, const double* __restrict__ src, double h, double keep) {
  pdl_wait();
  pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= w.V) return;
  const int vp = w.vpad;
  const int k = w.slot_loc[v];
  const int m = w.slot_m[v];
  const V3 c{F(src, CX, vp, v), F(src, CY, vp, v), F(src, CZ, vp, v)};
  double s = F(src, S, vp, v);
  if (w.classic && !w.pinned[v]) {
    double ratio = 0.0;
    int count = 0;
    for (int d = -1; d <= 0; ++d) {
      const int e = k + d;
      if (e < 0 || e >= m) continue;
      const int se = v + d;
      const V3 a{F(src, CX, vp, se), F(src, CY, vp, se), F(src, CZ, vp, se)};
      const V3 b{F(src, CX, vp, se + 1), F(src, CY, vp, se + 1), F(src, CZ, vp, se + 1)};
      const double cur = norm(b - a);
      ratio += sqrt(F(w.estat, LEN, vp, se) / fmax(cur, 1e-12));
      ++count;
    }
    s = fmax(F(w.vstat, SBAR, vp, v) * ratio / count, kMinScale);
  }
  const V3 pc{F(w.prev, CX, vp, v), F(w.prev, CY, vp, v), F(w.prev, CZ, vp, v)};
  const V3 cv = (keep * (c - pc)) / h;
  Fr(w.X, CX, vp, v) = c.x;
  Fr(w.X, CY, vp, v) = c.y;
  Fr(w.X, CZ, vp, v) = c.z;
  Fr(w.X, S, vp, v) = s;
  Fr(w.vel, VX, vp, v) = cv.x;
  Fr(w.vel, VY, vp, v) = cv.y;
  Fr(w.vel, VZ, vp, v) = cv.z;
  Fr(w.vel, VS, vp, v) = keep * (s - F(w.prev, S, vp, v)) / h;
  if (k < m) {
    const Q4 q{F(src, QW, vp, v), F(src, QX, vp, v), F(src, QY, vp, v), F(src, QZ, vp, v)};
    const Q4 pq{F(w.prev, QW, vp, v), F(w.prev, QX, vp, v), F(w.prev, QY, vp, v), F(w.prev, QZ, vp, v)};
    Fr(w.X, QW, vp, v) = q.w;
    Fr(w.X, QX, vp, v) = q.x;
    Fr(w.X, QY, vp, v) = q.y;
    Fr(w.X, QZ, vp, v) = q.z;
    const V3 av = (keep * 2.0 * qvec(relative_rotation(pq, q))) / h;
    Fr(w.vel, WX, vp, v) = av.x;
    Fr(w.vel, WY, vp, v) = av.y;
    Fr(w.vel, WZ, vp, v) = av.z;
  }
}

__global__ void k_copy_state(int V, int vpad, const double* __restrict__ src, double* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
#pragma unroll
  for (int f = 0; f < kStateFields; ++f) dst[static_cast<long long>(f) * vpad + v] = src[static_cast<long long>(f) * vpad + v];
}

}  // namespace

void launch_animate_predict(const World& w, const double* anim, const AnimLayout& al, const int* pm_slot,
                            const int* act_rod_off, const int* act_list, double* act_applied, const int* act_rods,
                            int n_act_rods, const double* gravity_h, double h, int substep, unsigned long long* err,
                            const Collide* pills, cudaStream_t st) {
  if (al.n_pm > 0) launch_kernel(k_pin_motions, (al.n_pm + 127) / 128, 128, 0, st, g_pdl, w, anim, al, pm_slot);
  // act_static follows act_applied in the same allocation (see solver.cu)
  ActArgs aa{act_rod_off, act_list, act_applied, act_rods, act_applied + al.n_act, n_act_rods};
  const V3 g{gravity_h[0], gravity_h[1], gravity_h[2]};
  if (w.max_rod_n <= 32) {  // activation + prediction in one launch
    launch_kernel(k_predict_rods, n_act_rods + (w.R + kPredictRodsPerCta - 1) / kPredictRodsPerCta,
                  32 * kPredictRodsPerCta, 0, st, g_pdl, w, anim, al, g, h, substep, err, aa, pills ? *pills : Collide{},
                  pills ? 1 : 0);
    return;
  }
  if (n_act_rods > 0) launch_kernel(k_activation, n_act_rods, 128, 0, st, g_pdl, w, anim, al, aa);
  const int b = (w.V + 127) / 128;
  launch_kernel(k_predict_vertices, b, 128, 0, st, g_pdl, w, anim, al, g, h, substep, err);
  launch_kernel(k_predict_elements, b, 128, 0, st, g_pdl, w, h, substep, err);
}

void launch_finalize_from(const World& w, const double* src, double h, double keep, cudaStream_t st) {
  launch_kernel(k_finalize, (w.V + 127) / 128, 128, 0, st, g_pdl, w, src, h, keep);
}

void launch_copy_state(const World& w, const double* src, double* dst, cudaStream_t st) {
  launch_kernel(k_copy_state, (w.V + 127) / 128, 128, 0, st, g_pdl, w.V, w.vpad, src, dst);
}

}  // namespace vdev
