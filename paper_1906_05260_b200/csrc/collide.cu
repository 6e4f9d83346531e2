// Pill-pill collision: rod_pills (collision.cpp:275-296), bounding spheres (:137-153), the
// uniform-grid broad phase (:184-238) and the dichotomous narrow phase (:55-135, :251-273),
// plus half-plane block generation (solver.cpp:227-249). Compiled with --fmad=false so the
// narrow phase, the cell keys and every pill geometry value match the reference bit for bit.
//
// Broad phase on the GPU: the grid is an open-addressing hash table of cell keys built with
// atomicCAS (one representative pill per cell), a count -> exclusive scan -> scatter counting
// sort of pill ids into cells (with cell-sorted copies of the per-pill data the pair scan
// reads), then a 27-cell scan per pill (small worlds) or per cell (large worlds) that (1) counts
// every allowed pair j > i (StepReport.broad_pairs, exactly the reference's candidate count)
// and (2) keeps the pairs that can penetrate (bounding spheres, then segment distance). The
// candidate list is unordered; the narrow-phase hits are put in the reference's (i, j) order
// afterwards (k_ct_order in one CTA, or count -> scan -> scatter -> per-i sort).
#include <algorithm>
#include <cfloat>

#include <cstdlib>

#include "kernels.cuh"
#include "pill.cuh"
#include "pillbounds.cuh"
#include "vmath.cuh"

namespace vdev {

using namespace vm;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double pair_distance(const PillV& a, const PillPrep& b, double alpha, double& beta) {
  const V3 ca = (1.0 - alpha) * a.c0 + alpha * a.c1;
  const double ra = (1.0 - alpha) * a.r0 + alpha * a.r1;
  bool deg;
  double t;
  const double d = project(ca, b, t, deg);
  beta = t;
  return d - ra;
}
__device__ __forceinline__ bool pill_less(const PillV& a, const PillV& b) {  // collision.cpp:65-74
  if (a.c0.x != b.c0.x) return a.c0.x < b.c0.x;
  if (a.c0.y != b.c0.y) return a.c0.y < b.c0.y;
  if (a.c0.z != b.c0.z) return a.c0.z < b.c0.z;
  if (a.c1.x != b.c1.x) return a.c1.x < b.c1.x;
  if (a.c1.y != b.c1.y) return a.c1.y < b.c1.y;
  if (a.c1.z != b.c1.z) return a.c1.z < b.c1.z;
  if (a.r0 != b.r0) return a.r0 < b.r0;
  return a.r1 < b.r1;
}
// deepest_penetration, collision.cpp:78-135, in two parts: the dichotomous search (which does not
// depend on the warm start) and the final evaluations of lo, hi and the warm alpha. Split so the
// narrow phase can look the warm start up on another lane while the search runs.
struct DeepState {
  PillV pa;
  PillPrep pb;
  bool swapped;
  double lo, hi, best, best_a, best_b;
};
__device__ __forceinline__ void deepest_search(const PillV& A, const PillV& B, int iterations, DeepState& s) {
  s.swapped = pill_less(B, A);
  s.pa = s.swapped ? B : A;
  s.pb = prep_pill(s.swapped ? A : B);
  double lo = 0.0, hi = 1.0;
  double best_a = 0.5, best_b = 0.0;
  double best = pair_distance(s.pa, s.pb, 0.5, best_b);
  const double delta = 1e-6;
  for (int it = 0; it < iterations; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double x1 = mid - delta, x2 = mid + delta;
    double b1 = 0.0, b2 = 0.0;
    const double f1 = pair_distance(s.pa, s.pb, x1, b1);
    const double f2 = pair_distance(s.pa, s.pb, x2, b2);
    if (f1 < best) {
      best = f1;
      best_a = x1;
      best_b = b1;
    }
    if (f2 < best) {
      best = f2;
      best_a = x2;
      best_b = b2;
    }
    if (f1 <= f2) hi = x2;
    else lo = x1;
  }
  s.lo = lo;
  s.hi = hi;
  s.best = best;
  s.best_a = best_a;
  s.best_b = best_b;
}
__device__ __forceinline__ void deepest_finish(const DeepState& s, double warm, double& alpha_out, double& beta_out,
                                               double& dist_out) {
  if (s.swapped && warm >= 0.0) warm = -1.0;
  double best = s.best, best_a = s.best_a, best_b = s.best_b;
  const double cands[3] = {s.lo, s.hi, warm};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double cand = cands[k];
    if (cand < 0.0 || cand > 1.0) continue;
    double bc = 0.0;
    const double fc = pair_distance(s.pa, s.pb, cand, bc);
    if (fc < best) {
      best = fc;
      best_a = cand;
      best_b = bc;
    }
  }
  dist_out = best;
  if (s.swapped) {
    alpha_out = best_b;
    beta_out = best_a;
  } else {
    alpha_out = best_a;
    beta_out = best_b;
  }
}
__device__ void deepest(const PillV& A, const PillV& B, int iterations, double warm, double& alpha_out,
                        double& beta_out, double& dist_out) {
  DeepState s;
  deepest_search(A, B, iterations, s);
  deepest_finish(s, warm, alpha_out, beta_out, dist_out);
}
__device__ __forceinline__ unsigned long long pair_key(uint32_t ia, uint32_t ib) {  // collision.cpp:240-249
  if (ia > ib) {
    const uint32_t t = ia;
    ia = ib;
    ib = t;
  }
  return (static_cast<unsigned long long>(ia) << 32) | ib;
}
__device__ __forceinline__ uint32_t pill_id(int rod, int el) {
  return (static_cast<uint32_t>(rod + 1) << 16) | (static_cast<uint32_t>(el + 1) & 0xffffu);
}

__device__ __forceinline__ unsigned long long cell_hash(long long x, long long y, long long z, int scene) {
  unsigned long long h = static_cast<unsigned long long>(x) * 73856093ull ^
                         static_cast<unsigned long long>(y) * 19349663ull ^
                         static_cast<unsigned long long>(z) * 83492791ull ^
                         static_cast<unsigned long long>(scene) * 0x9e3779b97f4a7c15ull;
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  return h;
}

// pair_allowed, collision.cpp:172-180.
__device__ __forceinline__ bool pair_allowed(int ra, int ga, bool sa, int ea, int rb, int gb, int eb) {
  if (ra < 0 && rb < 0) return false;
  if (ga >= 0 && ga == gb) return false;
  if (ra >= 0 && ra == rb) {
    if (!sa) return false;
    if (abs(ea - eb) <= 1) return false;
  }
  return true;
}

// ---- pipeline kernels ----------------------------------------------------------------------

// rod_pills from the predicted state + the posed kinematic pills of this substep. bounds != 0
// (single-scene worlds; the broad phase's resets already ran): each pill's bounding sphere and the
// max radius too (k_bounds' work, one launch less).
__global__ void k_build_pills(World w, Collide c, const double* __restrict__ anim, AnimLayout al, int bounds,
                              int substep, unsigned long long* err) {
  pdl_wait();
  pdl_trigger();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long bits = 0;
  if (v < w.V) {
    const int k = w.slot_loc[v], m = w.slot_m[v];
    if (k < m) {
      const int r = w.slot_rod[v];
      const int i = v - r;
      const int vp = w.vpad;
      const double* X = w.X;
      const PillV p{V3{X[CX * vp + v], X[CY * vp + v], X[CZ * vp + v]},
                    V3{X[CX * vp + v + 1], X[CY * vp + v + 1], X[CZ * vp + v + 1]},
                    X[S * vp + v] * w.vstat[RBAR * vp + v], X[S * vp + v + 1] * w.vstat[RBAR * vp + v + 1]};
      double2* o = reinterpret_cast<double2*>(c.pill + 8ll * i);
      o[0] = make_double2(p.c0.x, p.c0.y);
      o[1] = make_double2(p.c0.z, p.c1.x);
      o[2] = make_double2(p.c1.y, p.c1.z);
      o[3] = make_double2(p.r0, p.r1);
      if (bounds) bits = pill_bounds(c, p, i, substep, err);
    }
  }
  if (v < al.n_kin) {
    const double* kp = anim + al.off_kin + 8 * v;
    const int i = w.E + v;
    for (int f = 0; f < 8; ++f) c.pill[8ll * i + f] = kp[f];
    if (bounds) {
      const unsigned long long b2 = pill_bounds(c, PillV{V3{kp[0], kp[1], kp[2]}, V3{kp[3], kp[4], kp[5]}, kp[6], kp[7]},
                                                i, substep, err);
      bits = b2 > bits ? b2 : bits;
    }
  }
  if (bounds) {  // warp max, one atomic per warp (max is order independent)
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_down_sync(0xffffffffu, bits, o);
      bits = x > bits ? x : bits;
    }
    if ((threadIdx.x & 31) == 0 && bits) atomicMax(c.maxr_bits, bits);
  }
}

// Bounding spheres, max radius, finiteness (broad_phase, collision.cpp:189-196).
__global__ void k_bounds(Collide c, int substep, unsigned long long* err) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long bits = 0;
  if (i < c.P) bits = pill_bounds(c, load_pill(c.pill, c.P, i), i, substep, err);
  // warp max, one atomic per warp (max is order independent); a batch keeps one max per scene
  const int sc = c.pill_scene && i < c.P ? c.pill_scene[i] : 0;
  const int sc0 = __shfl_sync(0xffffffffu, sc, 0);
  if (__all_sync(0xffffffffu, sc == sc0 || i >= c.P)) {
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_down_sync(0xffffffffu, bits, o);
      bits = v > bits ? v : bits;
    }
    if ((threadIdx.x & 31) == 0 && bits) atomicMax(c.pill_scene ? &c.scene_maxr[sc0] : c.maxr_bits, bits);
  } else if (bits) {
    atomicMax(&c.scene_maxr[sc], bits);
  }
}

__device__ __forceinline__ double cell_inv(const Collide& c, int scene) {
  const double maxr =
      __longlong_as_double(static_cast<long long>(c.pill_scene ? c.scene_maxr[scene] : *c.maxr_bits));
  const double cell = fmax(2.0 * maxr, 1e-12);  // collision.cpp:197-198
  return 1.0 / cell;
}
__device__ __forceinline__ long long key1(double x, double inv) {
  const double f = floor(x * inv);
  return isfinite(f) ? static_cast<long long>(f) : 0;
}

__global__ void k_insert(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.P) return;
  const int scene = c.pill_scene ? c.pill_scene[i] : 0;
  const double inv = cell_inv(c, scene);
  const long long kx = key1(c.bsph[i], inv), ky = key1(c.bsph[c.P + i], inv), kz = key1(c.bsph[2 * c.P + i], inv);
  c.cellkey[i] = kx;
  c.cellkey[c.P + i] = ky;
  c.cellkey[2 * c.P + i] = kz;
  __threadfence();
  const unsigned mask = static_cast<unsigned>(c.T - 1);
  unsigned h = static_cast<unsigned>(cell_hash(kx, ky, kz, scene)) & mask;
  int rep = 0;
  while (true) {
    int e = atomicCAS(&c.table[h], -1, i);
    if (e == -1) {  // new cell, i is its representative
      rep = 1;
      break;
    }
    const long long ex = static_cast<volatile long long*>(c.cellkey)[e];
    const long long ey = static_cast<volatile long long*>(c.cellkey)[c.P + e];
    const long long ez = static_cast<volatile long long*>(c.cellkey)[2 * c.P + e];
    if (ex == kx && ey == ky && ez == kz && (!c.pill_scene || c.pill_scene[e] == scene)) break;
    h = (h + 1) & mask;
  }
  c.pill_cell[i] = static_cast<int>(h);
  c.rep_flag[i] = rep;
  atomicAdd(&c.cell_count[h], 1);
}

// Non-empty cells listed in representative-pill order (spatially coherent, deterministic), each
// with the spans (first position in the cell-sorted arrays, size) of its half-stencil
// neighbourhood (see k_pairs_cell): the cell itself and its 13 lexicographically positive
// neighbours. The representative's thread probes the 13 neighbours' hash chains side by side
// (first probes, key checks and span loads each issued together), so the pair scan starts from
// ready spans instead of walking those chains cell by cell.
constexpr int kHalfStencil = 14;
__device__ __forceinline__ int find_cell(const Collide& c, long long kx, long long ky, long long kz, int scene);
__global__ void __launch_bounds__(128) k_cell_list(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int P = c.P;
  const unsigned mask = static_cast<unsigned>(c.T - 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    if (!c.rep_flag[i]) continue;
    const int ci = c.rep_pos[i];
    const int h = c.pill_cell[i];
    c.cell_list[ci] = h;
    const int scene = c.pill_scene ? c.pill_scene[i] : 0;
    const long long kx = c.cellkey[i], ky = c.cellkey[P + i], kz = c.cellkey[2 * P + i];
    // first probes of the 13 chains side by side: (span, key) of each hashed slot
    int a0[kHalfStencil - 1], a1[kHalfStencil - 1];
    bool hit[kHalfStencil - 1];
#pragma unroll
    for (int l = 1; l < kHalfStencil; ++l) {  // offsets (o/9-1, (o/3)%3-1, o%3-1), o = 13 + l
      const int o = 13 + l;
      const long long x = kx + (o / 9 - 1), y = ky + ((o / 3) % 3 - 1), z = kz + (o % 3 - 1);
      const int hh = static_cast<int>(static_cast<unsigned>(cell_hash(x, y, z, scene)) & mask);
      a0[l - 1] = c.cell_start[hh];
      a1[l - 1] = c.cell_start[hh + 1];
      const longlong4 k = c.slot_key[hh];
      hit[l - 1] = k.x == x && k.y == y && k.z == z && k.w == scene;
    }
    int2* span = c.cell_span + static_cast<long long>(kHalfStencil) * ci;
    span[0] = make_int2(c.cell_start[h], c.cell_start[h + 1] - c.cell_start[h]);
#pragma unroll
    for (int l = 1; l < kHalfStencil; ++l) {
      const int o = 13 + l;
      int2 v = make_int2(0, 0);
      if (a0[l - 1] != a1[l - 1]) {  // occupied slot
        if (hit[l - 1]) {
          v = make_int2(a0[l - 1], a1[l - 1] - a0[l - 1]);
        } else {  // rare: another cell in the slot, follow the chain
          const int hn = find_cell(c, kx + (o / 9 - 1), ky + ((o / 3) % 3 - 1), kz + (o % 3 - 1), scene);
          if (hn >= 0) v = make_int2(c.cell_start[hn], c.cell_start[hn + 1] - c.cell_start[hn]);
        }
      }
      span[l] = v;
    }
  }
}

__global__ void k_scatter(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.P) return;
  const int h = c.pill_cell[i];
  const int pos = c.cell_start[h] + atomicAdd(&c.cell_cursor[h], 1);
  c.cell_items[pos] = i;
  if (c.rep_flag[i])  // the slot's key, read beside cell_start by find_cell (one load round per probe)
    c.slot_key[h] = make_longlong4(c.cellkey[i], c.cellkey[c.P + i], c.cellkey[2 * c.P + i], c.pill_scene ? c.pill_scene[i] : 0);
  // cell-sorted copies of what the pair scan reads per neighbour: contiguous per cell, so the
  // scan's loads are coalesced and need no second indirection
  c.cell_attr[pos] = make_int4(i, c.pill_rod[i], c.pill_group[i], 2 * c.pill_el[i] + (c.pill_self[i] ? 1 : 0));
  double2* sp = reinterpret_cast<double2*>(c.cell_sph) + 2 * pos;
  sp[0] = make_double2(c.bsph[i], c.bsph[c.P + i]);
  sp[1] = make_double2(c.bsph[2 * c.P + i], c.bsph[3 * c.P + i]);
}

// The half-stencil span holding flattened item k: the largest d with off[d] <= k (off[0] = 0,
// off[14] = the total > k); empty spans share their start with the next, which this picks.
__device__ __forceinline__ int span_of(const int* off, int k) {
  int lo = 0, hi = 13;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= k) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// The table slot of cell (kx, ky, kz, scene), or -1 (after k_scatter). An occupied slot has a
// non-empty span in cell_start, and its key in slot_key: the three loads of a probe are
// independent, so each probe of the linear chain costs one load round; the chain ends at the
// first empty slot.
__device__ __forceinline__ int find_cell(const Collide& c, long long kx, long long ky, long long kz, int scene) {
  const unsigned mask = static_cast<unsigned>(c.T - 1);
  unsigned h = static_cast<unsigned>(cell_hash(kx, ky, kz, scene)) & mask;
  while (true) {
    const int a = c.cell_start[h], b = c.cell_start[h + 1];
    const longlong4 k = c.slot_key[h];
    if (a == b) return -1;
    if (k.x == kx && k.y == ky && k.z == kz && k.w == scene) return static_cast<int>(h);
    h = (h + 1) & mask;
  }
}

// Conservative "can these pills penetrate" test on the bounding spheres: a pair whose spheres
// are separated by more than a relative 1e-9 has a strictly positive deepest-penetration
// distance, so dropping it cannot change the contact set.
__device__ __forceinline__ bool spheres_touch(const Collide& c, int i, int j) {
  const double dx = c.bsph[i] - c.bsph[j], dy = c.bsph[c.P + i] - c.bsph[c.P + j],
               dz = c.bsph[2 * c.P + i] - c.bsph[2 * c.P + j];
  const double rr = (c.bsph[3 * c.P + i] + c.bsph[3 * c.P + j]) * (1.0 + 1e-9) + 1e-12;
  return dx * dx + dy * dy + dz * dz <= rr * rr;
}

// Warm alpha of `key` in a list increasing in (scene, key) — scene-major in a batch, where the
// pair ids are scene-local (the same pair_key as the scene alone).
__device__ __forceinline__ double warm_lookup(const unsigned long long* keys, const int* scenes, const double* alpha,
                                              int n, int scene, unsigned long long key) {
  int lo = 0, hi = n;  // lower_bound: first inserted wins on duplicate keys
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool less = scenes ? (scenes[mid] < scene || (scenes[mid] == scene && keys[mid] < key)) : keys[mid] < key;
    if (less) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && keys[lo] == key && (!scenes || scenes[lo] == scene)) ? alpha[lo] : -1.0;
}

// Squared distance between segments [p0,p1] and [q0,q1] (closest points of two segments,
// clamped parametric solution).
__device__ __forceinline__ double seg_seg_dist2(const V3& p0, const V3& p1, const V3& q0, const V3& q1) {
  const V3 d1 = p1 - p0, d2 = q1 - q0, r = p0 - q0;
  const double a = dot(d1, d1), e = dot(d2, d2), f = dot(d2, r);
  double s = 0.0, t = 0.0;
  if (a <= 1e-300 && e <= 1e-300) return sqnorm(r);
  if (a <= 1e-300) {
    t = fmin(fmax(f / e, 0.0), 1.0);
  } else {
    const double cc = dot(d1, r);
    if (e <= 1e-300) {
      s = fmin(fmax(-cc / a, 0.0), 1.0);
    } else {
      const double b = dot(d1, d2);
      const double denom = a * e - b * b;
      s = denom > 0.0 ? fmin(fmax((b * f - cc * e) / denom, 0.0), 1.0) : 0.0;
      t = (b * s + f) / e;
      if (t < 0.0) {
        t = 0.0;
        s = fmin(fmax(-cc / a, 0.0), 1.0);
      } else if (t > 1.0) {
        t = 1.0;
        s = fmin(fmax((b - cc) / a, 0.0), 1.0);
      }
    }
  }
  const V3 x = (p0 + s * d1) - (q0 + t * d2);
  return sqnorm(x);
}

// Conservative "can these pills penetrate" test. A pill lies inside its axis segment dilated by
// max(r0, r1), and every value deepest_penetration evaluates is >= dist(segments) - rmax_a -
// rmax_b (collision.cpp:9-61), so a pair whose segments are farther apart than the summed max
// radii (with a 1e-9 relative + 1e-12 absolute margin for rounding) has a strictly positive
// computed distance: dropping it cannot change the contact set. First the bounding spheres,
// then the exact segment distance.
__device__ __forceinline__ bool may_penetrate(const Collide& c, int i, int j) {
  const int P = c.P;
  const double dx = c.bsph[i] - c.bsph[j], dy = c.bsph[P + i] - c.bsph[P + j], dz = c.bsph[2 * P + i] - c.bsph[2 * P + j];
  const double rs = (c.bsph[3 * P + i] + c.bsph[3 * P + j]) * (1.0 + 1e-9) + 1e-12;
  if (dx * dx + dy * dy + dz * dz > rs * rs) return false;
  const PillV a = load_pill(c.pill, P, i), b = load_pill(c.pill, P, j);
  const double rr = (fmax(a.r0, a.r1) + fmax(b.r0, b.r1)) * (1.0 + 1e-9) + 1e-12;
  return seg_seg_dist2(a.c0, a.c1, b.c0, b.c1) <= rr * rr;
}

// One WARP per pill i. Lanes 0..26 probe the 27 cells of i's 3x3x3 block in parallel; the warp
// then strides over the flattened list of their items (uniform work per lane, kPairUnroll items
// per lane in flight), reading the cell-sorted copies (cell_attr, cell_sph) written by k_scatter.
// It counts every allowed pair j > i (broad_phase, collision.cpp:213-226 — StepReport.broad_pairs)
// and keeps the pairs whose bounding spheres touch (prefilter; all allowed pairs without it). Kept pairs
// collect in a per-warp shared buffer; the CTA reserves its slots with one atomic at the end
// (a full buffer flushes early with its own). The list is unordered; contacts are put in (i, j)
// order after the narrow phase.
// may_penetrate's exact segment test (out of line: keeps the pair scan's registers low)
__device__ __noinline__ bool segments_close(const double* __restrict__ pill, int P, int i, int j) {
  const PillV a = load_pill(pill, P, i), b = load_pill(pill, P, j);
  const double rr = (fmax(a.r0, a.r1) + fmax(b.r0, b.r1)) * (1.0 + 1e-9) + 1e-12;
  return seg_seg_dist2(a.c0, a.c1, b.c0, b.c1) <= rr * rr;
}
constexpr int kPairWarps = 8;
// 64 registers (4 CTAs per SM) keep all of C3's 3,712 pill warps in one wave; two items per lane
// in flight fit in them without spilling (measured: 15 us vs 18-20 us at 80 registers / 2 waves).
constexpr int kPairUnroll = 2;
constexpr int kPairBuf = 64;
__global__ void __launch_bounds__(32 * kPairWarps, 4) k_pairs_warp(Collide c, int prefilter, int* broad_total,
                                                                int* cand_total, int* out_i, int* out_j) {
  pdl_wait();
  pdl_trigger();
  constexpr int kHalf = 14;  // half stencil (see k_pairs_cell): the own cell + 13 positive offsets
  __shared__ int s_start[kPairWarps][kHalf];
  __shared__ int s_off[kPairWarps][kHalf + 1];
  __shared__ int s_buf[kPairWarps][kPairBuf];
  __shared__ int s_cnt[kPairWarps], s_broad[kPairWarps];
  __shared__ int s_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = c.P;
  const int i = blockIdx.x * kPairWarps + warp;
  const bool live = i < P;
  int size = 0;
  const int scene = live && c.pill_scene ? c.pill_scene[i] : 0;
  if (live && lane < kHalf) {
    const int o = 13 + lane;
    const int h = find_cell(c, c.cellkey[i] + (o / 9 - 1), c.cellkey[P + i] + ((o / 3) % 3 - 1),
                            c.cellkey[2 * P + i] + (o % 3 - 1), scene);
    if (h >= 0) {
      s_start[warp][lane] = c.cell_start[h];
      size = c.cell_start[h + 1] - c.cell_start[h];
    }
  }
  int incl = size;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane < kHalf) s_off[warp][lane + 1] = incl;
  if (lane == 0) s_off[warp][0] = 0;
  const int total = __shfl_sync(0xffffffffu, incl, kHalf - 1);
  __syncwarp();
  int ri = 0, gi = 0, ei = 0;
  bool si = false;
  double xi = 0, yi = 0, zi = 0, Ri = 0;
  if (live) {
    ri = c.pill_rod[i];
    gi = c.pill_group[i];
    ei = c.pill_el[i];
    si = c.pill_self[i] != 0;
    xi = c.bsph[i];
    yi = c.bsph[P + i];
    zi = c.bsph[2 * P + i];
    Ri = c.bsph[3 * P + i];
  }
  const int4* __restrict__ attr = c.cell_attr;
  const double2* __restrict__ sph = reinterpret_cast<const double2*>(c.cell_sph);
  const long long cap = c.cand_cap;
  int broad = 0, nbuf = 0, cur_d = 0;  // the span of the lane's current item (span_of)
  auto flush = [&]() {  // rare: the survivor buffer is full — reserve its slots with its own atomic
    int base = 0;
    if (lane == 0) base = atomicAdd(cand_total, nbuf);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int q = lane; q < nbuf; q += 32)
      if (base + q < cap) {
        out_i[base + q] = min(i, s_buf[warp][q]);
        out_j[base + q] = max(i, s_buf[warp][q]);
      }
    __syncwarp();
    nbuf = 0;
  };
  auto push = [&](bool keep, int j) {  // warp-uniform call: append the lanes' kept j
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) return;
    if (nbuf + __popc(m) > kPairBuf) flush();
    if (keep) s_buf[warp][nbuf + __popc(m & ((1u << lane) - 1))] = j;
    nbuf += __popc(m);
    __syncwarp();
  };
  if (live)
    for (int k0 = 0; k0 < total; k0 += 32 * kPairUnroll) {
      int4 at[kPairUnroll];
      double2 s01[kPairUnroll], s23[kPairUnroll];
      bool own[kPairUnroll];  // item from pill i's own cell (there only j > i counts)
#pragma unroll
      for (int u = 0; u < kPairUnroll; ++u) {
        const int k = k0 + u * 32 + lane;
        at[u].x = -1;
        own[u] = false;
        if (k < total) {
          cur_d = span_of(s_off[warp], k);
          own[u] = cur_d == 0;
          const int pos = s_start[warp][cur_d] + (k - s_off[warp][cur_d]);
          at[u] = attr[pos];
          s01[u] = sph[2 * pos];
          s23[u] = sph[2 * pos + 1];
        }
      }
#pragma unroll
      for (int u = 0; u < kPairUnroll; ++u) {
        const int j = at[u].x;
        bool cand = false;
        // pair_allowed(pills[min], pills[max]): its only asymmetry is the first pill's self_collide
        const bool s_first = j > i ? si : (at[u].w & 1) != 0;
        if (j >= 0 && (!own[u] || j > i) && pair_allowed(ri, gi, s_first, ei, at[u].y, at[u].z, at[u].w >> 1)) {
          ++broad;
          cand = true;
          if (prefilter) {  // spheres_touch on the cell-sorted copies
            const double dx = xi - s01[u].x, dy = yi - s01[u].y, dz = zi - s23[u].x;
            const double rs = (Ri + s23[u].y) * (1.0 + 1e-9) + 1e-12;
            cand = dx * dx + dy * dy + dz * dz <= rs * rs;
          }
        }
        push(cand, j);
      }
    }
  for (int o = 16; o > 0; o >>= 1) broad += __shfl_down_sync(0xffffffffu, broad, o);
  if (lane == 0) {
    s_cnt[warp] = nbuf;
    s_broad[warp] = broad;
    if (broad && c.pill_scene) atomicAdd(&c.scene_acc[scene].broad_pairs, broad);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int sum = 0, bsum = 0;
    for (int w = 0; w < kPairWarps; ++w) {
      const int v = s_cnt[w];
      s_cnt[w] = sum;
      sum += v;
      bsum += s_broad[w];
    }
    s_base = sum ? atomicAdd(cand_total, sum) : 0;
    if (bsum) atomicAdd(broad_total, bsum);
  }
  __syncthreads();
  const long long base = static_cast<long long>(s_base) + s_cnt[warp];
  for (int q = lane; q < nbuf; q += 32)
    if (base + q < cap) {
      out_i[base + q] = min(i, s_buf[warp][q]);
      out_j[base + q] = max(i, s_buf[warp][q]);
    }
}

// One WARP per non-empty grid cell (table slot), over a HALF stencil: the cell itself and the 13
// neighbours whose offset is lexicographically positive, so every pair of distinct cells is
// visited from exactly one side (the reference's 27-cell scan with j > i visits each pair from
// both sides and drops one). The 14 spans come ready from k_cell_list (lane l loads span l; the
// next cell's spans are loaded while this one is scanned). The cell's member pills are staged
// in shared memory from the cell-sorted copies (cell_attr, cell_sph), and the warp strides over
// the flattened neighbourhood items j, loading each j once and testing it against every member
// i. It counts every allowed pair once — j > i within the cell, any order across cells,
// evaluated as pair_allowed(pills[min], pills[max]) (its one asymmetric operand, the first
// pill's self_collide, is taken from the lower index; the sphere test is symmetric: commutative
// sums and squared differences) — for broad_phase (collision.cpp:213-226,
// StepReport.broad_pairs; the reference has no overlap test), and keeps the pairs whose bounding
// spheres touch (prefilter; all allowed pairs without it) as (min, max). Kept pairs collect in a
// per-warp shared buffer flushed with one atomic per fill. The list is unordered; contacts are
// put in (i, j) order after the narrow phase.
constexpr int kCellWarps = 8;
constexpr int kCellPathMinPills = 1 << 16;
constexpr int kCellBuf = 128;
__global__ void __launch_bounds__(32 * kCellWarps) k_pairs_cell(Collide c, int prefilter, int* broad_total,
                                                                int* cand_total) {
  pdl_wait();
  pdl_trigger();
  constexpr int kHalf = kHalfStencil;
  __shared__ int s_start[kCellWarps][kHalf];
  __shared__ int s_off[kCellWarps][kHalf + 1];
  __shared__ int4 s_ma[kCellWarps][32];
  __shared__ double2 s_m01[kCellWarps][32], s_m23[kCellWarps][32];
  __shared__ int s_buf[kCellWarps][2][kCellBuf];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = c.P;
  const int ncells = c.rep_pos[P];
  const int4* __restrict__ attr = c.cell_attr;
  const double2* __restrict__ sph = reinterpret_cast<const double2*>(c.cell_sph);
  const int cstride = gridDim.x * kCellWarps;
  int broad = 0, nbuf = 0, scene_broad_done = 0;
  int ci = blockIdx.x * kCellWarps + warp;
  int2 nspan = make_int2(0, 0);
  if (ci < ncells && lane < kHalf) nspan = c.cell_span[static_cast<long long>(kHalf) * ci + lane];
  for (; ci < ncells; ci += cstride) {
  const int2 span = nspan;
  if (ci + cstride < ncells && lane < kHalf) nspan = c.cell_span[static_cast<long long>(kHalf) * (ci + cstride) + lane];
  const int size = lane < kHalf ? span.y : 0;
  if (lane < kHalf) s_start[warp][lane] = span.x;
  int incl = size;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane < kHalf) s_off[warp][lane + 1] = incl;
  if (lane == 0) s_off[warp][0] = 0;
  const int total = __shfl_sync(0xffffffffu, incl, kHalf - 1);
  const int mbase = __shfl_sync(0xffffffffu, span.x, 0);
  const int n_c = __shfl_sync(0xffffffffu, span.y, 0);
  auto flush = [&]() {
    int base = 0;
    if (lane == 0) base = atomicAdd(cand_total, nbuf);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int q = lane; q < nbuf; q += 32) {
      const long long p = static_cast<long long>(base) + q;
      if (p < c.cand_cap) {
        c.cand_i[p] = s_buf[warp][0][q];
        c.cand_j[p] = s_buf[warp][1][q];
      }
    }
    __syncwarp();
    nbuf = 0;
  };
  int scene = 0;
  for (int ib = 0; ib < n_c; ib += 32) {
    const int nm = min(32, n_c - ib);
    __syncwarp();
    if (lane < nm) {
      const int pos = mbase + ib + lane;
      s_ma[warp][lane] = attr[pos];
      s_m01[warp][lane] = sph[2 * pos];
      s_m23[warp][lane] = sph[2 * pos + 1];
    }
    __syncwarp();
    if (ib == 0 && c.pill_scene) scene = c.pill_scene[s_ma[warp][0].x];
    int cur_d = 0;  // the span of the lane's current item (span_of)
    for (int k0 = 0; k0 < total; k0 += 32) {
      const int k = k0 + lane;
      int4 at = make_int4(-1, 0, 0, 0);
      double2 j01 = make_double2(0, 0), j23 = make_double2(0, 0);
      if (k < total) {
        cur_d = span_of(s_off[warp], k);
        const int pos = s_start[warp][cur_d] + (k - s_off[warp][cur_d]);
        at = attr[pos];
        j01 = sph[2 * pos];
        j23 = sph[2 * pos + 1];
      }
      const int j = at.x;
      const bool sj = (at.w & 1) != 0;
      for (int m = 0; m < nm; ++m) {
        const int4 mi = s_ma[warp][m];
        const int i = mi.x;
        bool cand = false;
        // pair_allowed(pills[min], pills[max]): its only asymmetry is the first pill's self_collide
        if (j >= 0 && (cur_d > 0 || j > i) &&
            pair_allowed(mi.y, mi.z, j > i ? (mi.w & 1) != 0 : sj, mi.w >> 1, at.y, at.z, at.w >> 1)) {
          ++broad;
          if (prefilter) {  // spheres_touch, same arithmetic
            const double2 m01 = s_m01[warp][m], m23 = s_m23[warp][m];
            const double dx = m01.x - j01.x, dy = m01.y - j01.y, dz = m23.x - j23.x;
            const double rr = (m23.y + j23.y) * (1.0 + 1e-9) + 1e-12;
            cand = dx * dx + dy * dy + dz * dz <= rr * rr;
          } else {
            cand = true;
          }
        }
        const unsigned msk = __ballot_sync(0xffffffffu, cand);
        if (msk) {
          if (nbuf + __popc(msk) > kCellBuf) flush();
          if (cand) {
            const int q = nbuf + __popc(msk & ((1u << lane) - 1));
            s_buf[warp][0][q] = min(i, j);
            s_buf[warp][1][q] = max(i, j);
          }
          nbuf += __popc(msk);
        }
      }
    }
  }
  __syncwarp();
  if (nbuf) flush();
  if (c.pill_scene) {  // batch: per-scene count (a cell belongs to one scene)
    int b = broad;
    for (int o = 16; o > 0; o >>= 1) b += __shfl_down_sync(0xffffffffu, b, o);
    if (lane == 0 && b) atomicAdd(&c.scene_acc[scene].broad_pairs, b);
    broad = 0;
    scene_broad_done += b;
  }
  }  // cells of this warp
  for (int o = 16; o > 0; o >>= 1) broad += __shfl_down_sync(0xffffffffu, broad, o);
  if (lane == 0 && (broad || scene_broad_done)) atomicAdd(broad_total, broad + scene_broad_done);
}

// Exact conservative segment test (see may_penetrate) over the sphere-filtered candidates;
// survivors are compacted (warp-aggregated append) into cand2 so the expensive narrow phase
// runs without divergence.
__global__ void k_seg_filter(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCAND];
  const int lane = threadIdx.x & 31;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long q0 = blockIdx.x * static_cast<long long>(blockDim.x); q0 < n; q0 += stride) {
    const long long q = q0 + threadIdx.x;
    int i = 0, j = 0;
    bool keep = false;
    if (q < n) {
      i = c.cand_i[q];
      j = c.cand_j[q];
      const PillV A = load_pill(c.pill, c.P, i), B = load_pill(c.pill, c.P, j);
      const double rr = (fmax(A.r0, A.r1) + fmax(B.r0, B.r1)) * (1.0 + 1e-9) + 1e-12;
      keep = seg_seg_dist2(A.c0, A.c1, B.c0, B.c1) <= rr * rr;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    int base = 0;
    if (lane == 0 && mask) base = atomicAdd(&c.scalars[SC_NCAND2], __popc(mask));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
      const long long k = base + __popc(mask & ((1u << lane) - 1));
      c.cand2_i[k] = i;  // k < n <= cand_cap
      c.cand2_j[k] = j;
    }
  }
}

// Narrow phase over the unordered candidates; penetrating pairs are appended (warp-aggregated)
// to the raw contact list. Large worlds (kQuad = false, throughput-bound): one thread per
// candidate. Small worlds (latency-bound): four lanes per candidate: each step of the dichotomous search
// evaluates x1 and x2 on two lanes at once (a pair_distance is a ~1k-cycle dependent FP64 chain
// of two square roots and a division), the start value and the final lo / hi / warm candidates
// run side by side, and the fourth lane does the exact segment test and the warm-start binary
// search while the first step runs. Every evaluation is the reference's, on the same inputs,
// and the comparisons happen in the reference's order: the result is bit-identical to deepest().
// raw_idx >= 0 (k_pairs_warp's path): the candidates are the first scalars[raw_idx] (unclamped)
// sphere-touching pairs in cand_i/cand_j; the count is clamped here (k_clamp_raw's job on the
// other path) and each pair first passes k_seg_filter's exact segment test.
template <bool kQuad>
__global__ void __launch_bounds__(kQuad ? 64 : 256, kQuad ? 1 : 3) k_narrow_append(Collide c, int split_warm, int raw_idx, int seg_test) {
  pdl_wait();
  pdl_trigger();
  int n = c.scalars[SC_NCAND2];
  const int* ci = c.cand2_i;
  const int* cj = c.cand2_j;
  if (raw_idx >= 0) {
    const int t = c.scalars[raw_idx];
    n = t > c.cand_cap ? static_cast<int>(c.cand_cap) : t;
    if (t > c.cand_cap && blockIdx.x == 0 && threadIdx.x == 0) atomicExch(&c.scalars[SC_OVF], 1);
    ci = c.cand_i;
    cj = c.cand_j;
  }
  const int nrr = c.scalars[SC_NRR_PREV], nrk = c.scalars[SC_NRK_PREV];
  if (!kQuad) {  // large worlds (throughput-bound): one thread per candidate, deepest() as is
    const int lane = threadIdx.x & 31;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long q0 = blockIdx.x * static_cast<long long>(blockDim.x); q0 < n; q0 += stride) {
      const long long q = q0 + threadIdx.x;
      int i = 0, j = 0;
      double al = 0, be = 0, d = 1.0;
      if (q < n) {
        i = ci[q];
        j = cj[q];
      }
      if (q < n && (!seg_test || segments_close(c.pill, c.P, i, j))) {
        const unsigned long long key = pair_key(c.pill_id[i], c.pill_id[j]);
        const int scene = c.pill_scene ? c.pill_scene[i] : 0;
        double warm;
        if (!split_warm || (c.pill_rod[i] >= 0 && c.pill_rod[j] >= 0))
          warm = warm_lookup(c.warm_rr_key, c.warm_rr_scene, c.warm_rr_alpha, nrr, scene, key);
        else
          warm = warm_lookup(c.warm_rk_key, c.warm_rk_scene, c.warm_rk_alpha, nrk, scene, key);
        deepest(load_pill(c.pill, c.P, i), load_pill(c.pill, c.P, j), c.iters_dich, warm, al, be, d);
      }
      const bool hit = q < n && d < 0.0;
      const unsigned mask = __ballot_sync(0xffffffffu, hit);
      int base = 0;
      if (lane == 0 && mask) base = atomicAdd(&c.scalars[SC_NCT_RAW], __popc(mask));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (hit) {
        const long long k = base + __popc(mask & ((1u << lane) - 1));
        if (k < c.contact_cap) {
          c.raw_i[k] = i;
          c.raw_j[k] = j;
          c.raw_ab[k] = al;
          c.raw_ab[c.contact_cap + k] = be;
        }
      }
    }
    return;
  }
  const int lane = threadIdx.x & 31, r = lane & 3, gb = lane & ~3;
  const double delta = 1e-6;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t0 = blockIdx.x * static_cast<long long>(blockDim.x); (t0 >> 2) < n; t0 += stride) {
    const long long q = (t0 + threadIdx.x) >> 2;  // t0 is CTA-uniform: whole warps iterate together
    const bool live = q < n;
    int i = 0, j = 0;
    if (live) {
      i = ci[q];
      j = cj[q];
    }
    // phase A: lanes 0 / 1 evaluate the first iteration's x1 / x2, lane 2 the start value at 0.5
    // (none depends on another); lane 3 runs the exact segment test and the warm-start lookup
    bool keep = false, swapped = false;
    double warm = -1.0, f = 0.0, b = 0.0;
    PillV pa{};
    PillPrep pb{};
    if (live) {
      if (r == 3) {
        keep = !seg_test || segments_close(c.pill, c.P, i, j);
        if (keep) {
          const unsigned long long key = pair_key(c.pill_id[i], c.pill_id[j]);
          const int scene = c.pill_scene ? c.pill_scene[i] : 0;
          if (!split_warm || (c.pill_rod[i] >= 0 && c.pill_rod[j] >= 0))
            warm = warm_lookup(c.warm_rr_key, c.warm_rr_scene, c.warm_rr_alpha, nrr, scene, key);
          else
            warm = warm_lookup(c.warm_rk_key, c.warm_rk_scene, c.warm_rk_alpha, nrk, scene, key);
        }
      } else {
        const PillV A = load_pill(c.pill, c.P, i), B = load_pill(c.pill, c.P, j);
        swapped = pill_less(B, A);
        pa = swapped ? B : A;
        pb = prep_pill(swapped ? A : B);
        const double mid = 0.5 * (0.0 + 1.0);
        f = pair_distance(pa, pb, r == 2 ? 0.5 : (r == 0 ? mid - delta : mid + delta), b);
      }
    }
    keep = __shfl_sync(0xffffffffu, static_cast<int>(keep), gb + 3) != 0;
    warm = __shfl_sync(0xffffffffu, warm, gb + 3);
    // the dichotomous search (deepest_penetration, collision.cpp:78-135): every lane of the group
    // keeps the same state from the shuffled evaluations; lanes 0 / 1 evaluate x1 / x2
    double best = __shfl_sync(0xffffffffu, f, gb + 2), best_b = __shfl_sync(0xffffffffu, b, gb + 2);
    double best_a = 0.5, lo = 0.0, hi = 1.0;
    for (int it = 0; it < c.iters_dich; ++it) {
      const double mid = 0.5 * (lo + hi);
      const double x1 = mid - delta, x2 = mid + delta;
      if (it > 0 && live && r < 2) f = pair_distance(pa, pb, r == 0 ? x1 : x2, b);
      const double f1 = __shfl_sync(0xffffffffu, f, gb), b1 = __shfl_sync(0xffffffffu, b, gb);
      const double f2 = __shfl_sync(0xffffffffu, f, gb + 1), b2 = __shfl_sync(0xffffffffu, b, gb + 1);
      if (f1 < best) {
        best = f1;
        best_a = x1;
        best_b = b1;
      }
      if (f2 < best) {
        best = f2;
        best_a = x2;
        best_b = b2;
      }
      if (f1 <= f2) hi = x2;
      else lo = x1;
    }
    // final candidates lo, hi, warm on lanes 0, 1, 2; compared in that order on lane 0
    if (swapped && warm >= 0.0) warm = -1.0;
    const double cand = r == 0 ? lo : (r == 1 ? hi : warm);
    bool valid = false;
    double fc = 0.0, bc = 0.0;
    if (live && keep && r < 3 && !(cand < 0.0 || cand > 1.0)) {
      valid = true;
      fc = pair_distance(pa, pb, cand, bc);
    }
    double al = 0, be = 0, d = 1.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const bool vk = __shfl_sync(0xffffffffu, static_cast<int>(valid), gb + k) != 0;
      const double ck = __shfl_sync(0xffffffffu, cand, gb + k);
      const double fk = __shfl_sync(0xffffffffu, fc, gb + k), bk = __shfl_sync(0xffffffffu, bc, gb + k);
      if (vk && fk < best) {
        best = fk;
        best_a = ck;
        best_b = bk;
      }
    }
    if (keep) {
      d = best;
      al = swapped ? best_b : best_a;
      be = swapped ? best_a : best_b;
    }
    const bool hit = live && r == 0 && d < 0.0;
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    int base = 0;
    if (lane == 0 && mask) base = atomicAdd(&c.scalars[SC_NCT_RAW], __popc(mask));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (hit) {
      const long long k = base + __popc(mask & ((1u << lane) - 1));
      if (k < c.contact_cap) {
        c.raw_i[k] = i;
        c.raw_j[k] = j;
        c.raw_ab[k] = al;
        c.raw_ab[c.contact_cap + k] = be;
      }
    }
  }
}

// (i, j) ordering of the raw contacts: count per pill i -> scan -> scatter -> per-i sort by j.
__global__ void k_ct_count(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCT];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    atomicAdd(&c.ct_cnt[c.raw_i[k]], 1);
}
__global__ void k_ct_scatter(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCT];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int i = c.raw_i[k];
    const int pos = c.ct_off[i] + atomicAdd(&c.ct_cur[i], 1);
    c.ct_a[pos] = i;
    c.ct_b[pos] = c.raw_j[k];
    c.ct_alpha[pos] = c.raw_ab[k];
    c.ct_beta[pos] = c.raw_ab[c.contact_cap + k];
  }
}
__device__ void sort_pill_contacts(const Collide& c, int i);
__global__ void k_ct_sort(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < c.P) sort_pill_contacts(c, i);
}
// pill i's contacts sorted by j (the pairs are unique): up to 8 in registers — all loads in flight
// together, a fixed compare-exchange network, one store round — else an insertion sort in place
__device__ void sort_pill_contacts(const Collide& c, int i) {
  const int s0 = c.ct_off[i], s1 = c.ct_off[i + 1];
#ifndef VROD_CT_SORT_GLOBAL
  constexpr int kR = 8;
  if (s1 - s0 <= 1) return;
  if (s1 - s0 <= kR) {
    int kj[kR];
    double ka[kR], kb[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const bool in = s0 + u < s1;
      kj[u] = in ? c.ct_b[s0 + u] : 0x7fffffff;
      ka[u] = in ? c.ct_alpha[s0 + u] : 0.0;
      kb[u] = in ? c.ct_beta[s0 + u] : 0.0;
    }
#pragma unroll
    for (int a = 1; a < kR; ++a)
#pragma unroll
      for (int b = a; b > 0; --b)
        if (kj[b - 1] > kj[b]) {
          const int tj = kj[b - 1];
          kj[b - 1] = kj[b];
          kj[b] = tj;
          const double ta = ka[b - 1];
          ka[b - 1] = ka[b];
          ka[b] = ta;
          const double tb = kb[b - 1];
          kb[b - 1] = kb[b];
          kb[b] = tb;
        }
#pragma unroll
    for (int u = 0; u < kR; ++u)
      if (s0 + u < s1) {
        c.ct_b[s0 + u] = kj[u];
        c.ct_alpha[s0 + u] = ka[u];
        c.ct_beta[s0 + u] = kb[u];
      }
    return;
  }
#endif
  for (int a = s0 + 1; a < s1; ++a) {
    const int kj = c.ct_b[a];
    const double ka = c.ct_alpha[a], kb = c.ct_beta[a];
    int b = a - 1;
    while (b >= s0 && c.ct_b[b] > kj) {
      c.ct_b[b + 1] = c.ct_b[b];
      c.ct_alpha[b + 1] = c.ct_alpha[b];
      c.ct_beta[b + 1] = c.ct_beta[b];
      --b;
    }
    c.ct_b[b + 1] = kj;
    c.ct_alpha[b + 1] = ka;
    c.ct_beta[b + 1] = kb;
  }
}
__global__ void k_clamp_raw(int* scalars, int raw, int out, long long cap, int ovf_code) {
  pdl_wait();
  pdl_trigger();
  const int t = scalars[raw];
  if (t > cap) atomicExch(&scalars[SC_OVF], ovf_code);
  scalars[out] = t > cap ? static_cast<int>(cap) : t;
}

// (i, j) ordering of the raw contacts in ONE CTA (small worlds: one launch instead of five).
// Up to `smem_cap` contacts the unique keys (i, j) + raw index, packed in 64 bits, go to shared
// memory: up to 1024 each key's rank is counted directly (one thread per key), beyond that a
// bitonic sort (padded to the next power of two) runs over just the warps it needs. More contacts: the counting sort of
// the multi-launch path (count per i, scan, scatter, per-i insertion sort) run by this CTA in
// global memory — slow but correct; the host then switches the next recording to the
// multi-launch path. Either way the output is the same total (i, j) order.
constexpr int kOrderThreads = 1024;
__device__ __forceinline__ int block_excl_1024(int v, int* total, int* ws) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int y = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    ws[lane] = y;
  }
  __syncthreads();
  const int r = (wid ? ws[wid - 1] : 0) + x - v;
  *total = ws[31];
  __syncthreads();
  return r;
}
// The warm-start list entry of ordered contact k (pair key, frozen alpha; k_warm_build without the
// kinematic split) and the substep's contact counters (k_warm_counts), for the fused small-world
// ordering kernel.
__device__ __forceinline__ void warm_rr_put(const Collide& c, int k, int a, int b, double alpha) {
  const unsigned long long key = pair_key(c.pill_id[a], c.pill_id[b]);
  const int scene = c.pill_scene ? c.pill_scene[a] : 0;
  if (c.pill_scene) {
    atomicAdd(&c.scene_acc[scene].contact_count, 1);
    c.warm_rr_scene[k] = scene;
  }
  c.warm_rr_key[k] = key;
  c.warm_rr_alpha[k] = alpha;
}
__device__ __forceinline__ void warm_counts_unsplit(const Collide& c, StepAccum* acc, int n) {
  atomicAdd(&acc->contact_count, n);
  atomicAdd(&acc->broad_pairs, c.scalars[SC_BROAD]);
  if (c.scalars[SC_NCT_RAW] > acc->max_contacts) acc->max_contacts = c.scalars[SC_NCT_RAW];
  if (c.scalars[SC_NCAND_RAW] > acc->max_candidates) acc->max_candidates = c.scalars[SC_NCAND_RAW];
  c.scalars[SC_NRK_PREV] = 0;
  c.scalars[SC_NRR_PREV] = n;
}

// `acc` non-null (small worlds without kinematic pills): the ordering kernel also clamps the raw
// contact count (k_clamp_raw), builds the warm-start list (k_warm_build) and the counters
// (k_warm_counts) — three launches less per substep, the same writes.
__global__ void __launch_bounds__(kOrderThreads) k_ct_order(Collide c, int smem_cap, StepAccum* acc) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ unsigned long long okey[];  // smem_cap packed keys
  __shared__ int ws[32];
  const int tid = threadIdx.x;
  int n;
  if (acc) {  // k_clamp_raw (contacts) + k_warm_counts
    const int raw = c.scalars[SC_NCT_RAW];
    n = raw > c.contact_cap ? static_cast<int>(c.contact_cap) : raw;
    if (tid == 0) {
      if (raw > c.contact_cap) atomicExch(&c.scalars[SC_OVF], 2);
      c.scalars[SC_NCT] = n;
      warm_counts_unsplit(c, acc, n);
    }
  } else {
    n = c.scalars[SC_NCT];
  }
  if (n == 0) return;
  if (n <= smem_cap && c.P <= 65536) {
    // packed key (i << 48 | j << 32 | raw index): pill ids < 2^16 here, so sorting the packed
    // words sorts by (i, j) and carries the raw index along
    const bool rank = n <= kOrderThreads;
    int m = 2;
    while (m < n) m <<= 1;
    // only the warps the sort needs take part (named barrier over `act` threads)
    const int act = rank ? (n + 31) & ~31 : min(kOrderThreads, m >> 1);
    if (tid >= act) return;
    auto bar = [act]() { asm volatile("bar.sync 1, %0;" ::"r"(act) : "memory"); };
    const int fill = rank ? (n + 1) & ~1 : m;
    for (int k = tid; k < fill; k += act)
      okey[k] = k < n ? (static_cast<unsigned long long>(c.raw_i[k]) << 48) |
                            (static_cast<unsigned long long>(c.raw_j[k]) << 32) | static_cast<unsigned>(k)
                      : ~0ull;
    bar();
    auto emit = [&](int r, unsigned long long key) {
      const int q = static_cast<int>(key & 0xffffffffu);
      const int a = static_cast<int>(key >> 48), b = static_cast<int>((key >> 32) & 0xffffu);
      const double alpha = c.raw_ab[q];
      c.ct_a[r] = a;
      c.ct_b[r] = b;
      c.ct_alpha[r] = alpha;
      c.ct_beta[r] = c.raw_ab[c.contact_cap + q];
      if (acc) warm_rr_put(c, r, a, b, alpha);
    };
    if (rank) {  // one key per thread: its rank among the (unique) keys, broadcast pair reads
      if (tid >= n) return;
      const unsigned long long key = okey[tid];
      const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(okey);
      int r = 0;
#pragma unroll 4
      for (int q = 0; q < fill / 2; ++q) {
        const ulonglong2 v = k2[q];
        r += (v.x < key) + (v.y < key);
      }
      emit(r, key);
      return;
    }
    for (int size = 2; size <= m; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = tid; t < (m >> 1); t += act) {
          const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
          const unsigned long long x = okey[lo], y = okey[hi];
          if ((x > y) == ((lo & size) == 0)) {
            okey[lo] = y;
            okey[hi] = x;
          }
        }
        bar();
      }
    for (int k = tid; k < n; k += act) emit(k, okey[k]);
    return;
  }
  const int P = c.P;
  for (int k = tid; k <= P; k += kOrderThreads) {
    c.ct_cnt[k] = 0;
    c.ct_cur[k] = 0;
  }
  __syncthreads();
  for (int k = tid; k < n; k += kOrderThreads) atomicAdd(&c.ct_cnt[c.raw_i[k]], 1);
  __syncthreads();
  int carry = 0;
  for (int b = 0; b < P; b += kOrderThreads) {
    const int v = b + tid < P ? c.ct_cnt[b + tid] : 0;
    int total;
    const int ex = block_excl_1024(v, &total, ws);
    if (b + tid < P) c.ct_off[b + tid] = carry + ex;
    carry += total;
  }
  if (tid == 0) c.ct_off[P] = carry;
  __syncthreads();
  for (int k = tid; k < n; k += kOrderThreads) {
    const int i = c.raw_i[k];
    const int pos = c.ct_off[i] + atomicAdd(&c.ct_cur[i], 1);
    c.ct_a[pos] = i;
    c.ct_b[pos] = c.raw_j[k];
    c.ct_alpha[pos] = c.raw_ab[k];
    c.ct_beta[pos] = c.raw_ab[c.contact_cap + k];
  }
  __syncthreads();
  for (int i = tid; i < P; i += kOrderThreads) sort_pill_contacts(c, i);
  if (acc) {
    __syncthreads();
    for (int k = tid; k < n; k += kOrderThreads) warm_rr_put(c, k, c.ct_a[k], c.ct_b[k], c.ct_alpha[k]);
  }
}

// Narrow phase over the candidate list (find_contacts, collision.cpp:261-271).
__global__ void k_narrow(Collide c, int split_warm, int store_d) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCAND];
  const int nrr = c.scalars[SC_NRR_PREV], nrk = c.scalars[SC_NRK_PREV];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = c.cand_i[q], j = c.cand_j[q];
    const unsigned long long key = pair_key(c.pill_id[i], c.pill_id[j]);
    double warm;
    if (!split_warm || (c.pill_rod[i] >= 0 && c.pill_rod[j] >= 0))
      warm = warm_lookup(c.warm_rr_key, nullptr, c.warm_rr_alpha, nrr, 0, key);
    else
      warm = warm_lookup(c.warm_rk_key, nullptr, c.warm_rk_alpha, nrk, 0, key);
    double al, be, d;
    deepest(load_pill(c.pill, c.P, i), load_pill(c.pill, c.P, j), c.iters_dich, warm, al, be, d);
    c.cand_flag[q] = d < 0.0 ? 1 : 0;
    c.cand_ab[q] = al;
    c.cand_ab[c.cand_cap + q] = be;
    if (store_d) c.cand_ab[2 * c.cand_cap + q] = d;
  }
}

__global__ void k_compact_contacts(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCAND];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    if (!c.cand_flag[q]) continue;
    const long long k = c.cand_pos[q];
    if (k >= c.contact_cap) continue;
    c.ct_a[k] = c.cand_i[q];
    c.ct_b[k] = c.cand_j[q];
    c.ct_alpha[k] = c.cand_ab[q];
    c.ct_beta[k] = c.cand_ab[c.cand_cap + q];
    if (c.ct_dist) c.ct_dist[k] = c.cand_ab[2 * c.cand_cap + q];
  }
}


__global__ void k_cand_to_raw(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCAND];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    c.raw_i[k] = c.cand_i[k];
    c.raw_j[k] = c.cand_j[k];
    c.raw_ab[k] = 0.0;
    c.raw_ab[c.contact_cap + k] = 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c.scalars[SC_NCT] = n;
}

// Warm list for the next substep: (pair key, alpha) of the new contacts (solver.cpp:210-214).
// Rod-rod contacts in (i, j) order have increasing keys; contacts with a kinematic pill are
// kept in a second list, also increasing in key, so both are searchable by lower_bound.
__global__ void k_warm_flags(Collide c) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCT];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    c.rk_flag[k] = (c.pill_rod[c.ct_a[k]] < 0 || c.pill_rod[c.ct_b[k]] < 0) ? 1 : 0;
}
__global__ void k_warm_build(Collide c, int split) {
  pdl_wait();
  pdl_trigger();
  const int n = c.scalars[SC_NCT];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const unsigned long long key = pair_key(c.pill_id[c.ct_a[k]], c.pill_id[c.ct_b[k]]);
    const int scene = c.pill_scene ? c.pill_scene[c.ct_a[k]] : 0;
    if (c.pill_scene) atomicAdd(&c.scene_acc[scene].contact_count, 1);
    if (!split) {
      c.warm_rr_key[k] = key;
      c.warm_rr_alpha[k] = c.ct_alpha[k];
      if (c.pill_scene) c.warm_rr_scene[k] = scene;
    } else if (c.rk_flag[k]) {
      const int p = c.rk_pos[k];
      c.warm_rk_key[p] = key;
      c.warm_rk_alpha[p] = c.ct_alpha[k];
      if (c.pill_scene) c.warm_rk_scene[p] = scene;
    } else {
      const int p = k - c.rk_pos[k];
      c.warm_rr_key[p] = key;
      c.warm_rr_alpha[p] = c.ct_alpha[k];
      if (c.pill_scene) c.warm_rr_scene[p] = scene;
    }
  }
}
// The step report's collision counters (solver.cpp:203-225) and the sizes of the warm lists the
// next substep looks up.
__global__ void k_warm_counts(Collide c, int split, StepAccum* acc) {
  pdl_wait();
  pdl_trigger();
  atomicAdd(&acc->contact_count, c.scalars[SC_NCT]);
  atomicAdd(&acc->broad_pairs, c.scalars[SC_BROAD]);
  if (c.scalars[SC_NCT_RAW] > acc->max_contacts) acc->max_contacts = c.scalars[SC_NCT_RAW];
  if (c.scalars[SC_NCAND_RAW] > acc->max_candidates) acc->max_candidates = c.scalars[SC_NCAND_RAW];
  const int n = c.scalars[SC_NCT];
  const int nrk = split ? c.rk_pos[n] : 0;
  c.scalars[SC_NRK_PREV] = nrk;
  c.scalars[SC_NRR_PREV] = n - nrk;
}

// Half-plane blocks (solver.cpp:229-249): plane-major, then global vertex order.
__global__ void k_hp_flags(World w, Collide c) {
  pdl_wait();
  pdl_trigger();
  const long long n = static_cast<long long>(c.n_planes) * w.V;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(q / w.V);
    const int v = static_cast<int>(q - static_cast<long long>(p) * w.V);
    if (c.plane_scene && c.plane_scene[p] != w.rod_scene[w.slot_rod[v]]) {  // batch: own scene's planes only
      c.hp_flag[q] = 0;
      continue;
    }
    const int vp = w.vpad;
    const double* pl = c.planes + 4 * p;
    const V3 nrm{pl[0], pl[1], pl[2]};
    const V3 x{w.X[CX * vp + v], w.X[CY * vp + v], w.X[CZ * vp + v]};
    const double wr = w.X[S * vp + v] * w.vstat[RBAR * vp + v];
    const double clearance = dot(nrm, x) - pl[3] - wr;
    c.hp_flag[q] = clearance < 0.5 * wr ? 1 : 0;
  }
}
__global__ void k_hp_compact(World w, Collide c) {
  pdl_wait();
  pdl_trigger();
  const long long n = static_cast<long long>(c.n_planes) * w.V;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!c.hp_flag[q]) continue;
    const int k = c.hp_pos[q];
    const int p = static_cast<int>(q / w.V);
    c.hp_slot[k] = static_cast<int>(q - static_cast<long long>(p) * w.V);
    c.hp_plane[k] = p;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c.scalars[SC_NHP] = c.hp_pos[n];
}

// ---- standalone fine-grained entry points ----------------------------------------------------

struct PillAoS {  // vrod_pill layout
  double c0[3], c1[3], r0, r1;
  int rod, element, group, self_collide;
};
__device__ __forceinline__ PillV from_aos(const PillAoS& p) {
  return PillV{V3{p.c0[0], p.c0[1], p.c0[2]}, V3{p.c1[0], p.c1[1], p.c1[2]}, p.r0, p.r1};
}
__global__ void k_pill_project(long long n, const double* __restrict__ x, const PillAoS* __restrict__ pills,
                               double* t, double* d, uint8_t* deg) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const PillPrep p = prep_pill(from_aos(pills[i]));
    double tt;
    bool g;
    const double dd = project(V3{x[3 * i], x[3 * i + 1], x[3 * i + 2]}, p, tt, g);
    t[i] = tt;
    d[i] = dd;
    deg[i] = g ? 1 : 0;
  }
}
__global__ void k_deepest(long long n, const PillAoS* __restrict__ a, const PillAoS* __restrict__ b, int iters,
                          const double* __restrict__ warm, double* alpha, double* beta, double* dist) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double al, be, d;
    deepest(from_aos(a[i]), from_aos(b[i]), iters, warm ? warm[i] : -1.0, al, be, d);
    alpha[i] = al;
    beta[i] = be;
    dist[i] = d;
  }
}

int grid_for(long long n) {
  const long long b = (n + kThreads - 1) / kThreads;
  return static_cast<int>(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}
// The narrow phase is FP64-issue-bound per SM (≈ 6k FP64-heavy instructions per candidate
// warp): two-warp CTAs, so the live candidates (a prefix of the grid) spread over all SMs
// instead of queueing on the few SMs that 256-thread CTAs would put them on.
constexpr int kNarrowThreads = 64;
int narrow_grid(long long cand_cap) {
  const long long b = (4 * cand_cap + kNarrowThreads - 1) / kNarrowThreads;
  return static_cast<int>(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

}  // namespace

// Broad + narrow phase on the pill arrays already in `c` (pill, pill_rod/el/group/self/id).
// prefilter=0 keeps every allowed pair (the standalone broad_phase contract).
void launch_narrow_only(Collide& c, int split_warm, int store_d, cudaStream_t st) {
  const int g = grid_for(c.cand_cap);
  launch_kernel(k_narrow, g, kThreads, 0, st, g_pdl, c, split_warm, store_d);
  scan_exclusive(c.cand_flag, c.cand_pos, c.cand_cap, c.scalars + SC_NCAND, c.scan_tmp, c.scan_parts, st);
  launch_kernel(k_compact_contacts, g, kThreads, 0, st, g_pdl, c);
}

// Puts the first scalars[SC_NCT] raw (i, j, alpha, beta) records into (i, j) order in ct_*.
int order_cap_for(int P) {
  const char* env = std::getenv("VROD_CT_ORDER_CAP");  // tests: 0 forces the single-CTA fallback, -1 the multi-launch path
  if (env) return std::atoi(env);
  return P < kCellPathMinPills ? 4096 : -1;
}

void launch_order_contacts(Collide& c, cudaStream_t st, StepAccum* fuse_acc) {
  if (c.order_smem_cap >= 0) {  // one CTA (small worlds)
    const std::size_t smem = 8ull * (c.order_smem_cap + 2);
    cudaFuncSetAttribute(k_ct_order, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    launch_kernel(k_ct_order, 1, kOrderThreads, smem, st, g_pdl, c, c.order_smem_cap, fuse_acc);
    return;
  }
  const int g = grid_for(c.contact_cap);
  FillList f;
  f.add(c.ct_cnt, c.P + 1, 0);
  f.add(c.ct_cur, c.P + 1, 0);
  launch_fill(f, st);
  launch_kernel(k_ct_count, g, kThreads, 0, st, g_pdl, c);
  scan_exclusive(c.ct_cnt, c.ct_off, c.P, nullptr, c.scan_tmp, c.scan_parts, st);
  launch_kernel(k_ct_scatter, g, kThreads, 0, st, g_pdl, c);
  launch_kernel(k_ct_sort, (c.P + kThreads - 1) / kThreads, kThreads, 0, st, g_pdl, c);
}

// Broad + narrow phase on the pill arrays already in `c` (pill, pill_rod/el/group/self/id).
// prefilter=0 keeps every allowed pair (the standalone broad_phase contract); with do_narrow=0
// the (unordered) candidates are left in cand_i/cand_j, scalars[SC_NCAND].
cudaEvent_t g_broad_mark = nullptr;

// The broad phase's per-call resets, one fill launch.
bool g_broad_resets_done = false;
bool g_pills_built = false;

void broad_reset_list(const Collide& c, int do_narrow, FillList& f) {
  f.add(c.maxr_bits, 2, 0);
  if (c.pill_scene) f.add(c.scene_maxr, 2ll * c.n_scenes, 0);
  f.add(c.table, c.T, -1);
  f.add(c.cell_count, c.T, 0);
  f.add(c.cell_cursor, c.T, 0);
  f.add(c.scalars + SC_BROAD, 1, 0);
  f.add(c.scalars + SC_NCAND_RAW, 1, 0);
  f.add(c.scalars + SC_NCT_RAW, 1, 0);
  if (do_narrow) f.add(c.scalars + SC_NCAND2, 1, 0);  // k_seg_filter's counter
}

void launch_broad_resets(Collide& c, int do_narrow, cudaStream_t st) {
  FillList f;
  broad_reset_list(c, do_narrow, f);
  launch_fill(f, st);
}

bool launch_broad_narrow(Collide& c, int substep, unsigned long long* err, int prefilter, int do_narrow,
                         int split_warm, int store_d, cudaStream_t st, StepAccum* fuse_acc, bool prepared) {
  (void)store_d;
  const int P = c.P;
  const int b = (P + kThreads - 1) / kThreads;
  if (!prepared) launch_broad_resets(c, do_narrow, st);  // else: resets, bounds and max radius done by the caller
  bool fused_seg = false;
  if (P > 0) {
    if (!prepared) launch_kernel(k_bounds, b, kThreads, 0, st, g_pdl, c, substep, err);
    launch_kernel(k_insert, b, kThreads, 0, st, g_pdl, c);
  }
  scan_exclusive(c.cell_count, c.cell_start, c.T, nullptr, c.scan_tmp, c.scan_parts, st);
  if (P > 0) {
    launch_kernel(k_scatter, b, kThreads, 0, st, g_pdl, c);
    // VROD_BROAD_CELL_MIN overrides the switch-over size (tests run small worlds down both paths)
    const char* env = std::getenv("VROD_BROAD_CELL_MIN");
    const int cell_min = env ? std::atoi(env) : kCellPathMinPills;
    if (P < cell_min) {  // small worlds: one warp per pill, a single launch
      fused_seg = do_narrow && prefilter;
      launch_kernel(k_pairs_warp, (P + kPairWarps - 1) / kPairWarps, 32 * kPairWarps, 0, st, g_pdl, c, prefilter,
                    c.scalars + SC_BROAD, c.scalars + SC_NCAND_RAW, c.cand_i, c.cand_j);
    } else {  // large worlds: one warp per non-empty cell, neighbourhood loads shared by its pills
      scan_exclusive(c.rep_flag, c.rep_pos, P, nullptr, c.scan_tmp, c.scan_parts, st);
      launch_kernel(k_cell_list, (P + 127) / 128, 128, 0, st, g_pdl, c);
      launch_kernel(k_pairs_cell, std::min((P + kCellWarps - 1) / kCellWarps, 148 * 16), 32 * kCellWarps, 0, st,
                    g_pdl, c, prefilter, c.scalars + SC_BROAD, c.scalars + SC_NCAND_RAW);
    }
  }
  if (g_broad_mark) cudaEventRecord(g_broad_mark, st);  // end of the broad phase (phase timing)
  if (fused_seg) {  // k_narrow_append clamps the count and runs the exact segment test itself
    launch_kernel(k_narrow_append<true>, narrow_grid(c.cand_cap), kNarrowThreads, 0, st, g_pdl, c, split_warm,
                  int(SC_NCAND_RAW), 1);
  } else {
    launch_kernel(k_clamp_raw, 1, 1, 0, st, g_pdl, c.scalars, SC_NCAND_RAW, SC_NCAND, c.cand_cap, 1);
    if (!do_narrow) return false;
    launch_kernel(k_seg_filter, grid_for(c.cand_cap), kThreads, 0, st, g_pdl, c);
    launch_kernel(k_narrow_append<false>, grid_for(c.cand_cap), kThreads, 0, st, g_pdl, c, split_warm, -1, 0);
  }
  // small worlds without kinematic pills: the ordering kernel clamps the count and builds the warm list
  const bool fused = fuse_acc && c.order_smem_cap >= 0 && !split_warm;
  if (!fused) launch_kernel(k_clamp_raw, 1, 1, 0, st, g_pdl, c.scalars, SC_NCT_RAW, SC_NCT, c.contact_cap, 2);
  launch_order_contacts(c, st, fused ? fuse_acc : nullptr);
  return fused;
}

// Standalone broad_phase: every allowed pair, in the reference's (i, j) order.
void launch_broad_ordered(Collide& c, unsigned long long* err, cudaStream_t st) {
  launch_broad_narrow(c, 0, err, 0, 0, 0, 0, st, nullptr, false);
  launch_kernel(k_cand_to_raw, grid_for(c.cand_cap), kThreads, 0, st, g_pdl, c);
  launch_order_contacts(c, st, nullptr);
}

void launch_collide(const World& w, Collide& c, const double* anim, const AnimLayout& al, int substep,
                    unsigned long long* err, StepAccum* acc, int possible, cudaStream_t st) {
  const int nb = (std::max(w.V, al.n_kin) + kThreads - 1) / kThreads;
  // single-scene worlds: the broad phase's resets first, then the pills with their bounding spheres
  const bool fused_bounds = possible && !c.pill_scene;
  // (g_broad_resets_done: the step prologue already did them, see Solver::record_step)
  if (fused_bounds && !g_broad_resets_done) launch_broad_resets(c, 1, st);
  g_broad_resets_done = false;
  // (g_pills_built: the prediction launch built the pills and bounds, launch_animate_predict)
  if (!(g_pills_built && fused_bounds))
    launch_kernel(k_build_pills, nb, kThreads, 0, st, g_pdl, w, c, anim, al, fused_bounds ? 1 : 0, substep, err);
  g_pills_built = false;
  if (!possible) {  // no pair can pass pair_allowed: only broad_phase's finiteness check remains
    if (c.P >= 2) launch_kernel(k_bounds, (c.P + kThreads - 1) / kThreads, kThreads, 0, st, g_pdl, c, substep, err);
    return;
  }
  const int split = w.K > 0 ? 1 : 0;
  if (launch_broad_narrow(c, substep, err, 1, 1, split, 0, st, acc, fused_bounds)) return;  // warm list built by the ordering
  const int g = grid_for(c.contact_cap);
  if (split) {
    launch_kernel(k_warm_flags, g, kThreads, 0, st, g_pdl, c);
    scan_exclusive(c.rk_flag, c.rk_pos, c.contact_cap, c.scalars + SC_NCT, c.scan_tmp, c.scan_parts, st);
  }
  launch_kernel(k_warm_build, g, kThreads, 0, st, g_pdl, c, split);
  launch_kernel(k_warm_counts, 1, 1, 0, st, g_pdl, c, split, acc);
}

void launch_halfplanes(const World& w, Collide& c, cudaStream_t st) {
  if (c.n_planes == 0) return;
  const long long n = static_cast<long long>(c.n_planes) * w.V;
  const int g = grid_for(n);
  launch_kernel(k_hp_flags, g, kThreads, 0, st, g_pdl, w, c);
  scan_exclusive(c.hp_flag, c.hp_pos, n, nullptr, c.scan_tmp, c.scan_parts, st);
  launch_kernel(k_hp_compact, g, kThreads, 0, st, g_pdl, w, c);
}

void launch_pill_project(long long n, const double* x, const double* pills, double* t, double* d, uint8_t* deg,
                         cudaStream_t st) {
  if (n <= 0) return;
  launch_kernel(k_pill_project, grid_for(n), kThreads, 0, st, g_pdl, n, x, reinterpret_cast<const PillAoS*>(pills), t, d, deg);
}

void launch_deepest(long long n, const double* a, const double* b, int iters, const double* warm, double* alpha,
                    double* beta, double* dist, cudaStream_t st) {
  if (n <= 0) return;
  launch_kernel(k_deepest, grid_for(n), kThreads, 0, st, g_pdl, n, reinterpret_cast<const PillAoS*>(a), reinterpret_cast<const PillAoS*>(b), iters, warm, alpha, beta, dist);
}

}  // namespace vdev
