// Pill-pill collision: rod_pills (collision.cpp:275-296), bounding spheres (:137-153), the
// uniform-grid broad phase (:184-238) and the dichotomous narrow phase (:55-135, :251-273),
// plus half-plane block generation (solver.cpp:227-249). Compiled with --fmad=false so the
// narrow phase, the cell keys and every pill geometry value match the reference bit for bit.
//
// Broad phase on the GPU: the grid is an open-addressing hash table of cell keys built with
// atomicCAS (one representative pill per cell), a count -> exclusive scan -> scatter counting
// sort of pill ids into cells, then per pill a 27-cell scan that (1) counts every allowed pair
// j > i (StepReport.broad_pairs, exactly the reference's candidate count) and (2) keeps the
// pairs whose bounding spheres overlap — the only pairs that can penetrate — sorted by j.
// Candidates are therefore in (i, j) order like the reference's pair list, and so are the
// contacts after the stream compaction of the narrow-phase hits.
#include <algorithm>
#include <cfloat>

#include "kernels.cuh"
#include "vmath.cuh"

namespace vdev {

using namespace vm;

namespace {

constexpr int kThreads = 256;

struct PillV {
  V3 c0, c1;
  double r0, r1;
};

__device__ __forceinline__ PillV load_pill(const double* __restrict__ pill, int P, int i) {
  return PillV{V3{pill[i], pill[P + i], pill[2 * P + i]}, V3{pill[3 * P + i], pill[4 * P + i], pill[5 * P + i]},
               pill[6 * P + i], pill[7 * P + i]};
}

// pill_project (collision.cpp:15-49) with the per-pill constants (axis, length, unit axis,
// cone slope) computed once per query pill: same operations on the same inputs, so the
// results are identical to evaluating them inside every call.
struct PillPrep {
  V3 c0, c1;
  double r0, r1;
  bool degenerate;
  double l;
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
  if (!q.degenerate) {
    q.j = axis / q.l;
    const double sin_t = (p.r1 - p.r0) / q.l;
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
  double t = (a + b * p.tan_t) / p.l;
  t = fmin(fmax(t, 0.0), 1.0);
  t_out = t;
  const V3 c = (1.0 - t) * p.c0 + t * p.c1;  // pill_distance_at, collision.cpp:9-13
  const double r = (1.0 - t) * p.r0 + t * p.r1;
  return norm(x - c) - r;
}
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
// deepest_penetration, collision.cpp:78-135.
__device__ void deepest(const PillV& A, const PillV& B, int iterations, double warm, double& alpha_out,
                        double& beta_out, double& dist_out) {
  const bool swapped = pill_less(B, A);
  const PillV& pa = swapped ? B : A;
  const PillPrep pb = prep_pill(swapped ? A : B);
  if (swapped && warm >= 0.0) warm = -1.0;
  double lo = 0.0, hi = 1.0;
  double best_a = 0.5, best_b = 0.0;
  double best = pair_distance(pa, pb, 0.5, best_b);
  const double delta = 1e-6;
  for (int it = 0; it < iterations; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double x1 = mid - delta, x2 = mid + delta;
    double b1 = 0.0, b2 = 0.0;
    const double f1 = pair_distance(pa, pb, x1, b1);
    const double f2 = pair_distance(pa, pb, x2, b2);
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
  const double cands[3] = {lo, hi, warm};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double cand = cands[k];
    if (cand < 0.0 || cand > 1.0) continue;
    double bc = 0.0;
    const double fc = pair_distance(pa, pb, cand, bc);
    if (fc < best) {
      best = fc;
      best_a = cand;
      best_b = bc;
    }
  }
  dist_out = best;
  if (swapped) {
    alpha_out = best_b;
    beta_out = best_a;
  } else {
    alpha_out = best_a;
    beta_out = best_b;
  }
}
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

__device__ __forceinline__ unsigned long long cell_hash(long long x, long long y, long long z) {
  unsigned long long h = static_cast<unsigned long long>(x) * 73856093ull ^
                         static_cast<unsigned long long>(y) * 19349663ull ^
                         static_cast<unsigned long long>(z) * 83492791ull;
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

// rod_pills from the predicted state + the posed kinematic pills of this substep.
__global__ void k_build_pills(World w, Collide c, const double* __restrict__ anim, AnimLayout al) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  const int P = c.P;
  if (v < w.V) {
    const int k = w.slot_loc[v], m = w.slot_m[v];
    if (k < m) {
      const int r = w.slot_rod[v];
      const int i = v - r;
      const int vp = w.vpad;
      const double* X = w.X;
      c.pill[i] = X[CX * vp + v];
      c.pill[P + i] = X[CY * vp + v];
      c.pill[2 * P + i] = X[CZ * vp + v];
      c.pill[3 * P + i] = X[CX * vp + v + 1];
      c.pill[4 * P + i] = X[CY * vp + v + 1];
      c.pill[5 * P + i] = X[CZ * vp + v + 1];
      c.pill[6 * P + i] = X[S * vp + v] * w.vstat[RBAR * vp + v];
      c.pill[7 * P + i] = X[S * vp + v + 1] * w.vstat[RBAR * vp + v + 1];
    }
  }
  if (v < al.n_kin) {
    const double* kp = anim + al.off_kin + 8 * v;
    const int i = w.E + v;
    for (int f = 0; f < 8; ++f) c.pill[f * P + i] = kp[f];
  }
}

// Bounding spheres, max radius, finiteness (broad_phase, collision.cpp:189-196).
__global__ void k_bounds(Collide c, int substep, unsigned long long* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.P) return;
  const PillV p = load_pill(c.pill, c.P, i);
  V3 ctr;
  double r;
  bounding_sphere(p, ctr, r);
  c.bsph[i] = ctr.x;
  c.bsph[c.P + i] = ctr.y;
  c.bsph[2 * c.P + i] = ctr.z;
  c.bsph[3 * c.P + i] = r;
  if (!(finite3(ctr) && isfinite(r))) {
    if (c.P >= 2) atomicMin(err, err_code(substep, ERR_BROAD, 0, i));
    return;
  }
  atomicMax(c.maxr_bits, static_cast<unsigned long long>(__double_as_longlong(r)));  // r >= 0
}

__device__ __forceinline__ double cell_inv(const Collide& c) {
  const double maxr = __longlong_as_double(static_cast<long long>(*c.maxr_bits));
  const double cell = fmax(2.0 * maxr, 1e-12);  // collision.cpp:197-198
  return 1.0 / cell;
}
__device__ __forceinline__ long long key1(double x, double inv) {
  const double f = floor(x * inv);
  return isfinite(f) ? static_cast<long long>(f) : 0;
}

__global__ void k_insert(Collide c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.P) return;
  const double inv = cell_inv(c);
  const long long kx = key1(c.bsph[i], inv), ky = key1(c.bsph[c.P + i], inv), kz = key1(c.bsph[2 * c.P + i], inv);
  c.cellkey[i] = kx;
  c.cellkey[c.P + i] = ky;
  c.cellkey[2 * c.P + i] = kz;
  __threadfence();
  const unsigned mask = static_cast<unsigned>(c.T - 1);
  unsigned h = static_cast<unsigned>(cell_hash(kx, ky, kz)) & mask;
  while (true) {
    int e = atomicCAS(&c.table[h], -1, i);
    if (e == -1) break;  // new cell, i is its representative
    const long long ex = static_cast<volatile long long*>(c.cellkey)[e];
    const long long ey = static_cast<volatile long long*>(c.cellkey)[c.P + e];
    const long long ez = static_cast<volatile long long*>(c.cellkey)[2 * c.P + e];
    if (ex == kx && ey == ky && ez == kz) break;
    h = (h + 1) & mask;
  }
  c.pill_cell[i] = static_cast<int>(h);
  atomicAdd(&c.cell_count[h], 1);
}

__global__ void k_scatter(Collide c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.P) return;
  const int h = c.pill_cell[i];
  const int pos = c.cell_start[h] + atomicAdd(&c.cell_cursor[h], 1);
  c.cell_items[pos] = i;
}

__device__ __forceinline__ int find_cell(const Collide& c, long long kx, long long ky, long long kz) {
  const unsigned mask = static_cast<unsigned>(c.T - 1);
  unsigned h = static_cast<unsigned>(cell_hash(kx, ky, kz)) & mask;
  while (true) {
    const int e = c.table[h];
    if (e < 0) return -1;
    if (c.cellkey[e] == kx && c.cellkey[c.P + e] == ky && c.cellkey[2 * c.P + e] == kz) return static_cast<int>(h);
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

template <bool kFill>
__global__ void k_candidates(Collide c, int prefilter, int* broad_total) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int broad = 0, cand = 0;
  if (i < c.P) {
    const long long kx = c.cellkey[i], ky = c.cellkey[c.P + i], kz = c.cellkey[2 * c.P + i];
    const int ri = c.pill_rod[i], gi = c.pill_group[i], ei = c.pill_el[i];
    const bool si = c.pill_self[i] != 0;
    long long base = 0;
    if (kFill) base = c.cand_off[i];
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const int h = find_cell(c, kx + dx, ky + dy, kz + dz);
          if (h < 0) continue;
          const int s0 = c.cell_start[h], s1 = c.cell_start[h + 1];
          for (int q = s0; q < s1; ++q) {
            const int j = c.cell_items[q];
            if (j <= i) continue;
            if (!pair_allowed(ri, gi, si, ei, c.pill_rod[j], c.pill_group[j], c.pill_el[j])) continue;
            ++broad;
            if (prefilter && !spheres_touch(c, i, j)) continue;
            if (kFill) {
              const long long pos = base + cand;
              if (pos < c.cand_cap) {
                c.cand_j[pos] = j;
                c.cand_i[pos] = i;
              }
            }
            ++cand;
          }
        }
    if (!kFill) c.cand_count[i] = cand;
    if (kFill) {  // insertion sort of this pill's segment by j (deterministic (i, j) order)
      const long long end = min(base + cand, c.cand_cap);
      for (long long a = base + 1; a < end; ++a) {
        const int key = c.cand_j[a];
        long long b = a - 1;
        while (b >= base && c.cand_j[b] > key) {
          c.cand_j[b + 1] = c.cand_j[b];
          --b;
        }
        c.cand_j[b + 1] = key;
      }
    }
  }
  if (!kFill && broad_total) {
    // warp-aggregate the broad-phase pair count
    for (int o = 16; o > 0; o >>= 1) broad += __shfl_down_sync(0xffffffffu, broad, o);
    if ((threadIdx.x & 31) == 0 && broad) atomicAdd(broad_total, broad);
  }
}

__global__ void k_clamp_count(const int* total, long long cap, int* out, int* ovf) {
  const int t = *total;
  if (t > cap) atomicExch(ovf, 1);
  *out = t > cap ? static_cast<int>(cap) : t;
}

__device__ __forceinline__ double warm_lookup(const unsigned long long* keys, const double* alpha, int n,
                                              unsigned long long key) {
  int lo = 0, hi = n;  // lower_bound: first inserted wins on duplicate keys
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && keys[lo] == key) ? alpha[lo] : -1.0;
}

// Narrow phase over the candidate list (find_contacts, collision.cpp:261-271).
__global__ void k_narrow(Collide c, int split_warm, int store_d) {
  const int n = c.scalars[SC_NCAND];
  const int nrr = c.scalars[SC_NRR_PREV], nrk = c.scalars[SC_NRK_PREV];
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = c.cand_i[q], j = c.cand_j[q];
    const unsigned long long key = pair_key(c.pill_id[i], c.pill_id[j]);
    double warm;
    if (!split_warm || (c.pill_rod[i] >= 0 && c.pill_rod[j] >= 0)) warm = warm_lookup(c.warm_rr_key, c.warm_rr_alpha, nrr, key);
    else warm = warm_lookup(c.warm_rk_key, c.warm_rk_alpha, nrk, key);
    double al, be, d;
    deepest(load_pill(c.pill, c.P, i), load_pill(c.pill, c.P, j), c.iters_dich, warm, al, be, d);
    c.cand_flag[q] = d < 0.0 ? 1 : 0;
    c.cand_ab[q] = al;
    c.cand_ab[c.cand_cap + q] = be;
    if (store_d) c.cand_ab[2 * c.cand_cap + q] = d;
  }
}

__global__ void k_compact_contacts(Collide c) {
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

__global__ void k_contact_count(Collide c, StepAccum* acc) {
  const int n = c.cand_pos[c.scalars[SC_NCAND]];
  if (n > c.contact_cap) atomicExch(&c.scalars[SC_OVF], 2);
  const int nc = n > c.contact_cap ? static_cast<int>(c.contact_cap) : n;
  c.scalars[SC_NCT] = nc;
  atomicAdd(&acc->contact_count, nc);
  atomicAdd(&acc->broad_pairs, c.scalars[SC_BROAD]);
  if (n > acc->max_contacts) acc->max_contacts = n;
  if (c.cand_off[c.P] > acc->max_candidates) acc->max_candidates = c.cand_off[c.P];
}

// Warm list for the next substep: (pair key, alpha) of the new contacts (solver.cpp:210-214).
// Rod-rod contacts in (i, j) order have increasing keys; contacts with a kinematic pill are
// kept in a second list, also increasing in key, so both are searchable by lower_bound.
__global__ void k_warm_flags(Collide c) {
  const int n = c.scalars[SC_NCT];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    c.rk_flag[k] = (c.pill_rod[c.ct_a[k]] < 0 || c.pill_rod[c.ct_b[k]] < 0) ? 1 : 0;
}
__global__ void k_warm_build(Collide c, int split) {
  const int n = c.scalars[SC_NCT];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const unsigned long long key = pair_key(c.pill_id[c.ct_a[k]], c.pill_id[c.ct_b[k]]);
    if (!split) {
      c.warm_rr_key[k] = key;
      c.warm_rr_alpha[k] = c.ct_alpha[k];
    } else if (c.rk_flag[k]) {
      const int p = c.rk_pos[k];
      c.warm_rk_key[p] = key;
      c.warm_rk_alpha[p] = c.ct_alpha[k];
    } else {
      const int p = k - c.rk_pos[k];
      c.warm_rr_key[p] = key;
      c.warm_rr_alpha[p] = c.ct_alpha[k];
    }
  }
}
__global__ void k_warm_counts(Collide c, int split) {
  const int n = c.scalars[SC_NCT];
  const int nrk = split ? c.rk_pos[n] : 0;
  c.scalars[SC_NRK_PREV] = nrk;
  c.scalars[SC_NRR_PREV] = n - nrk;
}

// Half-plane blocks (solver.cpp:229-249): plane-major, then global vertex order.
__global__ void k_hp_flags(World w, Collide c) {
  const long long n = static_cast<long long>(c.n_planes) * w.V;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(q / w.V);
    const int v = static_cast<int>(q - static_cast<long long>(p) * w.V);
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

}  // namespace

// Broad + narrow phase on the pill arrays already in `c` (pill, pill_rod/el/group/self/id).
// prefilter=0 keeps every allowed pair (the standalone broad_phase contract).
void launch_narrow_only(Collide& c, int split_warm, int store_d, cudaStream_t st) {
  const int g = grid_for(c.cand_cap);
  k_narrow<<<g, kThreads, 0, st>>>(c, split_warm, store_d);
  scan_exclusive(c.cand_flag, c.cand_pos, c.cand_cap, c.scalars + SC_NCAND, c.scan_tmp, c.scan_parts, st);
  k_compact_contacts<<<g, kThreads, 0, st>>>(c);
}

void launch_broad_narrow(Collide& c, int substep, unsigned long long* err, int prefilter, int do_narrow,
                         int split_warm, int store_d, cudaStream_t st) {
  const int P = c.P;
  const int b = (P + kThreads - 1) / kThreads;
  cudaMemsetAsync(c.maxr_bits, 0, sizeof(unsigned long long), st);
  cudaMemsetAsync(c.table, 0xff, sizeof(int) * c.T, st);
  cudaMemsetAsync(c.cell_count, 0, sizeof(int) * c.T, st);
  cudaMemsetAsync(c.cell_cursor, 0, sizeof(int) * c.T, st);
  cudaMemsetAsync(c.scalars + SC_BROAD, 0, sizeof(int), st);
  if (P > 0) {
    k_bounds<<<b, kThreads, 0, st>>>(c, substep, err);
    k_insert<<<b, kThreads, 0, st>>>(c);
  }
  scan_exclusive(c.cell_count, c.cell_start, c.T, nullptr, c.scan_tmp, c.scan_parts, st);
  if (P > 0) {
    k_scatter<<<b, kThreads, 0, st>>>(c);
    k_candidates<false><<<b, kThreads, 0, st>>>(c, prefilter, c.scalars + SC_BROAD);
  }
  scan_exclusive(c.cand_count, c.cand_off, P, nullptr, c.scan_tmp, c.scan_parts, st);
  if (P > 0) k_candidates<true><<<b, kThreads, 0, st>>>(c, prefilter, nullptr);
  k_clamp_count<<<1, 1, 0, st>>>(c.cand_off + P, c.cand_cap, c.scalars + SC_NCAND, c.scalars + SC_OVF);
  if (!do_narrow) return;
  launch_narrow_only(c, split_warm, store_d, st);
}

void launch_collide(const World& w, Collide& c, const double* anim, const AnimLayout& al, int substep,
                    unsigned long long* err, StepAccum* acc, int possible, cudaStream_t st) {
  const int nb = (std::max(w.V, al.n_kin) + kThreads - 1) / kThreads;
  k_build_pills<<<nb, kThreads, 0, st>>>(w, c, anim, al);
  if (!possible) {  // no pair can pass pair_allowed: only broad_phase's finiteness check remains
    if (c.P >= 2) k_bounds<<<(c.P + kThreads - 1) / kThreads, kThreads, 0, st>>>(c, substep, err);
    return;
  }
  const int split = w.K > 0 ? 1 : 0;
  launch_broad_narrow(c, substep, err, 1, 1, split, 0, st);
  k_contact_count<<<1, 1, 0, st>>>(c, acc);
  const int g = grid_for(c.contact_cap);
  if (split) {
    k_warm_flags<<<g, kThreads, 0, st>>>(c);
    scan_exclusive(c.rk_flag, c.rk_pos, c.contact_cap, c.scalars + SC_NCT, c.scan_tmp, c.scan_parts, st);
  }
  k_warm_build<<<g, kThreads, 0, st>>>(c, split);
  k_warm_counts<<<1, 1, 0, st>>>(c, split);
}

void launch_halfplanes(const World& w, Collide& c, cudaStream_t st) {
  if (c.n_planes == 0) return;
  const long long n = static_cast<long long>(c.n_planes) * w.V;
  const int g = grid_for(n);
  k_hp_flags<<<g, kThreads, 0, st>>>(w, c);
  scan_exclusive(c.hp_flag, c.hp_pos, n, nullptr, c.scan_tmp, c.scan_parts, st);
  k_hp_compact<<<g, kThreads, 0, st>>>(w, c);
}

void launch_pill_project(long long n, const double* x, const double* pills, double* t, double* d, uint8_t* deg,
                         cudaStream_t st) {
  if (n <= 0) return;
  k_pill_project<<<grid_for(n), kThreads, 0, st>>>(n, x, reinterpret_cast<const PillAoS*>(pills), t, d, deg);
}

void launch_deepest(long long n, const double* a, const double* b, int iters, const double* warm, double* alpha,
                    double* beta, double* dist, cudaStream_t st) {
  if (n <= 0) return;
  k_deepest<<<grid_for(n), kThreads, 0, st>>>(n, reinterpret_cast<const PillAoS*>(a),
                                              reinterpret_cast<const PillAoS*>(b), iters, warm, alpha, beta, dist);
}

}  // namespace vdev
