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
#include "ext.cuh"
#include "kernels.cuh"
#include "vmath.cuh"

namespace vdev {

using namespace vm;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double F(const double* a, int f, int vpad, int i) {
  return a[static_cast<long long>(f) * vpad + i];
}

__device__ __forceinline__ V3 ldc(const double* X, int vp, int v) { return V3{F(X, CX, vp, v), F(X, CY, vp, v), F(X, CZ, vp, v)}; }

// ---- external blocks ----------------------------------------------------------------------

// resolve with the pill's first slot known (v = pill + rod, or -1 for a kinematic pill)
__device__ __forceinline__ ExtGeom resolve_at(const World& w, const Collide& c, const double* X, int pill, int v) {
  ExtGeom g;
  if (v >= 0) {
    const int vp = w.vpad;
    g.c0 = ldc(X, vp, v);
    g.c1 = ldc(X, vp, v + 1);
    g.rb0 = F(w.vstat, RBAR, vp, v);
    g.rb1 = F(w.vstat, RBAR, vp, v + 1);
    g.r0 = F(X, S, vp, v) * g.rb0;
    g.r1 = F(X, S, vp, v + 1) * g.rb1;
    g.v0 = v;
  } else {
    g.c0 = V3{c.pill[8ll * pill], c.pill[8ll * pill + 1], c.pill[8ll * pill + 2]};
    g.c1 = V3{c.pill[8ll * pill + 3], c.pill[8ll * pill + 4], c.pill[8ll * pill + 5]};
    g.r0 = c.pill[8ll * pill + 6];
    g.r1 = c.pill[8ll * pill + 7];
    g.rb0 = g.rb1 = 0.0;
    g.v0 = -1;
  }
  return g;
}
__device__ __forceinline__ ExtGeom resolve(const World& w, const Collide& c, const double* X, int pill) {
  const int rod = c.pill_rod[pill];
  return resolve_at(w, c, X, pill, rod >= 0 ? pill + rod : -1);
}

// Residual of an external block (contact / half-plane only), for the end-of-step penetration.
// The endpoints' first slots come from ct_va / ct_vb (stored by the incidence setup); xrec
// (nullable): the slot records, when they hold X's centers and scales (not in classic mode,
// whose post-step scales change X after the last sweep).
__device__ double ext_residual(const World& w, const Collide& c, const double* X, const double* xrec, int b, int npins,
                               int nct) {
  const int vp = w.vpad;
  if (b < npins + nct) {
    const int k = b - npins;
    ExtGeom A, B;
    if (xrec) {
      double ic[2], is[2];
      A = resolve_rec(xrec, c, c.ct_a[k], c.ct_va[k], ic, is);
      B = resolve_rec(xrec, c, c.ct_b[k], c.ct_vb[k], ic, is);
    } else {
      A = resolve_at(w, c, X, c.ct_a[k], c.ct_va[k]);
      B = resolve_at(w, c, X, c.ct_b[k], c.ct_vb[k]);
    }
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

__global__ void __launch_bounds__(256, 4) k_ext_solve(World w, Collide c, const double* __restrict__ X,
                                                     SweepParams sp, int* singular, unsigned long long* err) {
  if (sp.pdl) {
    pdl_wait();
    pdl_trigger();
  }
  const int elastic_blocks = sp.elastic_blocks;
  const int npins = sp.n_pins;
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  int nsing = 0;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    const long long ls = c.ext_cap;
    auto sing = [&]() {  // singular block (counted; per scene in a batch's last sweep)
      ++nsing;
      if (sp.scene_singular) atomicAdd(&sp.scene_singular[ext_scene(w, c, b, npins, nct)], 1);
    };
    // the block's record (32 B, coalesced by block): the per-launch sweeps' gathers form every
    // endpoint's correction from it (Collide::ext_rec)
    const ExtResult r = ext_block(w, c, X, w.xrec, c.ext_lam, ls, b, sp, [](int, int, double, double, double, double) {},
                                  nullptr, nct);
    double2* rec = reinterpret_cast<double2*>(c.ext_rec + 4ll * b);
    rec[0] = make_double2(r.rec[0], r.rec[1]);
    rec[1] = make_double2(r.rec[2], r.rec[3]);
    for (int d = 0; d < r.nlam; ++d) c.ext_lam[d * ls + b] = r.lam[d];
    if (r.singular) sing();
    if (r.bad)
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
  pdl_wait();
  pdl_trigger();
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    int slots[4];
    const int ne = ext_endpoints(c, b, npins, nct, slots);
    for (int e = 0; e < ne; ++e)
      if (slots[e] >= 0) atomicAdd(&c.ext_cnt[slots[e]], 1);
    if (b >= npins && b < npins + nct) {
      c.ct_va[b - npins] = slots[0];
      c.ct_vb[b - npins] = slots[2];
    }
    c.ext_lam[b] = 0.0;  // SoA, stride ext_cap
    c.ext_lam[c.ext_cap + b] = 0.0;
    c.ext_lam[2 * c.ext_cap + b] = 0.0;
  }
}
__global__ void k_ext_fill(Collide c, int npins) {
  pdl_wait();
  pdl_trigger();
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    int slots[4];
    int ne;
    if (b >= npins && b < npins + nct) {  // a contact's endpoint slots, as k_ext_count stored them
      const int va = c.ct_va[b - npins], vb = c.ct_vb[b - npins];
      slots[0] = va;
      slots[1] = va >= 0 ? va + 1 : -1;
      slots[2] = vb;
      slots[3] = vb >= 0 ? vb + 1 : -1;
      ne = vb >= 0 ? 4 : 2;
    } else {
      ne = ext_endpoints(c, b, npins, nct, slots);
    }
    for (int e = 0; e < ne; ++e) {
      if (slots[e] < 0) continue;
      const int pos = c.ext_off[slots[e]] + atomicAdd(&c.ext_cur[slots[e]], 1);
      c.ext_items[pos] = (b << 2) | e;
    }
  }
}
// The frozen alpha / beta an incidence entry's gather scales its contact's correction by.
__device__ __forceinline__ double entry_ab(const Collide& c, int key, int npins, int nct) {
  const int k = (key >> 2) - npins;
  return k >= 0 && k < nct ? ((key & 3) < 2 ? c.ct_alpha[k] : c.ct_beta[k]) : 0.0;
}

// Orders each slot's incidence entries by (block, endpoint): one warp per slot; up to 32 entries
// are ranked in registers (keys are distinct), longer lists fall back to an insertion sort. Each
// entry's alpha / beta is stored beside it (ext_ab), so the sweeps' gathers read it contiguously.
// A slot's list, whole warp: ranked in registers up to 32 entries (keys are distinct), longer
// lists by an insertion sort on lane 0.
__device__ __forceinline__ void ext_sort_slot_warp(const Collide& c, int s0, int n, int npins, int nct, int lane) {
  if (n <= 32) {
    const int key = lane < n ? c.ext_items[s0 + lane] : 0x7fffffff;
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += __shfl_sync(0xffffffffu, key, j) < key ? 1 : 0;
    __syncwarp();
    if (lane < n) {
      c.ext_items[s0 + rank] = key;
      c.ext_pos[key] = s0 + rank;
      c.ext_ab[s0 + rank] = entry_ab(c, key, npins, nct);
    }
  } else if (lane == 0) {
    const int s1 = s0 + n;
    for (int a = s0 + 1; a < s1; ++a) {  // insertion sort: block order, then endpoint
      const int key = c.ext_items[a];
      int b = a - 1;
      while (b >= s0 && c.ext_items[b] > key) {
        c.ext_items[b + 1] = c.ext_items[b];
        --b;
      }
      c.ext_items[b + 1] = key;
    }
    for (int a = s0; a < s1; ++a) {
      c.ext_pos[c.ext_items[a]] = a;
      c.ext_ab[a] = entry_ab(c, c.ext_items[a], npins, nct);
    }
  }
  __syncwarp();
}

#ifndef VROD_EXT_SORT_G
#define VROD_EXT_SORT_G 16  // C4: incidence setup 0.352 -> 0.334 ms per substep (8: 0.334, A/B)
#endif
// Each warp takes 32 / kG consecutive slots at a time, one kG-lane group per slot: lists of up to
// kG entries are ranked inside their group, longer ones afterwards by the whole warp.
__global__ void k_ext_sort(Collide c, int V, int npins) {
  pdl_wait();
  pdl_trigger();
  constexpr int kG = VROD_EXT_SORT_G, kPer = 32 / kG;
  const int nct = c.scalars[SC_NCT];
  const int lane = threadIdx.x & 31, sub = lane / kG, gl = lane % kG;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int v0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kPer; v0 < V; v0 += warps * kPer) {
    if (kG == 32) {
      const int s0 = c.ext_off[v0], n = c.ext_off[v0 + 1] - s0;
      if (n > 0) ext_sort_slot_warp(c, s0, n, npins, nct, lane);
      continue;
    }
    const int v = v0 + sub;
    int s0 = 0, n = 0;
    if (v < V) {
      s0 = c.ext_off[v];
      n = c.ext_off[v + 1] - s0;
    }
    const bool small = n <= kG;
    const int key = small && gl < n ? c.ext_items[s0 + gl] : 0x7fffffff;
    int rank = 0;
#pragma unroll
    for (int j = 0; j < kG; ++j) rank += __shfl_sync(0xffffffffu, key, sub * kG + j) < key ? 1 : 0;
    __syncwarp();
    if (small && gl < n) {
      c.ext_items[s0 + rank] = key;
      c.ext_pos[key] = s0 + rank;
      c.ext_ab[s0 + rank] = entry_ab(c, key, npins, nct);
    }
    unsigned big = __ballot_sync(0xffffffffu, !small && gl == 0);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int bs0 = __shfl_sync(0xffffffffu, s0, src), bn = __shfl_sync(0xffffffffu, n, src);
      ext_sort_slot_warp(c, bs0, bn, npins, nct, lane);
    }
  }
}

// Small worlds whose slot counters fit in shared memory (V <= kExtSmemSlots): the same setup as
// k_ext_setup_small, with the per-slot counts, offsets and cursors — and the entries, when they
// fit — in shared memory, so each phase costs shared-memory atomics and one block barrier instead
// of a global-memory round trip; ext_off / ext_items / ext_pos / ext_ab are written once at the end.
constexpr int kExtSmemThreads = 1024;
constexpr int kExtSmemSlots = 12288;
constexpr int kExtSmemItems = 8192;
unsigned ext_smem_bytes(int V) { return static_cast<unsigned>((2 * (V + 1) + kExtSmemItems) * sizeof(int)); }
__global__ void __launch_bounds__(kExtSmemThreads) k_ext_setup_smem(Collide c, int V, int npins) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ int s_ext[];
  int* s_off = s_ext;              // V + 1: counts, then exclusive offsets
  int* s_cur = s_ext + V + 1;      // V + 1: fill cursors
  int* s_items = s_cur + V + 1;    // kExtSmemItems
  __shared__ int ws[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int v = tid; v <= V; v += kExtSmemThreads) {
    s_off[v] = 0;
    s_cur[v] = 0;
  }
  __syncthreads();
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  for (int b = tid; b < n; b += kExtSmemThreads) {  // k_ext_count
    int slots[4];
    const int ne = ext_endpoints(c, b, npins, nct, slots);
    for (int e = 0; e < ne; ++e)
      if (slots[e] >= 0) atomicAdd(&s_off[slots[e]], 1);
    if (b >= npins && b < npins + nct) {
      c.ct_va[b - npins] = slots[0];
      c.ct_vb[b - npins] = slots[2];
    }
    c.ext_lam[b] = 0.0;
    c.ext_lam[c.ext_cap + b] = 0.0;
    c.ext_lam[2 * c.ext_cap + b] = 0.0;
  }
  __syncthreads();
  int carry = 0;  // exclusive scan in place, s_off[0, V) -> s_off[0, V]
  for (int b0 = 0; b0 < V; b0 += kExtSmemThreads) {
    const int x = b0 + tid < V ? s_off[b0 + tid] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) ws[wid] = incl;
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
    if (b0 + tid < V) s_off[b0 + tid] = carry + (wid ? ws[wid - 1] : 0) + incl - x;
    carry += ws[31];
    __syncthreads();
  }
  if (tid == 0) s_off[V] = carry;
  __syncthreads();
  const int total = s_off[V];
  for (int v = tid; v <= V; v += kExtSmemThreads) c.ext_off[v] = s_off[v];
  int* items = total <= kExtSmemItems ? s_items : c.ext_items;  // entries in shared memory when they fit
  for (int b = tid; b < n; b += kExtSmemThreads) {  // k_ext_fill
    int slots[4];
    const int ne = ext_endpoints(c, b, npins, nct, slots);
    for (int e = 0; e < ne; ++e) {
      if (slots[e] < 0) continue;
      items[s_off[slots[e]] + atomicAdd(&s_cur[slots[e]], 1)] = (b << 2) | e;
    }
  }
  __syncthreads();
  // k_ext_sort: warps over 32 consecutive slots at a time, ranking the busy slots' entries in
  // place (no global memory on this loop's path) ...
  for (int v0 = 32 * wid; v0 < V; v0 += kExtSmemThreads) {
    const int vl = v0 + lane;
    const int ml = vl < V ? s_off[vl + 1] - s_off[vl] : 0;
    unsigned busy = __ballot_sync(0xffffffffu, ml > 0);
    while (busy) {
      const int src = __ffs(busy) - 1;
      busy &= busy - 1;
      const int s0 = s_off[v0 + src], m = __shfl_sync(0xffffffffu, ml, src);
      if (m <= 32) {
        const int key = lane < m ? items[s0 + lane] : 0x7fffffff;
        int rank = 0;
        for (int j = 0; j < m; ++j) rank += __shfl_sync(0xffffffffu, key, j) < key ? 1 : 0;
        if (lane < m) items[s0 + rank] = key;
      } else {
        __syncwarp();
        if (lane == 0) {  // insertion sort in place
          for (int a = s0 + 1; a < s0 + m; ++a) {
            const int key = items[a];
            int b = a - 1;
            while (b >= s0 && items[b] > key) {
              items[b + 1] = items[b];
              --b;
            }
            items[b + 1] = key;
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // ... then every entry's outputs in one parallel pass (the alpha / beta loads all in flight)
  for (int q = tid; q < total; q += kExtSmemThreads) {
    const int key = items[q];
    c.ext_items[q] = key;
    c.ext_pos[key] = q;
    c.ext_ab[q] = entry_ab(c, key, npins, nct);
  }
}

// Small worlds: the whole external-block incidence setup (k_ext_count, the scan, k_ext_fill,
// k_ext_sort) in ONE CTA of 1024 threads, phase by phase with block barriers — same entries,
// same order, one launch instead of five.
constexpr int kExtSetupThreads = 1024;
__global__ void __launch_bounds__(kExtSetupThreads) k_ext_setup_small(Collide c, int V, int npins) {
  pdl_wait();
  pdl_trigger();
  __shared__ int ws[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int v = tid; v <= V; v += kExtSetupThreads) {
    c.ext_cnt[v] = 0;
    if (v < V) c.ext_cur[v] = 0;
  }
  __syncthreads();
  const int nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  for (int b = tid; b < n; b += kExtSetupThreads) {  // k_ext_count
    int slots[4];
    const int ne = ext_endpoints(c, b, npins, nct, slots);
    for (int e = 0; e < ne; ++e)
      if (slots[e] >= 0) atomicAdd(&c.ext_cnt[slots[e]], 1);
    if (b >= npins && b < npins + nct) {
      c.ct_va[b - npins] = slots[0];
      c.ct_vb[b - npins] = slots[2];
    }
    c.ext_lam[b] = 0.0;
    c.ext_lam[c.ext_cap + b] = 0.0;
    c.ext_lam[2 * c.ext_cap + b] = 0.0;
  }
  __syncthreads();
  int carry = 0;  // exclusive scan ext_cnt[0, V) -> ext_off[0, V]
  for (int b0 = 0; b0 < V; b0 += kExtSetupThreads) {
    const int x = b0 + tid < V ? c.ext_cnt[b0 + tid] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) ws[wid] = incl;
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
    if (b0 + tid < V) c.ext_off[b0 + tid] = carry + (wid ? ws[wid - 1] : 0) + incl - x;
    carry += ws[31];
    __syncthreads();
  }
  if (tid == 0) c.ext_off[V] = carry;
  __syncthreads();
  for (int b = tid; b < n; b += kExtSetupThreads) {  // k_ext_fill
    int slots[4];
    const int ne = ext_endpoints(c, b, npins, nct, slots);
    for (int e = 0; e < ne; ++e) {
      if (slots[e] < 0) continue;
      const int pos = c.ext_off[slots[e]] + atomicAdd(&c.ext_cur[slots[e]], 1);
      c.ext_items[pos] = (b << 2) | e;
    }
  }
  __syncthreads();
  // k_ext_sort: each warp takes 32 consecutive slots at a time, finds the ones with entries with
  // one ballot (most slots have none), and sorts just those
  for (int v0 = 32 * wid; v0 < V; v0 += kExtSetupThreads) {
    const int vl = v0 + lane;
    const int ml = vl < V ? c.ext_off[vl + 1] - c.ext_off[vl] : 0;
    unsigned busy = __ballot_sync(0xffffffffu, ml > 0);
    while (busy) {
      const int src = __ffs(busy) - 1;
      busy &= busy - 1;
      const int v = v0 + src;
      const int s0 = c.ext_off[v], m = __shfl_sync(0xffffffffu, ml, src), s1 = s0 + m;
      if (m <= 32) {
        const int key = lane < m ? c.ext_items[s0 + lane] : 0x7fffffff;
        int rank = 0;
        for (int j = 0; j < m; ++j) rank += __shfl_sync(0xffffffffu, key, j) < key ? 1 : 0;
        __syncwarp();
        if (lane < m) {
          c.ext_items[s0 + rank] = key;
          c.ext_pos[key] = s0 + rank;
          c.ext_ab[s0 + rank] = entry_ab(c, key, npins, nct);
        }
        __syncwarp();
      } else {
        if (lane == 0) {
          for (int a = s0 + 1; a < s1; ++a) {
            const int key = c.ext_items[a];
            int b = a - 1;
            while (b >= s0 && c.ext_items[b] > key) {
              c.ext_items[b + 1] = c.ext_items[b];
              --b;
            }
            c.ext_items[b + 1] = key;
          }
          for (int a = s0; a < s1; ++a) {
            c.ext_pos[c.ext_items[a]] = a;
            c.ext_ab[a] = entry_ab(c, c.ext_items[a], npins, nct);
          }
        }
        __syncwarp();
      }
    }
  }
}

// ---- end-of-substep report (elastic_residual_norms, constraints.cpp:558-596, and
//      end_of_step_penetration, solver.cpp:291-299) ----------------------------------------

constexpr int kRepThreads = 256;

// Residual terms of the elastic blocks owned by slot v (element v, interior vertex v):
// acc[kind] += length weight * |W|^2, acc[8 + kind] += length weight.
__device__ __forceinline__ void slot_residual_terms(const World& w, const double* __restrict__ X, int classic, int v,
                                                    double (&acc)[16]) {
  {
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
}

// eval_constraint(...).W of every elastic block (constraints.cpp:106-214), written at the block's
// index in the reference's order: rod block base + element pass (k * ne + rank) or vertex pass
// (m * ne + (k - 1) * nv + rank). Same formulas as slot_residual_terms.
__global__ void k_block_residuals(World w, const double* __restrict__ X, int classic, double* __restrict__ out) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < w.V; v += gridDim.x * blockDim.x) {
    const int vp = w.vpad;
    const int k = w.slot_loc[v], m = w.slot_m[v], r = w.slot_rod[v];
    const int ek = w.rod_ekinds[r], vk = w.rod_vkinds[r];
    const int ne = __popc(ek), nv = __popc(vk);
    const long long base = w.rod_block_base[r];
    auto put = [&](long long b, double x, double y, double z) {
      out[3 * b] = x;
      out[3 * b + 1] = y;
      out[3 * b + 2] = z;
    };
    if (k < m) {
      const V3 c0 = ldc(X, vp, v), c1 = ldc(X, vp, v + 1);
      const double s0 = F(X, S, vp, v), s1 = F(X, S, vp, v + 1);
      const double sb0 = F(w.vstat, SBAR, vp, v), sb1 = F(w.vstat, SBAR, vp, v + 1);
      const double l = F(w.estat, LEN, vp, v), l0 = F(w.estat, LEN0, vp, v), tbar = F(w.estat, TDOT, vp, v);
      const M3 R = qmat(Q4{F(X, QW, vp, v), F(X, QX, vp, v), F(X, QY, vp, v), F(X, QZ, vp, v)});
      const V3 wv = col(R, 2);
      const long long b0 = base + static_cast<long long>(k) * ne;
      if (ek & EK_SZ) {
        const V3 W = (c1 - c0) / l - tbar * wv;
        put(b0 + __popc(ek & (EK_SZ - 1)), W.x, W.y, W.z);
      }
      if (ek & EK_CS) put(b0 + __popc(ek & (EK_CS - 1)), 0.5 * (s0 + s1) - 0.5 * (sb0 + sb1), 0, 0);
      if (ek & EK_SS) put(b0 + __popc(ek & (EK_SS - 1)), (s1 - s0) / l - F(w.estat, SGRAD, vp, v), 0, 0);
      if (ek & EK_VS) {
        const double smid = 0.5 * (s0 + s1), smr = 0.5 * (sb0 + sb1);
        const V3 W = (smid * smid) * ((c1 - c0) / l0) - (smr * smr * tbar) * wv;
        put(b0 + __popc(ek & (EK_VS - 1)), W.x, W.y, W.z);
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
      const long long b0 = base + static_cast<long long>(m) * ne + static_cast<long long>(k - 1) * nv;
      if (vk & VK_BT) {
        const V3 om = (4.0 / (la + lb)) * qvec(pr);
        const double s = classic ? sbar : s0;
        const V3 W = s * om - sbar * darb;
        put(b0 + __popc(vk & (VK_BT - 1)), W.x, W.y, W.z);
      }
      if (vk & VK_SB) {
        const double sm = F(X, S, vp, v - 1), spp = F(X, S, vp, v + 1);
        put(b0 + __popc(vk & (VK_SB - 1)), ((spp - s0) / lb - (s0 - sm) / la) - F(w.estat, SLAP, vp, v - 1), 0, 0);
      }
      const double inv_len0 = 4.0 / (la0 + lb0);
      for (int cc = 0; cc < 2; ++cc) {
        const int bit = cc == 0 ? VK_VBU : VK_VBV;
        if (!(vk & bit)) continue;
        const double om = inv_len0 * (cc == 0 ? pr.x : pr.y);
        const double rest_om = (cc == 0 ? darb.x : darb.y) * (la + lb) / (la0 + lb0);
        put(b0 + __popc(vk & (bit - 1)), s0 * s0 * s0 * om - sbar * sbar * sbar * rest_om, 0, 0);
      }
    }
  }
}

// get_state's output layout, packed on the device (one D2H copy, contiguous host copies):
// centers 3V | scales V | frames 4E (wxyz) | center velocities 3V | scale velocities V |
// angular velocities 3E, in the C-ABI's global slot / compact element order (element e of slot
// v is e = v - rod(v): every rod has one more vertex than elements).
__global__ void k_pack_state(World w, const double* __restrict__ X, int E, double* __restrict__ out) {
  const int V = w.V, vp = w.vpad;
  double* c = out;
  double* s = c + 3ll * V;
  double* q = s + V;
  double* cv = q + 4ll * E;
  double* sv = cv + 3ll * V;
  double* av = sv + V;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    c[3ll * v] = F(X, CX, vp, v);
    c[3ll * v + 1] = F(X, CY, vp, v);
    c[3ll * v + 2] = F(X, CZ, vp, v);
    s[v] = F(X, S, vp, v);
    cv[3ll * v] = F(w.vel, VX, vp, v);
    cv[3ll * v + 1] = F(w.vel, VY, vp, v);
    cv[3ll * v + 2] = F(w.vel, VZ, vp, v);
    sv[v] = F(w.vel, VS, vp, v);
    if (w.slot_loc[v] < w.slot_m[v]) {
      const long long e = v - w.slot_rod[v];
      for (int f = 0; f < 4; ++f) q[4 * e + f] = F(X, QW + f, vp, v);
      for (int f = 0; f < 3; ++f) av[3 * e + f] = F(w.vel, WX + f, vp, v);
    }
  }
}

// ---- Solver::kinetic_energy / total_volume (solver.cpp:400-430, rod.cpp:178-187) on the device.
// The terms are computed in parallel; the sums run in the reference's sequential order (one
// thread, or one thread per rod for the per-rod volumes), so the results are the same bits.
// terms: 4 per slot — vertex kinetic, scale kinetic, element kinetic, element volume.
__global__ void k_energy_terms(World w, const double* __restrict__ X, const double* __restrict__ cw,
                               const double* __restrict__ sw, double* __restrict__ terms) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < w.V; v += gridDim.x * blockDim.x) {
    const int vp = w.vpad;
    const V3 u{F(w.vel, VX, vp, v), F(w.vel, VY, vp, v), F(w.vel, VZ, vp, v)};
    const double svel = F(w.vel, VS, vp, v);
    terms[4ll * v] = 0.5 * cw[v] * sqnorm(u);
    terms[4ll * v + 1] = 0.5 * sw[v] * svel * svel;
    if (w.slot_loc[v] < w.slot_m[v]) {
      const double base = F(w.estat, TWB, vp, v);
      const V3 tw{0.25 * base, 0.25 * base, 0.5 * base};
      const V3 om{F(w.vel, WX, vp, v), F(w.vel, WY, vp, v), F(w.vel, WZ, vp, v)};
      terms[4ll * v + 2] = 0.5 * dot(om, cwmul(tw, om));
      const double s = 0.5 * (F(X, S, vp, v) + F(X, S, vp, v + 1));
      const double rr = 0.5 * (F(w.vstat, RBAR, vp, v) + F(w.vstat, RBAR, vp, v + 1));
      terms[4ll * v + 3] = kPi * (s * rr) * (s * rr) * norm(ldc(X, vp, v + 1) - ldc(X, vp, v));
    }
  }
}
// per rod: its elements' volume terms in order (rod.cpp:178-187)
__global__ void k_rod_volumes(World w, const double* __restrict__ terms, double* __restrict__ rod_vol) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < w.R; r += gridDim.x * blockDim.x) {
    const int v0 = w.rod_vbase[r], m = w.rod_n[r] - 1;
    double v = 0.0;
    for (int e = 0; e < m; ++e) v += terms[4ll * (v0 + e) + 3];
    rod_vol[r] = v;
  }
}
// one thread: kinetic energy in the reference's order (vertices, then elements), volume over rods
__global__ void k_energy_sum(World w, const double* __restrict__ terms, const double* __restrict__ cw,
                             const double* __restrict__ rod_vol, int classic, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double en = 0.0;
  for (int v = 0; v < w.V; ++v) {
    if (isinf(cw[v])) continue;  // inv_center == 0
    en += terms[4ll * v];
    if (!classic) en += terms[4ll * v + 1];
  }
  for (int v = 0; v < w.V; ++v)
    if (w.slot_loc[v] < w.slot_m[v]) en += terms[4ll * v + 2];
  double vol = 0.0;
  for (int r = 0; r < w.R; ++r) vol += rod_vol[r];
  out[0] = en;
  out[1] = vol;
}

__device__ __forceinline__ void report_partial_block(const World& w, const double* __restrict__ X, int classic,
                                                     double* partials, int blk) {
  const int v = blk * kRepThreads + threadIdx.x;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  if (v < w.V) slot_residual_terms(w, X, classic, v, acc);
  // fixed-order reduction: a shuffle tree per warp, then the warps' sums in warp order
  __shared__ double red[16][kRepThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    double x = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[q][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    double x = red[threadIdx.x][0];
    for (int k = 1; k < kRepThreads / 32; ++k) x += red[threadIdx.x][k];
    partials[16ll * blk + threadIdx.x] = x;
  }
}
__global__ void k_report_partial(World w, const double* __restrict__ X, int classic, double* partials) {
  pdl_wait();
  pdl_trigger();
  report_partial_block(w, X, classic, partials, blockIdx.x);
}

// Sums the per-CTA partials: 16 quantities x `parts`, one CTA of 256 threads, each thread a
// strided fixed subset, then a fixed tree — deterministic, no atomics.
__device__ __forceinline__ void report_final_block(const double* partials, int parts, double* out8) {
  __shared__ double red[16][kRepThreads / 16];
  const int q = threadIdx.x & 15, lane = threadIdx.x >> 4;  // 16 threads per quantity
  double acc = 0.0;
  for (int b = lane; b < parts; b += kRepThreads / 16) acc += partials[16ll * b + q];
  red[q][lane] = acc;
  __syncthreads();
  for (int s = kRepThreads / 32; s > 0; s >>= 1) {
    if (lane < s) red[q][lane] += red[q][lane + s];
    __syncthreads();
  }
  if (threadIdx.x < 8) {
    const double num = red[threadIdx.x][0], den = red[threadIdx.x + 8][0];
    out8[threadIdx.x] = den > 0 ? sqrt(num / den) : 0.0;
  }
}
__global__ void k_report_final(const double* partials, int parts, double* out8) {
  pdl_wait();
  pdl_trigger();
  report_final_block(partials, parts, out8);
}

__device__ __forceinline__ void penetration_part(const World& w, const Collide& c, const double* __restrict__ X,
                                                 const double* __restrict__ xrec, StepAccum* acc) {
  const int npins = c.n_pins;
  const int nct = c.scalars[SC_NCT];
  const int n = nct + c.scalars[SC_NHP];
  double deepest = 0.0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const double pen = -ext_residual(w, c, X, xrec, npins + q, npins, nct);
    if (pen > deepest) deepest = pen;
    if (c.pill_scene && pen > 0.0) {  // batch: per-scene max as well
      const int scene = q < nct ? c.pill_scene[c.ct_a[q]] : c.plane_scene[c.hp_plane[q - nct]];
      atomicMax(reinterpret_cast<unsigned long long*>(&c.scene_acc[scene].max_penetration),
                static_cast<unsigned long long>(__double_as_longlong(pen)));
    }
  }
  for (int o = 16; o > 0; o >>= 1) deepest = fmax(deepest, __shfl_down_sync(0xffffffffu, deepest, o));
  if ((threadIdx.x & 31) == 0 && deepest > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(&acc->max_penetration),
              static_cast<unsigned long long>(__double_as_longlong(deepest)));
}
__global__ void k_penetration(World w, Collide c, const double* __restrict__ X, StepAccum* acc) {
  pdl_wait();
  pdl_trigger();
  penetration_part(w, c, X, nullptr, acc);
}

// The end of a single-scene substep in one launch: the max penetration over the contact and
// half-plane blocks, then — in the last CTA to finish (ticket counter, reset by that CTA) — the
// residual norms from k_report_partial's partials (the same fixed-order tree as k_report_final)
// and the substep's singular count / error word (solver.cpp:335, 370-375).
// kPartials: the residual partials too (block b < parts computes partial b, k_report_partial's
// work and partition), so the whole report is one launch.
template <bool kPartials>
__global__ void k_report_tail(World w, Collide c, const double* __restrict__ X, const double* __restrict__ xrec,
                              StepAccum* acc, int do_pen,
                              double* partials, int parts, const int* singular_last, int last,
                              const unsigned long long* err, unsigned* counter, int classic) {
  pdl_wait();
  pdl_trigger();
  if (kPartials && static_cast<int>(blockIdx.x) < parts) {
    report_partial_block(w, X, classic, partials, blockIdx.x);
    if (threadIdx.x < 16) __threadfence();  // the partial, before this block's ticket
  }
  if (do_pen) penetration_part(w, c, X, xrec, acc);
  __shared__ int is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  report_final_block(partials, parts, acc->residuals);
  if (threadIdx.x == 0) {
    *counter = 0;
    acc->skipped_singular += *singular_last;
    if (last) {
      unsigned long long e = *err;
      if (c.scalars[SC_OVF]) e = err_code(0, ERR_CAPACITY, c.scalars[SC_OVF], 0);  // results invalid
      acc->error = e;
    }
  }
}

// Batch: per-scene residual norms of the scene's slot range (one CTA per scene, fixed tree),
// overwriting the previous substep's (Solver::step keeps the last substep's, solver.cpp:370).
__global__ void k_report_scene(World w, const double* __restrict__ X, int classic) {
  pdl_wait();
  pdl_trigger();
  const int sc = blockIdx.x;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int v = w.scene_vbase[sc] + threadIdx.x; v < w.scene_vbase[sc + 1]; v += kRepThreads)
    slot_residual_terms(w, X, classic, v, acc);
  __shared__ double red[kRepThreads];
  __shared__ double res[16];
  for (int q = 0; q < 16; ++q) {
    red[threadIdx.x] = acc[q];
    __syncthreads();
    for (int s = kRepThreads / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) res[q] = red[0];
    __syncthreads();
  }
  if (threadIdx.x < 8) {
    const double num = res[threadIdx.x], den = res[threadIdx.x + 8];
    w.scene_acc[sc].residuals[threadIdx.x] = den > 0 ? sqrt(num / den) : 0.0;
  }
}

// Batch: fold the last sweep's per-scene singular counts into the step totals.
__global__ void k_scene_singular(World w, int* scene_singular) {
  pdl_wait();
  pdl_trigger();
  for (int sc = blockIdx.x * blockDim.x + threadIdx.x; sc < w.n_scenes; sc += gridDim.x * blockDim.x) {
    w.scene_acc[sc].skipped_singular += scene_singular[sc];
    scene_singular[sc] = 0;
  }
}

int grid_for(long long n) {
  const long long b = (n + kThreads - 1) / kThreads;
  return static_cast<int>(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

int report_parts(int V) { return (V + kRepThreads - 1) / kRepThreads; }

void launch_ext_setup(const World& w, Collide& c, cudaStream_t st) {
  if (c.order_smem_cap >= 0 && w.V <= kExtSmemSlots && !std::getenv("VROD_EXT_SETUP_GLOBAL")) {
    static const cudaError_t attr = cudaFuncSetAttribute(k_ext_setup_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         ext_smem_bytes(kExtSmemSlots));
    (void)attr;  // a failure surfaces as a launch error
    launch_kernel(k_ext_setup_smem, 1, kExtSmemThreads, ext_smem_bytes(w.V), st, g_pdl, c, w.V, c.n_pins);
    return;
  }
  if (c.order_smem_cap >= 0 && w.V < (1 << 16)) {  // small worlds (same switch as the contact ordering)
    launch_kernel(k_ext_setup_small, 1, kExtSetupThreads, 0, st, g_pdl, c, w.V, c.n_pins);
    return;
  }
  FillList f;
  f.add(c.ext_cnt, w.V + 1, 0);
  f.add(c.ext_cur, w.V, 0);
  launch_fill(f, st);
  const int g = grid_for(c.ext_cap);
  launch_kernel(k_ext_count, g, kThreads, 0, st, g_pdl, c, c.n_pins);
  scan_exclusive(c.ext_cnt, c.ext_off, w.V, nullptr, c.scan_tmp, c.scan_parts, st);
  launch_kernel(k_ext_fill, g, kThreads, 0, st, g_pdl, c, c.n_pins);
  launch_kernel(k_ext_sort, grid_for(32ll * w.V), kThreads, 0, st, g_pdl, c, w.V, c.n_pins);
}

void launch_ext_solve(const World& w, Collide& c, const double* X, const SweepParams& sp, int* singular_counter,
                      unsigned long long* err, cudaStream_t st) {
  if (c.ext_cap > 0)
    launch_kernel(k_ext_solve, grid_for(c.ext_cap), kThreads, 0, st, sp.pdl != 0, w, c, X, sp, singular_counter, err);
}

void launch_iteration(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp,
                      int* singular_counter, unsigned long long* err, cudaStream_t st) {
  launch_ext_solve(w, c, X, sp, singular_counter, err, st);
  launch_rod_sweep(w, c, X, Y, sp, singular_counter, err, st);
}

void launch_residuals(const World& w, const double* X, int classic, double* partials, int parts, double* out8,
                      cudaStream_t st) {
  launch_kernel(k_report_partial, parts, kRepThreads, 0, st, g_pdl, w, X, classic, partials);
  launch_kernel(k_report_final, 1, kRepThreads, 0, st, g_pdl, partials, parts, out8);
}

void launch_pack_state(const World& w, const double* X, int E, double* out, cudaStream_t st) {
  launch_kernel(k_pack_state, grid_for(w.V), kThreads, 0, st, false, w, X, E, out);
}

void launch_energy(const World& w, const double* X, const double* cw, const double* sw, int classic, double* terms,
                   double* rod_vol, double* out, cudaStream_t st) {
  launch_kernel(k_energy_terms, grid_for(w.V), kThreads, 0, st, false, w, X, cw, sw, terms);
  launch_kernel(k_rod_volumes, grid_for(w.R), kThreads, 0, st, false, w, terms, rod_vol);
  launch_kernel(k_energy_sum, 1, 32, 0, st, false, w, terms, cw, rod_vol, classic, out);
}

void launch_block_residuals(const World& w, const double* X, int classic, double* out, cudaStream_t st) {
  launch_kernel(k_block_residuals, grid_for(w.V), kThreads, 0, st, false, w, X, classic, out);
}

void launch_scene_report(const World& w, const double* X, int classic, int* scene_singular, cudaStream_t st) {
  launch_kernel(k_report_scene, w.n_scenes, kRepThreads, 0, st, g_pdl, w, X, classic);
  launch_kernel(k_scene_singular, (w.n_scenes + kThreads - 1) / kThreads, kThreads, 0, st, g_pdl, w, scene_singular);
}

void launch_report_tail(const World& w, Collide& c, const double* X, const double* xrec, int classic, StepAccum* acc,
                        bool do_pen,
                        double* partials, int parts, const int* singular_last, int last, const unsigned long long* err,
                        unsigned* counter, cudaStream_t st) {
  // small worlds: the partials in the same launch (latency); large ones (C4: 0.31 vs 0.21 ms): separate
  const bool fused = parts <= 148;
  if (!fused) launch_kernel(k_report_partial, parts, kRepThreads, 0, st, g_pdl, w, X, classic, partials);
  const int g = std::max(do_pen ? grid_for(c.contact_cap + c.hp_cap) : 1, fused ? parts : 1);
  launch_kernel(fused ? k_report_tail<true> : k_report_tail<false>, g, kRepThreads, 0, st, g_pdl, w, c, X, xrec, acc,
                do_pen ? 1 : 0, partials, parts, singular_last, last, err, counter, classic);
}

void launch_penetration(const World& w, Collide& c, const double* X, StepAccum* acc, cudaStream_t st) {
  launch_kernel(k_penetration, grid_for(c.contact_cap + c.hp_cap), kThreads, 0, st, g_pdl, w, c, X, acc);
}

}  // namespace vdev
