// The rod stencil of one averaged-Jacobi sweep (jacobi_sweep, constraints.cpp:491-556): every
// elastic block of every rod evaluated and solved against the snapshot X, all corrections
// gathered per DOF in the reference's block order, averaged and applied into Y.
//
// CTA = 4 warps over a tile of 64 consecutive slots (62 owned + 1 halo slot each side). The
// blocks of the tile are evaluated kind-major (eval_constraint :101-270 + solve_block
// :400-487): work item = (kind present in the tile, position), so each warp runs one block
// formula over 32 positions. Per-block results go to shared memory; then one thread per owned slot gathers —
// element pass of element k-1 then k, vertex pass of vertex k-1, k, k+1, then the external
// blocks (soft pins, contacts, half-planes) through the slot-sorted incidence list — divides
// by the number of active touching blocks, clamps the scale and renormalizes the frame
// (constraints.cpp:509-554). The shapes of all expressions follow the reference, so with
// --fmad=false the result is the reference's arithmetic bit for bit; there are no atomics on
// the data path (bitwise run-to-run determinism) and no colouring (Jacobi
// snapshot semantics, test_sweep.cpp:132-142).
#include <cstdlib>

#include "ext.cuh"
#include "kernels.cuh"
#include "shape.cuh"
#include "vmath.cuh"

namespace vdev {

using namespace vm;

namespace {

// Tile of TP computed positions start-1 .. start+TP-2 (TP-2 owned), staged slots start-2 ..
// start+TP-1. TP = 64 for large worlds; 32 when 64-wide tiles would leave SMs idle.
// Warps per CTA: 4 for 64-wide tiles; 8 for 32-wide tiles (small worlds are latency-bound:
// one item round per thread instead of two).
template <int TP>
constexpr int warps_for() { return TP == 32 ? 8 : 4; }

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }

// Per-position block results (written by the kind warps, read by the gather).
struct PosRes {
  double sz_dc0[3], sz_dc1[3], sz_dt[3];
  double cs[2], ss[2];
  double vs_dc0[3], vs_dc1[3], vs_ds[2], vs_dt[3];
  double bt_ds, bt_dta[3], bt_dtb[3];
  double sb[3];  // ds_{j-1}, ds_j, ds_{j+1}
  double vb_ds[2], vb_dta[2][3], vb_dtb[2][3];
  double pad;  // 49-double stride: lane-consecutive records fall in distinct banks
};
enum : int { A_SZ = 0, A_CS, A_SS, A_VS, A_BT, A_SB, A_VBU, A_VBV, kKinds };

// Staged fields (rows of Tile::st), one column per slot start-2 .. start+63.
enum StageRow : int {
  T_CX = 0, T_CY, T_CZ, T_S, T_QW, T_QX, T_QY, T_QZ,  // snapshot X
  T_SBAR, T_IC, T_IS,                                  // static vertex fields
  T_ITX, T_ITY, T_ITZ,                                 // inverse theta weights
  T_LEN, T_LEN0, T_TDOT, T_SGRAD, T_SLAP, T_DARBX, T_DARBY, T_DARBZ,
  T_KSZ, T_KCS, T_KSS, T_KVS, T_KBT0, T_KBT1, T_KBT2, T_KSB, T_KVB,
  T_LAM,                                               // + LamField: multipliers before the sweep
  kStageRows = T_LAM + kLamFields
};
constexpr int kKindSZ = 1 << A_SZ, kKindCS = 1 << A_CS, kKindSS = 1 << A_SS, kKindVS = 1 << A_VS,
              kKindBT = 1 << A_BT, kKindSB = 1 << A_SB, kKindVBU = 1 << A_VBU, kKindVBV = 1 << A_VBV;
constexpr int kKindVB = kKindVBU | kKindVBV;
constexpr int kAllKinds = 0xff;

// Per staged row: which kinds read it (rows nobody in the tile needs are not loaded), and where
// it comes from (array: 0 X, 1 vertex statics, 2 element statics, 3 lambda_in; field index).
constexpr int kNeedSBAR = kKindCS | kKindVS | kKindBT | kKindSB | kKindVB;
constexpr int kNeedITXY = kKindSZ | kKindVS | kKindBT | kKindVB;
constexpr int kNeedLEN = kKindSZ | kKindSS | kKindBT | kKindSB | kKindVB;
__constant__ uint8_t kRowNeed[kStageRows] = {
    kAllKinds, kAllKinds, kAllKinds, kAllKinds, kAllKinds, kAllKinds, kAllKinds, kAllKinds,  // X
    kNeedSBAR, kAllKinds, kAllKinds,                                                      // SBAR IC IS
    kNeedITXY, kNeedITXY, kKindBT | kKindVB,                                              // IT xyz
    kNeedLEN, kKindVS | kKindVB, kKindSZ | kKindVS, kKindSS, kKindSB,                       // LEN LEN0 TDOT SGRAD SLAP
    kKindBT | kKindVB, kKindBT | kKindVB, kKindBT,                                         // DARB xyz
    kKindSZ, kKindCS, kKindSS, kKindVS, kKindBT, 0, kKindBT, kKindSB, kKindVB,  // inverse stiffnesses (KBT1 == KBT0)
    kKindSZ, kKindSZ, kKindSZ, kKindCS, kKindSS, kKindVS, kKindVS, kKindVS,                 // lambda element pass
    kKindBT, kKindBT, kKindBT, kKindSB, kKindVBU, kKindVBV};                                // lambda vertex pass
__constant__ uint8_t kRowArr[kStageRows] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2,
                                            2, 2, 2, 2, 2, 2, 2, 2, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3};
__constant__ uint8_t kRowField[kStageRows] = {
    CX, CY, CZ, S, QW, QX, QY, QZ, SBAR, IC, IS, ITX, ITY, ITZ, LEN, LEN0, TDOT, SGRAD, SLAP, DARBX, DARBY, DARBZ,
    KSZ, KCS, KSS, KVS, KBT0, KBT1, KBT2, KSB, KVB,
    L_SZ0, L_SZ1, L_SZ2, L_CS, L_SS, L_VS0, L_VS1, L_VS2, L_BT0, L_BT1, L_BT2, L_SB, L_VBU, L_VBV};
static_assert(kStageRows == 45, "row tables");

constexpr int kTileEntries = 160;

template <int TP>
struct Tile {
  static constexpr int kTilePos = TP, kTileStage = TP + 2;
  double st[kStageRows][kTileStage];
  PosRes res[kTilePos];
  int loc[kTilePos], m[kTilePos], kinds[kTilePos], bbase[kTilePos];
  unsigned wmask[(kTilePos + 31) / 32];  // OR of the kinds present, per 32 positions
  int klist[kKinds];              // the kinds present, ascending
  uint8_t act[kKinds][kTilePos];
  alignas(8) unsigned long long bar;  // mbarrier of the bulk (TMA) staging
};

// The persistent kernel's tile: incidence offsets of the owned slots and the first kTileEntries
// incidence entries, staged once per substep (item, contact constants), with their per-sweep
// corrections.
template <int TP>
struct PTile : Tile<TP> {
  static_assert(sizeof(PosRes) * TP >= 2 * kShapeScratch * sizeof(double), "shape scratch in res");
  int eoff[TP];
  int ent_next;                   // dynamic entry distribution of the current sweep
  int e_item[kTileEntries];
  ContactRef e_ref[kTileEntries];
  alignas(16) double e_out[kTileEntries][4];  // read and written as double2
  ShapeCache shape;                            // static data of this CTA's shape-matching chain
};

// Phase 0: per-position metadata of the tile (rod-local index, element count, kinds, block base),
// the OR of the kinds present and their ascending list. Ends with __syncthreads(); returns the
// kind mask.
template <int TP>
__device__ __forceinline__ unsigned tile_meta(Tile<TP>& t, const World& w, int start) {
  constexpr int kWarps = warps_for<TP>();
  constexpr int kTilePos = TP;
  const int V = w.V;
  const int tid = threadIdx.x, lane = tid & 31;
  // every lane of every warp takes part in the kind reduction (tiles need not be multiples of 32)
  for (int i0 = tid & ~31; i0 < kTilePos; i0 += 32 * kWarps) {
    const int i = i0 + lane;
    const int p = start - 1 + i;
    int k = -1, m = 0, kinds = 0, bb = 0;
    if (i < kTilePos && p >= 0 && p < V) {
      const int r = w.slot_rod[p];
      k = w.slot_loc[p];
      m = w.slot_m[p];
      kinds = w.rod_ekinds[r] | (w.rod_vkinds[r] << 4);
      bb = w.rod_block_base[r];
    }
    const unsigned wm = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(kinds));
    if (lane == 0) t.wmask[i0 >> 5] = wm;
    if (i < kTilePos) {
      t.loc[i] = k;
      t.m[i] = m;
      t.kinds[i] = kinds;
      t.bbase[i] = bb;
#pragma unroll
      for (int a = 0; a < kKinds; ++a) t.act[a][i] = 0;
    }
  }
  __syncthreads();
  unsigned mask = 0;
#pragma unroll
  for (int i = 0; i < (kTilePos + 31) / 32; ++i) mask |= t.wmask[i];
  if (tid < kKinds && (mask & (1u << tid))) t.klist[__popc(mask & ((1u << tid) - 1))] = tid;  // n-th kind present
  return mask;
}

// Phase 1: stage rows [r0, r1) that the tile's kinds read: 16-byte cp.async chunks (start-2 is
// even and rows are 256-byte aligned), all in flight at once; slots outside [0, V) are
// zero-filled. The caller waits (cp.async.wait_all + __syncthreads).
template <int TP>
__device__ __forceinline__ void stage_rows(Tile<TP>& t, const World& w, const double* X, const double* lam_in, int start,
                                           unsigned mask, int r0, int r1) {
  constexpr int kWarps = warps_for<TP>();
  constexpr int kChunks = (TP + 2) / 2;
  const int V = w.V, vp = w.vpad;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid >= 32 * kWarps) return;  // the persistent kernel's external-block warp stages nothing
  for (int r = r0 + (tid >> 5); r < r1; r += kWarps) {  // one warp per row, lanes over its chunks
    if (!(kRowNeed[r] & mask)) continue;
    const int arr = kRowArr[r];
    const double* row = (arr == 0 ? X : arr == 1 ? w.vstat : arr == 2 ? w.estat : lam_in) +
                        static_cast<long long>(kRowField[r]) * vp;
    for (int j = lane; j < kChunks; j += 32) {
      const int v = start - 2 + 2 * j;
      const int valid = v < 0 ? 0 : min(2, V - v);
      const double* src = row + (valid > 0 ? v : 0);
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&t.st[r][2 * j]));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(8 * max(valid, 0)));
    }
  }
}

// Phase 2: every elastic block of the tile evaluated and solved against the staged snapshot
// (eval_constraint :101-270 + solve_block :400-487), results to t.res, activity to t.act.
struct NoPost {
  __device__ void operator()(int&, unsigned long long&) const {}
};

// post(nsing, bad): extra per-thread work after the items, counted in the same reduction.
// ---- 1D bulk copies (TMA engine) global -> shared, completion on an mbarrier ----------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Interior tiles of the per-sweep kernel: every needed row segment (TP + 2 doubles, 16-byte
// aligned, a multiple of 16 bytes) is ONE bulk copy issued by the lanes of warp 0, all
// completing on the tile's mbarrier (initialised by tile_meta's caller). A handful of
// instructions per row instead of a cp.async loop per thread.
template <int TP>
__device__ __forceinline__ void stage_rows_bulk(Tile<TP>& t, const World& w, const double* X, const double* lam_in,
                                                int start, unsigned mask) {
  constexpr unsigned kBytes = (TP + 2) * sizeof(double);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    unsigned total = 0;
    for (int r = 0; r < kStageRows; ++r) total += (kRowNeed[r] & mask) ? kBytes : 0u;
    if (lane == 0) mbar_arrive_expect(&t.bar, total);
    __syncwarp();
    for (int r = lane; r < kStageRows; r += 32) {
      if (!(kRowNeed[r] & mask)) continue;
      const int arr = kRowArr[r];
      const double* row = (arr == 0 ? X : arr == 1 ? w.vstat : arr == 2 ? w.estat : lam_in) +
                          static_cast<long long>(kRowField[r]) * w.vpad;
      bulk_g2s(&t.st[r][0], row + (start - 2), kBytes, &t.bar);
    }
  }
}

template <int TP, bool kLamSmem, class Post = NoPost>
__device__ __forceinline__ void solve_items(Tile<TP>& t, const World& w, const SweepParams& sp, int start, unsigned mask,
                                            int* singular, unsigned long long* err, Post&& post = Post()) {
  constexpr int kWarps = warps_for<TP>();
  constexpr int kTilePos = TP, kTileOwned = TP - 2;
  const int vp = w.vpad;
  const int tid = threadIdx.x, lane = tid & 31;
  const double h2 = sp.h2, beta = sp.beta;
  int nsing = 0;
  unsigned long long bad = kNoError;
  // Work items (kind, position), kind-major over the kinds present in the tile: 64 positions
  // per kind, so every warp evaluates a single kind (no divergence between block formulas)
  // and all four warps share the tile's work whatever its kind mix.
  const int items = __popc(mask) * kTilePos;
  for (int item = tid; item < items; item += 32 * kWarps) {
    const int pi = item % kTilePos;
    const int kind = t.klist[item / kTilePos];
    const int k = t.loc[pi];
    if (k < 0) continue;
    const int p = start - 1 + pi;
    const int m = t.m[pi];
    const int ek = t.kinds[pi] & 15, vk = t.kinds[pi] >> 4;
    const bool owned = pi >= 1 && pi <= kTileOwned;
    const int si = pi + 1;  // staging index of p
    PosRes& R = t.res[pi];
    // Multipliers: per slot, ping-ponged in HBM (only the owner writes lam_out), or kept in the
    // tile's shared rows (persistent kernel: halo positions are updated identically by both
    // neighbouring tiles, so every copy stays equal to the owner's).
    auto put_lam = [&](int f, double v) {
      if (kLamSmem)
        t.st[T_LAM + f][si] = v;
      else if (owned)
        sp.lam_out[f * (long long)vp + p] = v;
    };
    auto keep_lam = [&](int f0, int nf) {
      if (kLamSmem || !owned) return;
      for (int f = f0; f < f0 + nf; ++f) sp.lam_out[f * (long long)vp + p] = t.st[T_LAM + f][si];
    };
    auto sing = [&]() {  // singular block: counted by its owner (per scene in a batch's last sweep)
      if (!owned) return;
      ++nsing;
      if (sp.scene_singular) atomicAdd(&sp.scene_singular[w.rod_scene[w.slot_rod[p]]], 1);
    };
    auto fail = [&](int local) { bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, t.bbase[pi] + local)); };
    const int ne = __popc(ek), nv = __popc(vk);

    if (k < m && kind < A_BT) {  // element pass of element k (constraints.cpp:302-314)
      const V3 c0{t.st[T_CX][si], t.st[T_CY][si], t.st[T_CZ][si]}, c1{t.st[T_CX][si + 1], t.st[T_CY][si + 1], t.st[T_CZ][si + 1]};
      const double s0 = t.st[T_S][si], s1 = t.st[T_S][si + 1];
      const double ic0 = t.st[T_IC][si], ic1 = t.st[T_IC][si + 1], is0 = t.st[T_IS][si], is1 = t.st[T_IS][si + 1];
      const V3 it{t.st[T_ITX][si], t.st[T_ITY][si], t.st[T_ITZ][si]};
      const int lbase = k * ne;
      if (kind == A_SZ && (ek & EK_SZ)) {  // StretchZ (:106-119), dim 3
        const M3 Rm = qmat(Q4{t.st[T_QW][si], t.st[T_QX][si], t.st[T_QY][si], t.st[T_QZ][si]});
        const double tbar = t.st[T_TDOT][si];
        const double l = t.st[T_LEN][si];
        const double inv_l = 1.0 / l;
        const V3 dzc = (c1 - c0) / l;
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
        const double kinv = t.st[T_KSZ][si];
        double rhs[3], dl[3];
        const double lam[3] = {t.st[T_LAM + L_SZ0][si], t.st[T_LAM + L_SZ1][si], t.st[T_LAM + L_SZ2][si]};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          M[d][d] = M[d][d] + kinv;
          rhs[d] = W[d] - kinv * lam[d];
        }
        if (solve3(M, rhs, beta, dl)) {
          const double f0 = -h2 * ic0, f1 = -h2 * ic1;
          bool ok = true;
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            R.sz_dc0[d] = f0 * (-inv_l * dl[d]);
            R.sz_dc1[d] = f1 * (inv_l * dl[d]);
            ok = ok && isfinite(dl[d]) && isfinite(R.sz_dc0[d]) && isfinite(R.sz_dc1[d]);
          }
          const double jt0 = (J0[0] * dl[0] + J0[1] * dl[1]) + J0[2] * dl[2];
          const double jt1 = (J1[0] * dl[0] + J1[1] * dl[1]) + J1[2] * dl[2];
          R.sz_dt[0] = -h2 * (it.x * jt0);
          R.sz_dt[1] = -h2 * (it.y * jt1);
          R.sz_dt[2] = 0.0;
          t.act[A_SZ][pi] = 1;
          put_lam(L_SZ0, lam[0] + dl[0]);
          put_lam(L_SZ1, lam[1] + dl[1]);
          put_lam(L_SZ2, lam[2] + dl[2]);
          if (owned) {
            if (!(ok && isfinite(R.sz_dt[0]) && isfinite(R.sz_dt[1]))) fail(lbase + __popc(ek & (EK_SZ - 1)));
          }
        } else {
          sing();
          keep_lam(L_SZ0, 3);
        }
      }
      if (kind == A_CS && (ek & EK_CS)) {  // CrossSection (:120-129), dim 1
        const double W = 0.5 * (s0 + s1) - 0.5 * (t.st[T_SBAR][si] + t.st[T_SBAR][si + 1]);
        double M = 0.0;
        if (is0 != 0.0) M = M + (h2 * is0 * 0.5) * 0.5;
        if (is1 != 0.0) M = M + (h2 * is1 * 0.5) * 0.5;
        const double kinv = t.st[T_KCS][si];
        const double lam = t.st[T_LAM + L_CS][si];
        M = M + kinv;
        if (M > 1e-250) {
          const double dl = beta * (W - kinv * lam) / M;
          R.cs[0] = -h2 * is0 * (0.5 * dl);
          R.cs[1] = -h2 * is1 * (0.5 * dl);
          t.act[A_CS][pi] = 1;
          put_lam(L_CS, lam + dl);
          if (owned) {
            if (!(isfinite(dl) && isfinite(R.cs[0]) && isfinite(R.cs[1]))) fail(lbase + __popc(ek & (EK_CS - 1)));
          }
        } else {
          sing();
          keep_lam(L_CS, 1);
        }
      }
      if (kind == A_SS && (ek & EK_SS)) {  // SurfaceStretch (:130-138), dim 1
        const double l = t.st[T_LEN][si];
        const double W = (s1 - s0) / l - t.st[T_SGRAD][si];
        const double j0 = -1.0 / l, j1 = 1.0 / l;
        double M = 0.0;
        if (is0 != 0.0) M = M + (h2 * is0 * j0) * j0;
        if (is1 != 0.0) M = M + (h2 * is1 * j1) * j1;
        const double kinv = t.st[T_KSS][si];
        const double lam = t.st[T_LAM + L_SS][si];
        M = M + kinv;
        if (M > 1e-250) {
          const double dl = beta * (W - kinv * lam) / M;
          R.ss[0] = -h2 * is0 * (j0 * dl);
          R.ss[1] = -h2 * is1 * (j1 * dl);
          t.act[A_SS][pi] = 1;
          put_lam(L_SS, lam + dl);
          if (owned) {
            if (!(isfinite(dl) && isfinite(R.ss[0]) && isfinite(R.ss[1]))) fail(lbase + __popc(ek & (EK_SS - 1)));
          }
        } else {
          sing();
          keep_lam(L_SS, 1);
        }
      }
      if (kind == A_VS && (ek & EK_VS)) {  // VolumeStretch (:169-188), dim 3
        const M3 Rm = qmat(Q4{t.st[T_QW][si], t.st[T_QX][si], t.st[T_QY][si], t.st[T_QZ][si]});
        const double tbar = t.st[T_TDOT][si];
        const double l0 = t.st[T_LEN0][si];
        const double smid = 0.5 * (s0 + s1);
        const double smr = 0.5 * (t.st[T_SBAR][si] + t.st[T_SBAR][si + 1]);
        const V3 dzc = (c1 - c0) / l0;
        const V3 wv = col(Rm, 2);
        const double ka = smid * smid, kb = smr * smr * tbar;
        const double W[3] = {ka * dzc.x - kb * wv.x, ka * dzc.y - kb * wv.y, ka * dzc.z - kb * wv.z};
        const double jc = smid * smid / l0;
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
        const double kinv = t.st[T_KVS][si];
        double rhs[3], dl[3];
        const double lam[3] = {t.st[T_LAM + L_VS0][si], t.st[T_LAM + L_VS1][si], t.st[T_LAM + L_VS2][si]};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          M[d][d] = M[d][d] + kinv;
          rhs[d] = W[d] - kinv * lam[d];
        }
        if (solve3(M, rhs, beta, dl)) {
          const double f0 = -h2 * ic0, f1 = -h2 * ic1;
          bool ok = true;
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            R.vs_dc0[d] = f0 * (-jc * dl[d]);
            R.vs_dc1[d] = f1 * (jc * dl[d]);
            ok = ok && isfinite(dl[d]) && isfinite(R.vs_dc0[d]) && isfinite(R.vs_dc1[d]);
          }
          const double jd = (js[0] * dl[0] + js[1] * dl[1]) + js[2] * dl[2];
          R.vs_ds[0] = -h2 * is0 * jd;
          R.vs_ds[1] = -h2 * is1 * jd;
          const double jt0 = (J0[0] * dl[0] + J0[1] * dl[1]) + J0[2] * dl[2];
          const double jt1 = (J1[0] * dl[0] + J1[1] * dl[1]) + J1[2] * dl[2];
          R.vs_dt[0] = -h2 * (it.x * jt0);
          R.vs_dt[1] = -h2 * (it.y * jt1);
          R.vs_dt[2] = 0.0;
          t.act[A_VS][pi] = 1;
          put_lam(L_VS0, lam[0] + dl[0]);
          put_lam(L_VS1, lam[1] + dl[1]);
          put_lam(L_VS2, lam[2] + dl[2]);
          if (owned) {
            if (!(ok && isfinite(R.vs_ds[0]) && isfinite(R.vs_ds[1]) && isfinite(R.vs_dt[0]) && isfinite(R.vs_dt[1])))
              fail(lbase + __popc(ek & (EK_VS - 1)));
          }
        } else {
          sing();
          keep_lam(L_VS0, 3);
        }
      }
    }

    if (k >= 1 && k <= m - 1 && kind >= A_BT) {  // vertex pass of vertex k (:315-327)
      const Q4 qa{t.st[T_QW][si - 1], t.st[T_QX][si - 1], t.st[T_QY][si - 1], t.st[T_QZ][si - 1]};
      const Q4 qb{t.st[T_QW][si], t.st[T_QX][si], t.st[T_QY][si], t.st[T_QZ][si]};
      const double sm = t.st[T_S][si - 1], s0 = t.st[T_S][si], spp = t.st[T_S][si + 1];
      const double is0 = t.st[T_IS][si];
      const V3 ita{t.st[T_ITX][si - 1], t.st[T_ITY][si - 1], t.st[T_ITZ][si - 1]};
      const V3 itb{t.st[T_ITX][si], t.st[T_ITY][si], t.st[T_ITZ][si]};
      const double sbar = t.st[T_SBAR][si];
      const double la = t.st[T_LEN][si - 1], lb = t.st[T_LEN][si];
      const int lbase = m * ne + (k - 1) * nv;
      Q4 pr{1, 0, 0, 0};
      if (vk & (VK_BT | VK_VBU | VK_VBV)) pr = relative_rotation(qa, qb);
      // 0.5*(-+p.w I + [p_v]x) (constraints.cpp:50-51)
      const double Da[3][3] = {{0.5 * -pr.w, 0.5 * -pr.z, 0.5 * pr.y},
                               {0.5 * pr.z, 0.5 * -pr.w, 0.5 * -pr.x},
                               {0.5 * -pr.y, 0.5 * pr.x, 0.5 * -pr.w}};
      const double Db[3][3] = {{0.5 * pr.w, 0.5 * -pr.z, 0.5 * pr.y},
                               {0.5 * pr.z, 0.5 * pr.w, 0.5 * -pr.x},
                               {0.5 * -pr.y, 0.5 * pr.x, 0.5 * pr.w}};
      if (kind == A_BT && (vk & VK_BT)) {  // BendTwist (:139-155), dim 3
        const double inv_len = 4.0 / (la + lb);
        const V3 om = inv_len * qvec(pr);
        const double s = sp.classic ? sbar : s0;
        const V3 darb{t.st[T_DARBX][si - 1], t.st[T_DARBY][si - 1], t.st[T_DARBZ][si - 1]};
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
        const double kinv[3] = {t.st[T_KBT0][si], t.st[T_KBT0][si],
                                t.st[T_KBT2][si]};
        const double lam[3] = {t.st[T_LAM + L_BT0][si], t.st[T_LAM + L_BT1][si], t.st[T_LAM + L_BT2][si]};
        double rhs[3], dl[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          M[d][d] = M[d][d] + kinv[d];
          rhs[d] = W[d] - kinv[d] * lam[d];
        }
        if (solve3(M, rhs, beta, dl)) {
          bool ok = isfinite(dl[0]) && isfinite(dl[1]) && isfinite(dl[2]);
          R.bt_ds = 0.0;
          if (!sp.classic) {
            R.bt_ds = -h2 * is0 * ((omv[0] * dl[0] + omv[1] * dl[1]) + omv[2] * dl[2]);
            ok = ok && isfinite(R.bt_ds);
          }
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            R.bt_dta[b] = -h2 * (comp(ita, b) * ((Ja[0][b] * dl[0] + Ja[1][b] * dl[1]) + Ja[2][b] * dl[2]));
            R.bt_dtb[b] = -h2 * (comp(itb, b) * ((Jb[0][b] * dl[0] + Jb[1][b] * dl[1]) + Jb[2][b] * dl[2]));
            ok = ok && isfinite(R.bt_dta[b]) && isfinite(R.bt_dtb[b]);
          }
          t.act[A_BT][pi] = 1;
          put_lam(L_BT0, lam[0] + dl[0]);
          put_lam(L_BT1, lam[1] + dl[1]);
          put_lam(L_BT2, lam[2] + dl[2]);
          if (owned) {
            if (!ok) fail(lbase + __popc(vk & (VK_BT - 1)));
          }
        } else {
          sing();
          keep_lam(L_BT0, 3);
        }
      }
      if (kind == A_SB && (vk & VK_SB)) {  // SurfaceBending (:156-168), dim 1
        const double lap = (spp - s0) / lb - (s0 - sm) / la;
        const double W = lap - t.st[T_SLAP][si - 1];
        const double jm = 1.0 / la, j0 = -1.0 / la - 1.0 / lb, jp = 1.0 / lb;
        const double ism = t.st[T_IS][si - 1], isp = t.st[T_IS][si + 1];
        double M = 0.0;
        if (ism != 0.0) M = M + (h2 * ism * jm) * jm;
        if (is0 != 0.0) M = M + (h2 * is0 * j0) * j0;
        if (isp != 0.0) M = M + (h2 * isp * jp) * jp;
        const double kinv = t.st[T_KSB][si];
        const double lam = t.st[T_LAM + L_SB][si];
        M = M + kinv;
        if (M > 1e-250) {
          const double dl = beta * (W - kinv * lam) / M;
          R.sb[0] = -h2 * ism * (jm * dl);
          R.sb[1] = -h2 * is0 * (j0 * dl);
          R.sb[2] = -h2 * isp * (jp * dl);
          t.act[A_SB][pi] = 1;
          put_lam(L_SB, lam + dl);
          if (owned) {
            if (!(isfinite(dl) && isfinite(R.sb[0]) && isfinite(R.sb[1]) && isfinite(R.sb[2])))
              fail(lbase + __popc(vk & (VK_SB - 1)));
          }
        } else {
          sing();
          keep_lam(L_SB, 1);
        }
      }
      if (kind >= A_VBU) {  // VolumeBendU / V (:189-214), dim 1
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int bit = cc == 0 ? VK_VBU : VK_VBV;
          if (kind != A_VBU + cc || !(vk & bit)) continue;
          const double la0 = t.st[T_LEN0][si - 1], lb0 = t.st[T_LEN0][si];
          const double inv_len0 = 4.0 / (la0 + lb0);
          const double om = inv_len0 * (cc == 0 ? pr.x : pr.y);
          const double darb = t.st[cc == 0 ? T_DARBX : T_DARBY][si - 1];
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
          const double kinv = t.st[T_KVB][si];
          const int lf = cc == 0 ? L_VBU : L_VBV;
          const double lam = t.st[T_LAM + lf][si];
          M = M + kinv;
          if (M > 1e-250) {
            const double dl = beta * (W - kinv * lam) / M;
            R.vb_ds[cc] = -h2 * is0 * (js * dl);
            bool ok = isfinite(dl) && isfinite(R.vb_ds[cc]);
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              R.vb_dta[cc][b] = -h2 * (comp(ita, b) * (ja[b] * dl));
              R.vb_dtb[cc][b] = -h2 * (comp(itb, b) * (jb[b] * dl));
              ok = ok && isfinite(R.vb_dta[cc][b]) && isfinite(R.vb_dtb[cc][b]);
            }
            t.act[cc == 0 ? A_VBU : A_VBV][pi] = 1;
            put_lam(lf, lam + dl);
            if (owned) {
              if (!ok) fail(lbase + __popc(vk & (bit - 1)));
            }
          } else {
            sing();
            keep_lam(lf, 1);
          }
        }
      }
    }
  }
  if (sp.dbg && (threadIdx.x & 31) == 0) sp.dbg[threadIdx.x >> 5] = gtimer();  // VROD_TRACE: items done
  post(nsing, bad);
  if (sp.dbg && (threadIdx.x & 31) == 0) sp.dbg[16 + (threadIdx.x >> 5)] = gtimer();  // + external entries
  if (__any_sync(0xffffffffu, nsing != 0 || bad != kNoError)) {  // rare: singular blocks / errors
    for (int o = 16; o > 0; o >>= 1) {
      nsing += __shfl_down_sync(0xffffffffu, nsing, o);
      const unsigned long long b2 = __shfl_down_sync(0xffffffffu, bad, o);
      bad = umin64(bad, b2);
    }
    if (lane == 0) {
      if (nsing) atomicAdd(singular, nsing);
      if (bad != kNoError) atomicMin(err, bad);
    }
  }
  __syncthreads();

}

// Phase 3: one thread per owned slot gathers the corrections of every block touching it in the
// reference's block order (constraints.cpp:509-534) — element pass of element k-1 then k,
// vertex pass of vertex k-1, k, k+1, then the external blocks through `ext` — divides by the
// number of active touching blocks and applies (:537-554) into Y (and the slot record).
template <int TP, class ExtGather>
__device__ __forceinline__ void gather_apply(const Tile<TP>& t, const World& w, const SweepParams& sp, int start, double* Y,
                                             double* xrec_out, ExtGather&& ext) {
  constexpr int kWarps = warps_for<TP>();
  constexpr int kTileOwned = TP - 2;
  const int vp = w.vpad;
  const int tid = threadIdx.x, lane = tid & 31;
  // Small (latency-bound) tiles: two threads per slot (adjacent warps), role 0 gathers and
  // applies the center and scale (elastic + external blocks), role 1 the frame (elastic blocks
  // only; external blocks have no theta slots) — two shorter dependency chains instead of one.
  // Large (issue-bound) tiles: one thread per slot does all three (role 2).
  constexpr bool kSplit = TP == 32;
  const int role = kSplit ? (tid >> 5) & 1 : 2;
  for (int pi = kSplit ? 1 + lane + 32 * (tid >> 6) : 1 + tid; pi <= kTileOwned; pi += kSplit ? 16 * kWarps : 32 * kWarps) {
    const int k = t.loc[pi];
    if (k < 0) continue;
    const int p = start - 1 + pi;
    const int m = t.m[pi];
    const int si = pi + 1;
    const bool prev_el = k >= 1, has_el = k < m, prev_vx = k - 1 >= 1, has_vx = k >= 1 && k <= m - 1,
               next_vx = k + 1 <= m - 1;
    const PosRes& A = t.res[pi - 1];  // element k-1 / vertex k-1
    const PosRes& B = t.res[pi];      // element k / vertex k
    const PosRes& N = t.res[pi + 1];  // vertex k+1
    V3 csum{0, 0, 0};
    int ccnt = 0;
    double ssum = 0.0;
    int scnt = 0;
    V3 tsum{0, 0, 0};
    int tcnt = 0;
    auto addc = [&](const double* d) {
      if (role == 1) return;
      csum = csum + V3{d[0], d[1], d[2]};
      ++ccnt;
    };
    auto adds = [&](double d) {
      if (role == 1) return;
      ssum += d;
      ++scnt;
    };
    auto addt = [&](const double* d) {
      if (role == 0) return;
      tsum = tsum + V3{d[0], d[1], d[2]};
      ++tcnt;
    };
    // element pass: element k-1 (this vertex is its c1/s1), then element k (c0/s0, theta)
    if (prev_el) {
      if (t.act[A_SZ][pi - 1]) addc(A.sz_dc1);
      if (t.act[A_CS][pi - 1]) adds(A.cs[1]);
      if (t.act[A_SS][pi - 1]) adds(A.ss[1]);
      if (t.act[A_VS][pi - 1]) {
        addc(A.vs_dc1);
        adds(A.vs_ds[1]);
      }
    }
    if (has_el) {
      if (t.act[A_SZ][pi]) {
        addc(B.sz_dc0);
        addt(B.sz_dt);
      }
      if (t.act[A_CS][pi]) adds(B.cs[0]);
      if (t.act[A_SS][pi]) adds(B.ss[0]);
      if (t.act[A_VS][pi]) {
        addc(B.vs_dc0);
        adds(B.vs_ds[0]);
        addt(B.vs_dt);
      }
    }
    // vertex pass: vertex k-1 (SurfaceBending s_{j+1}), vertex k, vertex k+1
    if (prev_vx && t.act[A_SB][pi - 1]) adds(A.sb[2]);
    if (has_vx) {
      if (t.act[A_BT][pi]) {
        if (!sp.classic) adds(B.bt_ds);
        addt(B.bt_dtb);
      }
      if (t.act[A_SB][pi]) adds(B.sb[1]);
      if (t.act[A_VBU][pi]) {
        adds(B.vb_ds[0]);
        addt(B.vb_dtb[0]);
      }
      if (t.act[A_VBV][pi]) {
        adds(B.vb_ds[1]);
        addt(B.vb_dtb[1]);
      }
    }
    if (next_vx) {
      if (t.act[A_BT][pi + 1]) addt(N.bt_dta);
      if (t.act[A_SB][pi + 1]) adds(N.sb[0]);
      if (t.act[A_VBU][pi + 1]) addt(N.vb_dta[0]);
      if (t.act[A_VBV][pi + 1]) addt(N.vb_dta[1]);
    }
    if (role != 1) {
      ext(p, addc, adds);
      V3 cn{t.st[T_CX][si], t.st[T_CY][si], t.st[T_CZ][si]};
      if (ccnt > 0) cn = cn + csum / static_cast<double>(ccnt);
      double sn = t.st[T_S][si];
      if (scnt > 0) sn = fmax(sn + ssum / static_cast<double>(scnt), kMinScale);
      Y[CX * (long long)vp + p] = cn.x;
      Y[CY * (long long)vp + p] = cn.y;
      Y[CZ * (long long)vp + p] = cn.z;
      Y[S * (long long)vp + p] = sn;
      if (xrec_out) {
        double2* xr = reinterpret_cast<double2*>(xrec_out + 8ll * p);
        xr[0] = make_double2(cn.x, cn.y);
        xr[1] = make_double2(cn.z, sn);
      }
    }
    if (role != 0) {
      Q4 qn{t.st[T_QW][si], t.st[T_QX][si], t.st[T_QY][si], t.st[T_QZ][si]};
      if (has_el && tcnt > 0) qn = apply_increment(qn, tsum / static_cast<double>(tcnt));
      Y[QW * (long long)vp + p] = qn.w;
      Y[QX * (long long)vp + p] = qn.x;
      Y[QY * (long long)vp + p] = qn.y;
      Y[QZ * (long long)vp + p] = qn.z;
    }
  }
}



// The external blocks touching a slot (entries [e0, e1)), in block order (incidence entries are slot-sorted, then
// block-sorted): each entry holds the block's correction of this endpoint (ext_contrib, kExtNone
// markers for "no update" / "no scale update"). Chunks of 4 entries: all loads of a chunk are
// issued before the first add (the markers only predicate the adds), so a slot's list costs one
// latency per chunk.
template <class AddC, class AddS>
__device__ __forceinline__ void gather_entries(const Collide& c, int e0, int e1, AddC& addc, AddS& adds,
                                               const double* local = nullptr, int local_q0 = 0, int local_n = 0) {
  for (int q0 = e0; q0 < e1; q0 += 4) {
    double2 o01[4], o23[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u < e1 ? q0 + u : e0;
      const int i = q - local_q0;  // entries staged in shared memory (persistent kernel)
      const double2* o = reinterpret_cast<const double2*>(i >= 0 && i < local_n ? local + 4ll * i : c.ext_contrib + 4ll * q);
      o01[u] = o[0];
      o23[u] = o[1];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (q0 + u >= e1 || is_ext_none(o01[u].x)) continue;
      const double d[3] = {o01[u].x, o01[u].y, o23[u].x};
      addc(d);
      if (!is_ext_none(o23[u].y)) adds(o23[u].y);
    }
  }
}

// Writes an endpoint's correction into its incidence entry o (4 doubles; flag 0 = no update from
// the block; kExtNone in ds = no scale update).
__device__ __forceinline__ void put_entry(double* out, int flag, double x, double y, double z, double ds) {
  double2* o = reinterpret_cast<double2*>(out);
  if (flag) {
    o[0] = make_double2(x, y);
    o[1] = make_double2(z, (flag & kExtScale) ? ds : ext_none());
  } else {
    o[0].x = ext_none();
  }
}

// One sweep per launch (large worlds; every world when the persistent kernel does not apply).
template <int TP>
__global__ void __launch_bounds__(32 * warps_for<TP>(), TP == 32 ? 2 : 4) k_rod_sweep(World w, Collide c, const double* __restrict__ X,
                                                          double* __restrict__ Y, SweepParams sp, int* singular,
                                                          unsigned long long* err, int has_ext) {
  constexpr int kWarps = warps_for<TP>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kTileOwned = TP - 2;
  Tile<TP>& t = *reinterpret_cast<Tile<TP>*>(smem_raw);
  if (sp.pdl == 1) {  // predecessor wrote X: wait before staging
    pdl_wait();
    pdl_trigger();
  }
  const int V = w.V;
  const int start = blockIdx.x * kTileOwned;
  const int tid = threadIdx.x;
  // interior tiles stage with bulk copies: the whole window [start-2, start+TP) lies inside
  // every row's allocation (rows are vpad doubles)
  const bool bulk = start >= 2 && start + TP <= w.vpad;
  if (bulk && tid == 0) mbar_init(&t.bar);  // made visible by tile_meta's __syncthreads
  const unsigned mask = tile_meta(t, w, start);
  if (bulk)
    stage_rows_bulk(t, w, X, sp.lam_in, start, mask);
  else
    stage_rows(t, w, X, sp.lam_in, start, mask, 0, kStageRows);
  // The ext solve of this iteration (the predecessor) writes the tile's incidence entries.
  // Large worlds (64-wide tiles, bandwidth-bound): wait for it here and prefetch the tile's
  // entry range into L2 so the gather after the block solves finds it on chip. Small worlds
  // (latency-bound): solve the tile's blocks first, overlapping the ext solve's tail, and wait
  // just before the gather.
  constexpr bool kEarlyWait = TP != 32;
  if (kEarlyWait && sp.pdl == 2) {
    pdl_wait();
    pdl_trigger();
  }
  if (kEarlyWait && has_ext) {
    const int e0 = c.ext_off[max(start, 0)], e1 = c.ext_off[min(start + kTileOwned, V)];
    const char* lo = reinterpret_cast<const char*>(c.ext_contrib + 4ll * e0);
    const char* hi = reinterpret_cast<const char*>(c.ext_contrib + 4ll * e1);
    for (const char* a = lo + 128ll * tid; a < hi; a += 128ll * 32 * kWarps)
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a));
  }
  if (bulk)
    mbar_wait(&t.bar, 0);
  else
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();

  solve_items<TP, false>(t, w, sp, start, mask, singular, err);

  if (!kEarlyWait && sp.pdl == 2) {
    pdl_wait();
    pdl_trigger();
  }
  gather_apply(t, w, sp, start, Y, has_ext ? w.xrec : nullptr, [&](int p, auto& addc, auto& adds) {
    if (has_ext) gather_entries(c, c.ext_off[p], c.ext_off[p + 1], addc, adds);
  });
}

// Grid-wide barrier of the persistent kernel (all CTAs co-resident: cooperative launch). The
// counter is zeroed before each launch; `target` advances by gridDim.x per barrier.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// The whole iteration loop of one substep (solver.cpp:330-339) for small single-scene worlds,
// in ONE launch: one CTA per tile, all tiles co-resident, a grid barrier after each sweep and
// after each shape-matching level. What the per-launch path moves through HBM every sweep
// stays on chip: the tile's static rows are staged once, the elastic multipliers live in the
// tile's shared rows (never written back; they are reset every substep anyway), and the
// external blocks are not solved by a separate kernel: every incidence entry re-solves its block
// in the gather (ext_block, ext.cuh — the same arithmetic as k_ext_solve, so the same bits)
// and only the block's owner entry commits its multiplier (ping-pong lam_ext[2]) and counts
// singular / non-finite outcomes. The slot records are ping-ponged too (xrec[2]), so blocks
// solved by other tiles during a sweep always see the snapshot.
// Aux CTAs (the SMs the tiles leave idle): all external blocks of the sweep, one thread per
// block (ext_block, the k_ext_solve code), corrections into the slot-sorted incidence entries;
// then a release of `ext_done` for the tiles' gathers.
template <int TP>
__device__ __forceinline__ void aux_ext_phase(const World& w, const Collide& c, const PersistParams& pp,
                                              const SweepParams& sp, const double* cur, const double* xr_cur,
                                              const double* el_cur, double* el_nxt, int it, int* singular,
                                              unsigned long long* err) {
  const int kThreadsPerCta = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int npins = sp.n_pins, nct = c.scalars[SC_NCT];
  const int n = npins + nct + c.scalars[SC_NHP];
  int nsing = 0;
  unsigned long long bad = kNoError;
  for (int b = (blockIdx.x - pp.tiles) * kThreadsPerCta + tid; b < n; b += pp.n_aux * kThreadsPerCta) {
    const ExtResult r = ext_block(
        w, c, cur, xr_cur, el_cur, c.ext_cap, b, sp,
        [&](int e, int flag, double x, double y, double z, double ds) {
          put_entry(c.ext_contrib + 4ll * c.ext_pos[4 * b + e], flag, x, y, z, ds);
        },
        nullptr, nct);
    for (int d = 0; d < r.nlam; ++d) el_nxt[d * c.ext_cap + b] = r.lam[d];
    if (r.singular) ++nsing;
    if (r.bad) bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, it, static_cast<unsigned long long>(sp.elastic_blocks) + b));
  }
  if (__any_sync(0xffffffffu, nsing != 0 || bad != kNoError)) {
    for (int o = 16; o > 0; o >>= 1) {
      nsing += __shfl_down_sync(0xffffffffu, nsing, o);
      bad = umin64(bad, __shfl_down_sync(0xffffffffu, bad, o));
    }
    if (lane == 0) {
      if (nsing) atomicAdd(singular, nsing);
      if (bad != kNoError) atomicMin(err, bad);
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    atomicAdd(pp.ext_done, 1u);
  }
}

// The whole iteration loop of one substep (solver.cpp:330-339) for small single-scene worlds,
// in ONE launch: one CTA per tile, all CTAs co-resident, a grid barrier after each sweep and
// after each shape-matching phase. What the per-launch path moves through HBM every sweep
// stays on chip: the tile's static rows are staged once, the elastic multipliers live in the
// tile's shared rows (never written back; they are reset every substep anyway).
//
// When SMs are left over (pp.n_aux > 0, e.g. C3: 128 tiles + 20 aux CTAs on 148 SMs), the aux
// CTAs solve the external blocks during each sweep (released to the tiles through ext_done, so
// the tiles with contacts no longer finish late) and run the shape matching; their small code
// stays hot in their instruction caches. Otherwise (n_aux = 0) every incidence entry of a
// tile's owned slots re-solves its block in the tile (ext_block — the same arithmetic as
// k_ext_solve, so the same bits) and only the block's owner entry commits its multiplier
// (ping-pong lam_ext[2]) and counts; all CTAs share the shape work. The slot records are
// ping-ponged (xrec[2]), so blocks solved elsewhere during a sweep always see the snapshot.
template <int TP, bool kExactShape>
__global__ void __launch_bounds__(32 * (warps_for<TP>() + 1), 1) k_iterate(World w, Collide c, Groups g, PersistParams pp,
                                                                      SweepParams sp, int* singular,
                                                                      unsigned long long* err) {
  constexpr int kWarps = warps_for<TP>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kTileOwned = TP - 2, kTileStage = TP + 2;
  PTile<TP>& t = *reinterpret_cast<PTile<TP>*>(smem_raw);
  const bool is_aux = blockIdx.x >= pp.tiles;
  const bool inline_ext = pp.n_aux == 0;
  const int nct = pp.has_ext ? c.scalars[SC_NCT] : 0;  // the substep's contact count
  const int start = is_aux ? 0 : blockIdx.x * kTileOwned;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int has_ext = pp.has_ext;
  unsigned mask = 0;
  int ent_q0 = 0, ent_n = 0;  // staged entries: [ent_q0, ent_q0 + ent_n)
  if (!is_aux) {
    mask = tile_meta(t, w, start);
    stage_rows(t, w, nullptr, nullptr, start, mask, T_SBAR, T_LAM);  // statics: once per substep
    if (has_ext) {
      for (int i = tid; i <= kTileOwned; i += 32 * kWarps) t.eoff[i] = c.ext_off[min(start + i, w.V)];
      const int q0 = c.ext_off[start], q1 = c.ext_off[min(start + kTileOwned, w.V)];
      ent_q0 = q0;
      ent_n = min(q1 - q0, kTileEntries);
      if (inline_ext) {
        const int npins = sp.n_pins;
        for (int i = tid; i < ent_n; i += 32 * kWarps) {
          const int item = c.ext_items[q0 + i];
          t.e_item[i] = item;
          const int b = item >> 2;
          if (b >= npins && b < npins + nct) t.e_ref[i] = contact_ref(c, b - npins);
        }
      }
    }
    for (int i = tid; i < kLamFields * kTileStage; i += 32 * kWarps) t.st[T_LAM + i / kTileStage][i % kTileStage] = 0.0;
  }
  // the groups of the chain this CTA's warp 0 runs (chain u = CTA index, see the shape pass)
  const int my_chain = inline_ext ? blockIdx.x : blockIdx.x - pp.tiles;
  const bool cache_shape = g.G > 0 && g.nchains > 0 && my_chain >= 0 && my_chain < g.nchains;
  if (cache_shape) shape_cache_fill(t.shape, w, g, g.chain_groups, g.chain_off[my_chain], g.chain_off[my_chain + 1]);
  double* cur = pp.X;
  double* nxt = pp.Y;
  double* xr_cur = pp.xrec[0];
  double* xr_nxt = pp.xrec[1];
  double* el_cur = pp.lam_ext[0];
  double* el_nxt = pp.lam_ext[1];
  unsigned target = 0;
  int ntr = 0;
  auto mark = [&]() {  // debug phase trace (VROD_TRACE=1): CTA 0, one timestamp per phase
    if (pp.trace && blockIdx.x == 0 && tid == 0 && ntr < kTraceCap - 1) {
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      pp.trace[1 + ntr++] = ns;
      pp.trace[0] = ntr;
    }
  };
  mark();
  if (pp.trace && blockIdx.x == 0 && tid == 0) pp.trace[598] = g.nchains > 0 ? 1 : pp.levels;
  for (int it = 0; it < pp.iterations; ++it) {
    sp.iter = it;
    if (is_aux) {
      if (has_ext) aux_ext_phase<TP>(w, c, pp, sp, cur, xr_cur, el_cur, el_nxt, it, singular + it, err);
    } else {
      if (it > 0) {
        for (int i = tid; i < kKinds * TP; i += 32 * kWarps) t.act[i / TP][i % TP] = 0;
      }
      if (tid == 0) t.ent_next = 0;  // published by the __syncthreads below
      stage_rows(t, w, cur, nullptr, start, mask, 0, T_SBAR);
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncthreads();
      mark();
      // Inline external blocks: every incidence entry of the tile's owned slots (a contiguous
      // range) re-solves its block on the snapshot, one thread per entry, after that thread's
      // elastic items — entries go to the warps of the cheapest kinds first — and writes its
      // endpoint's correction into the entry; the block's owner entry commits the multiplier.
      auto ext_entries = [&](int& nsing, unsigned long long& bad) {
        if (!has_ext || !inline_ext) return;
        // Dynamic distribution: every warp takes the next 32 entries from a shared counter once
        // it is done with its elastic items — the CTA's extra warp (no items) at once, the warps
        // of the cheap kinds early, the heavy ones rarely. Each entry's result is independent of
        // which warp computes it.
        const int q0 = t.eoff[0], q1 = t.eoff[kTileOwned];
        for (;;) {
          int b0 = 0;
          if (lane == 0) b0 = atomicAdd(&t.ent_next, 32);
          b0 = __shfl_sync(0xffffffffu, b0, 0);
          if (b0 >= q1 - q0) break;
          const int q = q0 + b0 + lane;
          if (q >= q1) continue;
          const int i = q - ent_q0;
          const bool staged = i < ent_n;
          const int item = staged ? t.e_item[i] : c.ext_items[q];
          const int b = item >> 2, e = item & 3;
          double* out = staged ? t.e_out[i] : c.ext_contrib + 4ll * q;
          const ExtResult res = ext_block(
              w, c, cur, xr_cur, el_cur, c.ext_cap, b, sp,
              [&](int e2, int flag, double x, double y, double z, double ds) {
                if (e2 == e) put_entry(out, flag, x, y, z, ds);
              },
              staged && b >= sp.n_pins && b < sp.n_pins + nct ? &t.e_ref[i] : nullptr, nct);
          if (e == res.owner) {  // the block's owner entry commits it
            for (int d = 0; d < res.nlam; ++d) el_nxt[d * c.ext_cap + b] = res.lam[d];
            if (res.singular) ++nsing;
            if (res.bad)
              bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, it, static_cast<unsigned long long>(sp.elastic_blocks) + b));
          }
        }
      };
      // VROD_TRACE: per-warp phase ends of one CTA (pp.trace_cta, default 0) in iteration 1
      sp.dbg = pp.trace && it == 1 && blockIdx.x == pp.trace_cta ? pp.trace + 900 : nullptr;
      if (sp.dbg && tid == 0) pp.trace[899] = gtimer();
      solve_items<TP, true>(t, w, sp, start, mask, singular + it, err, ext_entries);  // ends with __syncthreads()
      mark();
      if (has_ext && !inline_ext) {  // the aux CTAs' external blocks of this sweep
        if (tid == 0) {
          const unsigned want = (it + 1u) * static_cast<unsigned>(pp.n_aux);
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(pp.ext_done) : "memory");
          } while (v < want);
        }
        __syncthreads();
        // the tile's entries in one coalesced copy (all loads in flight), then the gather reads
        // them from shared memory
        const double2* src = reinterpret_cast<const double2*>(c.ext_contrib + 4ll * ent_q0);
        double2* dst = reinterpret_cast<double2*>(&t.e_out[0][0]);
        for (int i = tid; i < 2 * ent_n; i += 32 * kWarps) dst[i] = __ldcg(src + i);
        __syncthreads();
      }
      gather_apply(t, w, sp, start, nxt, has_ext ? xr_nxt : nullptr, [&](int p, auto& addc, auto& adds) {
        if (has_ext)
          gather_entries(c, t.eoff[p - start], t.eoff[p - start + 1], addc, adds, &t.e_out[0][0], ent_q0, ent_n);
      });
      mark();
      if (pp.trace && it == 1 && tid == 0) pp.trace[700 + blockIdx.x] = gtimer();
    }
    grid_sync(pp.bar, target);
    mark();
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
    tmp = xr_cur;
    xr_cur = xr_nxt;
    xr_nxt = tmp;
    tmp = el_cur;
    el_cur = el_nxt;
    el_nxt = tmp;
    if (g.G > 0 && (it + 1) % pp.sm_period == 0) {  // shape matching (shape.cuh)
      // One warp per work unit: a dependency chain of groups (one barrier in all), or one group
      // of the current level (a barrier per level); the aux CTAs' warps when there are any. A
      // single call site keeps one copy of the group code in the kernel.
      const bool workers = inline_ext || is_aux;
      const int ncta = inline_ext ? gridDim.x : pp.n_aux, cta = inline_ext ? blockIdx.x : blockIdx.x - pp.tiles;
      const int gw = warp * ncta + cta, nw = static_cast<int>(blockDim.x >> 5) * ncta;
      const bool chains = g.nchains > 0;
      const int phases = chains ? 1 : pp.levels;
      for (int l = 0; l < phases; ++l) {
        const int u0 = chains ? 0 : pp.level_off[l], u1 = chains ? g.nchains : pp.level_off[l + 1];
        for (int u = u0 + gw; workers && u < u1; u += nw) {
          const int k0 = chains ? g.chain_off[u] : u, k1 = chains ? g.chain_off[u + 1] : u + 1;
          for (int k = k0; k < k1; ++k) {
            const bool tr = pp.trace && it == 1 && (chains ? u == 28 : u == u0);
            // exact path: warps 0 and 1 order their member sums through the tile's block-result
            // rows (idle between sweeps), other warps use shuffles
            double* scratch = kExactShape && warp < 2 && !is_aux
                                  ? reinterpret_cast<double*>(&t.res[0]) + warp * kShapeScratch
                                  : nullptr;
            shape_group<kExactShape ? 1 : 0>(w, g, cur, xr_cur, chains ? g.chain_groups[k] : g.level_groups[k], lane,
                        tr ? pp.trace + 600 + 8 * (chains ? k - k0 : l) : nullptr, cache_shape ? &t.shape : nullptr,
                        nullptr, scratch);
            __syncwarp();
          }
        }
        grid_sync(pp.bar, target);
        mark();
      }
    }
  }
}

template <int TP>
void launch_tiles(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp, int* singular_counter,
                  unsigned long long* err, cudaStream_t st) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_rod_sweep<TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(Tile<TP>));
  (void)attr;  // a failure surfaces as a launch error
  const int has_ext = c.ext_cap > 0 ? 1 : 0;
  const int blocks = (w.V + TP - 3) / (TP - 2);
  launch_kernel(k_rod_sweep<TP>, blocks, 32 * warps_for<TP>(), sizeof(Tile<TP>), st, sp.pdl != 0, w, c, X, Y, sp, singular_counter,
                err, has_ext);
}

constexpr int kPersistTP = 32;

}  // namespace

void launch_rod_sweep(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp,
                      int* singular_counter, unsigned long long* err, cudaStream_t st) {
  // 64-wide tiles once they fill every SM twice over (148 SMs x 2 x 62 slots).
  if (w.V >= 2 * 148 * 62)
    launch_tiles<64>(w, c, X, Y, sp, singular_counter, err, st);
  else
    launch_tiles<32>(w, c, X, Y, sp, singular_counter, err, st);
}

int persistent_aux_ctas(const World& w) {
  // the SMs the tiles leave idle (one CTA per SM), at least 2 to be worth it, at most 32
  const int tiles = (w.V + kPersistTP - 3) / (kPersistTP - 2);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int spare = sms - tiles;
  return spare >= 2 ? (spare > 32 ? 32 : spare) : 0;
}

int persistent_tiles(const World& w) {
  if (w.n_scenes != 1 || w.V <= 0) return 0;
  const int tiles = (w.V + kPersistTP - 3) / (kPersistTP - 2);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(PTile<kPersistTP>);
  for (auto* k : {k_iterate<kPersistTP, false>, k_iterate<kPersistTP, true>})
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 0;
  for (auto* k : {k_iterate<kPersistTP, false>, k_iterate<kPersistTP, true>}) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 32 * (warps_for<kPersistTP>() + 1), smem) != cudaSuccess) return 0;
    per_sm = per_sm == 0 ? n : (n < per_sm ? n : per_sm);
  }
  return tiles <= per_sm * sms ? tiles : 0;
}

void launch_iterate_persistent(const World& w, Collide& c, const Groups& g, const PersistParams& pp, const SweepParams& sp,
                               int* singular_counters, unsigned long long* err, cudaStream_t st) {
  // pp.bar and pp.ext_done must be zero (Solver's fill)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pp.tiles + pp.n_aux);
  cfg.blockDim = dim3(32 * (warps_for<kPersistTP>() + 1));  // + the external-block warp
  cfg.dynamicSmemBytes = sizeof(PTile<kPersistTP>);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (g.exact)
    cudaLaunchKernelEx(&cfg, k_iterate<kPersistTP, true>, w, c, g, pp, sp, singular_counters, err);
  else
    cudaLaunchKernelEx(&cfg, k_iterate<kPersistTP, false>, w, c, g, pp, sp, singular_counters, err);
}

}  // namespace vdev
