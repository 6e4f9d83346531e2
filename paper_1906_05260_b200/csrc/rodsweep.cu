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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "blocks.cuh"
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
  alignas(8) uint8_t act[kTilePos][kKinds];  // per position: one byte per block kind (read as one 64-bit word)
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
      for (int a = 0; a < kKinds; ++a) t.act[i][a] = 0;
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

// One 2D tensor copy (a box of rows x columns of a field-major FP64 array, as encoded in `map`)
// into shared memory at dst (128-byte aligned), completing on the mbarrier `bar`; col: the box's
// first column (slot), even.
__device__ __forceinline__ void tma_rows(void* dst, const CUtensorMap* map, int col, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(0), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of the same box (no shared memory, no completion): cp.async.bulk.prefetch.tensor.
__device__ __forceinline__ void tma_prefetch_rows(const CUtensorMap* map, int col) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(col), "r"(0)
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

    if (k < m && kind < A_BT) {  // element pass of element k (constraints.cpp:302-314), blocks.cuh
      const V3 c0{t.st[T_CX][si], t.st[T_CY][si], t.st[T_CZ][si]}, c1{t.st[T_CX][si + 1], t.st[T_CY][si + 1], t.st[T_CZ][si + 1]};
      const double s0 = t.st[T_S][si], s1 = t.st[T_S][si + 1];
      const double ic0 = t.st[T_IC][si], ic1 = t.st[T_IC][si + 1], is0 = t.st[T_IS][si], is1 = t.st[T_IS][si + 1];
      const V3 it{t.st[T_ITX][si], t.st[T_ITY][si], t.st[T_ITZ][si]};
      const Q4 q{t.st[T_QW][si], t.st[T_QX][si], t.st[T_QY][si], t.st[T_QZ][si]};
      const int lbase = k * ne;
      if (kind == A_SZ && (ek & EK_SZ)) {  // StretchZ (:106-119), dim 3
        const double lam[3] = {t.st[T_LAM + L_SZ0][si], t.st[T_LAM + L_SZ1][si], t.st[T_LAM + L_SZ2][si]};
        double ln[3];
        bool ok = true;
        if (blk::stretch_z(c0, c1, ic0, ic1, it, q, t.st[T_TDOT][si], t.st[T_LEN][si], t.st[T_KSZ][si], lam, h2, beta,
                           R.sz_dc0, R.sz_dc1, R.sz_dt, ln, ok)) {
          t.act[pi][A_SZ] = 1;
          put_lam(L_SZ0, ln[0]);
          put_lam(L_SZ1, ln[1]);
          put_lam(L_SZ2, ln[2]);
          if (owned && !ok) fail(lbase + __popc(ek & (EK_SZ - 1)));
        } else {
          sing();
          keep_lam(L_SZ0, 3);
        }
      }
      if (kind == A_CS && (ek & EK_CS)) {  // CrossSection (:120-129), dim 1
        double ln;
        bool ok = true;
        if (blk::cross_section(s0, s1, t.st[T_SBAR][si], t.st[T_SBAR][si + 1], is0, is1, t.st[T_KCS][si],
                               t.st[T_LAM + L_CS][si], h2, beta, R.cs, ln, ok)) {
          t.act[pi][A_CS] = 1;
          put_lam(L_CS, ln);
          if (owned && !ok) fail(lbase + __popc(ek & (EK_CS - 1)));
        } else {
          sing();
          keep_lam(L_CS, 1);
        }
      }
      if (kind == A_SS && (ek & EK_SS)) {  // SurfaceStretch (:130-138), dim 1
        double ln;
        bool ok = true;
        if (blk::surface_stretch(s0, s1, t.st[T_LEN][si], t.st[T_SGRAD][si], is0, is1, t.st[T_KSS][si],
                                 t.st[T_LAM + L_SS][si], h2, beta, R.ss, ln, ok)) {
          t.act[pi][A_SS] = 1;
          put_lam(L_SS, ln);
          if (owned && !ok) fail(lbase + __popc(ek & (EK_SS - 1)));
        } else {
          sing();
          keep_lam(L_SS, 1);
        }
      }
      if (kind == A_VS && (ek & EK_VS)) {  // VolumeStretch (:169-188), dim 3
        const double lam[3] = {t.st[T_LAM + L_VS0][si], t.st[T_LAM + L_VS1][si], t.st[T_LAM + L_VS2][si]};
        double ln[3];
        bool ok = true;
        if (blk::volume_stretch(c0, c1, s0, s1, t.st[T_SBAR][si], t.st[T_SBAR][si + 1], ic0, ic1, is0, is1, it, q,
                                t.st[T_TDOT][si], t.st[T_LEN0][si], t.st[T_KVS][si], lam, h2, beta, R.vs_dc0, R.vs_dc1,
                                R.vs_ds, R.vs_dt, ln, ok)) {
          t.act[pi][A_VS] = 1;
          put_lam(L_VS0, ln[0]);
          put_lam(L_VS1, ln[1]);
          put_lam(L_VS2, ln[2]);
          if (owned && !ok) fail(lbase + __popc(ek & (EK_VS - 1)));
        } else {
          sing();
          keep_lam(L_VS0, 3);
        }
      }
    }

    if (k >= 1 && k <= m - 1 && kind >= A_BT) {  // vertex pass of vertex k (:315-327), blocks.cuh
      const Q4 qa{t.st[T_QW][si - 1], t.st[T_QX][si - 1], t.st[T_QY][si - 1], t.st[T_QZ][si - 1]};
      const Q4 qb{t.st[T_QW][si], t.st[T_QX][si], t.st[T_QY][si], t.st[T_QZ][si]};
      const double sm = t.st[T_S][si - 1], s0 = t.st[T_S][si], spp = t.st[T_S][si + 1];
      const double is0 = t.st[T_IS][si];
      const V3 ita{t.st[T_ITX][si - 1], t.st[T_ITY][si - 1], t.st[T_ITZ][si - 1]};
      const V3 itb{t.st[T_ITX][si], t.st[T_ITY][si], t.st[T_ITZ][si]};
      const double sbar = t.st[T_SBAR][si];
      const double la = t.st[T_LEN][si - 1], lb = t.st[T_LEN][si];
      const int lbase = m * ne + (k - 1) * nv;
      const blk::VertexFrame vf = blk::vertex_frame(qa, qb, (vk & (VK_BT | VK_VBU | VK_VBV)) != 0);
      if (kind == A_BT && (vk & VK_BT)) {  // BendTwist (:139-155), dim 3
        const V3 darb{t.st[T_DARBX][si - 1], t.st[T_DARBY][si - 1], t.st[T_DARBZ][si - 1]};
        const double lam[3] = {t.st[T_LAM + L_BT0][si], t.st[T_LAM + L_BT1][si], t.st[T_LAM + L_BT2][si]};
        double ln[3];
        bool ok = true;
        if (blk::bend_twist(vf, s0, sbar, is0, ita, itb, la, lb, darb, t.st[T_KBT0][si], t.st[T_KBT2][si], lam,
                            sp.classic, h2, beta, R.bt_ds, R.bt_dta, R.bt_dtb, ln, ok)) {
          t.act[pi][A_BT] = 1;
          put_lam(L_BT0, ln[0]);
          put_lam(L_BT1, ln[1]);
          put_lam(L_BT2, ln[2]);
          if (owned && !ok) fail(lbase + __popc(vk & (VK_BT - 1)));
        } else {
          sing();
          keep_lam(L_BT0, 3);
        }
      }
      if (kind == A_SB && (vk & VK_SB)) {  // SurfaceBending (:156-168), dim 1
        double ln;
        bool ok = true;
        if (blk::surface_bending(sm, s0, spp, la, lb, t.st[T_SLAP][si - 1], t.st[T_IS][si - 1], is0,
                                 t.st[T_IS][si + 1], t.st[T_KSB][si], t.st[T_LAM + L_SB][si], h2, beta, R.sb, ln, ok)) {
          t.act[pi][A_SB] = 1;
          put_lam(L_SB, ln);
          if (owned && !ok) fail(lbase + __popc(vk & (VK_SB - 1)));
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
          const int lf = cc == 0 ? L_VBU : L_VBV;
          double ln;
          bool ok = true;
          if (blk::volume_bend(cc, vf, s0, sbar, is0, ita, itb, la, lb, t.st[T_LEN0][si - 1], t.st[T_LEN0][si],
                               t.st[cc == 0 ? T_DARBX : T_DARBY][si - 1], t.st[T_KVB][si], t.st[T_LAM + lf][si], h2,
                               beta, R.vb_ds[cc], R.vb_dta[cc], R.vb_dtb[cc], ln, ok)) {
            t.act[pi][cc == 0 ? A_VBU : A_VBV] = 1;
            put_lam(lf, ln);
            if (owned && !ok) fail(lbase + __popc(vk & (bit - 1)));
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
    // the activity flags of the three positions, one 64-bit load each (byte = kind): no shared
    // memory round trip per flag on the gather's path (C3: 391.4 -> 386.7 us per step)
    const unsigned long long fa = *reinterpret_cast<const unsigned long long*>(&t.act[pi - 1][0]);
    const unsigned long long fb = *reinterpret_cast<const unsigned long long*>(&t.act[pi][0]);
    const unsigned long long fn = *reinterpret_cast<const unsigned long long*>(&t.act[pi + 1][0]);
    auto on = [](unsigned long long f, int kind) { return ((f >> (8 * kind)) & 0xffu) != 0; };
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
      if (on(fa, A_SZ)) addc(A.sz_dc1);
      if (on(fa, A_CS)) adds(A.cs[1]);
      if (on(fa, A_SS)) adds(A.ss[1]);
      if (on(fa, A_VS)) {
        addc(A.vs_dc1);
        adds(A.vs_ds[1]);
      }
    }
    if (has_el) {
      if (on(fb, A_SZ)) {
        addc(B.sz_dc0);
        addt(B.sz_dt);
      }
      if (on(fb, A_CS)) adds(B.cs[0]);
      if (on(fb, A_SS)) adds(B.ss[0]);
      if (on(fb, A_VS)) {
        addc(B.vs_dc0);
        adds(B.vs_ds[0]);
        addt(B.vs_dt);
      }
    }
    // vertex pass: vertex k-1 (SurfaceBending s_{j+1}), vertex k, vertex k+1
    if (prev_vx && on(fa, A_SB)) adds(A.sb[2]);
    if (has_vx) {
      if (on(fb, A_BT)) {
        if (!sp.classic) adds(B.bt_ds);
        addt(B.bt_dtb);
      }
      if (on(fb, A_SB)) adds(B.sb[1]);
      if (on(fb, A_VBU)) {
        adds(B.vb_ds[0]);
        addt(B.vb_dtb[0]);
      }
      if (on(fb, A_VBV)) {
        adds(B.vb_ds[1]);
        addt(B.vb_dtb[1]);
      }
    }
    if (next_vx) {
      if (on(fn, A_BT)) addt(N.bt_dta);
      if (on(fn, A_SB)) adds(N.sb[0]);
      if (on(fn, A_VBU)) addt(N.vb_dta[0]);
      if (on(fn, A_VBV)) addt(N.vb_dta[1]);
    }
    if (role != 1) {
      ext(p, addc, adds);
      V3 cn{t.st[T_CX][si], t.st[T_CY][si], t.st[T_CZ][si]};
      if (ccnt > 0) cn = cn + csum / static_cast<double>(ccnt);
      double sn = t.st[T_S][si];
      if (scnt > 0) sn = fmax(sn + qdiv(ssum, static_cast<double>(scnt)), kMinScale);
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

// The external blocks touching slot p (incidence entries [e0, e1), block order) from the blocks'
// records (Collide::ext_rec, written by k_ext_solve): pins and half-planes carry their single
// endpoint's correction, contacts their normal and dlambda, from which the endpoint's correction
// is re-formed exactly as ext_block forms it (contact_endpoint) with the entry's frozen alpha /
// beta (Collide::ext_ab, beside the entry). Chunks of 4 entries, software-pipelined: a chunk's
// entries (static for the substep) are loaded while the previous chunk's records are in flight,
// and all loads of a chunk are issued before its first add. `pre`: the first chunk's entries,
// loaded by the caller ahead of time (before waiting for the ext solve). ic, is, rb: the slot's
// inverse weights and rest radius.
struct EntryChunk {
  int it[4];
  double ab[4];
};
__device__ __forceinline__ EntryChunk load_entries(const Collide& c, int q0, int e0, int e1) {
  EntryChunk ch;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int q = q0 + u < e1 ? q0 + u : e0;
    ch.it[u] = c.ext_items[q];
    ch.ab[u] = c.ext_ab[q];
  }
  return ch;
}
template <class AddC, class AddS>
__device__ __forceinline__ void gather_recs(const Collide& c, int e0, int e1, int npins, int nct, double h2, double ic,
                                            double is, double rb, AddC& addc, AddS& adds, EntryChunk nxt) {
  for (int q0 = e0; q0 < e1; q0 += 4) {
    const EntryChunk ch = nxt;
    double2 r01[4], r23[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2* rr = reinterpret_cast<const double2*>(c.ext_rec + 4ll * (ch.it[u] >> 2));
      r01[u] = rr[0];
      r23[u] = rr[1];
    }
    if (q0 + 4 < e1) nxt = load_entries(c, q0 + 4, e0, e1);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (q0 + u >= e1) continue;
      const int b = ch.it[u] >> 2, e = ch.it[u] & 3;
      if (b < npins) {  // soft pin: center only
        if (is_ext_none(r01[u].x)) continue;
        const double d[3] = {r01[u].x, r01[u].y, r23[u].x};
        addc(d);
      } else if (b < npins + nct) {  // contact
        if (is_ext_none(r23[u].y)) continue;
        double o[3], os;
        contact_endpoint(e, ch.ab[u], r01[u].x, r01[u].y, r23[u].x, r23[u].y, h2, ic, is, rb, o, os);
        addc(o);
        adds(os);
      } else {  // half-plane
        if (is_ext_none(r01[u].x)) continue;
        const double d[3] = {r01[u].x, r01[u].y, r23[u].x};
        addc(d);
        adds(r23[u].y);
      }
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
  extern __shared__ __align__(128) unsigned char smem_raw[];
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
  if (kEarlyWait && has_ext) {  // the tile's incidence items, for the gather after the block solves
    const int e0 = c.ext_off[max(start, 0)], e1 = c.ext_off[min(start + kTileOwned, V)];
    const char* lo = reinterpret_cast<const char*>(c.ext_items + e0);
    const char* hi = reinterpret_cast<const char*>(c.ext_items + e1);
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
  const int nct = has_ext ? c.scalars[SC_NCT] : 0;
  gather_apply(t, w, sp, start, Y, has_ext ? w.xrec : nullptr, [&](int p, auto& addc, auto& adds) {
    if (!has_ext) return;
    const int e0 = c.ext_off[p], e1 = c.ext_off[p + 1];
    if (e0 == e1) return;
    const int si = p - start + 2;
    gather_recs(c, e0, e1, sp.n_pins, nct, sp.h2, t.st[T_IC][si], t.st[T_IS][si], w.vstat[RBAR * (long long)w.vpad + p],
                addc, adds, load_entries(c, e0, e0, e1));
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
                                                                      unsigned long long* err,
                                                                      const __grid_constant__ CUtensorMap tm_x0,
                                                                      const __grid_constant__ CUtensorMap tm_x1) {
  constexpr int kWarps = warps_for<TP>();
  extern __shared__ __align__(128) unsigned char smem_raw[];
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
    if (tid == 0) mbar_init(&t.bar);  // the per-sweep tensor copy of the snapshot rows (published by tile_meta)
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
        for (int i = tid; i < kKinds * TP; i += 32 * kWarps) t.act[i / kKinds][i % kKinds] = 0;
      }
      if (tid == 0) {
        t.ent_next = 0;  // published by the __syncthreads below
        // the snapshot rows (CX .. QZ, slots start-2 .. start+31) in ONE tensor copy; the other CTAs'
        // gathers wrote them before the grid barrier (generic proxy): order them before the async read
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        mbar_arrive_expect(&t.bar, static_cast<unsigned>(kStateFields * kTileStage * sizeof(double)));
        tma_rows(&t.st[T_CX][0], (it & 1) ? &tm_x1 : &tm_x0, start - 2, &t.bar);
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");  // the substep's static rows (first sweep)
      mbar_wait(&t.bar, static_cast<unsigned>(it & 1));
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

// ---- warp-per-rod sweep (every rod <= 32 vertices: C4, C5) -----------------------------------
// One warp per rod, lane k = the rod's slot k (vertex k, element k). Each lane loads its slot's
// snapshot, static rows and multipliers straight into registers (coalesced rows), takes what its
// blocks need from the neighbouring lanes by shuffle, solves the element-pass blocks of element k
// and the vertex-pass blocks of vertex k (blocks.cuh: the tile sweep's arithmetic, so the same
// bits), and gathers in the reference's block order (constraints.cpp:509-534): element k-1's and
// element k's results, then vertex k-1's, k's and k+1's — the neighbours' by shuffle — then the
// external blocks through the incidence list. No shared memory, no halo recomputation, no
// block barrier; a lane owns its slot's multipliers, so they are updated in place.
constexpr int kWarpRodsPerCta = 4;

__device__ __forceinline__ double shup(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shdn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ int shup_i(int v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ int shdn_i(int v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// Staged rows of one rod (warp), one 128-byte aligned block per source array (the TMA tensor
// copy's shared-memory destination must be 128-byte aligned): snapshot X, vertex statics, the
// sweep's element statics (EStatField LEN .. ITZ), multipliers. The box starts at an even slot
// (the copy's inner start coordinate must be 16-byte aligned, measured: an odd FP64 start is an
// illegal instruction), base = (vb - 1) rounded down to even (0 for the first rod), and spans 36
// columns: the rod's <= 32 slots and one neighbour each side; columns past the arrays arrive
// zero-filled. `lead` keeps the first rod's column -1 (never used) inside shared memory.
constexpr int kWCols = 36;
struct alignas(128) WarpStage {
  double lead[16];
  alignas(128) double x[kStateFields][kWCols];
  alignas(128) double vs[kVStatFields][kWCols];
  alignas(128) double es[kSweepEStatFields][kWCols];
  alignas(128) double lm[kLamFields][kWCols];
  alignas(8) unsigned long long bar;
};
constexpr unsigned kWarpStageBytes =
    (kStateFields + kVStatFields + kSweepEStatFields + kLamFields) * kWCols * sizeof(double);

// kStaged: the rod's rows are first copied into shared memory by the TMA engine — four 2D tensor
// copies (X, vertex statics, element statics, multipliers) issued by one lane, completing on one
// mbarrier — and every operand, the lane's own and its neighbours', is read from there;
// otherwise each lane loads its own rows and takes the neighbours' by shuffle.
template <int kMinBlocks, bool kStaged, bool kAll = false>
__global__ void __launch_bounds__(32 * kWarpRodsPerCta, kMinBlocks) k_rod_sweep_warp(World w, Collide c, const double* __restrict__ X,
                                                                      double* __restrict__ Y, SweepParams sp,
                                                                      int* singular, unsigned long long* err,
                                                                      int has_ext, const __grid_constant__ CUtensorMap tm_x,
                                                                      const __grid_constant__ CUtensorMap tm_vs,
                                                                      const __grid_constant__ CUtensorMap tm_es,
                                                                      const __grid_constant__ CUtensorMap tm_lm) {
  if (sp.pdl == 1) {  // predecessor wrote X: wait before loading
    pdl_wait();
    pdl_trigger();
  }
  const int r = blockIdx.x * kWarpRodsPerCta + (threadIdx.x >> 5);
  if (r >= w.R) return;  // whole warps only
  const int k = threadIdx.x & 31;
  const int n = w.rod_n[r], m = n - 1, vb = w.rod_vbase[r];
  // kAll (every rod has every kind): the kind tests below are compile-time true (C4: -1.3 %)
  const int ek = kAll ? 15 : w.rod_ekinds[r], vk = kAll ? 15 : w.rod_vkinds[r], bb = w.rod_block_base[r];
  const int ne = __popc(ek), nv = __popc(vk);
  const bool valid = k < n;
  const long long vp = w.vpad;
  const int p = vb + (valid ? k : 0);
  const double h2 = sp.h2, beta = sp.beta;
  const double* L = sp.lam_in;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WarpStage& ws = reinterpret_cast<WarpStage*>(smem_raw)[threadIdx.x >> 5];
  const int base = vb >= 1 ? (vb - 1) & ~1 : 0;
  const int col = vb - base + k;
  if constexpr (kStaged) {
    if (k == 0) {
      mbar_init(&ws.bar);
      mbar_arrive_expect(&ws.bar, kWarpStageBytes);
      tma_rows(&ws.x[0][0], &tm_x, base, &ws.bar);
      tma_rows(&ws.vs[0][0], &tm_vs, base, &ws.bar);
      tma_rows(&ws.es[0][0], &tm_es, base, &ws.bar);
      tma_rows(&ws.lm[0][0], &tm_lm, base, &ws.bar);
      // the rows of rod r + sp.prefetch_rods, which a warp of a later wave takes, into L2: its
      // own tensor copies then hit L2
      const int rf = r + sp.prefetch_rods;
      if (sp.prefetch_rods > 0 && rf < w.R) {
        const int vf = w.rod_vbase[rf];
        const int bf = vf >= 1 ? (vf - 1) & ~1 : 0;
        tma_prefetch_rows(&tm_x, bf);
        tma_prefetch_rows(&tm_vs, bf);
        tma_prefetch_rows(&tm_es, bf);
        tma_prefetch_rows(&tm_lm, bf);
      }
    }
    __syncwarp();
    mbar_wait(&ws.bar, 0);
  }
  // the lane's own value of (array, field) and a neighbour's (d = +-1)
  auto SM = [&](int a, int f, int cc) -> double {
    return a == 0 ? ws.x[f][cc] : a == 1 ? ws.vs[f][cc] : a == 2 ? ws.es[f][cc] : ws.lm[f][cc];
  };
  auto G = [&](int a, int f) -> double {
    if constexpr (kStaged)
      return SM(a, f, col);
    else
      return valid ? (a == 0 ? X : a == 1 ? w.vstat : a == 2 ? w.estat : L)[f * vp + p] : 0.0;
  };
  auto GN = [&](int a, int f, int d) -> double {
    if constexpr (kStaged)
      return SM(a, f, col + d);
    else
      return d > 0 ? shdn(G(a, f)) : shup(G(a, f));
  };
  int nsing = 0;
  unsigned long long bad = kNoError;
  auto fail = [&](int local) { bad = umin64(bad, err_code(sp.substep, ERR_SWEEP, sp.iter, bb + local)); };
  auto sing = [&]() {
    ++nsing;
    if (sp.scene_singular) atomicAdd(&sp.scene_singular[w.rod_scene[r]], 1);
  };
  auto put_lam = [&](int f, double v) { sp.lam_out[f * vp + p] = v; };
  // The gather sums (constraints.cpp:509-534) are built as the blocks are solved, kind by kind,
  // keeping the reference's order: the three accumulators are independent, and within each the
  // terms go element k-1, element k, vertex k-1, vertex k, vertex k+1 — a term that must wait for
  // a later one is held in a register meanwhile. So only a few results are alive at a time.
  V3 csum{0, 0, 0}, tsum{0, 0, 0};
  double ssum = 0.0;
  int ccnt = 0, scnt = 0, tcnt = 0;
  auto addc = [&](const double* d) {
    csum = csum + V3{d[0], d[1], d[2]};
    ++ccnt;
  };
  auto adds = [&](double d) {
    ssum += d;
    ++scnt;
  };
  auto addt = [&](const double* d) {
    tsum = tsum + V3{d[0], d[1], d[2]};
    ++tcnt;
  };
  const bool el = valid && k < m;         // element k exists
  const bool pel = valid && k >= 1;       // element k-1 exists
  // ---- this slot's snapshot ----
  const V3 c0{G(0, CX), G(0, CY), G(0, CZ)};
  const double s0 = G(0, S);
  const Q4 q{G(0, QW), G(0, QX), G(0, QY), G(0, QZ)};
  const double sbar = G(1, SBAR), is0 = G(1, IS);
  const V3 it{G(2, ITX), G(2, ITY), G(2, ITZ)};
  const double len = G(2, LEN);

  // ---- element pass of element k (constraints.cpp:302-314) ----
  double b_sz[3] = {0, 0, 0}, b_vs[3] = {0, 0, 0}, b_cs = 0.0, b_ss = 0.0, b_vsds = 0.0;  // element k's c0 / s0 terms
  int bact = 0;
  {
    const double ic0 = G(1, IC);
    const V3 c1{GN(0, CX, 1), GN(0, CY, 1), GN(0, CZ, 1)};
    const double s1 = GN(0, S, 1), ic1 = GN(1, IC, 1), is1 = GN(1, IS, 1), sbar1 = GN(1, SBAR, 1);
    const int lbase = k * ne;
    if (ek & EK_SZ) {  // StretchZ (:106-119)
      double dc1[3] = {0, 0, 0}, dt[3];
      int act = 0;
      if (el) {
        const double lam[3] = {G(3, L_SZ0), G(3, L_SZ1), G(3, L_SZ2)};
        double ln[3];
        bool ok = true;
        if (blk::stretch_z(c0, c1, ic0, ic1, it, q, G(2, TDOT), len, G(2, KSZ), lam, h2, beta, b_sz, dc1,
                           dt, ln, ok)) {
          act = 1;
          put_lam(L_SZ0, ln[0]);
          put_lam(L_SZ1, ln[1]);
          put_lam(L_SZ2, ln[2]);
          addt(dt);
          if (!ok) fail(lbase + __popc(ek & (EK_SZ - 1)));
        } else {
          sing();
          put_lam(L_SZ0, lam[0]);
          put_lam(L_SZ1, lam[1]);
          put_lam(L_SZ2, lam[2]);
        }
      }
      bact |= act << A_SZ;
      const double a[3] = {shup(dc1[0]), shup(dc1[1]), shup(dc1[2])};
      const int pa = shup_i(act);
      if (pel && pa) addc(a);
    }
    if (ek & EK_CS) {  // CrossSection (:120-129)
      double ds[2] = {0, 0};
      int act = 0;
      if (el) {
        const double lam = G(3, L_CS);
        double ln;
        bool ok = true;
        if (blk::cross_section(s0, s1, sbar, sbar1, is0, is1, G(2, KCS), lam, h2, beta, ds, ln, ok)) {
          act = 1;
          put_lam(L_CS, ln);
          if (!ok) fail(lbase + __popc(ek & (EK_CS - 1)));
        } else {
          sing();
          put_lam(L_CS, lam);
        }
      }
      b_cs = ds[0];
      bact |= act << A_CS;
      const double a = shup(ds[1]);
      const int pa = shup_i(act);
      if (pel && pa) adds(a);
    }
    if (ek & EK_SS) {  // SurfaceStretch (:130-138)
      double ds[2] = {0, 0};
      int act = 0;
      if (el) {
        const double lam = G(3, L_SS);
        double ln;
        bool ok = true;
        if (blk::surface_stretch(s0, s1, len, G(2, SGRAD), is0, is1, G(2, KSS), lam, h2, beta, ds, ln,
                                 ok)) {
          act = 1;
          put_lam(L_SS, ln);
          if (!ok) fail(lbase + __popc(ek & (EK_SS - 1)));
        } else {
          sing();
          put_lam(L_SS, lam);
        }
      }
      b_ss = ds[0];
      bact |= act << A_SS;
      const double a = shup(ds[1]);
      const int pa = shup_i(act);
      if (pel && pa) adds(a);
    }
    if (ek & EK_VS) {  // VolumeStretch (:169-188)
      double dc1[3] = {0, 0, 0}, ds[2] = {0, 0}, dt[3];
      int act = 0;
      if (el) {
        const double lam[3] = {G(3, L_VS0), G(3, L_VS1), G(3, L_VS2)};
        double ln[3];
        bool ok = true;
        if (blk::volume_stretch(c0, c1, s0, s1, sbar, sbar1, ic0, ic1, is0, is1, it, q, G(2, TDOT),
                                G(2, LEN0), G(2, KVS), lam, h2, beta, b_vs, dc1, ds, dt, ln, ok)) {
          act = 1;
          put_lam(L_VS0, ln[0]);
          put_lam(L_VS1, ln[1]);
          put_lam(L_VS2, ln[2]);
          addt(dt);
          if (!ok) fail(lbase + __popc(ek & (EK_VS - 1)));
        } else {
          sing();
          put_lam(L_VS0, lam[0]);
          put_lam(L_VS1, lam[1]);
          put_lam(L_VS2, lam[2]);
        }
      }
      b_vsds = ds[0];
      bact |= act << A_VS;
      const double a[3] = {shup(dc1[0]), shup(dc1[1]), shup(dc1[2])};
      const double ads = shup(ds[1]);
      const int pa = shup_i(act);
      if (pel && pa) {
        addc(a);
        adds(ads);
      }
    }
  }
  // element k's own terms (c0 / s0 side) after all of element k-1's
  if (el) {
    if (bact & (1 << A_SZ)) addc(b_sz);
    if (bact & (1 << A_CS)) adds(b_cs);
    if (bact & (1 << A_SS)) adds(b_ss);
    if (bact & (1 << A_VS)) {
      addc(b_vs);
      adds(b_vsds);
    }
  }

  // ---- vertex pass of interior vertex k (constraints.cpp:315-327) ----
  {
    const bool vx = valid && k >= 1 && k <= m - 1;  // vertex k is interior
    const bool nvx = valid && k + 1 <= m - 1;        // vertex k+1 is interior
    const Q4 qa{GN(0, QW, -1), GN(0, QX, -1), GN(0, QY, -1), GN(0, QZ, -1)};
    const V3 ita{GN(2, ITX, -1), GN(2, ITY, -1), GN(2, ITZ, -1)};
    const double la = GN(2, LEN, -1);
    const double lb = len;
    const int lbase = m * ne + (k - 1) * nv;
    const blk::VertexFrame vf = blk::vertex_frame(qa, q, (vk & (VK_BT | VK_VBU | VK_VBV)) != 0);
    double bt_ds = 0.0;
    int bt_act = 0;
    double n_bta[3] = {0, 0, 0};
    int n_bt = 0;
    if (vk & VK_BT) {  // BendTwist (:139-155)
      const V3 darb_a{GN(2, DARBX, -1), GN(2, DARBY, -1), GN(2, DARBZ, -1)};
      double dta[3] = {0, 0, 0}, dtb[3];
      if (vx) {
        const double lam[3] = {G(3, L_BT0), G(3, L_BT1), G(3, L_BT2)};
        double ln[3];
        bool ok = true;
        if (blk::bend_twist(vf, s0, sbar, is0, ita, it, la, lb, darb_a, G(2, KBT0), G(2, KBT2), lam,
                            sp.classic, h2, beta, bt_ds, dta, dtb, ln, ok)) {
          bt_act = 1;
          put_lam(L_BT0, ln[0]);
          put_lam(L_BT1, ln[1]);
          put_lam(L_BT2, ln[2]);
          addt(dtb);
          if (!ok) fail(lbase + __popc(vk & (VK_BT - 1)));
        } else {
          sing();
          put_lam(L_BT0, lam[0]);
          put_lam(L_BT1, lam[1]);
          put_lam(L_BT2, lam[2]);
        }
      }
      n_bta[0] = shdn(dta[0]);
      n_bta[1] = shdn(dta[1]);
      n_bta[2] = shdn(dta[2]);
      n_bt = shdn_i(bt_act);
    }
    double sb_mid = 0.0, n_sb0 = 0.0;
    int sb_act = 0, n_sb = 0;
    {
      double a_sb2 = 0.0;
      int p_sb = 0;
      if (vk & VK_SB) {  // SurfaceBending (:156-168)
        const double sm = GN(0, S, -1), ism = GN(1, IS, -1), slap_a = GN(2, SLAP, -1);
        const double spp = GN(0, S, 1), isp = GN(1, IS, 1);
        double ds[3] = {0, 0, 0};
        if (vx) {
          const double lam = G(3, L_SB);
          double ln;
          bool ok = true;
          if (blk::surface_bending(sm, s0, spp, la, lb, slap_a, ism, is0, isp, G(2, KSB), lam, h2, beta, ds, ln,
                                   ok)) {
            sb_act = 1;
            put_lam(L_SB, ln);
            if (!ok) fail(lbase + __popc(vk & (VK_SB - 1)));
          } else {
            sing();
            put_lam(L_SB, lam);
          }
        }
        sb_mid = ds[1];
        a_sb2 = shup(ds[2]);
        p_sb = shup_i(sb_act);
        n_sb0 = shdn(ds[0]);
        n_sb = shdn_i(sb_act);
      }
      // scale terms: vertex k-1's s_{j+1}, then vertex k's (BendTwist, SurfaceBending; the volume
      // bends follow below)
      if (valid && k - 1 >= 1 && p_sb) adds(a_sb2);
      if (vx && bt_act && !sp.classic) adds(bt_ds);
      if (vx && sb_act) adds(sb_mid);
    }
    double n_vb[2][3] = {{0, 0, 0}, {0, 0, 0}};
    int n_vba[2] = {0, 0};
    if (vk & (VK_VBU | VK_VBV)) {  // VolumeBendU / V (:189-214)
      const double la0 = GN(2, LEN0, -1), lb0 = G(2, LEN0);
      const double dax = GN(2, DARBX, -1), day = GN(2, DARBY, -1);
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int bit = cc == 0 ? VK_VBU : VK_VBV;
        if (!(vk & bit)) continue;
        const int lf = cc == 0 ? L_VBU : L_VBV;
        double ds = 0.0, dta[3] = {0, 0, 0}, dtb[3];
        int act = 0;
        if (vx) {
          const double lam = G(3, lf);
          double ln;
          bool ok = true;
          if (blk::volume_bend(cc, vf, s0, sbar, is0, ita, it, la, lb, la0, lb0, cc == 0 ? dax : day,
                               G(2, KVB), lam, h2, beta, ds, dta, dtb, ln, ok)) {
            act = 1;
            put_lam(lf, ln);
            adds(ds);
            addt(dtb);
            if (!ok) fail(lbase + __popc(vk & (bit - 1)));
          } else {
            sing();
            put_lam(lf, lam);
          }
        }
        n_vb[cc][0] = shdn(dta[0]);
        n_vb[cc][1] = shdn(dta[1]);
        n_vb[cc][2] = shdn(dta[2]);
        n_vba[cc] = shdn_i(act);
      }
    }
    // vertex k+1's terms last
    if (nvx) {
      if (n_bt) addt(n_bta);
      if (n_sb) adds(n_sb0);
      if (n_vba[0]) addt(n_vb[0]);
      if (n_vba[1]) addt(n_vb[1]);
    }
  }
  // singular / error counts of this warp's blocks
  if (__any_sync(0xffffffffu, nsing != 0 || bad != kNoError)) {
    for (int o = 16; o > 0; o >>= 1) {
      nsing += __shfl_down_sync(0xffffffffu, nsing, o);
      bad = umin64(bad, __shfl_down_sync(0xffffffffu, bad, o));
    }
    if (k == 0) {
      if (nsing) atomicAdd(singular, nsing);
      if (bad != kNoError) atomicMin(err, bad);
    }
  }
  // the slot's incidence entries are static for the substep: the first chunk is loaded before
  // waiting for this iteration's ext solve (the predecessor), which writes the block records and
  // reads the slot records this sweep rewrites
  int e0 = 0, e1 = 0;
  EntryChunk first{};
  if (has_ext && valid) {
    e0 = c.ext_off[p];
    e1 = c.ext_off[p + 1];
    if (e0 < e1) first = load_entries(c, e0, e0, e1);
  }
  if (sp.pdl == 2) {
    pdl_wait();
    pdl_trigger();
  }
  if (!valid) return;
  if (e0 < e1) gather_recs(c, e0, e1, sp.n_pins, c.scalars[SC_NCT], h2, G(1, IC), is0, G(1, RBAR), addc, adds, first);
  // ---- apply (constraints.cpp:537-554) ----
  V3 cn = c0;
  if (ccnt > 0) cn = cn + csum / static_cast<double>(ccnt);
  double sn = s0;
  if (scnt > 0) sn = fmax(sn + qdiv(ssum, static_cast<double>(scnt)), kMinScale);
  Y[CX * vp + p] = cn.x;
  Y[CY * vp + p] = cn.y;
  Y[CZ * vp + p] = cn.z;
  Y[S * vp + p] = sn;
  if (has_ext) {
    double2* xr = reinterpret_cast<double2*>(w.xrec + 8ll * p);
    xr[0] = make_double2(cn.x, cn.y);
    xr[1] = make_double2(cn.z, sn);
  }
  Q4 qn = q;
  if (k < m && tcnt > 0) qn = apply_increment(qn, tsum / static_cast<double>(tcnt));
  Y[QW * vp + p] = qn.w;
  Y[QX * vp + p] = qn.x;
  Y[QY * vp + p] = qn.y;
  Y[QZ * vp + p] = qn.z;
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

// Tensor map of the first `rows` fields of a field-major FP64 array (row stride vpad doubles):
// boxes of rows x cols, zero fill out of range. Encoded once per (array, rows, vpad) through the
// driver entry point (no libcuda link), then passed by value as a __grid_constant__ parameter.
CUtensorMap rows_map(const double* base, int rows, int vpad, int cols = kWCols) {
  static const auto encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr)
      throw std::runtime_error("CUDA error: cuTensorMapEncodeTiled is unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(static_cast<const void*>(base), rows, vpad, cols);
  const auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(vpad), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(vpad) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(cols), static_cast<cuuint32_t>(rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("CUDA error: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  cache.emplace(key, map);
  return map;
}

}  // namespace

void launch_rod_sweep(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp,
                      int* singular_counter, unsigned long long* err, cudaStream_t st) {
  // every rod fits a warp: one warp per rod (VROD_ROD_WARP=0 forces the tiles, for A/B runs)
  const bool warp_ok = !(std::getenv("VROD_ROD_WARP") && std::getenv("VROD_ROD_WARP")[0] == '0');
  if (warp_ok && w.max_rod_n <= 32 && w.R > 0) {
    const int has_ext = c.ext_cap > 0 ? 1 : 0;
    // VROD_WARP_TMA=0: operands by per-lane loads and shuffles instead of the staged rows (A/B)
    const bool staged = !(std::getenv("VROD_WARP_TMA") && std::getenv("VROD_WARP_TMA")[0] == '0');
    // 3 CTAs per SM (168 registers, no spills) measured fastest at C4 with the tensor staging
    const int minb = std::getenv("VROD_WARP_MINB") ? std::atoi(std::getenv("VROD_WARP_MINB")) : 3;
    const size_t smem = staged ? kWarpRodsPerCta * sizeof(WarpStage) : 0;
    // L2 prefetch distance in rods (VROD_WARP_PREFETCH, 0 = off). Measured at C4: 444 (148 x 3)
    // sweep 3.33 -> 3.29 ms per substep; 222 / 888 / 1776 / 3552 less; also prefetching the
    // incidence entries is slower (lane 0's extra offset loads)
    SweepParams spp = sp;
    spp.prefetch_rods = std::getenv("VROD_WARP_PREFETCH") ? std::atoi(std::getenv("VROD_WARP_PREFETCH")) : 444;
    const CUtensorMap tx = rows_map(X, kStateFields, w.vpad), tv = rows_map(w.vstat, kVStatFields, w.vpad),
                      te = rows_map(w.estat, kSweepEStatFields, w.vpad), tl = rows_map(sp.lam_in, kLamFields, w.vpad);
    static const bool attrs = [] {
      for (auto* k : {k_rod_sweep_warp<2, true>, k_rod_sweep_warp<3, true>, k_rod_sweep_warp<4, true>,
                      k_rod_sweep_warp<3, true, true>})
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kWarpRodsPerCta * sizeof(WarpStage));
      return true;
    }();
    (void)attrs;
    auto* kern = staged ? (minb <= 2 ? k_rod_sweep_warp<2, true> : minb == 3 ? k_rod_sweep_warp<3, true> : k_rod_sweep_warp<4, true>)
                        : (minb <= 2 ? k_rod_sweep_warp<2, false> : minb == 3 ? k_rod_sweep_warp<3, false> : k_rod_sweep_warp<4, false>);
    if (staged && minb == 3 && w.all_kinds) kern = k_rod_sweep_warp<3, true, true>;
    launch_kernel(kern, (w.R + kWarpRodsPerCta - 1) / kWarpRodsPerCta, 32 * kWarpRodsPerCta, smem, st, sp.pdl != 0, w,
                  c, X, Y, spp, singular_counter, err, has_ext, tx, tv, te, tl);
    return;
  }
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
  const CUtensorMap t0 = rows_map(pp.X, kStateFields, w.vpad, kPersistTP + 2),
                    t1 = rows_map(pp.Y, kStateFields, w.vpad, kPersistTP + 2);
  if (g.exact)
    cudaLaunchKernelEx(&cfg, k_iterate<kPersistTP, true>, w, c, g, pp, sp, singular_counters, err, t0, t1);
  else
    cudaLaunchKernelEx(&cfg, k_iterate<kPersistTP, false>, w, c, g, pp, sp, singular_counters, err, t0, t1);
}

}  // namespace vdev
