// Device-resident data layout of one solver world (build target:
// SoA FP64 by global slot).
//
// Index space: ONE slot index for vertices and elements. Rod r owns slots
// [vbase[r], vbase[r] + n_r); slot vbase[r]+k holds vertex k (center, scale) and, for
// k < n_r - 1, element k (frame) — the last slot of each rod carries no element. This is the
// reference's DofLayout (layout.h:17-41) with element slots padded by one per rod, so every
// per-vertex and per-element array is read with the same coalesced index and a rod's stencil
// (elements k-1,k / vertices k-1..k+1) is a contiguous window.
//
// Every field is a separate FP64 array of `vpad` doubles ("field f of array A" = A + f*vpad),
// i.e. structure-of-arrays with 256-byte aligned rows.
#pragma once

#include <cstdint>

namespace vdev {

// Dynamic state fields (two ping-pong copies + the pre-predict snapshot).
enum StateField : int { CX = 0, CY, CZ, S, QW, QX, QY, QZ, kStateFields };
// Velocity fields.
enum VelField : int { VX = 0, VY, VZ, VS, WX, WY, WZ, kVelFields };
// Static per-vertex fields.
enum VStatField : int { RBAR = 0, SBAR, IC, IS, kVStatFields };
// Per-element rest fields (element k of a rod at its slot). DARB*/SLAP are the rest Darboux
// vector / scale laplacian of interior vertex k+1 (reference index j-1 = k).
// The rows a sweep reads come first (LEN .. ITZ, kSweepEStatFields), so the warp-per-rod sweep
// stages them with ONE 2D tensor copy per rod (rodsweep.cu).
enum EStatField : int {
  LEN = 0, LEN0, TDOT, SGRAD, SLAP, DARBX, DARBY, DARBZ,
  // Stiffness rows hold the INVERSE stiffness inverse_stiffness(k) (constraints.cpp:274-278),
  // computed once at setup / on activation refresh instead of once per block per sweep.
  KSZ, KCS, KSS, KVS,     // element-pass (StretchZ/VolumeStretch are Constant)
  KBT0, KBT1, KBT2, KSB, KVB,  // vertex-pass of vertex k (VolumeBendU == V; KBT1 == KBT0 always)
  ITX, ITY, ITZ,          // inverse theta weights (refreshed every substep)
  kSweepEStatFields,
  RQW = kSweepEStatFields, RQX, RQY, RQZ,
  A2E,      // pi * rmid^2
  A4EP,     // 0.25 * pi * pow(rmid, 4)   (refresh_stiffness form, constraints.cpp:352)
  A4VP,     // 0.25 * pi * pow(r_k, 4) of vertex k (constraints.cpp:357,363)
  TWB,                    // theta weight base rho*s_mid^2*pi*r^4*l0 (weights = 0.25,0.25,0.5 x base)
  kEStatFields
};
// Elastic multipliers per slot: element pass then vertex pass (constraints.cpp:302-327).
enum LamField : int {
  L_SZ0 = 0, L_SZ1, L_SZ2, L_CS, L_SS, L_VS0, L_VS1, L_VS2,
  L_BT0, L_BT1, L_BT2, L_SB, L_VBU, L_VBV, kLamFields
};

// Element-pass kind bits (ekinds) and vertex-pass kind bits (vkinds), per rod.
enum : uint8_t { EK_SZ = 1, EK_CS = 2, EK_SS = 4, EK_VS = 8 };
enum : uint8_t { VK_BT = 1, VK_SB = 2, VK_VBU = 4, VK_VBV = 8 };

// Error word: min over (substep, stage, iteration, index); decoded on the host.
enum ErrStage : uint64_t { ERR_PREDICT = 0, ERR_BROAD = 1, ERR_SWEEP = 2, ERR_CAPACITY = 3 };
__host__ __device__ inline uint64_t err_code(uint64_t substep, uint64_t stage, uint64_t iter, uint64_t idx) {
  return (substep << 56) | (stage << 52) | ((iter & 0xfffff) << 32) | (idx & 0xffffffffull);
}
constexpr uint64_t kNoError = ~0ull;

struct StepAccum {  // device-side StepReport accumulation (solver.cpp:363-388)
  double residuals[8];
  double max_penetration;
  int contact_count;
  int broad_pairs;
  int skipped_singular;
  int pad;
  unsigned long long error;
  long long max_candidates;  // capacity diagnostics
  long long max_contacts;
};

// Per-scene StepReport accumulation when the world is a batch of independent scenes
// (BASELINE config C5). Same semantics as StepAccum, per scene.
struct SceneAcc {
  double residuals[8];
  double max_penetration;
  int contact_count;
  int broad_pairs;
  int skipped_singular;
  int pad;
};

struct World {
  // Batch of independent scenes: rods of scene s are [scene_rod_base[s], scene_rod_base[s+1]),
  // their slots contiguous [scene_vbase[s], scene_vbase[s+1]). n_scenes == 1: arrays null.
  int n_scenes = 1;
  int* rod_scene = nullptr;
  int* scene_vbase = nullptr;
  SceneAcc* scene_acc = nullptr;
  int R = 0;          // rods
  int V = 0;          // slots (= total vertices)
  int vpad = 0;       // field stride
  int E = 0;          // compact element count (= rod pills)
  int K = 0;          // kinematic pills
  int P = 0;          // pills = E + K
  int classic = 0;    // ScaleMode::kPostStepLengthRatio
  int max_rod_n = 0;  // longest rod (vertices): <= 32 selects the warp-per-rod sweep
  int all_kinds = 0;  // every rod has all 8 block kinds: the warp sweep's kind tests fold away
  int has_bones = 0;
  int has_loads = 0;

  // per rod
  int* rod_vbase = nullptr;
  int* rod_n = nullptr;
  int* rod_block_base = nullptr;
  int* rod_material = nullptr;
  int* rod_group = nullptr;
  uint8_t* rod_self = nullptr;
  uint8_t* rod_ekinds = nullptr;
  uint8_t* rod_vkinds = nullptr;
  int* rod_bone_off = nullptr;   // CSR into bone ids/weights (R+1)
  int* rod_bones = nullptr;
  double* bone_w = nullptr;      // per slot: bone_count of its rod weights, at slot_bw_off
  int* slot_bw_off = nullptr;
  uint8_t* load_flags = nullptr; // per rod: bit0 force, bit1 torque, bit2 scale load

  // per slot
  int* slot_rod = nullptr;
  int* slot_loc = nullptr;
  int* slot_m = nullptr;         // element count of the owning rod
  uint8_t* pinned = nullptr;
  double* vstat = nullptr;       // kVStatFields x vpad
  double* estat = nullptr;       // kEStatFields x vpad
  double* mat = nullptr;         // materials: 8 doubles each (MaterialParams order)

  // state
  double* X = nullptr;           // kStateFields x vpad, canonical between steps
  double* Y = nullptr;           // ping-pong partner
  double* prev = nullptr;        // snapshot after animate
  double* vel = nullptr;         // kVelFields x vpad
  double* lam = nullptr;         // kLamFields x vpad
  double* loads = nullptr;       // 3 force + 3 torque + 1 scale load per slot (7 x vpad)
  // AoS mirror of what the external blocks read per slot, 64 B records: c xyz, s (current
  // iterate; written by predict, the rod sweep and shape matching), rbar, 1/w_c, 1/w_s (static).
  // One record = two 32-byte sectors, instead of seven scattered SoA sectors per endpoint.
  double* xrec = nullptr;
};

}  // namespace vdev
