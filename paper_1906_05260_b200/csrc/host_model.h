// Host-side scene model and setup path of the product.
//
// Holds what the C-ABI scene builder receives (the reference's vrod::Scene, scene.h:109-126),
// validates it with the reference's checks and messages (Scene::validate, scene.cpp:63-157),
// and derives everything the device needs once: DofLayout (layout.cpp:7-73) in slot form,
// per-rod emitted constraint kinds and block bases (constraints.cpp:282-329), stiffness,
// shape-matching groups with their rest data (bundling.cpp:17-48) and a dependency-level
// schedule, and the per-substep animation inputs (pin motions, activation amounts, bone
// poses — scene.cpp:22-61) that the host evaluates exactly as the reference does.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "vmath.cuh"

namespace vhost {

using vm::Q4;
using vm::V3;

struct SimulationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
inline void require(bool cond, const std::string& what) {
  if (!cond) throw std::invalid_argument(what);
}
inline void require_index(bool cond, const std::string& what) {
  if (!cond) throw std::out_of_range(what);
}
inline void require_index(int i, int count, const std::string& what) {
  if (i < 0 || i >= count) throw std::out_of_range(what + " out of range");
}

constexpr double kInf = std::numeric_limits<double>::infinity();

struct Material {
  double sx = 1e4, sy = 1e4, sz = 1e4, bx = 1e3, by = 1e3, bz = 0.0, vol = 1e6, rho = 1000.0;
};
struct Settings {
  double dt = 1.0 / 60.0;
  int iterations = 20, substeps = 1;
  double beta = 0.75;
  V3 g{0, 0, -9.81};
  int dich = 10, sm_period = 2;
  double contact_k = kInf, damping = 0.0;
  bool deterministic = false;
  int scale_mode = 0;
};
struct RodData {
  int n = 0;
  // rest (RodRestPose)
  std::vector<V3> rc;
  std::vector<double> rs, r, len, len0;
  std::vector<Q4> rq;
  std::vector<V3> darb;
  std::vector<double> tdot, sgrad, slap;
  // state (RodState)
  std::vector<V3> c, cv, av;
  std::vector<double> s, sv;
  std::vector<Q4> q;
  std::vector<uint8_t> pinned;
  int material = 0, group = -1;
  bool self_collide = false;
  std::vector<int> bones;
  std::vector<double> bone_w;  // n x bones
};
struct PillData {
  V3 c0{0, 0, 0}, c1{0, 0, 0};
  double r0 = 0, r1 = 0;
  int rod = -1, element = -1, group = -1;
  bool self_collide = false;
};
struct Key {
  double t;
  V3 p;
  Q4 r;
};
struct BoneData {
  std::vector<Key> keys;
  V3 position_at(double t) const;  // scene.cpp:22-34
  Q4 rotation_at(double t) const;  // scene.cpp:36-48 (Eigen slerp)
};
struct KinPill {
  PillData pill;
  int bone = -1;
};
struct PinMotion {
  int rod, vertex;
  V3 start, target;
  double t0, t1;
  V3 position_at(double t) const;  // scene.cpp:50-55
};
struct SoftPin {
  int rod, vertex;
  V3 target;
  double k;
};
struct Activation {
  int rod;
  double factor, t_start, t_end;
  int first, last;
  double amount_at(double t) const;  // scene.cpp:57-61
};

struct SceneData {
  std::vector<RodData> rods;
  std::vector<Material> materials;
  std::vector<std::pair<V3, double>> planes;
  std::vector<KinPill> kpills;
  std::vector<BoneData> bones;
  std::vector<std::vector<std::pair<int, int>>> bundles;
  std::vector<PinMotion> pin_motions;
  std::vector<SoftPin> soft_pins;
  std::vector<Activation> activations;
  Settings settings;

  void validate() const;  // Scene::validate, scene.cpp:63-157
};

// A batch of independent scenes merged into one world (BASELINE config C5): rods, materials,
// planes, kinematic pills, bones, bundles, pins and activations concatenated scene by scene,
// indices re-based. Each scene is validated on its own (same messages); all must share one
// SolverSettings. Block order inside the merged world keeps every slot's reference order:
// elastic (rods ascending), then pins, contacts and half-planes, each scene-major.
struct BatchLayout {
  int scenes = 1;
  std::vector<int> rod_base;     // scenes + 1
  std::vector<int> plane_scene;  // per plane
  std::vector<int> kpill_scene;  // per kinematic pill
};
SceneData merge_scenes(const std::vector<const SceneData*>& scenes, BatchLayout& layout);

// make_rest_pose, rod.cpp:60-112 (fills the rest fields of `rod`).
void make_rest_pose(RodData& rod, const std::vector<V3>& centers, const std::vector<double>& radii,
                    const std::vector<double>& scales);
void validate_rest(const RodData& rod);  // RodRestPose::validate, rod.cpp:15-34

// Everything derived once at Solver construction.
struct Setup {
  int R = 0, V = 0, E = 0, vpad = 0;
  std::vector<int> vbase, ebase, block_base;
  std::vector<uint8_t> ekinds, vkinds;
  int elastic_blocks = 0;
  // shape matching
  struct Group {
    std::vector<int> slot;   // member vertex slot
    std::vector<int> eslot;  // member frame slot (element min(v, m-1))
    std::vector<V3> rc;
    std::vector<double> rs;
    std::vector<vm::M3> rR;
    std::vector<Q4> qR;      // Quat(rest frame matrix)
    V3 rcent{0, 0, 0};
    double denom = 0;
    bool serial_apply = false;
  };
  std::vector<Group> groups;
  std::vector<int> group_level;
  int levels = 0;
  // Chain schedule of the groups (empty when the frame dependencies are not chains):
  // chain c = chain_groups[chain_off[c] .. chain_off[c+1]), in the reference's group order.
  std::vector<int> chain_off, chain_groups;
  // pin motions after dedupe (last one per vertex wins, like the reference's sequential writes)
  std::vector<int> pin_motion_ids;
};

Setup build_setup(const SceneData& s);

int element_kinds(const Material& m, bool scale_kinds);
int vertex_kinds(const Material& m, bool scale_kinds);
int popcount4(int bits);

}  // namespace vhost
