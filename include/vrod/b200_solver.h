// vrod::b200::Solver — the drop-in C++ facade over the B200 C-ABI (include/vrod_capi.h).
//
// A reference caller (proj/tools/vrod_main.cpp, proj/core/src/metrics.cpp, the doctest suites)
// switches from the CPU solver to the B200 one by naming vrod::b200::Solver where it named
// vrod::Solver (solver.h:54-115) and linking libvrod_b200.so. Everything the caller sees keeps the
// reference's types (Scene, StepReport, DofLayout, ExternalLoads, Pill, PillTransform,
// BundleGroup) and the reference's exceptions with its exact messages.
//
// Header-only: it needs the reference's public headers (proj/core/include) for those types, and
// make_bundle_group (bundling.h:38) from the reference core library for bundles() — setup-time
// host data; nothing on the step() path runs on the CPU.
//
// State ownership: the device is authoritative. scene() returns a host mirror of the live
// state, refreshed lazily after each step (one vrod_solver_get_state); edits made through the
// mutable scene() are detected at the next step() (compared with what was pulled) and written
// back with vrod_solver_set_state — the reference's "write scene().rods[r].state between steps"
// (SURVEY.md §7 hard part 5). Activation-refreshed rest data (rod.cpp:164-176) is mirrored too.
#pragma once

#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vrod/bundling.h"
#include "vrod/layout.h"
#include "vrod/scene.h"
#include "vrod/skinning.h"
#include "vrod/solver.h"  // StepReport, PhaseTimings, ExternalLoads (shared types)
#include "vrod_capi.h"

namespace vrod::b200 {

/// Status code -> the reference's exception type with its message (types.h:25-28,67-77).
inline void check(int status) {
  if (status == VROD_OK) return;
  const std::string msg = vrod_last_error();
  switch (status) {
    case VROD_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VROD_OUT_OF_RANGE: throw std::out_of_range(msg);
    case VROD_SIMULATION_ERROR: throw vrod::SimulationError(msg);
    default: throw std::runtime_error(msg);  // VROD_DEVICE_ERROR / runtime: no CPU fallback
  }
}

namespace detail {

inline void put3(double* p, const Vec3& v) {
  p[0] = v.x();
  p[1] = v.y();
  p[2] = v.z();
}
inline void putq(double* p, const Quat& q) {  // C-ABI order w, x, y, z
  p[0] = q.w();
  p[1] = q.x();
  p[2] = q.y();
  p[3] = q.z();
}
inline Vec3 get3(const double* p) { return Vec3(p[0], p[1], p[2]); }
inline Quat getq(const double* p) { return Quat(p[0], p[1], p[2], p[3]); }

inline vrod_settings to_c(const SolverSettings& s) {
  vrod_settings c{};
  c.dt = s.dt;
  c.iterations = s.iterations;
  c.substeps = s.substeps;
  c.beta = s.beta;
  put3(c.gravity, s.gravity);
  c.dichotomous_iterations = s.dichotomous_iterations;
  c.shape_match_period = s.shape_match_period;
  c.contact_stiffness = s.contact_stiffness;
  c.velocity_damping = s.velocity_damping;
  c.deterministic = s.deterministic ? 1 : 0;
  c.scale_mode = static_cast<int32_t>(s.scale_mode);
  return c;
}

inline vrod_material to_c(const MaterialParams& m) {
  return vrod_material{m.stretch_x, m.stretch_y, m.stretch_z, m.bend_x, m.bend_y, m.bend_z, m.volume, m.density};
}

inline vrod_pill to_c(const Pill& p) {
  vrod_pill c{};
  put3(c.c0, p.c0);
  put3(c.c1, p.c1);
  c.r0 = p.r0;
  c.r1 = p.r1;
  c.rod = p.rod;
  c.element = p.element;
  c.group = p.group;
  c.self_collide = p.self_collide ? 1 : 0;
  return c;
}

inline Pill from_c(const vrod_pill& c) {
  Pill p;
  p.c0 = get3(c.c0);
  p.c1 = get3(c.c1);
  p.r0 = c.r0;
  p.r1 = c.r1;
  p.rod = c.rod;
  p.element = c.element;
  p.group = c.group;
  p.self_collide = c.self_collide != 0;
  return p;
}

inline PillTransform from_c(const vrod_pill_transform& c) {
  PillTransform t;
  t.center = get3(c.center);
  t.scale = c.scale;
  t.rotation = getq(c.rotation);
  return t;
}

inline StepReport from_c(const vrod_step_report& r) {
  StepReport out;
  out.step = r.step;
  out.time = r.time;
  out.residuals.assign(r.residuals, r.residuals + 8);
  out.max_penetration = r.max_penetration;
  out.contact_count = r.contact_count;
  out.broad_pairs = r.broad_pairs;
  out.skipped_singular = r.skipped_singular;
  out.dof_count = r.dof_count;
  out.timings = PhaseTimings{r.predict_ms, r.broad_ms, r.narrow_ms, r.solve_ms, r.finalize_ms, r.total_ms};
  return out;
}

/// Flat C-ABI copy of one Rod (vrod_rod_desc points into it).
struct RodBuffers {
  std::vector<double> rest_centers, rest_frames, darboux, centers, frames, center_vel, angular_vel, bone_w;
  vrod_rod_desc desc{};

  explicit RodBuffers(const Rod& rod) {
    const RodRestPose& rp = rod.rest;
    const RodState& st = rod.state;
    const int n = rp.vertex_count(), m = rp.element_count();
    rest_centers.resize(3 * rp.centers.size());
    for (std::size_t i = 0; i < rp.centers.size(); ++i) put3(&rest_centers[3 * i], rp.centers[i]);
    rest_frames.resize(4 * rp.frames.size());
    for (std::size_t i = 0; i < rp.frames.size(); ++i) putq(&rest_frames[4 * i], rp.frames[i]);
    darboux.resize(3 * rp.darboux.size());
    for (std::size_t i = 0; i < rp.darboux.size(); ++i) put3(&darboux[3 * i], rp.darboux[i]);
    centers.resize(3 * st.centers.size());
    for (std::size_t i = 0; i < st.centers.size(); ++i) put3(&centers[3 * i], st.centers[i]);
    frames.resize(4 * st.frames.size());
    for (std::size_t i = 0; i < st.frames.size(); ++i) putq(&frames[4 * i], st.frames[i]);
    center_vel.resize(3 * st.center_vel.size());
    for (std::size_t i = 0; i < st.center_vel.size(); ++i) put3(&center_vel[3 * i], st.center_vel[i]);
    angular_vel.resize(3 * st.angular_vel.size());
    for (std::size_t i = 0; i < st.angular_vel.size(); ++i) put3(&angular_vel[3 * i], st.angular_vel[i]);
    for (const auto& row : rod.bone_weights) bone_w.insert(bone_w.end(), row.begin(), row.end());
    // Scene::validate (already run) checks centers and frames; the reference leaves the other state
    // arrays unchecked (and reads them out of bounds); the flat copy needs them sized
    require(st.scales.size() == st.centers.size() && st.center_vel.size() == st.centers.size() &&
                st.scale_vel.size() == st.centers.size() && static_cast<int>(st.angular_vel.size()) == m,
            "rod state arrays must match the vertex / element counts");
    desc.vertex_count = n;
    desc.material = rod.material;
    desc.collision_group = rod.collision_group;
    desc.self_collide = rod.self_collide ? 1 : 0;
    desc.rest_centers = rest_centers.data();
    desc.rest_scales = rp.scales.data();
    desc.radii = rp.radii.data();
    desc.lengths = rp.lengths.data();
    desc.initial_lengths = rp.initial_lengths.data();
    desc.rest_frames = rest_frames.data();
    desc.darboux = darboux.data();
    desc.tangent_dots = rp.tangent_dots.data();
    desc.scale_grads = rp.scale_grads.data();
    desc.scale_laplacians = rp.scale_laplacians.data();
    desc.centers = centers.data();
    desc.scales = st.scales.data();
    desc.frames = frames.data();
    desc.center_vel = center_vel.data();
    desc.scale_vel = st.scale_vel.data();
    desc.angular_vel = angular_vel.data();
    desc.pinned = rod.pinned.empty() ? nullptr : rod.pinned.data();
    desc.bone_count = static_cast<int32_t>(rod.bones.size());
    desc.bones = rod.bones.empty() ? nullptr : rod.bones.data();
    desc.bone_weights = bone_w.empty() ? nullptr : bone_w.data();
  }
};

/// Scene (scene.h:109-126) -> a C-ABI scene handle. Probes and the skin setup are caller-side
/// data (metrics / CLI) and stay in the mirror.
class CScene {
 public:
  explicit CScene(const Scene& scene) {
    check(vrod_scene_create(&s_));
    try {
      const vrod_settings st = to_c(scene.settings);
      check(vrod_scene_set_settings(s_, &st));
      for (const MaterialParams& m : scene.materials) {
        const vrod_material cm = to_c(m);
        check(vrod_scene_add_material(s_, &cm));
      }
      for (const Rod& r : scene.rods) {
        RodBuffers b(r);
        check(vrod_scene_add_rod(s_, &b.desc));
      }
      for (const HalfPlane& p : scene.planes) {
        double nrm[3];
        put3(nrm, p.normal);
        check(vrod_scene_add_plane(s_, nrm, p.offset));
      }
      for (const Bone& b : scene.bones) {
        std::vector<double> t, pos, rot;
        for (const RigidKeyframe& k : b.keys) {
          t.push_back(k.t);
          pos.insert(pos.end(), {k.position.x(), k.position.y(), k.position.z()});
          rot.insert(rot.end(), {k.rotation.w(), k.rotation.x(), k.rotation.y(), k.rotation.z()});
        }
        check(vrod_scene_add_bone(s_, static_cast<int32_t>(b.keys.size()), t.data(), pos.data(), rot.data()));
      }
      for (const KinematicPill& kp : scene.kinematic_pills) {
        const vrod_pill cp = to_c(kp.pill);
        check(vrod_scene_add_kinematic_pill(s_, &cp, kp.bone));
      }
      for (const auto& members : scene.bundles) {
        std::vector<int32_t> rods, verts;
        for (const BundleMember& mb : members) {
          rods.push_back(mb.rod);
          verts.push_back(mb.vertex);
        }
        check(vrod_scene_add_bundle(s_, static_cast<int32_t>(members.size()), rods.data(), verts.data()));
      }
      for (const PinMotion& pm : scene.pin_motions) {
        double a[3], b[3];
        put3(a, pm.start);
        put3(b, pm.target);
        check(vrod_scene_add_pin_motion(s_, pm.rod, pm.vertex, a, b, pm.t0, pm.t1));
      }
      for (const SoftPin& sp : scene.soft_pins) {
        double t[3];
        put3(t, sp.target);
        check(vrod_scene_add_soft_pin(s_, sp.rod, sp.vertex, t, sp.stiffness));
      }
      for (const Activation& a : scene.activations)
        check(vrod_scene_add_activation(s_, a.rod, a.factor, a.t_start, a.t_end, a.first_element, a.last_element));
    } catch (...) {
      vrod_scene_destroy(s_);
      throw;
    }
  }
  ~CScene() { vrod_scene_destroy(s_); }
  CScene(const CScene&) = delete;
  CScene& operator=(const CScene&) = delete;
  const vrod_scene* get() const { return s_; }

 private:
  vrod_scene* s_ = nullptr;
};

}  // namespace detail

/// Drop-in for vrod::Solver (solver.h:54-115) running the substep on one B200.
class Solver {
 public:
  explicit Solver(Scene scene) : scene_(std::move(scene)) {
    scene_.validate();  // the reference's own checks and messages, before any C-ABI call (solver.cpp:103)
    {
      detail::CScene cs(scene_);
      check(vrod_solver_create(cs.get(), &h_));
    }
    vrod_solver_info info{};
    check(vrod_solver_get_info(h_, &info));
    V_ = info.total_vertices;
    E_ = info.total_elements;
    build_layout_mirror(info);
    for (const auto& members : scene_.bundles) groups_.push_back(make_bundle_group(scene_.rods, members));
  }
  ~Solver() {
    if (h_) vrod_solver_destroy(h_);
  }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;
  Solver(Solver&& o) noexcept { *this = std::move(o); }
  Solver& operator=(Solver&& o) noexcept {
    if (this != &o) {
      if (h_) vrod_solver_destroy(h_);
      h_ = std::exchange(o.h_, nullptr);
      scene_ = std::move(o.scene_);
      layout_ = std::move(o.layout_);
      groups_ = std::move(o.groups_);
      loads_ = std::move(o.loads_);
      pulled_ = std::move(o.pulled_);
      V_ = o.V_;
      E_ = o.E_;
      stale_ = o.stale_;
      loads_pushed_ = o.loads_pushed_;
    }
    return *this;
  }

  /// Solver::step(), solver.cpp:363-388. Throws SimulationError on a non-finite state.
  StepReport step() {
    sync_to_device();
    vrod_step_report r{};
    const int status = vrod_solver_step(h_, &r);
    stale_ = true;
    check(status);
    return detail::from_c(r);
  }

  /// Solver::probe_convergence, solver.cpp:390-398: iterations x 8 residual RMS rows.
  std::vector<std::vector<double>> probe_convergence(int iterations) {
    sync_to_device();
    std::vector<double> flat(static_cast<std::size_t>(iterations > 0 ? iterations : 0) * 8);
    const int status = vrod_solver_probe_convergence(h_, iterations, flat.data());
    if (status == VROD_OK || status == VROD_SIMULATION_ERROR) stale_ = true;
    check(status);
    std::vector<std::vector<double>> log(static_cast<std::size_t>(iterations));
    for (int i = 0; i < iterations; ++i) log[i].assign(flat.begin() + 8 * i, flat.begin() + 8 * i + 8);
    return log;
  }

  const Scene& scene() const {
    pull();
    return scene_;
  }
  Scene& scene() {
    pull();
    return scene_;
  }
  const DofLayout& layout() const {
    refresh_theta_weights();
    return layout_;
  }
  double time() const { return info().time; }
  int step_index() const { return info().step_index; }
  int dof_count() const { return layout_.dof_count; }
  ExternalLoads& loads() { return loads_; }
  std::span<const BundleGroup> bundles() const { return groups_; }  // rest data; warm rotations live on the device

  double kinetic_energy() const {
    const_cast<Solver*>(this)->sync_to_device();
    double v = 0.0;
    check(vrod_solver_energy(h_, &v, nullptr, nullptr));
    return v;
  }
  double total_volume() const {
    const_cast<Solver*>(this)->sync_to_device();
    double v = 0.0;
    check(vrod_solver_energy(h_, nullptr, &v, nullptr));
    return v;
  }
  double total_rest_volume() const {
    double v = 0.0;
    check(vrod_solver_energy(h_, nullptr, nullptr, &v));
    return v;
  }
  std::vector<Pill> current_pills() const {
    const_cast<Solver*>(this)->sync_to_device();
    int64_t n = 0;
    check(vrod_solver_current_pills(h_, 0, &n, nullptr));
    std::vector<vrod_pill> c(static_cast<std::size_t>(n));
    check(vrod_solver_current_pills(h_, n, &n, c.data()));
    std::vector<Pill> out;
    out.reserve(c.size());
    for (const vrod_pill& p : c) out.push_back(detail::from_c(p));
    return out;
  }
  std::vector<PillTransform> pill_transforms() const {
    const_cast<Solver*>(this)->sync_to_device();
    int64_t n = 0;
    check(vrod_solver_pill_transforms(h_, 0, &n, nullptr));
    std::vector<vrod_pill_transform> c(static_cast<std::size_t>(n));
    check(vrod_solver_pill_transforms(h_, n, &n, c.data()));
    std::vector<PillTransform> out;
    out.reserve(c.size());
    for (const vrod_pill_transform& t : c) out.push_back(detail::from_c(t));
    return out;
  }

  /// Product options (state_prefetch, exact_shape_matching, phase_timing), vrod_capi.h.
  void set_option(const char* name, int64_t value) { check(vrod_solver_set_option(h_, name, value)); }
  vrod_solver* handle() { return h_; }

 private:
  vrod_solver_info info() const {
    vrod_solver_info i{};
    check(vrod_solver_get_info(h_, &i));
    return i;
  }

  // DofLayout (layout.h:17-41) of the device world, read back once; theta weights on demand.
  void build_layout_mirror(const vrod_solver_info& info) {
    DofLayout& L = layout_;
    const int R = info.rod_count;
    std::vector<int32_t> sizes(R);
    check(vrod_solver_get_rod_sizes(h_, sizes.data()));
    L.total_vertices = V_;
    L.total_elements = E_;
    L.dof_count = info.dof_count;
    int v = 0, e = 0;
    for (int r = 0; r < R; ++r) {
      L.vertex_base.push_back(v);
      L.element_base.push_back(e);
      for (int k = 0; k < sizes[r]; ++k) {
        L.vertex_rod.push_back(r);
        L.vertex_local.push_back(k);
        const auto& pin = scene_.rods[r].pinned;
        L.pinned.push_back(!pin.empty() && pin[k] ? 1 : 0);
        if (k + 1 < sizes[r]) {
          L.element_rod.push_back(r);
          L.element_local.push_back(k);
        }
      }
      v += sizes[r];
      e += sizes[r] - 1;
    }
    L.center_weight.resize(V_);
    L.scale_weight.resize(V_);
    L.inv_center.resize(V_);
    L.inv_scale.resize(V_);
    L.theta_weight.resize(E_);
    L.inv_theta.resize(E_);
    check(vrod_solver_get_weights(h_, L.center_weight.data(), L.scale_weight.data(), nullptr));
    check(vrod_solver_get_inverse_weights(h_, L.inv_center.data(), L.inv_scale.data(), nullptr));
    refresh_theta_weights();
  }

  void refresh_theta_weights() const {
    std::vector<double> tw(3 * static_cast<std::size_t>(E_)), it(3 * static_cast<std::size_t>(E_));
    check(vrod_solver_get_weights(h_, nullptr, nullptr, tw.data()));
    check(vrod_solver_get_inverse_weights(h_, nullptr, nullptr, it.data()));
    for (int e = 0; e < E_; ++e) {
      layout_.theta_weight[e] = detail::get3(&tw[3 * e]);
      layout_.inv_theta[e] = detail::get3(&it[3 * e]);
    }
  }

  struct Flat {
    std::vector<double> c, s, q, cv, sv, av;
  };

  Flat flatten() const {
    Flat f;
    f.c.reserve(3 * V_);
    f.s.reserve(V_);
    f.q.reserve(4 * E_);
    f.cv.reserve(3 * V_);
    f.sv.reserve(V_);
    f.av.reserve(3 * E_);
    double b[4];
    for (const Rod& rod : scene_.rods) {
      const RodState& st = rod.state;
      for (const Vec3& x : st.centers) detail::put3(b, x), f.c.insert(f.c.end(), b, b + 3);
      f.s.insert(f.s.end(), st.scales.begin(), st.scales.end());
      for (const Quat& x : st.frames) detail::putq(b, x), f.q.insert(f.q.end(), b, b + 4);
      for (const Vec3& x : st.center_vel) detail::put3(b, x), f.cv.insert(f.cv.end(), b, b + 3);
      f.sv.insert(f.sv.end(), st.scale_vel.begin(), st.scale_vel.end());
      for (const Vec3& x : st.angular_vel) detail::put3(b, x), f.av.insert(f.av.end(), b, b + 3);
    }
    return f;
  }

  static bool same(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), sizeof(double) * a.size()) == 0);
  }

  // Device -> mirror (scene_.rods[*].state and the activation-refreshed rest data).
  void pull() const {
    if (!stale_) return;
    Flat f;
    f.c.resize(3 * V_);
    f.s.resize(V_);
    f.q.resize(4 * E_);
    f.cv.resize(3 * V_);
    f.sv.resize(V_);
    f.av.resize(3 * E_);
    check(vrod_solver_get_state(h_, f.c.data(), f.s.data(), f.q.data(), f.cv.data(), f.sv.data(), f.av.data()));
    std::vector<double> len(E_), darb(3 * static_cast<std::size_t>(E_)), grad(E_), lap(E_);
    check(vrod_solver_get_rest(h_, len.data(), darb.data(), grad.data(), lap.data()));
    int v = 0, e = 0;
    for (Rod& rod : scene_.rods) {
      RodState& st = rod.state;
      RodRestPose& rp = rod.rest;
      const int n = static_cast<int>(st.centers.size());
      for (int k = 0; k < n; ++k, ++v) {
        st.centers[k] = detail::get3(&f.c[3 * v]);
        st.scales[k] = f.s[v];
        st.center_vel[k] = detail::get3(&f.cv[3 * v]);
        st.scale_vel[k] = f.sv[v];
      }
      for (int k = 0; k + 1 < n; ++k, ++e) {
        st.frames[k] = detail::getq(&f.q[4 * e]);
        st.angular_vel[k] = detail::get3(&f.av[3 * e]);
        rp.lengths[k] = len[e];
        rp.scale_grads[k] = grad[e];
        if (k + 2 < n) {
          rp.darboux[k] = detail::get3(&darb[3 * e]);
          rp.scale_laplacians[k] = lap[e];
        }
      }
    }
    pulled_ = std::move(f);
    stale_ = false;
  }

  // Mirror edits (scene() writes between steps) and loads() -> device.
  void sync_to_device() {
    if (!stale_) {
      const Flat f = flatten();
      if (!(same(f.c, pulled_.c) && same(f.s, pulled_.s) && same(f.q, pulled_.q) && same(f.cv, pulled_.cv) &&
            same(f.sv, pulled_.sv) && same(f.av, pulled_.av))) {
        check(vrod_solver_set_state(h_, f.c.data(), f.s.data(), f.q.data(), f.cv.data(), f.sv.data(), f.av.data()));
        pulled_ = f;
      }
    }
    push_loads();
  }

  // ExternalLoads (solver.h:35-41), resolved like predict_all (solver.cpp:155-167): an empty outer
  // vector = no load; an empty per-rod vector = no load on that rod.
  void push_loads() {
    const bool any = !loads_.force_density.empty() || !loads_.torque.empty() || !loads_.scale_load.empty();
    if (!any && !loads_pushed_) return;
    const int R = static_cast<int>(scene_.rods.size());
    std::vector<double> fd(3 * static_cast<std::size_t>(V_), 0.0), tq(3 * static_cast<std::size_t>(E_), 0.0),
        sl(E_, 0.0);
    std::vector<uint8_t> fdr(R, 0), tqr(R, 0), slr(R, 0);
    bool has_fd = false, has_tq = false, has_sl = false;
    for (int r = 0; r < R; ++r) {
      const int v0 = layout_.vertex_base[r], e0 = layout_.element_base[r];
      const int n = static_cast<int>(scene_.rods[r].state.centers.size());
      if (r < static_cast<int>(loads_.force_density.size()) && !loads_.force_density[r].empty()) {
        require(static_cast<int>(loads_.force_density[r].size()) == n, "external force size must match the rod");
        for (int k = 0; k < n; ++k) detail::put3(&fd[3 * (v0 + k)], loads_.force_density[r][k]);
        fdr[r] = has_fd = true;
      }
      if (r < static_cast<int>(loads_.torque.size()) && !loads_.torque[r].empty()) {
        require(static_cast<int>(loads_.torque[r].size()) == n - 1, "external torque size must match the rod");
        for (int k = 0; k < n - 1; ++k) detail::put3(&tq[3 * (e0 + k)], loads_.torque[r][k]);
        tqr[r] = has_tq = true;
      }
      if (r < static_cast<int>(loads_.scale_load.size()) && !loads_.scale_load[r].empty()) {
        require(static_cast<int>(loads_.scale_load[r].size()) == n - 1, "external scale load size must match the rod");
        for (int k = 0; k < n - 1; ++k) sl[e0 + k] = loads_.scale_load[r][k];
        slr[r] = has_sl = true;
      }
    }
    check(vrod_solver_set_loads(h_, has_fd ? fd.data() : nullptr, fdr.data(), has_tq ? tq.data() : nullptr,
                                tqr.data(), has_sl ? sl.data() : nullptr, slr.data()));
    loads_pushed_ = any;
  }

  mutable Scene scene_;
  vrod_solver* h_ = nullptr;
  mutable DofLayout layout_;
  std::vector<BundleGroup> groups_;
  ExternalLoads loads_;
  mutable Flat pulled_;
  int V_ = 0, E_ = 0;
  mutable bool stale_ = true;
  bool loads_pushed_ = false;
};

}  // namespace vrod::b200
