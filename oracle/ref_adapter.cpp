// C-ABI adapter over the REFERENCE implementation — TEST INFRASTRUCTURE ONLY.
//
// Linked with the reference's own, unmodified hot-path sources (compiled from
// /root/reference/proj/core/src against shim/Eigen by oracle/Makefile) into
// oracle/_ref/libvrod_ref.so. It implements include/vrod_capi.h by calling the reference
// C++ API directly (vrod::Scene, vrod::Solver, broad_phase, ...), so tests and bench.py can
// drive the reference exactly like the product. Never shipped, never on the product path.

#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

// The contact list of the last substep is private in the reference Solver
// (solver.h:106-108); this test adapter reads it for contact-set parity checks.
#define private public
#include "vrod/solver.h"
#undef private
#include "vrod/bundling.h"
#include "vrod/collision.h"
#include "vrod/constraints.h"
#include "vrod/layout.h"
#include "vrod/rod.h"
#include "vrod/scene.h"
#include "vrod/skinning.h"
#include "vrod_capi.h"

using namespace vrod;

namespace {

thread_local std::string g_error;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return VROD_OK;
  } catch (const SimulationError& e) {
    g_error = e.what();
    return VROD_SIMULATION_ERROR;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return VROD_OUT_OF_RANGE;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return VROD_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_error = e.what();
    return VROD_RUNTIME_ERROR;
  }
}

Vec3 v3(const double* p) { return Vec3(p[0], p[1], p[2]); }
Quat q4(const double* p) { return Quat(p[0], p[1], p[2], p[3]); }
void put3(double* p, const Vec3& v) {
  p[0] = v.x();
  p[1] = v.y();
  p[2] = v.z();
}
void put4(double* p, const Quat& q) {
  p[0] = q.w();
  p[1] = q.x();
  p[2] = q.y();
  p[3] = q.z();
}

Pill to_pill(const vrod_pill& p) {
  Pill o;
  o.c0 = v3(p.c0);
  o.c1 = v3(p.c1);
  o.r0 = p.r0;
  o.r1 = p.r1;
  o.rod = p.rod;
  o.element = p.element;
  o.group = p.group;
  o.self_collide = p.self_collide != 0;
  return o;
}
vrod_pill from_pill(const Pill& p) {
  vrod_pill o;
  put3(o.c0, p.c0);
  put3(o.c1, p.c1);
  o.r0 = p.r0;
  o.r1 = p.r1;
  o.rod = p.rod;
  o.element = p.element;
  o.group = p.group;
  o.self_collide = p.self_collide ? 1 : 0;
  return o;
}

}  // namespace

struct vrod_scene {
  Scene scene;
};
struct vrod_skin {
  TriMesh mesh;
  SkinBinding binding;
};
// A batch (vrod_batch_create) is N independent reference solvers stepped in lockstep — the
// reference has no batch API of its own.
struct vrod_solver {
  std::unique_ptr<Solver> solver;
  std::vector<std::unique_ptr<Solver>> batch;
  std::vector<StepReport> last;
};
namespace {
Solver& one(const vrod_solver* h) {
  if (!h->solver) throw std::invalid_argument("this query needs a single-scene solver (not a batch)");
  return *h->solver;
}
std::vector<Solver*> all(const vrod_solver* h) {
  std::vector<Solver*> v;
  if (h->solver) v.push_back(h->solver.get());
  for (const auto& b : h->batch) v.push_back(b.get());
  return v;
}
void put_report(const StepReport& r, vrod_step_report* out) {
  std::memset(out, 0, sizeof(*out));
  out->step = r.step;
  out->time = r.time;
  for (int k = 0; k < 8 && k < static_cast<int>(r.residuals.size()); ++k) out->residuals[k] = r.residuals[k];
  out->max_penetration = r.max_penetration;
  out->contact_count = r.contact_count;
  out->broad_pairs = r.broad_pairs;
  out->skipped_singular = r.skipped_singular;
  out->dof_count = r.dof_count;
  out->predict_ms = r.timings.predict_ms;
  out->broad_ms = r.timings.broad_ms;
  out->narrow_ms = r.timings.narrow_ms;
  out->solve_ms = r.timings.solve_ms;
  out->finalize_ms = r.timings.finalize_ms;
  out->total_ms = r.timings.total_ms;
}
void put_transform(const PillTransform& t, vrod_pill_transform* o) {
  put3(o->center, t.center);
  o->scale = t.scale;
  put4(o->rotation, t.rotation);
}
PillTransform to_transform(const vrod_pill_transform& t) {
  PillTransform o;
  o.center = v3(t.center);
  o.scale = t.scale;
  o.rotation = q4(t.rotation);
  return o;
}
template <class T, class Put>
void put_list(const std::vector<T>& v, int64_t cap, int64_t* count, Put&& put) {
  for (std::size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) put(v[i], i);
  *count = static_cast<int64_t>(v.size());
}
}  // namespace

extern "C" {

const char* vrod_last_error(void) { return g_error.c_str(); }
const char* vrod_backend_name(void) { return "reference-cpu"; }
int32_t vrod_capi_version(void) { return VROD_CAPI_VERSION; }

void vrod_default_material(vrod_material* out) {
  const MaterialParams m;
  *out = {m.stretch_x, m.stretch_y, m.stretch_z, m.bend_x, m.bend_y, m.bend_z, m.volume, m.density};
}

void vrod_default_settings(vrod_settings* out) {
  const SolverSettings s;
  out->dt = s.dt;
  out->iterations = s.iterations;
  out->substeps = s.substeps;
  out->beta = s.beta;
  put3(out->gravity, s.gravity);
  out->dichotomous_iterations = s.dichotomous_iterations;
  out->shape_match_period = s.shape_match_period;
  out->contact_stiffness = s.contact_stiffness;
  out->velocity_damping = s.velocity_damping;
  out->deterministic = s.deterministic ? 1 : 0;
  out->scale_mode = static_cast<int32_t>(s.scale_mode);
}

int vrod_make_rest_pose(int32_t n, const double* centers, int32_t radii_count, const double* radii,
                        int32_t scales_count, const double* scales, vrod_rest_pose_out* out) {
  return guarded([&] {
    std::vector<Vec3> c(static_cast<std::size_t>(std::max(0, n)));
    for (int i = 0; i < n; ++i) c[i] = v3(centers + 3 * i);
    const RodRestPose rest =
        make_rest_pose(c, std::span<const double>(radii, static_cast<std::size_t>(radii_count)),
                       std::span<const double>(scales, static_cast<std::size_t>(scales_count)));
    const int m = rest.element_count();
    for (int i = 0; i < n; ++i) {
      out->rest_scales[i] = rest.scales[i];
      out->radii[i] = rest.radii[i];
    }
    for (int e = 0; e < m; ++e) {
      out->lengths[e] = rest.lengths[e];
      out->initial_lengths[e] = rest.initial_lengths[e];
      put4(out->rest_frames + 4 * e, rest.frames[e]);
      out->tangent_dots[e] = rest.tangent_dots[e];
      out->scale_grads[e] = rest.scale_grads[e];
    }
    for (int j = 0; j + 1 < m; ++j) {
      put3(out->darboux + 3 * j, rest.darboux[j]);
      out->scale_laplacians[j] = rest.scale_laplacians[j];
    }
  });
}

int vrod_scene_create(vrod_scene** out) {
  return guarded([&] { *out = new vrod_scene(); });
}
void vrod_scene_destroy(vrod_scene* scene) { delete scene; }

int vrod_scene_set_settings(vrod_scene* s, const vrod_settings* in) {
  return guarded([&] {
    SolverSettings& o = s->scene.settings;
    o.dt = in->dt;
    o.iterations = in->iterations;
    o.substeps = in->substeps;
    o.beta = in->beta;
    o.gravity = v3(in->gravity);
    o.dichotomous_iterations = in->dichotomous_iterations;
    o.shape_match_period = in->shape_match_period;
    o.contact_stiffness = in->contact_stiffness;
    o.velocity_damping = in->velocity_damping;
    o.deterministic = in->deterministic != 0;
    o.scale_mode = static_cast<ScaleMode>(in->scale_mode);
  });
}

int vrod_scene_add_material(vrod_scene* s, const vrod_material* m) {
  return guarded([&] {
    MaterialParams p;
    p.stretch_x = m->stretch_x;
    p.stretch_y = m->stretch_y;
    p.stretch_z = m->stretch_z;
    p.bend_x = m->bend_x;
    p.bend_y = m->bend_y;
    p.bend_z = m->bend_z;
    p.volume = m->volume;
    p.density = m->density;
    s->scene.materials.push_back(p);
  });
}

int vrod_scene_add_rod(vrod_scene* s, const vrod_rod_desc* d) {
  return guarded([&] {
    const int n = d->vertex_count;
    const int m = n - 1;
    Rod rod;
    RodRestPose& r = rod.rest;
    RodState& st = rod.state;
    for (int i = 0; i < n; ++i) {
      r.centers.push_back(v3(d->rest_centers + 3 * i));
      r.scales.push_back(d->rest_scales[i]);
      r.radii.push_back(d->radii[i]);
      st.centers.push_back(v3(d->centers + 3 * i));
      st.scales.push_back(d->scales[i]);
      st.center_vel.push_back(v3(d->center_vel + 3 * i));
      st.scale_vel.push_back(d->scale_vel[i]);
      rod.pinned.push_back(d->pinned ? d->pinned[i] : 0);
    }
    for (int e = 0; e < m; ++e) {
      r.lengths.push_back(d->lengths[e]);
      r.initial_lengths.push_back(d->initial_lengths[e]);
      r.frames.push_back(q4(d->rest_frames + 4 * e));
      r.tangent_dots.push_back(d->tangent_dots[e]);
      r.scale_grads.push_back(d->scale_grads[e]);
      st.frames.push_back(q4(d->frames + 4 * e));
      st.angular_vel.push_back(v3(d->angular_vel + 3 * e));
    }
    for (int j = 0; j + 1 < m; ++j) {
      r.darboux.push_back(v3(d->darboux + 3 * j));
      r.scale_laplacians.push_back(d->scale_laplacians[j]);
    }
    rod.material = d->material;
    rod.collision_group = d->collision_group;
    rod.self_collide = d->self_collide != 0;
    for (int b = 0; b < d->bone_count; ++b) rod.bones.push_back(d->bones[b]);
    if (d->bone_count > 0) {
      for (int i = 0; i < n; ++i) {
        rod.bone_weights.emplace_back(d->bone_weights + static_cast<std::size_t>(i) * d->bone_count,
                                      d->bone_weights + static_cast<std::size_t>(i + 1) * d->bone_count);
      }
    }
    s->scene.rods.push_back(std::move(rod));
  });
}

int vrod_scene_add_plane(vrod_scene* s, const double normal[3], double offset) {
  return guarded([&] { s->scene.planes.push_back({v3(normal), offset}); });
}

int vrod_scene_add_bone(vrod_scene* s, int32_t k, const double* t, const double* pos, const double* rot) {
  return guarded([&] {
    Bone b;
    for (int i = 0; i < k; ++i) b.keys.push_back({t[i], v3(pos + 3 * i), q4(rot + 4 * i)});
    s->scene.bones.push_back(std::move(b));
  });
}

int vrod_scene_add_kinematic_pill(vrod_scene* s, const vrod_pill* p, int32_t bone) {
  return guarded([&] {
    KinematicPill kp;
    kp.pill = to_pill(*p);
    kp.bone = bone;
    s->scene.kinematic_pills.push_back(kp);
  });
}

int vrod_scene_add_bundle(vrod_scene* s, int32_t count, const int32_t* rods, const int32_t* verts) {
  return guarded([&] {
    std::vector<BundleMember> members;
    for (int i = 0; i < count; ++i) members.push_back({rods[i], verts[i]});
    s->scene.bundles.push_back(std::move(members));
  });
}

int vrod_scene_add_pin_motion(vrod_scene* s, int32_t rod, int32_t vertex, const double start[3],
                              const double target[3], double t0, double t1) {
  return guarded([&] { s->scene.pin_motions.push_back({rod, vertex, v3(start), v3(target), t0, t1}); });
}

int vrod_scene_add_soft_pin(vrod_scene* s, int32_t rod, int32_t vertex, const double target[3],
                            double stiffness) {
  return guarded([&] { s->scene.soft_pins.push_back({rod, vertex, v3(target), stiffness}); });
}

int vrod_scene_add_activation(vrod_scene* s, int32_t rod, double factor, double t_start, double t_end,
                              int32_t first_element, int32_t last_element) {
  return guarded([&] {
    Activation a;
    a.rod = rod;
    a.factor = factor;
    a.t_start = t_start;
    a.t_end = t_end;
    a.first_element = first_element;
    a.last_element = last_element;
    s->scene.activations.push_back(a);
  });
}

int vrod_scene_validate(const vrod_scene* s) {
  return guarded([&] { s->scene.validate(); });
}

int vrod_solver_create(const vrod_scene* s, vrod_solver** out) {
  return guarded([&] {
    auto h = std::make_unique<vrod_solver>();
    h->solver = std::make_unique<Solver>(s->scene);
    *out = h.release();
  });
}
void vrod_solver_destroy(vrod_solver* s) { delete s; }

int vrod_batch_create(int32_t n, const vrod_scene* const* scenes, vrod_solver** out) {
  return guarded([&] {
    if (n < 1 || !scenes) throw std::invalid_argument("batch needs at least one scene");
    auto h = std::make_unique<vrod_solver>();
    for (int i = 0; i < n; ++i) h->batch.push_back(std::make_unique<Solver>(scenes[i]->scene));
    *out = h.release();
  });
}
int vrod_solver_scene_count(const vrod_solver* s, int32_t* count) {
  return guarded([&] { *count = static_cast<int32_t>(all(s).size()); });
}
int vrod_solver_scene_reports(const vrod_solver* s, int32_t capacity, vrod_step_report* reports) {
  return guarded([&] {
    if (capacity < static_cast<int32_t>(s->last.size())) throw std::invalid_argument("scene report capacity too small");
    for (std::size_t i = 0; i < s->last.size(); ++i) put_report(s->last[i], reports + i);
  });
}

int vrod_solver_step(vrod_solver* s, vrod_step_report* out) {
  return guarded([&] {
    s->last.clear();
    StepReport tot;
    tot.residuals.assign(8, 0.0);
    for (Solver* sv : all(s)) {
      s->last.push_back(sv->step());
      const StepReport& r = s->last.back();
      if (s->solver) {
        tot = r;
        break;
      }
      tot.step = r.step;
      tot.time = r.time;
      for (int k = 0; k < 8 && k < static_cast<int>(r.residuals.size()); ++k)
        tot.residuals[k] = std::max(tot.residuals[k], r.residuals[k]);
      tot.max_penetration = std::max(tot.max_penetration, r.max_penetration);
      tot.contact_count += r.contact_count;
      tot.broad_pairs += r.broad_pairs;
      tot.skipped_singular += r.skipped_singular;
      tot.dof_count += r.dof_count;
      tot.timings.total_ms += r.timings.total_ms;
    }
    put_report(tot, out);
  });
}

int vrod_solver_probe_convergence(vrod_solver* s, int32_t iterations, double* log) {
  return guarded([&] {
    const auto rows = one(s).probe_convergence(iterations);
    for (std::size_t i = 0; i < rows.size(); ++i)
      for (int k = 0; k < 8; ++k) log[i * 8 + k] = rows[i][k];
  });
}

int vrod_solver_get_info(const vrod_solver* s, vrod_solver_info* info) {
  return guarded([&] {
    std::memset(info, 0, sizeof(*info));
    for (const Solver* p : all(s)) {
      const Solver& sv = *p;
      info->rod_count += static_cast<int32_t>(sv.scene().rods.size());
      info->total_vertices += sv.layout().total_vertices;
      info->total_elements += sv.layout().total_elements;
      info->dof_count += sv.dof_count();
      info->step_index = sv.step_index();
      info->bundle_count += static_cast<int32_t>(sv.bundles().size());
      info->elastic_blocks += static_cast<int32_t>(sv.elastic_.size());
      info->time = sv.time();
    }
  });
}

int vrod_solver_get_rod_sizes(const vrod_solver* s, int32_t* counts) {
  return guarded([&] {
    int i = 0;
    for (const Solver* p : all(s))
      for (const Rod& rod : p->scene().rods) counts[i++] = rod.rest.vertex_count();
  });
}

int vrod_solver_get_state(vrod_solver* s, double* c, double* sc, double* f, double* cv, double* sv,
                          double* av) {
  return guarded([&] {
    std::size_t vi = 0, ei = 0;
    for (const Solver* p : all(s))
      for (const Rod& rod : p->scene().rods) {
        for (int v = 0; v < rod.rest.vertex_count(); ++v, ++vi) {
          if (c) put3(c + 3 * vi, rod.state.centers[v]);
          if (sc) sc[vi] = rod.state.scales[v];
          if (cv) put3(cv + 3 * vi, rod.state.center_vel[v]);
          if (sv) sv[vi] = rod.state.scale_vel[v];
        }
        for (int e = 0; e < rod.rest.element_count(); ++e, ++ei) {
          if (f) put4(f + 4 * ei, rod.state.frames[e]);
          if (av) put3(av + 3 * ei, rod.state.angular_vel[e]);
        }
      }
  });
}

// Product options (include/vrod_capi.h): the CPU path is always the reference's exact order and
// copies state on demand, so the options are accepted and change nothing here.
int vrod_solver_set_option(vrod_solver*, const char* name, int64_t) {
  return guarded([&] {
    const std::string n = name ? name : "";
    vrod::require(n == "state_prefetch" || n == "exact_shape_matching" || n == "phase_timing", "unknown solver option");
  });
}
int vrod_solver_set_state(vrod_solver* s, const double* c, const double* sc, const double* f,
                          const double* cv, const double* sv, const double* av) {
  return guarded([&] {
    std::size_t vi = 0, ei = 0;
    for (Rod& rod : one(s).scene().rods) {
      for (int v = 0; v < rod.rest.vertex_count(); ++v, ++vi) {
        if (c) rod.state.centers[v] = v3(c + 3 * vi);
        if (sc) rod.state.scales[v] = sc[vi];
        if (cv) rod.state.center_vel[v] = v3(cv + 3 * vi);
        if (sv) rod.state.scale_vel[v] = sv[vi];
      }
      for (int e = 0; e < rod.rest.element_count(); ++e, ++ei) {
        if (f) rod.state.frames[e] = q4(f + 4 * ei);
        if (av) rod.state.angular_vel[e] = v3(av + 3 * ei);
      }
    }
  });
}

int vrod_solver_get_rest(vrod_solver* s, double* lengths, double* darboux, double* grads, double* laps) {
  return guarded([&] {
    std::size_t ei = 0;
    for (const Rod& rod : one(s).scene().rods) {
      const int m = rod.rest.element_count();
      for (int e = 0; e < m; ++e, ++ei) {
        if (lengths) lengths[ei] = rod.rest.lengths[e];
        if (grads) grads[ei] = rod.rest.scale_grads[e];
        const bool interior = e + 1 < m;
        if (darboux) put3(darboux + 3 * ei, interior ? rod.rest.darboux[e] : Vec3::Zero());
        if (laps) laps[ei] = interior ? rod.rest.scale_laplacians[e] : 0.0;
      }
    }
  });
}

int vrod_solver_set_loads(vrod_solver* s, const double* fd, const uint8_t* fd_rods, const double* tq,
                          const uint8_t* tq_rods, const double* sl, const uint8_t* sl_rods) {
  return guarded([&] {
    ExternalLoads& L = one(s).loads();
    const auto& rods = one(s).scene().rods;
    const std::size_t nr = rods.size();
    L.force_density.clear();
    L.torque.clear();
    L.scale_load.clear();
    if (fd) L.force_density.resize(nr);
    if (tq) L.torque.resize(nr);
    if (sl) L.scale_load.resize(nr);
    std::size_t vi = 0, ei = 0;
    for (std::size_t r = 0; r < nr; ++r) {
      const int n = rods[r].rest.vertex_count();
      const int m = rods[r].rest.element_count();
      if (fd && (!fd_rods || fd_rods[r]))
        for (int v = 0; v < n; ++v) L.force_density[r].push_back(v3(fd + 3 * (vi + v)));
      if (tq && (!tq_rods || tq_rods[r]))
        for (int e = 0; e < m; ++e) L.torque[r].push_back(v3(tq + 3 * (ei + e)));
      if (sl && (!sl_rods || sl_rods[r]))
        for (int e = 0; e < m; ++e) L.scale_load[r].push_back(sl[ei + e]);
      vi += n;
      ei += m;
    }
  });
}

int vrod_solver_energy(vrod_solver* s, double* ke, double* vol, double* rest_vol) {
  return guarded([&] {
    if (ke) *ke = one(s).kinetic_energy();
    if (vol) *vol = one(s).total_volume();
    if (rest_vol) *rest_vol = one(s).total_rest_volume();
  });
}

int vrod_solver_get_inverse_weights(vrod_solver* s, double* ic, double* is, double* it) {
  return guarded([&] {
    const DofLayout& L = one(s).layout();
    for (int v = 0; v < L.total_vertices; ++v) {
      if (ic) ic[v] = L.inv_center[v];
      if (is) is[v] = L.inv_scale[v];
    }
    for (int e = 0; e < L.total_elements; ++e)
      if (it) put3(it + 3 * e, L.inv_theta[e]);
  });
}

int vrod_solver_get_weights(vrod_solver* s, double* cw, double* sw, double* tw) {
  return guarded([&] {
    const DofLayout& L = one(s).layout();
    for (int v = 0; v < L.total_vertices; ++v) {
      if (cw) cw[v] = L.center_weight[v];
      if (sw) sw[v] = L.scale_weight[v];
    }
    for (int e = 0; e < L.total_elements; ++e)
      if (tw) put3(tw + 3 * e, L.theta_weight[e]);
  });
}

int vrod_solver_get_contacts(vrod_solver* s, int64_t cap, int64_t* count, int32_t* a, int32_t* b,
                             double* alpha, double* beta) {
  return guarded([&] {
    int64_t k = 0;
    for (const ConstraintBlock& blk : one(s).contact_blocks_) {
      if (blk.kind != ConstraintKind::kContact) continue;
      if (k < cap) {
        if (a) a[k] = blk.pill_a;
        if (b) b[k] = blk.aux;
        if (alpha) alpha[k] = blk.alpha;
        if (beta) beta[k] = blk.beta;
      }
      ++k;
    }
    *count = k;
  });
}

int vrod_solver_current_pills(vrod_solver* s, int64_t cap, int64_t* count, vrod_pill* out) {
  return guarded([&] {
    const auto pills = one(s).current_pills();
    for (std::size_t i = 0; i < pills.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = from_pill(pills[i]);
    *count = static_cast<int64_t>(pills.size());
  });
}

int vrod_pill_project(int64_t n, const double* x, const vrod_pill* pills, double* t, double* d,
                      uint8_t* degenerate) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      const PillProjection p = pill_project(v3(x + 3 * i), to_pill(pills[i]));
      if (t) t[i] = p.t;
      if (d) d[i] = p.distance;
      if (degenerate) degenerate[i] = p.degenerate ? 1 : 0;
    }
  });
}

int vrod_deepest_penetration(int64_t n, const vrod_pill* a, const vrod_pill* b, int32_t iters,
                             const double* warm, double* alpha, double* beta, double* dist) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      const PillOverlap o = deepest_penetration(to_pill(a[i]), to_pill(b[i]), iters, warm ? warm[i] : -1.0);
      alpha[i] = o.alpha;
      beta[i] = o.beta;
      dist[i] = o.distance;
    }
  });
}

int vrod_broad_phase(int64_t n, const vrod_pill* pills, int64_t cap, int64_t* count, int32_t* pairs) {
  return guarded([&] {
    std::vector<Pill> p;
    p.reserve(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) p.push_back(to_pill(pills[i]));
    const auto out = broad_phase(p);
    for (std::size_t k = 0; k < out.size() && static_cast<int64_t>(k) < cap; ++k) {
      pairs[2 * k] = out[k].first;
      pairs[2 * k + 1] = out[k].second;
    }
    *count = static_cast<int64_t>(out.size());
  });
}

int vrod_find_contacts(int64_t n, const vrod_pill* pills, int64_t npairs, const int32_t* pairs,
                       int32_t iters, int64_t nwarm, const uint64_t* wkeys, const double* walpha,
                       int64_t cap, int64_t* count, int32_t* pa, int32_t* pb, double* alpha,
                       double* beta, double* dist) {
  return guarded([&] {
    std::vector<Pill> p;
    for (int64_t i = 0; i < n; ++i) p.push_back(to_pill(pills[i]));
    std::vector<std::pair<int, int>> pr;
    for (int64_t k = 0; k < npairs; ++k) pr.emplace_back(pairs[2 * k], pairs[2 * k + 1]);
    std::vector<std::pair<std::uint64_t, double>> warm;
    for (int64_t k = 0; k < nwarm; ++k) warm.emplace_back(wkeys[k], walpha[k]);
    const auto out = find_contacts(p, pr, iters, wkeys ? &warm : nullptr);
    for (std::size_t k = 0; k < out.size() && static_cast<int64_t>(k) < cap; ++k) {
      pa[k] = out[k].pill_a;
      pb[k] = out[k].pill_b;
      alpha[k] = out[k].alpha;
      beta[k] = out[k].beta;
      dist[k] = out[k].distance;
    }
    *count = static_cast<int64_t>(out.size());
  });
}

int vrod_solver_pill_transforms(vrod_solver* s, int64_t cap, int64_t* count, vrod_pill_transform* out) {
  return guarded([&] {
    put_list(one(s).pill_transforms(), cap, count, [&](const PillTransform& t, std::size_t i) { put_transform(t, out + i); });
  });
}
int vrod_solver_rest_pill_transforms(vrod_solver* s, int64_t cap, int64_t* count, vrod_pill_transform* out) {
  return guarded([&] {
    put_list(rod_rest_pill_transforms(one(s).scene().rods), cap, count,
             [&](const PillTransform& t, std::size_t i) { put_transform(t, out + i); });
  });
}
int vrod_solver_rest_pills(vrod_solver* s, int64_t cap, int64_t* count, vrod_pill* out) {
  return guarded([&] {
    put_list(rod_rest_pills(one(s).scene().rods), cap, count, [&](const Pill& p, std::size_t i) { out[i] = from_pill(p); });
  });
}
int vrod_skin_bind(int32_t nv, const double* verts, int32_t nt, const int32_t* tris, int32_t np, const vrod_pill* pills,
                   const vrod_pill_transform* rest, int32_t max_influences, double epsilon, vrod_skin** out) {
  return guarded([&] {
    auto sk = std::make_unique<vrod_skin>();
    for (int32_t v = 0; v < nv; ++v) sk->mesh.vertices.push_back(v3(verts + 3 * v));
    for (int32_t t = 0; t < nt; ++t) sk->mesh.triangles.push_back({tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]});
    std::vector<Pill> p;
    std::vector<PillTransform> tr;
    for (int32_t i = 0; i < np; ++i) {
      p.push_back(to_pill(pills[i]));
      tr.push_back(to_transform(rest[i]));
    }
    sk->binding = bind_skin(sk->mesh, p, tr, max_influences, epsilon);
    *out = sk.release();
  });
}
void vrod_skin_destroy(vrod_skin* sk) { delete sk; }
int vrod_skin_smooth(vrod_skin* sk, int32_t iterations) {
  return guarded([&] { smooth_binding(sk->binding, sk->mesh, iterations); });
}
int vrod_skin_get_binding(const vrod_skin* sk, int32_t* offsets, int32_t* pills, double* weights, int32_t* nnz,
                          int32_t* clamped) {
  return guarded([&] {
    const SkinBinding& b = sk->binding;
    if (offsets) std::copy(b.offsets.begin(), b.offsets.end(), offsets);
    if (pills) std::copy(b.pills.begin(), b.pills.end(), pills);
    if (weights) std::copy(b.weights.begin(), b.weights.end(), weights);
    *nnz = static_cast<int32_t>(b.pills.size());
    *clamped = b.clamped_vertices;
  });
}
int vrod_skin_deform(vrod_skin* sk, int32_t np, const vrod_pill_transform* cur, double* out) {
  return guarded([&] {
    std::vector<PillTransform> tr;
    for (int32_t i = 0; i < np; ++i) tr.push_back(to_transform(cur[i]));
    std::vector<Vec3> o;
    deform_mesh(sk->binding, tr, sk->mesh, o);
    for (std::size_t v = 0; v < o.size(); ++v) put3(out + 3 * v, o[v]);
  });
}
int vrod_solver_shape_match(vrod_solver* s, int32_t cap, int32_t* count, double* fits) {
  return guarded([&] {
    int32_t k = 0;
    for (Solver* sv : all(s))
      for (BundleGroup& g : sv->groups_) {
        const SimilarityFit f = apply_shape_match(g, sv->scene().rods);
        if (fits && k < cap) {
          double* o = fits + 14ll * k;
          o[0] = f.scale;
          put3(o + 1, f.translation);
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) o[4 + 3 * a + b] = f.rotation(a, b);
          o[13] = f.degenerate ? 1.0 : 0.0;
        }
        ++k;
      }
    *count = k;
  });
}
int vrod_solver_jacobi_sweep(vrod_solver* s, double h, double beta, int32_t* active, int32_t* singular) {
  return guarded([&] {
    Solver& sv = one(s);
    std::vector<ConstraintBlock> blocks = sv.elastic_;
    blocks.insert(blocks.end(), sv.pin_blocks_.begin(), sv.pin_blocks_.end());
    for (ConstraintBlock& b : blocks) b.lambda = Vec3::Zero();
    const EvalContext ctx{sv.scene_.rods, &sv.layout_, sv.pills_, sv.scene_.planes, sv.pin_targets_, sv.classic_};
    const SweepOutcome o = jacobi_sweep(blocks, sv.scene_.rods, ctx, h, beta, sv.scratch_);
    if (active) *active = o.active;
    if (singular) *singular = o.skipped_singular;
  });
}
int vrod_solver_elastic_residuals(vrod_solver* s, int64_t cap, int64_t* count, double* W) {
  return guarded([&] {
    Solver& sv = one(s);
    const EvalContext ctx{sv.scene_.rods, &sv.layout_, sv.pills_, sv.scene_.planes, sv.pin_targets_, sv.classic_};
    const int64_t n = static_cast<int64_t>(sv.elastic_.size());
    for (int64_t i = 0; i < n && i < cap && W; ++i) {
      const ResidualEval ev = eval_constraint(sv.elastic_[i], ctx);
      for (int d = 0; d < 3; ++d) W[3 * i + d] = ev.W[d];
    }
    *count = n;
  });
}
int vrod_extract_rotation(int64_t n, const double* B, const double* guess, int32_t max_iterations, double tolerance,
                          double* out) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      Mat3 m;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m(a, b) = B[9 * i + 3 * a + b];
      put4(out + 4 * i, extract_rotation(m, q4(guess + 4 * i), max_iterations, tolerance));
    }
  });
}
int vrod_skin_deform_solver(vrod_skin* sk, vrod_solver* s, double* out) {
  return guarded([&] {
    std::vector<Vec3> o;
    deform_mesh(sk->binding, one(s).pill_transforms(), sk->mesh, o);
    if (out)
      for (std::size_t v = 0; v < o.size(); ++v) put3(out + 3 * v, o[v]);
  });
}

uint64_t vrod_pair_key(const vrod_pill* a, const vrod_pill* b) { return pair_key(to_pill(*a), to_pill(*b)); }

}  // extern "C"
