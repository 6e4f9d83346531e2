// The product's C-ABI (include/vrod_capi.h): the drop-in boundary for the reference's C++ core
// API. Scene building is plain host data; vrod_solver_* drive the CUDA Solver (solver.cu);
// the fine-grained collision entry points run on the GPU (standalone.cu). Exceptions map to
// status codes with the reference's messages (types.h:25-28, 67-77).
#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vrod_bench.h"
#include "../../include/vrod_capi.h"
#include "host_model.h"
#include "skin.h"
#include "solver.h"
#include "standalone.h"

using namespace vhost;
using vm::Q4;
using vm::V3;

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
  } catch (const DeviceError& e) {
    g_error = e.what();
    return VROD_DEVICE_ERROR;
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

V3 v3(const double* p) { return V3{p[0], p[1], p[2]}; }
Q4 q4(const double* p) { return Q4{p[0], p[1], p[2], p[3]}; }
void put3(double* p, const V3& v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
void put4(double* p, const Q4& q) {
  p[0] = q.w;
  p[1] = q.x;
  p[2] = q.y;
  p[3] = q.z;
}
PillData to_pill(const vrod_pill& p) {
  PillData o;
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

}  // namespace

struct vrod_scene {
  SceneData scene;
};
struct vrod_solver {
  std::unique_ptr<Solver> s;
};
struct vrod_skin {
  std::unique_ptr<Skin> k;
};
namespace {
void put_transform(const double* t, vrod_pill_transform* o) {  // device layout: center, scale, wxyz
  std::copy(t, t + 3, o->center);
  o->scale = t[3];
  std::copy(t + 4, t + 8, o->rotation);
}
void get_transform(const vrod_pill_transform& t, double* o) {
  std::copy(t.center, t.center + 3, o);
  o[3] = t.scale;
  std::copy(t.rotation, t.rotation + 4, o + 4);
}
// rod_rest_pill_transforms, skinning.cpp:24-37 (setup-time, host)
std::vector<double> rest_transforms(const SceneData& sc) {
  std::vector<double> out;
  for (const RodData& r : sc.rods)
    for (int e = 0; e + 1 < r.n; ++e) {
      const V3 c = 0.5 * (r.rc[e] + r.rc[e + 1]);
      const Q4& q = r.rq[e];
      out.insert(out.end(), {c.x, c.y, c.z, 0.5 * (r.rs[e] + r.rs[e + 1]), q.w, q.x, q.y, q.z});
    }
  return out;
}
// rod_rest_pills, skinning.cpp:39-57 (setup-time, host)
std::vector<PillData> rest_pills(const SceneData& sc) {
  std::vector<PillData> out;
  for (int ri = 0; ri < static_cast<int>(sc.rods.size()); ++ri) {
    const RodData& r = sc.rods[ri];
    for (int e = 0; e + 1 < r.n; ++e) {
      PillData p;
      p.c0 = r.rc[e];
      p.c1 = r.rc[e + 1];
      p.r0 = r.rs[e] * r.r[e];
      p.r1 = r.rs[e + 1] * r.r[e + 1];
      p.rod = ri;
      p.element = e;
      out.push_back(p);
    }
  }
  return out;
}
void put_pill(const PillData& p, vrod_pill* o) {
  put3(o->c0, p.c0);
  put3(o->c1, p.c1);
  o->r0 = p.r0;
  o->r1 = p.r1;
  o->rod = p.rod;
  o->element = p.element;
  o->group = p.group;
  o->self_collide = p.self_collide ? 1 : 0;
}
}  // namespace

extern "C" {

const char* vrod_last_error(void) { return g_error.c_str(); }
const char* vrod_backend_name(void) { return "b200-cuda"; }
int32_t vrod_capi_version(void) { return VROD_CAPI_VERSION; }

void vrod_default_material(vrod_material* o) {
  const Material m;
  *o = {m.sx, m.sy, m.sz, m.bx, m.by, m.bz, m.vol, m.rho};
}
void vrod_default_settings(vrod_settings* o) {
  const Settings s;
  o->dt = s.dt;
  o->iterations = s.iterations;
  o->substeps = s.substeps;
  o->beta = s.beta;
  put3(o->gravity, s.g);
  o->dichotomous_iterations = s.dich;
  o->shape_match_period = s.sm_period;
  o->contact_stiffness = s.contact_k;
  o->velocity_damping = s.damping;
  o->deterministic = 0;
  o->scale_mode = 0;
}

int vrod_make_rest_pose(int32_t n, const double* centers, int32_t nr, const double* radii, int32_t ns,
                        const double* scales, vrod_rest_pose_out* out) {
  return guarded([&] {
    std::vector<V3> c;
    for (int i = 0; i < n; ++i) c.push_back(v3(centers + 3 * i));
    RodData rod;
    make_rest_pose(rod, c, std::vector<double>(radii, radii + nr),
                   std::vector<double>(scales, scales + (scales ? ns : 0)));
    const int m = n - 1;
    for (int i = 0; i < n; ++i) {
      out->rest_scales[i] = rod.rs[i];
      out->radii[i] = rod.r[i];
    }
    for (int e = 0; e < m; ++e) {
      out->lengths[e] = rod.len[e];
      out->initial_lengths[e] = rod.len0[e];
      put4(out->rest_frames + 4 * e, rod.rq[e]);
      out->tangent_dots[e] = rod.tdot[e];
      out->scale_grads[e] = rod.sgrad[e];
    }
    for (int j = 0; j + 1 < m; ++j) {
      put3(out->darboux + 3 * j, rod.darb[j]);
      out->scale_laplacians[j] = rod.slap[j];
    }
  });
}

int vrod_scene_create(vrod_scene** out) {
  return guarded([&] { *out = new vrod_scene(); });
}
void vrod_scene_destroy(vrod_scene* s) { delete s; }

int vrod_scene_set_settings(vrod_scene* s, const vrod_settings* in) {
  return guarded([&] {
    Settings& o = s->scene.settings;
    o.dt = in->dt;
    o.iterations = in->iterations;
    o.substeps = in->substeps;
    o.beta = in->beta;
    o.g = v3(in->gravity);
    o.dich = in->dichotomous_iterations;
    o.sm_period = in->shape_match_period;
    o.contact_k = in->contact_stiffness;
    o.damping = in->velocity_damping;
    o.deterministic = in->deterministic != 0;
    o.scale_mode = in->scale_mode;
  });
}
int vrod_scene_add_material(vrod_scene* s, const vrod_material* m) {
  return guarded([&] {
    s->scene.materials.push_back(
        Material{m->stretch_x, m->stretch_y, m->stretch_z, m->bend_x, m->bend_y, m->bend_z, m->volume, m->density});
  });
}
int vrod_scene_add_rod(vrod_scene* s, const vrod_rod_desc* d) {
  return guarded([&] {
    const int n = d->vertex_count, m = n - 1;
    if (n < 2) throw std::invalid_argument("rest pose: need at least 2 vertices");
    RodData rod;
    rod.n = n;
    for (int i = 0; i < n; ++i) {
      rod.rc.push_back(v3(d->rest_centers + 3 * i));
      rod.rs.push_back(d->rest_scales[i]);
      rod.r.push_back(d->radii[i]);
      rod.c.push_back(v3(d->centers + 3 * i));
      rod.s.push_back(d->scales[i]);
      rod.cv.push_back(v3(d->center_vel + 3 * i));
      rod.sv.push_back(d->scale_vel[i]);
      rod.pinned.push_back(d->pinned ? d->pinned[i] : 0);
    }
    for (int e = 0; e < m; ++e) {
      rod.len.push_back(d->lengths[e]);
      rod.len0.push_back(d->initial_lengths[e]);
      rod.rq.push_back(q4(d->rest_frames + 4 * e));
      rod.tdot.push_back(d->tangent_dots[e]);
      rod.sgrad.push_back(d->scale_grads[e]);
      rod.q.push_back(q4(d->frames + 4 * e));
      rod.av.push_back(v3(d->angular_vel + 3 * e));
    }
    for (int j = 0; j + 1 < m; ++j) {
      rod.darb.push_back(v3(d->darboux + 3 * j));
      rod.slap.push_back(d->scale_laplacians[j]);
    }
    rod.material = d->material;
    rod.group = d->collision_group;
    rod.self_collide = d->self_collide != 0;
    for (int b = 0; b < d->bone_count; ++b) rod.bones.push_back(d->bones[b]);
    if (d->bone_count > 0) rod.bone_w.assign(d->bone_weights, d->bone_weights + static_cast<std::size_t>(n) * d->bone_count);
    s->scene.rods.push_back(std::move(rod));
  });
}
int vrod_scene_add_plane(vrod_scene* s, const double normal[3], double offset) {
  return guarded([&] { s->scene.planes.emplace_back(v3(normal), offset); });
}
int vrod_scene_add_bone(vrod_scene* s, int32_t k, const double* t, const double* pos, const double* rot) {
  return guarded([&] {
    BoneData b;
    for (int i = 0; i < k; ++i) b.keys.push_back(Key{t[i], v3(pos + 3 * i), q4(rot + 4 * i)});
    s->scene.bones.push_back(std::move(b));
  });
}
int vrod_scene_add_kinematic_pill(vrod_scene* s, const vrod_pill* p, int32_t bone) {
  return guarded([&] { s->scene.kpills.push_back(KinPill{to_pill(*p), bone}); });
}
int vrod_scene_add_bundle(vrod_scene* s, int32_t count, const int32_t* rods, const int32_t* verts) {
  return guarded([&] {
    std::vector<std::pair<int, int>> m;
    for (int i = 0; i < count; ++i) m.emplace_back(rods[i], verts[i]);
    s->scene.bundles.push_back(std::move(m));
  });
}
int vrod_scene_add_pin_motion(vrod_scene* s, int32_t rod, int32_t vertex, const double start[3],
                              const double target[3], double t0, double t1) {
  return guarded([&] { s->scene.pin_motions.push_back(PinMotion{rod, vertex, v3(start), v3(target), t0, t1}); });
}
int vrod_scene_add_soft_pin(vrod_scene* s, int32_t rod, int32_t vertex, const double target[3], double k) {
  return guarded([&] { s->scene.soft_pins.push_back(SoftPin{rod, vertex, v3(target), k}); });
}
int vrod_scene_add_activation(vrod_scene* s, int32_t rod, double factor, double t_start, double t_end, int32_t first,
                              int32_t last) {
  return guarded([&] { s->scene.activations.push_back(Activation{rod, factor, t_start, t_end, first, last}); });
}
int vrod_scene_validate(const vrod_scene* s) {
  return guarded([&] { s->scene.validate(); });
}

int vrod_solver_create(const vrod_scene* s, vrod_solver** out) {
  return guarded([&] {
    auto h = std::make_unique<vrod_solver>();
    h->s = std::make_unique<Solver>(s->scene);
    *out = h.release();
  });
}
void vrod_solver_destroy(vrod_solver* s) { delete s; }

static void put_report(const Report& r, vrod_step_report* out) {
  std::memset(out, 0, sizeof(*out));
  out->step = r.step;
  out->time = r.time;
  for (int k = 0; k < 8; ++k) out->residuals[k] = r.residuals[k];
  out->max_penetration = r.max_pen;
  out->contact_count = r.contacts;
  out->broad_pairs = r.broad;
  out->skipped_singular = r.singular;
  out->dof_count = r.dof;
  out->predict_ms = r.predict_ms;
  out->broad_ms = r.broad_ms;
  out->narrow_ms = r.narrow_ms;
  out->solve_ms = r.solve_ms;
  out->finalize_ms = r.finalize_ms;
  out->total_ms = r.total_ms;
}

int vrod_solver_step(vrod_solver* h, vrod_step_report* out) {
  return guarded([&] {
    Report r = h->s->step();
    if (h->s->scene_count() > 1) {  // batch total: maxima over scenes, counters summed (saturating)
      for (int k = 0; k < 8; ++k) r.residuals[k] = 0.0;
      r.max_pen = 0.0;
      long long ct = 0, bp = 0, sg = 0;
      for (const Report& sr : h->s->scene_reports()) {
        for (int k = 0; k < 8; ++k) r.residuals[k] = std::max(r.residuals[k], sr.residuals[k]);
        r.max_pen = std::max(r.max_pen, sr.max_pen);
        ct += sr.contacts;
        bp += sr.broad;
        sg += sr.singular;
      }
      const auto sat = [](long long v) { return static_cast<int>(std::min<long long>(v, 2147483647ll)); };
      r.contacts = sat(ct);
      r.broad = sat(bp);
      r.singular = sat(sg);
    }
    put_report(r, out);
  });
}

int vrod_batch_create(int32_t n, const vrod_scene* const* scenes, vrod_solver** out) {
  return guarded([&] {
    require(n >= 1 && scenes != nullptr, "batch needs at least one scene");
    std::vector<const SceneData*> list;
    for (int i = 0; i < n; ++i) list.push_back(&scenes[i]->scene);
    BatchLayout layout;
    const SceneData merged = merge_scenes(list, layout);
    auto h = std::make_unique<vrod_solver>();
    h->s = std::make_unique<Solver>(merged, &layout);
    *out = h.release();
  });
}
int vrod_solver_scene_count(const vrod_solver* h, int32_t* count) {
  return guarded([&] { *count = h->s->scene_count(); });
}
int vrod_solver_scene_reports(const vrod_solver* h, int32_t capacity, vrod_step_report* reports) {
  return guarded([&] {
    const std::vector<Report> rs = h->s->scene_reports();
    require(capacity >= static_cast<int32_t>(rs.size()), "scene report capacity too small");
    for (std::size_t i = 0; i < rs.size(); ++i) put_report(rs[i], reports + i);
  });
}
int vrod_solver_probe_convergence(vrod_solver* h, int32_t iterations, double* log) {
  return guarded([&] {
    const std::vector<double> rows = h->s->probe_convergence(iterations);
    std::memcpy(log, rows.data(), sizeof(double) * rows.size());
  });
}
int vrod_solver_get_info(const vrod_solver* h, vrod_solver_info* info) {
  return guarded([&] {
    const Solver& s = *h->s;
    std::memset(info, 0, sizeof(*info));
    info->rod_count = s.rod_count();
    info->total_vertices = s.total_vertices();
    info->total_elements = s.total_elements();
    info->dof_count = s.dof_count();
    info->step_index = s.step_index();
    info->bundle_count = s.bundle_count();
    info->elastic_blocks = s.elastic_blocks();
    info->time = s.time();
  });
}
int vrod_solver_get_rod_sizes(const vrod_solver* h, int32_t* counts) {
  return guarded([&] {
    const auto& rods = h->s->scene().rods;
    for (std::size_t r = 0; r < rods.size(); ++r) counts[r] = rods[r].n;
  });
}
int vrod_solver_get_state(vrod_solver* h, double* c, double* sc, double* f, double* cv, double* sv, double* av) {
  return guarded([&] { h->s->get_state(c, sc, f, cv, sv, av); });
}
int vrod_solver_set_option(vrod_solver* h, const char* name, int64_t value) {
  return guarded([&] {
    require(name != nullptr && h->s->set_option(name, value), "unknown solver option");
  });
}
int vrod_solver_set_state(vrod_solver* h, const double* c, const double* sc, const double* f, const double* cv,
                          const double* sv, const double* av) {
  return guarded([&] { h->s->set_state(c, sc, f, cv, sv, av); });
}
int vrod_solver_get_rest(vrod_solver* h, double* lengths, double* darb, double* grads, double* laps) {
  return guarded([&] { h->s->get_rest(lengths, darb, grads, laps); });
}
int vrod_solver_set_loads(vrod_solver* h, const double* fd, const uint8_t* fdr, const double* tq, const uint8_t* tqr,
                          const double* sl, const uint8_t* slr) {
  return guarded([&] { h->s->set_loads(fd, fdr, tq, tqr, sl, slr); });
}
int vrod_solver_energy(vrod_solver* h, double* ke, double* vol, double* rvol) {
  return guarded([&] { h->s->energy(ke, vol, rvol); });
}
int vrod_solver_get_weights(vrod_solver* h, double* cw, double* sw, double* tw) {
  return guarded([&] { h->s->weights(cw, sw, tw); });
}
int vrod_solver_get_inverse_weights(vrod_solver* h, double* ic, double* is, double* it) {
  return guarded([&] { h->s->inverse_weights(ic, is, it); });
}
int vrod_solver_get_contacts(vrod_solver* h, int64_t cap, int64_t* count, int32_t* a, int32_t* b, double* alpha,
                             double* beta) {
  return guarded([&] { *count = h->s->contacts(cap, a, b, alpha, beta); });
}
int vrod_solver_pill_transforms(vrod_solver* h, int64_t cap, int64_t* count, vrod_pill_transform* out) {
  return guarded([&] {
    const std::vector<double> t = h->s->pill_transforms();
    const int64_t n = static_cast<int64_t>(t.size() / 8);
    for (int64_t i = 0; i < n && i < cap; ++i) put_transform(t.data() + 8 * i, out + i);
    *count = n;
  });
}
int vrod_solver_rest_pill_transforms(vrod_solver* h, int64_t cap, int64_t* count, vrod_pill_transform* out) {
  return guarded([&] {
    const std::vector<double> t = rest_transforms(h->s->scene());
    const int64_t n = static_cast<int64_t>(t.size() / 8);
    for (int64_t i = 0; i < n && i < cap; ++i) put_transform(t.data() + 8 * i, out + i);
    *count = n;
  });
}
int vrod_solver_rest_pills(vrod_solver* h, int64_t cap, int64_t* count, vrod_pill* out) {
  return guarded([&] {
    const auto p = rest_pills(h->s->scene());
    for (std::size_t i = 0; i < p.size() && static_cast<int64_t>(i) < cap; ++i) put_pill(p[i], out + i);
    *count = static_cast<int64_t>(p.size());
  });
}
int vrod_skin_bind(int32_t nv, const double* verts, int32_t nt, const int32_t* tris, int32_t np, const vrod_pill* pills,
                   const vrod_pill_transform* rest, int32_t max_influences, double epsilon, vrod_skin** out) {
  return guarded([&] {
    std::vector<V3> v(nv > 0 ? nv : 0);
    for (int32_t i = 0; i < nv; ++i) v[i] = v3(verts + 3 * i);
    std::vector<std::array<int, 3>> t(nt > 0 ? nt : 0);
    for (int32_t i = 0; i < nt; ++i) t[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    std::vector<PillData> p(np > 0 ? np : 0);
    std::vector<double> tr(8ull * p.size());
    for (int32_t i = 0; i < np; ++i) {
      p[i] = to_pill(pills[i]);
      get_transform(rest[i], tr.data() + 8ll * i);
    }
    auto sk = std::make_unique<vrod_skin>();
    sk->k = std::make_unique<Skin>(v, t, p, tr, max_influences, epsilon);
    *out = sk.release();
  });
}
void vrod_skin_destroy(vrod_skin* sk) { delete sk; }
int vrod_skin_smooth(vrod_skin* sk, int32_t iterations) {
  return guarded([&] { sk->k->smooth(iterations); });
}
int vrod_skin_get_binding(const vrod_skin* sk, int32_t* offsets, int32_t* pills, double* weights, int32_t* nnz,
                          int32_t* clamped) {
  return guarded([&] { sk->k->get_binding(offsets, pills, weights, nnz, clamped); });
}
int vrod_skin_deform(vrod_skin* sk, int32_t np, const vrod_pill_transform* cur, double* out) {
  return guarded([&] {
    std::vector<double> t(8ull * (np > 0 ? np : 0));
    for (int32_t i = 0; i < np; ++i) get_transform(cur[i], t.data() + 8ll * i);
    sk->k->deform(np, t.data(), out);
  });
}
int vrod_skin_deform_solver(vrod_skin* sk, vrod_solver* h, double* out) {
  return guarded([&] { sk->k->deform_solver(*h->s, out); });
}

int vrod_solver_shape_match(vrod_solver* h, int32_t cap, int32_t* count, double* fits) {
  return guarded([&] {
    const std::vector<double> f = h->s->shape_match();
    const int32_t n = static_cast<int32_t>(f.size() / 14);
    if (fits) std::copy(f.begin(), f.begin() + 14ll * std::min(n, std::max(cap, 0)), fits);
    *count = n;
  });
}
int vrod_solver_jacobi_sweep(vrod_solver* h, double step, double beta, int32_t* active, int32_t* singular) {
  return guarded([&] {
    const auto o = h->s->jacobi_sweep(step, beta);
    if (active) *active = o.first;
    if (singular) *singular = o.second;
  });
}
int vrod_solver_elastic_residuals(vrod_solver* h, int64_t cap, int64_t* count, double* W) {
  return guarded([&] {
    const std::vector<double> r = h->s->elastic_residuals();
    const int64_t n = static_cast<int64_t>(r.size() / 3);
    if (W) std::copy(r.begin(), r.begin() + 3 * std::min(n, std::max<int64_t>(cap, 0)), W);
    *count = n;
  });
}
int vrod_extract_rotation(int64_t n, const double* B, const double* guess, int32_t max_iterations, double tolerance,
                          double* out) {
  return guarded([&] { gpu_extract_rotation(n, B, guess, max_iterations, tolerance, out); });
}

int vrod_solver_current_pills(vrod_solver* h, int64_t cap, int64_t* count, vrod_pill* out) {
  return guarded([&] {
    const auto pills = h->s->current_pills();
    for (std::size_t i = 0; i < pills.size() && static_cast<int64_t>(i) < cap; ++i) {
      const PillData& p = pills[i];
      put3(out[i].c0, p.c0);
      put3(out[i].c1, p.c1);
      out[i].r0 = p.r0;
      out[i].r1 = p.r1;
      out[i].rod = p.rod;
      out[i].element = p.element;
      out[i].group = p.group;
      out[i].self_collide = p.self_collide ? 1 : 0;
    }
    *count = static_cast<int64_t>(pills.size());
  });
}

int vrod_pill_project(int64_t n, const double* x, const vrod_pill* pills, double* t, double* d, uint8_t* deg) {
  return guarded([&] { gpu_pill_project(n, x, pills, t, d, deg); });
}
int vrod_deepest_penetration(int64_t n, const vrod_pill* a, const vrod_pill* b, int32_t iters, const double* warm,
                             double* alpha, double* beta, double* dist) {
  return guarded([&] { gpu_deepest(n, a, b, iters, warm, alpha, beta, dist); });
}
int vrod_broad_phase(int64_t n, const vrod_pill* pills, int64_t cap, int64_t* count, int32_t* pairs) {
  return guarded([&] { *count = gpu_broad_phase(n, pills, cap, pairs); });
}
int vrod_find_contacts(int64_t n, const vrod_pill* pills, int64_t np, const int32_t* pairs, int32_t iters, int64_t nw,
                       const uint64_t* wk, const double* wa, int64_t cap, int64_t* count, int32_t* pa, int32_t* pb,
                       double* alpha, double* beta, double* dist) {
  return guarded([&] { *count = gpu_find_contacts(n, pills, np, pairs, iters, nw, wk, wa, cap, pa, pb, alpha, beta, dist); });
}
int vrod_bench_run(vrod_solver* h, int32_t steps, int64_t flush_bytes, double* device_ms, int64_t* kernels) {
  return guarded([&] {
    *device_ms = h->s->bench_run(steps, flush_bytes);
    if (kernels) *kernels = h->s->kernel_nodes_per_step();
  });
}
int vrod_bench_kernel_times(vrod_solver* h, int32_t steps, double* ms, int64_t* launches) {
  return guarded([&] {
    long long l[Solver::kCategories];
    h->s->kernel_times(steps, ms, l);
    for (int c = 0; c < Solver::kCategories; ++c) launches[c] = l[c];
  });
}
int vrod_bench_trace(vrod_solver* h, int32_t cap, int64_t* out, int32_t* count) {
  return guarded([&] {
    std::vector<long long> t(cap > 0 ? cap : -cap);
    *count = h->s->trace(t.data(), cap);
    for (int i = 0; i < *count; ++i) out[i] = t[i];
  });
}
int vrod_bench_skin_deform(vrod_skin* sk, vrod_solver* h, int32_t iterations, double* ms, double* deform_ms) {
  return guarded([&] { sk->k->bench(*h->s, iterations, ms, deform_ms); });
}
int vrod_bench_last_counts(vrod_solver* h, int64_t* cand, int64_t* ct) {
  return guarded([&] {
    if (cand) *cand = h->s->last_max_candidates();
    if (ct) *ct = h->s->last_max_contacts();
  });
}

uint64_t vrod_pair_key(const vrod_pill* a, const vrod_pill* b) {  // collision.cpp:240-249
  auto id = [](const vrod_pill& p) {
    return (static_cast<uint32_t>(p.rod + 1) << 16) | (static_cast<uint32_t>(p.element + 1) & 0xffffu);
  };
  uint32_t ia = id(*a), ib = id(*b);
  if (ia > ib) std::swap(ia, ib);
  return (static_cast<uint64_t>(ia) << 32) | ib;
}

}  // extern "C"
