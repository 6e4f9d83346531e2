// Host setup path of the product: validation, rest pose, layout, constraint kinds, bundle
// groups, animation inputs. See host_model.h for the reference functions each part follows.
#include "host_model.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <set>

namespace vhost {

using namespace vm;

static bool is_unit(const Q4& q, double tol = 1e-6) { return std::abs(qnorm(q) - 1.0) <= tol; }

// ---- scene.cpp:22-61 -----------------------------------------------------------------------

V3 BoneData::position_at(double t) const {
  if (keys.empty()) return V3{0, 0, 0};
  if (t <= keys.front().t) return keys.front().p;
  if (t >= keys.back().t) return keys.back().p;
  for (std::size_t k = 1; k < keys.size(); ++k) {
    if (t <= keys[k].t) {
      const double span = keys[k].t - keys[k - 1].t;
      const double f = span > 0.0 ? (t - keys[k - 1].t) / span : 1.0;
      return (1.0 - f) * keys[k - 1].p + f * keys[k].p;
    }
  }
  return keys.back().p;
}

static Q4 slerp(const Q4& a, double t, const Q4& b) {  // Eigen QuaternionBase::slerp
  const double one = 1.0 - std::numeric_limits<double>::epsilon();
  const double d = qdot(a, b);
  const double absD = std::abs(d);
  double s0, s1;
  if (absD >= one) {
    s0 = 1.0 - t;
    s1 = t;
  } else {
    const double theta = std::acos(absD);
    const double sinTheta = std::sin(theta);
    s0 = std::sin((1.0 - t) * theta) / sinTheta;
    s1 = std::sin(t * theta) / sinTheta;
  }
  if (d < 0.0) s1 = -s1;
  return Q4{s0 * a.w + s1 * b.w, s0 * a.x + s1 * b.x, s0 * a.y + s1 * b.y, s0 * a.z + s1 * b.z};
}

Q4 BoneData::rotation_at(double t) const {
  if (keys.empty()) return Q4{1, 0, 0, 0};
  if (t <= keys.front().t) return keys.front().r;
  if (t >= keys.back().t) return keys.back().r;
  for (std::size_t k = 1; k < keys.size(); ++k) {
    if (t <= keys[k].t) {
      const double span = keys[k].t - keys[k - 1].t;
      const double f = span > 0.0 ? (t - keys[k - 1].t) / span : 1.0;
      return slerp(keys[k - 1].r, f, keys[k].r);
    }
  }
  return keys.back().r;
}

V3 PinMotion::position_at(double t) const {
  if (t <= t0) return start;
  if (t >= t1) return target;
  const double f = (t - t0) / (t1 - t0);
  return (1.0 - f) * start + f * target;
}

double Activation::amount_at(double t) const {
  if (t <= t_start) return 0.0;
  if (t >= t_end) return 1.0;
  return (t - t_start) / (t_end - t_start);
}

// ---- rod.cpp -------------------------------------------------------------------------------

void validate_rest(const RodData& r) {  // rod.cpp:15-34
  const int n = static_cast<int>(r.rc.size());
  const int m = static_cast<int>(r.rq.size());
  require(n >= 2, "rest pose: need at least 2 vertices");
  require(m == n - 1, "rest pose: frame count must be vertex count - 1");
  require(r.rs.size() == r.rc.size(), "rest pose: scales size mismatch");
  require(r.r.size() == r.rc.size(), "rest pose: radii size mismatch");
  require(static_cast<int>(r.len.size()) == m, "rest pose: lengths size mismatch");
  require(static_cast<int>(r.len0.size()) == m, "rest pose: initial lengths size mismatch");
  require(static_cast<int>(r.tdot.size()) == m, "rest pose: tangent dots size mismatch");
  require(static_cast<int>(r.sgrad.size()) == m, "rest pose: scale grads size mismatch");
  require(static_cast<int>(r.darb.size()) == std::max(0, m - 1), "rest pose: darboux size mismatch");
  require(static_cast<int>(r.slap.size()) == std::max(0, m - 1), "rest pose: scale laplacians size mismatch");
  for (double l : r.len) require(l > 0, "rest pose: element length must be > 0");
  for (double l : r.len0) require(l > 0, "rest pose: element length must be > 0");
  for (double x : r.r) require(x > 0, "rest pose: radius must be > 0");
  for (double x : r.rs) require(x > 0, "rest pose: scale must be > 0");
  for (const Q4& f : r.rq) require(is_unit(f), "rest pose: frame quaternion not unit");
}

static V3 darboux_vector(const Q4& qa, const Q4& qb, double la, double lb) {  // rod.cpp:157-162
  require(is_unit(qa) && is_unit(qb), "darboux_vector: quaternions must be unit norm");
  require(la > 0 && lb > 0, "darboux_vector: lengths must be > 0");
  return (4.0 / (la + lb)) * qvec(relative_rotation(qa, qb));
}

void make_rest_pose(RodData& rod, const std::vector<V3>& centers, const std::vector<double>& radii,
                    const std::vector<double>& scales) {  // rod.cpp:60-112
  const int n = static_cast<int>(centers.size());
  require(n >= 2, "make_rest_pose: need at least 2 vertices");
  const int m = n - 1;
  rod.n = n;
  rod.rc = centers;
  if (radii.size() == 1) {
    rod.r.assign(n, radii[0]);
  } else {
    require(static_cast<int>(radii.size()) == n, "make_rest_pose: radii must be uniform or per vertex");
    rod.r = radii;
  }
  if (scales.empty()) {
    rod.rs.assign(n, 1.0);
  } else if (scales.size() == 1) {
    rod.rs.assign(n, scales[0]);
  } else {
    require(static_cast<int>(scales.size()) == n, "make_rest_pose: scales must be uniform or per vertex");
    rod.rs = scales;
  }
  rod.len.resize(m);
  std::vector<V3> tan(m);
  for (int e = 0; e < m; ++e) {
    const V3 d = rod.rc[e + 1] - rod.rc[e];
    rod.len[e] = norm(d);
    require(rod.len[e] > 0, "make_rest_pose: coincident consecutive centers");
    tan[e] = d / rod.len[e];
  }
  rod.len0 = rod.len;
  rod.rq.resize(m);
  rod.rq[0] = qnormalized(qfrom_two_vectors(V3{0, 0, 1}, tan[0]));
  for (int e = 1; e < m; ++e) {
    const Q4 dq = qnormalized(qfrom_two_vectors(tan[e - 1], tan[e]));
    rod.rq[e] = qnormalized(qmul(dq, rod.rq[e - 1]));
    if (qdot(rod.rq[e], rod.rq[e - 1]) < 0) rod.rq[e] = qneg(rod.rq[e]);
  }
  rod.tdot.resize(m);
  for (int e = 0; e < m; ++e) rod.tdot[e] = dot(col(qmat(rod.rq[e]), 2), tan[e]);
  rod.sgrad.resize(m);
  for (int e = 0; e < m; ++e) rod.sgrad[e] = (rod.rs[e + 1] - rod.rs[e]) / rod.len[e];
  rod.darb.resize(std::max(0, m - 1));
  rod.slap.resize(std::max(0, m - 1));
  for (int j = 1; j < m; ++j) {
    rod.darb[j - 1] = darboux_vector(rod.rq[j - 1], rod.rq[j], rod.len[j - 1], rod.len[j]);
    rod.slap[j - 1] = (rod.rs[j + 1] - rod.rs[j]) / rod.len[j] - (rod.rs[j] - rod.rs[j - 1]) / rod.len[j - 1];
  }
  validate_rest(rod);
}

// ---- scene.cpp:8-20, 63-157 ----------------------------------------------------------------

static void validate_settings(const Settings& s) {
  require(s.dt > 0.0 && std::isfinite(s.dt), "settings.dt must be positive and finite");
  require(s.iterations >= 1, "settings.iterations must be at least 1");
  require(s.substeps >= 1, "settings.substeps must be at least 1");
  require(s.beta > 0.0 && s.beta <= 1.0, "settings.beta must be in (0, 1]");
  require(finite3(s.g), "settings.gravity must be finite");
  require(s.dich >= 1, "settings.dichotomous_iterations must be at least 1");
  require(s.sm_period >= 1, "settings.shape_match_period must be at least 1");
  require(s.contact_k > 0.0, "settings.contact_stiffness must be positive");
  require(s.damping >= 0.0 && s.damping < 1.0, "settings.velocity_damping must be in [0, 1)");
}

static void validate_material(const Material& m) {  // rod.cpp:8-13
  require(m.sx >= 0 && m.sy >= 0 && m.sz >= 0, "material: stretch stiffness must be >= 0");
  require(m.bx >= 0 && m.by >= 0 && m.bz >= 0, "material: bend stiffness must be >= 0");
  require(m.vol >= 0, "material: volume stiffness must be >= 0");
  require(m.rho > 0, "material: density must be > 0");
}

void SceneData::validate() const {
  validate_settings(settings);
  require(!materials.empty(), "scene needs at least one material");
  for (const Material& m : materials) validate_material(m);
  const int rc = static_cast<int>(rods.size());
  for (int r = 0; r < rc; ++r) {
    const RodData& rod = rods[r];
    validate_rest(rod);
    const std::string where = "rod " + std::to_string(r);
    require_index(rod.material, static_cast<int>(materials.size()), where + " material");
    const int n = static_cast<int>(rod.rc.size());
    require(static_cast<int>(rod.pinned.size()) == n, where + " pinned flags size");
    require(static_cast<int>(rod.c.size()) == n, where + " state size");
    require(rod.q.size() == rod.rq.size(), where + " frame count");
    if (!rod.bones.empty()) {
      const std::size_t nb = rod.bones.size();
      require(rod.bone_w.size() == static_cast<std::size_t>(n) * nb, where + " bone weights per vertex");
      for (int b : rod.bones) require_index(b, static_cast<int>(bones.size()), where + " bone index");
      for (int v = 0; v < n; ++v) {
        double sum = 0.0;
        for (std::size_t b = 0; b < nb; ++b) sum += rod.bone_w[v * nb + b];
        require(std::abs(sum - 1.0) < 1e-6, where + " bone weights must sum to 1");
      }
    }
  }
  for (const auto& p : planes) require(std::abs(norm(p.first) - 1.0) < 1e-9, "plane normal must be unit length");
  for (const KinPill& kp : kpills) {
    require(kp.pill.rod < 0, "kinematic pill must not reference a rod");
    require(kp.pill.r0 > 0.0 && kp.pill.r1 > 0.0, "kinematic pill radii must be positive");
    require(finite3(kp.pill.c0) && finite3(kp.pill.c1), "kinematic pill centers must be finite");
    require(kp.bone < static_cast<int>(bones.size()), "kinematic pill bone out of range");
    if (kp.bone >= 0) require(!bones[kp.bone].keys.empty(), "kinematic pill bone has no keyframes");
  }
  // one flag per (rod, vertex): linear in the member count (batches merge ~10^7 members)
  std::vector<std::size_t> vbase(rc + 1, 0);
  for (int r = 0; r < rc; ++r) vbase[r + 1] = vbase[r] + rods[r].rc.size();
  std::vector<uint8_t> seen(bundles.empty() ? 0 : vbase[rc], 0);
  for (const auto& members : bundles) {
    require(members.size() >= 2, "bundle needs at least two members");
    for (const auto& [mr, mv] : members) {
      require_index(mr, rc, "bundle member rod");
      require_index(mv, static_cast<int>(rods[mr].rc.size()), "bundle member vertex");
      uint8_t& f = seen[vbase[mr] + mv];
      require(!f, "bundle groups must not share a vertex");
      f = 1;
    }
  }
  for (const PinMotion& pm : pin_motions) {
    require_index(pm.rod, rc, "pin motion rod");
    require_index(pm.vertex, static_cast<int>(rods[pm.rod].rc.size()), "pin motion vertex");
    require(rods[pm.rod].pinned[pm.vertex] != 0, "pin motion requires a pinned vertex");
    require(pm.t1 >= pm.t0, "pin motion must have t1 >= t0");
  }
  for (const SoftPin& sp : soft_pins) {
    require_index(sp.rod, rc, "soft pin rod");
    require_index(sp.vertex, static_cast<int>(rods[sp.rod].rc.size()), "soft pin vertex");
    require(sp.k > 0.0, "soft pin stiffness must be positive");
  }
  for (const Activation& a : activations) {
    require_index(a.rod, rc, "activation rod");
    require(a.factor >= 0.0 && a.factor < 1.0, "activation factor must be in [0, 1)");
    require(a.t_end >= a.t_start, "activation must have t_end >= t_start");
    const int m = static_cast<int>(rods[a.rod].rq.size());
    require(a.first >= 0 && a.first < m, "activation first element");
    require(a.last == -1 || (a.last >= a.first && a.last < m), "activation last element");
  }
}

// ---- constraint kinds (constraints.cpp:282-329) -------------------------------------------

int element_kinds(const Material& m, bool scale_kinds) {
  const double kxy = m.sx + m.sy;
  int k = 0;
  if (m.sz > 0) k |= 1;
  if (scale_kinds && kxy > 0) k |= 2 | 4;
  if (scale_kinds && m.vol > 0) k |= 8;
  return k;
}
int vertex_kinds(const Material& m, bool scale_kinds) {
  const double kxy = m.sx + m.sy;
  const double bxy = m.bx + m.by;
  int k = 0;
  if (m.sz > 0 || kxy > 0) k |= 1;
  if (scale_kinds && bxy > 0) k |= 2;
  if (scale_kinds && m.vol > 0) k |= 4 | 8;
  return k;
}
int popcount4(int b) { return (b & 1) + ((b >> 1) & 1) + ((b >> 2) & 1) + ((b >> 3) & 1); }

Setup build_setup(const SceneData& s) {
  Setup out;
  const bool scale_kinds = s.settings.scale_mode == 0;
  out.R = static_cast<int>(s.rods.size());
  out.vbase.resize(out.R);
  out.ebase.resize(out.R);
  out.block_base.resize(out.R);
  out.ekinds.resize(out.R);
  out.vkinds.resize(out.R);
  int blocks = 0;
  for (int r = 0; r < out.R; ++r) {
    const RodData& rod = s.rods[r];
    out.vbase[r] = out.V;
    out.ebase[r] = out.E;
    out.V += rod.n;
    out.E += rod.n - 1;
    const Material& mat = s.materials[rod.material];
    out.ekinds[r] = static_cast<uint8_t>(element_kinds(mat, scale_kinds));
    out.vkinds[r] = static_cast<uint8_t>(vertex_kinds(mat, scale_kinds));
    out.block_base[r] = blocks;
    const int m = rod.n - 1;
    blocks += m * popcount4(out.ekinds[r]) + std::max(0, m - 1) * popcount4(out.vkinds[r]);
  }
  out.elastic_blocks = blocks;
  out.vpad = std::max(32, (out.V + 31) / 32 * 32);

  // Shape-matching groups (make_bundle_group, bundling.cpp:17-48) + level schedule.
  // frame slot -> highest level that wrote it so far; per-slot stamps find a group's distinct
  // frames (flat arrays: batches merge ~10^6 groups)
  std::vector<int> last_level(out.V, -1), stamp(out.V, -1), last_writer(out.V, -1);
  // chain schedule: a group's predecessor is the last earlier group that wrote one of its frames
  std::vector<int> pred, nsucc;
  bool chains_ok = true;
  for (const auto& members : s.bundles) {
    const int gid = static_cast<int>(out.groups.size());
    Setup::Group g;
    require(!members.empty(), "bundle group needs at least one member");
    const int n = static_cast<int>(members.size());
    V3 cent{0, 0, 0};
    for (const auto& [mr, mv] : members) {
      require_index(mr, out.R, "bundle member rod");
      require_index(mv, s.rods[mr].n, "bundle member vertex");
      cent = cent + s.rods[mr].rc[mv];
    }
    cent = cent / static_cast<double>(n);
    g.rcent = cent;
    double denom = 0.0;
    std::vector<int> frames;
    for (const auto& [mr, mv] : members) {
      const RodData& rod = s.rods[mr];
      const int e = std::min(mv, rod.n - 2);
      const V3 c = rod.rc[mv] - cent;
      const double sc = rod.rs[mv];
      const M3 R = qmat(rod.rq[e]);
      g.slot.push_back(out.vbase[mr] + mv);
      g.eslot.push_back(out.vbase[mr] + e);
      g.rc.push_back(c);
      g.rs.push_back(sc);
      g.rR.push_back(R);
      g.qR.push_back(qfrom_mat(R));
      denom += sqnorm(c) + 3.0 * sc * sc;
      const int f = out.vbase[mr] + e;
      if (stamp[f] == gid) {
        g.serial_apply = true;
      } else {
        stamp[f] = gid;
        frames.push_back(f);
      }
    }
    g.denom = denom;
    int level = 0;
    for (int f : frames)
      if (last_level[f] >= 0) level = std::max(level, last_level[f] + 1);
    for (int f : frames) last_level[f] = std::max(last_level[f], level);
    int p = -1;
    for (int f : frames) {
      const int lw = last_writer[f];
      if (lw < 0) continue;
      if (p >= 0 && lw != p) chains_ok = false;  // two predecessors: not a chain
      p = lw;
    }
    for (int f : frames) last_writer[f] = gid;
    pred.push_back(p);
    nsucc.push_back(0);
    if (p >= 0 && ++nsucc[p] > 1) chains_ok = false;  // a fork: not a chain
    out.group_level.push_back(level);
    out.levels = std::max(out.levels, level + 1);
    out.groups.push_back(std::move(g));
  }

  // Chains: each group has <= 1 predecessor and <= 1 successor, so the dependency graph is a set
  // of chains; one warp runs a chain's groups in order and chains run concurrently.
  if (chains_ok && !out.groups.empty()) {
    const int G = static_cast<int>(out.groups.size());
    std::vector<int> next(G, -1);
    for (int gi = 0; gi < G; ++gi)
      if (pred[gi] >= 0) next[pred[gi]] = gi;
    out.chain_off.push_back(0);
    for (int gi = 0; gi < G; ++gi) {
      if (pred[gi] >= 0) continue;  // not a chain head
      for (int k = gi; k >= 0; k = next[k]) out.chain_groups.push_back(k);
      out.chain_off.push_back(static_cast<int>(out.chain_groups.size()));
    }
  }

  // Pin motions: sequential writes in the reference, so the last motion per vertex wins.
  std::map<std::pair<int, int>, int> last_pm;
  for (int i = 0; i < static_cast<int>(s.pin_motions.size()); ++i)
    last_pm[{s.pin_motions[i].rod, s.pin_motions[i].vertex}] = i;
  for (int i = 0; i < static_cast<int>(s.pin_motions.size()); ++i)
    if (last_pm[{s.pin_motions[i].rod, s.pin_motions[i].vertex}] == i) out.pin_motion_ids.push_back(i);
  return out;
}

}  // namespace vhost

namespace vhost {

static bool same_settings(const Settings& a, const Settings& b) {
  return a.dt == b.dt && a.iterations == b.iterations && a.substeps == b.substeps && a.beta == b.beta &&
         a.g.x == b.g.x && a.g.y == b.g.y && a.g.z == b.g.z && a.dich == b.dich && a.sm_period == b.sm_period &&
         a.contact_k == b.contact_k && a.damping == b.damping && a.deterministic == b.deterministic &&
         a.scale_mode == b.scale_mode;
}

SceneData merge_scenes(const std::vector<const SceneData*>& scenes, BatchLayout& layout) {
  require(!scenes.empty(), "batch needs at least one scene");
  SceneData out;
  out.settings = scenes[0]->settings;
  layout = BatchLayout{};
  layout.scenes = static_cast<int>(scenes.size());
  layout.rod_base.push_back(0);
  for (std::size_t si = 0; si < scenes.size(); ++si) {
    const SceneData& s = *scenes[si];
    s.validate();
    require(same_settings(s.settings, out.settings), "batch scene " + std::to_string(si) +
                                                         ": all scenes of a batch must share one SolverSettings");
    const int rb = static_cast<int>(out.rods.size());
    const int mb = static_cast<int>(out.materials.size());
    const int bb = static_cast<int>(out.bones.size());
    for (RodData rod : s.rods) {
      rod.material += mb;
      for (int& b : rod.bones) b += bb;
      out.rods.push_back(std::move(rod));
    }
    out.materials.insert(out.materials.end(), s.materials.begin(), s.materials.end());
    for (const auto& p : s.planes) {
      out.planes.push_back(p);
      layout.plane_scene.push_back(static_cast<int>(si));
    }
    for (KinPill kp : s.kpills) {
      if (kp.bone >= 0) kp.bone += bb;
      out.kpills.push_back(kp);
      layout.kpill_scene.push_back(static_cast<int>(si));
    }
    out.bones.insert(out.bones.end(), s.bones.begin(), s.bones.end());
    for (auto members : s.bundles) {
      for (auto& m : members) m.first += rb;
      out.bundles.push_back(std::move(members));
    }
    for (PinMotion pm : s.pin_motions) {
      pm.rod += rb;
      out.pin_motions.push_back(pm);
    }
    for (SoftPin sp : s.soft_pins) {
      sp.rod += rb;
      out.soft_pins.push_back(sp);
    }
    for (Activation a : s.activations) {
      a.rod += rb;
      out.activations.push_back(a);
    }
    layout.rod_base.push_back(static_cast<int>(out.rods.size()));
  }
  return out;
}

}  // namespace vhost
