// CPU restatement of the VIPER rod-solver substep — TEST INFRASTRUCTURE ONLY.
//
// This is the parity ORACLE for the B200 product (paper_1906_05260_b200). It restates the
// reference's hot path (`/root/reference/proj/core/src/{rod,layout,constraints,collision,
// bundling,scene,solver}.cpp`) function by function, each citing the file:line it follows,
// and exports the same C-ABI as the product (include/vrod_capi.h). Its arithmetic order
// mirrors the reference compiled against oracle/shim/Eigen (oracle/_ref), and
// tests/test_oracle_pinning.py pins it there bit for bit. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline leg load it — never the product path.

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "vrod_capi.h"
#include "vrod_oracle_math.h"

using namespace vo;

namespace {

constexpr double kPi = 3.141592653589793;  // std::numbers::pi (types.h:18)
constexpr double kMinScale = 1e-4;         // types.h:22
constexpr double kInf = std::numeric_limits<double>::infinity();

struct SimulationError : std::runtime_error {  // types.h:25-28
  using std::runtime_error::runtime_error;
};
inline void require(bool cond, const std::string& what) {  // types.h:67-69
  if (!cond) throw std::invalid_argument(what);
}
inline void require_index(bool cond, const std::string& what) {  // types.h:71-73
  if (!cond) throw std::out_of_range(what);
}
inline void require_index(int i, int count, const std::string& what) {  // types.h:75-77
  if (i < 0 || i >= count) throw std::out_of_range(what + " out of range");
}

// ---- data model (rod.h:13-74, scene.h:25-126) --------------------------------------------

struct Material {
  double sx = 1e4, sy = 1e4, sz = 1e4, bx = 1e3, by = 1e3, bz = 0.0, vol = 1e6, rho = 1000.0;
  void validate() const {  // rod.cpp:8-13
    require(sx >= 0 && sy >= 0 && sz >= 0, "material: stretch stiffness must be >= 0");
    require(bx >= 0 && by >= 0 && bz >= 0, "material: bend stiffness must be >= 0");
    require(vol >= 0, "material: volume stiffness must be >= 0");
    require(rho > 0, "material: density must be > 0");
  }
};

struct Rest {  // RodRestPose, rod.h:30-46
  std::vector<V3> c;
  std::vector<double> s, r, len, len0;
  std::vector<Q> q;
  std::vector<V3> darb;
  std::vector<double> tdot, sgrad, slap;
  int n() const { return static_cast<int>(c.size()); }
  int m() const { return static_cast<int>(q.size()); }
  void validate() const {  // rod.cpp:15-34
    const int nn = n(), mm = m();
    require(nn >= 2, "rest pose: need at least 2 vertices");
    require(mm == nn - 1, "rest pose: frame count must be vertex count - 1");
    require(s.size() == c.size(), "rest pose: scales size mismatch");
    require(r.size() == c.size(), "rest pose: radii size mismatch");
    require(static_cast<int>(len.size()) == mm, "rest pose: lengths size mismatch");
    require(static_cast<int>(len0.size()) == mm, "rest pose: initial lengths size mismatch");
    require(static_cast<int>(tdot.size()) == mm, "rest pose: tangent dots size mismatch");
    require(static_cast<int>(sgrad.size()) == mm, "rest pose: scale grads size mismatch");
    require(static_cast<int>(darb.size()) == std::max(0, mm - 1), "rest pose: darboux size mismatch");
    require(static_cast<int>(slap.size()) == std::max(0, mm - 1), "rest pose: scale laplacians size mismatch");
    for (double l : len) require(l > 0, "rest pose: element length must be > 0");
    for (double l : len0) require(l > 0, "rest pose: element length must be > 0");
    for (double x : r) require(x > 0, "rest pose: radius must be > 0");
    for (double x : s) require(x > 0, "rest pose: scale must be > 0");
    for (const Q& f : q) require(is_unit(f), "rest pose: frame quaternion not unit");
  }
};

struct State {  // RodState, rod.h:50-60
  std::vector<V3> c;
  std::vector<double> s;
  std::vector<Q> q;
  std::vector<V3> cv;
  std::vector<double> sv;
  std::vector<V3> av;
};

struct Rod {  // rod.h:64-74
  Rest rest;
  State st;
  int material = 0;
  std::vector<uint8_t> pinned;
  int group = -1;
  bool self_collide = false;
  std::vector<int> bones;
  std::vector<std::vector<double>> bone_w;
};

struct Pill {  // collision.h:16-25
  V3 c0, c1;
  double r0 = 0, r1 = 0;
  int rod = -1, element = -1, group = -1;
  bool self_collide = false;
};
struct Plane {
  V3 n{0, 0, 1};
  double off = 0;
};
struct Key {
  double t;
  V3 p;
  Q r;
};
struct Bone {  // scene.h:49-53, scene.cpp:22-48
  std::vector<Key> keys;
  V3 position_at(double t) const {
    if (keys.empty()) return V3{0, 0, 0};
    if (t <= keys.front().t) return keys.front().p;
    if (t >= keys.back().t) return keys.back().p;
    for (std::size_t k = 1; k < keys.size(); ++k) {
      if (t <= keys[k].t) {
        const double span = keys[k].t - keys[k - 1].t;
        const double f = span > 0.0 ? (t - keys[k - 1].t) / span : 1.0;
        return add(mul(1.0 - f, keys[k - 1].p), mul(f, keys[k].p));
      }
    }
    return keys.back().p;
  }
  Q rotation_at(double t) const {
    if (keys.empty()) return Q{1, 0, 0, 0};
    if (t <= keys.front().t) return keys.front().r;
    if (t >= keys.back().t) return keys.back().r;
    for (std::size_t k = 1; k < keys.size(); ++k) {
      if (t <= keys[k].t) {
        const double span = keys[k].t - keys[k - 1].t;
        const double f = span > 0.0 ? (t - keys[k - 1].t) / span : 1.0;
        return qslerp(keys[k - 1].r, f, keys[k].r);
      }
    }
    return keys.back().r;
  }
};
struct KinPill {
  Pill pill;
  int bone = -1;
};
struct PinMotion {  // scene.h:62-71, scene.cpp:50-55
  int rod = 0, vertex = 0;
  V3 start, target;
  double t0 = 0, t1 = 0;
  V3 position_at(double t) const {
    if (t <= t0) return start;
    if (t >= t1) return target;
    const double f = (t - t0) / (t1 - t0);
    return add(mul(1.0 - f, start), mul(f, target));
  }
};
struct SoftPin {
  int rod = 0, vertex = 0;
  V3 target;
  double k = kInf;
};
struct Activation {  // scene.h:84-92, scene.cpp:57-61
  int rod = 0;
  double factor = 0.2, t_start = 0.0, t_end = 1.0;
  int first = 0, last = -1;
  double amount_at(double t) const {
    if (t <= t_start) return 0.0;
    if (t >= t_end) return 1.0;
    return (t - t_start) / (t_end - t_start);
  }
};
struct Settings {  // scene.h:25-39
  double dt = 1.0 / 60.0;
  int iterations = 20, substeps = 1;
  double beta = 0.75;
  V3 g{0, 0, -9.81};
  int dich = 10, sm_period = 2;
  double contact_k = kInf, damping = 0.0;
  bool deterministic = false;
  int scale_mode = 0;
  void validate() const {  // scene.cpp:8-20
    require(dt > 0.0 && std::isfinite(dt), "settings.dt must be positive and finite");
    require(iterations >= 1, "settings.iterations must be at least 1");
    require(substeps >= 1, "settings.substeps must be at least 1");
    require(beta > 0.0 && beta <= 1.0, "settings.beta must be in (0, 1]");
    require(finite(g), "settings.gravity must be finite");
    require(dich >= 1, "settings.dichotomous_iterations must be at least 1");
    require(sm_period >= 1, "settings.shape_match_period must be at least 1");
    require(contact_k > 0.0, "settings.contact_stiffness must be positive");
    require(damping >= 0.0 && damping < 1.0, "settings.velocity_damping must be in [0, 1)");
  }
};

struct Scene {  // scene.h:109-126
  std::vector<Rod> rods;
  std::vector<Material> materials;
  std::vector<Plane> planes;
  std::vector<KinPill> kpills;
  std::vector<Bone> bones;
  std::vector<std::vector<std::pair<int, int>>> bundles;
  std::vector<PinMotion> pin_motions;
  std::vector<SoftPin> soft_pins;
  std::vector<Activation> activations;
  Settings settings;

  void validate() const {  // scene.cpp:63-157 (skin/probe checks are out of scope)
    settings.validate();
    require(!materials.empty(), "scene needs at least one material");
    for (const Material& m : materials) m.validate();
    const int rc = static_cast<int>(rods.size());
    for (int r = 0; r < rc; ++r) {
      const Rod& rod = rods[r];
      rod.rest.validate();
      const std::string where = "rod " + std::to_string(r);
      require_index(rod.material, static_cast<int>(materials.size()), where + " material");
      const int n = rod.rest.n();
      require(static_cast<int>(rod.pinned.size()) == n, where + " pinned flags size");
      require(static_cast<int>(rod.st.c.size()) == n, where + " state size");
      require(static_cast<int>(rod.st.q.size()) == rod.rest.m(), where + " frame count");
      if (!rod.bones.empty()) {
        require(static_cast<int>(rod.bone_w.size()) == n, where + " bone weights per vertex");
        for (int b : rod.bones) require_index(b, static_cast<int>(bones.size()), where + " bone index");
        for (int v = 0; v < n; ++v) {
          require(rod.bone_w[v].size() == rod.bones.size(), where + " bone weight row size");
          double sum = 0.0;
          for (double w : rod.bone_w[v]) sum += w;
          require(std::abs(sum - 1.0) < 1e-6, where + " bone weights must sum to 1");
        }
      }
    }
    for (const Plane& p : planes) require(std::abs(norm(p.n) - 1.0) < 1e-9, "plane normal must be unit length");
    for (const KinPill& kp : kpills) {
      require(kp.pill.rod < 0, "kinematic pill must not reference a rod");
      require(kp.pill.r0 > 0.0 && kp.pill.r1 > 0.0, "kinematic pill radii must be positive");
      require(finite(kp.pill.c0) && finite(kp.pill.c1), "kinematic pill centers must be finite");
      require(kp.bone < static_cast<int>(bones.size()), "kinematic pill bone out of range");
      if (kp.bone >= 0) require(!bones[kp.bone].keys.empty(), "kinematic pill bone has no keyframes");
    }
    std::set<std::pair<int, int>> seen;
    for (const auto& members : bundles) {
      require(members.size() >= 2, "bundle needs at least two members");
      for (const auto& [mr, mv] : members) {
        require_index(mr, rc, "bundle member rod");
        require_index(mv, rods[mr].rest.n(), "bundle member vertex");
        require(seen.insert({mr, mv}).second, "bundle groups must not share a vertex");
      }
    }
    for (const PinMotion& pm : pin_motions) {
      require_index(pm.rod, rc, "pin motion rod");
      require_index(pm.vertex, rods[pm.rod].rest.n(), "pin motion vertex");
      require(rods[pm.rod].pinned[pm.vertex] != 0, "pin motion requires a pinned vertex");
      require(pm.t1 >= pm.t0, "pin motion must have t1 >= t0");
    }
    for (const SoftPin& sp : soft_pins) {
      require_index(sp.rod, rc, "soft pin rod");
      require_index(sp.vertex, rods[sp.rod].rest.n(), "soft pin vertex");
      require(sp.k > 0.0, "soft pin stiffness must be positive");
    }
    for (const Activation& a : activations) {
      require_index(a.rod, rc, "activation rod");
      require(a.factor >= 0.0 && a.factor < 1.0, "activation factor must be in [0, 1)");
      require(a.t_end >= a.t_start, "activation must have t_end >= t_start");
      const int m = rods[a.rod].rest.m();
      require(a.first >= 0 && a.first < m, "activation first element");
      require(a.last == -1 || (a.last >= a.first && a.last < m), "activation last element");
    }
  }
};

// ---- rod model (rod.cpp) -------------------------------------------------------------------

// relative_rotation, rod.cpp:151-155.
Q relative_rotation(const Q& qa, const Q& qb) {
  Q p = qmul(qconj(qa), qb);
  if (p.w < 0) p = Q{-p.w, -p.x, -p.y, -p.z};
  return p;
}
// darboux_vector, rod.cpp:157-162.
V3 darboux_vector(const Q& qa, const Q& qb, double la, double lb) {
  require(is_unit(qa) && is_unit(qb), "darboux_vector: quaternions must be unit norm");
  require(la > 0 && lb > 0, "darboux_vector: lengths must be > 0");
  const Q p = relative_rotation(qa, qb);
  return mul(4.0 / (la + lb), qvec(p));
}
// refresh_length_derived, rod.cpp:42-56.
void refresh_length_derived(Rest& r) {
  const int m = r.m();
  r.sgrad.resize(m);
  for (int e = 0; e < m; ++e) r.sgrad[e] = (r.s[e + 1] - r.s[e]) / r.len[e];
  r.darb.resize(std::max(0, m - 1));
  r.slap.resize(std::max(0, m - 1));
  for (int j = 1; j < m; ++j) {
    r.darb[j - 1] = darboux_vector(r.q[j - 1], r.q[j], r.len[j - 1], r.len[j]);
    r.slap[j - 1] = (r.s[j + 1] - r.s[j]) / r.len[j] - (r.s[j] - r.s[j - 1]) / r.len[j - 1];
  }
}
// make_rest_pose, rod.cpp:60-112.
Rest make_rest_pose(const std::vector<V3>& centers, const std::vector<double>& radii,
                    const std::vector<double>& scales) {
  const int n = static_cast<int>(centers.size());
  require(n >= 2, "make_rest_pose: need at least 2 vertices");
  const int m = n - 1;
  Rest r;
  r.c = centers;
  if (radii.size() == 1) {
    r.r.assign(n, radii[0]);
  } else {
    require(static_cast<int>(radii.size()) == n, "make_rest_pose: radii must be uniform or per vertex");
    r.r = radii;
  }
  if (scales.empty()) {
    r.s.assign(n, 1.0);
  } else if (scales.size() == 1) {
    r.s.assign(n, scales[0]);
  } else {
    require(static_cast<int>(scales.size()) == n, "make_rest_pose: scales must be uniform or per vertex");
    r.s = scales;
  }
  r.len.resize(m);
  std::vector<V3> tangents(m);
  for (int e = 0; e < m; ++e) {
    const V3 d = sub(r.c[e + 1], r.c[e]);
    r.len[e] = norm(d);
    require(r.len[e] > 0, "make_rest_pose: coincident consecutive centers");
    tangents[e] = divs(d, r.len[e]);
  }
  r.len0 = r.len;
  r.q.resize(m);
  Q f0 = qfrom_two_vectors(V3{0, 0, 1}, tangents[0]);  // minimal_rotation, types.h:57-61
  qnormalize(f0);
  r.q[0] = f0;
  for (int e = 1; e < m; ++e) {
    Q dq = qfrom_two_vectors(tangents[e - 1], tangents[e]);
    qnormalize(dq);
    r.q[e] = qnormalized(qmul(dq, r.q[e - 1]));
    if (qdot(r.q[e], r.q[e - 1]) < 0) r.q[e] = Q{-r.q[e].w, -r.q[e].x, -r.q[e].y, -r.q[e].z};
  }
  r.tdot.resize(m);
  for (int e = 0; e < m; ++e) r.tdot[e] = dot(qmat(r.q[e]).col(2), tangents[e]);
  refresh_length_derived(r);
  r.validate();
  return r;
}
// apply_activation, rod.cpp:164-176.
void apply_activation(Rest& r, double a, double factor, int first, int last) {
  const int m = r.m();
  if (last < 0) last = m - 1;
  require_index(first >= 0 && last < m && first <= last, "apply_activation: element range out of bounds");
  const double scale = 1.0 - a * factor;
  require(scale > 0, "apply_activation: activation would collapse rest lengths");
  for (int e = first; e <= last; ++e) r.len[e] = r.len0[e] * scale;
  refresh_length_derived(r);
}
// current_volume / rest_volume, rod.cpp:178-197.
double current_volume(const State& st, const Rest& r) {
  double v = 0.0;
  for (int e = 0; e < r.m(); ++e) {
    const double s = 0.5 * (st.s[e] + st.s[e + 1]);
    const double rr = 0.5 * (r.r[e] + r.r[e + 1]);
    const double len = norm(sub(st.c[e + 1], st.c[e]));
    v += kPi * (s * rr) * (s * rr) * len;
  }
  return v;
}
double rest_volume(const Rest& r) {
  double v = 0.0;
  for (int e = 0; e < r.m(); ++e) {
    const double s = 0.5 * (r.s[e] + r.s[e + 1]);
    const double rr = 0.5 * (r.r[e] + r.r[e + 1]);
    v += kPi * (s * rr) * (s * rr) * r.len0[e];
  }
  return v;
}

// ---- layout (layout.cpp) -------------------------------------------------------------------

struct Layout {  // DofLayout, layout.h:17-41
  std::vector<int> vbase, ebase;
  int V = 0, E = 0, dof = 0;
  std::vector<double> cw, sw, ic, is;
  std::vector<V3> tw, it;
  std::vector<uint8_t> pinned;
  std::vector<int> vrod, vloc, erod, eloc;
  int vslot(int r, int v) const { return vbase[r] + v; }
  int eslot(int r, int e) const { return ebase[r] + e; }
};

// refresh_orientation_inertia, layout.cpp:76-93.
void refresh_orientation_inertia(Layout& L, const std::vector<Rod>& rods, const std::vector<Material>& mats) {
  for (int r = 0; r < static_cast<int>(rods.size()); ++r) {
    const Rod& rod = rods[r];
    const double rho = mats[rod.material].rho;
    for (int e = 0; e < rod.rest.m(); ++e) {
      const double rbar = 0.5 * (rod.rest.r[e] + rod.rest.r[e + 1]);
      const double smid = 0.5 * (rod.st.s[e] + rod.st.s[e + 1]);
      const double r4 = kPi * rbar * rbar * rbar * rbar;
      const double base = rho * smid * smid * r4 * rod.rest.len0[e];
      const V3 w{0.25 * base, 0.25 * base, 0.5 * base};
      const int slot = L.eslot(r, e);
      L.tw[slot] = w;
      L.it[slot] = V3{1.0 / w.x, 1.0 / w.y, 1.0 / w.z};
    }
  }
}
// build_layout, layout.cpp:7-73.
Layout build_layout(const std::vector<Rod>& rods, const std::vector<Material>& mats) {
  Layout L;
  const int nr = static_cast<int>(rods.size());
  L.vbase.resize(nr);
  L.ebase.resize(nr);
  for (int r = 0; r < nr; ++r) {
    L.vbase[r] = L.V;
    L.ebase[r] = L.E;
    L.V += rods[r].rest.n();
    L.E += rods[r].rest.m();
  }
  L.dof = 4 * L.V + 3 * L.E;
  L.cw.assign(L.V, 0.0);
  L.sw.assign(L.V, 0.0);
  L.ic.assign(L.V, 0.0);
  L.is.assign(L.V, 0.0);
  L.pinned.assign(L.V, 0);
  L.tw.assign(L.E, V3{});
  L.it.assign(L.E, V3{});
  L.vrod.resize(L.V);
  L.vloc.resize(L.V);
  L.erod.resize(L.E);
  L.eloc.resize(L.E);
  for (int r = 0; r < nr; ++r) {
    for (int v = 0; v < rods[r].rest.n(); ++v) {
      L.vrod[L.vslot(r, v)] = r;
      L.vloc[L.vslot(r, v)] = v;
    }
    for (int e = 0; e < rods[r].rest.m(); ++e) {
      L.erod[L.eslot(r, e)] = r;
      L.eloc[L.eslot(r, e)] = e;
    }
  }
  for (int r = 0; r < nr; ++r) {
    const Rod& rod = rods[r];
    const double rho = mats[rod.material].rho;
    const int n = rod.rest.n();
    for (int v = 0; v < n; ++v) {
      double lump = 0.0;
      if (v > 0) lump += 0.5 * rod.rest.len0[v - 1];
      if (v < n - 1) lump += 0.5 * rod.rest.len0[v];
      const double rbar = rod.rest.r[v];
      const int slot = L.vslot(r, v);
      const bool pin = !rod.pinned.empty() && rod.pinned[v] != 0;
      L.pinned[slot] = pin ? 1 : 0;
      if (pin) {
        L.cw[slot] = kInf;
        L.sw[slot] = kInf;
        L.ic[slot] = 0.0;
        L.is[slot] = 0.0;
      } else {
        const double cw = kPi * rbar * rbar * rho * lump;
        const double sw = 0.5 * kPi * rbar * rbar * rbar * rbar * rho * lump;
        L.cw[slot] = cw;
        L.sw[slot] = sw;
        L.ic[slot] = 1.0 / cw;
        L.is[slot] = 1.0 / sw;
      }
    }
  }
  refresh_orientation_inertia(L, rods, mats);
  return L;
}

// ---- constraints (constraints.cpp) ---------------------------------------------------------

enum Kind : int {
  kStretchZ = 0, kCrossSection, kSurfaceStretch, kBendTwist, kSurfaceBending, kVolumeStretch,
  kVolumeBendU, kVolumeBendV, kContact, kHalfPlane, kPin
};
const char* kind_name(int k) {  // constraints.cpp:11-26
  static const char* names[] = {"stretch_z", "cross_section", "surface_stretch", "bend_twist",
                                "surface_bending", "volume_stretch", "volume_bend_u", "volume_bend_v",
                                "contact", "half_plane", "pin"};
  return (k >= 0 && k < 11) ? names[k] : "unknown";
}
int residual_dim(int k) {  // constraints.cpp:28-38
  return (k == kStretchZ || k == kBendTwist || k == kVolumeStretch || k == kPin) ? 3 : 1;
}

struct Block {  // ConstraintBlock, constraints.h:37-48
  int kind = kStretchZ;
  bool unilateral = false;
  int rod = -1, loc = -1, aux = -1, pill_a = -1;
  double alpha = 0, beta = 0;
  V3 k{0, 0, 0};
  V3 lambda{0, 0, 0};
};

struct Eval {  // ResidualEval, constraints.h:55-67
  int dim = 1;
  V3 W{0, 0, 0};
  int nc = 0, ns = 0, nt = 0;
  int cslot[4], sslot[4], tslot[2];
  M3 cj[4];
  V3 sj[4];
  M3 tj[2];
};

struct Ctx {  // EvalContext, constraints.h:73-80
  const std::vector<Rod>* rods;
  const Layout* L;
  const std::vector<Pill>* pills;
  const std::vector<Plane>* planes;
  const std::vector<V3>* pin_targets;
  bool classic = false;
};

M3 diag(double d) {
  M3 o;
  o(0, 0) = o(1, 1) = o(2, 2) = d;
  return o;
}
// axis_column_derivative (constraints.cpp:43-45): -R * [e_z]x == [-R.col1, R.col0, 0].
M3 axis_column_derivative(const M3& R) {
  M3 o;
  for (int i = 0; i < 3; ++i) {
    o(i, 0) = -R(i, 1);
    o(i, 1) = R(i, 0);
    o(i, 2) = 0.0;
  }
  return o;
}
// dimag_dqa / dimag_dqb (constraints.cpp:50-51): 0.5 * (-+p.w I + [p_v]x).
M3 dimag(const Q& p, double wsign) {
  const double w = wsign * p.w;
  M3 o;
  o(0, 0) = 0.5 * w;
  o(0, 1) = 0.5 * -p.z;
  o(0, 2) = 0.5 * p.y;
  o(1, 0) = 0.5 * p.z;
  o(1, 1) = 0.5 * w;
  o(1, 2) = 0.5 * -p.x;
  o(2, 0) = 0.5 * -p.y;
  o(2, 1) = 0.5 * p.x;
  o(2, 2) = 0.5 * w;
  return o;
}
M3 row0(const V3& v) {
  M3 o;
  o(0, 0) = v.x;
  o(0, 1) = v.y;
  o(0, 2) = v.z;
  return o;
}
void push_c(Eval& ev, int slot, const M3& j) {
  ev.cslot[ev.nc] = slot;
  ev.cj[ev.nc++] = j;
}
void push_s(Eval& ev, int slot, const V3& j) {
  ev.sslot[ev.ns] = slot;
  ev.sj[ev.ns++] = j;
}
void push_t(Eval& ev, int slot, const M3& j) {
  ev.tslot[ev.nt] = slot;
  ev.tj[ev.nt++] = j;
}

struct PillGeom {  // constraints.cpp:69-97
  V3 c0, c1;
  double r0 = 0, r1 = 0, rb0 = 0, rb1 = 0;
  int v0 = -1, v1 = -1;
};
PillGeom resolve_pill(int idx, const Ctx& ctx) {
  const Pill& p = (*ctx.pills)[idx];
  PillGeom g;
  if (p.rod >= 0) {
    const Rod& rod = (*ctx.rods)[p.rod];
    g.c0 = rod.st.c[p.element];
    g.c1 = rod.st.c[p.element + 1];
    g.rb0 = rod.rest.r[p.element];
    g.rb1 = rod.rest.r[p.element + 1];
    g.r0 = rod.st.s[p.element] * g.rb0;
    g.r1 = rod.st.s[p.element + 1] * g.rb1;
    g.v0 = ctx.L->vslot(p.rod, p.element);
    g.v1 = ctx.L->vslot(p.rod, p.element + 1);
  } else {
    g.c0 = p.c0;
    g.c1 = p.c1;
    g.r0 = p.r0;
    g.r1 = p.r1;
  }
  return g;
}

// eval_constraint, constraints.cpp:101-270.
Eval eval_constraint(const Block& b, const Ctx& ctx) {
  Eval ev;
  ev.dim = residual_dim(b.kind);
  switch (b.kind) {
    case kStretchZ: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int e = b.loc;
      const double l = rod.rest.len[e];
      const M3 R = qmat(rod.st.q[e]);
      const V3 w = R.col(2);
      const double tbar = rod.rest.tdot[e];
      const V3 dzc = divs(sub(rod.st.c[e + 1], rod.st.c[e]), l);
      ev.W = sub(dzc, mul(tbar, w));
      push_c(ev, ctx.L->vslot(b.rod, e), diag(-1.0 / l));
      push_c(ev, ctx.L->vslot(b.rod, e + 1), diag(1.0 / l));
      push_t(ev, ctx.L->eslot(b.rod, e), mscale(-tbar, axis_column_derivative(R)));
      break;
    }
    case kCrossSection: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int e = b.loc;
      const double smid = 0.5 * (rod.st.s[e] + rod.st.s[e + 1]);
      const double smid_rest = 0.5 * (rod.rest.s[e] + rod.rest.s[e + 1]);
      ev.W.x = smid - smid_rest;
      push_s(ev, ctx.L->vslot(b.rod, e), V3{0.5, 0, 0});
      push_s(ev, ctx.L->vslot(b.rod, e + 1), V3{0.5, 0, 0});
      break;
    }
    case kSurfaceStretch: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int e = b.loc;
      const double l = rod.rest.len[e];
      ev.W.x = (rod.st.s[e + 1] - rod.st.s[e]) / l - rod.rest.sgrad[e];
      push_s(ev, ctx.L->vslot(b.rod, e), V3{-1.0 / l, 0, 0});
      push_s(ev, ctx.L->vslot(b.rod, e + 1), V3{1.0 / l, 0, 0});
      break;
    }
    case kBendTwist: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int j = b.loc;
      const double la = rod.rest.len[j - 1], lb = rod.rest.len[j];
      const Q p = relative_rotation(rod.st.q[j - 1], rod.st.q[j]);
      const double inv_len = 4.0 / (la + lb);
      const V3 omega = mul(inv_len, qvec(p));
      const double s = ctx.classic ? rod.rest.s[j] : rod.st.s[j];
      ev.W = sub(mul(s, omega), mul(rod.rest.s[j], rod.rest.darb[j - 1]));
      if (!ctx.classic) push_s(ev, ctx.L->vslot(b.rod, j), omega);
      push_t(ev, ctx.L->eslot(b.rod, j - 1), mscale(s * inv_len, dimag(p, -1.0)));
      push_t(ev, ctx.L->eslot(b.rod, j), mscale(s * inv_len, dimag(p, 1.0)));
      break;
    }
    case kSurfaceBending: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int j = b.loc;
      const double la = rod.rest.len[j - 1], lb = rod.rest.len[j];
      const double lap = (rod.st.s[j + 1] - rod.st.s[j]) / lb - (rod.st.s[j] - rod.st.s[j - 1]) / la;
      ev.W.x = lap - rod.rest.slap[j - 1];
      push_s(ev, ctx.L->vslot(b.rod, j - 1), V3{1.0 / la, 0, 0});
      push_s(ev, ctx.L->vslot(b.rod, j), V3{-1.0 / la - 1.0 / lb, 0, 0});
      push_s(ev, ctx.L->vslot(b.rod, j + 1), V3{1.0 / lb, 0, 0});
      break;
    }
    case kVolumeStretch: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int e = b.loc;
      const double l0 = rod.rest.len0[e];
      const M3 R = qmat(rod.st.q[e]);
      const V3 w = R.col(2);
      const double tbar = rod.rest.tdot[e];
      const double smid = 0.5 * (rod.st.s[e] + rod.st.s[e + 1]);
      const double smid_rest = 0.5 * (rod.rest.s[e] + rod.rest.s[e + 1]);
      const V3 dzc = divs(sub(rod.st.c[e + 1], rod.st.c[e]), l0);
      ev.W = sub(mul(smid * smid, dzc), mul(smid_rest * smid_rest * tbar, w));
      push_c(ev, ctx.L->vslot(b.rod, e), diag(-smid * smid / l0));
      push_c(ev, ctx.L->vslot(b.rod, e + 1), diag(smid * smid / l0));
      push_s(ev, ctx.L->vslot(b.rod, e), mul(smid, dzc));
      push_s(ev, ctx.L->vslot(b.rod, e + 1), mul(smid, dzc));
      push_t(ev, ctx.L->eslot(b.rod, e), mscale(-smid_rest * smid_rest * tbar, axis_column_derivative(R)));
      break;
    }
    case kVolumeBendU:
    case kVolumeBendV: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int j = b.loc;
      const int comp = b.kind == kVolumeBendU ? 0 : 1;
      const double la0 = rod.rest.len0[j - 1], lb0 = rod.rest.len0[j];
      const Q p = relative_rotation(rod.st.q[j - 1], rod.st.q[j]);
      const double inv_len0 = 4.0 / (la0 + lb0);
      const double omega_c = inv_len0 * qvec(p)[comp];
      const double rest_omega_c = rod.rest.darb[j - 1][comp] * (rod.rest.len[j - 1] + rod.rest.len[j]) / (la0 + lb0);
      const double s = rod.st.s[j];
      const double sbar = rod.rest.s[j];
      ev.W.x = s * s * s * omega_c - sbar * sbar * sbar * rest_omega_c;
      push_s(ev, ctx.L->vslot(b.rod, j), V3{3.0 * s * s * omega_c, 0, 0});
      const M3 da = mscale(s * s * s * inv_len0, dimag(p, -1.0));
      const M3 db = mscale(s * s * s * inv_len0, dimag(p, 1.0));
      push_t(ev, ctx.L->eslot(b.rod, j - 1), row0(da.row(comp)));
      push_t(ev, ctx.L->eslot(b.rod, j), row0(db.row(comp)));
      break;
    }
    case kContact: {
      const PillGeom a = resolve_pill(b.pill_a, ctx);
      const PillGeom c = resolve_pill(b.aux, ctx);
      const double al = b.alpha, be = b.beta;
      const V3 ca = add(mul(1.0 - al, a.c0), mul(al, a.c1));
      const V3 cb = add(mul(1.0 - be, c.c0), mul(be, c.c1));
      const double ra = (1.0 - al) * a.r0 + al * a.r1;
      const double rb = (1.0 - be) * c.r0 + be * c.r1;
      V3 nrm = sub(ca, cb);
      const double dist = norm(nrm);
      if (dist < 1e-12) {
        ev.dim = 1;
        ev.W.x = 0.0;
        break;
      }
      nrm = divs(nrm, dist);
      ev.W.x = dist - ra - rb;
      if (a.v0 >= 0) {
        push_c(ev, a.v0, row0(mul(1.0 - al, nrm)));
        push_c(ev, a.v1, row0(mul(al, nrm)));
        push_s(ev, a.v0, V3{-(1.0 - al) * a.rb0, 0, 0});
        push_s(ev, a.v1, V3{-al * a.rb1, 0, 0});
      }
      if (c.v0 >= 0) {
        push_c(ev, c.v0, row0(mul(-(1.0 - be), nrm)));
        push_c(ev, c.v1, row0(mul(-be, nrm)));
        push_s(ev, c.v0, V3{-(1.0 - be) * c.rb0, 0, 0});
        push_s(ev, c.v1, V3{-be * c.rb1, 0, 0});
      }
      break;
    }
    case kHalfPlane: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const Plane& pl = (*ctx.planes)[b.aux];
      const int v = b.loc;
      const double rbar = rod.rest.r[v];
      ev.W.x = dot(pl.n, rod.st.c[v]) - pl.off - rod.st.s[v] * rbar;
      push_c(ev, ctx.L->vslot(b.rod, v), row0(pl.n));
      push_s(ev, ctx.L->vslot(b.rod, v), V3{-rbar, 0, 0});
      break;
    }
    case kPin: {
      const Rod& rod = (*ctx.rods)[b.rod];
      const int v = b.loc;
      ev.W = sub(rod.st.c[v], (*ctx.pin_targets)[b.aux]);
      push_c(ev, ctx.L->vslot(b.rod, v), diag(1.0));
      break;
    }
  }
  return ev;
}

// inverse_stiffness, constraints.cpp:274-278.
double inverse_stiffness(double k) {
  if (std::isinf(k)) return 0.0;
  if (k <= 0.0) return 1e30;
  return std::min(1.0 / k, 1e30);
}

// assemble_rod_constraints, constraints.cpp:282-329.
std::vector<Block> assemble_rod_constraints(const Rod& rod, const Material& mat, int ri, bool scale_kinds) {
  mat.validate();
  rod.rest.validate();
  std::vector<Block> blocks;
  const Rest& r = rod.rest;
  const int m = r.m();
  const double kxy = mat.sx + mat.sy;
  const double bxy = mat.bx + mat.by;
  auto emit = [&](int kind, int loc, const V3& k) {
    if (maxc(k) <= 0.0) return;
    Block b;
    b.kind = kind;
    b.rod = ri;
    b.loc = loc;
    b.k = k;
    blocks.push_back(b);
  };
  for (int e = 0; e < m; ++e) {
    const double rmid = 0.5 * (r.r[e] + r.r[e + 1]);
    const double a2 = kPi * rmid * rmid;
    const double a4 = 0.25 * kPi * rmid * rmid * rmid * rmid;
    const double l = r.len[e], l0 = r.len0[e];
    const double kz = a2 * mat.sz * l;
    emit(kStretchZ, e, V3{kz, kz, kz});
    if (scale_kinds) {
      emit(kCrossSection, e, V3{a2 * kxy * l, 0, 0});
      emit(kSurfaceStretch, e, V3{a4 * kxy * l, 0, 0});
      const double kv = a2 * mat.vol * l0;
      emit(kVolumeStretch, e, V3{kv, kv, kv});
    }
  }
  for (int j = 1; j < m; ++j) {
    const double rv = r.r[j];
    const double a4 = 0.25 * kPi * rv * rv * rv * rv;
    const double lw = 0.5 * (r.len[j - 1] + r.len[j]);
    const double lw0 = 0.5 * (r.len0[j - 1] + r.len0[j]);
    emit(kBendTwist, j, V3{a4 * mat.sz * lw, a4 * mat.sz * lw, a4 * kxy * lw});
    if (scale_kinds) {
      emit(kSurfaceBending, j, V3{a4 * bxy * lw, 0, 0});
      emit(kVolumeBendU, j, V3{2.0 * a4 * mat.vol * lw0, 0, 0});
      emit(kVolumeBendV, j, V3{2.0 * a4 * mat.vol * lw0, 0, 0});
    }
  }
  return blocks;
}

// refresh_stiffness, constraints.cpp:331-372 (note std::pow, unlike assembly).
void refresh_stiffness(Block* blocks, int count, const std::vector<Rod>& rods, const std::vector<Material>& mats) {
  for (int i = 0; i < count; ++i) {
    Block& b = blocks[i];
    if (b.rod < 0) continue;
    const Rod& rod = rods[b.rod];
    const Rest& r = rod.rest;
    const Material& mat = mats[rod.material];
    const double kxy = mat.sx + mat.sy;
    switch (b.kind) {
      case kStretchZ: {
        const double rmid = 0.5 * (r.r[b.loc] + r.r[b.loc + 1]);
        const double k = kPi * rmid * rmid * mat.sz * r.len[b.loc];
        b.k = V3{k, k, k};
        break;
      }
      case kCrossSection: {
        const double rmid = 0.5 * (r.r[b.loc] + r.r[b.loc + 1]);
        b.k = V3{kPi * rmid * rmid * kxy * r.len[b.loc], 0, 0};
        break;
      }
      case kSurfaceStretch: {
        const double rmid = 0.5 * (r.r[b.loc] + r.r[b.loc + 1]);
        const double a4 = 0.25 * kPi * std::pow(rmid, 4);
        b.k = V3{a4 * kxy * r.len[b.loc], 0, 0};
        break;
      }
      case kBendTwist: {
        const double a4 = 0.25 * kPi * std::pow(r.r[b.loc], 4);
        const double lw = 0.5 * (r.len[b.loc - 1] + r.len[b.loc]);
        b.k = V3{a4 * mat.sz * lw, a4 * mat.sz * lw, a4 * kxy * lw};
        break;
      }
      case kSurfaceBending: {
        const double a4 = 0.25 * kPi * std::pow(r.r[b.loc], 4);
        const double lw = 0.5 * (r.len[b.loc - 1] + r.len[b.loc]);
        b.k = V3{a4 * (mat.bx + mat.by) * lw, 0, 0};
        break;
      }
      default:
        break;
    }
  }
}

struct Update {  // BlockUpdate, constraints.cpp:385-397
  bool active = false, singular = false, finite = true;
  int nc = 0, ns = 0, nt = 0;
  int cs[4], ss[4], ts[2];
  V3 dc[4];
  double ds[4];
  V3 dt[2];
  V3 dl{0, 0, 0};
};

// solve_block, constraints.cpp:400-487.
Update solve_block(const Block& b, const Ctx& ctx, double h, double beta) {
  Update up;
  const Eval ev = eval_constraint(b, ctx);
  const int dim = ev.dim;
  if (b.unilateral && ev.W.x >= 0.0 && b.lambda.x == 0.0) return up;
  const Layout& L = *ctx.L;
  const double h2 = h * h;
  M3 M;
  for (int i = 0; i < ev.nc; ++i) {
    const double invw = L.ic[ev.cslot[i]];
    if (invw == 0.0) continue;
    const double s = h2 * invw;
    const M3& J = ev.cj[i];
    for (int p = 0; p < dim; ++p)
      for (int q = 0; q < dim; ++q) {
        const double a0 = s * J(p, 0), a1 = s * J(p, 1), a2 = s * J(p, 2);
        M(p, q) = M(p, q) + ((a0 * J(q, 0) + a1 * J(q, 1)) + a2 * J(q, 2));
      }
  }
  for (int i = 0; i < ev.ns; ++i) {
    const double invw = L.is[ev.sslot[i]];
    if (invw == 0.0) continue;
    const double s = h2 * invw;
    const V3& j = ev.sj[i];
    for (int p = 0; p < dim; ++p)
      for (int q = 0; q < dim; ++q) M(p, q) = M(p, q) + (s * j[p]) * j[q];
  }
  for (int i = 0; i < ev.nt; ++i) {
    const V3& invw = L.it[ev.tslot[i]];
    const M3& J = ev.tj[i];
    for (int p = 0; p < dim; ++p) {
      // ((h2 * J) * diag(invw)) row p
      const double b0 = (h2 * J(p, 0)) * invw.x, b1 = (h2 * J(p, 1)) * invw.y, b2 = (h2 * J(p, 2)) * invw.z;
      for (int q = 0; q < dim; ++q) M(p, q) = M(p, q) + ((b0 * J(q, 0) + b1 * J(q, 1)) + b2 * J(q, 2));
    }
  }
  V3 kinv{0, 0, 0};
  for (int d = 0; d < dim; ++d) {
    kinv[d] = inverse_stiffness(b.k[d]);
    M(d, d) = M(d, d) + kinv[d];
  }
  V3 rhs{0, 0, 0};
  for (int d = 0; d < dim; ++d) rhs[d] = ev.W[d] - kinv[d] * b.lambda[d];
  V3 dl{0, 0, 0};
  if (dim == 1) {
    if (M(0, 0) <= 1e-250) {
      up.singular = true;
      return up;
    }
    dl.x = beta * rhs.x / M(0, 0);
  } else {
    double md = std::abs(M(0, 0));  // cwiseAbs().maxCoeff(), column-major scan
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) md = std::max(md, std::abs(M(i, j)));
    md = std::max(md, 1e-300);
    auto h3 = [&](int a, int bb, int c) { return M(0, a) * (M(1, bb) * M(2, c) - M(1, c) * M(2, bb)); };
    const double det = h3(0, 1, 2) - h3(1, 0, 2) + h3(2, 0, 1);
    if (std::abs(det) <= 1e-14 * md * md * md) {
      up.singular = true;
      return up;
    }
    auto cof = [&](int i, int j) {
      const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      return M(i1, j1) * M(i2, j2) - M(i1, j2) * M(i2, j1);
    };
    const double c0 = cof(0, 0), c1 = cof(1, 0), c2 = cof(2, 0);
    const double d = (c0 * M(0, 0) + c1 * M(1, 0)) + c2 * M(2, 0);
    const double invdet = 1.0 / d;
    M3 inv;
    inv(0, 0) = c0 * invdet;
    inv(0, 1) = c1 * invdet;
    inv(0, 2) = c2 * invdet;
    inv(1, 0) = cof(0, 1) * invdet;
    inv(1, 1) = cof(1, 1) * invdet;
    inv(1, 2) = cof(2, 1) * invdet;
    inv(2, 0) = cof(0, 2) * invdet;
    inv(2, 1) = cof(1, 2) * invdet;
    inv(2, 2) = cof(2, 2) * invdet;
    dl = mvmul(mscale(beta, inv), rhs);
  }
  if (b.unilateral && b.lambda.x + dl.x > 0.0) dl.x = -b.lambda.x;
  up.active = true;
  up.dl = dl;
  up.finite = finite(dl);
  up.nc = ev.nc;
  up.ns = ev.ns;
  up.nt = ev.nt;
  for (int i = 0; i < ev.nc; ++i) {
    const int slot = ev.cslot[i];
    up.cs[i] = slot;
    const M3& J = ev.cj[i];
    V3 v;
    for (int k = 0; k < 3; ++k) {
      double acc = J(0, k) * dl[0];
      for (int d = 1; d < dim; ++d) acc = acc + J(d, k) * dl[d];
      v[k] = acc;
    }
    up.dc[i] = mul(-h2 * L.ic[slot], v);
    if (!finite(up.dc[i])) up.finite = false;
  }
  for (int i = 0; i < ev.ns; ++i) {
    const int slot = ev.sslot[i];
    up.ss[i] = slot;
    const V3& j = ev.sj[i];
    const double dd = dim == 1 ? j[0] * dl[0] : (j[0] * dl[0] + j[1] * dl[1]) + j[2] * dl[2];
    up.ds[i] = -h2 * L.is[slot] * dd;
    if (!std::isfinite(up.ds[i])) up.finite = false;
  }
  for (int i = 0; i < ev.nt; ++i) {
    const int slot = ev.tslot[i];
    up.ts[i] = slot;
    const M3& J = ev.tj[i];
    V3 jt;
    for (int k = 0; k < 3; ++k) {
      double acc = J(0, k) * dl[0];
      for (int d = 1; d < dim; ++d) acc = acc + J(d, k) * dl[d];
      jt[k] = acc;
    }
    up.dt[i] = mul(-h2, cwmul(L.it[slot], jt));
    if (!finite(up.dt[i])) up.finite = false;
  }
  return up;
}

struct Scratch {  // SweepScratch, constraints.h:102-110
  std::vector<V3> csum, tsum;
  std::vector<double> ssum;
  std::vector<int> ccount, scount, tcount;
  void resize(const Layout& L) {
    csum.assign(L.V, V3{});
    ssum.assign(L.V, 0.0);
    tsum.assign(L.E, V3{});
    ccount.assign(L.V, 0);
    scount.assign(L.V, 0);
    tcount.assign(L.E, 0);
  }
};

struct SweepOutcome {
  int active = 0, skipped_singular = 0;
};

// thread_count / parallel_for, parallel.h:12-46: VROD_THREADS workers (clamped to the hardware),
// contiguous chunks, index-addressed results — so the outcome is independent of scheduling. (The
// reference's own multi-threaded run crashes on its thread_local update buffer, DESIGN.md §2;
// this restatement keeps one shared buffer.)
int thread_count() {  // read per sweep (like parallel.h), so one process can compare thread counts
  const char* env = std::getenv("VROD_THREADS");
  if (!env) return 1;
  static const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  return std::clamp(std::atoi(env), 1, hw);
}
template <typename Fn>
void parallel_for(int n, int threads, Fn&& fn) {
  if (n <= 0) return;
  if (threads <= 1 || n == 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  threads = std::min(threads, n);
  std::vector<std::thread> pool;
  const int chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back([b, e, &fn] {
      for (int i = b; i < e; ++i) fn(i);
    });
  }
  for (std::thread& th : pool) th.join();
}

// jacobi_sweep, constraints.cpp:491-556 (block solves on VROD_THREADS workers, :497-500).
SweepOutcome jacobi_sweep(std::vector<Block>& blocks, std::vector<Rod>& rods, const Ctx& ctx, double h,
                          double beta, Scratch& sc) {
  const Layout& L = *ctx.L;
  const int n = static_cast<int>(blocks.size());
  SweepOutcome out;
  std::vector<Update> ups(static_cast<std::size_t>(n));
  parallel_for(n, thread_count(), [&](int i) { ups[i] = solve_block(blocks[i], ctx, h, beta); });
  std::fill(sc.csum.begin(), sc.csum.end(), V3{});
  std::fill(sc.ssum.begin(), sc.ssum.end(), 0.0);
  std::fill(sc.tsum.begin(), sc.tsum.end(), V3{});
  std::fill(sc.ccount.begin(), sc.ccount.end(), 0);
  std::fill(sc.scount.begin(), sc.scount.end(), 0);
  std::fill(sc.tcount.begin(), sc.tcount.end(), 0);
  for (int i = 0; i < n; ++i) {
    Update& up = ups[i];
    if (up.singular) {
      ++out.skipped_singular;
      continue;
    }
    if (!up.active) continue;
    if (!up.finite)
      throw SimulationError(std::string("non-finite update from constraint ") + kind_name(blocks[i].kind) + " #" +
                            std::to_string(i));
    ++out.active;
    blocks[i].lambda = add(blocks[i].lambda, up.dl);
    for (int k = 0; k < up.nc; ++k) {
      sc.csum[up.cs[k]] = add(sc.csum[up.cs[k]], up.dc[k]);
      ++sc.ccount[up.cs[k]];
    }
    for (int k = 0; k < up.ns; ++k) {
      sc.ssum[up.ss[k]] += up.ds[k];
      ++sc.scount[up.ss[k]];
    }
    for (int k = 0; k < up.nt; ++k) {
      sc.tsum[up.ts[k]] = add(sc.tsum[up.ts[k]], up.dt[k]);
      ++sc.tcount[up.ts[k]];
    }
  }
  for (int slot = 0; slot < L.V; ++slot) {
    Rod& rod = rods[L.vrod[slot]];
    const int v = L.vloc[slot];
    if (sc.ccount[slot] > 0) rod.st.c[v] = add(rod.st.c[v], divs(sc.csum[slot], sc.ccount[slot]));
    if (sc.scount[slot] > 0) {
      const double s = rod.st.s[v] + sc.ssum[slot] / sc.scount[slot];
      rod.st.s[v] = std::max(s, kMinScale);
    }
  }
  for (int slot = 0; slot < L.E; ++slot) {
    if (sc.tcount[slot] == 0) continue;
    Rod& rod = rods[L.erod[slot]];
    const int e = L.eloc[slot];
    rod.st.q[e] = apply_increment(rod.st.q[e], divs(sc.tsum[slot], sc.tcount[slot]));
  }
  return out;
}

// elastic_residual_norms, constraints.cpp:558-596.
std::vector<double> elastic_residual_norms(const Block* blocks, int count, const Ctx& ctx) {
  std::vector<double> num(8, 0.0), den(8, 0.0);
  for (int i = 0; i < count; ++i) {
    const Block& b = blocks[i];
    if (b.kind >= 8) continue;
    const Rest& r = (*ctx.rods)[b.rod].rest;
    double lw = 0.0;
    switch (b.kind) {
      case kStretchZ:
      case kCrossSection:
      case kSurfaceStretch: lw = r.len[b.loc]; break;
      case kVolumeStretch: lw = r.len0[b.loc]; break;
      case kBendTwist:
      case kSurfaceBending: lw = 0.5 * (r.len[b.loc - 1] + r.len[b.loc]); break;
      case kVolumeBendU:
      case kVolumeBendV: lw = 0.5 * (r.len0[b.loc - 1] + r.len0[b.loc]); break;
      default: break;
    }
    const Eval ev = eval_constraint(b, ctx);
    const double sq = ev.dim == 1 ? ev.W.x * ev.W.x : sqnorm(ev.W);
    num[b.kind] += lw * sq;
    den[b.kind] += lw;
  }
  std::vector<double> out(8, 0.0);
  for (int k = 0; k < 8; ++k)
    if (den[k] > 0) out[k] = std::sqrt(num[k] / den[k]);
  return out;
}

// ---- collision (collision.cpp) -------------------------------------------------------------

struct Projection {
  double t = 0, d = 0;
  bool degenerate = false;
};
// pill_distance_at, collision.cpp:9-13.
double pill_distance_at(const V3& x, const Pill& p, double t) {
  const V3 c = add(mul(1.0 - t, p.c0), mul(t, p.c1));
  const double r = (1.0 - t) * p.r0 + t * p.r1;
  return norm(sub(x, c)) - r;
}
// pill_project, collision.cpp:15-49.
Projection pill_project(const V3& x, const Pill& p) {
  Projection out;
  const V3 axis = sub(p.c1, p.c0);
  const double l = norm(axis);
  if (l <= std::abs(p.r0 - p.r1) || l < 1e-14) {
    const double d0 = norm(sub(x, p.c0)) - p.r0;
    const double d1 = norm(sub(x, p.c1)) - p.r1;
    out.degenerate = true;
    if (d0 <= d1) {
      out.t = 0.0;
      out.d = d0;
    } else {
      out.t = 1.0;
      out.d = d1;
    }
    return out;
  }
  const V3 j = divs(axis, l);
  const V3 y = sub(x, p.c0);
  const double a = dot(y, j);
  const double b = norm(sub(y, mul(a, j)));
  const double sin_t = (p.r1 - p.r0) / l;
  const double tan_t = sin_t / std::sqrt(std::max(1e-16, 1.0 - sin_t * sin_t));
  double t = (a + b * tan_t) / l;
  t = std::clamp(t, 0.0, 1.0);
  out.t = t;
  out.d = pill_distance_at(x, p, t);
  return out;
}
// pair_distance, collision.cpp:55-61.
double pair_distance(const Pill& a, const Pill& b, double alpha, double& beta) {
  const V3 ca = add(mul(1.0 - alpha, a.c0), mul(alpha, a.c1));
  const double ra = (1.0 - alpha) * a.r0 + alpha * a.r1;
  const Projection pr = pill_project(ca, b);
  beta = pr.t;
  return pr.d - ra;
}
// pill_less, collision.cpp:65-74.
bool pill_less(const Pill& a, const Pill& b) {
  for (int i = 0; i < 3; ++i)
    if (a.c0[i] != b.c0[i]) return a.c0[i] < b.c0[i];
  for (int i = 0; i < 3; ++i)
    if (a.c1[i] != b.c1[i]) return a.c1[i] < b.c1[i];
  if (a.r0 != b.r0) return a.r0 < b.r0;
  return a.r1 < b.r1;
}
struct Overlap {
  double alpha = 0, beta = 0, d = 0;
};
// deepest_penetration, collision.cpp:78-135.
Overlap deepest_penetration(const Pill& a, const Pill& b, int iterations, double warm) {
  const bool swapped = pill_less(b, a);
  const Pill& pa = swapped ? b : a;
  const Pill& pb = swapped ? a : b;
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
  for (double cand : cands) {
    if (cand < 0.0 || cand > 1.0) continue;
    double bc = 0.0;
    const double fc = pair_distance(pa, pb, cand, bc);
    if (fc < best) {
      best = fc;
      best_a = cand;
      best_b = bc;
    }
  }
  Overlap o;
  o.d = best;
  if (swapped) {
    o.alpha = best_b;
    o.beta = best_a;
  } else {
    o.alpha = best_a;
    o.beta = best_b;
  }
  return o;
}
// bounding_sphere, collision.cpp:137-153.
void bounding_sphere(const Pill& p, V3& center, double& radius) {
  const V3 axis = sub(p.c1, p.c0);
  const double l = norm(axis);
  if (l + p.r1 <= p.r0) {
    center = p.c0;
    radius = p.r0;
    return;
  }
  if (l + p.r0 <= p.r1) {
    center = p.c1;
    radius = p.r1;
    return;
  }
  const double u = 0.5 * (l + p.r1 - p.r0);
  center = add(p.c0, mul(u / l, axis));
  radius = 0.5 * (l + p.r0 + p.r1);
}
// pair_allowed, collision.cpp:172-180.
bool pair_allowed(const Pill& a, const Pill& b) {
  if (a.rod < 0 && b.rod < 0) return false;
  if (a.group >= 0 && a.group == b.group) return false;
  if (a.rod >= 0 && a.rod == b.rod) {
    if (!a.self_collide) return false;
    if (std::abs(a.element - b.element) <= 1) return false;
  }
  return true;
}
// broad_phase, collision.cpp:184-238. The grid is an ordered map keyed by the cell triple;
// per-i candidate lists are sorted by j, so the result equals the reference's for any map.
std::vector<std::pair<int, int>> broad_phase(const std::vector<Pill>& pills) {
  const int n = static_cast<int>(pills.size());
  std::vector<std::pair<int, int>> pairs;
  if (n < 2) return pairs;
  std::vector<V3> centers(n);
  std::vector<double> radii(n);
  double max_radius = 0.0;
  for (int i = 0; i < n; ++i) {
    bounding_sphere(pills[i], centers[i], radii[i]);
    require(finite(centers[i]) && std::isfinite(radii[i]), "broad_phase: non-finite pill");
    max_radius = std::max(max_radius, radii[i]);
  }
  const double cell = std::max(2.0 * max_radius, 1e-12);
  const double inv_cell = 1.0 / cell;
  using K = std::tuple<int64_t, int64_t, int64_t>;
  auto key_of = [&](const V3& p) {
    return K{static_cast<int64_t>(std::floor(p.x * inv_cell)), static_cast<int64_t>(std::floor(p.y * inv_cell)),
             static_cast<int64_t>(std::floor(p.z * inv_cell))};
  };
  std::map<K, std::vector<int>> grid;
  for (int i = 0; i < n; ++i) grid[key_of(centers[i])].push_back(i);
  std::vector<int> js;
  for (int i = 0; i < n; ++i) {
    const K base = key_of(centers[i]);
    js.clear();
    for (int64_t dx = -1; dx <= 1; ++dx)
      for (int64_t dy = -1; dy <= 1; ++dy)
        for (int64_t dz = -1; dz <= 1; ++dz) {
          const auto it = grid.find(K{std::get<0>(base) + dx, std::get<1>(base) + dy, std::get<2>(base) + dz});
          if (it == grid.end()) continue;
          for (int j : it->second)
            if (j > i && pair_allowed(pills[i], pills[j])) js.push_back(j);
        }
    std::sort(js.begin(), js.end());
    for (int j : js) pairs.emplace_back(i, j);
  }
  return pairs;
}
// pair_key, collision.cpp:240-249.
uint64_t pair_key(const Pill& a, const Pill& b) {
  auto id = [](const Pill& p) {
    const uint32_t rod = static_cast<uint32_t>(p.rod + 1);
    const uint32_t el = static_cast<uint32_t>(p.element + 1);
    return (rod << 16) | (el & 0xffffu);
  };
  uint32_t ia = id(a), ib = id(b);
  if (ia > ib) std::swap(ia, ib);
  return (static_cast<uint64_t>(ia) << 32) | ib;
}
struct Contact {
  int a, b;
  double alpha, beta, d;
};
// find_contacts, collision.cpp:251-273.
std::vector<Contact> find_contacts(const std::vector<Pill>& pills, const std::vector<std::pair<int, int>>& pairs,
                                   int iters, const std::vector<std::pair<uint64_t, double>>* warm) {
  std::unordered_map<uint64_t, double> wm;
  if (warm)
    for (const auto& [k, v] : *warm) wm.emplace(k, v);  // first insertion wins
  std::vector<Contact> out;
  for (const auto& [i, j] : pairs) {
    double wa = -1.0;
    if (warm) {
      const auto it = wm.find(pair_key(pills[i], pills[j]));
      if (it != wm.end()) wa = it->second;
    }
    const Overlap o = deepest_penetration(pills[i], pills[j], iters, wa);
    if (o.d < 0.0) out.push_back({i, j, o.alpha, o.beta, o.d});
  }
  return out;
}
// rod_pills, collision.cpp:275-296.
std::vector<Pill> rod_pills(const std::vector<Rod>& rods) {
  std::vector<Pill> pills;
  for (int r = 0; r < static_cast<int>(rods.size()); ++r) {
    const Rod& rod = rods[r];
    for (int e = 0; e < rod.rest.m(); ++e) {
      Pill p;
      p.c0 = rod.st.c[e];
      p.c1 = rod.st.c[e + 1];
      p.r0 = rod.st.s[e] * rod.rest.r[e];
      p.r1 = rod.st.s[e + 1] * rod.rest.r[e + 1];
      p.rod = r;
      p.element = e;
      p.group = rod.group;
      p.self_collide = rod.self_collide;
      pills.push_back(p);
    }
  }
  return pills;
}

// ---- bundle shape matching (bundling.cpp) ---------------------------------------------------

struct Group {  // BundleGroup, bundling.h:28-36
  std::vector<std::pair<int, int>> members;
  std::vector<V3> rc;
  std::vector<double> rs;
  std::vector<M3> rR;
  V3 rcent;
  double denom = 0.0;
  Q warm{1, 0, 0, 0};
};
int member_element(const Rod& rod, int v) { return std::min(v, rod.rest.m() - 1); }  // bundling.cpp:11-13

// make_bundle_group, bundling.cpp:17-48.
Group make_bundle_group(const std::vector<Rod>& rods, std::vector<std::pair<int, int>> members) {
  require(!members.empty(), "bundle group needs at least one member");
  Group g;
  g.members = std::move(members);
  const int n = static_cast<int>(g.members.size());
  V3 cent{0, 0, 0};
  for (const auto& [mr, mv] : g.members) {
    require_index(mr, static_cast<int>(rods.size()), "bundle member rod");
    require_index(mv, rods[mr].rest.n(), "bundle member vertex");
    cent = add(cent, rods[mr].rest.c[mv]);
  }
  cent = divs(cent, n);
  g.rcent = cent;
  double denom = 0.0;
  for (const auto& [mr, mv] : g.members) {
    const Rod& rod = rods[mr];
    const V3 c = sub(rod.rest.c[mv], cent);
    const double s = rod.rest.s[mv];
    g.rc.push_back(c);
    g.rs.push_back(s);
    g.rR.push_back(qmat(rod.rest.q[member_element(rod, mv)]));
    denom += sqnorm(c) + 3.0 * s * s;
  }
  g.denom = denom;
  return g;
}
// extract_rotation, bundling.cpp:50-67.
Q extract_rotation(const M3& B, const Q& guess, int max_it = 100, double tol = 1e-9) {
  Q q = qnormalized(guess);
  for (int it = 0; it < max_it; ++it) {
    const M3 R = qmat(q);
    V3 omega{0, 0, 0};
    double d = 0.0;
    for (int a = 0; a < 3; ++a) {
      omega = add(omega, cross(R.col(a), B.col(a)));
      d += dot(R.col(a), B.col(a));
    }
    omega = divs(omega, std::abs(d) + 1e-9);
    const double angle = norm(omega);
    if (angle < tol) break;
    q = qnormalized(qmul(qfrom_angle_axis(angle, divs(omega, angle)), q));
  }
  return q;
}
struct Fit {
  double scale = 1.0;
  M3 R = diag(1.0);
  V3 t{0, 0, 0};
  bool degenerate = false;
};
// fit_similarity, bundling.cpp:69-114.
Fit fit_similarity(Group& g, const std::vector<Rod>& rods) {
  const int n = static_cast<int>(g.members.size());
  Fit fit;
  V3 cent{0, 0, 0};
  for (const auto& [mr, mv] : g.members) cent = add(cent, rods[mr].st.c[mv]);
  cent = divs(cent, n);
  M3 B;
  for (int i = 0; i < n; ++i) {
    const auto [mr, mv] = g.members[i];
    const Rod& rod = rods[mr];
    const V3 c = sub(rod.st.c[mv], cent);
    const double s = rod.st.s[mv];
    const M3 R = qmat(rod.st.q[member_element(rod, mv)]);
    madd(B, mmul(mscale(s * g.rs[i], R), mtrans(g.rR[i])));
    M3 outer;
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) outer(p, q) = c[p] * g.rc[i][q];
    madd(B, outer);
  }
  if (mfrob(B) < 1e-12 || g.denom < 1e-300) {
    fit.degenerate = true;
    fit.t = sub(cent, g.rcent);
    return fit;
  }
  g.warm = extract_rotation(B, g.warm);
  fit.R = qmat(g.warm);
  double numer = 0.0;
  for (int i = 0; i < n; ++i) {
    const auto [mr, mv] = g.members[i];
    const Rod& rod = rods[mr];
    const V3 c = sub(rod.st.c[mv], cent);
    const double s = rod.st.s[mv];
    const M3 R = qmat(rod.st.q[member_element(rod, mv)]);
    numer += (s * g.rs[i]) * mcwise_sum(mmul(fit.R, g.rR[i]), R);
    numer += dot(c, mvmul(fit.R, g.rc[i]));
  }
  fit.scale = std::max(numer / g.denom, kMinScale);
  fit.t = sub(cent, mul(fit.scale, mvmul(fit.R, g.rcent)));
  return fit;
}
// apply_shape_match, bundling.cpp:116-133.
Fit apply_shape_match(Group& g, std::vector<Rod>& rods) {
  const Fit fit = fit_similarity(g, rods);
  if (fit.degenerate) return fit;
  const int n = static_cast<int>(g.members.size());
  for (int i = 0; i < n; ++i) {
    const auto [mr, mv] = g.members[i];
    Rod& rod = rods[mr];
    const int e = member_element(rod, mv);
    if (!rod.pinned[mv]) {
      rod.st.c[mv] = add(mul(fit.scale, mvmul(fit.R, add(g.rc[i], g.rcent))), fit.t);
      rod.st.s[mv] = std::max(fit.scale * g.rs[i], kMinScale);
    }
    rod.st.q[e] = qnormalized(qmul(qfrom_mat(fit.R), qfrom_mat(g.rR[i])));
  }
  return fit;
}

// ---- solver (solver.cpp) --------------------------------------------------------------------

struct Loads {  // ExternalLoads, solver.h:35-41
  std::vector<std::vector<V3>> fd, tq;
  std::vector<std::vector<double>> sl;
};

// predict_rod, solver.cpp:21-73.
void predict_rod(Rod& rod, const Material& mat, const V3& g, double h, const std::vector<V3>* fd,
                 const std::vector<V3>* tq, const std::vector<double>* sl) {
  const int n = rod.rest.n(), m = rod.rest.m();
  const double h2 = h * h;
  const double rho = mat.rho;
  for (int v = 0; v < n; ++v) {
    if (rod.pinned[v]) continue;
    V3 accel = g;
    if (fd) {
      require(finite((*fd)[v]), "external force must be finite");
      accel = add(accel, divs((*fd)[v], rho));
    }
    rod.st.c[v] = add(rod.st.c[v], add(mul(h, rod.st.cv[v]), mul(h2, accel)));
    double ds = h * rod.st.sv[v];
    if (sl) {
      double gamma = 0.0;
      int count = 0;
      if (v > 0) {
        gamma += (*sl)[v - 1];
        ++count;
      }
      if (v < m) {
        gamma += (*sl)[v];
        ++count;
      }
      gamma /= count;
      require(std::isfinite(gamma), "external scale load must be finite");
      const double r = rod.rest.r[v];
      ds += 2.0 * h2 * gamma / (kPi * r * r * r * r * rho);
    }
    rod.st.s[v] = std::max(rod.st.s[v] + ds, kMinScale);
  }
  for (int e = 0; e < m; ++e) {
    V3 dth = mul(h, rod.st.av[e]);
    if (tq) {
      require(finite((*tq)[e]), "external torque must be finite");
      const double smid = 0.5 * (rod.st.s[e] + rod.st.s[e + 1]);
      const double rmid = 0.5 * (rod.rest.r[e] + rod.rest.r[e + 1]);
      const double r4 = rmid * rmid * rmid * rmid;
      const V3 bt = qrot(qconj(rod.st.q[e]), (*tq)[e]);
      const V3 ii{4.0 / (kPi * r4), 4.0 / (kPi * r4), 2.0 / (kPi * r4)};
      dth = add(dth, mul(h2 / (smid * smid * rho), cwmul(ii, bt)));
    }
    rod.st.q[e] = apply_increment(rod.st.q[e], dth);
  }
}
// warm_start_lbs, solver.cpp:75-100.
void warm_start_lbs(Rod& rod, const std::vector<Bone>& bones, double t_prev, double t_new) {
  if (rod.bones.empty()) return;
  const int n = rod.rest.n();
  const int bc = static_cast<int>(rod.bones.size());
  std::vector<Q> rp(bc), rn(bc);
  std::vector<V3> pp(bc), pn(bc);
  for (int b = 0; b < bc; ++b) {
    const Bone& bone = bones[rod.bones[b]];
    rp[b] = bone.rotation_at(t_prev);
    rn[b] = bone.rotation_at(t_new);
    pp[b] = bone.position_at(t_prev);
    pn[b] = bone.position_at(t_new);
  }
  for (int v = 0; v < n; ++v) {
    if (rod.pinned[v]) continue;
    const V3 c = rod.st.c[v];
    V3 blended{0, 0, 0};
    for (int b = 0; b < bc; ++b) {
      const Q delta = qmul(rn[b], qconj(rp[b]));
      blended = add(blended, mul(rod.bone_w[v][b], add(qrot(delta, sub(c, pp[b])), pn[b])));
    }
    rod.st.c[v] = blended;
  }
}

struct Report {
  int step = 0;
  double time = 0.0;
  std::vector<double> residuals = std::vector<double>(8, 0.0);
  double max_pen = 0.0;
  int contacts = 0, broad = 0, singular = 0, dof = 0;
};

class Solver {  // solver.h:54-115 / solver.cpp:102-442
 public:
  explicit Solver(Scene sc) : s_(std::move(sc)) {
    s_.validate();
    classic_ = s_.settings.scale_mode == 1;
    L_ = build_layout(s_.rods, s_.materials);
    if (classic_) std::fill(L_.is.begin(), L_.is.end(), 0.0);
    scratch_.resize(L_);
    for (int r = 0; r < static_cast<int>(s_.rods.size()); ++r) {
      const int begin = static_cast<int>(elastic_.size());
      auto blocks = assemble_rod_constraints(s_.rods[r], s_.materials[s_.rods[r].material], r, !classic_);
      elastic_.insert(elastic_.end(), blocks.begin(), blocks.end());
      ranges_.emplace_back(begin, static_cast<int>(elastic_.size()));
    }
    for (int i = 0; i < static_cast<int>(s_.soft_pins.size()); ++i) {
      const SoftPin& sp = s_.soft_pins[i];
      Block b;
      b.kind = kPin;
      b.rod = sp.rod;
      b.loc = sp.vertex;
      b.aux = i;
      b.k = V3{sp.k, sp.k, sp.k};
      pins_.push_back(b);
      pin_targets_.push_back(sp.target);
    }
    for (const auto& members : s_.bundles) groups_.push_back(make_bundle_group(s_.rods, members));
  }

  Report step() {  // solver.cpp:363-388
    const int substeps = s_.settings.substeps;
    const double h = s_.settings.dt / substeps;
    Report total;
    for (int s = 0; s < substeps; ++s) {
      Report part = substep(h, s_.settings.iterations, nullptr);
      total.residuals = part.residuals;
      total.max_pen = std::max(total.max_pen, part.max_pen);
      total.contacts += part.contacts;
      total.broad += part.broad;
      total.singular += part.singular;
      total.dof = part.dof;
    }
    ++step_index_;
    total.step = step_index_;
    total.time = time_;
    return total;
  }

  std::vector<std::vector<double>> probe_convergence(int iterations) {  // solver.cpp:390-398
    require(iterations >= 1, "probe needs at least one iteration");
    std::vector<std::vector<double>> log;
    const double h = s_.settings.dt / s_.settings.substeps;
    substep(h, iterations, &log);
    ++step_index_;
    return log;
  }

  double kinetic_energy() const {  // solver.cpp:400-418
    double en = 0.0;
    for (int slot = 0; slot < L_.V; ++slot) {
      if (L_.ic[slot] == 0.0) continue;
      const Rod& rod = s_.rods[L_.vrod[slot]];
      const int v = L_.vloc[slot];
      en += 0.5 * L_.cw[slot] * sqnorm(rod.st.cv[v]);
      if (L_.is[slot] > 0.0) en += 0.5 * L_.sw[slot] * rod.st.sv[v] * rod.st.sv[v];
    }
    for (int slot = 0; slot < L_.E; ++slot) {
      const Rod& rod = s_.rods[L_.erod[slot]];
      const V3& w = rod.st.av[L_.eloc[slot]];
      en += 0.5 * dot(w, cwmul(L_.tw[slot], w));
    }
    return en;
  }
  double total_volume() const {
    double v = 0.0;
    for (const Rod& rod : s_.rods) v += current_volume(rod.st, rod.rest);
    return v;
  }
  double total_rest_volume() const {
    double v = 0.0;
    for (const Rod& rod : s_.rods) v += rest_volume(rod.rest);
    return v;
  }
  std::vector<Pill> current_pills() const {  // solver.cpp:432-436
    std::vector<Pill> p = rod_pills(s_.rods);
    append_kinematic_pills(time_, p);
    return p;
  }

  Scene s_;
  Layout L_;
  std::vector<Block> elastic_, pins_, contacts_, sweep_;
  std::vector<std::pair<int, int>> ranges_;
  std::vector<V3> pin_targets_;
  std::vector<Group> groups_;
  std::vector<Pill> pills_;
  std::vector<std::pair<uint64_t, double>> warm_;
  std::vector<double> applied_;
  struct Saved {
    std::vector<V3> c;
    std::vector<double> s;
    std::vector<Q> q;
  };
  std::vector<Saved> prev_;
  Scratch scratch_;
  Loads loads_;
  double time_ = 0.0;
  int step_index_ = 0;
  bool classic_ = false;

  Ctx ctx() const { return Ctx{&s_.rods, &L_, &pills_, &s_.planes, &pin_targets_, classic_}; }

 private:

  void animate(double t_new) {  // solver.cpp:138-154
    for (const PinMotion& pm : s_.pin_motions) s_.rods[pm.rod].st.c[pm.vertex] = pm.position_at(t_new);
    applied_.resize(s_.activations.size(), -1.0);
    for (std::size_t i = 0; i < s_.activations.size(); ++i) {
      const Activation& a = s_.activations[i];
      const double amt = a.amount_at(t_new);
      if (amt == applied_[i]) continue;
      apply_activation(s_.rods[a.rod].rest, amt, a.factor, a.first, a.last);
      applied_[i] = amt;
      const auto [begin, end] = ranges_[a.rod];
      refresh_stiffness(elastic_.data() + begin, end - begin, s_.rods, s_.materials);
    }
  }

  void predict_all(double h, double t_prev, double t_new) {  // solver.cpp:156-183
    const bool has = !loads_.fd.empty() || !loads_.tq.empty() || !loads_.sl.empty();
    for (int r = 0; r < static_cast<int>(s_.rods.size()); ++r) {
      Rod& rod = s_.rods[r];
      const std::vector<V3>* fd = nullptr;
      const std::vector<V3>* tq = nullptr;
      const std::vector<double>* sl = nullptr;
      if (has) {
        if (r < static_cast<int>(loads_.fd.size()) && !loads_.fd[r].empty()) fd = &loads_.fd[r];
        if (r < static_cast<int>(loads_.tq.size()) && !loads_.tq[r].empty()) tq = &loads_.tq[r];
        if (r < static_cast<int>(loads_.sl.size()) && !loads_.sl[r].empty()) sl = &loads_.sl[r];
      }
      if (classic_) sl = nullptr;
      predict_rod(rod, s_.materials[rod.material], s_.settings.g, h, fd, tq, sl);
      if (classic_)
        for (int v = 0; v < rod.rest.n(); ++v) rod.st.sv[v] = 0.0;
      warm_start_lbs(rod, s_.bones, t_prev, t_new);
      for (const V3& c : rod.st.c)
        if (!finite(c)) throw SimulationError("non-finite prediction in rod " + std::to_string(r));
    }
  }

  void append_kinematic_pills(double t, std::vector<Pill>& pills) const {  // solver.cpp:185-197
    for (const KinPill& kp : s_.kpills) {
      Pill p = kp.pill;
      if (kp.bone >= 0) {
        const Bone& bone = s_.bones[kp.bone];
        const Q rot = bone.rotation_at(t);
        const V3 pos = bone.position_at(t);
        p.c0 = add(qrot(rot, p.c0), pos);
        p.c1 = add(qrot(rot, p.c1), pos);
      }
      pills.push_back(p);
    }
  }

  void collide(double t_new, Report& rep) {  // solver.cpp:199-251
    pills_ = rod_pills(s_.rods);
    append_kinematic_pills(t_new, pills_);
    const auto pairs = broad_phase(pills_);
    rep.broad += static_cast<int>(pairs.size());
    const auto found = find_contacts(pills_, pairs, s_.settings.dich, &warm_);
    warm_.clear();
    contacts_.clear();
    for (const Contact& c : found) {
      warm_.emplace_back(pair_key(pills_[c.a], pills_[c.b]), c.alpha);
      Block b;
      b.kind = kContact;
      b.unilateral = true;
      b.pill_a = c.a;
      b.aux = c.b;
      b.alpha = c.alpha;
      b.beta = c.beta;
      b.k = V3{s_.settings.contact_k, 0, 0};
      contacts_.push_back(b);
    }
    rep.contacts += static_cast<int>(contacts_.size());
    for (int p = 0; p < static_cast<int>(s_.planes.size()); ++p) {
      const Plane& pl = s_.planes[p];
      for (int r = 0; r < static_cast<int>(s_.rods.size()); ++r) {
        const Rod& rod = s_.rods[r];
        for (int v = 0; v < rod.rest.n(); ++v) {
          const double wr = rod.st.s[v] * rod.rest.r[v];
          const double clearance = dot(pl.n, rod.st.c[v]) - pl.off - wr;
          if (clearance < 0.5 * wr) {
            Block b;
            b.kind = kHalfPlane;
            b.unilateral = true;
            b.rod = r;
            b.loc = v;
            b.aux = p;
            b.k = V3{s_.settings.contact_k, 0, 0};
            contacts_.push_back(b);
          }
        }
      }
    }
  }

  void post_step_scales() {  // solver.cpp:253-271
    for (Rod& rod : s_.rods) {
      const int n = rod.rest.n(), m = rod.rest.m();
      for (int v = 0; v < n; ++v) {
        if (rod.pinned[v]) continue;
        double ratio = 0.0;
        int count = 0;
        for (int e : {v - 1, v}) {
          if (e < 0 || e >= m) continue;
          const double cur = norm(sub(rod.st.c[e + 1], rod.st.c[e]));
          ratio += std::sqrt(rod.rest.len[e] / std::max(cur, 1e-12));
          ++count;
        }
        rod.st.s[v] = std::max(rod.rest.s[v] * ratio / count, kMinScale);
        rod.st.sv[v] = 0.0;
      }
    }
  }

  void finalize_velocities(double h) {  // solver.cpp:273-289
    const double keep = 1.0 - s_.settings.damping;
    for (int r = 0; r < static_cast<int>(s_.rods.size()); ++r) {
      Rod& rod = s_.rods[r];
      const Saved& pv = prev_[r];
      for (int v = 0; v < rod.rest.n(); ++v) {
        rod.st.cv[v] = divs(mul(keep, sub(rod.st.c[v], pv.c[v])), h);
        rod.st.sv[v] = keep * (rod.st.s[v] - pv.s[v]) / h;
      }
      for (int e = 0; e < rod.rest.m(); ++e) {
        const Q d = relative_rotation(pv.q[e], rod.st.q[e]);
        rod.st.av[e] = divs(mul(keep * 2.0, qvec(d)), h);
      }
    }
  }

  double end_of_step_penetration() {  // solver.cpp:291-299
    double deepest = 0.0;
    const Ctx c = ctx();
    for (const Block& b : contacts_) deepest = std::max(deepest, -eval_constraint(b, c).W.x);
    return deepest;
  }

  Report substep(double h, int iterations, std::vector<std::vector<double>>* log) {  // solver.cpp:301-361
    Report rep;
    rep.dof = L_.dof;
    const double t_prev = time_;
    const double t_new = time_ + h;
    animate(t_new);
    prev_.resize(s_.rods.size());
    for (std::size_t r = 0; r < s_.rods.size(); ++r) {
      prev_[r].c = s_.rods[r].st.c;
      prev_[r].s = s_.rods[r].st.s;
      prev_[r].q = s_.rods[r].st.q;
    }
    predict_all(h, t_prev, t_new);
    refresh_orientation_inertia(L_, s_.rods, s_.materials);
    collide(t_new, rep);
    sweep_.clear();
    sweep_.insert(sweep_.end(), elastic_.begin(), elastic_.end());
    sweep_.insert(sweep_.end(), pins_.begin(), pins_.end());
    sweep_.insert(sweep_.end(), contacts_.begin(), contacts_.end());
    for (Block& b : sweep_) b.lambda = V3{0, 0, 0};
    const Ctx c = ctx();
    for (int it = 0; it < iterations; ++it) {
      const SweepOutcome o = jacobi_sweep(sweep_, s_.rods, c, h, s_.settings.beta, scratch_);
      rep.singular = o.skipped_singular;
      if (!groups_.empty() && (it + 1) % s_.settings.sm_period == 0)
        for (Group& g : groups_) apply_shape_match(g, s_.rods);
      if (log) log->push_back(elastic_residual_norms(sweep_.data(), static_cast<int>(elastic_.size()), c));
    }
    std::copy(sweep_.begin(), sweep_.begin() + static_cast<long>(elastic_.size()), elastic_.begin());
    contacts_.assign(sweep_.begin() + static_cast<long>(elastic_.size() + pins_.size()), sweep_.end());
    if (classic_) post_step_scales();
    finalize_velocities(h);
    time_ = t_new;
    rep.residuals = elastic_residual_norms(elastic_.data(), static_cast<int>(elastic_.size()), c);
    rep.max_pen = end_of_step_penetration();
    return rep;
  }
};

// ---- C-ABI glue --------------------------------------------------------------------------

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
// ---- skinning (skinning.cpp) ------------------------------------------------------------

struct PillTransform {  // skinning.h:19-25
  V3 center{0, 0, 0};
  double scale = 1.0;
  Q rotation{1, 0, 0, 0};
};
// rod_pill_transforms, skinning.cpp:9-22.
std::vector<PillTransform> rod_pill_transforms(const std::vector<Rod>& rods) {
  std::vector<PillTransform> out;
  for (const Rod& rod : rods)
    for (int e = 0; e < rod.rest.m(); ++e)
      out.push_back({mul(0.5, add(rod.st.c[e], rod.st.c[e + 1])), 0.5 * (rod.st.s[e] + rod.st.s[e + 1]), rod.st.q[e]});
  return out;
}
// rod_rest_pill_transforms, skinning.cpp:24-37.
std::vector<PillTransform> rod_rest_pill_transforms(const std::vector<Rod>& rods) {
  std::vector<PillTransform> out;
  for (const Rod& rod : rods)
    for (int e = 0; e < rod.rest.m(); ++e)
      out.push_back({mul(0.5, add(rod.rest.c[e], rod.rest.c[e + 1])), 0.5 * (rod.rest.s[e] + rod.rest.s[e + 1]),
                     rod.rest.q[e]});
  return out;
}
// rod_rest_pills, skinning.cpp:39-57.
std::vector<Pill> rod_rest_pills(const std::vector<Rod>& rods) {
  std::vector<Pill> out;
  for (int r = 0; r < static_cast<int>(rods.size()); ++r) {
    const Rod& rod = rods[r];
    for (int e = 0; e < rod.rest.m(); ++e) {
      Pill p;
      p.c0 = rod.rest.c[e];
      p.c1 = rod.rest.c[e + 1];
      p.r0 = rod.rest.s[e] * rod.rest.r[e];
      p.r1 = rod.rest.s[e + 1] * rod.rest.r[e + 1];
      p.rod = r;
      p.element = e;
      out.push_back(p);
    }
  }
  return out;
}
struct SkinBinding {  // skinning.h:31-40
  std::vector<int> offsets, pills;
  std::vector<double> weights;
  std::vector<PillTransform> rest;
  int max_influences = 8;
  int clamped_vertices = 0;
};
struct TriMesh {
  std::vector<V3> vertices;
  std::vector<std::array<int, 3>> triangles;
};
// Top-`keep` selection of partial_sort (score descending, pill ascending), renormalized over the
// kept scores in that order, then listed by pill (skinning.cpp:80-93, 145-157).
void keep_top(std::vector<std::pair<double, int>>& scored, int max_influences, SkinBinding& b) {
  const int keep = std::min<int>(max_influences, static_cast<int>(scored.size()));
  std::partial_sort(scored.begin(), scored.begin() + keep, scored.end(), [](const auto& x, const auto& y) {
    return x.first != y.first ? x.first > y.first : x.second < y.second;
  });
  double total = 0.0;
  for (int k = 0; k < keep; ++k) total += scored[k].first;
  std::sort(scored.begin(), scored.begin() + keep, [](const auto& x, const auto& y) { return x.second < y.second; });
  for (int k = 0; k < keep; ++k) {
    b.pills.push_back(scored[k].second);
    b.weights.push_back(scored[k].first / total);
  }
}
// bind_skin, skinning.cpp:59-105.
SkinBinding bind_skin(const TriMesh& mesh, const std::vector<Pill>& pills, const std::vector<PillTransform>& rest,
                      int max_influences, double epsilon) {
  require(!pills.empty(), "skin binding needs at least one pill");
  require(pills.size() == rest.size(), "pill list and transform list must match");
  require(max_influences >= 1, "max_influences must be at least 1");
  require(epsilon > 0.0, "epsilon must be positive");
  SkinBinding b;
  b.max_influences = max_influences;
  b.rest = rest;
  const int nv = static_cast<int>(mesh.vertices.size()), np = static_cast<int>(pills.size());
  b.offsets.assign(nv + 1, 0);
  std::vector<std::pair<double, int>> scored(np);
  for (int v = 0; v < nv; ++v) {
    bool clamped = false;
    for (int p = 0; p < np; ++p) {
      const double d = pill_project(mesh.vertices[v], pills[p]).d;
      if (d < epsilon) clamped = clamped || d < 0.0;
      const double dc = std::max(d, epsilon);
      scored[p] = {1.0 / (dc * dc), p};
    }
    if (clamped) ++b.clamped_vertices;
    keep_top(scored, max_influences, b);
    b.offsets[v + 1] = static_cast<int>(b.pills.size());
  }
  return b;
}
// smooth_binding, skinning.cpp:107-163.
void smooth_binding(SkinBinding& b, const TriMesh& mesh, int iterations) {
  if (iterations <= 0) return;
  const int nv = static_cast<int>(mesh.vertices.size());
  std::vector<std::vector<int>> nb(nv);
  for (const auto& tri : mesh.triangles)
    for (int k = 0; k < 3; ++k) {
      const int a = tri[k], c = tri[(k + 1) % 3];
      nb[a].push_back(c);
      nb[c].push_back(a);
    }
  for (auto& l : nb) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  for (int it = 0; it < iterations; ++it) {
    SkinBinding n;
    n.offsets.push_back(0);
    for (int v = 0; v < nv; ++v) {
      std::map<int, double> blended;
      for (int k = b.offsets[v]; k < b.offsets[v + 1]; ++k) blended[b.pills[k]] += 0.5 * b.weights[k];
      if (!nb[v].empty()) {
        const double share = 0.5 / nb[v].size();
        for (int u : nb[v])
          for (int k = b.offsets[u]; k < b.offsets[u + 1]; ++k) blended[b.pills[k]] += share * b.weights[k];
      } else {
        for (int k = b.offsets[v]; k < b.offsets[v + 1]; ++k) blended[b.pills[k]] += 0.5 * b.weights[k];
      }
      std::vector<std::pair<double, int>> scored;
      for (const auto& [p, w] : blended) scored.push_back({w, p});
      keep_top(scored, b.max_influences, n);
      n.offsets.push_back(static_cast<int>(n.pills.size()));
    }
    b.offsets = std::move(n.offsets);
    b.pills = std::move(n.pills);
    b.weights = std::move(n.weights);
  }
}
// deform_mesh, skinning.cpp:165-185 (Eigen: conj(q) * v is _transformVector of the conjugate).
void deform_mesh(const SkinBinding& b, const std::vector<PillTransform>& cur, const TriMesh& mesh, std::vector<V3>& out) {
  require(cur.size() == b.rest.size(), "transform count changed since binding");
  const int nv = static_cast<int>(mesh.vertices.size());
  require(static_cast<int>(b.offsets.size()) == nv + 1, "binding does not match mesh");
  out.assign(nv, V3{0, 0, 0});
  for (int v = 0; v < nv; ++v) {
    const V3& rest = mesh.vertices[v];
    V3 blended{0, 0, 0};
    for (int k = b.offsets[v]; k < b.offsets[v + 1]; ++k) {
      const PillTransform& c = cur[b.pills[k]];
      const PillTransform& r = b.rest[b.pills[k]];
      const V3 local = qrot(qconj(r.rotation), sub(rest, r.center));
      blended = add(blended, mul(b.weights[k], add(c.center, mul(c.scale / r.scale, qrot(c.rotation, local)))));
    }
    out[v] = blended;
  }
}

V3 v3(const double* p) { return V3{p[0], p[1], p[2]}; }
Q q4(const double* p) { return Q{p[0], p[1], p[2], p[3]}; }
void put3(double* p, const V3& v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
void put4(double* p, const Q& q) {
  p[0] = q.w;
  p[1] = q.x;
  p[2] = q.y;
  p[3] = q.z;
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
// A batch (vrod_batch_create) is N independent reference solvers stepped in lockstep.
struct vrod_solver {
  std::unique_ptr<Solver> s;
  std::vector<std::unique_ptr<Solver>> batch;
  std::vector<Report> last;
};
namespace {
Solver& one(vrod_solver* h) {
  if (!h->s) throw std::invalid_argument("this query needs a single-scene solver (not a batch)");
  return *h->s;
}
const Solver& one(const vrod_solver* h) { return one(const_cast<vrod_solver*>(h)); }
std::vector<Solver*> all(const vrod_solver* h) {  // the scenes, in order
  std::vector<Solver*> v;
  if (h->s) v.push_back(h->s.get());
  for (const auto& b : h->batch) v.push_back(b.get());
  return v;
}
}  // namespace

extern "C" {

const char* vrod_last_error(void) { return g_error.c_str(); }
const char* vrod_backend_name(void) { return "oracle-cpu"; }
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
    const Rest r = make_rest_pose(c, std::vector<double>(radii, radii + nr),
                                  std::vector<double>(scales, scales + (scales ? ns : 0)));
    const int m = r.m();
    for (int i = 0; i < n; ++i) {
      out->rest_scales[i] = r.s[i];
      out->radii[i] = r.r[i];
    }
    for (int e = 0; e < m; ++e) {
      out->lengths[e] = r.len[e];
      out->initial_lengths[e] = r.len0[e];
      put4(out->rest_frames + 4 * e, r.q[e]);
      out->tangent_dots[e] = r.tdot[e];
      out->scale_grads[e] = r.sgrad[e];
    }
    for (int j = 0; j + 1 < m; ++j) {
      put3(out->darboux + 3 * j, r.darb[j]);
      out->scale_laplacians[j] = r.slap[j];
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
    Rod rod;
    for (int i = 0; i < n; ++i) {
      rod.rest.c.push_back(v3(d->rest_centers + 3 * i));
      rod.rest.s.push_back(d->rest_scales[i]);
      rod.rest.r.push_back(d->radii[i]);
      rod.st.c.push_back(v3(d->centers + 3 * i));
      rod.st.s.push_back(d->scales[i]);
      rod.st.cv.push_back(v3(d->center_vel + 3 * i));
      rod.st.sv.push_back(d->scale_vel[i]);
      rod.pinned.push_back(d->pinned ? d->pinned[i] : 0);
    }
    for (int e = 0; e < m; ++e) {
      rod.rest.len.push_back(d->lengths[e]);
      rod.rest.len0.push_back(d->initial_lengths[e]);
      rod.rest.q.push_back(q4(d->rest_frames + 4 * e));
      rod.rest.tdot.push_back(d->tangent_dots[e]);
      rod.rest.sgrad.push_back(d->scale_grads[e]);
      rod.st.q.push_back(q4(d->frames + 4 * e));
      rod.st.av.push_back(v3(d->angular_vel + 3 * e));
    }
    for (int j = 0; j + 1 < m; ++j) {
      rod.rest.darb.push_back(v3(d->darboux + 3 * j));
      rod.rest.slap.push_back(d->scale_laplacians[j]);
    }
    rod.material = d->material;
    rod.group = d->collision_group;
    rod.self_collide = d->self_collide != 0;
    for (int b = 0; b < d->bone_count; ++b) rod.bones.push_back(d->bones[b]);
    if (d->bone_count > 0)
      for (int i = 0; i < n; ++i)
        rod.bone_w.emplace_back(d->bone_weights + static_cast<std::size_t>(i) * d->bone_count,
                                d->bone_weights + static_cast<std::size_t>(i + 1) * d->bone_count);
    s->scene.rods.push_back(std::move(rod));
  });
}
int vrod_scene_add_plane(vrod_scene* s, const double normal[3], double offset) {
  return guarded([&] { s->scene.planes.push_back(Plane{v3(normal), offset}); });
}
int vrod_scene_add_bone(vrod_scene* s, int32_t k, const double* t, const double* pos, const double* rot) {
  return guarded([&] {
    Bone b;
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
int vrod_scene_add_activation(vrod_scene* s, int32_t rod, double factor, double t_start, double t_end,
                              int32_t first, int32_t last) {
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
}

int vrod_batch_create(int32_t n, const vrod_scene* const* scenes, vrod_solver** out) {
  return guarded([&] {
    require(n >= 1 && scenes != nullptr, "batch needs at least one scene");
    auto h = std::make_unique<vrod_solver>();
    for (int i = 0; i < n; ++i) {
      if (i > 0) {
        const Settings& a = scenes[0]->scene.settings;
        const Settings& b = scenes[i]->scene.settings;
        require(a.dt == b.dt && a.iterations == b.iterations && a.substeps == b.substeps && a.beta == b.beta &&
                    a.g.x == b.g.x && a.g.y == b.g.y && a.g.z == b.g.z && a.dich == b.dich && a.sm_period == b.sm_period && a.contact_k == b.contact_k &&
                    a.damping == b.damping && a.deterministic == b.deterministic && a.scale_mode == b.scale_mode,
                "batch scene " + std::to_string(i) + ": all scenes of a batch must share one SolverSettings");
      }
      h->batch.push_back(std::make_unique<Solver>(scenes[i]->scene));
    }
    *out = h.release();
  });
}
int vrod_solver_scene_count(const vrod_solver* h, int32_t* count) {
  return guarded([&] { *count = h->s ? 1 : static_cast<int32_t>(h->batch.size()); });
}
int vrod_solver_scene_reports(const vrod_solver* h, int32_t capacity, vrod_step_report* reports) {
  return guarded([&] {
    require(capacity >= static_cast<int32_t>(h->last.size()), "scene report capacity too small");
    for (std::size_t i = 0; i < h->last.size(); ++i) put_report(h->last[i], reports + i);
  });
}

int vrod_solver_step(vrod_solver* h, vrod_step_report* out) {
  return guarded([&] {
    if (!h->s) {  // batch: every scene alone, in order; the total as documented in vrod_capi.h
      h->last.clear();
      Report tot;
      for (auto& sv : h->batch) {
        h->last.push_back(sv->step());
        const Report& r = h->last.back();
        tot.step = r.step;
        tot.time = r.time;
        for (int k = 0; k < 8; ++k) tot.residuals[k] = std::max(tot.residuals[k], r.residuals[k]);
        tot.max_pen = std::max(tot.max_pen, r.max_pen);
        tot.contacts += r.contacts;
        tot.broad += r.broad;
        tot.singular += r.singular;
        tot.dof += r.dof;
      }
      put_report(tot, out);
      return;
    }
    const Report r = one(h).step();
    h->last.assign(1, r);
    std::memset(out, 0, sizeof(*out));
    out->step = r.step;
    out->time = r.time;
    for (int k = 0; k < 8; ++k) out->residuals[k] = r.residuals[k];
    out->max_penetration = r.max_pen;
    out->contact_count = r.contacts;
    out->broad_pairs = r.broad;
    out->skipped_singular = r.singular;
    out->dof_count = r.dof;
  });
}
int vrod_solver_probe_convergence(vrod_solver* h, int32_t iterations, double* log) {
  return guarded([&] {
    const auto rows = one(h).probe_convergence(iterations);
    for (std::size_t i = 0; i < rows.size(); ++i)
      for (int k = 0; k < 8; ++k) log[i * 8 + k] = rows[i][k];
  });
}
int vrod_solver_get_info(const vrod_solver* h, vrod_solver_info* info) {
  return guarded([&] {
    std::memset(info, 0, sizeof(*info));
    for (const Solver* sp : all(h)) {
      const Solver& s = *sp;
      info->rod_count += static_cast<int32_t>(s.s_.rods.size());
      info->total_vertices += s.L_.V;
      info->total_elements += s.L_.E;
      info->dof_count += s.L_.dof;
      info->step_index = s.step_index_;
      info->bundle_count += static_cast<int32_t>(s.groups_.size());
      info->elastic_blocks += static_cast<int32_t>(s.elastic_.size());
      info->time = s.time_;
    }
  });
}
int vrod_solver_get_rod_sizes(const vrod_solver* h, int32_t* counts) {
  return guarded([&] {
    int i = 0;
    for (const Solver* sp : all(h))
      for (const Rod& rod : sp->s_.rods) counts[i++] = rod.rest.n();
  });
}
int vrod_solver_get_state(vrod_solver* h, double* c, double* sc, double* f, double* cv, double* sv, double* av) {
  return guarded([&] {
    std::size_t vi = 0, ei = 0;
    for (const Solver* sp : all(h))
      for (const Rod& rod : sp->s_.rods) {
        for (int v = 0; v < rod.rest.n(); ++v, ++vi) {
          if (c) put3(c + 3 * vi, rod.st.c[v]);
          if (sc) sc[vi] = rod.st.s[v];
          if (cv) put3(cv + 3 * vi, rod.st.cv[v]);
          if (sv) sv[vi] = rod.st.sv[v];
        }
        for (int e = 0; e < rod.rest.m(); ++e, ++ei) {
          if (f) put4(f + 4 * ei, rod.st.q[e]);
          if (av) put3(av + 3 * ei, rod.st.av[e]);
        }
      }
  });
}
// Product options (include/vrod_capi.h): the CPU path is always the reference's exact order and
// copies state on demand, so the options are accepted and change nothing here.
int vrod_solver_set_option(vrod_solver*, const char* name, int64_t) {
  return guarded([&] {
    const std::string n = name ? name : "";
    require(n == "state_prefetch" || n == "exact_shape_matching" || n == "phase_timing", "unknown solver option");
  });
}
int vrod_solver_set_state(vrod_solver* h, const double* c, const double* sc, const double* f, const double* cv,
                          const double* sv, const double* av) {
  return guarded([&] {
    std::size_t vi = 0, ei = 0;
    for (Rod& rod : one(h).s_.rods) {
      for (int v = 0; v < rod.rest.n(); ++v, ++vi) {
        if (c) rod.st.c[v] = v3(c + 3 * vi);
        if (sc) rod.st.s[v] = sc[vi];
        if (cv) rod.st.cv[v] = v3(cv + 3 * vi);
        if (sv) rod.st.sv[v] = sv[vi];
      }
      for (int e = 0; e < rod.rest.m(); ++e, ++ei) {
        if (f) rod.st.q[e] = q4(f + 4 * ei);
        if (av) rod.st.av[e] = v3(av + 3 * ei);
      }
    }
  });
}
int vrod_solver_get_rest(vrod_solver* h, double* lengths, double* darb, double* grads, double* laps) {
  return guarded([&] {
    std::size_t ei = 0;
    for (const Rod& rod : one(h).s_.rods) {
      const int m = rod.rest.m();
      for (int e = 0; e < m; ++e, ++ei) {
        if (lengths) lengths[ei] = rod.rest.len[e];
        if (grads) grads[ei] = rod.rest.sgrad[e];
        const bool in = e + 1 < m;
        if (darb) put3(darb + 3 * ei, in ? rod.rest.darb[e] : V3{});
        if (laps) laps[ei] = in ? rod.rest.slap[e] : 0.0;
      }
    }
  });
}
int vrod_solver_set_loads(vrod_solver* h, const double* fd, const uint8_t* fdr, const double* tq,
                          const uint8_t* tqr, const double* sl, const uint8_t* slr) {
  return guarded([&] {
    Loads& L = one(h).loads_;
    const auto& rods = one(h).s_.rods;
    const std::size_t nr = rods.size();
    L = Loads{};
    if (fd) L.fd.resize(nr);
    if (tq) L.tq.resize(nr);
    if (sl) L.sl.resize(nr);
    std::size_t vi = 0, ei = 0;
    for (std::size_t r = 0; r < nr; ++r) {
      const int n = rods[r].rest.n(), m = rods[r].rest.m();
      if (fd && (!fdr || fdr[r]))
        for (int v = 0; v < n; ++v) L.fd[r].push_back(v3(fd + 3 * (vi + v)));
      if (tq && (!tqr || tqr[r]))
        for (int e = 0; e < m; ++e) L.tq[r].push_back(v3(tq + 3 * (ei + e)));
      if (sl && (!slr || slr[r]))
        for (int e = 0; e < m; ++e) L.sl[r].push_back(sl[ei + e]);
      vi += n;
      ei += m;
    }
  });
}
int vrod_solver_energy(vrod_solver* h, double* ke, double* vol, double* rvol) {
  return guarded([&] {
    if (ke) *ke = one(h).kinetic_energy();
    if (vol) *vol = one(h).total_volume();
    if (rvol) *rvol = one(h).total_rest_volume();
  });
}
int vrod_solver_get_inverse_weights(vrod_solver* h, double* ic, double* is, double* it) {
  return guarded([&] {
    const Layout& L = one(h).L_;
    for (int v = 0; v < L.V; ++v) {
      if (ic) ic[v] = L.ic[v];
      if (is) is[v] = L.is[v];
    }
    for (int e = 0; e < L.E; ++e)
      if (it) put3(it + 3 * e, L.it[e]);
  });
}
int vrod_solver_get_weights(vrod_solver* h, double* cw, double* sw, double* tw) {
  return guarded([&] {
    const Layout& L = one(h).L_;
    for (int v = 0; v < L.V; ++v) {
      if (cw) cw[v] = L.cw[v];
      if (sw) sw[v] = L.sw[v];
    }
    for (int e = 0; e < L.E; ++e)
      if (tw) put3(tw + 3 * e, L.tw[e]);
  });
}
int vrod_solver_get_contacts(vrod_solver* h, int64_t cap, int64_t* count, int32_t* a, int32_t* b, double* alpha,
                             double* beta) {
  return guarded([&] {
    int64_t k = 0;
    for (const Block& blk : one(h).contacts_) {
      if (blk.kind != kContact) continue;
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
int vrod_solver_current_pills(vrod_solver* h, int64_t cap, int64_t* count, vrod_pill* out) {
  return guarded([&] {
    const auto p = one(h).current_pills();
    for (std::size_t i = 0; i < p.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = from_pill(p[i]);
    *count = static_cast<int64_t>(p.size());
  });
}
int vrod_pill_project(int64_t n, const double* x, const vrod_pill* pills, double* t, double* d, uint8_t* deg) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      const Projection p = pill_project(v3(x + 3 * i), to_pill(pills[i]));
      if (t) t[i] = p.t;
      if (d) d[i] = p.d;
      if (deg) deg[i] = p.degenerate ? 1 : 0;
    }
  });
}
int vrod_deepest_penetration(int64_t n, const vrod_pill* a, const vrod_pill* b, int32_t iters, const double* warm,
                             double* alpha, double* beta, double* dist) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      const Overlap o = deepest_penetration(to_pill(a[i]), to_pill(b[i]), iters, warm ? warm[i] : -1.0);
      alpha[i] = o.alpha;
      beta[i] = o.beta;
      dist[i] = o.d;
    }
  });
}
int vrod_broad_phase(int64_t n, const vrod_pill* pills, int64_t cap, int64_t* count, int32_t* pairs) {
  return guarded([&] {
    std::vector<Pill> p;
    for (int64_t i = 0; i < n; ++i) p.push_back(to_pill(pills[i]));
    const auto out = broad_phase(p);
    for (std::size_t k = 0; k < out.size() && static_cast<int64_t>(k) < cap; ++k) {
      pairs[2 * k] = out[k].first;
      pairs[2 * k + 1] = out[k].second;
    }
    *count = static_cast<int64_t>(out.size());
  });
}
int vrod_find_contacts(int64_t n, const vrod_pill* pills, int64_t np, const int32_t* pairs, int32_t iters,
                       int64_t nw, const uint64_t* wk, const double* wa, int64_t cap, int64_t* count, int32_t* pa,
                       int32_t* pb, double* alpha, double* beta, double* dist) {
  return guarded([&] {
    std::vector<Pill> p;
    for (int64_t i = 0; i < n; ++i) p.push_back(to_pill(pills[i]));
    std::vector<std::pair<int, int>> pr;
    for (int64_t k = 0; k < np; ++k) pr.emplace_back(pairs[2 * k], pairs[2 * k + 1]);
    std::vector<std::pair<uint64_t, double>> warm;
    for (int64_t k = 0; k < nw; ++k) warm.emplace_back(wk[k], wa[k]);
    const auto out = find_contacts(p, pr, iters, wk ? &warm : nullptr);
    for (std::size_t k = 0; k < out.size() && static_cast<int64_t>(k) < cap; ++k) {
      pa[k] = out[k].a;
      pb[k] = out[k].b;
      alpha[k] = out[k].alpha;
      beta[k] = out[k].beta;
      dist[k] = out[k].d;
    }
    *count = static_cast<int64_t>(out.size());
  });
}
uint64_t vrod_pair_key(const vrod_pill* a, const vrod_pill* b) { return pair_key(to_pill(*a), to_pill(*b)); }

}  // extern "C"

namespace {

void put_transform(const PillTransform& t, vrod_pill_transform* o) {
  put3(o->center, t.center);
  o->scale = t.scale;
  put4(o->rotation, t.rotation);
}
PillTransform to_transform(const vrod_pill_transform& t) { return {v3(t.center), t.scale, q4(t.rotation)}; }
}  // namespace

extern "C" {

int vrod_solver_pill_transforms(vrod_solver* s, int64_t cap, int64_t* count, vrod_pill_transform* out) {
  return guarded([&] {
    const auto v = rod_pill_transforms(one(s).s_.rods);
    for (std::size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) put_transform(v[i], out + i);
    *count = static_cast<int64_t>(v.size());
  });
}
int vrod_solver_rest_pill_transforms(vrod_solver* s, int64_t cap, int64_t* count, vrod_pill_transform* out) {
  return guarded([&] {
    const auto v = rod_rest_pill_transforms(one(s).s_.rods);
    for (std::size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) put_transform(v[i], out + i);
    *count = static_cast<int64_t>(v.size());
  });
}
int vrod_solver_rest_pills(vrod_solver* s, int64_t cap, int64_t* count, vrod_pill* out) {
  return guarded([&] {
    const auto v = rod_rest_pills(one(s).s_.rods);
    for (std::size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = from_pill(v[i]);
    *count = static_cast<int64_t>(v.size());
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
    std::vector<V3> o;
    deform_mesh(sk->binding, tr, sk->mesh, o);
    for (std::size_t v = 0; v < o.size(); ++v) put3(out + 3 * v, o[v]);
  });
}
int vrod_solver_shape_match(vrod_solver* s, int32_t cap, int32_t* count, double* fits) {
  return guarded([&] {
    int32_t k = 0;
    for (Solver* sv : all(s))
      for (Group& g : sv->groups_) {
        const Fit f = apply_shape_match(g, sv->s_.rods);
        if (fits && k < cap) {
          double* o = fits + 14ll * k;
          o[0] = f.scale;
          o[1] = f.t.x;
          o[2] = f.t.y;
          o[3] = f.t.z;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) o[4 + 3 * a + b] = f.R(a, b);
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
    std::vector<Block> blocks = sv.elastic_;
    blocks.insert(blocks.end(), sv.pins_.begin(), sv.pins_.end());
    for (Block& b : blocks) b.lambda = V3{0, 0, 0};
    const SweepOutcome o = jacobi_sweep(blocks, sv.s_.rods, sv.ctx(), h, beta, sv.scratch_);
    if (active) *active = o.active;
    if (singular) *singular = o.skipped_singular;
  });
}
int vrod_solver_elastic_residuals(vrod_solver* s, int64_t cap, int64_t* count, double* W) {
  return guarded([&] {
    Solver& sv = one(s);
    const Ctx c = sv.ctx();
    const int64_t n = static_cast<int64_t>(sv.elastic_.size());
    for (int64_t i = 0; i < n && i < cap && W; ++i) {
      const Eval ev = eval_constraint(sv.elastic_[i], c);
      for (int d = 0; d < 3; ++d) W[3 * i + d] = ev.W[d];
    }
    *count = n;
  });
}
int vrod_extract_rotation(int64_t n, const double* B, const double* guess, int32_t max_iterations, double tolerance,
                          double* out) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      M3 m;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m(a, b) = B[9 * i + 3 * a + b];
      const Q q = extract_rotation(m, q4(guess + 4 * i), max_iterations, tolerance);
      put4(out + 4 * i, q);
    }
  });
}
int vrod_skin_deform_solver(vrod_skin* sk, vrod_solver* s, double* out) {
  return guarded([&] {
    std::vector<V3> o;
    deform_mesh(sk->binding, rod_pill_transforms(one(s).s_.rods), sk->mesh, o);
    if (out)
      for (std::size_t v = 0; v < o.size(); ++v) put3(out + 3 * v, o[v]);
  });
}

}  // extern "C"
