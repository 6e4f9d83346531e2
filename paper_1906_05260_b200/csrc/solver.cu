// Host orchestration of the product Solver (reference: Solver, solver.cpp:102-442).
//
// Construction validates the scene, derives the setup (host_model.cpp), lays the world out in
// device memory (world.cuh) and uploads it once. step() evaluates the per-substep animation
// inputs on the host exactly like the reference (pin paths, activation amounts, bone poses),
// then replays ONE CUDA graph holding every kernel of every substep of the step — predict,
// collide, the I Jacobi sweeps with shape matching, finalize, report — and reads back a single
// StepReport. Nothing leaves the device between steps.
#include "solver.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <map>

namespace vhost {

using namespace vm;
using vdev::StepAccum;

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

template <typename T>
T* Solver::dalloc(std::size_t n) {
  void* p = nullptr;
  const std::size_t bytes = std::max<std::size_t>(n, 1) * sizeof(T);
  check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  check_cuda(cudaMemsetAsync(p, 0, bytes, stream_), "cudaMemset");
  allocs_.push_back(p);
  return static_cast<T*>(p);
}

template <typename T>
static void upload(T* dst, const std::vector<T>& src, cudaStream_t st) {
  if (!src.empty()) check_cuda(cudaMemcpyAsync(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
}

static int next_pow2(long long x) {
  int p = 64;
  while (p < x) p <<= 1;
  return p;
}

Solver::Solver(const SceneData& scene, const BatchLayout* batch) : scene_(scene) {
  if (batch && batch->scenes > 1) {
    batch_ = *batch;
    n_scenes_ = batch->scenes;
  }
  scene_.validate();
  // assemble_rod_constraints validates material and rest pose again (constraints.cpp:284-285)
  setup_ = build_setup(scene_);
  classic_ = scene_.settings.scale_mode == 1;
  const int R = setup_.R, V = setup_.V, vpad = setup_.vpad;
  const int K = static_cast<int>(scene_.kpills.size());
  for (const auto& rod : scene_.rods)
    if (rod.n + 1 >= 65536) throw std::invalid_argument("rod too long for the pair_key warm-start ids (>= 65535 elements)");
  for (int sc = 0; sc < n_scenes_; ++sc) {  // pair ids are scene-local
    const int rods = n_scenes_ > 1 ? batch_.rod_base[sc + 1] - batch_.rod_base[sc] : R;
    if (rods + 1 >= 65536) throw std::invalid_argument("too many rods for the pair_key warm-start ids (>= 65535)");
  }
  for (const auto& kp : scene_.kpills)
    if (kp.pill.element != -1) throw std::invalid_argument("kinematic pills with element != -1 are not supported");

  check_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");

  // ---- world -------------------------------------------------------------------------------
  w_.R = R;
  w_.V = V;
  w_.vpad = vpad;
  w_.E = setup_.E;
  w_.K = K;
  w_.P = setup_.E + K;
  w_.classic = classic_ ? 1 : 0;
  w_.rod_vbase = dalloc<int>(R);
  w_.rod_n = dalloc<int>(R);
  w_.rod_block_base = dalloc<int>(R);
  w_.rod_material = dalloc<int>(R);
  w_.rod_group = dalloc<int>(R);
  w_.rod_self = dalloc<uint8_t>(R);
  w_.rod_ekinds = dalloc<uint8_t>(R);
  w_.rod_vkinds = dalloc<uint8_t>(R);
  w_.load_flags = dalloc<uint8_t>(R);
  w_.slot_rod = dalloc<int>(vpad);
  w_.slot_loc = dalloc<int>(vpad);
  w_.slot_m = dalloc<int>(vpad);
  w_.pinned = dalloc<uint8_t>(vpad);
  w_.vstat = dalloc<double>(static_cast<std::size_t>(vdev::kVStatFields) * vpad);
  w_.estat = dalloc<double>(static_cast<std::size_t>(vdev::kEStatFields) * vpad);
  w_.mat = dalloc<double>(8 * scene_.materials.size());
  w_.X = dalloc<double>(static_cast<std::size_t>(vdev::kStateFields) * vpad);
  w_.Y = dalloc<double>(static_cast<std::size_t>(vdev::kStateFields) * vpad);
  w_.prev = dalloc<double>(static_cast<std::size_t>(vdev::kStateFields) * vpad);
  w_.vel = dalloc<double>(static_cast<std::size_t>(vdev::kVelFields) * vpad);
  w_.lam = dalloc<double>(2ull * vdev::kLamFields * vpad);  // ping-pong pair
  w_.loads = dalloc<double>(7ull * vpad);
  w_.xrec = dalloc<double>(8ull * vpad);
  int nbones_total = 0;
  for (const auto& rod : scene_.rods) nbones_total += static_cast<int>(rod.bones.size());
  w_.has_bones = nbones_total > 0;
  w_.rod_bone_off = dalloc<int>(R + 1);
  w_.rod_bones = dalloc<int>(nbones_total);
  w_.slot_bw_off = dalloc<int>(vpad);
  long long bw_total = 0;
  for (const auto& rod : scene_.rods) bw_total += static_cast<long long>(rod.n) * rod.bones.size();
  w_.bone_w = dalloc<double>(bw_total);

  // ---- collision ---------------------------------------------------------------------------
  c_.P = w_.P;
  c_.T = next_pow2(2ll * std::max(c_.P, 1));
  c_.n_planes = static_cast<int>(scene_.planes.size());
  c_.n_pins = static_cast<int>(scene_.soft_pins.size());
  c_.iters_dich = scene_.settings.dich;
  // Can any pair pass pair_allowed (collision.cpp:172-180)?
  {
    bool any = false;
    std::map<int, int> groups;  // group -> rods with that group (>= 0)
    int ungrouped = 0;
    for (const auto& rod : scene_.rods) {
      if (rod.group >= 0) groups[rod.group]++;
      else ++ungrouped;
      if (rod.self_collide && rod.n >= 4) any = true;
    }
    if (ungrouped + static_cast<int>(groups.size()) >= 2) any = true;
    if (ungrouped >= 1 && R >= 2) any = true;
    for (const auto& kp : scene_.kpills)
      for (const auto& rod : scene_.rods)
        if (kp.pill.group < 0 || kp.pill.group != rod.group) any = true;
    collide_possible_ = any && c_.P >= 2;
  }
  ext_possible_ = collide_possible_ || c_.n_planes > 0 || c_.n_pins > 0;
  // Capacities (overflow raises a capacity error, never truncates). A batch of scenes gets a
  // third of the single-scene headroom: its scenes are small and independent.
  const long long cand_per_pill = n_scenes_ > 1 ? 8 : 24, ct_per_pill = n_scenes_ > 1 ? 4 : 12;
  c_.cand_cap = collide_possible_ ? std::max<long long>(1 << 16, cand_per_pill * c_.P) : 0;
  c_.contact_cap = collide_possible_ ? std::max<long long>(1 << 15, ct_per_pill * c_.P) : 0;
  c_.hp_cap = c_.n_planes * V;
  c_.ext_cap = ext_possible_ ? c_.n_pins + c_.contact_cap + c_.hp_cap : 0;
  c_.pill = dalloc<double>(8ull * std::max(c_.P, 1));
  c_.pill_rod = dalloc<int>(c_.P);
  c_.pill_el = dalloc<int>(c_.P);
  c_.pill_group = dalloc<int>(c_.P);
  c_.pill_self = dalloc<uint8_t>(c_.P);
  c_.pill_id = dalloc<uint32_t>(c_.P);
  c_.bsph = dalloc<double>(4ull * std::max(c_.P, 1));
  c_.cellkey = dalloc<long long>(3ull * std::max(c_.P, 1));
  c_.table = dalloc<int>(c_.T);
  c_.cell_count = dalloc<int>(c_.T);
  c_.cell_start = dalloc<int>(c_.T + 1);
  c_.cell_cursor = dalloc<int>(c_.T);
  c_.slot_key = dalloc<longlong4>(c_.T);
  c_.cell_items = dalloc<int>(c_.P);
  c_.order_smem_cap = vdev::order_cap_for(c_.P);
  c_.cell_attr = dalloc<int4>(std::max(c_.P, 1));
  c_.cell_sph = dalloc<double>(4ull * std::max(c_.P, 1));
  c_.pill_cell = dalloc<int>(c_.P);
  c_.rep_flag = dalloc<int>(c_.P + 1);
  c_.rep_pos = dalloc<int>(c_.P + 1);
  c_.cell_list = dalloc<int>(c_.P);
  c_.cell_span = dalloc<int2>(14ull * std::max(c_.P, 1));
  c_.cand_i = dalloc<int>(c_.cand_cap);
  c_.cand_j = dalloc<int>(c_.cand_cap);
  c_.cand2_i = dalloc<int>(c_.cand_cap);
  c_.cand2_j = dalloc<int>(c_.cand_cap);
  c_.raw_i = dalloc<int>(c_.contact_cap);
  c_.raw_j = dalloc<int>(c_.contact_cap);
  c_.raw_ab = dalloc<double>(2 * c_.contact_cap);
  c_.ct_cnt = dalloc<int>(c_.P + 1);
  c_.ct_off = dalloc<int>(c_.P + 1);
  c_.ct_cur = dalloc<int>(c_.P + 1);
  c_.ct_a = dalloc<int>(c_.contact_cap);
  c_.ct_b = dalloc<int>(c_.contact_cap);
  c_.ct_alpha = dalloc<double>(c_.contact_cap);
  c_.ct_beta = dalloc<double>(c_.contact_cap);
  c_.ct_va = dalloc<int>(c_.contact_cap);
  c_.ct_vb = dalloc<int>(c_.contact_cap);
  c_.warm_rr_key = dalloc<unsigned long long>(c_.contact_cap);
  c_.warm_rr_alpha = dalloc<double>(c_.contact_cap);
  c_.warm_rk_key = dalloc<unsigned long long>(K > 0 ? c_.contact_cap : 1);
  c_.warm_rk_alpha = dalloc<double>(K > 0 ? c_.contact_cap : 1);
  c_.rk_flag = dalloc<int>(K > 0 ? c_.contact_cap + 1 : 1);
  c_.rk_pos = dalloc<int>(K > 0 ? c_.contact_cap + 1 : 1);
  c_.planes = dalloc<double>(4 * std::max(c_.n_planes, 1));
  c_.hp_flag = dalloc<int>(static_cast<std::size_t>(c_.hp_cap) + 1);
  c_.hp_pos = dalloc<int>(static_cast<std::size_t>(c_.hp_cap) + 1);
  c_.hp_slot = dalloc<int>(c_.hp_cap);
  c_.hp_plane = dalloc<int>(c_.hp_cap);
  c_.pin_slot = dalloc<int>(c_.n_pins);
  c_.pin_data = dalloc<double>(4 * std::max(c_.n_pins, 1));
  c_.ext_lam = dalloc<double>(3 * c_.ext_cap);
  c_.ext_contrib = dalloc<double>(16 * c_.ext_cap);
  c_.ext_rec = dalloc<double>(4 * c_.ext_cap);
  c_.ext_pos = dalloc<int>(4 * c_.ext_cap);
  c_.ext_cnt = dalloc<int>(V + 1);
  c_.ext_off = dalloc<int>(V + 1);
  c_.ext_cur = dalloc<int>(V);
  c_.ext_items = dalloc<int>(4 * c_.ext_cap);
  c_.ext_ab = dalloc<double>(4 * c_.ext_cap);
  c_.scalars = dalloc<int>(vdev::kScalars);
  c_.maxr_bits = dalloc<unsigned long long>(1);
  const long long scan_max = std::max<long long>({c_.cand_cap, static_cast<long long>(c_.T), static_cast<long long>(c_.P),
                                                  c_.contact_cap, static_cast<long long>(c_.hp_cap), static_cast<long long>(V)});
  c_.scan_parts = static_cast<int>(vdev::scan_partials_needed(scan_max));
  c_.scan_tmp = dalloc<int>(c_.scan_parts);

  // ---- batch of scenes ---------------------------------------------------------------------
  if (n_scenes_ > 1) {
    const int S = n_scenes_;
    w_.n_scenes = S;
    c_.n_scenes = S;
    w_.rod_scene = dalloc<int>(R);
    w_.scene_vbase = dalloc<int>(S + 1);
    w_.scene_acc = dalloc<vdev::SceneAcc>(S);
    c_.scene_acc = w_.scene_acc;
    c_.pill_scene = dalloc<int>(c_.P);
    c_.scene_maxr = dalloc<unsigned long long>(S);
    c_.plane_scene = dalloc<int>(c_.n_planes);
    c_.warm_rr_scene = dalloc<int>(c_.contact_cap);
    c_.warm_rk_scene = dalloc<int>(K > 0 ? c_.contact_cap : 1);
    d_scene_sing_ = dalloc<int>(S);
    check_cuda(cudaMallocHost(&h_scene_acc_, sizeof(vdev::SceneAcc) * S), "cudaMallocHost");
    std::vector<int> rod_scene(R), vb(S + 1), pill_scene;
    for (int sc = 0; sc < S; ++sc) {
      for (int r = batch_.rod_base[sc]; r < batch_.rod_base[sc + 1]; ++r) rod_scene[r] = sc;
      vb[sc] = batch_.rod_base[sc] < R ? setup_.vbase[batch_.rod_base[sc]] : V;
    }
    vb[S] = V;
    for (int sc = S - 1; sc >= 0; --sc)  // scenes without rods: empty range
      if (batch_.rod_base[sc] == batch_.rod_base[sc + 1]) vb[sc] = vb[sc + 1];
    for (int r = 0; r < R; ++r)
      for (int e = 0; e < scene_.rods[r].n - 1; ++e) pill_scene.push_back(rod_scene[r]);
    pill_scene.insert(pill_scene.end(), batch_.kpill_scene.begin(), batch_.kpill_scene.end());
    upload(w_.rod_scene, rod_scene, stream_);
    upload(w_.scene_vbase, vb, stream_);
    upload(c_.pill_scene, pill_scene, stream_);
    upload(c_.plane_scene, batch_.plane_scene, stream_);
  }

  // ---- shape matching ----------------------------------------------------------------------
  g_.G = static_cast<int>(setup_.groups.size());
  g_.levels = setup_.levels;
  // exact-order shape matching (shape.cuh shape_group_exact): VROD_SHAPE_EXACT=1
  g_.exact = std::getenv("VROD_SHAPE_EXACT") && std::getenv("VROD_SHAPE_EXACT")[0] == '1';
  {
    std::vector<int> off(1, 0), ms, mes, lvl_groups;
    std::vector<double> mrest, grest, warm;
    std::vector<uint8_t> serial;
    for (const auto& g : setup_.groups) {
      for (std::size_t i = 0; i < g.slot.size(); ++i) {
        ms.push_back(g.slot[i]);
        mes.push_back(g.eslot[i]);
        mrest.insert(mrest.end(), {g.rc[i].x, g.rc[i].y, g.rc[i].z, g.rs[i]});
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) mrest.push_back(g.rR[i].m[a][b]);
        mrest.insert(mrest.end(), {g.qR[i].w, g.qR[i].x, g.qR[i].y, g.qR[i].z});
      }
      off.push_back(static_cast<int>(ms.size()));
      grest.insert(grest.end(), {g.rcent.x, g.rcent.y, g.rcent.z, g.denom});
      warm.insert(warm.end(), {1.0, 0.0, 0.0, 0.0});
      serial.push_back(g.serial_apply ? 1 : 0);
    }
    level_off_.assign(g_.levels + 1, 0);
    for (int l = 0; l < g_.levels; ++l) {
      for (int gi = 0; gi < g_.G; ++gi)
        if (setup_.group_level[gi] == l) lvl_groups.push_back(gi);
      level_off_[l + 1] = static_cast<int>(lvl_groups.size());
    }
    g_.off = dalloc<int>(off.size());
    g_.mslot = dalloc<int>(ms.size());
    g_.meslot = dalloc<int>(mes.size());
    g_.mrest = dalloc<double>(mrest.size());
    g_.grest = dalloc<double>(grest.size());
    g_.warm = dalloc<double>(warm.size());
    g_.serial = dalloc<uint8_t>(serial.size());
    g_.level_groups = dalloc<int>(lvl_groups.size());
    upload(g_.off, off, stream_);
    upload(g_.mslot, ms, stream_);
    upload(g_.meslot, mes, stream_);
    upload(g_.mrest, mrest, stream_);
    upload(g_.grest, grest, stream_);
    upload(g_.warm, warm, stream_);
    upload(g_.serial, serial, stream_);
    upload(g_.level_groups, lvl_groups, stream_);
    if (!setup_.chain_groups.empty()) {
      g_.nchains = static_cast<int>(setup_.chain_off.size()) - 1;
      g_.chain_off = dalloc<int>(setup_.chain_off.size());
      g_.chain_groups = dalloc<int>(setup_.chain_groups.size());
      upload(g_.chain_off, setup_.chain_off, stream_);
      upload(g_.chain_groups, setup_.chain_groups, stream_);
    }
  }

  // ---- animation packet ----------------------------------------------------------------------
  al_.n_pm = static_cast<int>(setup_.pin_motion_ids.size());
  al_.n_act = static_cast<int>(scene_.activations.size());
  al_.n_bone = static_cast<int>(scene_.bones.size());
  al_.n_kin = K;
  al_.off_time = 0;
  al_.off_pm = 1;
  al_.off_act = al_.off_pm + 3 * al_.n_pm;
  al_.off_bone = al_.off_act + al_.n_act;
  al_.off_kin = al_.off_bone + 14 * al_.n_bone;
  al_.stride = al_.off_kin + 8 * al_.n_kin;
  const int S = scene_.settings.substeps;
  d_anim_ = dalloc<double>(static_cast<std::size_t>(al_.stride) * S);
  check_cuda(cudaMallocHost(&h_anim_, sizeof(double) * al_.stride * S), "cudaMallocHost");
  {
    std::vector<int> pm_slot;
    for (int id : setup_.pin_motion_ids) {
      const auto& pm = scene_.pin_motions[id];
      pm_slot.push_back(setup_.vbase[pm.rod] + pm.vertex);
    }
    d_pm_slot_ = dalloc<int>(pm_slot.size());
    upload(d_pm_slot_, pm_slot, stream_);
    // activations grouped per rod, in activation order
    std::map<int, std::vector<int>> per_rod;
    for (int i = 0; i < al_.n_act; ++i) per_rod[scene_.activations[i].rod].push_back(i);
    std::vector<int> rod_off(1, 0), list, rods;
    for (auto& [r, ids] : per_rod) {
      rods.push_back(r);
      list.insert(list.end(), ids.begin(), ids.end());
      rod_off.push_back(static_cast<int>(list.size()));
    }
    n_act_rods_ = static_cast<int>(rods.size());
    d_act_rod_off_ = dalloc<int>(rod_off.size());
    d_act_list_ = dalloc<int>(list.size());
    d_act_rods_ = dalloc<int>(rods.size());
    upload(d_act_rod_off_, rod_off, stream_);
    upload(d_act_list_, list, stream_);
    upload(d_act_rods_, rods, stream_);
    std::vector<double> act(al_.n_act, -1.0);  // applied_activation_ starts at -1 (solver.cpp:142)
    for (const auto& a : scene_.activations) act.insert(act.end(), {a.factor, double(a.first), double(a.last)});
    d_act_applied_ = dalloc<double>(act.size());
    upload(d_act_applied_, act, stream_);
  }

  d_acc_ = dalloc<StepAccum>(1);
  check_cuda(cudaMallocHost(&h_acc_, sizeof(StepAccum)), "cudaMallocHost");
  d_singular_ = dalloc<int>(std::max(scene_.settings.iterations, 1));
  d_err_ = dalloc<unsigned long long>(1);
  if (persist_ok_ && n_scenes_ == 1 && g_.levels <= vdev::kMaxPersistLevels) persist_tiles_ = vdev::persistent_tiles(w_);
  if (persist_tiles_ > 0) {
    xrec2_ = dalloc<double>(8ull * w_.vpad);
    ext_lam2_ = dalloc<double>(3 * std::max(c_.ext_cap, 1ll));
    d_bar_ = dalloc<unsigned>(2);  // grid barrier, aux ext releases
    // aux CTAs (external blocks + shape matching on the SMs the tiles leave idle) are opt-in:
    // measured at C3 they do not beat the inline scheme (586 vs 566 us/step), VROD_PERSIST_AUX=1
    persist_aux_ = (std::getenv("VROD_PERSIST_AUX") && std::getenv("VROD_PERSIST_AUX")[0] == '1')
                       ? vdev::persistent_aux_ctas(w_)
                       : 0;
    if (std::getenv("VROD_TRACE") && std::getenv("VROD_TRACE")[0] == '1') {
      d_trace_ = dalloc<unsigned long long>(vdev::kTraceCap);
      check_cuda(cudaMemset(d_trace_, 0, sizeof(unsigned long long) * vdev::kTraceCap), "trace");
    }
  }
  report_parts_ = vdev::report_parts(V);
  d_report_partials_ = dalloc<double>(16ull * std::max(report_parts_, 1));
  d_tail_counter_ = dalloc<unsigned>(1);

  upload_static();
  check_cuda(cudaStreamSynchronize(stream_), "setup");
}

Solver::~Solver() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (stream_) cudaStreamSynchronize(stream_);
  if (flush_buf_) cudaFree(flush_buf_);
  for (void* p : allocs_) cudaFree(p);
  if (h_anim_) cudaFreeHost(h_anim_);
  if (h_acc_) cudaFreeHost(h_acc_);
  if (h_scene_acc_) cudaFreeHost(h_scene_acc_);
  if (h_pack_) cudaFreeHost(h_pack_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (side_) cudaStreamDestroy(side_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Solver::upload_static() {
  const int R = setup_.R, vpad = setup_.vpad;
  const bool scale_kinds = !classic_;
  std::vector<int> vbase = setup_.vbase, rn(R), mat(R), grp(R), bone_off(1, 0), bones;
  std::vector<uint8_t> self(R);
  for (int r = 0; r < R; ++r) {
    const RodData& rod = scene_.rods[r];
    rn[r] = rod.n;
    mat[r] = rod.material;
    grp[r] = rod.group;
    self[r] = rod.self_collide ? 1 : 0;
    bones.insert(bones.end(), rod.bones.begin(), rod.bones.end());
    bone_off.push_back(static_cast<int>(bones.size()));
  }
  w_.max_rod_n = R ? *std::max_element(rn.begin(), rn.end()) : 0;
  upload(w_.rod_vbase, vbase, stream_);
  upload(w_.rod_n, rn, stream_);
  upload(w_.rod_block_base, setup_.block_base, stream_);
  upload(w_.rod_material, mat, stream_);
  upload(w_.rod_group, grp, stream_);
  upload(w_.rod_self, self, stream_);
  upload(w_.rod_ekinds, setup_.ekinds, stream_);
  upload(w_.rod_vkinds, setup_.vkinds, stream_);
  w_.all_kinds = R > 0 && std::all_of(setup_.ekinds.begin(), setup_.ekinds.end(), [](int k) { return k == 15; }) &&
                 std::all_of(setup_.vkinds.begin(), setup_.vkinds.end(), [](int k) { return k == 15; });
  upload(w_.rod_bone_off, bone_off, stream_);
  upload(w_.rod_bones, bones, stream_);
  std::vector<double> mats;
  for (const auto& m : scene_.materials) mats.insert(mats.end(), {m.sx, m.sy, m.sz, m.bx, m.by, m.bz, m.vol, m.rho});
  upload(w_.mat, mats, stream_);

  std::vector<int> srod(vpad, 0), sloc(vpad, 0), sm(vpad, 0), bw_off(vpad, 0);
  std::vector<uint8_t> pinned(vpad, 0);
  std::vector<double> vstat(static_cast<std::size_t>(vdev::kVStatFields) * vpad, 0.0);
  std::vector<double> estat(static_cast<std::size_t>(vdev::kEStatFields) * vpad, 0.0);
  std::vector<double> X(static_cast<std::size_t>(vdev::kStateFields) * vpad, 0.0);
  std::vector<double> vel(static_cast<std::size_t>(vdev::kVelFields) * vpad, 0.0);
  std::vector<double> bw;
  cw_.assign(setup_.V, 0.0);
  sw_.assign(setup_.V, 0.0);
  auto VS = [&](int f, int i) -> double& { return vstat[static_cast<std::size_t>(f) * vpad + i]; };
  auto ES = [&](int f, int i) -> double& { return estat[static_cast<std::size_t>(f) * vpad + i]; };
  auto XS = [&](int f, int i) -> double& { return X[static_cast<std::size_t>(f) * vpad + i]; };
  auto VL = [&](int f, int i) -> double& { return vel[static_cast<std::size_t>(f) * vpad + i]; };
  for (int r = 0; r < R; ++r) {
    const RodData& rod = scene_.rods[r];
    const Material& M = scene_.materials[rod.material];
    const double rho = M.rho, kxy = M.sx + M.sy, bxy = M.bx + M.by;
    const int n = rod.n, m = n - 1, v0 = setup_.vbase[r];
    for (int k = 0; k < n; ++k) {
      const int v = v0 + k;
      srod[v] = r;
      sloc[v] = k;
      sm[v] = m;
      bw_off[v] = static_cast<int>(bw.size());
      for (std::size_t b = 0; b < rod.bones.size(); ++b) bw.push_back(rod.bone_w[k * rod.bones.size() + b]);
      // build_layout, layout.cpp:46-69
      double lump = 0.0;
      if (k > 0) lump += 0.5 * rod.len0[k - 1];
      if (k < n - 1) lump += 0.5 * rod.len0[k];
      const double rbar = rod.r[k];
      const bool pin = rod.pinned[k] != 0;
      pinned[v] = pin ? 1 : 0;
      VS(vdev::RBAR, v) = rbar;
      VS(vdev::SBAR, v) = rod.rs[k];
      if (pin) {
        cw_[v] = kInf;
        sw_[v] = kInf;
        VS(vdev::IC, v) = 0.0;
        VS(vdev::IS, v) = 0.0;
      } else {
        const double cw = kPi * rbar * rbar * rho * lump;
        const double sw = 0.5 * kPi * rbar * rbar * rbar * rbar * rho * lump;
        cw_[v] = cw;
        sw_[v] = sw;
        VS(vdev::IC, v) = 1.0 / cw;
        VS(vdev::IS, v) = classic_ ? 0.0 : 1.0 / sw;  // classic: scale DOFs kinematic (solver.cpp:106-109)
      }
      XS(vdev::CX, v) = rod.c[k].x;
      XS(vdev::CY, v) = rod.c[k].y;
      XS(vdev::CZ, v) = rod.c[k].z;
      XS(vdev::S, v) = rod.s[k];
      VL(vdev::VX, v) = rod.cv[k].x;
      VL(vdev::VY, v) = rod.cv[k].y;
      VL(vdev::VZ, v) = rod.cv[k].z;
      VL(vdev::VS, v) = rod.sv[k];
      if (k < m) {
        XS(vdev::QW, v) = rod.q[k].w;
        XS(vdev::QX, v) = rod.q[k].x;
        XS(vdev::QY, v) = rod.q[k].y;
        XS(vdev::QZ, v) = rod.q[k].z;
        VL(vdev::WX, v) = rod.av[k].x;
        VL(vdev::WY, v) = rod.av[k].y;
        VL(vdev::WZ, v) = rod.av[k].z;
        ES(vdev::LEN, v) = rod.len[k];
        ES(vdev::LEN0, v) = rod.len0[k];
        ES(vdev::TDOT, v) = rod.tdot[k];
        ES(vdev::SGRAD, v) = rod.sgrad[k];
        if (k < m - 1) {
          ES(vdev::SLAP, v) = rod.slap[k];
          ES(vdev::DARBX, v) = rod.darb[k].x;
          ES(vdev::DARBY, v) = rod.darb[k].y;
          ES(vdev::DARBZ, v) = rod.darb[k].z;
        }
        ES(vdev::RQW, v) = rod.rq[k].w;
        ES(vdev::RQX, v) = rod.rq[k].x;
        ES(vdev::RQY, v) = rod.rq[k].y;
        ES(vdev::RQZ, v) = rod.rq[k].z;
        // assemble_rod_constraints element pass (constraints.cpp:302-314)
        const double rmid = 0.5 * (rod.r[k] + rod.r[k + 1]);
        const double a2 = kPi * rmid * rmid;
        const double a4 = 0.25 * kPi * rmid * rmid * rmid * rmid;
        const double l = rod.len[k], l0 = rod.len0[k];
        ES(vdev::A2E, v) = a2;
        ES(vdev::A4EP, v) = 0.25 * kPi * std::pow(rmid, 4);
        ES(vdev::KSZ, v) = inverse_stiffness(a2 * M.sz * l);
        ES(vdev::KCS, v) = inverse_stiffness(a2 * kxy * l);
        ES(vdev::KSS, v) = inverse_stiffness(a4 * kxy * l);
        ES(vdev::KVS, v) = inverse_stiffness(a2 * M.vol * l0);
        // refresh_orientation_inertia at construction (layout.cpp:76-93)
        const double smid = 0.5 * (rod.s[k] + rod.s[k + 1]);
        const double r4 = kPi * rmid * rmid * rmid * rmid;
        const double base = rho * smid * smid * r4 * l0;
        ES(vdev::TWB, v) = base;
        ES(vdev::ITX, v) = 1.0 / (0.25 * base);
        ES(vdev::ITY, v) = 1.0 / (0.25 * base);
        ES(vdev::ITZ, v) = 1.0 / (0.5 * base);
      }
      if (k >= 1 && k <= m - 1) {  // vertex pass (constraints.cpp:315-327)
        const double rv = rod.r[k];
        const double a4 = 0.25 * kPi * rv * rv * rv * rv;
        const double lw = 0.5 * (rod.len[k - 1] + rod.len[k]);
        const double lw0 = 0.5 * (rod.len0[k - 1] + rod.len0[k]);
        ES(vdev::A4VP, v) = 0.25 * kPi * std::pow(rv, 4);
        ES(vdev::KBT0, v) = inverse_stiffness(a4 * M.sz * lw);
        ES(vdev::KBT1, v) = inverse_stiffness(a4 * M.sz * lw);
        ES(vdev::KBT2, v) = inverse_stiffness(a4 * kxy * lw);
        ES(vdev::KSB, v) = inverse_stiffness(a4 * bxy * lw);
        ES(vdev::KVB, v) = inverse_stiffness(2.0 * a4 * M.vol * lw0);
      }
      (void)scale_kinds;
    }
  }
  upload(w_.slot_rod, srod, stream_);
  upload(w_.slot_loc, sloc, stream_);
  upload(w_.slot_m, sm, stream_);
  upload(w_.pinned, pinned, stream_);
  upload(w_.vstat, vstat, stream_);
  upload(w_.estat, estat, stream_);
  upload(w_.X, X, stream_);
  upload(w_.vel, vel, stream_);
  upload(w_.slot_bw_off, bw_off, stream_);
  {  // slot records for the external blocks: current c, s + static rbar, 1/w_c, 1/w_s
    std::vector<double> rec(8ull * vpad, 0.0);
    for (int p = 0; p < setup_.V; ++p) {
      double* o = rec.data() + 8ll * p;
      o[0] = XS(vdev::CX, p);
      o[1] = XS(vdev::CY, p);
      o[2] = XS(vdev::CZ, p);
      o[3] = XS(vdev::S, p);
      o[4] = VS(vdev::RBAR, p);
      o[5] = VS(vdev::IC, p);
      o[6] = VS(vdev::IS, p);
    }
    upload(w_.xrec, rec, stream_);
    if (xrec2_) upload(xrec2_, rec, stream_);  // statics of the persistent kernel's partner records
  }
  upload(w_.bone_w, bw, stream_);

  // static pill attributes: rod pills in (rod, element) order, then kinematic pills
  const int P = c_.P;
  std::vector<int> prod(P), pel(P), pgrp(P);
  std::vector<uint8_t> pself(P);
  std::vector<uint32_t> pid(P);
  int i = 0;
  for (int r = 0; r < R; ++r) {
    const RodData& rod = scene_.rods[r];
    for (int e = 0; e < rod.n - 1; ++e, ++i) {
      prod[i] = r;
      pel[i] = e;
      pgrp[i] = rod.group;
      pself[i] = rod.self_collide ? 1 : 0;
      const int local = n_scenes_ > 1 ? r - batch_.rod_base[std::upper_bound(batch_.rod_base.begin(), batch_.rod_base.end(), r) -
                                                         batch_.rod_base.begin() - 1]
                                      : r;  // pair ids are scene-local in a batch
      pid[i] = (static_cast<uint32_t>(local + 1) << 16) | (static_cast<uint32_t>(e + 1) & 0xffffu);
    }
  }
  for (const auto& kp : scene_.kpills) {
    prod[i] = -1;
    pel[i] = kp.pill.element;
    pgrp[i] = kp.pill.group;
    pself[i] = kp.pill.self_collide ? 1 : 0;
    pid[i] = (0u << 16) | (static_cast<uint32_t>(kp.pill.element + 1) & 0xffffu);
    ++i;
  }
  upload(c_.pill_rod, prod, stream_);
  upload(c_.pill_el, pel, stream_);
  upload(c_.pill_group, pgrp, stream_);
  upload(c_.pill_self, pself, stream_);
  upload(c_.pill_id, pid, stream_);
  std::vector<double> planes;
  for (const auto& p : scene_.planes) planes.insert(planes.end(), {p.first.x, p.first.y, p.first.z, p.second});
  upload(c_.planes, planes, stream_);
  std::vector<int> pin_slot;
  std::vector<double> pin_data;
  for (const auto& sp : scene_.soft_pins) {
    pin_slot.push_back(setup_.vbase[sp.rod] + sp.vertex);
    pin_data.insert(pin_data.end(), {sp.target.x, sp.target.y, sp.target.z, sp.k});
  }
  upload(c_.pin_slot, pin_slot, stream_);
  upload(c_.pin_data, pin_data, stream_);
  int zero_scalars[vdev::kScalars] = {0};
  check_cuda(cudaMemcpyAsync(c_.scalars, zero_scalars, sizeof(zero_scalars), cudaMemcpyHostToDevice, stream_), "scalars");
}

// Host evaluation of the per-substep animation inputs (scene.cpp:22-61, solver.cpp:138-197).
void Solver::fill_animation(int substeps, double h) {
  double t = time_;
  for (int s = 0; s < substeps; ++s) {
    const double t_prev = t;
    const double t_new = t + h;
    double* a = h_anim_ + static_cast<std::size_t>(al_.stride) * s;
    a[al_.off_time] = t_new;
    for (int i = 0; i < al_.n_pm; ++i) {
      const V3 p = scene_.pin_motions[setup_.pin_motion_ids[i]].position_at(t_new);
      a[al_.off_pm + 3 * i] = p.x;
      a[al_.off_pm + 3 * i + 1] = p.y;
      a[al_.off_pm + 3 * i + 2] = p.z;
    }
    for (int i = 0; i < al_.n_act; ++i) a[al_.off_act + i] = scene_.activations[i].amount_at(t_new);
    for (int b = 0; b < al_.n_bone; ++b) {
      const BoneData& bone = scene_.bones[b];
      const Q4 rp = bone.rotation_at(t_prev), rn = bone.rotation_at(t_new);
      const V3 pp = bone.position_at(t_prev), pn = bone.position_at(t_new);
      double* o = a + al_.off_bone + 14 * b;
      const double vals[14] = {rp.w, rp.x, rp.y, rp.z, rn.w, rn.x, rn.y, rn.z, pp.x, pp.y, pp.z, pn.x, pn.y, pn.z};
      std::memcpy(o, vals, sizeof(vals));
    }
    for (int k = 0; k < al_.n_kin; ++k) {
      PillData p = scene_.kpills[k].pill;
      if (scene_.kpills[k].bone >= 0) {
        const BoneData& bone = scene_.bones[scene_.kpills[k].bone];
        const Q4 rot = bone.rotation_at(t_new);
        const V3 pos = bone.position_at(t_new);
        p.c0 = qrot(rot, p.c0) + pos;
        p.c1 = qrot(rot, p.c1) + pos;
      }
      double* o = a + al_.off_kin + 8 * k;
      const double vals[8] = {p.c0.x, p.c0.y, p.c0.z, p.c1.x, p.c1.y, p.c1.z, p.r0, p.r1};
      std::memcpy(o, vals, sizeof(vals));
    }
    t = t_new;
  }
}

// Step prologue: the step accumulator and error word, plus the first substep's resets (the broad
// phase's and the iteration loop's, `f`), one launch instead of three.
__global__ void k_init_acc(StepAccum* acc, unsigned long long* err, int* scalars, vdev::FillList f) {
  vdev::pdl_wait();
  vdev::pdl_trigger();
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int a = 0; a < f.n; ++a)
    for (long long i = t; i < f.count[a]; i += stride) f.ptr[a][i] = f.value[a];
  if (t != 0) return;
  scalars[vdev::SC_OVF] = 0;
  for (int q = 0; q < 8; ++q) acc->residuals[q] = 0.0;
  acc->max_penetration = 0.0;
  acc->contact_count = 0;
  acc->broad_pairs = 0;
  acc->skipped_singular = 0;
  acc->error = ~0ull;
  acc->max_candidates = 0;
  acc->max_contacts = 0;
  *err = ~0ull;
}
// End of a substep: the last sweep's singular count (solver.cpp:335, 375); after the step's last
// substep also the error word (capacity overflow invalidates the results).
__global__ void k_end_substep(StepAccum* acc, const int* singular_last, int last, const unsigned long long* err,
                              const int* scalars) {
  vdev::pdl_wait();
  vdev::pdl_trigger();
  acc->skipped_singular += *singular_last;
  if (!last) return;
  unsigned long long e = *err;
  if (scalars[vdev::SC_OVF]) e = vdev::err_code(0, vdev::ERR_CAPACITY, scalars[vdev::SC_OVF], 0);  // results invalid
  acc->error = e;
}

// Records every kernel of one step (or, with probe_log, one probe substep) on stream_.
void Solver::record_step(double h, int substeps, int iterations, double* probe_log, Prof* prof) {
  cudaStream_t st = stream_;
  const double h2 = h * h;
  const double keep = 1.0 - scene_.settings.damping;
  const double g[3] = {scene_.settings.g.x, scene_.settings.g.y, scene_.settings.g.z};
  // profiling brackets (direct launches only): an event pair per kernel category
  auto begin = [&](int cat) {
    if (!prof) return;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    prof->cat.push_back(cat);
    prof->ev.push_back(a);
    prof->ev.push_back(b);
  };
  auto end = [&]() {
    if (prof) cudaEventRecord(prof->ev.back(), st);
  };
  // the collide bracket also marks the end of its broad phase (phase timing: broad vs narrow)
  auto begin_collide = [&]() {
    begin(CAT_COLLIDE);
    if (!prof) return;
    cudaEvent_t m;
    cudaEventCreate(&m);
    prof->broad_end.push_back(m);
    vdev::g_broad_mark = m;
  };
  // Programmatic dependent launch between the step's kernels (not when profiling: the event
  // brackets between categories would serialize them anyway).
  vdev::g_pdl = pdl_ && !prof;
  if (n_scenes_ > 1)
    check_cuda(cudaMemsetAsync(w_.scene_acc, 0, sizeof(vdev::SceneAcc) * n_scenes_, st), "scene report reset");
  // the first substep's resets ride on the prologue
  const bool persistent0 = persist_tiles_ > 0 && !probe_log;
  auto substep_resets = [&](vdev::FillList& f) {  // multipliers (per-launch path; the persistent kernel keeps
                                                 // them on chip), singular counters, grid-barrier counter
    if (!persistent0) f.add(w_.lam, 2ll * vdev::kLamFields * w_.vpad, 0);
    f.add(d_singular_, iterations, 0);
    if (persistent0) f.add(d_bar_, 2, 0);
  };
  const bool pro_broad = c_.P >= 1 && collide_possible_ && !c_.pill_scene;  // launch_collide's fused-bounds path
  {
    vdev::FillList f;
    if (pro_broad) vdev::broad_reset_list(c_, 1, f);
    substep_resets(f);
    long long mx = 1;
    for (int a = 0; a < f.n; ++a) mx = std::max(mx, f.count[a]);
    const long long b = std::min<long long>((mx + 255) / 256, 148 * 8);
    vdev::launch_kernel(k_init_acc, static_cast<unsigned>(b), 256, 0, st, vdev::g_pdl, d_acc_, d_err_, c_.scalars, f);
  }
  check_cuda(cudaMemcpyAsync(d_anim_, h_anim_, sizeof(double) * al_.stride * substeps, cudaMemcpyHostToDevice, st),
             "anim upload");
  for (int s = 0; s < substeps; ++s) {
    const double* anim = d_anim_ + static_cast<std::size_t>(al_.stride) * s;
    begin(CAT_PREDICT);
    // single-scene worlds of short rods without kinematic pills: the prediction launch also builds
    // the pills and their bounds, after the broad phase's resets (the prologue's for substep 0)
    const bool pills_in_predict = pro_broad && w_.max_rod_n <= 32 && w_.K == 0 && !std::getenv("VROD_PILLS_APART");
    if (pills_in_predict && s > 0) vdev::launch_broad_resets(c_, 1, st);
    vdev::launch_animate_predict(w_, anim, al_, d_pm_slot_, d_act_rod_off_, d_act_list_, d_act_applied_, d_act_rods_,
                                 n_act_rods_, g, h, s, d_err_, pills_in_predict ? &c_ : nullptr, st);
    vdev::g_pills_built = pills_in_predict;
    end();
    begin_collide();
    vdev::g_broad_resets_done = (s == 0 && pro_broad) || pills_in_predict;
    if (c_.P >= 1) vdev::launch_collide(w_, c_, anim, al_, s, d_err_, d_acc_, collide_possible_ ? 1 : 0, st);
    if (prof && vdev::g_broad_mark) {
      // no pair scan ran (nothing can collide): the broad phase ends here
      if (c_.P < 1 || !collide_possible_) cudaEventRecord(vdev::g_broad_mark, st);
      vdev::g_broad_mark = nullptr;
    }
    vdev::launch_halfplanes(w_, c_, st);
    end();
    begin(CAT_EXT_SETUP);
    if (ext_possible_) vdev::launch_ext_setup(w_, c_, st);
    const bool persistent = persist_tiles_ > 0 && !probe_log;
    if (s > 0) {  // per-substep resets (the first substep's ran in the prologue)
      vdev::FillList f;
      substep_resets(f);
      vdev::launch_fill(f, st);
    }
    end();
    double* cur = w_.X;
    double* nxt = w_.Y;
    vdev::SweepParams sp{h, h2, scene_.settings.beta, classic_ ? 1 : 0, 0, s, c_.n_pins, setup_.elastic_blocks,
                         vm::inverse_stiffness(scene_.settings.contact_k), 0, nullptr, nullptr, nullptr};
    const bool pdl = vdev::g_pdl;
    double* lam_a = w_.lam;
    double* lam_b = w_.lam + static_cast<std::size_t>(vdev::kLamFields) * w_.vpad;
    if (persistent) {  // the whole iteration loop in one launch
      vdev::PersistParams pp{};
      pp.X = cur;
      pp.Y = nxt;
      pp.xrec[0] = w_.xrec;
      pp.xrec[1] = xrec2_;
      pp.lam_ext[0] = c_.ext_lam;
      pp.lam_ext[1] = ext_lam2_;
      pp.bar = d_bar_;
      pp.ext_done = d_bar_ + 1;
      pp.tiles = persist_tiles_;
      pp.n_aux = persist_aux_;
      pp.trace = d_trace_;
      pp.trace_cta = std::getenv("VROD_TRACE_CTA") ? std::atoi(std::getenv("VROD_TRACE_CTA")) : 0;
      pp.iterations = iterations;
      pp.sm_period = scene_.settings.sm_period;
      pp.levels = g_.levels;
      pp.has_ext = c_.ext_cap > 0 ? 1 : 0;
      for (int l = 0; l <= g_.levels && g_.G > 0; ++l) pp.level_off[l] = level_off_[l];
      begin(CAT_ITERATE);
      vdev::launch_iterate_persistent(w_, c_, g_, pp, sp, d_singular_, d_err_, st);
      end();
      if (iterations & 1) std::swap(cur, nxt);
    }
    for (int it = 0; it < iterations && !persistent; ++it) {
      sp.iter = it;
      sp.scene_singular = (n_scenes_ > 1 && it == iterations - 1) ? d_scene_sing_ : nullptr;
      sp.lam_in = (it & 1) ? lam_b : lam_a;
      sp.lam_out = (it & 1) ? lam_a : lam_b;
      if (c_.ext_cap > 0) {
        begin(CAT_EXT_SOLVE);
        sp.pdl = pdl ? 1 : 0;
        vdev::launch_ext_solve(w_, c_, cur, sp, d_singular_ + it, d_err_, st);
        end();
      }
      begin(CAT_ROD_SWEEP);
      sp.pdl = !pdl ? 0 : (c_.ext_cap > 0 ? 2 : 1);
      vdev::launch_rod_sweep(w_, c_, cur, nxt, sp, d_singular_ + it, d_err_, st);
      end();
      std::swap(cur, nxt);
      if (g_.G > 0 && (it + 1) % scene_.settings.sm_period == 0) {
        begin(CAT_SHAPE);
        vdev::launch_shape_match(w_, g_, cur, level_off_.data(), pdl, st);
        end();
      }
      if (probe_log) vdev::launch_residuals(w_, cur, w_.classic, d_report_partials_, report_parts_, probe_log + 8 * it, st);
    }
    begin(CAT_REPORT);
    vdev::launch_finalize_from(w_, cur, h, keep, st);
    const bool fork = pack_in_graph_ && use_graph_ && s == substeps - 1 && !probe_log && !prof;
    if (fork) {  // get_state's pack + copy, as a side branch overlapping the report kernels
      check_cuda(cudaEventRecord(ev_fork_, st), "fork");
      check_cuda(cudaStreamWaitEvent(side_, ev_fork_, 0), "fork");
      enqueue_pack(side_);
      check_cuda(cudaEventRecord(ev_join_, side_), "join");
    }
    const bool do_pen = ext_possible_ && (c_.contact_cap + c_.hp_cap) > 0;
    if (n_scenes_ == 1) {  // partials, then one fused tail launch
      // the per-launch sweeps leave the final centers / scales in the slot records too (not the
      // persistent kernel's ping-pong, nor classic mode's post-step scales)
      const double* pen_xrec = !w_.classic && !persistent ? w_.xrec : nullptr;
      vdev::launch_report_tail(w_, c_, w_.X, pen_xrec, w_.classic, d_acc_, do_pen, d_report_partials_, report_parts_,
                               d_singular_ + (iterations - 1), s == substeps - 1 ? 1 : 0, d_err_, d_tail_counter_, st);
    } else {
      vdev::launch_residuals(w_, w_.X, w_.classic, d_report_partials_, report_parts_,
                             reinterpret_cast<double*>(reinterpret_cast<char*>(d_acc_) + offsetof(StepAccum, residuals)), st);
      if (do_pen) vdev::launch_penetration(w_, c_, w_.X, d_acc_, st);
      vdev::launch_scene_report(w_, w_.X, w_.classic, d_scene_sing_, st);
      vdev::launch_kernel(k_end_substep, 1, 1, 0, st, vdev::g_pdl, d_acc_, d_singular_ + (iterations - 1),
                          s == substeps - 1 ? 1 : 0, d_err_, c_.scalars);
    }
    if (fork) check_cuda(cudaStreamWaitEvent(st, ev_join_, 0), "join");
    end();
  }
  vdev::g_pdl = false;
  check_cuda(cudaMemcpyAsync(h_acc_, d_acc_, sizeof(StepAccum), cudaMemcpyDeviceToHost, st), "report download");
  if (n_scenes_ > 1)
    check_cuda(cudaMemcpyAsync(h_scene_acc_, w_.scene_acc, sizeof(vdev::SceneAcc) * n_scenes_, cudaMemcpyDeviceToHost, st),
               "scene report download");
}

static const char* kKindNames[11] = {"stretch_z", "cross_section", "surface_stretch", "bend_twist", "surface_bending",
                                     "volume_stretch", "volume_bend_u", "volume_bend_v", "contact", "half_plane", "pin"};

void Solver::check_error() {
  const unsigned long long e = h_acc_->error;
  if (e == vdev::kNoError) return;
  const int stage = static_cast<int>((e >> 52) & 0xf);
  const unsigned a = static_cast<unsigned>((e >> 32) & 0xfffff);
  const unsigned idx = static_cast<unsigned>(e & 0xffffffffu);
  if (stage == vdev::ERR_PREDICT) {
    const int r = static_cast<int>(a);
    const int n = scene_.rods[r].n;
    if (idx == 0xfffffffeu) throw SimulationError("non-finite prediction in rod " + std::to_string(r));
    if (idx < static_cast<unsigned>(2 * n)) {
      if (idx % 2 == 0) throw std::invalid_argument("external force must be finite");
      throw std::invalid_argument("external scale load must be finite");
    }
    throw std::invalid_argument("external torque must be finite");
  }
  if (stage == vdev::ERR_BROAD) throw std::invalid_argument("broad_phase: non-finite pill");
  if (stage == vdev::ERR_CAPACITY)
    throw std::runtime_error(a == 1 ? "collision candidate capacity exceeded" : "contact capacity exceeded");
  // sweep: map the global block index back to its kind (solver.cpp:324-328 block order)
  const int eb = setup_.elastic_blocks;
  std::string kind;
  if (static_cast<int>(idx) >= eb) {
    const int b = static_cast<int>(idx) - eb;
    kind = b < c_.n_pins ? "pin" : "contact_or_half_plane";
    if (b >= c_.n_pins) {
      int nct = 0;
      check_cuda(cudaMemcpy(&nct, c_.scalars + vdev::SC_NCT, sizeof(int), cudaMemcpyDeviceToHost), "nct");
      kind = (b - c_.n_pins) < nct ? "contact" : "half_plane";
    }
  } else {
    int r = static_cast<int>(std::upper_bound(setup_.block_base.begin(), setup_.block_base.end(), static_cast<int>(idx)) -
                             setup_.block_base.begin()) - 1;
    while (r > 0 && setup_.block_base[r] == setup_.block_base[r - 1] && setup_.block_base[r] > static_cast<int>(idx)) --r;
    const int local = static_cast<int>(idx) - setup_.block_base[r];
    const int m = scene_.rods[r].n - 1;
    const int ek = setup_.ekinds[r], vk = setup_.vkinds[r];
    const int ne = popcount4(ek), nv = popcount4(vk);
    int bits, rank;
    const int* order;
    static const int eorder[4] = {0, 1, 2, 5};  // StretchZ, CrossSection, SurfaceStretch, VolumeStretch
    static const int vorder[4] = {3, 4, 6, 7};  // BendTwist, SurfaceBending, VolumeBendU, VolumeBendV
    if (local < m * ne) {
      bits = ek;
      rank = local % ne;
      order = eorder;
    } else {
      bits = vk;
      rank = (local - m * ne) % nv;
      order = vorder;
    }
    int seen = -1, pick = 0;
    for (int b = 0; b < 4; ++b)
      if (bits & (1 << b)) {
        if (++seen == rank) {
          pick = order[b];
          break;
        }
      }
    kind = kKindNames[pick];
  }
  throw SimulationError("non-finite update from constraint " + kind + " #" + std::to_string(idx));
}

void Solver::ensure_graph() {
  if (graph_exec_) return;
  const int S = scene_.settings.substeps;
  const double h = scene_.settings.dt / S;
  cudaGraph_t graph;
  check_cuda(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
  record_step(h, S, scene_.settings.iterations, nullptr);
  check_cuda(cudaStreamEndCapture(stream_, &graph), "end capture");
  std::size_t n = 0;
  cudaGraphGetNodes(graph, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  cudaGraphGetNodes(graph, nodes.data(), &n);
  int kernels = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nd, &t);
    if (t == cudaGraphNodeTypeKernel) ++kernels;
  }
  kernels_per_step_ = kernels;
  check_cuda(cudaGraphInstantiate(&graph_exec_, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
}

long long Solver::kernel_nodes_per_step() {
  ensure_graph();
  return kernels_per_step_;
}

void Solver::pill_transforms_device(double* d_out) { vdev::launch_pill_transforms(w_, w_.X, d_out, stream_); }

std::vector<double> Solver::shape_match() {
  pack_fresh_ = false;
  std::vector<double> out(14ull * g_.G);
  if (g_.G == 0) return out;
  if (!d_fits_) d_fits_ = dalloc<double>(out.size());
  vdev::launch_shape_match(w_, g_, w_.X, level_off_.data(), false, stream_, d_fits_);
  check_cuda(cudaGetLastError(), "shape match launch");
  check_cuda(cudaMemcpyAsync(out.data(), d_fits_, out.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "shape match");
  check_cuda(cudaStreamSynchronize(stream_), "shape match");
  return out;
}

std::pair<int, int> Solver::jacobi_sweep(double h, double beta) {
  pack_fresh_ = false;
  cudaStream_t st = stream_;
  if (ext_possible_) {  // external blocks of this sweep: the soft pins only
    check_cuda(cudaMemsetAsync(c_.scalars + vdev::SC_NCT, 0, 2 * sizeof(int), st), "sweep reset");  // SC_NCT, SC_NHP
    vdev::launch_ext_setup(w_, c_, st);
  }
  {
    vdev::FillList f;
    f.add(w_.lam, 2ll * vdev::kLamFields * w_.vpad, 0);
    f.add(d_singular_, 1, 0);
    f.add(d_err_, 2, -1);
    vdev::launch_fill(f, st);
  }
  double* lam_a = w_.lam;
  double* lam_b = w_.lam + static_cast<std::size_t>(vdev::kLamFields) * w_.vpad;
  vdev::SweepParams sp{h, h * h, beta, classic_ ? 1 : 0, 0, 0, c_.n_pins, setup_.elastic_blocks,
                       vm::inverse_stiffness(scene_.settings.contact_k), 0, nullptr, lam_a, lam_b};
  vdev::launch_iteration(w_, c_, w_.X, w_.Y, sp, d_singular_, d_err_, st);
  vdev::launch_copy_state(w_, w_.Y, w_.X, st);
  check_cuda(cudaGetLastError(), "sweep launch");
  int singular = 0;
  unsigned long long err = 0;
  check_cuda(cudaMemcpyAsync(&singular, d_singular_, sizeof(int), cudaMemcpyDeviceToHost, st), "sweep");
  check_cuda(cudaMemcpyAsync(&err, d_err_, sizeof(err), cudaMemcpyDeviceToHost, st), "sweep");
  check_cuda(cudaStreamSynchronize(st), "sweep");
  h_acc_->error = err;
  check_error();
  return {setup_.elastic_blocks + c_.n_pins - singular, singular};
}

std::vector<double> Solver::elastic_residuals() {
  std::vector<double> out(3ull * setup_.elastic_blocks);
  if (out.empty()) return out;
  if (!d_blockw_) d_blockw_ = dalloc<double>(out.size());
  vdev::launch_block_residuals(w_, w_.X, w_.classic, d_blockw_, stream_);
  check_cuda(cudaGetLastError(), "residuals launch");
  check_cuda(cudaMemcpyAsync(out.data(), d_blockw_, out.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "residuals");
  check_cuda(cudaStreamSynchronize(stream_), "residuals");
  return out;
}

std::vector<double> Solver::pill_transforms() {
  std::vector<double> out(8ull * setup_.E);
  if (setup_.E == 0) return out;
  if (!d_ptrans_) d_ptrans_ = dalloc<double>(out.size());
  pill_transforms_device(d_ptrans_);
  check_cuda(cudaMemcpyAsync(out.data(), d_ptrans_, out.size() * sizeof(double), cudaMemcpyDeviceToHost, stream_),
             "pill transforms");
  check_cuda(cudaStreamSynchronize(stream_), "pill transforms");
  return out;
}

int Solver::trace(long long* out, int cap) {
  if (!d_trace_) return 0;
  std::vector<unsigned long long> h(vdev::kTraceCap);
  check_cuda(cudaMemcpy(h.data(), d_trace_, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost), "trace");
  if (cap < 0) {  // raw buffer
    const int n = std::min(-cap, vdev::kTraceCap);
    for (int i = 0; i < n; ++i) out[i] = static_cast<long long>(h[i]);
    return n;
  }
  const int n = static_cast<int>(std::min<unsigned long long>(h[0], static_cast<unsigned long long>(cap)));
  for (int i = 0; i < n; ++i) out[i] = static_cast<long long>(h[1 + i]);
  return n;
}
int Solver::contact_count_last() { return h_acc_->contact_count; }

double Solver::bench_run(int steps, long long flush_bytes) {
  pack_fresh_ = false;
  const int S = scene_.settings.substeps;
  const double h = scene_.settings.dt / S;
  ensure_graph();
  if (flush_bytes > 0 && flush_bytes_ < flush_bytes) {
    if (flush_buf_) cudaFree(flush_buf_);
    check_cuda(cudaMalloc(&flush_buf_, flush_bytes), "flush buffer");
    flush_bytes_ = flush_bytes;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double total = 0.0;
  for (int k = 0; k < steps; ++k) {
    fill_animation(S, h);
    if (flush_bytes > 0) check_cuda(cudaMemsetAsync(flush_buf_, k & 0xff, flush_bytes, stream_), "L2 flush");
    cudaEventRecord(a, stream_);
    check_cuda(cudaGraphLaunch(graph_exec_, stream_), "graph launch");
    cudaEventRecord(b, stream_);
    Report r;
    finish_step(h, S, &r);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    total += ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return total;
}

void Solver::kernel_times(int steps, double* ms, long long* launches) {
  pack_fresh_ = false;
  const int S = scene_.settings.substeps;
  const double h = scene_.settings.dt / S;
  for (int c = 0; c < kCategories; ++c) {
    ms[c] = 0.0;
    launches[c] = 0;
  }
  for (int k = 0; k < steps; ++k) {
    Prof prof;
    fill_animation(S, h);
    record_step(h, S, scene_.settings.iterations, nullptr, &prof);
    Report r;
    finish_step(h, S, &r);
    for (std::size_t i = 0; i < prof.cat.size(); ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, prof.ev[2 * i], prof.ev[2 * i + 1]);
      ms[prof.cat[i]] += t;
      launches[prof.cat[i]] += 1;
      cudaEventDestroy(prof.ev[2 * i]);
      cudaEventDestroy(prof.ev[2 * i + 1]);
    }
    for (cudaEvent_t m : prof.broad_end) cudaEventDestroy(m);
  }
}

// Device time per reference phase (solver.cpp:310-359: predict = animate + predict; broad =
// broad_phase; narrow = find_contacts + contact / half-plane blocks; solve = the sweeps and shape
// matching; finalize = velocities + report) from one profiled step's event brackets.
void Solver::phase_times(Prof& prof, Report* r) {
  std::size_t collide_k = 0;
  for (std::size_t i = 0; i < prof.cat.size(); ++i) {
    float t = 0.f;
    cudaEventElapsedTime(&t, prof.ev[2 * i], prof.ev[2 * i + 1]);
    switch (prof.cat[i]) {
      case CAT_PREDICT: r->predict_ms += t; break;
      case CAT_COLLIDE: {
        float b = t;
        if (collide_k < prof.broad_end.size()) cudaEventElapsedTime(&b, prof.ev[2 * i], prof.broad_end[collide_k]);
        ++collide_k;
        r->broad_ms += b;
        r->narrow_ms += t - b;
        break;
      }
      case CAT_EXT_SETUP: r->narrow_ms += t; break;  // contact / half-plane block generation
      case CAT_REPORT: r->finalize_ms += t; break;
      default: r->solve_ms += t; break;
    }
    cudaEventDestroy(prof.ev[2 * i]);
    cudaEventDestroy(prof.ev[2 * i + 1]);
  }
  for (cudaEvent_t m : prof.broad_end) cudaEventDestroy(m);
}

bool Solver::set_option(const std::string& name, long long value) {
  auto drop_graph = [&]() {
    if (graph_exec_) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
  };
  if (name == "state_prefetch") {
    const bool on = value != 0;
    if (on == prefetch_state_) return true;
    prefetch_state_ = on;
    pack_fresh_ = false;
    if (on && !d_pack_) {
      const std::size_t n = 8ull * setup_.V + 7ull * setup_.E;
      d_pack_ = dalloc<double>(n);
      check_cuda(cudaMallocHost(&h_pack_, sizeof(double) * std::max<std::size_t>(n, 1)), "cudaMallocHost");
    }
    if (on && use_graph_ && !side_) {
      check_cuda(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "cudaStreamCreate");
      check_cuda(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "cudaEventCreate");
      check_cuda(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "cudaEventCreate");
    }
    pack_in_graph_ = on && use_graph_;
    drop_graph();
    return true;
  }
  if (name == "exact_shape_matching") {
    g_.exact = value != 0 ? 1 : 0;
    drop_graph();
    return true;
  }
  if (name == "phase_timing") {
    phase_timing_ = value != 0;
    return true;
  }
  return false;
}

void Solver::finish_step(double h, int substeps, Report* out) {
  check_cuda(cudaStreamSynchronize(stream_), "step");
  check_cuda(cudaGetLastError(), "step kernels");
  for (int s = 0; s < substeps; ++s) time_ = time_ + h;
  last_max_cand_ = h_acc_->max_candidates;
  last_max_ct_ = h_acc_->max_contacts;
  if (c_.order_smem_cap >= 0 && last_max_ct_ > c_.order_smem_cap && !std::getenv("VROD_CT_ORDER_CAP") && graph_exec_) {
    // more contacts than the one-CTA sort holds: record the multi-launch ordering from now on
    c_.order_smem_cap = -1;
    cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
  }
  check_error();
  ++step_index_;
  out->step = step_index_;
  out->time = time_;
  std::memcpy(out->residuals, h_acc_->residuals, sizeof(out->residuals));
  out->max_pen = h_acc_->max_penetration;
  out->contacts = h_acc_->contact_count;
  out->broad = h_acc_->broad_pairs;
  out->singular = h_acc_->skipped_singular;
  out->dof = dof_count();
}

Report Solver::step() {
  const auto t0 = std::chrono::steady_clock::now();
  const int S = scene_.settings.substeps;
  const double h = scene_.settings.dt / S;
  fill_animation(S, h);
  Prof prof;
  const bool graph = use_graph_ && !phase_timing_;
  if (graph) {
    ensure_graph();
    check_cuda(cudaGraphLaunch(graph_exec_, stream_), "graph launch");
  } else {
    record_step(h, S, scene_.settings.iterations, nullptr, phase_timing_ ? &prof : nullptr);
  }
  pack_fresh_ = false;
  if (prefetch_state_ && !(graph && pack_in_graph_)) enqueue_pack(stream_);  // rides on the step's sync
  Report rr;
  finish_step(h, S, &rr);
  if (phase_timing_) phase_times(prof, &rr);
  pack_fresh_ = prefetch_state_;
  rr.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  last_report_ = rr;
  return rr;
}

std::vector<double> Solver::probe_convergence(int iterations) {
  pack_fresh_ = false;
  require(iterations >= 1, "probe needs at least one iteration");
  const double h = scene_.settings.dt / scene_.settings.substeps;
  if (iterations > scene_.settings.iterations) {
    // grow the per-iteration singular counters (graph is re-captured lazily)
    d_singular_ = dalloc<int>(iterations);
    if (graph_exec_) {
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
  }
  d_probe_ = dalloc<double>(8ull * iterations);
  fill_animation(1, h);
  record_step(h, 1, iterations, d_probe_);
  std::vector<double> log(8ull * iterations);
  check_cuda(cudaMemcpyAsync(log.data(), d_probe_, sizeof(double) * log.size(), cudaMemcpyDeviceToHost, stream_), "probe");
  check_cuda(cudaStreamSynchronize(stream_), "probe");
  time_ = time_ + h;
  check_error();
  ++step_index_;
  return log;
}

// ---- state access (global slot order with compact element numbering) -----------------------

void Solver::enqueue_pack(cudaStream_t st) {
  const std::size_t n = 8ull * setup_.V + 7ull * setup_.E;
  vdev::launch_pack_state(w_, w_.X, setup_.E, d_pack_, st);
  check_cuda(cudaMemcpyAsync(h_pack_, d_pack_, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "get_state");
}

void Solver::get_state(double* c, double* s, double* q, double* cv, double* sv, double* av) {
  if (!d_pack_) {
    const std::size_t n = 8ull * setup_.V + 7ull * setup_.E;
    d_pack_ = dalloc<double>(n);
    check_cuda(cudaMallocHost(&h_pack_, sizeof(double) * std::max<std::size_t>(n, 1)), "cudaMallocHost");
  }
  if (!pack_fresh_) {
    enqueue_pack(stream_);
    check_cuda(cudaStreamSynchronize(stream_), "get_state");
    pack_fresh_ = true;
  }
  const std::size_t V = static_cast<std::size_t>(setup_.V), E = static_cast<std::size_t>(setup_.E);
  const double* p = h_pack_;
  auto put = [&](double* dst, std::size_t n) {
    if (dst && n) std::memcpy(dst, p, sizeof(double) * n);
    p += n;
  };
  put(c, 3 * V);
  put(s, V);
  put(q, 4 * E);
  put(cv, 3 * V);
  put(sv, V);
  put(av, 3 * E);
}

void Solver::set_state(const double* c, const double* s, const double* q, const double* cv, const double* sv,
                       const double* av) {
  pack_fresh_ = false;
  const int vpad = setup_.vpad;
  std::vector<double> X(static_cast<std::size_t>(vdev::kStateFields) * vpad), vel(static_cast<std::size_t>(vdev::kVelFields) * vpad);
  check_cuda(cudaMemcpyAsync(X.data(), w_.X, sizeof(double) * X.size(), cudaMemcpyDeviceToHost, stream_), "set_state");
  check_cuda(cudaMemcpyAsync(vel.data(), w_.vel, sizeof(double) * vel.size(), cudaMemcpyDeviceToHost, stream_), "set_state");
  check_cuda(cudaStreamSynchronize(stream_), "set_state");
  int e = 0;
  for (int r = 0; r < setup_.R; ++r) {
    const int n = scene_.rods[r].n, v0 = setup_.vbase[r];
    for (int k = 0; k < n; ++k) {
      const int v = v0 + k;
      if (c) {
        X[vdev::CX * vpad + v] = c[3 * v];
        X[vdev::CY * vpad + v] = c[3 * v + 1];
        X[vdev::CZ * vpad + v] = c[3 * v + 2];
      }
      if (s) X[vdev::S * vpad + v] = s[v];
      if (cv) {
        vel[vdev::VX * vpad + v] = cv[3 * v];
        vel[vdev::VY * vpad + v] = cv[3 * v + 1];
        vel[vdev::VZ * vpad + v] = cv[3 * v + 2];
      }
      if (sv) vel[vdev::VS * vpad + v] = sv[v];
      if (k < n - 1) {
        if (q)
          for (int f = 0; f < 4; ++f) X[(vdev::QW + f) * vpad + v] = q[4 * e + f];
        if (av)
          for (int f = 0; f < 3; ++f) vel[(vdev::WX + f) * vpad + v] = av[3 * e + f];
        ++e;
      }
    }
  }
  check_cuda(cudaMemcpyAsync(w_.X, X.data(), sizeof(double) * X.size(), cudaMemcpyHostToDevice, stream_), "set_state");
  check_cuda(cudaMemcpyAsync(w_.vel, vel.data(), sizeof(double) * vel.size(), cudaMemcpyHostToDevice, stream_), "set_state");
  check_cuda(cudaStreamSynchronize(stream_), "set_state");
}

void Solver::get_rest(double* lengths, double* darb, double* grads, double* laps) {
  const int vpad = setup_.vpad;
  std::vector<double> es(static_cast<std::size_t>(vdev::kEStatFields) * vpad);
  check_cuda(cudaMemcpy(es.data(), w_.estat, sizeof(double) * es.size(), cudaMemcpyDeviceToHost), "get_rest");
  int e = 0;
  for (int r = 0; r < setup_.R; ++r) {
    const int m = scene_.rods[r].n - 1, v0 = setup_.vbase[r];
    for (int k = 0; k < m; ++k, ++e) {
      const int v = v0 + k;
      if (lengths) lengths[e] = es[vdev::LEN * vpad + v];
      if (grads) grads[e] = es[vdev::SGRAD * vpad + v];
      const bool in = k + 1 < m;
      if (darb)
        for (int f = 0; f < 3; ++f) darb[3 * e + f] = in ? es[(vdev::DARBX + f) * vpad + v] : 0.0;
      if (laps) laps[e] = in ? es[vdev::SLAP * vpad + v] : 0.0;
    }
  }
}

void Solver::set_loads(const double* fd, const uint8_t* fdr, const double* tq, const uint8_t* tqr, const double* sl,
                       const uint8_t* slr) {
  const int vpad = setup_.vpad, R = setup_.R;
  std::vector<double> L(7ull * vpad, 0.0);
  std::vector<uint8_t> flags(R, 0);
  int e = 0;
  for (int r = 0; r < R; ++r) {
    const int n = scene_.rods[r].n, v0 = setup_.vbase[r];
    if (fd && (!fdr || fdr[r])) flags[r] |= 1;
    if (tq && (!tqr || tqr[r])) flags[r] |= 2;
    if (sl && (!slr || slr[r])) flags[r] |= 4;
    for (int k = 0; k < n; ++k) {
      const int v = v0 + k;
      if (flags[r] & 1)
        for (int f = 0; f < 3; ++f) L[f * vpad + v] = fd[3 * v + f];
      if (k < n - 1) {
        if (flags[r] & 2)
          for (int f = 0; f < 3; ++f) L[(3 + f) * vpad + v] = tq[3 * e + f];
        if (flags[r] & 4) L[6 * vpad + v] = sl[e];
        ++e;
      }
    }
  }
  bool any = false;
  for (uint8_t f : flags) any = any || f;
  upload(w_.loads, L, stream_);
  upload(w_.load_flags, flags, stream_);
  check_cuda(cudaStreamSynchronize(stream_), "set_loads");
  if (w_.has_loads != (any ? 1 : 0)) {
    w_.has_loads = any ? 1 : 0;
    if (graph_exec_) {  // the flag is a kernel argument baked into the graph
      cudaGraphExecDestroy(graph_exec_);
      graph_exec_ = nullptr;
    }
  }
}

void Solver::energy(double* ke, double* vol, double* rest_vol) {
  // Solver::kinetic_energy (solver.cpp:400-418) and current_volume (rod.cpp:178-187) on the
  // device: terms in parallel, sums in the reference's sequential order (launch_energy).
  if (ke || vol) {
    const std::size_t V = static_cast<std::size_t>(setup_.V), R = static_cast<std::size_t>(setup_.R);
    if (!d_energy_) {
      d_energy_ = dalloc<double>(6 * V + R + 2);
      check_cuda(cudaMemcpyAsync(d_energy_ + 4 * V, cw_.data(), sizeof(double) * V, cudaMemcpyHostToDevice, stream_), "energy");
      check_cuda(cudaMemcpyAsync(d_energy_ + 5 * V, sw_.data(), sizeof(double) * V, cudaMemcpyHostToDevice, stream_), "energy");
    }
    double* terms = d_energy_;
    double* out = d_energy_ + 6 * V + R;
    vdev::launch_energy(w_, w_.X, d_energy_ + 4 * V, d_energy_ + 5 * V, classic_ ? 1 : 0, terms, d_energy_ + 6 * V, out,
                        stream_);
    double res[2];
    check_cuda(cudaMemcpyAsync(res, out, sizeof(res), cudaMemcpyDeviceToHost, stream_), "energy");
    check_cuda(cudaStreamSynchronize(stream_), "energy");
    if (ke) *ke = res[0];
    if (vol) *vol = res[1];
  }
  if (rest_vol) {  // rest_volume, rod.cpp:189-197
    double t = 0.0;
    for (const RodData& rod : scene_.rods) {
      double v = 0.0;
      for (int e = 0; e < rod.n - 1; ++e) {
        const double s = 0.5 * (rod.rs[e] + rod.rs[e + 1]);
        const double rr = 0.5 * (rod.r[e] + rod.r[e + 1]);
        v += kPi * (s * rr) * (s * rr) * rod.len0[e];
      }
      t += v;
    }
    *rest_vol = t;
  }
}

void Solver::weights(double* cw, double* sw, double* tw) {
  const int vpad = setup_.vpad;
  std::vector<double> twb(vpad);
  check_cuda(cudaMemcpy(twb.data(), w_.estat + static_cast<std::size_t>(vdev::TWB) * vpad, sizeof(double) * vpad,
                        cudaMemcpyDeviceToHost), "weights");
  int e = 0;
  for (int r = 0; r < setup_.R; ++r) {
    const int n = scene_.rods[r].n, v0 = setup_.vbase[r];
    for (int k = 0; k < n; ++k) {
      const int v = v0 + k;
      if (cw) cw[v] = cw_[v];
      if (sw) sw[v] = sw_[v];
      if (k < n - 1) {
        // refresh_orientation_inertia (layout.cpp:84-88): (0.25, 0.25, 0.5) x base
        const double b = twb[v];
        if (tw) {
          tw[3 * e] = 0.25 * b;
          tw[3 * e + 1] = 0.25 * b;
          tw[3 * e + 2] = 0.5 * b;
        }
        ++e;
      }
    }
  }
}

void Solver::inverse_weights(double* ic, double* is, double* it) {
  const int vpad = setup_.vpad;
  std::vector<double> vs(static_cast<std::size_t>(vdev::kVStatFields) * vpad), es(static_cast<std::size_t>(vdev::kEStatFields) * vpad);
  check_cuda(cudaMemcpy(vs.data(), w_.vstat, sizeof(double) * vs.size(), cudaMemcpyDeviceToHost), "weights");
  check_cuda(cudaMemcpy(es.data(), w_.estat, sizeof(double) * es.size(), cudaMemcpyDeviceToHost), "weights");
  int e = 0;
  for (int r = 0; r < setup_.R; ++r) {
    const int n = scene_.rods[r].n, v0 = setup_.vbase[r];
    for (int k = 0; k < n; ++k) {
      const int v = v0 + k;
      if (ic) ic[v] = vs[vdev::IC * vpad + v];
      if (is) is[v] = vs[vdev::IS * vpad + v];
      if (k < n - 1) {
        if (it)
          for (int f = 0; f < 3; ++f) it[3 * e + f] = es[(vdev::ITX + f) * vpad + v];
        ++e;
      }
    }
  }
}

long long Solver::contacts(long long cap, int* a, int* b, double* alpha, double* beta) {
  if (!collide_possible_) return 0;
  int n = 0;
  check_cuda(cudaMemcpy(&n, c_.scalars + vdev::SC_NCT, sizeof(int), cudaMemcpyDeviceToHost), "contacts");
  const long long k = std::min<long long>(cap, n);
  if (k > 0) {
    if (a) check_cuda(cudaMemcpy(a, c_.ct_a, sizeof(int) * k, cudaMemcpyDeviceToHost), "contacts");
    if (b) check_cuda(cudaMemcpy(b, c_.ct_b, sizeof(int) * k, cudaMemcpyDeviceToHost), "contacts");
    if (alpha) check_cuda(cudaMemcpy(alpha, c_.ct_alpha, sizeof(double) * k, cudaMemcpyDeviceToHost), "contacts");
    if (beta) check_cuda(cudaMemcpy(beta, c_.ct_beta, sizeof(double) * k, cudaMemcpyDeviceToHost), "contacts");
  }
  return n;
}

std::vector<PillData> Solver::current_pills() {  // Solver::current_pills, solver.cpp:432-436
  const int V = setup_.V;
  std::vector<double> c(3ull * V), s(V);
  get_state(c.data(), s.data(), nullptr, nullptr, nullptr, nullptr);
  std::vector<PillData> out;
  for (int r = 0; r < setup_.R; ++r) {
    const RodData& rod = scene_.rods[r];
    const int v0 = setup_.vbase[r];
    for (int e = 0; e < rod.n - 1; ++e) {
      PillData p;
      const int v = v0 + e;
      p.c0 = V3{c[3 * v], c[3 * v + 1], c[3 * v + 2]};
      p.c1 = V3{c[3 * v + 3], c[3 * v + 4], c[3 * v + 5]};
      p.r0 = s[v] * rod.r[e];
      p.r1 = s[v + 1] * rod.r[e + 1];
      p.rod = r;
      p.element = e;
      p.group = rod.group;
      p.self_collide = rod.self_collide;
      out.push_back(p);
    }
  }
  for (const auto& kp : scene_.kpills) {
    PillData p = kp.pill;
    if (kp.bone >= 0) {
      const BoneData& bone = scene_.bones[kp.bone];
      const Q4 rot = bone.rotation_at(time_);
      const V3 pos = bone.position_at(time_);
      p.c0 = qrot(rot, p.c0) + pos;
      p.c1 = qrot(rot, p.c1) + pos;
    }
    out.push_back(p);
  }
  return out;
}

}  // namespace vhost

namespace vhost {

std::vector<Report> Solver::scene_reports() const {
  if (n_scenes_ <= 1) return {last_report_};
  std::vector<Report> out(n_scenes_);
  for (int sc = 0; sc < n_scenes_; ++sc) {
    const vdev::SceneAcc& a = h_scene_acc_[sc];
    Report& r = out[sc];
    r.step = last_report_.step;
    r.time = last_report_.time;
    r.total_ms = last_report_.total_ms;
    r.contacts = a.contact_count;
    r.broad = a.broad_pairs;
    r.singular = a.skipped_singular;
    r.max_pen = a.max_penetration;
    for (int k = 0; k < 8; ++k) r.residuals[k] = a.residuals[k];
    int dof = 0;
    for (int rod = batch_.rod_base[sc]; rod < batch_.rod_base[sc + 1]; ++rod)
      dof += 4 * scene_.rods[rod].n + 3 * (scene_.rods[rod].n - 1);
    r.dof = dof;
  }
  return out;
}

}  // namespace vhost
