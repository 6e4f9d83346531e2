// Launch interfaces of the product's sm_100a kernels. One substep (solver.cpp:301-361) is:
//
//   animate      pin motions + activation rest refresh         integrate.cu
//   predict      prev snapshot, inertial prediction, LBS,      integrate.cu
//                orientation inertia
//   collide      pills -> bounding spheres -> hash grid ->     collide.cu
//                candidate count/fill -> narrow phase -> ordered contacts, half-planes
//   ext setup    external-block incidence (slot -> blocks)      sweep.cu
//   I x sweep    external blocks, fused rod stencil sweep       sweep.cu
//                (+ shape matching every period)               shape.cu
//   finalize     classic scales, velocities                    integrate.cu
//   report       residual RMS per kind, penetration            sweep.cu
//
// Everything is launched on one stream with device-side counts so a whole step is
// capturable in one CUDA graph.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "world.cuh"

namespace vdev {

// Per-substep collision / external-block buffers.
struct Collide {
  int P = 0;            // pills
  int n_scenes = 1;     // batch: see World
  int T = 0;            // hash table size (power of two >= 2P)
  long long cand_cap = 0;
  long long contact_cap = 0;
  int hp_cap = 0;
  int n_planes = 0;
  int n_pins = 0;
  int iters_dich = 10;
  // contact ordering: >= 0 runs k_ct_order (one CTA; bitonic sort in shared memory of up to this
  // many contacts, a single-CTA counting sort beyond); -1 the multi-launch counting sort
  int order_smem_cap = -1;
  int scan_parts = 0;

  // pills (SoA): c0xyz c1xyz r0 r1 = 8 fields x P
  double* pill = nullptr;
  int* pill_rod = nullptr;
  int* pill_el = nullptr;
  int* pill_group = nullptr;
  uint8_t* pill_self = nullptr;
  uint32_t* pill_id = nullptr;   // pair_key id (collision.cpp:241-245)
  double* bsph = nullptr;        // bounding spheres: cx cy cz R (4 x P)
  long long* cellkey = nullptr;  // 3 x P
  // grid
  int* table = nullptr;          // T: representative pill or -1
  int* cell_count = nullptr;     // T
  int* cell_start = nullptr;     // T+1
  int* cell_cursor = nullptr;    // T
  longlong4* slot_key = nullptr; // T: key (kx, ky, kz, scene) of an occupied table slot (written by k_scatter)
  int* cell_items = nullptr;     // P
  int4* cell_attr = nullptr;     // P, cell-sorted: (pill, rod, group, 2 * element + self)
  double* cell_sph = nullptr;    // 4 x P, cell-sorted AoS bounding spheres (cx cy cz R)
  int* pill_cell = nullptr;      // P
  int* rep_flag = nullptr;       // P+1: pill is its cell's representative
  int* rep_pos = nullptr;        // P+1: exclusive scan of rep_flag ([P] = cell count)
  int* cell_list = nullptr;      // P: non-empty table slots, representative order
  int2* cell_span = nullptr;     // 14 x P: per non-empty cell, its half-stencil neighbourhood spans (start, size)
  // candidates
  int* cand_count = nullptr;     // P+1
  int* cand_off = nullptr;       // P+1
  int* cand_i = nullptr;         // cand_cap
  int* cand_j = nullptr;
  int* cand2_i = nullptr;        // cand_cap: survivors of the exact segment test
  int* cand2_j = nullptr;
  int* cand_flag = nullptr;      // cand_cap+1
  int* cand_pos = nullptr;       // cand_cap+1
  double* cand_ab = nullptr;     // 3 x cand_cap (alpha, beta, distance)
  // contacts (current substep), ordered by (pill_a, pill_b)
  int* ct_a = nullptr;
  int* ct_b = nullptr;
  double* ct_alpha = nullptr;
  double* ct_beta = nullptr;
  double* ct_dist = nullptr;     // standalone find_contacts only
  int* ct_va = nullptr;          // first slot of each contact's pills (-1: kinematic), per substep
  int* ct_vb = nullptr;
  // raw (unordered) narrow-phase hits and the (i, j) ordering scratch
  int* raw_i = nullptr;          // contact_cap
  int* raw_j = nullptr;
  double* raw_ab = nullptr;      // 2 x contact_cap
  int* ct_cnt = nullptr;         // P+1
  int* ct_off = nullptr;         // P+1
  int* ct_cur = nullptr;         // P+1
  // warm-start lists from the previous substep (sorted by pair key)
  unsigned long long* warm_rr_key = nullptr;
  double* warm_rr_alpha = nullptr;
  unsigned long long* warm_rk_key = nullptr;
  double* warm_rk_alpha = nullptr;
  int* rk_flag = nullptr;        // contact_cap+1 scratch
  int* rk_pos = nullptr;
  // half-planes
  double* planes = nullptr;      // 4 x n_planes (nx ny nz offset)
  int* hp_flag = nullptr;        // n_planes*V + 1
  int* hp_pos = nullptr;
  int* hp_slot = nullptr;        // hp_cap
  int* hp_plane = nullptr;
  // pins (static): slot, target xyz, stiffness
  int* pin_slot = nullptr;
  double* pin_data = nullptr;    // 4 x n_pins
  // external blocks: pins | contacts | half-planes
  long long ext_cap = 0;
  double* ext_lam = nullptr;     // 3 x ext_cap, SoA: component d of block b at [d * ext_cap + b]
  // Results are written per incidence entry q (slot-sorted), so the sweep's gather reads
  // contiguous entries instead of chasing block ids.
  double* ext_contrib = nullptr; // 4 x (4 x ext_cap): entry q -> dc xyz, ds (kExtNone markers)
  // Per external block b, 4 doubles (k_ext_solve -> the per-launch sweeps' gathers): pin
  // {dc xyz, none}, half-plane {dc xyz, ds}, contact {unit normal xyz, dlambda}; kExtNone in
  // [0] (pin, half-plane) or [3] (contact) = no update. A contact's four endpoint corrections are
  // re-formed by each endpoint's gather from these (ext.cuh contact_endpoint), 32 B per contact
  // instead of 4 x 32 B of per-endpoint entries.
  double* ext_rec = nullptr;
  int* ext_pos = nullptr;        // 4 x ext_cap: (block << 2 | endpoint) -> entry q
  int* ext_cnt = nullptr;        // V+1 incidence counts
  int* ext_off = nullptr;        // V+1
  int* ext_cur = nullptr;        // V
  int* ext_items = nullptr;      // 4 x ext_cap entries (block << 2 | endpoint)
  double* ext_ab = nullptr;      // 4 x ext_cap, per entry q: its contact's alpha (endpoints 0, 1) /
                                 // beta (2, 3), 0 for pins and half-planes — frozen for the substep
  // batch of scenes (World::n_scenes > 1): pairs only within a scene, per-scene grid cell
  int* pill_scene = nullptr;     // P
  unsigned long long* scene_maxr = nullptr;  // per scene: max bounding radius bits
  int* plane_scene = nullptr;    // n_planes
  int* warm_rr_scene = nullptr;  // scene of each warm entry (lists are scene-major)
  int* warm_rk_scene = nullptr;
  SceneAcc* scene_acc = nullptr; // == World::scene_acc
  // device scalars
  int* scalars = nullptr;        // see Scalar enum
  unsigned long long* maxr_bits = nullptr;
  int* scan_tmp = nullptr;       // scan partials
};
enum : int { kExtCenter = 1, kExtScale = 2 };
// "No update" marker of an incidence entry: a NaN with a private payload in dc.x (the block
// made no update) or in ds (no scale update: soft pins). A computed non-finite update can never
// be applied silently — the ext solve flags it as the reference's SimulationError.
constexpr unsigned long long kExtNoneBits = 0x7ff4e0de00000001ull;
#ifdef __CUDACC__
__device__ __forceinline__ double ext_none() { return __longlong_as_double(static_cast<long long>(kExtNoneBits)); }
__device__ __forceinline__ bool is_ext_none(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(v)) == kExtNoneBits;
}
#endif
enum Scalar : int { SC_NCAND = 0, SC_NCT, SC_NHP, SC_NRR, SC_NRK, SC_NRR_PREV, SC_NRK_PREV, SC_BROAD, SC_OVF,
                    SC_NCAND_RAW, SC_NCT_RAW, SC_NCAND2, kScalars };

struct Groups {  // shape matching (bundling.cpp)
  int G = 0;
  int levels = 0;
  int* off = nullptr;            // G+1 member offsets
  int* mslot = nullptr;          // member vertex slot
  int* meslot = nullptr;         // member frame slot
  double* mrest = nullptr;       // 17 per member: rc(3) rs rR(9) qR(4)
  double* grest = nullptr;       // 4 per group: rcent(3) denom
  double* warm = nullptr;        // 4 per group: warm rotation (w,x,y,z), persistent
  uint8_t* serial = nullptr;
  int exact = 0;                 // exact-order path (shape.cuh shape_group_exact, VROD_SHAPE_EXACT)
  int* level_off = nullptr;      // host-side only (levels+1)
  int* level_groups = nullptr;   // device: group ids ordered by level
  // chain schedule (host_model.cpp), 0 chains when the frame dependencies are not chains
  int nchains = 0;
  int* chain_off = nullptr;      // nchains+1
  int* chain_groups = nullptr;
};

// Animation packet per substep (host-evaluated, uploaded once per step).
struct AnimLayout {
  int n_pm = 0, n_act = 0, n_bone = 0, n_kin = 0;
  int stride = 0;  // doubles per substep
  int off_time = 0, off_pm = 0, off_act = 0, off_bone = 0, off_kin = 0;
};

struct SweepParams {
  double h, h2, beta;
  int classic;
  int iter;            // iteration index (error word / singular counter)
  int substep;         // substep index within the step (error word)
  int n_pins;
  int elastic_blocks;  // first external block index in the reference's block list
  double contact_kinv;  // inverse_stiffness(settings.contact_stiffness), computed once on the host
  // Programmatic dependent launch inside the iteration loop: 0 off; 1 the kernel waits for its
  // predecessor before touching any state; 2 (rod sweep right after an ext solve) it stages
  // and solves its tile first and waits only before gathering the external contributions.
  int pdl;
  int* scene_singular;    // batch, last iteration only: per-scene singular-block counter
  const double* lam_in;  // elastic multipliers before this sweep (kLamFields x vpad)
  double* lam_out;       // after this sweep (ping-pong partner)
  unsigned long long* dbg = nullptr;  // debug trace (persistent kernel, VROD_TRACE=1)
  int prefetch_rods = 0;  // warp-per-rod sweep: L2 prefetch distance in rods (0: none)
};

// The persistent small-world iteration kernel (rodsweep.cu k_iterate): the whole iteration
// loop of one substep in one launch.
constexpr int kMaxPersistLevels = 8;
struct PersistParams {
  double* X;               // state at the start of the loop (w.X) and its ping-pong partner
  double* Y;
  double* xrec[2];         // slot records: [0] = w.xrec (written by predict), [1] its partner
  double* lam_ext[2];      // external-block multipliers: [0] = c.ext_lam (zeroed by ext setup)
  unsigned* bar;           // grid-barrier counter (zeroed before each launch)
  unsigned* ext_done;      // aux CTAs' external-block releases (zeroed before each launch)
  int tiles;               // tile CTAs; CTAs tiles .. tiles+n_aux-1 are aux CTAs
  int n_aux;
  int iterations;
  int sm_period;
  int levels;              // shape-matching levels (<= kMaxPersistLevels)
  int has_ext;
  int level_off[kMaxPersistLevels + 1];
  unsigned long long* trace;  // optional phase timestamps (globaltimer ns), see k_iterate
  int trace_cta;              // CTA whose per-warp phases are traced
};
constexpr int kTraceCap = 1024;

// Programmatic dependent launch (sm_90+): the next kernel in the stream may start while this
// one finishes; griddepcontrol.wait blocks until the predecessor grid has completed and its
// writes are visible. Each kernel triggers its dependents only after its own wait, so a
// kernel's pre-wait prologue overlaps only the post-wait tail of its predecessor.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Set by Solver::record_step while it records a step: every launch of the step then carries the
// programmatic-serialization attribute, and every kernel opens with pdl_wait(); pdl_trigger().
extern bool g_pdl;

template <typename... Exp, typename... Act>
inline void launch_kernel(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                          Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

// scan.cu
// Several int-array fills in ONE kernel launch (instead of a memset node each, which would also
// break the programmatic-dependent-launch chain of the step graph). Byte-zero fills of other
// types pass their size in ints.
constexpr int kMaxFills = 12;
struct FillList {
  int n = 0;
  int* ptr[kMaxFills];
  long long count[kMaxFills];
  int value[kMaxFills];
  void add(void* p, long long ints, int v) {
    if (!p || ints <= 0) return;
    ptr[n] = static_cast<int*>(p);
    count[n] = ints;
    value[n] = v;
    ++n;
  }
};
void launch_fill(const FillList& f, cudaStream_t st);
// The broad phase's per-substep resets (launch_broad_resets' list); g_broad_resets_done: the
// next launch_collide skips them (already done by the caller).
void broad_reset_list(const Collide& c, int do_narrow, FillList& f);
void launch_broad_resets(Collide& c, int do_narrow, cudaStream_t st);
extern bool g_broad_resets_done;
extern bool g_pills_built;  // the next launch_collide skips k_build_pills (built by the prediction launch)
void scan_exclusive(const int* in, int* out, long long n_cap, const int* n_dev, int* partials, int parts,
                    cudaStream_t st);
long long scan_partials_needed(long long n);

// integrate.cu
// animate (pin motions, activations) + predict_rod / warm_start_lbs / orientation inertia
// pills (non-null, rods <= 32 vertices only): the prediction launch also builds the rod pills and
// their bounding spheres (the broad-phase resets must have run), see launch_collide's pills_built.
void launch_animate_predict(const World& w, const double* anim, const AnimLayout& al, const int* pm_slot,
                            const int* act_rod_off, const int* act_list, double* act_applied, const int* act_rods,
                            int n_act_rods, const double* gravity_h, double h, int substep, unsigned long long* err,
                            const Collide* pills, cudaStream_t st);
void launch_finalize_from(const World& w, const double* src, double h, double keep, cudaStream_t st);
void launch_copy_state(const World& w, const double* src, double* dst, cudaStream_t st);

// collide.cu
// When set (phase timing, Solver::set_option "phase_timing"), recorded on the stream between the
// broad phase (pair scan) and the narrow phase of launch_collide.
extern cudaEvent_t g_broad_mark;
void launch_collide(const World& w, Collide& c, const double* anim, const AnimLayout& al, int substep,
                    unsigned long long* err, StepAccum* acc, int possible, cudaStream_t st);
// Returns true when the ordering kernel also built the warm-start list and counters (fuse_acc).
bool launch_broad_narrow(Collide& c, int substep, unsigned long long* err, int prefilter, int do_narrow,
                         int split_warm, int store_d, cudaStream_t st, StepAccum* fuse_acc = nullptr,
                         bool prepared = false);
void launch_narrow_only(Collide& c, int split_warm, int store_d, cudaStream_t st);
int order_cap_for(int P);  // Collide::order_smem_cap for a world of P pills
void launch_broad_ordered(Collide& c, unsigned long long* err, cudaStream_t st);
void launch_halfplanes(const World& w, Collide& c, cudaStream_t st);
// standalone fine-grained entry points (vrod_pill_project & co), on device arrays
void launch_pill_project(long long n, const double* x, const double* pills, double* t, double* d,
                         uint8_t* deg, cudaStream_t st);
void launch_deepest(long long n, const double* a, const double* b, int iters, const double* warm, double* alpha,
                    double* beta, double* dist, cudaStream_t st);

// sweep.cu
void launch_ext_setup(const World& w, Collide& c, cudaStream_t st);
void launch_iteration(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp,
                      int* singular_counter, unsigned long long* err, cudaStream_t st);
void launch_ext_solve(const World& w, Collide& c, const double* X, const SweepParams& sp, int* singular_counter,
                      unsigned long long* err, cudaStream_t st);
void launch_rod_sweep(const World& w, Collide& c, const double* X, double* Y, const SweepParams& sp,
                      int* singular_counter, unsigned long long* err, cudaStream_t st);
void launch_residuals(const World& w, const double* X, int classic, double* partials, int parts, double* out8,
                      cudaStream_t st);
void launch_penetration(const World& w, Collide& c, const double* X, StepAccum* acc, cudaStream_t st);
// batch: per-scene residual norms (one CTA per scene) and end-of-substep singular fold-in
void launch_scene_report(const World& w, const double* X, int classic, int* scene_singular, cudaStream_t st);
int report_parts(int V);
// k_report_partial only, and the fused end of a single-scene substep (penetration, residual
// norms from the partials, singular count / error word)
// The substep's report in one launch: residual partials (k_report_partial's partition), max
// penetration (from the slot records xrec when non-null: they must hold X's centers and scales),
// then the last CTA's fixed-order reduction, singular count and error word.
void launch_report_tail(const World& w, Collide& c, const double* X, const double* xrec, int classic, StepAccum* acc,
                        bool do_pen,
                        double* partials, int parts, const int* singular_last, int last, const unsigned long long* err,
                        unsigned* counter, cudaStream_t st);
// get_state's outputs packed contiguously (centers, scales, frames, velocities: 8V + 7E doubles)
void launch_pack_state(const World& w, const double* X, int E, double* out, cudaStream_t st);
// kinetic energy and total volume (out[0], out[1]) in the reference's summation order;
// terms: 4 x V scratch, rod_vol: R scratch; cw / sw: the layout's center / scale weights
void launch_energy(const World& w, const double* X, const double* cw, const double* sw, int classic, double* terms,
                   double* rod_vol, double* out, cudaStream_t st);
// eval_constraint(...).W of every elastic block, 3 doubles each, in block order
void launch_block_residuals(const World& w, const double* X, int classic, double* out, cudaStream_t st);

// rodsweep.cu: persistent iteration loop for small single-scene worlds. persistent_tiles()
// returns the number of co-resident tiles the world needs, or 0 when it does not fit.
int persistent_tiles(const World& w);
int persistent_aux_ctas(const World& w);
void launch_iterate_persistent(const World& w, Collide& c, const Groups& g, const PersistParams& pp, const SweepParams& sp,
                               int* singular_counters, unsigned long long* err, cudaStream_t st);

// skin.cu: rod_pill_transforms of the state X (8 doubles per rod pill: center, scale, wxyz)
void launch_pill_transforms(const World& w, const double* X, double* out, cudaStream_t st);

// shape.cu
void launch_shape_match(const World& w, const Groups& g, double* X, const int* level_off_host, bool pdl, cudaStream_t st,
                        double* fits = nullptr);  // fits: 14 doubles per group (SimilarityFit), or null
void launch_extract_rotation(long long n, const double* B, const double* guess, int max_iterations, double tolerance,
                             double* out, cudaStream_t st);

}  // namespace vdev
