// The product's Solver: vrod::Solver (solver.h:54-115 of the reference) on a B200.
// Owns the device world, replays one CUDA graph per step(), mirrors the reference's queries.
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "host_model.h"
#include "kernels.cuh"

namespace vhost {

struct Report {
  int step = 0, contacts = 0, broad = 0, singular = 0, dof = 0;
  double time = 0.0;
  double residuals[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double max_pen = 0.0;
  // PhaseTimings (solver.h:14-21 of the reference): device time per phase, summed over the
  // substeps, filled when the "phase_timing" option is on (else 0)
  double predict_ms = 0.0, broad_ms = 0.0, narrow_ms = 0.0, solve_ms = 0.0, finalize_ms = 0.0;
  double total_ms = 0.0;
};

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Solver {
 public:
  // batch != nullptr with batch->scenes > 1: `scene` is merge_scenes() of independent scenes
  explicit Solver(const SceneData& scene, const BatchLayout* batch = nullptr);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  Report step();
  std::vector<double> probe_convergence(int iterations);  // iterations x 8
  // Product options (no reference counterpart), include/vrod_capi.h vrod_solver_set_option:
  //  "state_prefetch"        1: every step also packs the state and copies it to pinned host
  //                          memory (a side branch of the step graph), so get_state after a step
  //                          costs no extra synchronisation; 0 (default): get_state copies on demand
  //  "exact_shape_matching"  1: the exact-order shape-matching path (bitwise equal to the
  //                          reference); 0: the latency-tuned one. Default: VROD_SHAPE_EXACT
  //  "phase_timing"          1: step() launches its kernels directly with CUDA events between the
  //                          reference's phases and fills Report::{predict,broad,narrow,solve,
  //                          finalize}_ms; 0 (default): one CUDA graph per step, phases unmeasured
  // Returns false for an unknown name.
  bool set_option(const std::string& name, long long value);

  int rod_count() const { return setup_.R; }
  int total_vertices() const { return setup_.V; }
  int total_elements() const { return setup_.E; }
  int dof_count() const { return 4 * setup_.V + 3 * setup_.E; }
  int step_index() const { return step_index_; }
  double time() const { return time_; }
  int bundle_count() const { return static_cast<int>(setup_.groups.size()); }
  int elastic_blocks() const { return setup_.elastic_blocks; }
  const SceneData& scene() const { return scene_; }

  // global slot order of the C-ABI (compact element numbering)
  void get_state(double* c, double* s, double* q, double* cv, double* sv, double* av);
  void set_state(const double* c, const double* s, const double* q, const double* cv, const double* sv,
                 const double* av);
  void get_rest(double* lengths, double* darb, double* grads, double* laps);
  void set_loads(const double* fd, const uint8_t* fdr, const double* tq, const uint8_t* tqr, const double* sl,
                 const uint8_t* slr);
  void energy(double* ke, double* vol, double* rest_vol);
  void inverse_weights(double* ic, double* is, double* it);
  void weights(double* cw, double* sw, double* tw);  // DofLayout weights (layout.h:25-27)
  long long contacts(long long cap, int* a, int* b, double* alpha, double* beta);
  std::vector<PillData> current_pills();
  // Solver::pill_transforms() (solver.cpp:438-440): rod pills, 8 doubles each (center, scale,
  // frame wxyz); the device variant writes into a device buffer on the solver's stream.
  std::vector<double> pill_transforms();
  // One apply_shape_match pass over every bundle group in group order (bundling.cpp:116-133) on
  // the live state; 14 doubles per group (SimilarityFit: scale, translation, rotation, degenerate).
  std::vector<double> shape_match();
  // jacobi_sweep (constraints.cpp:491-556) of the elastic blocks and soft pins, multipliers zero,
  // on the live state (contacts / half-planes excluded); returns {active, skipped_singular}.
  std::pair<int, int> jacobi_sweep(double h, double beta);
  // eval_constraint(...).W of every elastic block in block order, 3 doubles each.
  std::vector<double> elastic_residuals();
  void pill_transforms_device(double* d_out);
  // Per-scene reports of the last step (batch; a single scene returns one entry == step()).
  int scene_count() const { return n_scenes_; }
  std::vector<Report> scene_reports() const;

  // ---- bench / profiling (include/vrod_bench.h) ----
  enum Category { CAT_PREDICT = 0, CAT_COLLIDE, CAT_EXT_SETUP, CAT_EXT_SOLVE, CAT_ROD_SWEEP, CAT_SHAPE, CAT_REPORT,
                  CAT_ITERATE, kCategories };
  // steps graph replays, each bracketed by CUDA events on the solver stream; an L2-flushing
  // memset of flush_bytes runs (untimed) before every step. Returns summed device ms.
  double bench_run(int steps, long long flush_bytes);
  // steps direct-launched steps with event pairs around each kernel category.
  void kernel_times(int steps, double* ms, long long* launches);
  long long kernel_nodes_per_step();
  int contact_count_last();

  // diagnostics for bench.py
  long long last_max_candidates() const { return last_max_cand_; }
  long long last_max_contacts() const { return last_max_ct_; }
  cudaStream_t stream() const { return stream_; }
  int kernels_per_step() const { return kernels_per_step_; }
  void set_graphs(bool on) { use_graph_ = on; }

 private:
  struct Prof {
    std::vector<int> cat;
    std::vector<cudaEvent_t> ev;  // pairs
    std::vector<int> launches;
    std::vector<cudaEvent_t> broad_end;  // per CAT_COLLIDE bracket: end of the broad phase
  };
  bool phase_timing_ = false;
  void upload_static();
  void fill_animation(int substeps, double h);
  void record_step(double h, int substeps, int iterations, double* probe_log, Prof* prof = nullptr);
  void ensure_graph();
  void finish_step(double h, int substeps, Report* out);
  void phase_times(Prof& prof, Report* r);
  void* flush_buf_ = nullptr;
  long long flush_bytes_ = 0;
  void check_error();
  void download_state_cache();

  SceneData scene_;
  Setup setup_;
  bool classic_ = false;
  bool collide_possible_ = false;
  bool ext_possible_ = false;
  double time_ = 0.0;
  int step_index_ = 0;
  int kernels_per_step_ = 0;
  bool use_graph_ = true;
  // programmatic dependent launch in the iteration loop (VROD_PDL=0 disables, for A/B runs)
  bool pdl_ = !(std::getenv("VROD_PDL") && std::getenv("VROD_PDL")[0] == '0');
  // Persistent iteration kernel for small single-scene worlds (VROD_PERSIST=0 disables it).
  bool persist_ok_ = !(std::getenv("VROD_PERSIST") && std::getenv("VROD_PERSIST")[0] == '0');
  int persist_tiles_ = 0;
  int persist_aux_ = 0;              // aux CTAs of the persistent kernel (VROD_PERSIST_AUX=1)
  double* xrec2_ = nullptr;          // ping-pong partner of w_.xrec (persistent kernel)
  double* ext_lam2_ = nullptr;       // ping-pong partner of c_.ext_lam
  unsigned* d_bar_ = nullptr;        // grid-barrier counter
  double* d_ptrans_ = nullptr;       // pill transforms download buffer (lazy)
  double* d_fits_ = nullptr;         // shape_match() fit records (lazy)
  double* d_blockw_ = nullptr;       // elastic_residuals() output (lazy)
  double* d_energy_ = nullptr;
  unsigned* d_tail_counter_ = nullptr;  // k_report_tail's last-CTA ticket       // energy(): terms 4V, cw V, sw V, rod volumes R, out 2 (lazy)
  unsigned long long* d_trace_ = nullptr;  // VROD_TRACE=1: persistent-kernel phase timestamps
 public:
  int trace(long long* out, int cap);
 private:

  cudaStream_t stream_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  std::vector<void*> allocs_;
  template <typename T>
  T* dalloc(std::size_t n);

  vdev::World w_;
  vdev::Collide c_;
  vdev::Groups g_;
  vdev::AnimLayout al_;
  std::vector<int> level_off_;
  std::vector<double> cw_, sw_;          // layout weights (host copies)
  double* d_anim_ = nullptr;
  double* h_anim_ = nullptr;             // pinned
  int* d_pm_slot_ = nullptr;
  int* d_act_rod_off_ = nullptr;
  int* d_act_list_ = nullptr;
  int* d_act_rods_ = nullptr;
  double* d_act_applied_ = nullptr;      // applied amounts + static (factor, first, last)
  int n_act_rods_ = 0;
  vdev::StepAccum* d_acc_ = nullptr;
  vdev::StepAccum* h_acc_ = nullptr;     // pinned
  int* d_singular_ = nullptr;            // per iteration
  unsigned long long* d_err_ = nullptr;
  double* d_report_partials_ = nullptr;
  int report_parts_ = 0;
  double* d_probe_ = nullptr;
  long long last_max_cand_ = 0, last_max_ct_ = 0;
  // batch of scenes
  int n_scenes_ = 1;
  BatchLayout batch_;
  int* d_scene_sing_ = nullptr;
  vdev::SceneAcc* h_scene_acc_ = nullptr;  // pinned, n_scenes_ (batch only)
  Report last_report_;
  // get_state: the outputs packed on the device and copied into a pinned buffer. With the
  // "state_prefetch" option on, step() enqueues that pack + copy behind the step (one
  // synchronisation for both); any other state-changing call invalidates the copy.
  double* d_pack_ = nullptr;
  double* h_pack_ = nullptr;
  bool prefetch_state_ = false, pack_fresh_ = false;
  // with graphs: the pack + copy is a side branch of the step graph, forked after the last
  // finalize, so the copy overlaps the report kernels
  bool pack_in_graph_ = false;
  cudaStream_t side_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  void enqueue_pack(cudaStream_t st);
};

void check_cuda(cudaError_t e, const char* what);

}  // namespace vhost
