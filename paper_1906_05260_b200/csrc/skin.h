// Skinning on the device (skinning.h / skinning.cpp): bind_skin, smooth_binding, deform_mesh,
// and the per-frame pill transforms of a solver's live state. SURVEY.md §8(f) rows 2-3: the
// direct consumer of the substep's output (the CLI deforms the bound mesh every frame,
// vrod_main.cpp:52-73).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <vector>

#include "host_model.h"

namespace vhost {

class Solver;

// PillTransform (skinning.h:19-25), device layout: center xyz, scale, rotation wxyz.
constexpr int kTransformDoubles = 8;

class Skin {
 public:
  // bind_skin (skinning.cpp:59-105); validation messages follow the reference's require() calls.
  Skin(const std::vector<V3>& vertices, const std::vector<std::array<int, 3>>& triangles,
       const std::vector<PillData>& rest_pills, const std::vector<double>& rest_transforms /* 8 per pill */,
       int max_influences, double epsilon);
  ~Skin();
  Skin(const Skin&) = delete;
  Skin& operator=(const Skin&) = delete;

  void smooth(int iterations);  // smooth_binding, skinning.cpp:107-163
  // CSR of the binding (any pointer may be null)
  void get_binding(int* offsets, int* pills, double* weights, int* nnz, int* clamped) const;
  // deform_mesh (skinning.cpp:165-185) with host transforms (8 doubles per pill)
  void deform(int pill_count, const double* transforms, double* out);
  // pill transforms of the solver's live state + deform, on the solver's stream; out may be null
  void deform_solver(Solver& solver, double* out);
  int vertex_count() const { return nv_; }
  int pill_count() const { return np_; }
  // device output of the last deformation (3 doubles per vertex) and the bench helpers
  const double* device_out() const { return d_out_; }
  void deform_device(const double* d_transforms, cudaStream_t st);  // no host copies
  // bench: iterations x (pill transforms + deform) on the solver's stream, device-timed
  void bench(Solver& solver, int iterations, double* total_ms, double* deform_ms);

 private:
  int nv_ = 0, np_ = 0, keep_ = 0, max_influences_ = 8, clamped_ = 0;
  long long nnz_ = 0;
  std::vector<int> nb_off_, nb_list_;  // one-ring neighbours (sorted, unique), host CSR
  cudaStream_t stream_ = nullptr;
  double* d_verts_ = nullptr;       // 3 per vertex
  double* d_rest_ = nullptr;        // 8 per pill
  double* d_cur_ = nullptr;         // 8 per pill (host transforms upload)
  double* d_frame_ = nullptr;       // 8 per pill: cur transform with cur.scale / ref.scale
  int* d_off_ = nullptr;            // nv+1
  int* d_pills_ = nullptr;          // nv * keep (CSR packed in front)
  double* d_weights_ = nullptr;
  int* d_cnt_ = nullptr;            // per vertex influence count (smoothing)
  double* d_out_ = nullptr;         // 3 per vertex
  int* d_nb_off_ = nullptr;
  int* d_nb_ = nullptr;
  long long scratch_cap_ = 0;
  int* d_scr_pill_ = nullptr;       // smoothing scratch (pill, weight) per candidate
  double* d_scr_w_ = nullptr;
  long long* d_scr_off_ = nullptr;
  int* d_tmp_pills_ = nullptr;
  double* d_tmp_weights_ = nullptr;
  int* d_scan_tmp_ = nullptr;
  int scan_parts_ = 0;
};

}  // namespace vhost
