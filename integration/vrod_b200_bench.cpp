// cmd_bench on the drop-in (proj/tools/vrod_main.cpp:127-158): the reference CLI's throughput loop,
// with vrod::b200::Solver in place of vrod::Solver, over the reference's builtin scenarios
// (scenarios.cpp:296-306). `--impl both` also steps the reference's CPU solver on the same scene and
// compares every state array after the run (bitwise expected; shape-matching scenes bitwise with
// --exact, i.e. the exact_shape_matching option).
//
//   vrod_b200_bench builtin:<name> [--steps N] [--impl b200|reference|both] [--exact] [--phases]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "vrod/b200_solver.h"
#include "vrod/scenarios.h"

namespace {

using Clock = std::chrono::steady_clock;

vrod::Scene resolve_scene(const std::string& arg) {
  constexpr const char* kPrefix = "builtin:";
  if (arg.rfind(kPrefix, 0) != 0) throw std::invalid_argument("only builtin:<name> scenes (scene JSON is out of scope)");
  return vrod::make_builtin_scenario(arg.substr(std::string(kPrefix).size()));
}

// The loop body of cmd_bench, for either solver type.
template <class S>
int bench_loop(S& solver, int steps, const char* label) {
  vrod::PhaseTimings sum;
  const auto start = Clock::now();
  for (int i = 0; i < steps; ++i) {
    vrod::StepReport report;
    try {
      report = solver.step();
    } catch (const vrod::SimulationError& e) {
      std::fprintf(stderr, "simulation aborted at step %d (t=%.6g s): %s\n", solver.step_index() + 1, solver.time(),
                   e.what());
      return 1;
    }
    sum.predict_ms += report.timings.predict_ms;
    sum.broad_ms += report.timings.broad_ms;
    sum.narrow_ms += report.timings.narrow_ms;
    sum.solve_ms += report.timings.solve_ms;
    sum.finalize_ms += report.timings.finalize_ms;
    sum.total_ms += report.timings.total_ms;
  }
  const double wall_s = std::chrono::duration<double>(Clock::now() - start).count();
  const double n = steps > 0 ? static_cast<double>(steps) : 1.0;
  std::printf("[%s] rods: %zu, DOFs: %d\n", label, solver.scene().rods.size(), solver.dof_count());
  std::printf("[%s] steps: %d in %.3f s -> %.1f steps/s\n", label, steps, wall_s, steps > 0 ? steps / wall_s : 0.0);
  std::printf("[%s] per-step phase (ms): predict %.3f, broad %.3f, narrow %.3f, solve %.3f, finalize %.3f, total %.3f\n",
              label, sum.predict_ms / n, sum.broad_ms / n, sum.narrow_ms / n, sum.solve_ms / n, sum.finalize_ms / n,
              sum.total_ms / n);
  return 0;
}

double max_abs_diff(const vrod::Scene& a, const vrod::Scene& b, long long* mismatches) {
  double worst = 0.0;
  auto cmp = [&](double x, double y) {
    if (std::memcmp(&x, &y, sizeof(double)) != 0) ++*mismatches;
    worst = std::fmax(worst, std::fabs(x - y));
  };
  for (std::size_t r = 0; r < a.rods.size(); ++r) {
    const vrod::RodState& p = a.rods[r].state;
    const vrod::RodState& q = b.rods[r].state;
    for (std::size_t v = 0; v < p.centers.size(); ++v) {
      for (int k = 0; k < 3; ++k) cmp(p.centers[v][k], q.centers[v][k]), cmp(p.center_vel[v][k], q.center_vel[v][k]);
      cmp(p.scales[v], q.scales[v]);
      cmp(p.scale_vel[v], q.scale_vel[v]);
    }
    for (std::size_t e = 0; e < p.frames.size(); ++e) {
      for (int k = 0; k < 4; ++k) cmp(p.frames[e].coeffs()[k], q.frames[e].coeffs()[k]);
      for (int k = 0; k < 3; ++k) cmp(p.angular_vel[e][k], q.angular_vel[e][k]);
    }
  }
  return worst;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s builtin:<name> [--steps N] [--impl b200|reference|both] [--exact] [--phases]\n",
                 argv[0]);
    return 2;
  }
  const std::string scene_arg = argv[1];
  int steps = 100;
  std::string impl = "b200";
  bool exact = false, phases = false;
  for (int i = 2; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--steps") && i + 1 < argc) steps = std::atoi(argv[++i]);
    else if (!std::strcmp(argv[i], "--impl") && i + 1 < argc) impl = argv[++i];
    else if (!std::strcmp(argv[i], "--exact")) exact = true;
    else if (!std::strcmp(argv[i], "--phases")) phases = true;
  }
  try {
    const vrod::Scene scene = resolve_scene(scene_arg);
    int rc = 0;
    vrod::Scene gpu_final, ref_final;
    if (impl == "b200" || impl == "both") {
      vrod::b200::Solver solver(scene);
      if (exact) solver.set_option("exact_shape_matching", 1);
      if (phases) solver.set_option("phase_timing", 1);
      rc |= bench_loop(solver, steps, "b200");
      gpu_final = solver.scene();
    }
    if (impl == "reference" || impl == "both") {
      vrod::Solver solver(scene);
      rc |= bench_loop(solver, steps, "reference");
      ref_final = solver.scene();
    }
    if (impl == "both" && rc == 0) {
      long long mism = 0;
      const double d = max_abs_diff(gpu_final, ref_final, &mism);
      std::printf("parity: %s (state doubles differing: %lld, max |diff| %.3e)\n", mism == 0 ? "bitwise" : "differs",
                  mism, d);
      if (mism != 0 && exact) rc = 1;
    }
    return rc;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
