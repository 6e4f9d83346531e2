// Harness-side patch for two shipped defects in the reference's tests/test_solver.cpp
// (SURVEY.md §4): it names `RestPose` (the header type is `RodRestPose`, rod.h:30) and
// calls vrod::test helpers unqualified (:30,94,290). Force-included for that one file
// only; the reference source itself is compiled unmodified.
#pragma once
namespace vrod {
struct RodRestPose;
using RestPose = RodRestPose;
namespace test {}
using namespace test;
}  // namespace vrod

// test_solver.cpp:352-353 call make_rest_pose(centers, {0.05}, {}); std::span has no
// initializer_list constructor before C++26, so that line does not compile as C++20
// (a third shipped defect). This overload forwards to the real function unchanged.
#include <initializer_list>
#include <span>
#include "vrod/rod.h"
namespace vrod {
inline RodRestPose make_rest_pose(std::span<const Vec3> centers, std::initializer_list<double> radii,
                                  std::initializer_list<double> scales) {
  return make_rest_pose(centers, std::span<const double>(radii.begin(), radii.size()),
                        std::span<const double>(scales.begin(), scales.size()));
}
}  // namespace vrod
