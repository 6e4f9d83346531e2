// Force-included (after oracle/shim/test_solver_prelude.h) when the reference's own
// proj/tests/test_solver.cpp is compiled against the B200 drop-in: the reference's CPU class is
// declared under another name, and `Solver` — which the test file names through
// `using namespace vrod;` — becomes vrod::b200::Solver (include/vrod/b200_solver.h). The test
// source itself is compiled unmodified; every Solver it constructs steps on the GPU.
#pragma once
#define Solver Solver_reference_cpu_
#include "vrod/solver.h"
#undef Solver
#include "vrod/b200_solver.h"
namespace vrod {
using Solver = b200::Solver;
}  // namespace vrod
