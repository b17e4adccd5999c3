// solve_b200.hpp -- the adapter a `tempo` maintainer adds:
// tempo::solve / runtime::run_parallel dispatched to the B200 library through
// its C ABI (include/atmgrit.h).  Callers keep their Hierarchy, SolverConfig
// and SolveResult; the Application travels as a Phi descriptor because the C
// ABI cannot call back into a virtual Application::step per time step (the
// device runs thousands of steps concurrently).
//
// Built in this repository against the reference's own headers
// (/root/reference/proj/include) by tests/integration/Makefile, and checked
// against the reference's CPU solve by tests/test_gpu_integration.py.
#pragma once

#include <vector>

#include "tempo/problems/heat1d.hpp"
#include "tempo/runtime/parallel.hpp"
#include "tempo/solver.hpp"

namespace tempo {

/// problems::Heat1D (heat1d.hpp:20-76) as the B200 Phi descriptor: its
/// Options (not queryable after construction) plus an optional
/// initial-condition override.
struct Heat1DB200 {
    problems::Heat1D::Options opt;
    std::vector<double> ic;
};

/// SolverConfig::functional (solver_config.hpp:43) for NormKind::FunctionalChange:
/// a std::function cannot cross the C ABI, so the functional is named --
/// u.norm2() (the reference CLI's, run_config.cpp:241-243) or w.u.
struct FunctionalB200 {
    enum Kind { Norm2, Linear } kind = Norm2;
    std::vector<double> w;  ///< Linear: weights (vector_size() values)
};

/// solve() (solver.hpp:134-135) on one GPU.  Exceptions as the reference's
/// (errors.hpp:9-42).  trace receives one ("cycle", seconds) record per
/// iteration.
SolveResult solve_b200(const Heat1DB200& app, const Hierarchy& hier, const SolverConfig& cfg,
                       TraceSink trace = {}, const FunctionalB200* functional = nullptr);

namespace runtime {

/// run_parallel() (parallel.hpp:26-27): ParallelOptions::workers time shards
/// (the reference rank layout, layout.cpp:29-63) on one GPU; timeout applies
/// to multi-process runs (atm_runtime.timeout_ms).
SolveResult run_parallel_b200(const Heat1DB200& app, const Hierarchy& hier, const SolverConfig& cfg,
                              const ParallelOptions& opt, const FunctionalB200* functional = nullptr);

}  // namespace runtime
}  // namespace tempo
