// solve_b200.cpp -- see solve_b200.hpp.  The adapter INTEGRATION.md shows,
// compiled and tested in-tree.
#include "solve_b200.hpp"

#include <sstream>
#include <string>

#include "atmgrit.h"

namespace tempo {
namespace {

[[noreturn]] void raise(atm_status st, const std::string& msg, int iteration = 0) {
    switch (st) {
        case ATM_CONFIG_ERROR: throw ConfigError(msg);
        case ATM_DIVERGED: throw DivergenceError(iteration, msg);
        case ATM_NONLINEAR_FAIL: throw NonlinearSolveError(msg);
        default: throw RuntimeFault(0, msg);
    }
}

SolveResult run(const Heat1DB200& app, const Hierarchy& hier, const SolverConfig& cfg, int shards,
                int timeout_ms, const TraceSink& trace, const FunctionalB200* functional) {
    atm_problem p{};
    p.kind = ATM_PHI_HEAT1D;
    p.n = app.opt.n_dof;
    p.x0 = app.opt.x0;
    p.x1 = app.opt.x1;
    p.folded = app.opt.folded;
    p.manufactured = app.opt.manufactured_forcing;
    p.ic = app.ic.empty() ? nullptr : app.ic.data();

    atm_grid g{};
    g.t0 = hier.level(0).t0;
    g.tf = hier.level(0).tf;
    g.n_points = hier.level(0).n_points;
    g.n_m = static_cast<int>(hier.coarsening_factors().size());
    for (int l = 0; l < g.n_m; ++l) g.m[l] = hier.coarsening_factors()[static_cast<size_t>(l)];
    g.k = hier.k();

    atm_solver s{};
    s.mode = static_cast<int>(cfg.mode);  // same enumerator order (solver_config.hpp:13-25)
    s.relaxation = static_cast<int>(cfg.relaxation);
    s.nu = cfg.nu;
    s.max_iters = cfg.max_iters;
    s.tol = cfg.tol;
    s.norm = static_cast<int>(cfg.norm);
    if (cfg.norm == NormKind::FunctionalChange) {
        if (!functional)
            throw ConfigError("solve_b200: FunctionalChange needs the functional as a FunctionalB200 "
                              "(u.norm2() or weights)");
        s.functional_kind = functional->kind == FunctionalB200::Norm2 ? ATM_FUNCTIONAL_NORM2
                                                                      : ATM_FUNCTIONAL_LINEAR;
        if (functional->kind == FunctionalB200::Linear) {
            if (static_cast<int>(functional->w.size()) != p.n)
                throw ConfigError("solve_b200: functional weights must have vector_size() entries");
            s.functional_w = functional->w.data();
        }
    }
    s.initial_guess = static_cast<int>(cfg.initial_guess);
    s.seed = cfg.seed;
    s.coarse_substeps = cfg.coarse_substeps;
    std::vector<double> flat;
    if (cfg.initial_guess == InitialGuess::Provided) {
        if (static_cast<int>(cfg.provided.size()) != g.n_points)
            throw ConfigError("provided initial guess has the wrong number of points");
        flat.reserve(static_cast<size_t>(g.n_points) * p.n);
        for (const StateVector& v : cfg.provided) flat.insert(flat.end(), v.raw().begin(), v.raw().end());
        s.provided = flat.data();  // copied by atm_setup (atm_runtime.defer_guess = 0)
    }
    if (cfg.constant_value) s.constant_value = cfg.constant_value->raw().data();

    atm_runtime rt{};
    rt.n_shards = shards;  // time shards of the reference rank layout
    rt.timeout_ms = timeout_ms;
    rt.trace = trace ? 1 : 0;  // per-phase device timings (disables CUDA-graph replay)
    atm_ctx* ctx = nullptr;
    if (atm_status st = atm_create(&p, &g, &s, &rt, &ctx)) raise(st, atm_create_error());

    std::vector<double> norms(static_cast<size_t>(cfg.max_iters)), secs(norms.size());
    atm_report rep{};
    const atm_status st = atm_solve(ctx, &rep, norms.data(), secs.data());
    if (st != ATM_OK && st != ATM_NOT_CONVERGED) {
        const std::string msg = atm_last_error(ctx);
        atm_destroy(ctx);
        raise(st, msg, rep.iterations);
    }
    SolveResult out;
    ConvergenceReport& r = out.report;
    r.residual_norms.assign(norms.begin(), norms.begin() + rep.iterations);
    r.iteration_seconds.assign(secs.begin(), secs.begin() + rep.iterations);
    r.iterations = rep.iterations;
    r.converged = rep.converged != 0;
    r.stop_reason = rep.converged ? StopReason::Converged : StopReason::MaxIterations;
    char names[1024];
    double phase[32];
    const int np_ = atm_phase_times(ctx, names, sizeof(names), phase, 32);
    std::stringstream ss(names);
    std::string name;
    for (int i = 0; i < np_ && std::getline(ss, name, ','); ++i) r.timings[name] = phase[i];
    r.timings["total"] = rep.total_seconds;
    if (trace)
        for (int it = 0; it < rep.iterations; ++it) trace(it + 1, 0, "cycle", secs[static_cast<size_t>(it)]);

    // SpaceTimeState (space_time.hpp:20-32), shaped as CycleDriver::setup
    // sizes it (solver.cpp:84-96): u and g on every level, v and r on the
    // coarse levels.  Level-0 u is the solution; the other arrays are the
    // solver's working state, read back where the device holds them (the
    // linear two-level cycle keeps no coarse u, for instance) and zero
    // otherwise.
    const int n = p.n;
    out.state.levels.resize(static_cast<size_t>(hier.n_levels()));
    for (int l = 0; l < hier.n_levels(); ++l) {
        const int npl = hier.level(l).n_points;
        LevelState& ls = out.state.level(l);
        std::vector<StateVector>* arrs[4] = {&ls.u, &ls.g, &ls.v, &ls.r};  // atm_get_level's `which`
        for (int which = 0; which < 4; ++which) {
            if (which >= 2 && l == 0) continue;
            std::vector<double> buf(static_cast<size_t>(npl) * n, 0.0);
            if (atm_status e = atm_get_level(ctx, l, which, 0, npl, buf.data())) {
                const std::string msg = atm_last_error(ctx);
                atm_destroy(ctx);
                raise(e, msg);
            }
            auto& dst = *arrs[which];
            dst.reserve(static_cast<size_t>(npl));
            for (int i = 0; i < npl; ++i)
                dst.emplace_back(std::vector<double>(buf.begin() + static_cast<long>(i) * n,
                                                     buf.begin() + static_cast<long>(i + 1) * n));
        }
    }
    atm_destroy(ctx);
    return out;
}

}  // namespace

SolveResult solve_b200(const Heat1DB200& app, const Hierarchy& hier, const SolverConfig& cfg,
                       TraceSink trace, const FunctionalB200* functional) {
    return run(app, hier, cfg, 1, 0, trace, functional);
}

namespace runtime {

SolveResult run_parallel_b200(const Heat1DB200& app, const Hierarchy& hier, const SolverConfig& cfg,
                              const ParallelOptions& opt, const FunctionalB200* functional) {
    if (opt.workers < 1) throw ConfigError("run_parallel: need at least one worker");
    return run(app, hier, cfg, opt.workers, static_cast<int>(opt.timeout.count()), opt.trace, functional);
}

}  // namespace runtime
}  // namespace tempo
