// compare_main.cpp -- the adapter against the reference, both called through
// the reference's own API: tempo::solve / runtime::run_parallel (the compiled
// reference sources, oracle/_ref) and tempo::solve_b200 /
// runtime::run_parallel_b200 (this repository's GPU library) on the same
// Hierarchy and SolverConfig.  Prints one JSON line per case:
// iterations of both, the largest relative history difference and the
// relative l2 difference of the final level-0 state.
//
//   compare_b200 [case ...]    cases: config1 config1_p4 functional_norm2 fas_vcycle
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "solve_b200.hpp"
#include "tempo/hierarchy.hpp"

using namespace tempo;

namespace {

// Heat1D with an initial-condition override (Heat1D is final, sin(pi x) IC)
class HeatIC final : public Application {
public:
    HeatIC(problems::Heat1D::Options o, std::vector<double> ic) : inner_(o), ic_(std::move(ic)) {}
    int vector_size() const override { return inner_.vector_size(); }
    StateVector initial_condition() const override {
        return ic_.empty() ? inner_.initial_condition() : StateVector(ic_);
    }
    StateVector step(int l, int i, const StateVector& u) const override { return inner_.step(l, i, u); }
    StateVector forcing(int l, int i) const override { return inner_.forcing(l, i); }
    bool forcing_folded() const override { return inner_.forcing_folded(); }

protected:
    void on_configure() override { inner_.configure(levels_); }

private:
    problems::Heat1D inner_;
    std::vector<double> ic_;
};

std::vector<double> random_state(std::uint64_t seed, int n) {
    const StateVector v = tempo::random_state(seed, static_cast<std::size_t>(n));
    return v.raw();
}

struct Case {
    Heat1DB200 heat;
    Hierarchy hier;
    SolverConfig cfg;
    int workers = 1;
    FunctionalB200 functional;
};

Case make(const std::string& name) {
    if (name == "config1" || name == "config1_p4" || name == "functional_norm2") {
        // BASELINE config 1 (SURVEY 8(d) pins): n = 63, N_t = 1024, m = 16,
        // k = 2, FCF, u0 = sin(pi x) + 0.1 random_state(1, 63), guess seed 20
        problems::Heat1D::Options o;
        o.n_dof = 63;
        o.manufactured_forcing = false;
        std::vector<double> ic = random_state(1, 63);
        const double h = 1.0 / 64.0;
        for (int i = 0; i < 63; ++i) ic[static_cast<size_t>(i)] = std::sin(M_PI * h * (i + 1)) + 0.1 * ic[static_cast<size_t>(i)];
        SolverConfig cfg;
        cfg.relaxation = Relaxation::FCF;
        cfg.tol = 1e-10;
        cfg.max_iters = 100;
        cfg.initial_guess = InitialGuess::Random;
        cfg.seed = 20;
        Case c{{o, ic}, build_hierarchy(TimeGrid::make(0.0, 1.0, 1025), {16}, 2), cfg, 1, {}};
        if (name == "config1_p4") c.workers = 4;
        if (name == "functional_norm2") {
            c.cfg.norm = NormKind::FunctionalChange;
            c.cfg.functional = [](const StateVector& u) { return u.norm2(); };
            c.cfg.tol = 1e-9;
        }
        return c;
    }
    if (name == "fas_vcycle") {
        // folded manufactured forcing, three-level FAS V-cycle, coarse sub-steps
        problems::Heat1D::Options o;
        o.n_dof = 47;
        o.folded = true;
        SolverConfig cfg;
        cfg.mode = CycleMode::VCycle;
        cfg.tol = 1e-9;
        cfg.max_iters = 40;
        cfg.initial_guess = InitialGuess::Random;
        cfg.seed = 5;
        cfg.coarse_substeps = 2;
        return Case{{o, {}}, build_hierarchy(TimeGrid::make(0.0, 2.0, 257), {4, 4}, 4), cfg, 3, {}};
    }
    throw ConfigError("unknown case " + name);
}

void compare(const std::string& name) {
    Case c = make(name);
    HeatIC app(c.heat.opt, c.heat.ic);
    SolveResult ref, gpu;
    if (c.workers == 1) {
        ref = solve(app, c.hier, c.cfg);
        gpu = solve_b200(c.heat, c.hier, c.cfg, {}, &c.functional);
    } else {
        runtime::ParallelOptions po;
        po.workers = c.workers;
        ref = runtime::run_parallel(app, c.hier, c.cfg, po);
        gpu = runtime::run_parallel_b200(c.heat, c.hier, c.cfg, po, &c.functional);
    }
    // history agreement, scaled like tests/test_gpu_parity.py: residual
    // norms relative to themselves or to the first norm (tails sit near the
    // rounding floor).  FunctionalChange values are relative changes
    // |J(u) - J_prev| / |J_prev| (solver.cpp:380-396): two states that agree
    // to ~1e-15 give values that agree to ~1e-15 ABSOLUTELY, so they are
    // compared relative to themselves with an absolute floor of 1e-7 (i.e.
    // |a - b| <= 1e-6 |a| + 1e-13 under the test's 1e-6 bar)
    double hist = 0.0;
    const size_t nh = std::min(ref.report.residual_norms.size(), gpu.report.residual_norms.size());
    const double a0 = nh ? std::fabs(ref.report.residual_norms[0]) : 1.0;
    const bool fc = c.cfg.norm == NormKind::FunctionalChange;
    for (size_t i = 0; i < nh; ++i) {
        const double a = ref.report.residual_norms[i], b = gpu.report.residual_norms[i];
        const double d = std::fabs(a - b);
        const double rel = d / std::max(std::fabs(a), 1e-300);
        hist = std::max(hist, fc ? d / std::max(std::fabs(a), 1e-7) : std::min(rel, d / a0));
    }
    double num = 0.0, den = 0.0;
    const auto& ur = ref.state.level(0).u;
    const auto& ug = gpu.state.level(0).u;
    const bool same_shape = ur.size() == ug.size();
    for (size_t i = 0; same_shape && i < ur.size(); ++i)
        for (size_t q = 0; q < ur[i].size(); ++q) {
            const double d = ur[i][q] - ug[i][q];
            num += d * d;
            den += ur[i][q] * ur[i][q];
        }
    // the coarse levels' working arrays, where the device holds them
    // (nonzero): relative l2 against the reference's
    std::string coarse;
    for (int l = 0; l < c.hier.n_levels(); ++l) {
        const LevelState& lr = ref.state.level(l);
        const LevelState& lg = gpu.state.level(l);
        const std::vector<StateVector>* rs[4] = {&lr.u, &lr.g, &lr.v, &lr.r};
        const std::vector<StateVector>* gs[4] = {&lg.u, &lg.g, &lg.v, &lg.r};
        const char* nm[4] = {"u", "g", "v", "r"};
        for (int w = 0; w < 4; ++w) {
            if (rs[w]->size() != gs[w]->size() || (l == 0 && w == 0)) continue;
            double dn = 0.0, rn = 0.0, gn = 0.0;
            for (size_t i = 0; i < rs[w]->size(); ++i)
                for (size_t q = 0; q < (*rs[w])[i].size() && q < (*gs[w])[i].size(); ++q) {
                    const double a = (*rs[w])[i][q], b = (*gs[w])[i][q];
                    dn += (a - b) * (a - b);
                    rn += a * a;
                    gn += b * b;
                }
            if (gn == 0.0) continue;  // not held by the device
            char buf[96];
            std::snprintf(buf, sizeof(buf), "%s\"%s%d\": %.3e", coarse.empty() ? "" : ", ", nm[w], l,
                          rn > 0 ? std::sqrt(dn / rn) : std::sqrt(dn));
            coarse += buf;
        }
    }
    std::printf("{\"coarse_rel_l2\": {%s}}\n", coarse.c_str());
    std::printf("{\"case\": \"%s\", \"workers\": %d, \"ref_iterations\": %d, \"b200_iterations\": %d, "
                "\"ref_converged\": %s, \"b200_converged\": %s, \"history_max_rel\": %.3e, "
                "\"state_rel_l2\": %.3e, \"same_shape\": %s, \"b200_timings\": %zu, "
                "\"b200_iteration_seconds\": %zu}\n",
                name.c_str(), c.workers, ref.report.iterations, gpu.report.iterations,
                ref.report.converged ? "true" : "false", gpu.report.converged ? "true" : "false", hist,
                same_shape && den > 0 ? std::sqrt(num / den) : -1.0, same_shape ? "true" : "false",
                gpu.report.timings.size(), gpu.report.iteration_seconds.size());
}

}  // namespace

int main(int argc, char** argv) {
    std::vector<std::string> cases;
    for (int i = 1; i < argc; ++i) cases.push_back(argv[i]);
    if (cases.empty()) cases = {"config1", "config1_p4", "functional_norm2", "fas_vcycle"};
    try {
        for (const auto& c : cases) compare(c);
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 3;
    }
    return 0;
}
