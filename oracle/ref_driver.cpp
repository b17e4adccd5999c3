// ref_driver.cpp -- command-line driver around the UNMODIFIED reference
// library (`tempo`, /root/reference/proj/src/*.cpp compiled in place by
// oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY: used to generate golden fixtures
// (tests/golden/make_golden.py) and as the timed CPU reference arm
// (bench.py --impl reference).  It only calls the reference's public API:
// Application, build_hierarchy, SolverConfig, solve(), runtime::run_parallel().
//
// Problems the reference ships (heat1d, dahlquist) use its own Phi.  BASELINE
// configs 2-4 (2D heat with CG, Allen-Cahn with Newton) and Gray-Scott (whose
// reference Phi needs Eigen, absent) have no compilable reference Phi: for
// them `OracleApp` is an Application whose step()/forcing() call the C
// restatement's Phi (atm_oracle.c), so the reference's own CycleDriver /
// run_parallel drives the cycles -- pinning the cycle logic of those configs
// to the reference, with the Phi restated.
//
// Usage: tempo_ref key=value ...   (keys read in run()); prints one JSON line.

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "tempo/application.hpp"
#include "tempo/errors.hpp"
#include "tempo/hierarchy.hpp"
#include "tempo/problems/dahlquist.hpp"
#include "tempo/problems/heat1d.hpp"
#include "tempo/runtime/parallel.hpp"
#include "tempo/solver.hpp"

#include "atm_oracle.h"

using namespace tempo;

namespace {

std::map<std::string, std::string> g_kv;
int g_last_iter = 0;

std::string get(const std::string& k, const std::string& dflt) {
    auto it = g_kv.find(k);
    return it == g_kv.end() ? dflt : it->second;
}
double getd(const std::string& k, double d) {
    auto it = g_kv.find(k);
    return it == g_kv.end() ? d : std::stod(it->second);
}
int geti(const std::string& k, int d) {
    auto it = g_kv.find(k);
    return it == g_kv.end() ? d : std::stoi(it->second);
}

std::vector<double> read_bin(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw ConfigError("cannot open " + path);
    f.seekg(0, std::ios::end);
    const std::size_t bytes = static_cast<std::size_t>(f.tellg());
    f.seekg(0);
    std::vector<double> v(bytes / sizeof(double));
    f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(bytes));
    return v;
}

std::vector<int> int_list(const std::string& s) {
    std::vector<int> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) out.push_back(std::stoi(tok));
    return out;
}

std::vector<double> dbl_list(const std::string& s) {
    std::vector<double> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) out.push_back(std::stod(tok));
    return out;
}

/// Heat1D with an initial-condition override (configs 1 and 5 of
/// BASELINE.json); Heat1D itself is final with a hard-wired sin IC.
class HeatWithIC final : public Application {
public:
    HeatWithIC(problems::Heat1D::Options opt, std::vector<double> ic)
        : inner_(opt), ic_(std::move(ic)) {}
    int vector_size() const override { return inner_.vector_size(); }
    StateVector initial_condition() const override {
        return ic_.empty() ? inner_.initial_condition() : StateVector(ic_);
    }
    StateVector step(int level, int index, const StateVector& u) const override {
        return inner_.step(level, index, u);
    }
    StateVector forcing(int level, int index) const override {
        return inner_.forcing(level, index);
    }
    bool forcing_folded() const override { return inner_.forcing_folded(); }

protected:
    void on_configure() override { inner_.configure(levels_); }

private:
    problems::Heat1D inner_;
    std::vector<double> ic_;
};

/// Scalar linear fixture written from the definition in tests/support.hpp
/// (that header needs Eigen, absent here).
class ScalarFixture final : public Application {
public:
    ScalarFixture(std::vector<double> mult, double u0, bool folded, std::vector<double> ff)
        : mult_(std::move(mult)), u0_(u0), folded_(folded), ff_(std::move(ff)) {}
    int vector_size() const override { return 1; }
    StateVector initial_condition() const override { return StateVector(1, u0_); }
    StateVector step(int level, int index, const StateVector& u) const override {
        StateVector v(1);
        v[0] = mult_.at(static_cast<std::size_t>(level)) * u[0];
        if (folded_ && level == 0 && !ff_.empty()) v[0] += ff_.at(static_cast<std::size_t>(index));
        return v;
    }
    StateVector forcing(int level, int index) const override {
        StateVector v(1);
        v[0] = (!folded_ && level == 0 && !ff_.empty()) ? ff_.at(static_cast<std::size_t>(index)) : 0.0;
        return v;
    }
    bool forcing_folded() const override { return folded_; }

private:
    std::vector<double> mult_;
    double u0_;
    bool folded_;
    std::vector<double> ff_;
};

/// Application over the C restatement's Phi (atm_oracle.c: ac_step, h2_solve,
/// gs_step).  The restated Phi keeps scratch in its orc_driver, so concurrent
/// step() calls (application.hpp:31-32; run_parallel's worker threads) each
/// borrow a driver from a pool.  orc_create allocates no level arrays (those
/// come with orc_setup, never called here), so a driver is a few n-vectors.
class OracleApp final : public Application {
public:
    OracleApp(const orc_problem& p, const orc_grid& g, const orc_solver& s)
        : p_(p), g_(g), s_(s) {
        orc_driver* d = make();
        n_ = orc_vector_size(d);
        ic_.resize(static_cast<std::size_t>(n_));
        orc_initial_condition(d, ic_.data());
        folded_ = p.kind == ORC_ALLEN_CAHN || p.kind == ORC_GRAY_SCOTT || p.folded != 0;
        pool_.push_back(d);
    }
    ~OracleApp() override {
        for (orc_driver* d : pool_) orc_destroy(d);
    }
    int vector_size() const override { return n_; }
    StateVector initial_condition() const override { return StateVector(ic_); }
    StateVector step(int level, int index, const StateVector& u) const override {
        std::vector<double> out(static_cast<std::size_t>(n_));
        run(level, [&](orc_driver* d) { return orc_step(d, level, index, u.raw().data(), out.data()); });
        return StateVector(std::move(out));
    }
    StateVector forcing(int level, int index) const override {
        std::vector<double> out(static_cast<std::size_t>(n_));
        run(level, [&](orc_driver* d) { return orc_forcing(d, level, index, out.data()); });
        return StateVector(std::move(out));
    }
    bool forcing_folded() const override { return folded_; }

protected:
    // the restated Phi derives its per-level dt from the same grid rule
    // (hierarchy.cpp:42 / solver.cpp:30-43); refuse to run if they disagree
    void on_configure() override {
        for (int l = 0; l < n_levels(); ++l) {
            const int sub = l == n_levels() - 1 ? s_.coarse_substeps : 1;
            if (level(l).dt != orc_level_dt(&g_, l) || level(l).substeps != sub ||
                level(l).n_points != orc_level_points(&g_, l))
                throw ConfigError("OracleApp: level " + std::to_string(l) +
                                  " spec differs from the restated grid");
        }
    }

private:
    orc_driver* make() const {
        int st = 0;
        orc_driver* d = orc_create(&p_, &g_, &s_, &st);
        if (!d) throw ConfigError(std::string("oracle problem: ") + orc_create_error());
        return d;
    }
    template <class F>
    void run(int level, F&& f) const {
        (void)level;
        orc_driver* d = nullptr;
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (!pool_.empty()) {
                d = pool_.back();
                pool_.pop_back();
            }
        }
        if (!d) d = make();
        const int st = f(d);
        std::string err = st ? orc_error(d) : "";
        {
            std::lock_guard<std::mutex> lk(mu_);
            pool_.push_back(d);
        }
        if (st == ORC_NONLINEAR) throw NonlinearSolveError(err);
        if (st) throw ConfigError(err);
    }

    orc_problem p_;
    orc_grid g_;
    orc_solver s_;
    int n_ = 0;
    bool folded_ = false;
    std::vector<double> ic_;
    mutable std::mutex mu_;
    mutable std::vector<orc_driver*> pool_;
};

void write_json(const ConvergenceReport& rep, double seconds, int workers,
                const std::string& extra) {
    std::printf("{\"iterations\": %d, \"converged\": %s, \"seconds\": %.9g, \"workers\": %d",
                rep.iterations, rep.converged ? "true" : "false", seconds, workers);
    std::printf(", \"history\": [");
    for (std::size_t i = 0; i < rep.residual_norms.size(); ++i)
        std::printf("%s%.17g", i ? ", " : "", rep.residual_norms[i]);
    std::printf("], \"iteration_seconds\": [");
    for (std::size_t i = 0; i < rep.iteration_seconds.size(); ++i)
        std::printf("%s%.9g", i ? ", " : "", rep.iteration_seconds[i]);
    std::printf("], \"timings\": {");
    bool first = true;
    for (const auto& [k, v] : rep.timings) {
        std::printf("%s\"%s\": %.9g", first ? "" : ", ", k.c_str(), v);
        first = false;
    }
    std::printf("}%s}\n", extra.c_str());
}

int run() {
    const std::string problem = get("problem", "heat1d");
    std::unique_ptr<Application> app;
    int n = 1;
    if (problem == "heat1d") {
        problems::Heat1D::Options opt;
        opt.n_dof = geti("n", 1025);
        opt.x0 = getd("x0", 0.0);
        opt.x1 = getd("x1", 1.0);
        opt.folded = geti("folded", 0) != 0;
        opt.manufactured_forcing = geti("manufactured", 1) != 0;
        std::vector<double> ic;
        if (!get("ic_file", "").empty()) ic = read_bin(get("ic_file", ""));
        app = std::make_unique<HeatWithIC>(opt, ic);
        n = opt.n_dof;
    } else if (problem == "dahlquist") {
        app = std::make_unique<problems::Dahlquist>(getd("lambda", -1.0), getd("u0", 1.0),
                                                    geti("folded", 0) != 0);
    } else if (problem == "scalar") {
        std::vector<double> ff;
        if (!get("ff_file", "").empty()) ff = read_bin(get("ff_file", ""));
        app = std::make_unique<ScalarFixture>(dbl_list(get("mult", "0.5,0.25")),
                                              getd("u0", 1.0), geti("folded", 0) != 0, ff);
    } else if (problem == "allen_cahn" || problem == "heat2d" || problem == "gray_scott") {
        orc_problem p{};
        p.kind = problem == "allen_cahn" ? ORC_ALLEN_CAHN : problem == "heat2d" ? ORC_HEAT2D
                                                                               : ORC_GRAY_SCOTT;
        p.n = geti("n", 0);
        p.folded = geti("folded", 1);
        p.eps = getd("eps", 0.02);
        p.length = getd("length", 1.0);
        p.newton_tol = getd("newton_tol", p.kind == ORC_GRAY_SCOTT ? 1e-10 : 1e-12);
        p.newton_max = geti("newton_max", 30);
        p.nx = geti("nx", 0);
        p.cg_rtol = getd("cg_rtol", 1e-12);
        p.cg_max = geti("cg_max", 10000);
        // gray_scott.hpp:24-38 defaults
        p.gs_domain = getd("domain", 2.5);
        p.gs_feed = getd("feed", 0.024);
        p.gs_kill = getd("kill", 0.06);
        p.gs_du = getd("du", 8e-5);
        p.gs_dv = getd("dv", 4e-5);
        p.gs_linear_tol = getd("linear_tol", 1e-10);
        p.gs_reaction = geti("reaction", 1);
        p.gs_bounds_check = geti("bounds_check", 1);
        p.gs_bound_lo = getd("bound_lo", -1.0);
        p.gs_bound_hi = getd("bound_hi", 3.0);
        static std::vector<double> src, ic;
        if (!get("source_file", "").empty()) src = read_bin(get("source_file", ""));
        if (!get("ic_file", "").empty()) ic = read_bin(get("ic_file", ""));
        p.source = src.empty() ? nullptr : src.data();
        p.ic = ic.empty() ? nullptr : ic.data();
        orc_grid g{};
        g.t0 = getd("t0", 0.0);
        g.tf = getd("tf", 1.0);
        g.n_points = geti("n_points", 33);
        const std::vector<int> ms = int_list(get("m", "4"));
        g.n_m = static_cast<int>(ms.size());
        for (std::size_t i = 0; i < ms.size() && i < ORC_MAXL; ++i) g.m[i] = ms[i];
        g.k = geti("k", 2);
        orc_solver so{};
        so.mode = get("mode", "two-level") == "two-level" ? ORC_TWO_LEVEL : ORC_VCYCLE;
        so.tol = 1.0;
        so.max_iters = 1;
        so.nu = 1;
        so.coarse_substeps = geti("substeps", 1);
        auto oapp = std::make_unique<OracleApp>(p, g, so);
        n = oapp->vector_size();
        app = std::move(oapp);
    } else {
        throw ConfigError("unknown problem " + problem);
    }

    const TimeGrid grid = TimeGrid::make(getd("t0", 0.0), getd("tf", 1.0), geti("n_points", 33));
    const Hierarchy hier = build_hierarchy(grid, int_list(get("m", "4")), geti("k", 2));

    SolverConfig cfg;
    const std::string mode = get("mode", "two-level");
    cfg.mode = mode == "two-level" ? CycleMode::TwoLevel
             : mode == "v-cycle"   ? CycleMode::VCycle : CycleMode::NestedV;
    cfg.relaxation = get("relax", "F") == "FCF" ? Relaxation::FCF : Relaxation::F;
    cfg.nu = geti("nu", 1);
    cfg.max_iters = geti("max_iters", 100);
    cfg.tol = getd("tol", 1e-7);
    const std::string guess = get("guess", "constant");
    cfg.initial_guess = guess == "random" ? InitialGuess::Random
                      : guess == "provided" ? InitialGuess::Provided : InitialGuess::Constant;
    cfg.seed = static_cast<std::uint64_t>(std::stoull(get("seed", "0")));
    cfg.coarse_substeps = geti("substeps", 1);
    if (guess == "provided") {
        const std::vector<double> flat = read_bin(get("guess_file", ""));
        for (int i = 0; i < grid.n_points; ++i)
            cfg.provided.emplace_back(std::vector<double>(flat.begin() + static_cast<long>(i) * n,
                                                          flat.begin() + static_cast<long>(i + 1) * n));
    }
    if (get("norm", "l2") == "functional") {
        // functional=first: u[0]; norm2: u.norm2() (the reference CLI's,
        // run_config.cpp:241-243); weights: w.u in index order (w_file)
        cfg.norm = NormKind::FunctionalChange;
        const std::string fk = get("functional", "first");
        if (fk == "norm2") {
            cfg.functional = [](const StateVector& u) { return u.norm2(); };
        } else if (fk == "weights") {
            static std::vector<double> w;
            w = read_bin(get("w_file", ""));
            cfg.functional = [](const StateVector& u) {
                double s = 0.0;
                for (std::size_t q = 0; q < u.size(); ++q) s += w[q] * u[q];
                return s;
            };
        } else {
            cfg.functional = [](const StateVector& u) { return u[0]; };
        }
    }
    // fixed-iteration timing mode: the CPU reference arm of bench.py
    const int timing_iters = geti("timing_iters", 0);
    if (timing_iters > 0) {
        cfg.tol = 1e-300;
        cfg.max_iters = timing_iters;
    }

    int workers = geti("workers", 1);
    if (workers <= 0) workers = static_cast<int>(std::thread::hardware_concurrency());
    if (workers > hier.n_coarsest_points()) workers = hier.n_coarsest_points();

    const auto t0 = std::chrono::steady_clock::now();
    SolveResult result;
    // the highest iteration any phase finished (or unwound) in: on a failure
    // this names the failing cycle (PhaseTimer records during unwinding)
    std::mutex trace_mu;
    TraceSink trace = [&](int iter, int, const std::string&, double) {
        std::lock_guard<std::mutex> lk(trace_mu);
        if (iter > g_last_iter) g_last_iter = iter;
    };
    if (get("driver", "solve") == "solve" && workers == 1) {
        result = solve(*app, hier, cfg, trace);
    } else {
        runtime::ParallelOptions popt;
        popt.workers = workers;
        popt.timeout = std::chrono::milliseconds(geti("timeout_ms", 3600000));
        popt.trace = trace;
        result = runtime::run_parallel(*app, hier, cfg, popt);
    }
    const double seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    const std::string out_u = get("out_u", "");
    if (!out_u.empty()) {
        std::ofstream f(out_u, std::ios::binary);
        for (const StateVector& s : result.state.level(0).u)
            f.write(reinterpret_cast<const char*>(s.raw().data()),
                    static_cast<std::streamsize>(s.size() * sizeof(double)));
    }
    write_json(result.report, seconds, workers, "");
    return result.report.converged ? 0 : 1;
}

} // namespace

int main(int argc, char** argv) {
    for (int i = 1; i < argc; ++i) {
        const char* eq = std::strchr(argv[i], '=');
        if (!eq) continue;
        g_kv[std::string(argv[i], static_cast<std::size_t>(eq - argv[i]))] = std::string(eq + 1);
    }
    try {
        return run();
    } catch (const DivergenceError& e) {
        std::printf("{\"error\": \"diverged\", \"iteration\": %d, \"what\": \"%s\"}\n",
                    e.iteration(), e.what());
        return 3;
    } catch (const NonlinearSolveError& e) {
        std::printf("{\"error\": \"nonlinear\", \"last_iteration\": %d, \"what\": \"%s\"}\n",
                    g_last_iter, e.what());
        return 3;
    } catch (const ConfigError& e) {
        std::printf("{\"error\": \"config\", \"what\": \"%s\"}\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"runtime\", \"last_iteration\": %d, \"what\": \"%s\"}\n",
                    g_last_iter, e.what());
        return 3;
    }
}
