// ref_driver.cpp -- command-line driver around the UNMODIFIED reference
// library (`tempo`, /root/reference/proj/src/*.cpp compiled in place by
// oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY: used to generate golden fixtures
// (tests/golden/make_golden.py) and as the timed CPU reference arm
// (bench.py --impl reference).  It only calls the reference's public API:
// Application, build_hierarchy, SolverConfig, solve(), runtime::run_parallel().
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

using namespace tempo;

namespace {

std::map<std::string, std::string> g_kv;

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
        cfg.norm = NormKind::FunctionalChange;
        cfg.functional = [](const StateVector& u) { return u[0]; };
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
    if (get("driver", "solve") == "solve" && workers == 1) {
        result = solve(*app, hier, cfg);
    } else {
        runtime::ParallelOptions popt;
        popt.workers = workers;
        popt.timeout = std::chrono::milliseconds(600000);
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
    } catch (const ConfigError& e) {
        std::printf("{\"error\": \"config\", \"what\": \"%s\"}\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"runtime\", \"what\": \"%s\"}\n", e.what());
        return 3;
    }
}
