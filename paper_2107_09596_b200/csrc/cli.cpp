// cli.cpp -- `tempo_b200`: the reference's flat-config front end driving the
// GPU path through the C ABI.
//
// Restates the behaviour of the reference CLI (src/run_config.cpp:295-413,
// include/tempo/cli.hpp:12-64): one `key = value` per line, '#' comments,
// duplicate / unknown keys are ConfigErrors; `solve` writes
// `iter,residual_norm,seconds` rows plus a `converged,iterations,
// total_seconds` summary, `sweep-k` writes `m,k,k_over_ncpoints,iterations,
// parareal_equivalent` rows (k = 0 selects the full coarse grid).  Exit codes
// 0 converged / 1 not converged / 2 config error / 3 runtime fault.
// Problems: dahlquist, heat1d, grayscott (the reference's) plus allencahn,
// heat2d (the BASELINE configs 2-4 families).
//
//   tempo_b200 solve CONFIG [--out PATH] [--workers N]
//   tempo_b200 sweep-k CONFIG [--out PATH] [--workers N]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "atmgrit.h"

namespace {

enum Exit { kOk = 0, kNotConverged = 1, kConfig = 2, kFault = 3 };

struct ConfigErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Fault : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::string strip(const std::string& s) {
    const size_t a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    const size_t b = s.find_last_not_of(" \t\r\n");
    return s.substr(a, b - a + 1);
}

class Config {
public:
    static Config load(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw ConfigErr("cannot open config file '" + path + "'");
        Config c;
        std::string line;
        int no = 0;
        while (std::getline(in, line)) {
            ++no;
            const size_t hash = line.find('#');
            if (hash != std::string::npos) line.resize(hash);
            line = strip(line);
            if (line.empty()) continue;
            const size_t eq = line.find('=');
            if (eq == std::string::npos)
                throw ConfigErr("config line " + std::to_string(no) + ": expected 'key = value'");
            const std::string k = strip(line.substr(0, eq)), v = strip(line.substr(eq + 1));
            if (k.empty() || v.empty())
                throw ConfigErr("config line " + std::to_string(no) + ": empty key or value");
            if (!c.kv_.emplace(k, v).second) throw ConfigErr("config: duplicate key '" + k + "'");
        }
        return c;
    }
    bool has(const std::string& k) const { return kv_.count(k) != 0; }
    std::string str(const std::string& k) const {
        auto it = kv_.find(k);
        if (it == kv_.end()) throw ConfigErr("config: missing key '" + k + "'");
        return it->second;
    }
    std::string str(const std::string& k, const std::string& d) const { return has(k) ? str(k) : d; }
    double num(const std::string& k) const {
        const std::string s = str(k);
        size_t pos = 0;
        double v = 0;
        try {
            v = std::stod(s, &pos);
        } catch (...) {
            pos = 0;
        }
        if (pos != s.size() || s.empty())
            throw ConfigErr("config: key '" + k + "' is not a number: '" + s + "'");
        return v;
    }
    double num(const std::string& k, double d) const { return has(k) ? num(k) : d; }
    int integer(const std::string& k) const {
        const std::string s = str(k);
        size_t pos = 0;
        long v = 0;
        try {
            v = std::stol(s, &pos);
        } catch (...) {
            pos = 0;
        }
        if (pos != s.size() || s.empty())
            throw ConfigErr("config: key '" + k + "' is not an integer: '" + s + "'");
        return static_cast<int>(v);
    }
    int integer(const std::string& k, int d) const { return has(k) ? integer(k) : d; }
    std::vector<int> ints(const std::string& k) const {
        std::vector<int> out;
        std::stringstream ss(str(k));
        std::string part;
        while (std::getline(ss, part, ',')) {
            part = strip(part);
            if (part.empty()) continue;
            size_t pos = 0;
            int v = 0;
            try {
                v = std::stoi(part, &pos);
            } catch (...) {
                pos = 0;
            }
            if (pos != part.size())
                throw ConfigErr("config: key '" + k + "' has a non-integer entry '" + part + "'");
            out.push_back(v);
        }
        if (out.empty()) throw ConfigErr("config: key '" + k + "' is an empty list");
        return out;
    }
    void only(const std::vector<std::string>& allowed) const {
        for (const auto& kv : kv_) {
            bool ok = false;
            for (const auto& a : allowed) ok = ok || kv.first == a;
            if (!ok) throw ConfigErr("config: unknown key '" + kv.first + "'");
        }
    }

private:
    std::map<std::string, std::string> kv_;
};

std::vector<std::string> problem_keys(const std::string& p) {
    if (p == "dahlquist") return {"dahlquist.lambda", "dahlquist.u0"};
    if (p == "heat1d") return {"heat1d.dof", "heat1d.x0", "heat1d.x1"};
    if (p == "allencahn")
        return {"allencahn.n", "allencahn.eps", "allencahn.length", "allencahn.newton_tol",
                "allencahn.newton_max_iters", "allencahn.ic_seed", "allencahn.ic_amplitude"};
    if (p == "heat2d") return {"heat2d.nx", "heat2d.cg_rtol", "heat2d.cg_max_iters"};
    if (p == "grayscott")
        return {"grayscott.n",    "grayscott.domain",     "grayscott.feed",
                "grayscott.kill", "grayscott.du",         "grayscott.dv",
                "grayscott.newton_tol", "grayscott.newton_max_iters"};
    throw ConfigErr("config: unknown problem '" + p + "'");
}

std::vector<std::string> common_keys() {
    return {"problem",          "grid.t0",           "grid.tf",          "grid.n_points",
            "solver.mode",      "solver.relaxation", "solver.nu",        "solver.max_iters",
            "solver.tol",       "solver.initial_guess", "solver.seed",   "solver.coarse_substeps",
            "solver.norm",      "runtime.workers",   "runtime.trace",    "output.path"};
}

struct Built {
    atm_problem p{};
    atm_grid g{};
    atm_solver s{};
    atm_runtime rt{};
    std::vector<double> ic, fw;
    int n = 1;
};

// solver_config_from / application_from (run_config.cpp:207-262)
Built build(const Config& c, const std::vector<int>& m, int k, int workers) {
    Built b;
    const std::string mode = c.str("solver.mode", "two-level");
    if (mode == "two-level") b.s.mode = ATM_TWO_LEVEL;
    else if (mode == "v-cycle") b.s.mode = ATM_VCYCLE;
    else if (mode == "nested-v") b.s.mode = ATM_NESTED_V;
    else throw ConfigErr("config: solver.mode must be two-level, v-cycle or nested-v");
    const std::string relax = c.str("solver.relaxation", "F");
    if (relax == "F") b.s.relaxation = ATM_RELAX_F;
    else if (relax == "FCF") b.s.relaxation = ATM_RELAX_FCF;
    else throw ConfigErr("config: solver.relaxation must be F or FCF");
    b.s.nu = c.integer("solver.nu", 1);
    b.s.max_iters = c.integer("solver.max_iters", 100);
    b.s.tol = c.num("solver.tol");
    const std::string guess = c.str("solver.initial_guess", "constant");
    if (guess == "constant") b.s.initial_guess = ATM_GUESS_CONSTANT;
    else if (guess == "random") b.s.initial_guess = ATM_GUESS_RANDOM;
    else throw ConfigErr("config: solver.initial_guess must be constant or random");
    b.s.seed = static_cast<uint64_t>(c.integer("solver.seed", 0));
    b.s.coarse_substeps = c.integer("solver.coarse_substeps", 1);
    const bool folded = b.s.mode != ATM_TWO_LEVEL;

    const std::string prob = c.str("problem");
    if (prob == "dahlquist") {
        b.p.kind = ATM_PHI_DAHLQUIST;
        b.p.n = 1;
        b.p.lambda = c.num("dahlquist.lambda", -1.0);
        b.p.u0 = c.num("dahlquist.u0", 1.0);
        b.p.folded = folded;
    } else if (prob == "heat1d") {
        b.p.kind = ATM_PHI_HEAT1D;
        b.p.n = c.integer("heat1d.dof", 1025);
        b.p.x0 = c.num("heat1d.x0", 0.0);
        b.p.x1 = c.num("heat1d.x1", 1.0);
        b.p.folded = folded;
        b.p.manufactured = 1;  // Heat1D::Options default (heat1d.hpp:27); the CLI has no key for it
    } else if (prob == "allencahn") {
        b.p.kind = ATM_PHI_ALLEN_CAHN;
        b.p.n = c.integer("allencahn.n", 4096);
        b.p.eps = c.num("allencahn.eps", 0.02);
        b.p.length = c.num("allencahn.length", 1.0);
        b.p.newton_tol = c.num("allencahn.newton_tol", 1e-12);
        b.p.newton_max = c.integer("allencahn.newton_max_iters", 30);
        b.p.folded = 1;
        b.ic.resize(b.p.n);
        atm_random_state(static_cast<uint64_t>(c.integer("allencahn.ic_seed", 3)), b.p.n, b.ic.data());
        const double amp = c.num("allencahn.ic_amplitude", 0.05);
        for (double& v : b.ic) v *= amp;
    } else if (prob == "grayscott") {
        // GrayScott::Options defaults (gray_scott.hpp:24-38)
        b.p.kind = ATM_PHI_GRAY_SCOTT;
        b.p.nx = c.integer("grayscott.n", 32);
        b.p.n = 2 * b.p.nx * b.p.nx;
        b.p.gs_domain = c.num("grayscott.domain", 2.5);
        b.p.gs_feed = c.num("grayscott.feed", 0.024);
        b.p.gs_kill = c.num("grayscott.kill", 0.06);
        b.p.gs_du = c.num("grayscott.du", 8e-5);
        b.p.gs_dv = c.num("grayscott.dv", 4e-5);
        b.p.newton_tol = c.num("grayscott.newton_tol", 1e-10);
        b.p.newton_max = c.integer("grayscott.newton_max_iters", 30);
        b.p.gs_linear_tol = 1e-10;
        b.p.gs_reaction = 1;
        b.p.gs_bounds_check = 1;
        b.p.gs_bound_lo = -1.0;
        b.p.gs_bound_hi = 3.0;
        b.p.folded = 1;
    } else if (prob == "heat2d") {
        b.p.kind = ATM_PHI_HEAT2D;
        b.p.nx = c.integer("heat2d.nx", 127);
        b.p.n = b.p.nx * b.p.nx;
        b.p.cg_rtol = c.num("heat2d.cg_rtol", 1e-12);
        b.p.cg_max = c.integer("heat2d.cg_max_iters", 10000);
        b.p.folded = folded;
    } else {
        problem_keys(prob);  // throws with the reference's message
    }
    b.n = b.p.n;
    const std::string norm = c.str("solver.norm", "residual-2norm");
    if (norm == "residual-2norm") {
        b.s.norm = ATM_NORM_L2;
    } else if (norm == "functional-change") {
        // the reference CLI's functional is u.norm2() (run_config.cpp:241-243)
        b.s.norm = ATM_NORM_FUNCTIONAL;
        b.s.functional_kind = ATM_FUNCTIONAL_NORM2;
    } else {
        throw ConfigErr("config: solver.norm must be residual-2norm or functional-change");
    }
    b.g.t0 = c.num("grid.t0", 0.0);
    b.g.tf = c.num("grid.tf");
    b.g.n_points = c.integer("grid.n_points");
    if (m.size() > ATM_MAX_LEVELS - 1) throw ConfigErr("config: too many coarsening factors");
    b.g.n_m = static_cast<int>(m.size());
    for (size_t i = 0; i < m.size(); ++i) b.g.m[i] = m[i];
    b.g.k = k;
    b.rt.device = 0;
    b.rt.n_shards = workers;
    b.rt.world_size = 1;
    if (!b.ic.empty()) b.p.ic = b.ic.data();
    return b;
}

struct RunResult {
    std::vector<double> norms, secs;
    bool converged = false;
    int iterations = 0;
    double total = 0.0;
};

void check(atm_status st, atm_ctx* ctx) {
    if (st == ATM_OK || st == ATM_NOT_CONVERGED) return;
    const std::string msg = ctx ? atm_last_error(ctx) : atm_create_error();
    if (st == ATM_CONFIG_ERROR) throw ConfigErr(msg);
    throw Fault(msg);
}

// per-phase device seconds since setup, by name (atm_phase_times)
std::map<std::string, double> phase_seconds(atm_ctx* ctx) {
    char names[2048];
    double secs[64];
    const int k = atm_phase_times(ctx, names, sizeof(names), secs, 64);
    std::map<std::string, double> out;
    std::stringstream ss(names);
    std::string nm;
    for (int i = 0; i < k && std::getline(ss, nm, ','); ++i) out[nm] = secs[i];
    return out;
}

// drive (solver.cpp:398-435) one iteration at a time for per-iteration
// seconds; with a trace path, per-iteration phase rows `iter,rank,phase,
// seconds` like the reference's TraceSink (run_config.cpp:272-283), timed on
// the device with CUDA events
RunResult run(const Built& b, const std::string& trace_path = "") {
    RunResult r;
    atm_ctx* ctx = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    std::ofstream trace;
    Built bt = b;
    if (!trace_path.empty()) {
        trace.open(trace_path);
        if (!trace) throw ConfigErr("cannot open trace file '" + trace_path + "'");
        trace << "iter,rank,phase,seconds\n";
        trace.precision(17);
        bt.rt.trace = 1;
    }
    check(atm_create(&bt.p, &bt.g, &bt.s, &bt.rt, &ctx), nullptr);
    struct Guard {
        atm_ctx* c;
        ~Guard() { atm_destroy(c); }
    } guard{ctx};
    check(atm_setup(ctx), ctx);
    if (b.s.mode == ATM_NESTED_V) check(atm_nested_init(ctx), ctx);
    std::map<std::string, double> before;
    if (trace.is_open()) before = phase_seconds(ctx);
    for (int it = 1; it <= b.s.max_iters; ++it) {
        const auto a = std::chrono::steady_clock::now();
        double v = 0.0;
        check(atm_iterate(ctx, 1, &v), ctx);
        if (trace.is_open()) {
            const std::map<std::string, double> now = phase_seconds(ctx);
            for (const auto& kv : now) {
                const double d = kv.second - (before.count(kv.first) ? before[kv.first] : 0.0);
                if (d > 0.0) trace << it << ",0," << kv.first << ',' << d << '\n';
            }
            before = now;
        }
        r.secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
        r.norms.push_back(v);
        r.iterations = it;
        if (!std::isfinite(v))
            throw Fault("non-finite residual norm at iteration " + std::to_string(it));
        if (v <= b.s.tol) {
            r.converged = true;
            break;
        }
    }
    r.total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

int cmd_solve(const Config& c, const std::string& out_path, int workers_override) {
    std::vector<std::string> allowed = common_keys();
    allowed.push_back("solver.m");
    allowed.push_back("solver.k");
    for (const auto& k : problem_keys(c.str("problem"))) allowed.push_back(k);
    c.only(allowed);
    const int workers = workers_override > 0 ? workers_override : c.integer("runtime.workers", 1);
    const Built b = build(c, c.ints("solver.m"), c.integer("solver.k"), workers);
    const RunResult r = run(b, c.str("runtime.trace", ""));
    std::ofstream file;
    const std::string path = !out_path.empty() ? out_path : c.str("output.path", "");
    if (!path.empty()) {
        file.open(path);
        if (!file) throw ConfigErr("cannot open output file '" + path + "'");
    }
    std::ostream& out = file.is_open() ? file : std::cout;
    out.precision(17);
    out << "iter,residual_norm,seconds\n";
    for (size_t i = 0; i < r.norms.size(); ++i) out << (i + 1) << ',' << r.norms[i] << ',' << r.secs[i] << '\n';
    out << "converged,iterations,total_seconds\n";
    out << (r.converged ? 1 : 0) << ',' << r.iterations << ',' << r.total << '\n';
    return r.converged ? kOk : kNotConverged;
}

int cmd_sweep_k(const Config& c, const std::string& out_path, int workers_override) {
    std::vector<std::string> allowed = common_keys();
    allowed.push_back("sweep.m_values");
    allowed.push_back("sweep.k_values");
    for (const auto& k : problem_keys(c.str("problem"))) allowed.push_back(k);
    c.only(allowed);
    const int workers = workers_override > 0 ? workers_override : c.integer("runtime.workers", 1);
    std::ofstream file;
    const std::string path = !out_path.empty() ? out_path : c.str("output.path", "");
    if (!path.empty()) {
        file.open(path);
        if (!file) throw ConfigErr("cannot open output file '" + path + "'");
    }
    std::ostream& out = file.is_open() ? file : std::cout;
    out << "m,k,k_over_ncpoints,iterations,parareal_equivalent\n";
    const int npts = c.integer("grid.n_points");
    for (int m : c.ints("sweep.m_values")) {
        const int nc = (npts - 1) / m + 1;
        for (int kr : c.ints("sweep.k_values")) {
            const int k = kr == 0 ? nc : kr;
            const RunResult r = run(build(c, {m}, k, workers));
            out << m << ',' << k << ',' << static_cast<double>(k) / nc << ',' << r.iterations << ','
                << (k >= nc ? 1 : 0) << '\n';
            if (!r.converged)
                std::cerr << "warning: m=" << m << " k=" << k
                          << " did not converge within solver.max_iters\n";
        }
    }
    return kOk;
}

int usage() {
    std::cerr << "usage: tempo_b200 {solve|sweep-k} CONFIG [--out PATH] [--workers N]\n";
    return kConfig;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) return usage();
    const std::string cmd = argv[1], cfg_path = argv[2];
    std::string out;
    int workers = 0;
    for (int i = 3; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--out" && i + 1 < argc) out = argv[++i];
        else if (a == "--workers" && i + 1 < argc) workers = std::atoi(argv[++i]);
        else return usage();
    }
    try {
        const Config c = Config::load(cfg_path);
        if (cmd == "solve") return cmd_solve(c, out, workers);
        if (cmd == "sweep-k") return cmd_sweep_k(c, out, workers);
        return usage();
    } catch (const ConfigErr& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kConfig;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kFault;
    }
}
