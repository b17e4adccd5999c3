// capi.cpp -- extern "C" boundary (include/atmgrit.h) over atm::Engine.
// Every exception is mapped to an atm_status (errors.hpp:9-42 taxonomy).
#include <cstring>
#include <memory>
#include <string>

#include "atmgrit.h"
#include "engine.hpp"

struct atm_ctx {
    std::unique_ptr<atm::Engine> eng;
    std::string err;
};

namespace {

thread_local std::string g_create_err;

template <class F>
atm_status guard(atm_ctx* c, F&& f) {
    if (!c || !c->eng) return ATM_CONFIG_ERROR;
    try {
        return static_cast<atm_status>(f());
    } catch (const atm::Error& e) {
        c->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        c->err = e.what();
        return ATM_RUNTIME_FAULT;
    }
}

void fill_grid_hier(const atm_grid* g, atm::Hier* h) { *h = atm::make_hier(*g); }

}  // namespace

extern "C" {

int atm_abi_version(void) { return ATM_ABI_VERSION; }

const char* atm_create_error(void) { return g_create_err.c_str(); }

int atm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

atm_status atm_create(const atm_problem* problem, const atm_grid* grid, const atm_solver* solver,
                      const atm_runtime* runtime, atm_ctx** out) {
    if (!out || !problem || !grid || !solver) {
        g_create_err = "atm_create: null argument";
        return ATM_CONFIG_ERROR;
    }
    *out = nullptr;
    atm_runtime rt{};
    if (runtime) rt = *runtime;
    try {
        // the context is released to the caller only once the engine exists
        // (a ConfigError or CUDA fault in the constructor frees it here)
        auto c = std::make_unique<atm_ctx>();
        c->eng = std::make_unique<atm::Engine>(*problem, *grid, *solver, rt);
        *out = c.release();
        g_create_err.clear();
        return ATM_OK;
    } catch (const atm::Error& e) {
        g_create_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return ATM_RUNTIME_FAULT;
    }
}

void atm_destroy(atm_ctx* ctx) { delete ctx; }

const char* atm_last_error(const atm_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

atm_status atm_setup(atm_ctx* c) {
    return guard(c, [&] { c->eng->setup(); return 0; });
}

atm_status atm_nested_init(atm_ctx* c) {
    return guard(c, [&] { c->eng->nested_init(); return 0; });
}

atm_status atm_cycle(atm_ctx* c) {
    return guard(c, [&] { c->eng->cycle(); return 0; });
}

atm_status atm_residual_norm(atm_ctx* c, double* out) {
    return guard(c, [&] { *out = c->eng->residual_norm(); return 0; });
}

atm_status atm_solve(atm_ctx* c, atm_report* rep, double* norms, double* iteration_seconds) {
    return guard(c, [&] { return c->eng->solve(rep, norms, iteration_seconds); });
}

atm_status atm_iterate(atm_ctx* c, int count, double* norms) {
    return guard(c, [&] { c->eng->iterate(count, norms); return 0; });
}

atm_status atm_get_level(atm_ctx* c, int level, int which, int first, int count, double* out) {
    return guard(c, [&] { c->eng->get_level(level, which, first, count, out); return 0; });
}

atm_status atm_set_level(atm_ctx* c, int level, int which, int first, int count,
                         const double* in) {
    return guard(c, [&] { c->eng->set_level(level, which, first, count, in); return 0; });
}

int atm_level_points(const atm_ctx* c, int level) {
    return (c && c->eng && level >= 0 && level < c->eng->n_levels()) ? c->eng->level_points(level) : -1;
}

int atm_vector_size(const atm_ctx* c) { return (c && c->eng) ? c->eng->vector_size() : -1; }

int atm_n_levels(const atm_ctx* c) { return (c && c->eng) ? c->eng->n_levels() : -1; }

atm_status atm_apply_phi(atm_ctx* c, int level, int first_index, int count, const double* in,
                         double* out) {
    return guard(c, [&] { c->eng->apply_phi(level, first_index, count, in, out, false); return 0; });
}

atm_status atm_forcing(atm_ctx* c, int level, int first_index, int count, double* out) {
    return guard(c, [&] { c->eng->apply_phi(level, first_index, count, nullptr, out, true); return 0; });
}

atm_status atm_kernel_f_relax(atm_ctx* c, int level, int first_interval, int count) {
    return guard(c, [&] { c->eng->kernel_f_relax(level, first_interval, count); return 0; });
}

atm_status atm_kernel_c_relax(atm_ctx* c, int level, int first_c, int count) {
    return guard(c, [&] { c->eng->kernel_c_relax(level, first_c, count); return 0; });
}

atm_status atm_kernel_residual(atm_ctx* c, int level, int first, int count, double* out) {
    return guard(c, [&] { c->eng->kernel_residual(level, first, count, out); return 0; });
}

int atm_phase_times(const atm_ctx* c, char* names_csv, int names_cap, double* seconds, int cap) {
    if (!c || !c->eng) return 0;
    return c->eng->phase_times(names_csv, names_cap, seconds, cap);
}

int atm_phase_counts(const atm_ctx* c, int* counts, int cap) {
    if (!c || !c->eng) return 0;
    std::vector<double> secs(cap);
    return c->eng->phase_times(nullptr, 0, secs.data(), cap, counts);
}

atm_status atm_iterate_timed(atm_ctx* c, int count, double* norms, double* device_ms) {
    return guard(c, [&] {
        const double ms = c->eng->iterate_timed(count, norms);
        if (device_ms) *device_ms = ms;
        return 0;
    });
}

atm_status atm_host_register(void* ptr, size_t bytes) {
    return cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess ? ATM_OK
                                                                              : ATM_RUNTIME_FAULT;
}

atm_status atm_host_unregister(void* ptr) {
    return cudaHostUnregister(ptr) == cudaSuccess ? ATM_OK : ATM_RUNTIME_FAULT;
}

atm_status atm_last_iteration_stats(const atm_ctx* c, int* launches, double* sweep_ms) {
    if (!c || !c->eng) return ATM_CONFIG_ERROR;
    if (launches) *launches = c->eng->last_launches();
    if (sweep_ms) *sweep_ms = c->eng->last_sweep_ms();
    return ATM_OK;
}

atm_status atm_inner_iterations(atm_ctx* c, unsigned long long* out) {
    if (!c || !c->eng || !out) return ATM_CONFIG_ERROR;
    return guard(c, [&] { *out = c->eng->inner_iterations(); return 0; });
}

atm_status atm_host_traffic(const atm_ctx* c, unsigned long long* h2d, unsigned long long* d2h) {
    if (!c || !c->eng) return ATM_CONFIG_ERROR;
    c->eng->host_traffic(h2d, d2h);
    return ATM_OK;
}

// ---- host-only helpers ------------------------------------------------------

void atm_random_state(uint64_t seed, int n, double* out) {
    uint64_t s = seed;
    for (int i = 0; i < n; ++i) {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z = z ^ (z >> 31);
        out[i] = 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
    }
}

atm_status atm_build_layout(const atm_grid* grid, int workers, int* fine_lo, int* fine_hi,
                            int* coarse_lo, int* coarse_hi) {
    try {
        atm::Hier h;
        fill_grid_hier(grid, &h);
        const atm::Layout lay = atm::build_layout(h, workers);
        for (int r = 0; r < workers; ++r) {
            fine_lo[r] = lay.fine_lo[r];
            fine_hi[r] = lay.fine_hi[r];
            coarse_lo[r] = lay.coarse_lo[r];
            coarse_hi[r] = lay.coarse_hi[r];
        }
        return ATM_OK;
    } catch (const atm::Error& e) {
        g_create_err = e.what();
        return e.code;
    }
}

atm_status atm_rank_ranges(const atm_grid* grid, int workers, int rank, int* lo, int* hi,
                           int* iv_first, int* iv_count, int* c_first, int* c_count,
                           int* left_src, int* right_dst) {
    try {
        atm::Hier h;
        fill_grid_hier(grid, &h);
        const atm::Layout lay = atm::build_layout(h, workers);
        if (rank < 0 || rank >= workers) return ATM_CONFIG_ERROR;
        const atm::Ranges rr = atm::compute_ranges(h, lay, rank);
        for (int l = 0; l < h.L; ++l) {
            lo[l] = rr.lo[l];
            hi[l] = rr.hi[l];
            iv_first[l] = rr.iv_first[l];
            iv_count[l] = rr.iv_count[l];
            c_first[l] = rr.c_first[l];
            c_count[l] = rr.c_count[l];
            left_src[l] = rr.left_src[l];
            right_dst[l] = rr.right_dst[l];
        }
        return ATM_OK;
    } catch (const atm::Error& e) {
        g_create_err = e.what();
        return e.code;
    }
}

int atm_window_recvs(const atm_grid* grid, int workers, int rank, int* sends, int cap) {
    try {
        atm::Hier h;
        fill_grid_hier(grid, &h);
        const atm::Layout lay = atm::build_layout(h, workers);
        const int lc = h.coarsest();
        const atm::Ranges me = atm::compute_ranges(h, lay, rank);
        const int need_lo = std::max(0, me.lo[lc] - h.k + 1), need_hi = me.lo[lc] - 1;
        int cnt = 0;
        for (int q = 0; q < workers && need_hi >= need_lo; ++q) {
            if (q == rank) continue;
            const atm::Ranges rq = atm::compute_ranges(h, lay, q);
            const int a0 = std::max(need_lo, rq.lo[lc]), a1 = std::min(need_hi, rq.hi[lc]);
            if (a1 < a0) continue;
            if (cnt < cap) {
                sends[3 * cnt] = q;
                sends[3 * cnt + 1] = a0;
                sends[3 * cnt + 2] = a1 - a0 + 1;
            }
            ++cnt;
        }
        return cnt;
    } catch (const atm::Error& e) {
        g_create_err = e.what();
        return -1;
    }
}

atm_status atm_nccl_unique_id(void* out128) { return atm::nccl_unique_id(out128); }

}  // extern "C"
