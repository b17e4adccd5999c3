/*
 * atm_oracle.c -- CPU restatement of the AT-MGRIT reference path.
 *
 * TEST INFRASTRUCTURE ONLY (see atm_oracle.h).  Plain C, sequential, no
 * dependency on the product library.  Arrays are point-major: the state of
 * point i on a level lives at base + i*n.
 *
 * All reference citations are relative to /root/reference/proj.
 */
#include "atm_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

/* ------------------------------------------------------------------------ */
/* seeded fills                                                              */

/* state_vector.hpp:92-97 (splitmix64) and :99-102 (top 53 bits -> [0,1)) */
static uint64_t sm64_next(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* state_vector.hpp:108-118: entries 2*U[0,1) - 1 drawn in index order */
void orc_random_state(uint64_t seed, int n, double* out) {
    uint64_t s = seed;
    for (int i = 0; i < n; ++i) {
        const double unit = (double)(sm64_next(&s) >> 11) * 0x1.0p-53;
        out[i] = 2.0 * unit - 1.0;
    }
}

/* ------------------------------------------------------------------------ */
/* grids                                                                     */

/* hierarchy.cpp:35 -- n_coarse = (n_points - 1)/m + 1 per transition */
int orc_level_points(const orc_grid* g, int level) {
    int np = g->n_points;
    for (int l = 0; l < level; ++l) np = (np - 1) / g->m[l] + 1;
    return np;
}

/* time_grid.hpp:20 and hierarchy.cpp:42 -- dt_{l+1} = m_l * dt_l */
double orc_level_dt(const orc_grid* g, int level) {
    double dt = (g->tf - g->t0) / (double)(g->n_points - 1);
    for (int l = 0; l < level; ++l) dt = dt * g->m[l];
    return dt;
}

/* ------------------------------------------------------------------------ */
/* the driver object                                                         */

struct orc_driver {
    orc_problem p;
    orc_grid g;
    orc_solver s;
    int L, n;
    /* LevelSpec per level (application.hpp:11-16, solver.cpp:30-43) */
    double dt[ORC_MAXL], t0[ORC_MAXL];
    int np[ORC_MAXL], sub[ORC_MAXL];
    /* heat1d per-level factorization (heat1d.cpp:24-45) */
    double h;
    double* sinp;
    double* cpr[ORC_MAXL];
    double* inv[ORC_MAXL];
    double rr[ORC_MAXL], sdt[ORC_MAXL];
    /* heat2d per-level shift: A = (1/sdt) I - lap  */
    double* work;          /* scratch, several n-vectors               */
    double* ic;
    double* ff;            /* scalar fine forcing copy                 */
    double* fw;            /* functional weights copy                  */
    double* cval;          /* constant guess copy                      */
    double* prov;          /* provided guess copy                      */
    double* src;           /* heat2d source copy                       */
    /* per-level arrays */
    double* u[ORC_MAXL];
    double* gg[ORC_MAXL];
    double* v[ORC_MAXL];
    double* r[ORC_MAXL];
    double* rs;            /* level-0 residual scratch                 */
    double* gs_work;       /* gray-scott Newton / BiCGSTAB scratch     */
    double* prevf;         /* functional-change history per C-point    */
    int setup_done;
    int newton_fail;
    char err[256];
};

static char g_create_err[256];

static int fail(orc_driver* d, int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(d ? d->err : g_create_err, 256, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_error(const orc_driver* d) { return d->err; }
const char* orc_create_error(void) { return g_create_err; }

static double* vec(orc_driver* d, int level, int which, int i) {
    double* base = which == 0 ? d->u[level] : which == 1 ? d->gg[level]
                 : which == 2 ? d->v[level] : d->r[level];
    return base + (size_t)i * d->n;
}

static int cpoints(const orc_driver* d, int level) {
    return (d->np[level] - 1) / d->g.m[level] + 1;
}

/* hierarchy.cpp:7-22: one F-interval after each C-point c with c+1 <= last */
static int n_intervals(const orc_driver* d, int level) {
    const int m = d->g.m[level], last = d->np[level] - 1;
    const int nc = cpoints(d, level);
    return ((nc - 1) * m + 1 <= last) ? nc : nc - 1;
}

/* ------------------------------------------------------------------------ */
/* heat1d (heat1d.cpp)                                                       */

/* heat1d.cpp:47-60: (I + sub_dt L) x = rhs in place, precomputed Thomas */
static void heat_tridiag(const orc_driver* d, int level, double* x) {
    const int n = d->n;
    const double a = -d->rr[level];
    const double* inv = d->inv[level];
    const double* cp = d->cpr[level];
    double prev = 0.0;
    for (int i = 0; i < n; ++i) {
        prev = (x[i] - a * prev) * inv[i];
        x[i] = prev;
    }
    for (int i = n - 2; i >= 0; --i) x[i] -= cp[i] * x[i + 1];
}

/* heat1d.cpp:62-64 */
static double heat_time_factor(double t) { return -(sin(t) - kPi * kPi * cos(t)); }

/* heat1d.cpp:66-83: substep chain, forcing added before each solve */
static void heat_propagate(const orc_driver* d, int level, int index, const double* in,
                           double* out, int with_forcing) {
    const int n = d->n;
    if (out != in) memcpy(out, in, sizeof(double) * (size_t)n);
    for (int s = 1; s <= d->sub[level]; ++s) {
        if (with_forcing && d->p.manufactured) {
            const double t = (d->t0[level] + d->dt[level] * (index - 1)) + d->sdt[level] * s;
            const double theta = d->sdt[level] * heat_time_factor(t);
            for (int i = 0; i < n; ++i) out[i] += theta * d->sinp[i];
        }
        heat_tridiag(d, level, out);
    }
}

/* ------------------------------------------------------------------------ */
/* Allen-Cahn: backward Euler + Newton, periodic, cyclic tridiagonal J.      */
/* No reference counterpart; Newton stopping rule mirrors      */
/* gray_scott.cpp:113 stop = max(tol, tol*|res0|), cap -> NonlinearSolve.    */

/* cyclic tridiagonal solve, constant off-diagonal e, diagonal diag[],
 * via Sherman-Morrison: A = T + alpha*beta-corner; standard restatement. */
static void cyclic_tridiag(int n, double e, const double* diag, double* rhs, double* w1,
                           double* w2, double* w3) {
    /* A = tridiag(e, diag, e) + e*(E_{0,n-1} + E_{n-1,0}).
     * Write A = B + w w^T... use u = (gamma,0..,0,e), v = (1,0..,0,e/gamma). */
    const double gamma = -diag[0];
    /* B: diag with b0 - gamma, b_{n-1} - e*e/gamma */
    double* bd = w1;
    for (int i = 0; i < n; ++i) bd[i] = diag[i];
    bd[0] -= gamma;
    bd[n - 1] -= e * e / gamma;
    /* solve B y = rhs and B z = uvec with a Thomas sweep (shared factors) */
    double* cp = w2;   /* c' */
    double* z = w3;
    double den = bd[0];
    cp[0] = e / den;
    rhs[0] = rhs[0] / den;
    z[0] = gamma / den;
    for (int i = 1; i < n; ++i) {
        den = bd[i] - e * cp[i - 1];
        cp[i] = e / den;
        const double zi = (i == n - 1) ? e : 0.0;
        rhs[i] = (rhs[i] - e * rhs[i - 1]) / den;
        z[i] = (zi - e * z[i - 1]) / den;
    }
    for (int i = n - 2; i >= 0; --i) {
        rhs[i] -= cp[i] * rhs[i + 1];
        z[i] -= cp[i] * z[i + 1];
    }
    const double vy = rhs[0] + (e / gamma) * rhs[n - 1];
    const double vz = z[0] + (e / gamma) * z[n - 1];
    const double f = vy / (1.0 + vz);
    for (int i = 0; i < n; ++i) rhs[i] -= f * z[i];
}

/* residual F(u) = u - dt*(eps^2 D2 u + u - u^3) - u_prev (periodic) */
static void ac_residual(const orc_driver* d, double dt, const double* u, const double* up,
                        double* F) {
    const int n = d->n;
    const double hx = d->p.length / n;
    const double c = d->p.eps * d->p.eps / (hx * hx);
    for (int i = 0; i < n; ++i) {
        const double ul = u[(i + n - 1) % n], ur = u[(i + 1) % n], ui = u[i];
        const double lap = c * (ul - 2.0 * ui + ur);
        F[i] = ui - dt * (lap + ui - ui * ui * ui) - up[i];
    }
}

static double nrm2(int n, const double* x) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * x[i];
    return sqrt(s);
}

static int ac_step(orc_driver* d, int level, const double* in, double* out) {
    const int n = d->n;
    double* F = d->work;
    double* diag = F + n;
    double* w1 = diag + n;
    double* w2 = w1 + n;
    double* w3 = w2 + n;
    double* up = w3 + n;
    memcpy(up, in, sizeof(double) * (size_t)n);
    if (out != in) memcpy(out, in, sizeof(double) * (size_t)n);
    const double hx = d->p.length / n;
    const double c = d->p.eps * d->p.eps / (hx * hx);
    for (int s = 1; s <= d->sub[level]; ++s) {
        const double dt = d->sdt[level];
        ac_residual(d, dt, out, up, F);
        const double res0 = nrm2(n, F);
        const double stop = fmax(d->p.newton_tol, d->p.newton_tol * res0);
        int it = 0;
        double res = res0;
        while (res > stop) {
            if (it >= d->p.newton_max) {
                d->newton_fail = 1;
                return fail(d, ORC_NONLINEAR, "allen-cahn: Newton did not converge in %d iterations",
                            d->p.newton_max);
            }
            /* J = (1 + 2 dt c - dt + 3 dt u^2) on the diagonal, -dt c off */
            for (int i = 0; i < n; ++i)
                diag[i] = 1.0 + 2.0 * dt * c - dt + 3.0 * dt * out[i] * out[i];
            for (int i = 0; i < n; ++i) F[i] = -F[i];
            cyclic_tridiag(n, -dt * c, diag, F, w1, w2, w3);
            for (int i = 0; i < n; ++i) out[i] += F[i];
            ac_residual(d, dt, out, up, F);
            res = nrm2(n, F);
            ++it;
        }
        memcpy(up, out, sizeof(double) * (size_t)n);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* 2D heat: backward Euler, 5-point Laplacian (zero Dirichlet), CG per step.  */
/* No reference counterpart.  System: (I - dt*lap) x = b,      */
/* CG from x0 = b's source state (u_prev), stop |r| <= rtol*|b|.              */

static void h2_apply(const orc_driver* d, double dt, const double* x, double* y) {
    const int nx = d->p.nx;
    const double hh = 1.0 / (double)(nx + 1);
    const double c = dt / (hh * hh);
    for (int j = 0; j < nx; ++j) {
        for (int i = 0; i < nx; ++i) {
            const int q = j * nx + i;
            const double xw = i > 0 ? x[q - 1] : 0.0;
            const double xe = i < nx - 1 ? x[q + 1] : 0.0;
            const double xs = j > 0 ? x[q - nx] : 0.0;
            const double xn = j < nx - 1 ? x[q + nx] : 0.0;
            y[q] = (1.0 + 4.0 * c) * x[q] - c * (((xw + xe) + xs) + xn);
        }
    }
}

static double dotp(int n, const double* a, const double* b) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static int h2_solve(orc_driver* d, double dt, const double* b, double* x) {
    const int n = d->n;
    double* r = d->work;
    double* p = r + n;
    double* ap = p + n;
    h2_apply(d, dt, x, ap);
    for (int i = 0; i < n; ++i) r[i] = b[i] - ap[i];
    const double bn = sqrt(dotp(n, b, b));
    const double stop = d->p.cg_rtol * bn;
    double rr = dotp(n, r, r);
    memcpy(p, r, sizeof(double) * (size_t)n);
    int it = 0;
    while (sqrt(rr) > stop) {
        if (it >= d->p.cg_max)
            return fail(d, ORC_NONLINEAR, "heat2d: CG did not converge in %d iterations",
                        d->p.cg_max);
        h2_apply(d, dt, p, ap);
        const double alpha = rr / dotp(n, p, ap);
        for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] -= alpha * ap[i];
        const double rr_new = dotp(n, r, r);
        const double beta = rr_new / rr;
        rr = rr_new;
        for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        ++it;
    }
    return ORC_OK;
}

/* propagate like heat1d.cpp:66-83: per substep x <- A^{-1}(x + sdt*f) */
static int h2_propagate(orc_driver* d, int level, const double* in, double* out,
                        int with_forcing) {
    const int n = d->n;
    double* b = d->work + 3 * (size_t)n;
    if (out != in) memcpy(out, in, sizeof(double) * (size_t)n);
    for (int s = 1; s <= d->sub[level]; ++s) {
        memcpy(b, out, sizeof(double) * (size_t)n);
        if (with_forcing && d->src)
            for (int i = 0; i < n; ++i) b[i] += d->sdt[level] * d->src[i];
        const int st = h2_solve(d, d->sdt[level], b, out);
        if (st) return st;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Gray-Scott (gray_scott.cpp:16-190): periodic n x n cells on [0, domain]^2,  */
/* state [u; v]; backward Euler, Newton with the analytic Jacobian and an     */
/* inner BiCGSTAB with diagonal (Jacobi) preconditioning, right-              */
/* preconditioned, x0 = 0, |r|^2 <= tol^2 |b|^2, at most 2 dim iterations, a  */
/* restart when rho degenerates -- the published algorithm the reference      */
/* delegates to Eigen::BiCGSTAB (Eigen >= 3.3, absent here: parity unpinned). */

static int gs_nb(int n, int i, int j) { return ((i + n) % n) * n + (j + n) % n; }

/* reaction_terms (gray_scott.cpp:63-88) */
static void gs_rhs(const orc_driver* d, const double* w, double* f) {
    const int n = d->p.nx, cells = n * n;
    const double h = d->p.gs_domain / n, ih2 = 1.0 / (h * h);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const int c = i * n + j;
            const int N = gs_nb(n, i + 1, j), S = gs_nb(n, i - 1, j), E = gs_nb(n, i, j + 1),
                      W = gs_nb(n, i, j - 1);
            const double u = w[c], v = w[cells + c];
            const double lu = (w[N] + w[S] + w[E] + w[W] - 4.0 * u) * ih2;
            const double lv = (w[cells + N] + w[cells + S] + w[cells + E] + w[cells + W] - 4.0 * v) * ih2;
            double fu = d->p.gs_du * lu, fv = d->p.gs_dv * lv;
            if (d->p.gs_reaction) {
                const double uvv = u * v * v;
                fu += -uvv + d->p.gs_feed * (1.0 - u);
                fv += uvv - (d->p.gs_feed + d->p.gs_kill) * v;
            }
            f[c] = fu;
            f[cells + c] = fv;
        }
}

/* y = J x, J = I - dt f'(w) (the Jacobian of gray_scott.cpp:114-139) */
static void gs_jac(const orc_driver* d, double dt, const double* w, const double* x, double* y,
                   double* diag) {
    const int n = d->p.nx, cells = n * n;
    const double h = d->p.gs_domain / n, ih2 = 1.0 / (h * h);
    const double off = -dt * d->p.gs_du * ih2, offv = -dt * d->p.gs_dv * ih2;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const int c = i * n + j;
            const int N = gs_nb(n, i + 1, j), S = gs_nb(n, i - 1, j), E = gs_nb(n, i, j + 1),
                      W = gs_nb(n, i, j - 1);
            const double u = w[c], v = w[cells + c];
            double duu = 1.0 + dt * 4.0 * d->p.gs_du * ih2, dvv = 1.0 + dt * 4.0 * d->p.gs_dv * ih2;
            double cuv = 0.0, cvu = 0.0;
            if (d->p.gs_reaction) {
                duu += dt * (v * v + d->p.gs_feed);
                dvv += dt * (d->p.gs_feed + d->p.gs_kill) - dt * 2.0 * u * v;
                cuv = dt * 2.0 * u * v;
                cvu = -dt * v * v;
            }
            if (diag) {
                diag[c] = duu;
                diag[cells + c] = dvv;
            }
            if (x) {
                y[c] = duu * x[c] + off * (x[N] + x[S] + x[E] + x[W]) + cuv * x[cells + c];
                y[cells + c] = dvv * x[cells + c] +
                               offv * (x[cells + N] + x[cells + S] + x[cells + E] + x[cells + W]) +
                               cvu * x[c];
            }
        }
}

static double gs_dot(int m, const double* a, const double* b) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += a[i] * b[i];
    return s;
}

/* BiCGSTAB for J x = b, x0 = 0; returns 0 on convergence */
static int gs_bicgstab(const orc_driver* d, double dt, const double* w, const double* b, double* x,
                       double* ws) {
    const int m = 2 * d->p.nx * d->p.nx;
    double *r = ws, *r0 = r + m, *p = r0 + m, *v = p + m, *s = v + m, *t = s + m, *y = t + m,
           *z = y + m, *dg = z + m;
    gs_jac(d, dt, w, NULL, NULL, dg);
    for (int i = 0; i < m; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
        r0[i] = b[i];
        p[i] = v[i] = 0.0;
    }
    const double bb = gs_dot(m, b, b);
    const double tol2 = d->p.gs_linear_tol * d->p.gs_linear_tol * bb;
    double rr = gs_dot(m, r, r);
    if (rr <= tol2) return 0;
    double r0n = rr, rho = 1.0, alpha = 1.0, om = 1.0;
    const double eps2 = DBL_EPSILON * DBL_EPSILON;  /* Eigen BiCGSTAB: NumTraits<double>::epsilon()^2 */
    int it = 0, restarts = 0;
    const int maxit = 2 * m;
    while (rr > tol2 && it < maxit) {
        const double rho_old = rho;
        rho = gs_dot(m, r0, r);
        if (fabs(rho) < eps2 * r0n) {
            for (int i = 0; i < m; ++i) r0[i] = r[i];
            rho = r0n = gs_dot(m, r, r);
            if (restarts++ == 0) it = 0;
        }
        const double beta = (rho / rho_old) * (alpha / om);
        for (int i = 0; i < m; ++i) p[i] = r[i] + beta * (p[i] - om * v[i]);
        for (int i = 0; i < m; ++i) y[i] = p[i] / dg[i];
        gs_jac(d, dt, w, y, v, NULL);
        alpha = rho / gs_dot(m, r0, v);
        for (int i = 0; i < m; ++i) s[i] = r[i] - alpha * v[i];
        for (int i = 0; i < m; ++i) z[i] = s[i] / dg[i];
        gs_jac(d, dt, w, z, t, NULL);
        const double tt = gs_dot(m, t, t);
        om = tt > 0.0 ? gs_dot(m, t, s) / tt : 0.0;
        for (int i = 0; i < m; ++i) x[i] += alpha * y[i] + om * z[i];
        for (int i = 0; i < m; ++i) r[i] = s[i] - om * t[i];
        rr = gs_dot(m, r, r);
        ++it;
    }
    return rr <= tol2 ? 0 : 1;
}

/* backward_euler_solve (gray_scott.cpp:91-172) + step's bounds check (:174-190) */
static int gs_step(orc_driver* d, int level, const double* in, double* out) {
    const int m = 2 * d->p.nx * d->p.nx;
    /* own scratch: callers hand step() output slots inside d->work */
    double* f = d->gs_work;
    double* res = f + m;
    double* delta = res + m;
    double* prev = delta + m;
    double* ws = prev + m;
    if (out != in) memcpy(out, in, sizeof(double) * (size_t)m);
    for (int s = 1; s <= d->sub[level]; ++s) {
        const double dt = d->sdt[level];
        memcpy(prev, out, sizeof(double) * (size_t)m);
        gs_rhs(d, out, f);
        for (int i = 0; i < m; ++i) res[i] = out[i] - prev[i] - dt * f[i];
        const double norm0 = sqrt(gs_dot(m, res, res));
        const double stop = fmax(d->p.newton_tol, d->p.newton_tol * norm0);
        if (norm0 <= stop) continue;
        int ok = 0;
        for (int it = 0; it < d->p.newton_max; ++it) {
            if (gs_bicgstab(d, dt, out, res, delta, ws) != 0) {
                d->newton_fail = 1;
                return fail(d, ORC_NONLINEAR, "gray-scott: inner linear solve failed (dt = %g)", dt);
            }
            for (int i = 0; i < m; ++i) out[i] -= delta[i];
            gs_rhs(d, out, f);
            for (int i = 0; i < m; ++i) res[i] = out[i] - prev[i] - dt * f[i];
            if (sqrt(gs_dot(m, res, res)) <= stop) {
                ok = 1;
                break;
            }
        }
        if (!ok) {
            d->newton_fail = 1;
            return fail(d, ORC_NONLINEAR, "gray-scott: Newton did not reach %g within %d iterations",
                        d->p.newton_tol, d->p.newton_max);
        }
    }
    if (d->p.gs_bounds_check)
        for (int i = 0; i < m; ++i)
            if (!(out[i] >= d->p.gs_bound_lo && out[i] <= d->p.gs_bound_hi))
                return fail(d, ORC_NONLINEAR, "gray-scott: concentration left the bounding box");
    return ORC_OK;
}

/* initial_condition (gray_scott.cpp:38-61): u = 1, v = 0 plus a bump */
static void gs_initial(const orc_driver* d, double* w) {
    const int n = d->p.nx, cells = n * n;
    const double h = d->p.gs_domain / n;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const int c = i * n + j;
            const double x = (j + 0.5) * h, y = (i + 0.5) * h;
            double u = 1.0, v = 0.0;
            if (x >= 1.0 && x <= 1.5 && y >= 1.0 && y <= 1.5) {
                const double sx = sin(4.0 * kPi * x), sy = sin(4.0 * kPi * y);
                const double bump = 0.25 * sx * sx * sy * sy;
                u = 1.0 - 2.0 * bump;
                v = bump;
            }
            w[c] = u;
            w[cells + c] = v;
        }
}

/* ------------------------------------------------------------------------ */
/* Application::step / forcing / initial_condition                          */

static double dahl_mult(const orc_driver* d, int level) {
    /* dahlquist.hpp:36-42 */
    const double h = d->dt[level] / d->sub[level];
    const double m = 1.0 / (1.0 - d->p.lambda * h);
    double out = m;
    for (int s = 1; s < d->sub[level]; ++s) out *= m;
    return out;
}

int orc_step(orc_driver* d, int level, int index, const double* in, double* out) {
    switch (d->p.kind) {
        case ORC_HEAT1D:  /* heat1d.cpp:93-95 */
            heat_propagate(d, level, index, in, out, d->p.folded);
            return ORC_OK;
        case ORC_DAHLQUIST:  /* dahlquist.hpp:25-30 */
            out[0] = dahl_mult(d, level) * in[0];
            return ORC_OK;
        case ORC_SCALAR: {  /* tests/support.hpp:35-41 */
            double v = d->p.mult[level] * in[0];
            if (d->p.folded && level == 0 && d->ff) v += d->ff[index];
            out[0] = v;
            return ORC_OK;
        }
        case ORC_ALLEN_CAHN:
            return ac_step(d, level, in, out);
        case ORC_HEAT2D:
            return h2_propagate(d, level, in, out, d->p.folded);
        case ORC_GRAY_SCOTT:
            return gs_step(d, level, in, out);
    }
    return fail(d, ORC_CONFIG, "unknown problem kind");
}

int orc_forcing(orc_driver* d, int level, int index, double* out) {
    const int n = d->n;
    switch (d->p.kind) {
        case ORC_HEAT1D: {  /* heat1d.cpp:97-100: propagate(zero, with forcing) */
            memset(out, 0, sizeof(double) * (size_t)n);
            heat_propagate(d, level, index, out, out, 1);
            return ORC_OK;
        }
        case ORC_SCALAR:  /* tests/support.hpp:43-49 */
            out[0] = (!d->p.folded && level == 0 && d->ff) ? d->ff[index] : 0.0;
            return ORC_OK;
        case ORC_HEAT2D:
            memset(out, 0, sizeof(double) * (size_t)n);
            return h2_propagate(d, level, out, out, 1);
        default:  /* application.hpp:42-47 default: zeros */
            memset(out, 0, sizeof(double) * (size_t)n);
            return ORC_OK;
    }
}

void orc_initial_condition(orc_driver* d, double* out) {
    memcpy(out, d->ic, sizeof(double) * (size_t)d->n);
}

/* ------------------------------------------------------------------------ */
/* creation: hierarchy + configure + validate                                */

orc_driver* orc_create(const orc_problem* p, const orc_grid* g, const orc_solver* s,
                       int* status) {
    *status = ORC_CONFIG;
    /* time_grid.hpp:14-23 */
    if (g->n_points < 2) { fail(NULL, 2, "TimeGrid: need at least 2 points"); return NULL; }
    if (!(g->tf > g->t0)) { fail(NULL, 2, "TimeGrid: tf must exceed t0"); return NULL; }
    /* hierarchy.cpp:24-50 */
    if (g->n_m < 1 || g->n_m >= ORC_MAXL) {
        fail(NULL, 2, "hierarchy needs at least one coarsening factor");
        return NULL;
    }
    if (g->k < 1) { fail(NULL, 2, "local-grid distance k must be at least 1"); return NULL; }
    {
        int np = g->n_points;
        for (int l = 0; l < g->n_m; ++l) {
            if (g->m[l] < 2) {
                fail(NULL, 2, "coarsening factor must exceed 1, got %d", g->m[l]);
                return NULL;
            }
            const int nc = (np - 1) / g->m[l] + 1;
            if (nc < 2) {
                fail(NULL, 2, "coarsening exhausts the grid at level %d (%d points)", l + 1, nc);
                return NULL;
            }
            np = nc;
        }
    }
    if (s->coarse_substeps < 1) {
        fail(NULL, 2, "coarse_substeps must be at least 1");
        return NULL;
    }

    orc_driver* d = (orc_driver*)calloc(1, sizeof(orc_driver));
    d->p = *p;
    d->g = *g;
    d->s = *s;
    d->L = g->n_m + 1;
    const int scalar = (p->kind == ORC_DAHLQUIST || p->kind == ORC_SCALAR);
    d->n = scalar ? 1 : (p->kind == ORC_HEAT2D ? p->nx * p->nx
                         : p->kind == ORC_GRAY_SCOTT ? 2 * p->nx * p->nx : p->n);
    const int n = d->n;
    if (n < 1) { fail(NULL, 2, "problem: need at least one spatial unknown"); free(d); return NULL; }

    /* make_level_specs, solver.cpp:30-43: sub-steps on the coarsest level only */
    for (int l = 0; l < d->L; ++l) {
        d->np[l] = orc_level_points(g, l);
        d->dt[l] = orc_level_dt(g, l);
        d->t0[l] = g->t0;
        d->sub[l] = (l == d->L - 1) ? s->coarse_substeps : 1;
        d->sdt[l] = d->dt[l] / d->sub[l];
    }

    d->ic = (double*)calloc((size_t)n, sizeof(double));
    d->work = (double*)calloc((size_t)n * 16, sizeof(double));
    if (p->kind == ORC_HEAT1D) {
        /* heat1d.cpp:13-22 mesh and sin profile; :24-45 factorization */
        if (!(p->x1 > p->x0)) { fail(NULL, 2, "heat1d: x1 must exceed x0"); orc_destroy(d); return NULL; }
        d->h = (p->x1 - p->x0) / (double)(n + 1);
        d->sinp = (double*)calloc((size_t)n, sizeof(double));
        for (int i = 0; i < n; ++i) d->sinp[i] = sin(kPi * (p->x0 + d->h * (i + 1)));
        for (int l = 0; l < d->L; ++l) {
            d->rr[l] = d->sdt[l] / (d->h * d->h);
            const double a = -d->rr[l];
            const double b = 1.0 + 2.0 * d->rr[l];
            d->cpr[l] = (double*)calloc((size_t)n, sizeof(double));
            d->inv[l] = (double*)calloc((size_t)n, sizeof(double));
            double prev_c = 0.0;
            for (int i = 0; i < n; ++i) {
                const double den = b - a * prev_c;
                d->inv[l][i] = 1.0 / den;
                prev_c = a / den;
                d->cpr[l][i] = prev_c;
            }
        }
        memcpy(d->ic, d->sinp, sizeof(double) * (size_t)n);  /* heat1d.cpp:85-91 */
    } else if (p->kind == ORC_DAHLQUIST) {
        d->ic[0] = p->u0;
    } else if (p->kind == ORC_SCALAR) {
        d->ic[0] = p->u0;
        if (p->fine_forcing && p->n_ff > 0) {
            d->ff = (double*)calloc((size_t)p->n_ff, sizeof(double));
            memcpy(d->ff, p->fine_forcing, sizeof(double) * (size_t)p->n_ff);
        }
        if (p->n_mult < d->L) { fail(NULL, 2, "scalar: one multiplier per level"); orc_destroy(d); return NULL; }
    } else if (p->kind == ORC_ALLEN_CAHN) {
        if (!(p->eps > 0.0) || !(p->length > 0.0)) { fail(NULL, 2, "allen-cahn: bad eps/length"); orc_destroy(d); return NULL; }
    } else if (p->kind == ORC_GRAY_SCOTT) {
        /* gray_scott.cpp:16-36 */
        if (p->nx < 4) { fail(NULL, 2, "gray-scott: grid must be at least 4x4"); orc_destroy(d); return NULL; }
        if (!(p->gs_domain > 0.0)) { fail(NULL, 2, "gray-scott: domain size must be positive"); orc_destroy(d); return NULL; }
        gs_initial(d, d->ic);
        d->gs_work = (double*)calloc((size_t)n * 13, sizeof(double));
    } else if (p->kind == ORC_HEAT2D) {
        if (p->source) {
            d->src = (double*)calloc((size_t)n, sizeof(double));
            memcpy(d->src, p->source, sizeof(double) * (size_t)n);
        }
    } else {
        fail(NULL, 2, "unknown problem kind %d", p->kind);
        orc_destroy(d);
        return NULL;
    }
    if (p->ic) memcpy(d->ic, p->ic, sizeof(double) * (size_t)n);
    d->p.ic = NULL;
    d->p.fine_forcing = NULL;
    d->p.source = NULL;

    /* copies of caller-owned solver inputs */
    if (s->functional_w) {
        d->fw = (double*)malloc(sizeof(double) * (size_t)n);
        memcpy(d->fw, s->functional_w, sizeof(double) * (size_t)n);
    }
    if (s->constant_value) {
        d->cval = (double*)malloc(sizeof(double) * (size_t)n);
        memcpy(d->cval, s->constant_value, sizeof(double) * (size_t)n);
    }
    if (s->provided) {
        const size_t cnt = (size_t)g->n_points * n;
        d->prov = (double*)malloc(sizeof(double) * cnt);
        memcpy(d->prov, s->provided, sizeof(double) * cnt);
    }
    d->s.functional_w = NULL;
    d->s.constant_value = NULL;
    d->s.provided = NULL;

    /* CycleDriver::validate, solver.cpp:51-79 */
    const int folded = (p->kind == ORC_DAHLQUIST || p->kind == ORC_SCALAR ||
                        p->kind == ORC_HEAT1D || p->kind == ORC_HEAT2D) ? p->folded : 1;
    d->p.folded = folded;
    int st = ORC_OK;
    if (!(s->tol > 0.0)) st = fail(NULL, 2, "solver: tol must be positive");
    else if (s->max_iters < 1) st = fail(NULL, 2, "solver: max_iters must be at least 1");
    else if (s->relaxation == ORC_RELAX_FCF && s->nu < 1) st = fail(NULL, 2, "solver: FCF relaxation needs nu >= 1");
    else if (s->mode == ORC_TWO_LEVEL && d->L != 2) st = fail(NULL, 2, "two-level mode needs a two-level hierarchy");
    else if (s->mode == ORC_TWO_LEVEL && folded) st = fail(NULL, 2, "two-level residual-correction mode needs explicit forcing");
    else if (s->mode != ORC_TWO_LEVEL && !folded) st = fail(NULL, 2, "FAS cycles need forcing folded into the integrator");
    else if (s->norm == ORC_NORM_FUNCTIONAL && !d->fw) st = fail(NULL, 2, "functional-change stopping norm needs a functional");
    else if (s->initial_guess == ORC_GUESS_PROVIDED && !d->prov) st = fail(NULL, 2, "provided initial guess has the wrong number of points");
    if (st) { orc_destroy(d); return NULL; }
    *status = ORC_OK;
    return d;
}

void orc_destroy(orc_driver* d) {
    if (!d) return;
    free(d->sinp);
    for (int l = 0; l < ORC_MAXL; ++l) {
        free(d->cpr[l]); free(d->inv[l]);
        free(d->u[l]); free(d->gg[l]); free(d->v[l]); free(d->r[l]);
    }
    free(d->work); free(d->gs_work); free(d->ic); free(d->ff); free(d->fw); free(d->cval); free(d->prov);
    free(d->src); free(d->rs); free(d->prevf);
    free(d);
}

int orc_n_levels(const orc_driver* d) { return d->L; }
int orc_vector_size(const orc_driver* d) { return d->n; }

double* orc_array(orc_driver* d, int level, int which) {
    if (level < 0 || level >= d->L) return NULL;
    switch (which) {
        case 0: return d->u[level];
        case 1: return d->gg[level];
        case 2: return d->v[level];
        case 3: return d->r[level];
        case 4: return level == 0 ? d->rs : NULL;
    }
    return NULL;
}

/* ------------------------------------------------------------------------ */
/* kernels.cpp restatements                                                  */

/* kernels.cpp:7-17: u_i = Phi_i(u_{i-1}) + g_i over each F-interval */
int orc_k_f_relax(orc_driver* d, int level, int first_interval, int count) {
    const int n = d->n, m = d->g.m[level], last = d->np[level] - 1;
    for (int j = first_interval; j < first_interval + count; ++j) {
        const int c = j * m;
        const int stop = c + m - 1 < last ? c + m - 1 : last;
        for (int i = c + 1; i <= stop; ++i) {
            double* ui = vec(d, level, 0, i);
            const int st = orc_step(d, level, i, vec(d, level, 0, i - 1), ui);
            if (st) return st;
            const double* gi = vec(d, level, 1, i);
            for (int q = 0; q < n; ++q) ui[q] += gi[q];
        }
    }
    return ORC_OK;
}

/* kernels.cpp:19-28: C-points c > 0 from the preceding F-point */
int orc_k_c_relax(orc_driver* d, int level, int first_c, int count) {
    const int n = d->n, m = d->g.m[level];
    for (int j = first_c; j < first_c + count; ++j) {
        const int c = j * m;
        if (c == 0) continue;
        double* uc = vec(d, level, 0, c);
        const int st = orc_step(d, level, c, vec(d, level, 0, c - 1), uc);
        if (st) return st;
        const double* gc = vec(d, level, 1, c);
        for (int q = 0; q < n; ++q) uc[q] += gc[q];
    }
    return ORC_OK;
}

/* solver.cpp:174-185 / kernels.cpp:30-43 */
static int residual_at(orc_driver* d, int level, int i, double* r) {
    const int n = d->n;
    const double* ui = vec(d, level, 0, i);
    const double* gi = vec(d, level, 1, i);
    if (i == 0) {
        for (int q = 0; q < n; ++q) r[q] = gi[q] - ui[q];
        return ORC_OK;
    }
    const int st = orc_step(d, level, i, vec(d, level, 0, i - 1), r);
    if (st) return st;
    for (int q = 0; q < n; ++q) r[q] += gi[q];
    for (int q = 0; q < n; ++q) r[q] -= ui[q];
    return ORC_OK;
}

int orc_k_residual(orc_driver* d, int level, int first, int count, double* r_out) {
    for (int i = first; i < first + count; ++i) {
        const int st = residual_at(d, level, i, r_out + (size_t)(i - first) * d->n);
        if (st) return st;
    }
    return ORC_OK;
}

/* kernels.cpp:53-61 */
int orc_k_window_linear(orc_driver* d, int level, int lo, int size, const double* r_win,
                        double* out) {
    const int n = d->n;
    memcpy(out, r_win, sizeof(double) * (size_t)n);
    for (int s = 1; s < size; ++s) {
        const int st = orc_step(d, level, lo + s, out, out);
        if (st) return st;
        const double* rs = r_win + (size_t)s * n;
        for (int q = 0; q < n; ++q) out[q] += rs[q];
    }
    return ORC_OK;
}

/* kernels.cpp:63-77 */
int orc_k_window_fas(orc_driver* d, int level, int lo, int size, const double* v_win,
                     const double* r_win, double* out) {
    const int n = d->n;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
    for (int q = 0; q < n; ++q) out[q] = v_win[q] + r_win[q];
    for (int s = 1; s < size; ++s) {
        int st = orc_step(d, level, lo + s, out, out);
        if (!st) st = orc_step(d, level, lo + s, v_win + (size_t)(s - 1) * n, tmp);
        if (st) { free(tmp); return st; }
        const double* vs = v_win + (size_t)s * n;
        const double* rs = r_win + (size_t)s * n;
        for (int q = 0; q < n; ++q) out[q] += vs[q];
        for (int q = 0; q < n; ++q) out[q] -= tmp[q];
        for (int q = 0; q < n; ++q) out[q] += rs[q];
    }
    free(tmp);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* CycleDriver restatement (solver.cpp)                                      */

static void fill_level_rhs(orc_driver* d, int level) {
    /* solver.cpp:136-150 */
    const int n = d->n;
    for (int i = 0; i < d->np[level]; ++i) {
        double* gi = vec(d, level, 1, i);
        if (i == 0) memcpy(gi, d->ic, sizeof(double) * (size_t)n);
        else if (d->p.folded) memset(gi, 0, sizeof(double) * (size_t)n);
        else orc_forcing(d, level, i, gi);
    }
}

static double functional(const orc_driver* d, const double* u) {
    double s = 0.0;
    for (int q = 0; q < d->n; ++q) s += d->fw[q] * u[q];
    return s;
}

int orc_setup(orc_driver* d) {
    /* solver.cpp:81-109 */
    if (d->setup_done) return ORC_OK;
    const int n = d->n;
    for (int l = 0; l < d->L; ++l) {
        const size_t cnt = (size_t)d->np[l] * n;
        d->u[l] = (double*)calloc(cnt, sizeof(double));
        d->gg[l] = (double*)calloc(cnt, sizeof(double));
        if (l >= 1) {
            d->v[l] = (double*)calloc(cnt, sizeof(double));
            d->r[l] = (double*)calloc(cnt, sizeof(double));
        }
    }
    d->rs = (double*)calloc((size_t)d->np[0] * n, sizeof(double));
    /* fill_initial_guess, solver.cpp:111-134 */
    for (int i = 0; i < d->np[0]; ++i) {
        double* ui = vec(d, 0, 0, i);
        if (i == 0) { memcpy(ui, d->ic, sizeof(double) * (size_t)n); continue; }
        switch (d->s.initial_guess) {
            case ORC_GUESS_CONSTANT:
                memcpy(ui, d->cval ? d->cval : d->ic, sizeof(double) * (size_t)n);
                break;
            case ORC_GUESS_RANDOM:
                orc_random_state(d->s.seed + (uint64_t)i, n, ui);
                break;
            case ORC_GUESS_PROVIDED:
                memcpy(ui, d->prov + (size_t)i * n, sizeof(double) * (size_t)n);
                break;
        }
    }
    fill_level_rhs(d, 0);
    if (d->s.norm == ORC_NORM_FUNCTIONAL) {
        const int nc = cpoints(d, 0);
        d->prevf = (double*)calloc((size_t)nc, sizeof(double));
        for (int j = 0; j < nc; ++j) d->prevf[j] = functional(d, vec(d, 0, 0, j * d->g.m[0]));
    }
    d->setup_done = 1;
    return ORC_OK;
}

static int relax_level(orc_driver* d, int level) {
    /* solver.cpp:160-172 */
    int st = orc_k_f_relax(d, level, 0, n_intervals(d, level));
    if (st) return st;
    if (d->s.relaxation == ORC_RELAX_FCF) {
        for (int s = 0; s < d->s.nu; ++s) {
            st = orc_k_c_relax(d, level, 0, cpoints(d, level));
            if (!st) st = orc_k_f_relax(d, level, 0, n_intervals(d, level));
            if (st) return st;
        }
    }
    return ORC_OK;
}

static int restrict_to(orc_driver* d, int level) {
    /* solver.cpp:194-222 */
    const int n = d->n, m = d->g.m[level], nc = cpoints(d, level);
    const int relaxed = (level + 1) != d->L - 1;
    for (int j = 0; j < nc; ++j) {
        const double* uc = vec(d, level, 0, j * m);
        memcpy(vec(d, level + 1, 0, j), uc, sizeof(double) * (size_t)n);
        memcpy(vec(d, level + 1, 2, j), uc, sizeof(double) * (size_t)n);
        int st = residual_at(d, level, j * m, vec(d, level + 1, 3, j));
        if (st) return st;
        if (relaxed) {
            double* gj = vec(d, level + 1, 1, j);
            const double* vj = vec(d, level + 1, 2, j);
            const double* rj = vec(d, level + 1, 3, j);
            if (j == 0) {
                for (int q = 0; q < n; ++q) gj[q] = vj[q] + rj[q];
            } else {
                double* tmp = d->work + 6 * (size_t)n;
                st = orc_step(d, level + 1, j, vec(d, level, 0, (j - 1) * m), tmp);
                if (st) return st;
                for (int q = 0; q < n; ++q) gj[q] = vj[q] - tmp[q];
                for (int q = 0; q < n; ++q) gj[q] += rj[q];
            }
        }
    }
    return ORC_OK;
}

static int coarsest_fas(orc_driver* d) {
    /* solver.cpp:224-252 (sequential exchange returns every payload) */
    const int lc = d->L - 1, n = d->n, k = d->g.k;
    const int np = d->np[lc];
    for (int p = 0; p < np; ++p) {
        const int lo = p - k + 1 > 0 ? p - k + 1 : 0;
        const int st = orc_k_window_fas(d, lc, lo, p - lo + 1, vec(d, lc, 2, lo),
                                        vec(d, lc, 3, lo), vec(d, lc, 0, p));
        if (st) return st;
    }
    (void)n;
    return ORC_OK;
}

static int coarsest_linear(orc_driver* d) {
    /* solver.cpp:254-279 */
    const int n = d->n, k = d->g.k, m = d->g.m[0];
    const int np = d->np[1];
    double* e = d->work + 7 * (size_t)n;
    for (int p = 0; p < np; ++p) {
        const int lo = p - k + 1 > 0 ? p - k + 1 : 0;
        const int st = orc_k_window_linear(d, 1, lo, p - lo + 1, vec(d, 1, 3, lo), e);
        if (st) return st;
        double* uc = vec(d, 0, 0, p * m);
        for (int q = 0; q < n; ++q) uc[q] += e[q];
    }
    return ORC_OK;
}

static int correct_from(orc_driver* d, int level) {
    /* solver.cpp:281-292 */
    const int n = d->n, m = d->g.m[level], nc = cpoints(d, level);
    for (int j = 0; j < nc; ++j) {
        double* uc = vec(d, level, 0, j * m);
        const double* cu = vec(d, level + 1, 0, j);
        const double* cv = vec(d, level + 1, 2, j);
        for (int q = 0; q < n; ++q) uc[q] += cu[q] - cv[q];
    }
    return orc_k_f_relax(d, level, 0, n_intervals(d, level));
}

static int v_cycle(orc_driver* d, int level) {
    /* solver.cpp:294-303 */
    if (level == d->L - 1) return coarsest_fas(d);
    int st = relax_level(d, level);
    if (!st) st = restrict_to(d, level);
    if (!st) st = v_cycle(d, level + 1);
    if (!st) st = correct_from(d, level);
    return st;
}

static int two_level_cycle(orc_driver* d) {
    /* solver.cpp:305-320 */
    int st = relax_level(d, 0);
    if (st) return st;
    const int m = d->g.m[0], nc = cpoints(d, 0);
    for (int j = 0; j < nc; ++j) {
        st = residual_at(d, 0, j * m, vec(d, 1, 3, j));
        if (st) return st;
    }
    st = coarsest_linear(d);
    if (st) return st;
    return orc_k_f_relax(d, 0, 0, n_intervals(d, 0));
}

int orc_cycle(orc_driver* d) {
    /* solver.cpp:322-329 */
    orc_setup(d);
    return d->s.mode == ORC_TWO_LEVEL ? two_level_cycle(d) : v_cycle(d, 0);
}

int orc_nested_init(orc_driver* d) {
    /* solver.cpp:331-368 */
    const int lc = d->L - 1, n = d->n, k = d->g.k;
    orc_setup(d);
    for (int l = 0; l < lc; ++l) {
        const int m = d->g.m[l], nc = cpoints(d, l);
        for (int j = 0; j < nc; ++j)
            memcpy(vec(d, l + 1, 0, j), vec(d, l, 0, j * m), sizeof(double) * (size_t)n);
        fill_level_rhs(d, l + 1);
    }
    const int np = d->np[lc];
    if (k >= np) {
        /* solver.cpp:466-473 chain_forward */
        for (int i = 1; i < np; ++i) {
            double* ui = vec(d, lc, 0, i);
            const int st = orc_step(d, lc, i, vec(d, lc, 0, i - 1), ui);
            if (st) return st;
            const double* gi = vec(d, lc, 1, i);
            for (int q = 0; q < n; ++q) ui[q] += gi[q];
        }
    } else {
        /* windows start from the exchanged (pre-update) values, kernels.cpp:79-88 */
        double* snap = (double*)malloc(sizeof(double) * (size_t)np * n);
        memcpy(snap, d->u[lc], sizeof(double) * (size_t)np * n);
        for (int p = 0; p < np; ++p) {
            const int lo = p - k + 1 > 0 ? p - k + 1 : 0;
            double* up = vec(d, lc, 0, p);
            memcpy(up, snap + (size_t)lo * n, sizeof(double) * (size_t)n);
            for (int s = 1; s < p - lo + 1; ++s) {
                const int st = orc_step(d, lc, lo + s, up, up);
                if (st) { free(snap); return st; }
            }
        }
        free(snap);
    }
    for (int l = lc - 1; l >= 0; --l) {
        const int m = d->g.m[l], nc = cpoints(d, l);
        for (int j = 0; j < nc; ++j)
            memcpy(vec(d, l, 0, j * m), vec(d, l + 1, 0, j), sizeof(double) * (size_t)n);
        int st = orc_k_f_relax(d, l, 0, n_intervals(d, l));
        if (!st && l >= 1) st = v_cycle(d, l);
        if (st) return st;
    }
    return ORC_OK;
}

int orc_residual_norm(orc_driver* d, double* out) {
    /* solver.cpp:370-378 + kernels.cpp:90-101: per-point squares summed in order */
    orc_setup(d);
    const int n = d->n;
    double total = 0.0;
    for (int i = 0; i < d->np[0]; ++i) {
        double* ri = d->rs + (size_t)i * n;
        const int st = residual_at(d, 0, i, ri);
        if (st) return st;
        double sq = 0.0;
        for (int q = 0; q < n; ++q) sq += ri[q] * ri[q];
        total += sq;
    }
    *out = sqrt(total);
    return ORC_OK;
}

static int stopping_norm(orc_driver* d, double* out) {
    /* solver.cpp:380-396 */
    if (d->s.norm == ORC_NORM_L2) return orc_residual_norm(d, out);
    const int m = d->g.m[0], nc = cpoints(d, 0);
    double local_max = 0.0;
    for (int j = 0; j < nc; ++j) {
        const double val = functional(d, vec(d, 0, 0, j * m));
        const double prev = d->prevf[j];
        const double denom = fabs(prev) > 1e-300 ? fabs(prev) : 1e-300;
        const double rel = fabs(val - prev) / denom;
        local_max = local_max > rel ? local_max : rel;
        d->prevf[j] = val;
    }
    *out = local_max;
    return ORC_OK;
}

int orc_drive(orc_driver* d, double* history, int* iterations, int* converged) {
    /* solver.cpp:398-435 */
    *iterations = 0;
    *converged = 0;
    int st = orc_setup(d);
    if (!st && d->s.mode == ORC_NESTED_V) st = orc_nested_init(d);
    if (st) return st;
    for (int it = 1; it <= d->s.max_iters; ++it) {
        st = orc_cycle(d);
        double norm = 0.0;
        if (!st) st = stopping_norm(d, &norm);
        if (st) return st;
        history[it - 1] = norm;
        *iterations = it;
        if (!isfinite(norm))
            return fail(d, ORC_DIVERGED, "non-finite residual norm at iteration %d", it);
        if (norm <= d->s.tol) {
            *converged = 1;
            return ORC_OK;
        }
    }
    return ORC_NOT_CONVERGED;
}
