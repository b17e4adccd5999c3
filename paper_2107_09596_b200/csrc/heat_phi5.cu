// heat_phi5.cu -- 1D row Phi chains for sm_100a: Heat1D and Allen-Cahn.
//
// One CTA owns one state vector (a time point) in registers, blocked
// (thread t holds elements [t*L, t*L+L); L = 32 / 128 threads for the level-0
// sweeps of 2048 < n <= 4096, L <= 16 otherwise).  Rows move HBM -> smem by
// TMA (cp.async.bulk.tensor, 128B-swizzled so the blocked register view reads
// and writes smem conflict-free); produced rows leave by per-warp TMA stores
// of 1024-byte-aligned slices, so a stored row needs no CTA barrier and the
// stores overlap the next Phi.
//
// One Phi sub-step solves (I + sub_dt L) x = b, T = tridiag(a, b0, a) with
// a = -r, b0 = 1 + 2r (heat1d.cpp:24-60).  With (c*, d*) the fixed point of
// the Thomas recurrence, T = L_c U_c + delta e0 e0^T (delta = a c*), so
//     x = M^{-1} b - sigma x0 w,   M = L_c U_c, w = M^{-1} e0, x0 = (M^{-1} b)_0
// (Sherman-Morrison).  Every thread runs the constant-coefficient recurrences
// from registers.  On every chunk w lies in span{q, p_b}, the two vectors the
// blocked solve combines anyway, so the correction is two extra terms in the
// chunk's carry coefficients (only in the first `ncw` warps, where w is not
// negligible).  The periodic (Allen-Cahn) matrix adds the corner entries: a
// rank-2 Woodbury term with the right-end vector folded the same way.  (In
// fp64 this is more accurate than the serial Thomas sweep with its
// non-converged leading factors; see tests/test_gpu_parity.py.)
//
// M^{-1} b is evaluated with ONE CTA barrier:
//   1. forward local pass      y_loc = L^{-1} b on the chunk (zero carry-in)
//   2. forward warp scan of the chunk ends -> E (exclusive), warp total Tf
//   3. backward local pass     z_loc = U^{-1} y_loc   (the forward carry c_f
//      enters linearly as c_f q with q = U^{-1} p_f, precomputed)
//   4. backward warp scan of a = z_loc[0] + E q0 -> RA, warp total TA
//   5. publish (Tf, TA and the correction pick-ups), bar.sync, cross-warp
//      carries as fixed weighted sums (lane-parallel + xor tree)
//   6. x = z_loc + c_f q + c_b p_b (c_f, c_b include the correction)
// All multipliers are precomputed on the host (heat_level_host).
//
// Proxy rule: a buffer filled by TMA and read with ld.shared is handed back
// to TMA only after fence.proxy.async + bar.sync (write-after-read across
// the generic and async proxies).
//
// Reference semantics restated (file:line under /root/reference/proj):
//   Phi / step          heat1d.cpp:47-60 (Thomas), :66-83 (sub-steps, forcing)
//   F-relaxation        kernels.cpp:7-17      -> SW_F jobs
//   C-relaxation        kernels.cpp:19-28     -> SW_CRELAX jobs / fused SW_FCF
//   residual / restrict kernels.cpp:30-43, solver.cpp:174-185 -> tails, SW_RESID
//   window solves       kernels.cpp:53-88     -> heat_window_*_kernel
//   point squares       kernels.cpp:90-95     -> TAIL_SQ (fixed-order tree)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

#include "heat_kernels.cuh"
#include "tma.cuh"

namespace atm {

namespace cg = cooperative_groups;

// --------------------------------------------------------------------------
// host: fixed-point factors, correction vectors and every scan multiplier

HeatLevelHost heat_level_host(int n, int pitch, int L, double r_in, double shift, int substeps,
                              bool cyclic) {
    using LD = long double;
    HeatLevelHost H;
    H.n = n;
    H.pitch = pitch;
    H.L = L;
    H.substeps = substeps;
    H.cyclic = cyclic ? 1 : 0;
    const int nt = ((pitch + L - 1) / L + 127) / 128 * 128;
    H.nt = nt;
    const int npad = nt * L;
    // heat1d.cpp:28-31: r = sub_dt/h^2, a = -r, b = 1 + 2r (+ shift: the
    // Allen-Cahn linear part 1 + 2r - dt + s)
    H.r = r_in;
    const LD r = static_cast<LD>(H.r);
    const LD a = -r, b = 1.0L + 2.0L * r + static_cast<LD>(shift);
    // fixed point of c = a / (b - a c): the root of a c^2 - b c + a with |c| < 1
    const LD disc = (shift == 0.0) ? 1.0L + 4.0L * r : b * b - 4.0L * r * r;
    const LD c = 2.0L * a / (b + std::sqrt(disc));
    const LD d = b - a * c;
    H.beta_c = static_cast<double>(1.0L / d);
    H.gamma_c = static_cast<double>(r / d);
    H.cneg_c = static_cast<double>(-c);
    // correction vectors: wl = M^{-1} e0 (L_c: d* diag, a sub; U_c: 1 diag,
    // c* super), yf its forward (L_c^{-1}) values = the carries into every
    // chunk; cyclic: wr = M^{-1} e_{n-1} = (-c)^{n-1-i} / d
    std::vector<LD> w(n), yf(n), wr(n, 0.0L);
    {
        LD p = 0.0L;
        for (int i = 0; i < n; ++i) {
            p = ((i == 0 ? 1.0L : 0.0L) - a * p) / d;
            yf[i] = w[i] = p;
        }
        for (int i = n - 2; i >= 0; --i) w[i] -= c * w[i + 1];
        if (cyclic) {
            LD q = 1.0L / d;
            for (int i = n - 1; i >= 0; --i) {
                wr[i] = q;
                q *= -c;
            }
        }
    }
    H.w0 = w[0];
    H.wn = w[n - 1];
    H.wr0 = wr[0];
    H.wrn = wr[n - 1];
    // Woodbury: T = M + U C U^T, U = [e0, e_{n-1}], C = [[delta, a], [a, 0]]
    // (cyclic) or U = e0, C = delta; T^{-1} b = M^{-1} b - W S U^T M^{-1} b,
    // S = (C^{-1} + U^T W)^{-1}
    const LD delta = a * c;
    H.sigma = static_cast<double>(delta / (1.0L + delta * w[0]));
    H.S[0] = H.sigma;
    H.S[1] = H.S[2] = H.S[3] = 0.0;
    if (cyclic) {
        const LD m00 = w[0], m01 = 1.0L / a + wr[0];
        const LD m10 = 1.0L / a + w[n - 1], m11 = -delta / (a * a) + wr[n - 1];
        const LD det = m00 * m11 - m01 * m10;
        H.S[0] = static_cast<double>(m11 / det);
        H.S[1] = static_cast<double>(-m01 / det);
        H.S[2] = static_cast<double>(-m10 / det);
        H.S[3] = static_cast<double>(m00 / det);
    }
    LD wmax = 0.0L, wrmax = 0.0L;
    for (int i = 0; i < n; ++i) {
        wmax = std::max(wmax, std::fabs(w[i]));
        wrmax = std::max(wrmax, std::fabs(wr[i]));
    }
    int K = 0, KR = n;  // below 1e-20 of the peak past K (wl) and before KR (wr)
    for (int i = 0; i < n; ++i)
        if (std::fabs(w[i]) > 1e-20L * wmax) K = i + 1;
    if (cyclic)
        for (int i = n - 1; i >= 0; --i)
            if (std::fabs(wr[i]) > 1e-20L * wrmax) KR = i;
    H.ncw = (K + 32 * L - 1) / (32 * L);
    H.ncw_r0 = cyclic ? KR / (32 * L) : kMaxWarps;
    // effective per-element coefficients; padding elements (>= n) carry
    // gamma = 0 so no forward carry crosses them
    std::vector<double> eg(npad), ec(npad);
    for (int i = 0; i < npad; ++i) {
        eg[i] = i < n ? H.gamma_c : 0.0;
        ec[i] = H.cneg_c;
    }
    // per thread: p_f (forward carry influence), q = U^{-1} p_f, p_b
    std::vector<double> q(npad), pb(npad), Af(nt), Ab(nt), q0(nt);
    for (int t = 0; t < nt; ++t) {
        std::vector<double> pf(L);
        double p = 1.0;
        for (int e = 0; e < L; ++e) {
            p *= eg[t * L + e];
            pf[e] = p;
        }
        Af[t] = p;
        double z = 0.0;
        for (int e = L - 1; e >= 0; --e) {
            z = ec[t * L + e] * z + pf[e];
            q[t * L + e] = z;
        }
        q0[t] = q[t * L];
        p = 1.0;
        for (int e = L - 1; e >= 0; --e) {
            p *= ec[t * L + e];
            pb[t * L + e] = p;
        }
        Ab[t] = p;
    }
    // interior-thread vectors (constant coefficients, no padding), and q of
    // the thread holding element n-1
    H.powc.assign(3 * kMaxL, 0.0);
    {
        std::vector<double> pf(L);
        double p = 1.0;
        for (int e = 0; e < L; ++e) {
            p *= H.gamma_c;
            pf[e] = p;
        }
        double z = 0.0;
        for (int e = L - 1; e >= 0; --e) {
            z = H.cneg_c * z + pf[e];
            H.powc[e] = z;
        }
        p = 1.0;
        for (int e = L - 1; e >= 0; --e) {
            p *= H.cneg_c;
            H.powc[kMaxL + e] = p;
        }
        const int tl = (n - 1) / L;
        for (int e = 0; e < L; ++e) H.powc[2 * kMaxL + e] = q[tl * L + e];
    }
    // warp scans (Hillis-Steele; 0 where a lane has no partner)
    H.scan.assign(static_cast<size_t>(nt) * kScanPerThread, 0.0);
    const int nw = nt / 32;
    std::vector<double> AWf(nw), AWb(nw), TB(nw);
    for (int wi = 0; wi < nw; ++wi) {
        double pf = 1.0, pbw = 1.0;
        for (int l = 0; l < 32; ++l) pf *= Af[32 * wi + l];
        for (int l = 31; l >= 0; --l) pbw *= Ab[32 * wi + l];
        AWf[wi] = pf;
        AWb[wi] = pbw;
        std::vector<double> Pfex(32), RB(33, 0.0);
        for (int l = 0; l < 32; ++l) {
            double ex = 1.0;
            for (int u = 0; u < l; ++u) ex *= Af[32 * wi + u];
            Pfex[l] = ex;
        }
        // backward inclusive-from-the-right recurrence of b = Pfex * q0
        for (int l = 31; l >= 0; --l)
            RB[l] = Pfex[l] * q0[32 * wi + l] + Ab[32 * wi + l] * RB[l + 1];
        TB[wi] = RB[0];
        for (int l = 0; l < 32; ++l) {
            double* sc = &H.scan[static_cast<size_t>(32 * wi + l) * kScanPerThread];
            for (int dd = 0; dd < 5; ++dd) {
                const int off = 1 << dd;
                double mf = 0.0, mb = 0.0;
                if (l >= off) {
                    mf = 1.0;
                    for (int u = l - off + 1; u <= l; ++u) mf *= Af[32 * wi + u];
                }
                if (l + off <= 31) {
                    mb = 1.0;
                    for (int u = l; u <= l + off - 1; ++u) mb *= Ab[32 * wi + u];
                }
                sc[dd] = mf;
                sc[6 + dd] = mb;
            }
            sc[5] = Pfex[l];
            double exb = 1.0;
            for (int u = l + 1; u <= 31; ++u) exb *= Ab[32 * wi + u];
            sc[11] = exb;
            sc[12] = RB[l + 1];      // SB: coefficient of C_w in c_b
            sc[13] = q0[32 * wi + l];
        }
    }
    // wl on chunk t is cfw_t q_t + cbw_t p_b: cfw_t = the forward carry into
    // the chunk (for t = 0 the local forward of e0 is beta gamma^e = (beta /
    // gamma) p_f = -p_f / a), cbw_t = wl at the first element of the next
    // chunk; wr on chunk t is cbwr_t p_b
    {
        LD err = 0.0L;
        const int tl = (n - 1) / L;
        const int pl = n - tl * L;
        for (int t = 0; t < nt && t * L < n; ++t) {
            const LD cf = (t == 0) ? -1.0L / a : yf[t * L - 1];
            const LD cb = ((t + 1) * L < n) ? w[(t + 1) * L] : 0.0L;
            const LD cbr = !cyclic ? 0.0L
                           : (t < tl) ? wr[(t + 1) * L]
                                      : wr[n - 1] / static_cast<LD>(H.powc[kMaxL + pl - 1]);
            double* sc = &H.scan[static_cast<size_t>(t) * kScanPerThread];
            const int wt = t / 32;
            if (wt < H.ncw || wt >= H.ncw_r0) {
                sc[14] = static_cast<double>(cf);
                sc[15] = static_cast<double>(cb);
                sc[17] = static_cast<double>(cbr);
            }
            const int ne = std::min(L, n - t * L);
            for (int e = 0; e < ne; ++e) {
                const LD qe = (t == tl) ? static_cast<LD>(H.powc[2 * kMaxL + e])
                                        : static_cast<LD>(H.powc[e]);
                const LD pe = static_cast<LD>(H.powc[kMaxL + e]);
                err = std::max(err, std::fabs(cf * qe + cb * pe - w[t * L + e]) / wmax);
                if (cyclic) err = std::max(err, std::fabs(cbr * pe - wr[t * L + e]) / wrmax);
            }
        }
        H.fit_err = static_cast<double>(err);
    }
    // cross-warp weights (zero outside the causal range)
    H.wf.assign(kMaxWarps * kMaxWarps, 0.0);
    H.wb.assign(kMaxWarps * kMaxWarps, 0.0);
    H.wk.assign(kMaxWarps * kMaxWarps, 0.0);
    for (int wi = 0; wi < nw; ++wi) {
        for (int vv = 0; vv < wi; ++vv) {
            double p = 1.0;
            for (int u = vv + 1; u <= wi - 1; ++u) p *= AWf[u];
            H.wf[wi * kMaxWarps + vv] = p;
        }
        for (int vv = wi + 1; vv < nw; ++vv) {
            double p = 1.0;
            for (int u = wi + 1; u <= vv - 1; ++u) p *= AWb[u];
            H.wb[wi * kMaxWarps + vv] = p;
        }
    }
    // D_w = sum_{v>w} Wb[w][v] (TA_v + C_v TB_v), C_v = sum_{u<v} Wf[v][u] Tf_u
    //     = sum_v Wb[w][v] TA_v + sum_u K[w][u] Tf_u
    for (int wi = 0; wi < nw; ++wi)
        for (int u = 0; u < nw; ++u) {
            double k = 0.0;
            for (int vv = std::max(wi, u) + 1; vv < nw; ++vv)
                k += H.wb[wi * kMaxWarps + vv] * TB[vv] * H.wf[vv * kMaxWarps + u];
            H.wk[wi * kMaxWarps + u] = k;
        }
    // cyclic: x0 = (M^{-1} b)_0 and xn = (M^{-1} b)_{n-1} as fixed combinations
    // of the published warp totals and of thread 0's / thread tl's scalars:
    //   x0 = z0 + pb0 (Pb_ex0 D_0 + RA0),  D_w = sum_v wb[w][v] TA_v + wk[w][v] Tf_v
    //   xn = zl + ql (Pf_ex,tl C_wl + E_tl) + pbl (Pb_ex,tl D_wl + SB_tl C_wl + RA_tl)
    H.xw.assign(4 * kMaxWarps, 0.0);
    if (cyclic) {
        const int tl = (n - 1) / L, wl = tl / 32, pl = n - tl * L;
        const size_t KS = kScanPerThread;
        const double pb0 = H.powc[kMaxL], pbex0 = H.scan[11];
        const double ql = (pl < L) ? H.powc[2 * kMaxL + pl - 1] : H.powc[pl - 1];
        const double pbl = H.powc[kMaxL + pl - 1];
        const double pfe = H.scan[tl * KS + 5], pbe = H.scan[tl * KS + 11], sbl = H.scan[tl * KS + 12];
        for (int v = 0; v < nw; ++v) {
            H.xw[v] = pb0 * pbex0 * H.wk[v];
            H.xw[kMaxWarps + v] = pb0 * pbex0 * H.wb[v];
            H.xw[2 * kMaxWarps + v] = (ql * pfe + pbl * sbl) * H.wf[wl * kMaxWarps + v] +
                                      pbl * pbe * H.wk[wl * kMaxWarps + v];
            H.xw[3 * kMaxWarps + v] = pbl * pbe * H.wb[wl * kMaxWarps + v];
        }
        H.tl = tl;
        H.pl = pl;
        H.ql = ql;
        H.pbl = pbl;
    }
    // Sub-block local passes (plain heat rows with L = 16; tri_solve_sb): a chunk
    // runs as S = L / M independent chains of M elements.  sb_q = U^{-1} p_f
    // local to a fully real sub-block and sb_pb[e] = (-c)^{M - e} go to the
    // kernels as constant-bank operands.  A sub-block with only `real` < M
    // leading elements inside the row has q' = q - kappa p_b on them,
    // kappa = sum_{j >= real} (-c)^{j - M} gamma^{j + 1}: the thread holding
    // element n-1 folds kappa_b (powc row 2) into its sub-block c_b.
#ifndef ATM_NO_SUBBLOCK
    if (!cyclic && L == 16) {
        constexpr int M = 8;
        const int S = L / M;
        const LD g = static_cast<LD>(H.gamma_c), cn = static_cast<LD>(H.cneg_c);
        LD gp[M + 1], cp[M + 1];  // powers
        gp[0] = cp[0] = 1.0L;
        for (int e = 1; e <= M; ++e) {
            gp[e] = gp[e - 1] * g;
            cp[e] = cp[e - 1] * cn;
        }
        H.sb_m = M;
        H.sb_af = static_cast<double>(gp[M]);
        H.sb_ab = static_cast<double>(cp[M]);
        LD z = 0.0L;
        for (int e = M - 1; e >= 0; --e) {
            z = cn * z + gp[e + 1];
            H.sb_q[e] = static_cast<double>(z);
            H.sb_pb[e] = static_cast<double>(cp[M - e]);
        }
        const int tl = (n - 1) / L, pl = n - tl * L;  // the thread holding element n-1
        for (int b = 0; b < S; ++b) {
            const int real = std::max(0, std::min(M, pl - b * M));
            LD kap = 0.0L;
            for (int j = real; j < M; ++j) kap += gp[j + 1] / cp[M - j];
            H.powc[2 * kMaxL + b] = static_cast<double>(kap);
        }
    }
#endif
    return H;
}

// Rows split over a cluster (n > 5376): block q = elements [4096 q, 4096 q +
// n_q) of the row, n_q = min(4096, n - 4096 q), one CTA each.  With M_q =
// L_c U_c the constant-coefficient factorisation of block q,
//   T = blockdiag(M_q) + U C U^T,  U = [e_{s_0}, e_{e_0}, e_{s_1}, e_{e_1}, ...]
// (s_q, e_q: first and last element of block q), C = the Dirichlet delta at
// every block start and the coupling a between e_q and s_{q+1}; so
//   x = M^{-1} b - M^{-1} U s,  s = S' U^T M^{-1} b,  S' = (I + C U^T M^{-1} U)^{-1} C.
// Each block's M_q^{-1} e_{s_q} and M_q^{-1} e_{e_q} are the cyclic solve's
// two correction vectors (heat_level_host with cyclic = true), applied through
// the chunk carries exactly as the periodic Allen-Cahn matrix does; U^T M^{-1} b
// is every block's (x0, xn), exchanged over the cluster (tri_solve, CL).
HeatLevelHost heat_cluster_host(int n, int cl, double r, int substeps) {
    using LD = long double;
    std::vector<HeatLevelHost> B(static_cast<size_t>(cl));
    for (int q = 0; q < cl; ++q)
        B[q] = heat_level_host(std::min(4096, n - 4096 * q), 4096, 32, r, 0.0, substeps, true);
    HeatLevelHost H = B[0];
    H.n = n;
    H.pitch = 4096 * cl;
    H.cyclic = 0;
    H.scan.clear();
    H.wf.clear();
    H.wb.clear();
    H.wk.clear();
    H.powc.clear();
    H.xw.clear();
    H.blk.assign(static_cast<size_t>(8) * cl, 0.0);
    for (int q = 0; q < cl; ++q) {
        const HeatLevelHost& b = B[q];
        H.scan.insert(H.scan.end(), b.scan.begin(), b.scan.end());
        H.wf.insert(H.wf.end(), b.wf.begin(), b.wf.end());
        H.wb.insert(H.wb.end(), b.wb.begin(), b.wb.end());
        H.wk.insert(H.wk.end(), b.wk.begin(), b.wk.end());
        H.powc.insert(H.powc.end(), b.powc.begin(), b.powc.end());
        H.xw.insert(H.xw.end(), b.xw.begin(), b.xw.end());
        double* bk = &H.blk[static_cast<size_t>(8) * q];
        bk[0] = b.ncw;
        bk[1] = b.ncw_r0;
        bk[2] = b.tl;
        bk[3] = b.pl;
        bk[4] = b.ql;
        bk[5] = b.pbl;
        H.fit_err = std::max(H.fit_err, b.fit_err);
    }
    // S' = (I + C G)^{-1} C, G = U^T M^{-1} U (2x2 blocks on the diagonal)
    const int m2 = 2 * cl;
    const LD a = -static_cast<LD>(r), c = -static_cast<LD>(H.cneg_c);
    const LD delta = a * c;
    std::vector<LD> G(static_cast<size_t>(m2) * m2, 0.0L), Cm(G), A(G), X(G);
    for (int q = 0; q < cl; ++q) {
        const int i = 2 * q;
        G[i * m2 + i] = B[q].w0;
        G[i * m2 + i + 1] = B[q].wr0;
        G[(i + 1) * m2 + i] = B[q].wn;
        G[(i + 1) * m2 + i + 1] = B[q].wrn;
        Cm[i * m2 + i] = delta;
        if (q + 1 < cl) {
            Cm[(i + 1) * m2 + i + 2] = a;
            Cm[(i + 2) * m2 + i + 1] = a;
        }
    }
    for (int i = 0; i < m2; ++i)
        for (int j = 0; j < m2; ++j) {
            LD v = (i == j) ? 1.0L : 0.0L;
            for (int k = 0; k < m2; ++k) v += Cm[i * m2 + k] * G[k * m2 + j];
            A[i * m2 + j] = v;
            X[i * m2 + j] = Cm[i * m2 + j];
        }
    // Gauss-Jordan with partial pivoting: A X = C
    for (int col = 0; col < m2; ++col) {
        int piv = col;
        for (int i = col + 1; i < m2; ++i)
            if (std::fabs(A[i * m2 + col]) > std::fabs(A[piv * m2 + col])) piv = i;
        for (int j = 0; j < m2; ++j) {
            std::swap(A[col * m2 + j], A[piv * m2 + j]);
            std::swap(X[col * m2 + j], X[piv * m2 + j]);
        }
        const LD d = A[col * m2 + col];
        for (int j = 0; j < m2; ++j) {
            A[col * m2 + j] /= d;
            X[col * m2 + j] /= d;
        }
        for (int i = 0; i < m2; ++i) {
            if (i == col) continue;
            const LD f = A[i * m2 + col];
            if (f == 0.0L) continue;
            for (int j = 0; j < m2; ++j) {
                A[i * m2 + j] -= f * A[col * m2 + j];
                X[i * m2 + j] -= f * X[col * m2 + j];
            }
        }
    }
    H.cS.resize(static_cast<size_t>(m2) * m2);
    for (size_t i = 0; i < H.cS.size(); ++i) H.cS[i] = static_cast<double>(X[i]);
    return H;
}

// one point row into shared memory: R = pitch / 16 rows of the tensor map's
// [rows][16] view -- one box, or past 256 rows (the TMA box limit) two
// half-row boxes; pitch is then a multiple of 256, so the second half lands
// 1024-byte aligned and the 128-byte swizzle is that of one box
__device__ __forceinline__ void tma_load_row(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                             int R) {
    if (R <= 256) {
        tma_load_2d(dst, map, c0, c1, bar);
    } else {  // two half-row boxes (pitch a multiple of 256: 1024-byte aligned halves)
        tma_load_2d(dst, map, c0, c1, bar);
        tma_load_2d(static_cast<char*>(dst) + (R / 2) * 128, map, c0, c1 + R / 2, bar);
    }
}

// whole-row reduction global += shared (same boxes as the store)
__device__ __forceinline__ void tma_reduce_row(const CUtensorMap* map, int c0, int c1, const void* src, int R) {
    tma_reduce_add_2d(map, c0, c1, src);
    if (R > 256) tma_reduce_add_2d(map, c0, c1 + R / 2, static_cast<const char*>(src) + (R / 2) * 128);
}

// the matching whole-row store (bulk-group completion: one commit covers all boxes)
__device__ __forceinline__ void tma_store_row(const CUtensorMap* map, int c0, int c1, const void* src, int R) {
    tma_store_2d(map, c0, c1, src);
    if (R > 256) tma_store_2d(map, c0, c1 + R / 2, static_cast<const char*>(src) + (R / 2) * 128);
}

// --------------------------------------------------------------------------
// device: per-thread state, shared tables and the tridiagonal solve

// NW: warps per CTA of the instantiation (the cross-warp carry tree)
__host__ __device__ constexpr int warps_for(int L) { return L >= 32 ? 4 : (L == 16 ? 8 : 16); }

template <int L, int NW = warps_for(L), bool CL = false>
struct Lane {
    int t, lane, warp, nw, s;
    int q7, qx, qx1, ch0;  // swizzled row-staging geometry (L = 32: two 128-B rows)
    int pad0;            // first padding element of the chunk, L if none
    bool pad_last;       // pad0 == L - 1: only the chunk's last element is padding
    int par;             // parity of the warp-total slots (one barrier per Phi)
    bool corr, inside;   // carries the boundary correction; chunk inside the row
    double Mf[5], Pfex, Mb[5], Pbex, SB, q0;
    double cfw, cbw;     // correction carries of the chunk (left vector)
    // sub-block solve, the thread holding element n-1: kappa of its last
    // sub-block (and kappa (-c)^M) when only that one is short -- folded
    // off the carry chain; edge_slow: some other sub-block is short too
    double kapl, kapab;
    bool edge_slow;
    double cbwr;         // cyclic: right correction vector's p_b coefficient
    // cluster rows (CL): rank of the CTA in the cluster (its block of the
    // row) and the block's x_{n-1} pick-up (thread tl, element pl - 1)
    int q, btl, bpl;
    double bql, bpbl;
};

template <int L, int NW, bool CL>
__device__ __forceinline__ void lane_init(Lane<L, NW, CL>& ln, const HeatCoefDev& co) {
    ln.t = threadIdx.x;
    ln.lane = ln.t & 31;
    ln.warp = ln.t >> 5;
    ln.nw = blockDim.x >> 5;
    // the staging geometry is local to the CTA's part of the row; element
    // offsets (padding, forcing profile) and the tables are the row's
    const int sloc = ln.t * L;
    ln.q = 0;
    int gt = ln.t;
    if constexpr (CL) {
        ln.q = static_cast<int>(cg::this_cluster().block_rank());
        gt += ln.q * blockDim.x;
        const double* b = co.blk + 8 * ln.q;
        ln.corr = ln.warp < static_cast<int>(b[0]) || ln.warp >= static_cast<int>(b[1]);
        ln.btl = static_cast<int>(b[2]);
        ln.bpl = static_cast<int>(b[3]);
        ln.bql = b[4];
        ln.bpbl = b[5];
    } else {
        ln.corr = ln.warp < co.ncw || ln.warp >= co.ncw_r0;
        ln.btl = ln.bpl = 0;
        ln.bql = ln.bpbl = 0.0;
    }
    ln.s = gt * L;
    ln.inside = ln.s < co.pitch;  // chunks never straddle pitch (pitch % 16 == 0)
    ln.q7 = (sloc >> 4) << 7;
    ln.qx = (sloc >> 4) & 7;
    ln.ch0 = (sloc & 15) >> 1;
    ln.qx1 = (ln.qx + 1) & 7;
    ln.pad0 = (ln.s + L > co.n) ? max(0, co.n - ln.s) : L;
    ln.pad_last = ln.pad0 == L - 1;
    ln.par = 0;
    const double* sc = co.scan + gt * kScanPerThread;
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        ln.Mf[d] = __ldg(sc + d);
        ln.Mb[d] = __ldg(sc + 6 + d);
    }
    ln.Pfex = __ldg(sc + 5);
    ln.Pbex = __ldg(sc + 11);
    ln.SB = __ldg(sc + 12);
    ln.q0 = __ldg(sc + 13);
    ln.kapl = ln.kapab = 0.0;
    ln.edge_slow = false;
    if constexpr (L == 16 && !CL) {
        if (co.sb_m > 0 && ln.pad0 > 0 && ln.pad0 < L) {
            constexpr int S = L / 8;
            const double* kap = co.powc + 2 * kMaxL;
            for (int b = 0; b < S - 1; ++b) ln.edge_slow = ln.edge_slow || __ldg(kap + b) != 0.0;
            if (!ln.edge_slow) {
                ln.kapl = __ldg(kap + S - 1);
                ln.kapab = ln.kapl * co.sb_ab;
            }
        }
    }
    ln.cfw = ln.corr ? __ldg(sc + 14) : 0.0;
    ln.cbw = ln.corr ? __ldg(sc + 15) : 0.0;
    ln.cbwr = ln.corr ? __ldg(sc + 17) : 0.0;
}

struct Tabs {              // per-CTA copy of the level's small tables
    double wf[kMaxWarps * kMaxWarps];
    double wb[kMaxWarps * kMaxWarps];
    double wk[kMaxWarps * kMaxWarps];
    double powc[3 * kMaxL];  // q, p_b of interior threads; q of the padded last thread
    double pbex0;            // thread 0's Pb_ex
    double xw[4 * kMaxWarps];  // cyclic: x0 / xn weights of (Tf, TA)
};

struct Slots {                // small shared scratch
    double tf[2][kMaxWarps];  // forward warp totals (double-buffered by Phi parity)
    double ta[2][kMaxWarps];  // backward warp totals, C_w-free part
    double red[kMaxWarps];
    double z0[2], ra0[2];     // thread 0's z_loc[0] and RA_next (ncw > 1)
    double zl[2], el[2], ral[2];  // cyclic: thread tl's z_loc[pl-1], E, RA_next
    double nrm[2][kMaxWarps][2];  // Newton: per-warp residual square sums, max u^2
    double cz[2][kMaxCluster][2];  // cluster rows: every block's (x0, xn), by parity
    double csq[kMaxCluster];       // cluster rows: every block's tail square sum
    uint64_t bar[5];
};

// q: the CTA's block of a cluster row (its tables; 0 otherwise)
__device__ __forceinline__ void tabs_init(Tabs& tb, Slots& sl, const HeatCoefDev& co, int q = 0) {
    const double* wf = co.wf + q * kMaxWarps * kMaxWarps;
    const double* wb = co.wb + q * kMaxWarps * kMaxWarps;
    const double* wk = co.wk + q * kMaxWarps * kMaxWarps;
    for (int i = threadIdx.x; i < kMaxWarps * kMaxWarps; i += blockDim.x) {
        tb.wf[i] = wf[i];
        tb.wb[i] = wb[i];
        tb.wk[i] = wk[i];
    }
    for (int i = threadIdx.x; i < 3 * kMaxL; i += blockDim.x) tb.powc[i] = co.powc[q * 3 * kMaxL + i];
    if (threadIdx.x == 0) tb.pbex0 = co.scan[static_cast<size_t>(q) * blockDim.x * kScanPerThread + 11];
    for (int i = threadIdx.x; i < 4 * kMaxWarps; i += blockDim.x) tb.xw[i] = co.xw[q * 4 * kMaxWarps + i];
    // warp slots beyond the CTA are read with zero weights: keep them finite
    for (int i = threadIdx.x; i < 2 * kMaxWarps; i += blockDim.x) {
        sl.tf[i / kMaxWarps][i % kMaxWarps] = 0.0;
        sl.ta[i / kMaxWarps][i % kMaxWarps] = 0.0;
    }
}

// x[pad0 .. L) = 0 for the thread holding element n-1 (and fully padded
// threads).  A single padded element at the chunk end (n = 4095 and every
// n = k L - 1) is a select with no branch; otherwise a fall-through switch:
// one jump and L - pad0 moves for that thread instead of L predicated
// selects in its whole warp.
template <int L, int NW, bool CL>
__device__ __forceinline__ void zero_padding(double (&x)[L], const Lane<L, NW, CL>& ln) {
    x[L - 1] = ln.pad_last ? 0.0 : x[L - 1];
    if (ln.pad0 < L - 1) {
        switch (ln.pad0) {
        case 0: if constexpr (L > 0) x[0] = 0.0; [[fallthrough]];
        case 1: if constexpr (L > 1) x[1] = 0.0; [[fallthrough]];
        case 2: if constexpr (L > 2) x[2] = 0.0; [[fallthrough]];
        case 3: if constexpr (L > 3) x[3] = 0.0; [[fallthrough]];
        case 4: if constexpr (L > 4) x[4] = 0.0; [[fallthrough]];
        case 5: if constexpr (L > 5) x[5] = 0.0; [[fallthrough]];
        case 6: if constexpr (L > 6) x[6] = 0.0; [[fallthrough]];
        case 7: if constexpr (L > 7) x[7] = 0.0; [[fallthrough]];
        case 8: if constexpr (L > 8) x[8] = 0.0; [[fallthrough]];
        case 9: if constexpr (L > 9) x[9] = 0.0; [[fallthrough]];
        case 10: if constexpr (L > 10) x[10] = 0.0; [[fallthrough]];
        case 11: if constexpr (L > 11) x[11] = 0.0; [[fallthrough]];
        case 12: if constexpr (L > 12) x[12] = 0.0; [[fallthrough]];
        case 13: if constexpr (L > 13) x[13] = 0.0; [[fallthrough]];
        case 14: if constexpr (L > 14) x[14] = 0.0; [[fallthrough]];
        case 15: if constexpr (L > 15) x[15] = 0.0; [[fallthrough]];
        case 16: if constexpr (L > 16) x[16] = 0.0; [[fallthrough]];
        case 17: if constexpr (L > 17) x[17] = 0.0; [[fallthrough]];
        case 18: if constexpr (L > 18) x[18] = 0.0; [[fallthrough]];
        case 19: if constexpr (L > 19) x[19] = 0.0; [[fallthrough]];
        case 20: if constexpr (L > 20) x[20] = 0.0; [[fallthrough]];
        case 21: if constexpr (L > 21) x[21] = 0.0; [[fallthrough]];
        case 22: if constexpr (L > 22) x[22] = 0.0; [[fallthrough]];
        case 23: if constexpr (L > 23) x[23] = 0.0; [[fallthrough]];
        case 24: if constexpr (L > 24) x[24] = 0.0; [[fallthrough]];
        case 25: if constexpr (L > 25) x[25] = 0.0; [[fallthrough]];
        case 26: if constexpr (L > 26) x[26] = 0.0; [[fallthrough]];
        case 27: if constexpr (L > 27) x[27] = 0.0; [[fallthrough]];
        case 28: if constexpr (L > 28) x[28] = 0.0; [[fallthrough]];
        case 29: if constexpr (L > 29) x[29] = 0.0; [[fallthrough]];
        case 30: if constexpr (L > 30) x[30] = 0.0; [[fallthrough]];
        case 31: if constexpr (L > 31) x[31] = 0.0; [[fallthrough]];
        default: break;
        }
    }
}

// The blocked solve with sub-block local passes (plain heat rows with L = 16:
// the coarsest level of 2048 < n <= 5376, i.e. config 5's windows; the L = 32
// sweeps keep tri_solve -- see profiles/README.md, round 2).
// Every chunk is S = L / M sub-blocks whose M-long local chains run
// independently (4-way ILP on the FP64 pipe instead of 2 x L dependent
// DFMAs), and the sub-block carries are folded into the fix-up the blocked
// solve applies anyway: sub-block b gets its own pair (c_f, c_b),
//   c_f[b+1] = Y_b + gamma^M c_f[b]            (Y_b: the sub-block's local end)
//   c_b[b]   = z_{b+1} + c_f[b+1] q[0] + (-c)^M c_b[b+1]
// (z_{b+1}: first local backward value of sub-block b + 1), started from the
// thread's carries c_f[0] = c_f, c_b[S-1] = c_b.  Before the barrier the
// same two chains with zero thread carries give the thread's forward end B
// and first backward value zeta that the warp scans combine.  All fully real
// sub-blocks share one q and one p_b of M entries, read as constant-bank
// operands: the fix-up makes no shared-memory table reads (the LSU data
// pipe was the busiest unit of the Phi-bound sweeps).  The thread holding
// element n-1 has shorter sub-blocks: q' = q - kappa_b p_b there, folded
// into its c_b.  The thread-level tables (scan multipliers, cross-warp
// weights, boundary correction: a shift of the thread's two carries) are
// those of tri_solve.
template <int L, int NW, bool CL>
__device__ __forceinline__ void tri_solve_sb(double (&x)[L], const HeatCoefDev& co, Lane<L, NW, CL>& ln,
                                             const Tabs& tb, Slots& sl) {
    constexpr int M = 8, S = L / M;
    const double ab = co.sb_ab, q0c = co.sb_q[0];
    // sub-block carry multipliers: gamma^M across a fully real sub-block, 0
    // once the sub-block holds a padding element
    double af[S];
#pragma unroll
    for (int b = 0; b < S; ++b) af[b] = ((b + 1) * M <= ln.pad0) ? co.sb_af : 0.0;
    // effective right-carry coefficients ce[b] of the sub-blocks for forward
    // carries f[b] and the thread's right carry c; returns the chunk's first
    // backward value.  The chain ce[b] = ce[b+1] (-c)^M + T_b carries one FMA
    // per sub-block; kappa of a short last sub-block enters T_{S-2} and
    // ce[S-1] off the chain (kapl = 0 on every other thread).
    auto back_carries = [&](const double (&f)[S], double c, double (&ce)[S]) {
        double T[S];
#pragma unroll
        for (int b = 0; b < S - 1; ++b) T[b] = fma(f[b + 1], q0c, x[(b + 1) * M]);
        T[S - 2] = fma(-ln.kapab, f[S - 1], T[S - 2]);
        ce[S - 1] = fma(-ln.kapl, f[S - 1], c);
        ce[S - 2] = fma(c, ab, T[S - 2]);
#pragma unroll
        for (int b = S - 3; b >= 0; --b) ce[b] = fma(ce[b + 1], ab, T[b]);
        if (ln.edge_slow) {  // a short sub-block before the last one (n % L <= L - M)
            const double* kap = tb.powc + 2 * kMaxL;
            ce[S - 1] = fma(-kap[S - 1], f[S - 1], c);
#pragma unroll
            for (int b = S - 2; b >= 0; --b)
                ce[b] = fma(-kap[b], f[b], fma(ce[b + 1], ab, fma(f[b + 1], q0c, x[(b + 1) * M])));
        }
        return fma(ce[0], ab, fma(f[0], q0c, x[0]));
    };
    // 1. forward local, S independent chains
    {
        const double bb = co.beta_c, gg = co.gamma_c;
#pragma unroll
        for (int e = 0; e < M; ++e) {
#pragma unroll
            for (int b = 0; b < S; ++b) {
                const double prev = e == 0 ? 0.0 : x[b * M + e - 1];
                x[b * M + e] = fma(gg, prev, bb * x[b * M + e]);
            }
        }
        zero_padding<L>(x, ln);
    }
    double Y[S], eb[S];
#pragma unroll
    for (int b = 0; b < S; ++b) Y[b] = x[b * M + M - 1];
    eb[0] = 0.0;
    eb[1] = Y[0];
#pragma unroll
    for (int b = 2; b < S; ++b) eb[b] = fma(af[b - 1], eb[b - 1], Y[b - 1]);
    // 2. forward warp scan of the chunk ends
    double B = fma(af[S - 1], eb[S - 1], Y[S - 1]);
#pragma unroll
    for (int d = 0; d < 5; ++d) B = fma(ln.Mf[d], __shfl_up_sync(0xffffffffu, B, 1 << d), B);
    double E = __shfl_up_sync(0xffffffffu, B, 1);
    if (ln.lane == 0) E = 0.0;
    // 3. backward local on the uncorrected forward values, S independent chains
    {
        const double cc = co.cneg_c;
#pragma unroll
        for (int e = M - 2; e >= 0; --e) {
#pragma unroll
            for (int b = 0; b < S; ++b) x[b * M + e] = fma(cc, x[b * M + e + 1], x[b * M + e]);
        }
    }
    // the chunk's first backward value with zero carries into the thread
    double ce[S];
    const double zeta = back_carries(eb, 0.0, ce);
    // 4. backward warp scan of a = zeta + E q0
    double R = fma(E, ln.q0, zeta);
#pragma unroll
    for (int d = 0; d < 5; ++d) R = fma(ln.Mb[d], __shfl_down_sync(0xffffffffu, R, 1 << d), R);
    double RAn = __shfl_down_sync(0xffffffffu, R, 1);
    if (ln.lane == 31) RAn = 0.0;
    // 5. publish warp totals; one barrier; cross-warp carries (tri_solve)
    const int par = ln.par;
    if (ln.lane == 31) sl.tf[par][ln.warp] = B;
    if (ln.lane == 0) sl.ta[par][ln.warp] = R;
    const bool far = ln.corr && ln.warp > 0;
    double z00 = 0.0, ra0 = 0.0;
    if (co.ncw > 1) {
        if (ln.t == 0) {
            sl.z0[par] = zeta;
            sl.ra0[par] = RAn;
        }
    } else if (ln.corr) {
        z00 = __shfl_sync(0xffffffffu, zeta, 0);
        ra0 = __shfl_sync(0xffffffffu, RAn, 0);
    }
    __syncthreads();
    ln.par ^= 1;
    double cC, cD, cD0 = 0.0;
    {
        const int v = ln.lane & (NW - 1);
        const double tf = sl.tf[par][v], ta = sl.ta[par][v];
        const int row = ln.warp * kMaxWarps + v;
        cC = tb.wf[row] * tf;
        cD = fma(tb.wb[row], ta, tb.wk[row] * tf);
        if (far) cD0 = fma(tb.wb[v], ta, tb.wk[v] * tf);
#pragma unroll
        for (int off = NW / 2; off >= 1; off >>= 1) {
            cC += __shfl_xor_sync(0xffffffffu, cC, off);
            cD += __shfl_xor_sync(0xffffffffu, cD, off);
        }
        if (far) {
#pragma unroll
            for (int off = NW / 2; off >= 1; off >>= 1)
                cD0 += __shfl_xor_sync(0xffffffffu, cD0, off);
        }
    }
    double cf = fma(ln.Pfex, cC, E);
    double cb = fma(ln.Pbex, cD, fma(ln.SB, cC, RAn));
    if (ln.corr) {
        if (co.ncw > 1) {
            z00 = sl.z0[par];
            ra0 = sl.ra0[par];
        }
        const double x0 = fma(fma(tb.pbex0, far ? cD0 : cD, ra0), tb.powc[kMaxL], z00);
        const double ms = -co.sigma * x0;
        cf = fma(ms, ln.cfw, cf);
        cb = fma(ms, ln.cbw, cb);
    }
    // 6. sub-block carries, then x = z_loc + c_f[b] q + c_b[b] p_b
    {
        double cfb[S];
        cfb[0] = cf;
#pragma unroll
        for (int b = 1; b < S; ++b) cfb[b] = fma(af[b - 1], cfb[b - 1], Y[b - 1]);
        back_carries(cfb, cb, ce);
#pragma unroll
        for (int e = 0; e < M; ++e)
#pragma unroll
            for (int b = 0; b < S; ++b)
                x[b * M + e] = fma(ce[b], co.sb_pb[e], fma(cfb[b], co.sb_q[e], x[b * M + e]));
        zero_padding<L>(x, ln);
    }
}

// (I + sub_dt L) x = x, in place, over the CTA (heat1d.cpp:47-60); CYC:
// the periodic matrix with corner entries a (Allen-Cahn linear part).
// warps per CTA of the instantiation for chunk length L (a power of two):
// L = 32 -> 128 threads, L = 16 -> 256, L <= 8 -> 512

template <int L, bool CYC = false, int NW = warps_for(L), bool CL = false>
__device__ __forceinline__ void tri_solve(double (&x)[L], const HeatCoefDev& co, Lane<L, NW, CL>& ln,
                                          const Tabs& tb, Slots& sl) {
#ifndef ATM_NO_SUBBLOCK
    if constexpr (!CYC && !CL && L == 16) {
        tri_solve_sb<L>(x, co, ln, tb, sl);
        return;
    }
#endif
    // 1. forward local  y_i = beta x_i + gamma y_{i-1}
    double y = 0.0;
    {
        const double bb = co.beta_c, gg = co.gamma_c;
#pragma unroll
        for (int e = 0; e < L; ++e) {
            y = fma(gg, y, bb * x[e]);
            x[e] = y;
        }
        zero_padding<L>(x, ln);
        y = x[L - 1];
    }
    // 2. forward warp scan of the chunk ends
    double B = y;
#pragma unroll
    for (int d = 0; d < 5; ++d) B = fma(ln.Mf[d], __shfl_up_sync(0xffffffffu, B, 1 << d), B);
    double E = __shfl_up_sync(0xffffffffu, B, 1);
    if (ln.lane == 0) E = 0.0;
    // 3. backward local on the uncorrected forward values
    double z = 0.0;
    {
        const double cc = co.cneg_c;
#pragma unroll
        for (int e = L - 1; e >= 0; --e) {
            z = fma(cc, z, x[e]);
            x[e] = z;
        }
    }
    // 4. backward warp scan of a = z_loc[0] + E q0 (the C_w part is precomputed)
    double R = fma(E, ln.q0, z);
#pragma unroll
    for (int d = 0; d < 5; ++d) R = fma(ln.Mb[d], __shfl_down_sync(0xffffffffu, R, 1 << d), R);
    double RAn = __shfl_down_sync(0xffffffffu, R, 1);
    if (ln.lane == 31) RAn = 0.0;
    // 5. publish warp totals; one barrier; cross-warp carries.  The
    //    correction needs x0 = (M^{-1} b)_0 = z0 + c_b(thread 0) p_b[0]
    //    (thread 0 has no forward carry), c_b(thread 0) = Pb_ex0 D_0 + RA0:
    //    thread 0's z0 and RA0 travel by shuffle (ncw == 1) or smem.
    const int par = ln.par;
    if (ln.lane == 31) sl.tf[par][ln.warp] = B;
    if (ln.lane == 0) sl.ta[par][ln.warp] = R;
    // CL (cluster rows) runs the cyclic machinery: every block carries a left
    // and a right correction vector, coupled across the cluster below
    constexpr bool WB = CYC || CL;
    const bool far = !WB && ln.corr && ln.warp > 0;  // correction warp without warp 0's D
    double z00 = 0.0, ra0 = 0.0;
    if (WB) {
        const int tl = CL ? ln.btl : co.tl, pl = CL ? ln.bpl : co.pl;
        if (ln.t == 0) {
            sl.z0[par] = x[0];
            sl.ra0[par] = RAn;
        }
        if (ln.t == tl) {
            double zl = x[0];
#pragma unroll
            for (int e = 1; e < L; ++e)
                if (e == pl - 1) zl = x[e];
            sl.zl[par] = zl;
            sl.el[par] = E;
            sl.ral[par] = RAn;
        }
    } else if (co.ncw > 1) {
        if (ln.t == 0) {
            sl.z0[par] = x[0];
            sl.ra0[par] = RAn;
        }
    } else if (ln.corr) {
        z00 = __shfl_sync(0xffffffffu, x[0], 0);
        ra0 = __shfl_sync(0xffffffffu, RAn, 0);
    }
    __syncthreads();
    ln.par ^= 1;
    double cC, cD, cD0 = 0.0;
    double p0 = 0.0, pN = 0.0;
    {
        const int v = ln.lane & (NW - 1);
        const double tf = sl.tf[par][v], ta = sl.ta[par][v];
        const int row = ln.warp * kMaxWarps + v;
        cC = tb.wf[row] * tf;
        cD = fma(tb.wb[row], ta, tb.wk[row] * tf);
        if (far) cD0 = fma(tb.wb[v], ta, tb.wk[v] * tf);
        if (WB && ln.corr) {
            p0 = fma(tb.xw[v], tf, tb.xw[kMaxWarps + v] * ta);
            pN = fma(tb.xw[2 * kMaxWarps + v], tf, tb.xw[3 * kMaxWarps + v] * ta);
        }
#pragma unroll
        for (int off = NW / 2; off >= 1; off >>= 1) {
            cC += __shfl_xor_sync(0xffffffffu, cC, off);
            cD += __shfl_xor_sync(0xffffffffu, cD, off);
        }
        if (far) {
#pragma unroll
            for (int off = NW / 2; off >= 1; off >>= 1)
                cD0 += __shfl_xor_sync(0xffffffffu, cD0, off);
        }
        if (WB && ln.corr) {
#pragma unroll
            for (int off = NW / 2; off >= 1; off >>= 1) {
                p0 += __shfl_xor_sync(0xffffffffu, p0, off);
                pN += __shfl_xor_sync(0xffffffffu, pN, off);
            }
        }
    }
    double cf = fma(ln.Pfex, cC, E);
    double cb = fma(ln.Pbex, cD, fma(ln.SB, cC, RAn));
    if constexpr (CL) {
        // cluster rows: T = blockdiag(M_q) + U C U^T over every block's first
        // and last element (C: the Dirichlet delta at each block start, the
        // coupling a between neighbouring blocks); x = M^{-1}b - W s with
        // s = S' U^T M^{-1} b, S' = (I + C U^T W)^{-1} C (host, long double).
        // Every block's (x0, xn) goes to every CTA; all sum in one order.
        double x0 = 0.0, xn = 0.0;
        if (ln.corr) {
            x0 = fma(tb.powc[kMaxL], sl.ra0[par], sl.z0[par]) + p0;
            xn = fma(ln.bpbl, sl.ral[par], fma(ln.bql, sl.el[par], sl.zl[par])) + pN;
        }
        cg::cluster_group clu = cg::this_cluster();
        if (ln.t == 0)
            for (int r = 0; r < co.cl; ++r) {
                double* d = clu.map_shared_rank(&sl.cz[par][ln.q][0], r);
                d[0] = x0;
                d[1] = xn;
            }
        clu.sync();
        if (ln.corr) {
            const int m2 = 2 * co.cl;
            const double* r0 = co.cS + static_cast<size_t>(2 * ln.q) * m2;
            const double* r1 = r0 + m2;
            double s0 = 0.0, s1 = 0.0;
            for (int j = 0; j < co.cl; ++j) {
                const double zj0 = sl.cz[par][j][0], zj1 = sl.cz[par][j][1];
                s0 = fma(__ldg(r0 + 2 * j), zj0, fma(__ldg(r0 + 2 * j + 1), zj1, s0));
                s1 = fma(__ldg(r1 + 2 * j), zj0, fma(__ldg(r1 + 2 * j + 1), zj1, s1));
            }
            cf = fma(-s0, ln.cfw, cf);
            cb = fma(-s0, ln.cbw, fma(-s1, ln.cbwr, cb));
        }
    } else if (CYC) {
        if (ln.corr) {
            // Woodbury: s = S [x0, xn], x -= s0 wl + s1 wr
            const double x0 = fma(tb.powc[kMaxL], sl.ra0[par], sl.z0[par]) + p0;
            const double xn = fma(co.pbl, sl.ral[par], fma(co.ql, sl.el[par], sl.zl[par])) + pN;
            const double s0 = fma(co.S[0], x0, co.S[1] * xn);
            const double s1 = fma(co.S[2], x0, co.S[3] * xn);
            cf = fma(-s0, ln.cfw, cf);
            cb = fma(-s0, ln.cbw, fma(-s1, ln.cbwr, cb));
        }
    } else if (ln.corr) {
        if (co.ncw > 1) {
            z00 = sl.z0[par];
            ra0 = sl.ra0[par];
        }
        const double x0 = fma(fma(tb.pbex0, far ? cD0 : cD, ra0), tb.powc[kMaxL], z00);
        const double ms = -co.sigma * x0;
        cf = fma(ms, ln.cfw, cf);
        cb = fma(ms, ln.cbw, cb);
    }
    // 6. x = z_loc + c_f q + c_b p_b
    {
        const double* qv = (ln.pad0 < L) ? tb.powc + 2 * kMaxL : tb.powc;
#pragma unroll
        for (int e = 0; e < L; ++e) x[e] = fma(cb, tb.powc[kMaxL + e], fma(cf, qv[e], x[e]));
        zero_padding<L>(x, ln);
    }
}

// Phi_index on this level: S sub-steps, forcing added before each solve
// when `forced` (heat1d.cpp:66-83).
template <int L, int NW, bool CL>
__device__ __forceinline__ void phi(double (&x)[L], const HeatCoefDev& co, Lane<L, NW, CL>& ln,
                                    const Tabs& tb, Slots& sl, int index, int forced) {
    for (int s = 0; s < co.substeps; ++s) {
        if (forced) {
            const double th = __ldg(co.theta + static_cast<size_t>(index) * co.substeps + s);
#pragma unroll
            for (int e = 0; e < L; ++e) x[e] = fma(th, __ldg(co.prof + ln.s + e), x[e]);
        }
        tri_solve<L>(x, co, ln, tb, sl);
    }
}

// Allen-Cahn Phi: S backward-Euler sub-steps, each solved by Newton on
//   F(u) = u - dt (c (u_l - 2u + u_r) + u - u^3) - u_prev   (periodic),
//   J = A + D,  A = tridiag(-dt c, 1 + 2 dt c - dt, -dt c) cyclic, D = 3 dt u^2,
// with the Newton stopping rule of gray_scott.cpp:113 (stop = max(tol, tol
// |F_0|), cap -> NonlinearSolveError, :165-169).  J delta = -F is solved by
// Richardson on the shifted constant part A_s = A + s I (the fast cyclic
// solve): delta <- A_s^{-1}(-F - (D - s) delta), rate
// rho <= max(s, 3 dt umax^2 - s) / (1 - dt + s), iterated to rho^K <= eta.
// Chunk ends travel through smem (one barrier per residual); the residual
// norm and max u^2 ride on a second barrier.
template <int L, int NW, bool CL, bool PART>
__device__ __forceinline__ void ac_residual(const double (&u)[L], const double (&up)[L],
                                            double (&F)[L], const HeatCoefDev& co,
                                            const Lane<L, NW, CL>& ln, double* ends, double& sq,
                                            double& u2) {
    const int nt = blockDim.x;
    const bool last = ln.t == co.tl;
    const double dt = co.ac_dt, c = co.ac_c;
    sq = 0.0;
    u2 = 0.0;
    if constexpr (!PART) {
        // n a multiple of L: every real chunk is full (the instantiation for
        // every n % L == 0; PART handles the partial last chunk)
        ends[ln.t] = u[0];
        ends[nt + ln.t] = u[L - 1];
        __syncthreads();
        const bool real = ln.t <= co.tl;
        const double ul = ends[nt + (ln.t == 0 ? co.tl : ln.t - 1)];
        const double ur = ends[last ? 0 : ln.t + 1];
#pragma unroll
        for (int e = 0; e < L; ++e) {
            const double a = e == 0 ? ul : u[e - 1];
            const double b = e == L - 1 ? ur : u[e + 1];
            const double ui = u[e];
            const double lap = c * (a - 2.0 * ui + b);
            const double f = real ? ui - dt * (lap + ui - ui * ui * ui) - up[e] : 0.0;
            F[e] = f;
            sq = fma(f, f, sq);
            u2 = fmax(u2, ui * ui);
        }
        return;
    } else {
    // thread tl holds elements [tl L, tl L + pl) with element n-1 last: its
    // chunk end is u[pl - 1], whose periodic right neighbour is element 0
    double uend = u[L - 1];
    if (last) {
#pragma unroll
        for (int e = 0; e < L - 1; ++e)
            if (e == co.pl - 1) uend = u[e];
    }
    ends[ln.t] = u[0];
    ends[nt + ln.t] = uend;
    __syncthreads();
    const bool real = ln.t <= co.tl;
    const double ul = ends[nt + (ln.t == 0 ? co.tl : ln.t - 1)];
    const double ur = ends[last ? 0 : ln.t + 1];
    const int eend = last ? co.pl - 1 : L - 1;  // the chunk's last real element
#pragma unroll
    for (int e = 0; e < L; ++e) {
        const double a = e == 0 ? ul : u[e - 1];
        const double b = e == eend ? ur : (e == L - 1 ? 0.0 : u[e + 1]);
        const double ui = u[e];
        const double lap = c * (a - 2.0 * ui + b);
        const double f = (real && e <= eend) ? ui - dt * (lap + ui - ui * ui * ui) - up[e] : 0.0;
        F[e] = f;
        sq = fma(f, f, sq);
        u2 = fmax(u2, ui * ui);
    }
    }
}

template <int L, int NW, bool CL>
__device__ __forceinline__ void ac_reduce(double sq, double u2, const Lane<L, NW, CL>& ln, Slots& sl,
                                          int par, double& res, double& umax2) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, off);
        u2 = fmax(u2, __shfl_xor_sync(0xffffffffu, u2, off));
    }
    if (ln.lane == 0) {
        sl.nrm[par][ln.warp][0] = sq;
        sl.nrm[par][ln.warp][1] = u2;
    }
    __syncthreads();
    res = 0.0;
    umax2 = 0.0;
    for (int w = 0; w < ln.nw; ++w) {
        res += sl.nrm[par][w][0];
        umax2 = fmax(umax2, sl.nrm[par][w][1]);
    }
    res = sqrt(res);
}

template <int L, int NW, bool CL, bool PART = false>
__device__ __forceinline__ void ac_phi(double (&u)[L], const HeatCoefDev& co, Lane<L, NW, CL>& ln,
                                       const Tabs& tb, Slots& sl, double* ends) {
    int rpar = 0;
    for (int s = 0; s < co.substeps; ++s) {
        double up[L], F[L];
#pragma unroll
        for (int e = 0; e < L; ++e) up[e] = u[e];
        double sq, u2, res, umax2;
        ac_residual<L, NW, CL, PART>(u, up, F, co, ln, ends + rpar * 2 * blockDim.x, sq, u2);
        ac_reduce<L>(sq, u2, ln, sl, rpar, res, umax2);
        rpar ^= 1;
        const double stop = fmax(co.newton_tol, co.newton_tol * res);
        int it = 0;
        while (res > stop) {
            if (it >= co.newton_max) {
                if (ln.t == 0) atomicExch(co.fail, 1);
                break;
            }
            // inner iterations for this Newton step (uniform over the CTA)
            const double dt = co.ac_dt, sh = co.ac_shift;
            const double rho =
                fmax(sh, 3.0 * dt * fmax(umax2, co.ac_umax2) - sh) / (1.0 - dt + sh);
            int K = 1;
            for (double e = rho; e > co.inner_eta && K < 64; e *= rho) ++K;
            double d[L];
#pragma unroll
            for (int e = 0; e < L; ++e) d[e] = -F[e];
            tri_solve<L, true>(d, co, ln, tb, sl);
            for (int k = 1; k < K; ++k) {
#pragma unroll
                for (int e = 0; e < L; ++e) {
                    const double De = fma(3.0 * dt * u[e], u[e], -sh);
                    d[e] = fma(-De, d[e], -F[e]);
                }
                tri_solve<L, true>(d, co, ln, tb, sl);
            }
#pragma unroll
            for (int e = 0; e < L; ++e) u[e] += d[e];
            ac_residual<L, NW, CL, PART>(u, up, F, co, ln, ends + rpar * 2 * blockDim.x, sq, u2);
            ac_reduce<L>(sq, u2, ln, sl, rpar, res, umax2);
            rpar ^= 1;
            ++it;
        }
    }
}

// problem dispatch: P = 0 heat (forcing optional), P = 1 Allen-Cahn
template <int P, int L, int NW, bool CL>
__device__ __forceinline__ void phi_p(double (&x)[L], const HeatCoefDev& co, Lane<L, NW, CL>& ln,
                                      const Tabs& tb, Slots& sl, double* ends, int index,
                                      int forced) {
    if constexpr (P >= 1) ac_phi<L, NW, CL, P == 2>(x, co, ln, tb, sl, ends);
    else phi<L>(x, co, ln, tb, sl, index, forced);
}

// --------------------------------------------------------------------------
// device: swizzled row staging (TMA SWIZZLE_128B layout).  A thread's chunk
// lies in one 128-byte row q of the staging box; 16-byte unit c sits at
// position c ^ (q & 7).

// byte offset of element pair c (elements 2c, 2c+1) of this thread's chunk
template <int L, int NW, bool CL>
__device__ __forceinline__ int pair_off(const Lane<L, NW, CL>& ln, int c) {
    if constexpr (L == 32) {
        const int half = c >> 3, cc = c & 7;
        return ln.q7 + (half << 7) + ((cc ^ (half ? ln.qx1 : ln.qx)) << 4);
    } else {
        return ln.q7 + (((ln.ch0 + c) ^ ln.qx) << 4);
    }
}

template <int L, int NW, bool CL>
__device__ __forceinline__ void row_load(const char* buf, double (&x)[L], const Lane<L, NW, CL>& ln) {
    if (ln.inside) {
#pragma unroll
        for (int c = 0; c < L / 2; ++c) {
            const double2 v = *reinterpret_cast<const double2*>(buf + pair_off<L>(ln, c));
            x[2 * c] = v.x;
            x[2 * c + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < L; ++e) x[e] = 0.0;
    }
}

template <int L, int NW, bool CL>
__device__ __forceinline__ void row_store(char* buf, const double (&x)[L], const Lane<L, NW, CL>& ln) {
    if (ln.inside) {
#pragma unroll
        for (int c = 0; c < L / 2; ++c)
            *reinterpret_cast<double2*>(buf + pair_off<L>(ln, c)) = make_double2(x[2 * c], x[2 * c + 1]);
    }
}

// x = x + row, or x = x - row
template <int L, int NW, bool CL>
__device__ __forceinline__ void row_acc(const char* buf, double (&x)[L], const Lane<L, NW, CL>& ln,
                                        bool sub) {
    if (ln.inside) {
#pragma unroll
        for (int c = 0; c < L / 2; ++c) {
            const double2 v = *reinterpret_cast<const double2*>(buf + pair_off<L>(ln, c));
            if (sub) {
                x[2 * c] -= v.x;
                x[2 * c + 1] -= v.y;
            } else {
                x[2 * c] += v.x;
                x[2 * c + 1] += v.y;
            }
        }
    }
}

// fixed-order CTA reduction of sum x_e^2 (thread order, then warp xor tree,
// then warps in order): depends only on the CTA shape
template <int L, int NW, bool CL>
__device__ __forceinline__ double cta_sum_squares(const double (&x)[L], const Lane<L, NW, CL>& ln,
                                                  Slots& sl) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < L; ++e) s = fma(x[e], x[e], s);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (ln.lane == 0) sl.red[ln.warp] = s;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < ln.nw; ++w) tot += sl.red[w];
    if constexpr (CL) {
        // cluster rows: every block's sum to every CTA, added in block order
        cg::cluster_group clu = cg::this_cluster();
        if (ln.t == 0)
            for (int r = 0; r < static_cast<int>(clu.num_blocks()); ++r)
                *clu.map_shared_rank(&sl.csq[ln.q], r) = tot;
        clu.sync();
        tot = 0.0;
        for (int r = 0; r < static_cast<int>(clu.num_blocks()); ++r) tot += sl.csq[r];
    }
    return tot;
}

// 1024-aligned base inside the dynamic smem window, kept as a __shared__-
// derived pointer so every access compiles to LDS/STS
__device__ __forceinline__ char* smem_base(unsigned char* raw) {
#ifdef ATM_GENERIC_SMEM
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
#else
    const uint32_t mis = smem_u32(raw) & 1023u;
    return reinterpret_cast<char*>(raw + ((1024u - mis) & 1023u));
#endif
}

__host__ __device__ inline int row_bytes_al(int pitch) { return ((pitch * 8) + 1023) & ~1023; }

// --------------------------------------------------------------------------
// sweep kernel: F / fused FCF / C-relax / residual jobs over C-point indices
// smem: [S seed/tail][O0][O1 if n_out=2][A if add_g][Tabs][Slots]

template <int L, int NTMAX, int MINB, int P, bool CLU = false>
__global__ void __launch_bounds__(NTMAX, MINB)
    heat_sweep_kernel(const __grid_constant__ SweepArgs a, const __grid_constant__ CUtensorMap tm_u,
                      const __grid_constant__ CUtensorMap tm_g,
                      const __grid_constant__ CUtensorMap tm_out,
                      const __grid_constant__ CUtensorMap tm_uw,
                      const __grid_constant__ CUtensorMap tm_outw) {
    // L >= 4: every warp stores its own 1024-aligned slice of a row with its
    // own TMA store (no CTA barrier per produced row); L = 2: whole-row store
    constexpr bool kWarpStore = (L >= 4);
    extern __shared__ unsigned char smem_raw[];
    char* base = smem_base(smem_raw);
    // CLU: rows split over the cluster -- CTA q stages / moves only its part
    const int cl_ = CLU ? a.co.cl : 1;
    const int pitch = a.co.pitch;
    const int spitch = pitch / cl_;
    const int rb = row_bytes_al(spitch);
    const int nob = a.n_out;
    char* bufS = base;
    char* bufO0 = base + rb;
    char* bufO1 = base + (nob == 2 ? 2 : 1) * rb;
    char* bufA = base + (1 + nob) * rb;
    char* tl = base + (1 + nob + (a.add_g ? 1 : 0)) * rb;
    Tabs& tb = *reinterpret_cast<Tabs*>(tl);
    Slots& sl = *reinterpret_cast<Slots*>(tl + sizeof(Tabs));
    double* ends = reinterpret_cast<double*>(tl + sizeof(Tabs) + sizeof(Slots));
    uint64_t* barS = &sl.bar[0];
    uint64_t* barA = &sl.bar[1];
    const uint32_t bytes = static_cast<uint32_t>(spitch * 8);
    const int R = pitch >> 4, RS = spitch >> 4;

    Lane<L, NTMAX / 32, CLU> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    tabs_init(tb, sl, a.co, ln.q);
    const int qoff = ln.q * RS;  // the part's first row of the [.., 16] view
    // job distribution over clusters (CLU) or CTAs
    const int cid = CLU ? static_cast<int>(blockIdx.x) / cl_ : static_cast<int>(blockIdx.x);
    const int ncid = CLU ? static_cast<int>(gridDim.x) / cl_ : static_cast<int>(gridDim.x);
    if (t == 0) {
        mbar_init(barS, 1);
        mbar_init(barA, 1);
        mbar_fence_init();
        prefetch_tmap(&tm_u);
    }
    __syncthreads();
    if constexpr (CLU) cg::this_cluster().sync();  // every part of the row running before DSMEM use
    uint32_t phS = 0, phA = 0;
    int ob = 0;

    const long long Nj = a.j1 - a.j0;
    const int jb = a.j0 + static_cast<int>(Nj * cid / ncid);
    const int je = a.j0 + static_cast<int>(Nj * (cid + 1) / ncid);
    const int m = a.m, last = a.np - 1;
    // C-point-only u (u_div = m, F sweeps only): seed / tail rows J, J + 1
    const bool cpu = a.u_div > 1;
    const int ub = cpu ? a.u_base / a.u_div : a.u_base;
    bool seed_ready = false;
    const bool plain = (P == 0) && !a.add_g && !a.forced && a.co.substeps == 1;
    double x[L];

    // stage x into an output buffer and TMA-store it.  Per-warp stores: the
    // warp's lane 0 waits for the reads of its previous store from that
    // buffer only now, after the Phi (which the TMA read overlapped), and
    // __syncwarp hands the slice to the warp's lanes
    auto stage_out = [&](int row, const CUtensorMap* map, const CUtensorMap* mapw) {
        char* o = ob ? bufO1 : bufO0;
        if constexpr (kWarpStore) {
            if (ln.lane == 0) {
                if (nob == 2) bulk_wait_read<1>();
                else bulk_wait_read<0>();
            }
            __syncwarp();
        }
        row_store<L>(o, x, ln);
        fence_proxy_async();
        if constexpr (kWarpStore) {
            __syncwarp();
            const int gw = ln.q * ln.nw + ln.warp;  // warp of the row (cluster rows: CTA q's part)
            if (ln.lane == 0 && gw * 32 * L < pitch) {
                // streaming u rows (an array far larger than the L2): evict_first;
                // the policy is made here so that no register holds it across the Phi
                if (a.st_hint && mapw == &tm_uw)
                    tma_store_3d_hint(mapw, 0, gw * 2 * L, row, o + ln.warp * 256 * L,
                                      a.st_hint == 2 ? l2_policy_evict_last() : l2_policy_evict_first());
                else tma_store_3d(mapw, 0, gw * 2 * L, row, o + ln.warp * 256 * L);
                bulk_commit();
            }
        } else {
            __syncthreads();
            if (t == 0) {
                tma_store_row(map, 0, row * R + qoff, o, RS);
                bulk_commit();
            }
        }
        ob = (nob == 2) ? ob ^ 1 : 0;
    };
    // whole-row stores (L = 2): the issuer waits for the reads of the store
    // that last used the buffer before the Phi, whose barrier orders the rest
    auto release_staging = [&]() {
        if (!kWarpStore && t == 0) {
            if (nob == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
        }
    };

    for (int J = jb; J < je; ++J) {
        const int c = J * m;
        int start, end, store_from;
        switch (a.kind) {
            case SW_FCF:
                start = (J == 0) ? 0 : c - m;
                store_from = (J == 0) ? 1 : c;
                end = min(c + m - 1, last);
                break;
            case SW_CRELAX:
                start = c - 1;
                end = c;
                store_from = c;
                break;
            case SW_RESID:
                start = c - 1;
                end = c - 1;
                store_from = INT_MAX;
                break;
            default:  // SW_F
                start = c;
                end = min(c + m - 1, last);
                store_from = c + 1;
                break;
        }
        if (end < start) end = start;
        const int tail_i =
            (a.tail != TAIL_NONE && end + 1 <= last && ((end + 1) % m) == 0) ? end + 1 : -1;

        // ---- seed row
        if (!seed_ready) {
            if (t == 0) {
                mbar_expect_tx(barS, bytes);
                tma_load_row(bufS, &tm_u, 0, ((cpu ? J : start) - ub) * R + qoff, barS, RS);
            }
            mbar_wait(barS, phS);
            phS ^= 1;
        }
        row_load<L>(bufS, x, ln);
        fence_proxy_async();  // our reads of S before the TMA refill (WAR)
        __syncthreads();
        seed_ready = false;
        if (tail_i >= 0 && t == 0) {
            mbar_expect_tx(barS, bytes);
            tma_load_row(bufS, &tm_u, 0, ((cpu ? J + 1 : tail_i) - ub) * R + qoff, barS, RS);
        }

        // ---- chain steps u_i = Phi_i(u_{i-1}) (+ g_i)
        // Plain heat steps (one sub-step, no forcing, no stored g) with none
        // or all of the rows stored run loops without the per-step checks:
        // the Phi is latency-bound, and each uniform branch costs its issue
        // slot plus a reconvergence on the critical path.
        if (plain && !(store_from <= end && a.store != STORE_NONE)) {
            for (int i = start + 1; i <= end; ++i) tri_solve<L>(x, a.co, ln, tb, sl);
        } else if (plain && a.store == STORE_ALL && store_from == start + 1) {
            for (int i = start + 1; i <= end; ++i) {
                release_staging();
                tri_solve<L>(x, a.co, ln, tb, sl);
                stage_out(i - a.u_base, &tm_u, &tm_uw);
            }
        } else for (int i = start + 1; i <= end; ++i) {
            if (a.add_g && t == 0) {
                mbar_expect_tx(barA, bytes);
                tma_load_row(bufA, &tm_g, 0, (i - a.g_base) * R + qoff, barA, RS);
            }
            release_staging();
            phi_p<P, L>(x, a.co, ln, tb, sl, ends, i, a.forced);
            if (a.add_g) {
                mbar_wait(barA, phA);
                phA ^= 1;
                row_acc<L>(bufA, x, ln, false);
            }
            if (a.add_g) {
                // bufA consumed by every warp before the next step refills it
                // (the per-warp stores below carry no CTA barrier)
                fence_proxy_async();
                __syncthreads();
            }
            if (i >= store_from && store_row(a.store, i, m)) stage_out(i - a.u_base, &tm_u, &tm_uw);
        }

        // ---- tail: residual at the next C-point, r = Phi(u_last) + g_c - u_c
        if (tail_i >= 0) {
            if (a.add_g && t == 0) {
                mbar_expect_tx(barA, bytes);
                tma_load_row(bufA, &tm_g, 0, (tail_i - a.g_base) * R + qoff, barA, RS);
            }
            release_staging();
            if (plain) tri_solve<L>(x, a.co, ln, tb, sl);
            else phi_p<P, L>(x, a.co, ln, tb, sl, ends, tail_i, a.forced);
            if (a.add_g) {
                mbar_wait(barA, phA);
                phA ^= 1;
                row_acc<L>(bufA, x, ln, false);
            }
            mbar_wait(barS, phS);
            phS ^= 1;
            row_acc<L>(bufS, x, ln, true);
            if (a.kind == SW_F && J + 1 < je) seed_ready = true;  // S holds u[c_{J+1}]
            if (a.tail == TAIL_STORE) {
                stage_out(tail_i / m - a.out_base, &tm_out, &tm_outw);
            } else {
                const double tot = cta_sum_squares<L>(x, ln, sl);
                if (t == 0) a.sq[(tail_i - a.sq_base) / a.sq_div] = tot;
                if (a.tail == TAIL_BOTH) stage_out(tail_i / m - a.out_base, &tm_out, &tm_outw);
            }
        }
    }
    if (kWarpStore ? (ln.lane == 0) : (t == 0)) bulk_wait<0>();
    if constexpr (CLU) cg::this_cluster().sync();  // peers may still write our smem (DSMEM)
}

// --------------------------------------------------------------------------
// linear window kernel (kernels.cpp:53-61 + solver.cpp:271-278):
// e = r_lo, e = Psi_s(e) + r_s, fine u[c_p] += e.  Jobs are interleaved over
// CTAs (concurrent CTAs share r rows in L2); the r rows of the CTA's jobs
// form one stream, double-buffered two rows ahead; the fine C-point row is
// fetched into S ahead of its emit, updated in place and stored back.
// smem: [A0][A1][S][Tabs][Slots]

template <int L, int NTMAX, int MINB, int P, bool CLU = false>
__global__ void __launch_bounds__(NTMAX, MINB)
    heat_window_linear_kernel(const __grid_constant__ WindowArgs a,
                              const __grid_constant__ CUtensorMap tm_r,
                              const __grid_constant__ CUtensorMap tm_fine) {
    extern __shared__ unsigned char smem_raw[];
    char* base = smem_base(smem_raw);
    // CLU: rows split over the cluster -- CTA q stages / moves only its part
    const int cl_ = CLU ? a.co.cl : 1;
    const int pitch = a.co.pitch;
    const int spitch = pitch / cl_;
    const int rb = row_bytes_al(spitch);
    // L = 32 (three 128-thread CTAs per SM need <= 75 KB each): two r-row
    // stream buffers and no fine-row buffer -- an emit stages e into the
    // stream buffer it has just consumed and adds it to the fine C row with a
    // TMA reduction (fp64 add in the L2; one window per row, so the sum is
    // the load-add-store's), then refills the buffer once the reduction has
    // read it
    constexpr bool RED = (L == 32);
    constexpr int NB = 2;
    char* bufA0 = base;
    char* bufA1 = base + (NB - 1) * rb;
    // fine C rows: one buffer, or three (a.two_s: long prefix chains, whose
    // emits are back to back: row s + 2 is fetched at emit s into the buffer
    // of emit s - 1, whose store has had a whole step to drain, so neither
    // the store's smem read nor the load sits on the chain)
    const int NS = RED ? 0 : (a.two_s ? 3 : 1);
    char* bufS = base + NB * rb;
    Tabs& tb = *reinterpret_cast<Tabs*>(base + (NB + NS) * rb);
    Slots& sl = *reinterpret_cast<Slots*>(base + (NB + NS) * rb + sizeof(Tabs));
    double* ends = reinterpret_cast<double*>(base + (NB + NS) * rb + sizeof(Tabs) + sizeof(Slots));
    uint64_t* barA0 = &sl.bar[0];
    uint64_t* barA1 = &sl.bar[1];
    uint64_t* barS = &sl.bar[2];  // S_b uses sl.bar[2 + b] (Slots.bar has 5)
    const uint32_t bytes = static_cast<uint32_t>(spitch * 8);
    const int R = pitch >> 4, RS = spitch >> 4;

    Lane<L, NTMAX / 32, CLU> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    tabs_init(tb, sl, a.co, ln.q);
    const int qoff = ln.q * RS;  // the part's first row of the [.., 16] view
    // job distribution over clusters (CLU) or CTAs
    const int cid = CLU ? static_cast<int>(blockIdx.x) / cl_ : static_cast<int>(blockIdx.x);
    const int ncid = CLU ? static_cast<int>(gridDim.x) / cl_ : static_cast<int>(gridDim.x);
    if (t == 0) {
        mbar_init(barA0, 1);
        mbar_init(barA1, 1);
        for (int b = 0; b < NS; ++b) mbar_init(barS + b, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if constexpr (CLU) cg::this_cluster().sync();  // every part of the row running before DSMEM use
    uint32_t ph0 = 0, ph1 = 0, phS = 0;  // phS: bit b = phase of S_b

    const bool has_pre = a.pre_e1 >= a.pre_e0;
    const int n_ind = max(0, a.p1 - a.p0 + 1);
    const int Nj = (has_pre ? 1 : 0) + n_ind;
    const int G = ncid;
    if (cid >= Nj) return;  // (a cluster's CTAs share cid: they leave together)

    auto job_range = [&](int q, int& lo, int& e0, int& e1) {
        if (has_pre && q == 0) {
            lo = a.pre_lo;
            e0 = a.pre_e0;
            e1 = a.pre_e1;
        } else {
            const int p = a.p0 + q - (has_pre ? 1 : 0);
            lo = max(0, p - a.k + 1);
            e0 = e1 = p;
        }
    };
    // issue stream (thread 0): (iq, is_) = next r row to load
    int iq = cid, is_ = 0, ilo = 0, ie0 = 0, ie1 = -1;
    job_range(iq, ilo, ie0, ie1);
    is_ = ilo;
    auto issue_next = [&](int buf) {
        if (iq >= Nj) return;
        uint64_t* bar = buf ? barA1 : barA0;
        mbar_expect_tx(bar, bytes);
        tma_load_row(buf ? bufA1 : bufA0, &tm_r, 0, (is_ - a.x1_base) * R + qoff, bar, RS);
        if (++is_ > ie1) {
            iq += G;
            if (iq < Nj) {
                job_range(iq, ilo, ie0, ie1);
                is_ = ilo;
            }
        }
    };
    if (t == 0) {
        issue_next(0);
        if (NB == 2) issue_next(1);
    }
    int cb = 0;  // buffer of the next row to consume
    const bool plain = (P == 0) && !a.forced && a.co.substeps == 1;
    double x[L];
    auto consume = [&](bool add) {
        if (cb) {
            mbar_wait(barA1, ph1);
            ph1 ^= 1;
        } else {
            mbar_wait(barA0, ph0);
            ph0 ^= 1;
        }
        const char* buf = cb ? bufA1 : bufA0;
        if (add) row_acc<L>(buf, x, ln, false);
        else row_load<L>(buf, x, ln);
        fence_proxy_async();  // generic reads before the TMA refill (WAR)
        __syncthreads();
        if (t == 0) issue_next(cb);
        if (NB == 2) cb ^= 1;
    };

    if constexpr (RED) {
        // consume row s of the stream; when the step emits, the consumed
        // buffer carries e to the fine row before it is refilled
        auto step = [&](bool add, bool emit, int s) {
            if (cb) {
                mbar_wait(barA1, ph1);
                ph1 ^= 1;
            } else {
                mbar_wait(barA0, ph0);
                ph0 ^= 1;
            }
            char* buf = cb ? bufA1 : bufA0;
            if (add) row_acc<L>(buf, x, ln, false);
            else row_load<L>(buf, x, ln);
            if (emit) row_store<L>(buf, x, ln);  // each thread rewrites only what it read
            fence_proxy_async();  // reads before the refill (WAR), writes before the reduction
            __syncthreads();
            if (t == 0) {
                if (emit) {
                    tma_reduce_row(&tm_fine, 0, (s * a.out_stride - a.out_base) * R + qoff, buf, RS);
                    bulk_commit();
                    bulk_wait_read<0>();
                }
                issue_next(cb);
            }
            cb ^= 1;
        };
        for (int q = cid; q < Nj; q += G) {
            int lo, e0, e1;
            job_range(q, lo, e0, e1);
            step(false, lo >= e0, lo);  // e = r_lo
            for (int s = lo + 1; s <= e1; ++s) {
                if (plain) tri_solve<L>(x, a.co, ln, tb, sl);
                else phi_p<P, L>(x, a.co, ln, tb, sl, ends, s, a.forced);
                step(true, s >= e0, s);  // e = Psi(e) + r_s
            }
        }
    } else
    for (int q = cid; q < Nj; q += G) {
        int lo, e0, e1;
        job_range(q, lo, e0, e1);
        consume(false);  // e = r_lo
        const int f0 = max(e0, lo);  // first emitted C row of the job
        if (t == 0) {
            bulk_wait_read<0>();  // S free again
            for (int b = 0; b < (NS == 1 ? 1 : NS - 1) && f0 + b <= e1; ++b) {
                mbar_expect_tx(barS + b, bytes);
                tma_load_row(bufS + b * rb, &tm_fine, 0, ((f0 + b) * a.out_stride - a.out_base) * R + qoff,
                            barS + b, RS);
            }
        }
        for (int s = lo; s <= e1; ++s) {
            if (s > lo) {
                if (plain) tri_solve<L>(x, a.co, ln, tb, sl);
                else phi_p<P, L>(x, a.co, ln, tb, sl, ends, s, a.forced);
                consume(true);  // e = Psi(e) + r_s
            }
            if (s >= e0) {
                // fine.u[c_s] += e (emits rotate over the NS buffers)
                const int sb = (NS == 1) ? 0 : (s - f0) % NS;
                char* bs = bufS + sb * rb;
                mbar_wait(barS + sb, (phS >> sb) & 1);
                phS ^= 1u << sb;
                double y[L];
                row_load<L>(bs, y, ln);
#pragma unroll
                for (int e = 0; e < L; ++e) y[e] += x[e];
                row_store<L>(bs, y, ln);
                fence_proxy_async();
                __syncthreads();
                if (t == 0) {
                    tma_store_row(&tm_fine, 0, (s * a.out_stride - a.out_base) * R + qoff, bs, RS);
                    bulk_commit();
                    if (NS == 1) {
                        if (s + 1 <= e1) {
                            bulk_wait_read<0>();
                            mbar_expect_tx(barS, bytes);
                            tma_load_row(bufS, &tm_fine, 0, ((s + 1) * a.out_stride - a.out_base) * R + qoff,
                                        barS, RS);
                        }
                    } else if (s + NS - 1 <= e1) {
                        // row s + NS - 1 goes to the buffer of emit s - 1 (for
                        // s = f0 the never-used last buffer): all stores but
                        // this emit's have finished reading
                        const int nb = (s - f0 + NS - 1) % NS;
                        bulk_wait_read<1>();
                        mbar_expect_tx(barS + nb, bytes);
                        tma_load_row(bufS + nb * rb, &tm_fine, 0,
                                    ((s + NS - 1) * a.out_stride - a.out_base) * R + qoff, barS + nb, RS);
                    }
                }
            }
        }
    }
    if (t == 0) bulk_wait<0>();
    if constexpr (CLU) cg::this_cluster().sync();  // peers may still write our smem (DSMEM)
}

// --------------------------------------------------------------------------
// generic window kernel: FAS windows (kernels.cpp:63-77), nested forward
// windows (kernels.cpp:79-88), batched single-step applications (Phi of
// given rows, forcing, Psi(v_{j-1})) and the FAS coarse right-hand side
// (solver.cpp:214-218).  smem: [O0][O1][A1][A2][A3][Tabs][Slots]

template <int L, int NTMAX, int MINB, int P, bool CLU = false>
__global__ void __launch_bounds__(NTMAX, MINB)
    heat_window_kernel(const __grid_constant__ WindowArgs a,
                       const __grid_constant__ CUtensorMap tm_x1,
                       const __grid_constant__ CUtensorMap tm_x2,
                       const __grid_constant__ CUtensorMap tm_x3,
                       const __grid_constant__ CUtensorMap tm_out) {
    extern __shared__ unsigned char smem_raw[];
    char* base = smem_base(smem_raw);
    // CLU: rows split over the cluster -- CTA q stages / moves only its part
    const int cl_ = CLU ? a.co.cl : 1;
    const int pitch = a.co.pitch;
    const int spitch = pitch / cl_;
    const int rb = row_bytes_al(spitch);
    char* bufO0 = base;
    char* bufO1 = base + rb;
    char* bufA1 = base + 2 * rb;
    char* bufA2 = base + 3 * rb;
    char* bufA3 = base + 4 * rb;
    const bool three = (a.kind == WK_FAS || a.kind == WK_FAS_RHS);
    char* tl = base + (three ? 5 : 3) * rb;
    Tabs& tb = *reinterpret_cast<Tabs*>(tl);
    Slots& sl = *reinterpret_cast<Slots*>(tl + sizeof(Tabs));
    double* ends = reinterpret_cast<double*>(tl + sizeof(Tabs) + sizeof(Slots));
    uint64_t* barA = &sl.bar[1];
    const uint32_t bytes = static_cast<uint32_t>(spitch * 8);
    const int R = pitch >> 4, RS = spitch >> 4;

    Lane<L, NTMAX / 32, CLU> ln;
    lane_init<L>(ln, a.co);
    const int t = ln.t;
    tabs_init(tb, sl, a.co, ln.q);
    const int qoff = ln.q * RS;  // the part's first row of the [.., 16] view
    // job distribution over clusters (CLU) or CTAs
    const int cid = CLU ? static_cast<int>(blockIdx.x) / cl_ : static_cast<int>(blockIdx.x);
    const int ncid = CLU ? static_cast<int>(gridDim.x) / cl_ : static_cast<int>(gridDim.x);
    if (t == 0) {
        mbar_init(barA, 1);
        mbar_fence_init();
    }
    __syncthreads();
    if constexpr (CLU) cg::this_cluster().sync();  // every part of the row running before DSMEM use
    uint32_t phA = 0;
    int ob = 0;

    const bool has_pre = (a.kind == WK_FAS || a.kind == WK_FORWARD) && (a.pre_e1 >= a.pre_e0);
    const int n_ind = max(0, a.p1 - a.p0 + 1);
    const int Nj = (has_pre ? 1 : 0) + n_ind;
    double x[L];

    auto emit_store = [&](int row) {
        char* o = ob ? bufO1 : bufO0;
        // the store issued two emits ago read this buffer: wait for it
        if (t == 0) bulk_wait_read<1>();
        __syncthreads();
        row_store<L>(o, x, ln);
        fence_proxy_async();
        __syncthreads();
        if (t == 0) {
            tma_store_row(&tm_out, 0, (row - a.out_base) * R + qoff, o, RS);
            bulk_commit();
        }
        ob ^= 1;
    };

    for (int q = cid; q < Nj; q += ncid) {
        if (a.kind == WK_APPLY || a.kind == WK_FAS_RHS) {
            const int p = a.p0 + q;
            const int src = (a.kind == WK_FAS_RHS) ? p - 1 : p + a.seed_off;
            const uint32_t nb = a.seed_zero ? 0u : bytes;
            const uint32_t extra = (a.kind == WK_FAS_RHS) ? 2 * bytes : 0u;
            if (t == 0 && nb + extra) {
                mbar_expect_tx(barA, nb + extra);
                if (!a.seed_zero) tma_load_row(bufA1, &tm_x1, 0, (src - a.x1_base) * R + qoff, barA, RS);
                if (a.kind == WK_FAS_RHS) {
                    tma_load_row(bufA2, &tm_x2, 0, (p - a.x2_base) * R + qoff, barA, RS);
                    tma_load_row(bufA3, &tm_x3, 0, (p - a.x3_base) * R + qoff, barA, RS);
                }
            }
            if (nb + extra) {
                mbar_wait(barA, phA);
                phA ^= 1;
            }
            if (a.seed_zero) {
#pragma unroll
                for (int e = 0; e < L; ++e) x[e] = 0.0;
            } else {
                row_load<L>(bufA1, x, ln);
            }
            if (t == 0) bulk_wait_read<1>();
            phi_p<P, L>(x, a.co, ln, tb, sl, ends, a.idx0 + p, a.forced);
            if (a.kind == WK_FAS_RHS) {
                // g_j = (v_j - Psi_j(v_{j-1})) + r_j  (solver.cpp:214-218)
                double y[L];
                row_load<L>(bufA2, y, ln);
#pragma unroll
                for (int e = 0; e < L; ++e) y[e] -= x[e];
                row_acc<L>(bufA3, y, ln, false);
#pragma unroll
                for (int e = 0; e < L; ++e) x[e] = y[e];
            }
            emit_store(p);  // its fence + barrier also release bufA*
            continue;
        }

        int lo, e0, e1;
        if (has_pre && q == 0) {
            lo = a.pre_lo;
            e0 = a.pre_e0;
            e1 = a.pre_e1;
        } else {
            const int p = a.p0 + q - (has_pre ? 1 : 0);
            lo = max(0, p - a.k + 1);
            e0 = e1 = p;
        }
        // ---- seed: v_lo + r_lo (FAS), u_lo (forward)
        const bool fas = (a.kind == WK_FAS);
        if (t == 0) {
            mbar_expect_tx(barA, fas ? 2 * bytes : bytes);
            tma_load_row(bufA1, &tm_x1, 0, (lo - a.x1_base) * R + qoff, barA, RS);
            if (fas) tma_load_row(bufA2, &tm_x2, 0, (lo - a.x2_base) * R + qoff, barA, RS);
        }
        mbar_wait(barA, phA);
        phA ^= 1;
        if (fas) {
            row_load<L>(bufA2, x, ln);         // v_lo
            row_acc<L>(bufA1, x, ln, false);   // + r_lo
        } else {
            row_load<L>(bufA1, x, ln);
        }
        fence_proxy_async();
        __syncthreads();
        if (lo >= e0) emit_store(lo);
        for (int s = lo + 1; s <= e1; ++s) {
            if (t == 0 && fas) {
                mbar_expect_tx(barA, 3 * bytes);
                tma_load_row(bufA1, &tm_x1, 0, (s - a.x1_base) * R + qoff, barA, RS);
                tma_load_row(bufA2, &tm_x2, 0, (s - a.x2_base) * R + qoff, barA, RS);
                tma_load_row(bufA3, &tm_x3, 0, (s - a.x3_base) * R + qoff, barA, RS);
            }
            if (t == 0) bulk_wait_read<1>();
            phi_p<P, L>(x, a.co, ln, tb, sl, ends, s, a.forced);
            if (fas) {
                mbar_wait(barA, phA);
                phA ^= 1;
                // next = Psi(u) + v_s - Psi(v_{s-1}) + r_s  (kernels.cpp:69-74)
                row_acc<L>(bufA2, x, ln, false);
                row_acc<L>(bufA3, x, ln, true);
                row_acc<L>(bufA1, x, ln, false);
                fence_proxy_async();
                __syncthreads();
            }
            if (s >= e0) emit_store(s);
        }
    }
    if (t == 0) bulk_wait<0>();
    if constexpr (CLU) cg::this_cluster().sync();  // peers may still write our smem (DSMEM)
}

// --------------------------------------------------------------------------
// host launchers

// Allen-Cahn kernels also keep the chunk ends of the Newton residual
static size_t ends_bytes(const HeatCoefDev& co) {
    return co.prob == 1 ? sizeof(double) * 4 * static_cast<size_t>(co.nt) : 0;
}

// staged part of a row per CTA (cluster rows: 1 / cl of it)
static int staged_pitch(const HeatCoefDev& co) { return co.cl > 1 ? co.pitch / co.cl : co.pitch; }

size_t heat_sweep_smem(const SweepArgs& a) {
    const int rows = 1 + a.n_out + (a.add_g ? 1 : 0);
    return 1024 + static_cast<size_t>(rows) * row_bytes_al(staged_pitch(a.co)) + sizeof(Tabs) +
           sizeof(Slots) + ends_bytes(a.co);
}

size_t heat_window_smem(const WindowArgs& a) {
    int rows;
    if (a.kind == WK_LINEAR) rows = (a.co.L == 32 ? 2 : 3) + (a.two_s ? 2 : 0);
    else rows = (a.kind == WK_FAS || a.kind == WK_FAS_RHS) ? 5 : 3;
    return 1024 + static_cast<size_t>(rows) * row_bytes_al(staged_pitch(a.co)) + sizeof(Tabs) +
           sizeof(Slots) + ends_bytes(a.co);
}

namespace {

struct KernelPtrs {
    const void* sweep;
    const void* wlin;
    const void* win;
};

template <int L, int NT, int MB, bool CLU = false>
KernelPtrs kptrs() {
    return {reinterpret_cast<const void*>(heat_sweep_kernel<L, NT, MB, 0, CLU>),
            reinterpret_cast<const void*>(heat_window_linear_kernel<L, NT, MB, 0, CLU>),
            reinterpret_cast<const void*>(heat_window_kernel<L, NT, MB, 0, CLU>)};
}

// heat: L=16 serves 2048 < n <= 4096 with 256 threads; smaller L use up to
// 512.  Allen-Cahn (Newton Phi, FAS only): L = 8, up to 512 threads.
KernelPtrs select(const HeatCoefDev& co) {
    if (co.prob == 1) {
        // P = 2: n not a multiple of L (the last real chunk is partial)
        if (co.pl != co.L)
            return {reinterpret_cast<const void*>(heat_sweep_kernel<8, 512, 1, 2>), nullptr,
                    reinterpret_cast<const void*>(heat_window_kernel<8, 512, 1, 2>)};
        return {reinterpret_cast<const void*>(heat_sweep_kernel<8, 512, 1, 1>), nullptr,
                reinterpret_cast<const void*>(heat_window_kernel<8, 512, 1, 1>)};
    }
    // rows split over a cluster (n > 5376): every CTA a 4096-element part
    if (co.cl > 1) return kptrs<32, 128, 3, true>();
    // 4096 < n <= 5376: L = 32 with 256 threads (sweeps), L = 16 with up to
    // 512 (the coarsest level's windows)
    switch (co.L) {
        case 2: return kptrs<2, 512, 1>();
        case 4: return kptrs<4, 512, 1>();
        case 8: return kptrs<8, 512, 1>();
        case 32: return co.nt > 128 ? kptrs<32, 256, 1>() : kptrs<32, 128, 3>();
        default: return co.nt > 256 ? kptrs<16, 512, 1>() : kptrs<16, 256, 2>();
    }
}

void prepare(const void* fn) {
    static std::mutex mu;
    static std::map<const void*, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done[fn]) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    done[fn] = true;
}

int occupancy(const void* fn, int nt, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t>, int> cache;
    prepare(fn);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(fn, nt, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, nt, smem) != cudaSuccess) n = 1;
    n = std::max(1, n);
    cache[key] = n;
    return n;
}

// cluster rows: clusters of cl CTAs that can be resident at once
int max_clusters(const void* fn, int nt, size_t smem, int cl) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
    prepare(fn);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(fn, nt, smem, cl);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    // clusters of 9-16 CTAs are non-portable (opt-in)
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cfg.gridDim = dim3(cl * sms);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = 1;
    }
    cache[key] = n;
    return n;
}

// grid: CTAs, or for cluster rows (cl > 1) clusters, capped at what fits
int launch(const void* fn, int grid, int nt, size_t smem, cudaStream_t s, void** args, int cl = 1) {
    prepare(fn);
    if (cl <= 1) return static_cast<int>(cudaLaunchKernel(fn, dim3(grid), dim3(nt), args, smem, s));
    const int ncl = std::min(grid, max_clusters(fn, nt, smem, cl));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ncl * cl);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelExC(&cfg, fn, args));
}

}  // namespace

// CTAs per SM, or for cluster rows the clusters per SM rounded up (the
// launch caps the grid at the resident clusters)
int heat_sweep_occupancy(const SweepArgs& a) {
    const void* fn = select(a.co).sweep;
    if (a.co.cl > 1) return 1;
    return occupancy(fn, a.co.nt, heat_sweep_smem(a));
}

int heat_window_occupancy(const WindowArgs& a) {
    const KernelPtrs k = select(a.co);
    if (a.co.cl > 1) return 1;
    return occupancy(a.kind == WK_LINEAR ? k.wlin : k.win, a.co.nt, heat_window_smem(a));
}

int launch_heat_sweep(const SweepArgs& a, const CUtensorMap& u, const CUtensorMap& g,
                      const CUtensorMap& o, const CUtensorMap& uw, const CUtensorMap& ow, int grid,
                      cudaStream_t s) {
    if (grid <= 0) return 0;
    SweepArgs aa = a;
    CUtensorMap tu = u, tg = g, to = o, tuw = uw, tow = ow;
    void* args[] = {&aa, &tu, &tg, &to, &tuw, &tow};
    return launch(select(a.co).sweep, grid, a.co.nt, heat_sweep_smem(a), s, args, a.co.cl);
}

int launch_heat_window(const WindowArgs& a, const CUtensorMap& x1, const CUtensorMap& x2,
                       const CUtensorMap& x3, const CUtensorMap& o, int grid, cudaStream_t s) {
    if (grid <= 0) return 0;
    WindowArgs aa = a;
    CUtensorMap t1 = x1, t2 = x2, t3 = x3, to = o;
    const KernelPtrs k = select(a.co);
    if (a.kind == WK_LINEAR && !k.wlin) return static_cast<int>(cudaErrorInvalidValue);
    if (a.kind == WK_LINEAR) {
        void* args[] = {&aa, &t1, &to};
        return launch(k.wlin, grid, a.co.nt, heat_window_smem(a), s, args, a.co.cl);
    }
    void* args[] = {&aa, &t1, &t2, &t3, &to};
    return launch(k.win, grid, a.co.nt, heat_window_smem(a), s, args, a.co.cl);
}

}  // namespace atm
