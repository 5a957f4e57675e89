// Batched blocked Householder QR / complement / Jacobi orchestration.
//
// Every panel step advances all clusters of a batch together: one
// cooperative panel launch (k_hh.cu, the clusters' CTA groups side by side,
// in waves if they do not fit co-resident), then the trailing update
// A -= V T^T (V^T A) as a split-K DMMA GEMM, a T multiply and a DMMA GEMM.
#include "dense.h"

#include <algorithm>
#include <cstdlib>
#include <map>

#include "builders.h"

namespace h2f {

namespace {

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

constexpr int KCH = 1024;  // split-K chunk of the V^T A product

struct PanelPlan {
    int job, j0, nbp, Lp, ncta, chunk;
};

// CTA allocation of one wave: at least ceil(Lp / HH_CHUNK_MAX) CTAs per
// job, spare CTAs to the jobs with the most rows per CTA while a CTA keeps
// >= 128 rows (measured: the per-column work of wide slices outweighs the
// cost of a larger barrier group)
void size_wave(std::vector<PanelPlan>& w, int cap) {
    int total = 0;
    for (auto& p : w) {
        p.ncta = int(cdiv(p.Lp, HH_CHUNK_MAX));
        total += p.ncta;
    }
    for (;;) {
        PanelPlan* best = nullptr;
        double most = 0;
        for (auto& p : w) {
            const double per = double(p.Lp) / p.ncta;
            if (per >= 2.0 * 128 && per > most) {
                most = per;
                best = &p;
            }
        }
        if (!best || total >= cap) break;
        ++best->ncta;
        ++total;
    }
    for (auto& p : w) {
        int ch = int(cdiv(p.Lp, p.ncta));
        ch = std::max(HH_NB, (ch + 3) & ~3);
        p.chunk = ch;
        p.ncta = int(cdiv(p.Lp, ch));
    }
}

}  // namespace

void hh_factor(std::vector<HhJob>& jobs, Region& scr, bool keep) {
    cudaStream_t st = ctx().stream;
    const int cap = hh_panel_capacity(HH_CHUNK_MAX);
    if (cap < 1) throw Error(H2F_E_INTERNAL, "assertion: Householder panel kernel cannot be resident");
    int maxp = 0;
    std::vector<double*> vbuf(jobs.size(), nullptr);
    for (size_t i = 0; i < jobs.size(); ++i) {
        maxp = std::max<int>(maxp, int(cdiv(jobs[i].nfac, HH_NB)));
        jobs[i].Vt.clear();
        jobs[i].T.clear();
        if (!keep && jobs[i].nfac > 0 && jobs[i].M) vbuf[i] = scr.alloc_n<double>(int64_t(HH_NB) * jobs[i].L);
    }
    // block column pivoting: per job scratch, identity permutation
    struct PivScratch { double* norms; int32_t* order; int32_t* perm_tmp; double* tmp; };
    std::vector<PivScratch> piv(jobs.size(), PivScratch{nullptr, nullptr, nullptr, nullptr});
    for (size_t i = 0; i < jobs.size(); ++i) {
        HhJob& J = jobs[i];
        if (!J.perm || !J.M) continue;
        piv[i] = PivScratch{scr.alloc_n<double>(J.ntot), scr.alloc_n<int32_t>(J.ntot), scr.alloc_n<int32_t>(J.ntot),
                            scr.alloc_n<double>(int64_t(J.ntot) * J.ldm)};
        launch_iota(J.perm, J.ntot, st);
    }
    // pivoting at the first panels only: the sweep saving of the Jacobi
    // comes from moving the large-norm columns to the front (numpy study:
    // the same sweep counts as pivoting before every panel), while each
    // pivot step copies the whole trailing matrix
    static const int piv_panels = env_int("H2F_QR_PIVOT_PANELS", 6);
    for (int p = 0; p < maxp; ++p) {
        const int j0 = p * HH_NB;
        if (p < piv_panels) {
            std::vector<PivotTask> pt;
            int max_cols = 0, max_l = 0;
            for (size_t i = 0; i < jobs.size(); ++i) {
                const HhJob& J = jobs[i];
                if (!J.perm || !J.M || j0 >= J.nfac || J.ntot - j0 < 2) continue;
                pt.push_back(PivotTask{J.M, J.ldm, J.L, j0, J.ntot, piv[i].norms, piv[i].order, J.perm, piv[i].perm_tmp,
                                       piv[i].tmp});
                max_cols = std::max(max_cols, J.ntot);
                max_l = std::max(max_l, J.L);
            }
            if (!pt.empty()) launch_pivot_panel(upload(pt), int32_t(pt.size()), max_cols, max_l, st);
            // the reordered matrix lives in the other buffer from now on
            for (size_t i = 0; i < jobs.size(); ++i) {
                HhJob& J = jobs[i];
                if (!J.perm || !J.M || j0 >= J.nfac || J.ntot - j0 < 2) continue;
                std::swap(J.M, piv[i].tmp);
            }
        }
        std::vector<PanelPlan> all;
        for (size_t i = 0; i < jobs.size(); ++i) {
            const HhJob& J = jobs[i];
            if (j0 >= J.nfac) continue;
            all.push_back({int(i), j0, std::min(HH_NB, J.nfac - j0), J.L - j0, 0, 0});
        }
        if (all.empty()) break;
        GemmBuild gk, gu;
        std::vector<HhTmulTask> tm;
        int max_trail = 0;
        // trailing update of the panel's job: columns [j0 + nbp, ntot), rows [j0, L)
        auto add_trailing = [&](const PanelPlan& pp, const HhPanelTask& k) {
            HhJob& J = jobs[pp.job];
            // trailing update of columns [j0 + nbp, ntot), rows [j0, L)
            const int ntrail = J.ntot - (pp.j0 + pp.nbp);
            if (ntrail <= 0) return;
            const int L = pp.Lp, nch = int(cdiv(L, KCH));
            double* At = J.M + int64_t(pp.j0 + pp.nbp) * J.ldm + pp.j0;  // ntrail x L, ld ldm
            double* P = scr.alloc_n<double>(int64_t(nch) * pp.nbp * ntrail);
            double* W2 = scr.alloc_n<double>(int64_t(pp.nbp) * ntrail);
            for (int c = 0; c < nch; ++c) {
                const int kk = std::min(KCH, L - c * KCH);
                gk.add1(P + int64_t(c) * pp.nbp * ntrail, ntrail, pp.nbp, ntrail, GEMM_STORE,
                        contrib(k.Vt + int64_t(c) * KCH, L, 0, At + int64_t(c) * KCH, J.ldm, 1, kk));
            }
            tm.push_back(HhTmulTask{P, k.T, W2, nch, pp.nbp, ntrail, 1});
            max_trail = std::max(max_trail, ntrail);
            gu.add1(At, J.ldm, ntrail, L, GEMM_ADD, contrib(W2, ntrail, 1, k.Vt, L, 0, pp.nbp, -1.0));

        };
        // H2F_HH_CLUSTER=1: panels of HH_CHUNK_MAX < Lp <= 16 * HH_CLUSTER_CHUNK
        // rows as one thread-block cluster each (DSMEM exchange, cluster
        // barrier).  Measured on config 2: no gain over the
        // cooperative panel -- the per-column time is the slice's own
        // dot/update/syncthreads chain, not the inter-CTA barrier -- so the
        // cooperative panel stays the default.
        static const bool no_cluster = env_int("H2F_HH_CLUSTER", 0) == 0;
        {
            std::vector<PanelPlan> rest;
            std::map<int, std::vector<HhPanelTask>> by_cl;
            std::map<int, int> cl_chunk;
            for (auto& pp : all) {
                if (no_cluster || pp.Lp <= HH_CHUNK_MAX || pp.Lp > 16 * HH_CLUSTER_CHUNK) {
                    rest.push_back(pp);
                    continue;
                }
                HhJob& J = jobs[pp.job];
                if (!J.M) {  // plan-only (sharded): nothing to launch
                    J.Vt.push_back(nullptr);
                    J.T.push_back(nullptr);
                    continue;
                }
                // cluster size: ~rows_per_cta rows per CTA (the per-column
                // dot products and updates of a slice are the work between
                // two cluster barriers), 2..16 CTAs
                static const int rows_per_cta = env_int("H2F_HH_CLUSTER_ROWS", 256);
                int cl = 2;
                while (cl < 16 && int64_t(cl) * rows_per_cta < pp.Lp) cl *= 2;
                int ch = int(cdiv(pp.Lp, cl));
                ch = std::max(HH_NB, (ch + 3) & ~3);
                HhPanelTask k{};
                k.M = J.M;
                k.ldm = J.ldm;
                k.Vt = keep ? scr.alloc_n<double>(int64_t(HH_NB) * pp.Lp) : vbuf[pp.job];
                k.T = scr.alloc_n<double>(HH_NB * HH_NB);
                k.L = J.L;
                k.j0 = pp.j0;
                k.nbp = pp.nbp;
                k.chunk = ch;
                k.ncta = cl;
                by_cl[cl].push_back(k);
                cl_chunk[cl] = std::max(cl_chunk[cl], ch);
                J.Vt.push_back(k.Vt);
                J.T.push_back(k.T);
                add_trailing(pp, k);
            }
            for (auto& kv : by_cl) {
                cudaError_t e = launch_hh_panel_cluster(upload(kv.second), int32_t(kv.second.size()), kv.first,
                                                        cl_chunk[kv.first], st);
                if (e != cudaSuccess)
                    throw Error(H2F_E_CUDA, std::string("cluster Householder panel launch: ") + cudaGetErrorString(e));
            }
            all.swap(rest);
        }
        // waves of co-resident CTA groups
        std::vector<std::vector<PanelPlan>> waves(1);
        int used = 0;
        for (auto& pp : all) {
            const int need = int(cdiv(pp.Lp, HH_CHUNK_MAX));
            if (need > cap) throw Error(H2F_E_INTERNAL, "assertion: Householder panel taller than the device");
            if (used + need > cap) {
                waves.emplace_back();
                used = 0;
            }
            waves.back().push_back(pp);
            used += need;
        }
        for (auto& w : waves) {
            size_wave(w, cap);
            std::vector<HhPanelTask> tasks;
            std::vector<int32_t> owner;
            int cta0 = 0, max_chunk = HH_NB;
            uint32_t* bars = scr.alloc_n<uint32_t>(2 * int64_t(w.size()));
            H2F_CUDA(cudaMemsetAsync(bars, 0, sizeof(uint32_t) * 2 * w.size(), st));
            for (size_t t = 0; t < w.size(); ++t) {
                const PanelPlan& pp = w[t];
                HhJob& J = jobs[pp.job];
                if (!J.M) {
                    // plan-only job (another rank's cluster in a sharded
                    // factorization): it shaped the wave, nothing to launch
                    J.Vt.push_back(nullptr);
                    J.T.push_back(nullptr);
                    continue;
                }
                HhPanelTask k{};
                k.M = J.M;
                k.ldm = J.ldm;
                k.Vt = keep ? scr.alloc_n<double>(int64_t(HH_NB) * pp.Lp) : vbuf[pp.job];
                k.T = scr.alloc_n<double>(HH_NB * HH_NB);
                k.part = scr.alloc_n<double>(int64_t(2) * (pp.ncta + 1) * (HH_NB + 2));
                k.gram = scr.alloc_n<double>(int64_t(pp.ncta) * HH_NB * HH_NB);
                k.bar = bars + 2 * tasks.size();
                k.L = J.L;
                k.j0 = pp.j0;
                k.nbp = pp.nbp;
                k.chunk = pp.chunk;
                k.cta0 = cta0;
                k.ncta = pp.ncta;
                for (int c = 0; c < pp.ncta; ++c) owner.push_back(int32_t(tasks.size()));
                tasks.push_back(k);
                cta0 += pp.ncta;
                max_chunk = std::max(max_chunk, pp.chunk);
                J.Vt.push_back(k.Vt);
                J.T.push_back(k.T);
                add_trailing(pp, k);
            }
            if (tasks.empty()) continue;
            cudaError_t e = launch_hh_panel(upload(tasks), upload(owner), int32_t(owner.size()), max_chunk, st);
            if (e != cudaSuccess)
                throw Error(H2F_E_CUDA, std::string("cooperative Householder panel launch: ") + cudaGetErrorString(e));
        }
        gk.launch(-1);
        if (!tm.empty()) launch_hh_tmul(upload(tm), int32_t(tm.size()), max_trail, st);
        gu.launch(-1);
    }
}

void hh_apply_q(const std::vector<HhJob>& jobs, const std::vector<HhApply>& xs, Region& scr) {
    cudaStream_t st = ctx().stream;
    int maxp = 0;
    for (auto& J : jobs) maxp = std::max<int>(maxp, int(J.Vt.size()));
    for (int p = maxp - 1; p >= 0; --p) {
        GemmBuild g1, g2;
        std::vector<HhTmulTask> tm;
        int max_cols = 0;
        for (size_t i = 0; i < jobs.size(); ++i) {
            const HhJob& J = jobs[i];
            const HhApply& X = xs[i];
            if (p >= int(J.Vt.size()) || X.nx <= 0 || !J.M) continue;
            const int j0 = p * HH_NB, nbp = std::min(HH_NB, J.nfac - j0), L = J.L - j0;
            double* Xp = X.X + int64_t(j0) * X.ldx;  // L x nx
            double* P = scr.alloc_n<double>(int64_t(nbp) * X.nx);
            double* W = scr.alloc_n<double>(int64_t(nbp) * X.nx);
            g1.add1(P, X.nx, nbp, X.nx, GEMM_STORE, contrib(J.Vt[p], L, 0, Xp, X.ldx, 0, L));
            tm.push_back(HhTmulTask{P, J.T[p], W, 1, nbp, X.nx, 0});
            max_cols = std::max(max_cols, X.nx);
            g2.add1(Xp, X.ldx, L, X.nx, GEMM_ADD, contrib(J.Vt[p], L, 1, W, X.nx, 0, nbp, -1.0));
        }
        g1.launch(-1);
        if (!tm.empty()) launch_hh_tmul(upload(tm), int32_t(tm.size()), max_cols, st);
        g2.launch(-1);
    }
}

void reorth_batched(const std::vector<ReorthTask>& tasks, Region& scr) {
    GemmBuild g1, g2;
    std::vector<RowNormTask> rows;
    for (auto& t : tasks) {
        const int s = t.s, k = t.k, kp = t.kept;
        double* U = t.BT + int64_t(k) * s;  // kept x s, the rows to orthogonalise
        if (k > 0) {
            double* Cm = scr.alloc_n<double>(int64_t(k) * kp);
            // C (k x kp) = V^T U^T ;  U -= C^T V^T
            g1.add1(Cm, kp, k, kp, GEMM_STORE, contrib(t.V, t.ldv, 1, U, s, 1, s));
            g2.add1(U, s, kp, s, GEMM_ADD, contrib(Cm, kp, 1, t.V, t.ldv, 1, k, -1.0));
        }
        for (int j = 0; j < kp; ++j) rows.push_back(RowNormTask{U + int64_t(j) * s, s, 0});
    }
    g1.launch(-1);
    g2.launch(-1);
    launch_normalize_rows(upload(rows), int32_t(rows.size()), ctx().stream);
}

void qr_r_blocked(const std::vector<QrTask>& tasks, Region& scr, const std::vector<int32_t*>* perms) {
    std::vector<HhJob> jobs;
    std::vector<RExtractTask> ex;
    int maxn = 0;
    for (size_t ti = 0; ti < tasks.size(); ++ti) {
        const QrTask& t = tasks[ti];
        HhJob J;
        if (perms) J.perm = (*perms)[ti];
        J.M = t.Y;
        J.ldm = t.ldy;
        J.L = t.wf;
        J.ntot = t.s;
        J.nfac = std::min(t.s, t.wf);
        jobs.push_back(J);
        maxn = std::max(maxn, t.s);
    }
    hh_factor(jobs, scr, false);
    // R from each job's final buffer (pivoted jobs alternate between two)
    for (size_t ti = 0; ti < tasks.size(); ++ti)
        if (tasks[ti].Y) ex.push_back(RExtractTask{jobs[ti].M, tasks[ti].R, tasks[ti].ldy, jobs[ti].nfac, tasks[ti].s});
    if (!ex.empty()) launch_r_extract(upload(ex), int32_t(ex.size()), maxn, ctx().stream);
}

void complement_blocked(const std::vector<ComplementTask>& tasks, Region& scr) {
    cudaStream_t st = ctx().stream;
    std::vector<HhJob> jobs;
    std::vector<HhApply> xs;
    std::vector<EyeTask> eye;
    CopyBuild cp, zero;
    int maxr = 0;
    for (auto& t : tasks) {
        const int s = t.s, kt = t.kt, r = s - kt;
        HhJob J;
        J.M = t.W;
        J.ldm = s;
        J.L = s;
        J.ntot = kt;
        J.nfac = kt;
        jobs.push_back(J);
        if (!t.W) {  // plan-only (sharded factorization): shapes the waves only
            xs.push_back(HhApply{nullptr, s, 0});
            continue;
        }
        cp.add(t.W, s, kt, s, t.BT, s, 0, COPY_SET);     // the QR works on a copy of b_aug
        cp.add(t.Q + r, s, s, kt, t.BT, s, 1, COPY_SET);  // trailing columns: b_aug itself
        zero.zero(t.Q, s, s, r);
        if (r > 0) eye.push_back(EyeTask{t.Q, s, kt, r});
        xs.push_back(HhApply{t.Q, s, r});
        maxr = std::max(maxr, r);
    }
    zero.launch();
    cp.launch();
    if (!eye.empty()) launch_set_eye(upload(eye), int32_t(eye.size()), maxr, st);
    hh_factor(jobs, scr, true);
    hh_apply_q(jobs, xs, scr);
}

void blocked_lu(double* A, int64_t n, int32_t* piv, Region& scr, double* red, int kid_panel, int kid_misc,
                int kid_gemm) {
    cudaStream_t st = ctx().stream;
    if (n == 0) return;
    launch_absmax(A, n, int(n), int(n), red, st);
    const int nb = TOP_PANEL_NB;
    const int g = top_panel_grid(int(n));
    TopPanelScratch ps;
    ps.val = scr.alloc_n<double>(2 * g);
    ps.idx = scr.alloc_n<int>(2 * g);
    ps.rows = scr.alloc_n<double>(int64_t(2) * g * TOP_PANEL_NB);
    ps.rowk = scr.alloc_n<double>(2 * TOP_PANEL_NB);
    ps.bar = scr.alloc_n<unsigned>(2);
    for (int64_t k0 = 0; k0 < n; k0 += nb) {
        const int w = int(std::min<int64_t>(nb, n - k0));
        {
            ProfScope p(kid_panel, double(n - k0) * w * w, 16.0 * double(n - k0) * w);
            if (!launch_coop_panel_lu(A, n, int(n), int(k0), w, piv, ps, st))
                launch_panel_lu(A, n, int(n), int(k0), w, piv, st);
        }
        const int64_t rest = n - k0 - w;
        ProfScope p(kid_misc, double(rest) * w * w, 16.0 * double(n) * w + 16.0 * double(rest) * w);
        launch_row_swaps(A, n, int(n), int(k0), w, piv, int(k0), int(k0 + w), st);
        if (rest > 0) {
            launch_trsm_unit_lower_rows(A, n, int(k0), w, int(k0 + w), int(rest), st);
            GemmBuild gb;
            gb.add1(A + (k0 + w) * n + (k0 + w), n, int(rest), int(rest), GEMM_ADD,
                    contrib(A + (k0 + w) * n + k0, n, 0, A + k0 * n + (k0 + w), n, 0, w, -1.0));
            gb.launch(kid_gemm);
        }
    }
    launch_diag_absmin(A, n, int(n), red + 1, st);
}

namespace {

// one cooperative launch over `idx` tasks; block-cyclic unless forced pairwise
void jacobi_wave(const std::vector<SvdTask>& tasks, const std::vector<size_t>& idx, bool pairwise, double thresh,
                 Region& scr, std::vector<int32_t*>* flags_out) {
    cudaStream_t st = ctx().stream;
    int max_n = 1, max_m = 1;
    for (size_t i : idx) {
        max_n = std::max(max_n, tasks[i].n);
        max_m = std::max(max_m, tasks[i].m);
    }
    const int jb = jacobi_block_rows(max_n);
    const int cap = pairwise ? jacobi_coop_capacity(max_n, max_m) : jacobi_block_capacity(max_n, max_m);
    constexpr int WARPS = 8;  // pairs per CTA and step (pairwise version)
    std::vector<int> want;
    int total = 0;
    for (size_t i : idx) {
        const int m = tasks[i].m;
        want.push_back(std::max<int>(1, int(pairwise ? cdiv((m + 1) / 2, WARPS) : cdiv(m, 2 * jb))));
        total += want.back();
    }
    while (pairwise && total > cap) {  // the pairwise version loops over pairs: shrink to fit
        auto it = std::max_element(want.begin(), want.end());
        if (*it <= 1) break;
        --*it;
        --total;
    }
    if (total > cap) throw Error(H2F_E_INTERNAL, "assertion: too many clusters for the co-resident Jacobi");
    uint32_t* bars = scr.alloc_n<uint32_t>(2 * idx.size());
    int32_t* flags = scr.alloc_n<int32_t>(64 * idx.size());
    H2F_CUDA(cudaMemsetAsync(bars, 0, sizeof(uint32_t) * 2 * idx.size(), st));
    H2F_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * 64 * idx.size(), st));
    std::vector<CoopSvdTask> ct;
    std::vector<int32_t> owner;
    int cta0 = 0;
    for (size_t w = 0; w < idx.size(); ++w) {
        const SvdTask& t = tasks[idx[w]];
        if (!t.R) continue;  // plan-only (sharded factorization): sized the wave only
        for (int c = 0; c < want[w]; ++c) owner.push_back(int32_t(ct.size()));
        ct.push_back(CoopSvdTask{t, cta0, want[w], bars + 2 * w, flags + 64 * w, scr.alloc_n<double>(std::max(t.m, 1))});
        cta0 += want[w];
        if (flags_out) (*flags_out)[idx[w]] = flags + 64 * w;
    }
    if (ct.empty()) return;
    cudaError_t e = pairwise ? launch_jacobi_coop(upload(ct), int32_t(owner.size()), upload(owner), max_n, max_m,
                                                  thresh, st)
                             : launch_jacobi_block(upload(ct), int32_t(owner.size()), upload(owner), max_n, max_m,
                                                   thresh, st);
    if (e != cudaSuccess) throw Error(H2F_E_CUDA, std::string("cooperative Jacobi launch: ") + cudaGetErrorString(e));
}

}  // namespace

void jacobi_multi_cta(const std::vector<SvdTask>& tasks, double thresh, Region& scr, bool pairwise,
                      std::vector<int32_t*>* flags_out) {
    static const bool env_pairwise = std::getenv("H2F_JACOBI_PAIRWISE") != nullptr;
    if (flags_out) flags_out->assign(tasks.size(), nullptr);
    if (pairwise || env_pairwise) {
        std::vector<size_t> all(tasks.size());
        for (size_t i = 0; i < tasks.size(); ++i) all[i] = i;
        jacobi_wave(tasks, all, true, thresh, scr, flags_out);
        return;
    }
    int max_n = 1, max_m = 1;
    for (auto& t : tasks) {
        max_n = std::max(max_n, t.n);
        max_m = std::max(max_m, t.m);
    }
    const int jb = jacobi_block_rows(max_n);
    const int cap = jacobi_block_capacity(max_n, max_m);
    // waves of co-resident clusters; a cluster wider than the device runs pairwise
    std::vector<size_t> wave;
    int used = 0;
    for (size_t i = 0; i < tasks.size(); ++i) {
        const int need = std::max<int>(1, int(cdiv(tasks[i].m, 2 * jb)));
        if (need > cap) {
            jacobi_wave(tasks, {i}, true, thresh, scr, flags_out);
            continue;
        }
        if (used + need > cap) {
            jacobi_wave(tasks, wave, false, thresh, scr, flags_out);
            wave.clear();
            used = 0;
        }
        wave.push_back(i);
        used += need;
    }
    if (!wave.empty()) jacobi_wave(tasks, wave, false, thresh, scr, flags_out);
}

}  // namespace h2f
