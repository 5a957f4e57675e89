// Device H2 construction and recompression: the input of
// the factorization built where it is consumed, from the point set, the
// cluster tree and the block partition (host integer work, problem.py).
//
//   construction (h2core.py:128-185): Chebyshev grids per cluster, tensor
//     Lagrange leaf bases and transfers, kernel-evaluated couplings and
//     dense near-field blocks (k_build.cu);
//   orthogonalize_recompress (h2core.py:226-269): QR sweep (leaf to top),
//     SVD truncation at eps * sigma_0 (top to leaf) with the parent's kept
//     singular values as column weights, QR sweep again.
//
// Every per-cluster step of a level runs as one batch: blocked Householder
// QR with explicit Q (dense.cpp hh_factor / hh_apply_q), the augmentation's
// TSQR + one-sided Jacobi for the SVDs, and the DMMA task GEMM for every
// basis / coupling transform.  The host syncs once per level of the
// recompression (the kept counts fix the next shapes).
//
// Deviation from the reference (tolerance contract): inside
// one level of the recompression the reference updates clusters one after
// another, so a cluster's SVD sees couplings already projected by the
// neighbours processed before it; here every cluster of the level takes its
// SVD of the level's unprojected couplings and the couplings are projected
// on both sides afterwards (C <- U_s^T C U_t).  The two differ by the
// truncated part, O(eps) relative.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>

#include "builders.h"
#include "dense.h"
#include "h2mat.h"

namespace h2f {

namespace {

struct Coupling {
    int s, t;
    double* p;  // rk[s] x rk[t], row-major, contiguous
};

struct Builder {
    const h2f_build_desc& d;
    Region& R;
    cudaStream_t st;
    int dim, depth, top, nlev;
    int64_t N;
    std::vector<std::vector<int>> levels;
    std::vector<int> rk;                    // current rank per node (-1: no basis)
    std::vector<double*> grid, LB, T;      // grid points, leaf basis (n_c x rk), transfer (rk x rk[par])
    std::vector<std::vector<Coupling>> cpl;  // per level
    std::vector<std::vector<std::pair<int, bool>>> touch;  // node -> (coupling index, c is t)
    std::vector<double*> w;                 // kept singular values (device), per node
    double* pts = nullptr;

    Builder(const h2f_build_desc& dd, Region& r) : d(dd), R(r), st(ctx().stream) {
        dim = d.dim;
        depth = d.depth;
        top = d.top_level;
        nlev = depth + 1;
        N = d.num_nodes;
        levels.assign(nlev, {});
        for (int64_t c = 0; c < N; ++c) {
            if (d.level[c] < 0 || d.level[c] >= nlev) throw Error(H2F_E_ARG, "node level out of range");
            levels[d.level[c]].push_back(int(c));
        }
        rk.assign(N, -1);
        grid.assign(N, nullptr);
        LB.assign(N, nullptr);
        T.assign(N, nullptr);
        w.assign(N, nullptr);
        touch.assign(N, {});
        cpl.assign(nlev, {});
    }

    std::vector<double*> dense_buf;         // per dense pair (absorb path); empty: evaluate at pack time

    bool leaf(int c) const { return d.child_left[c] < 0; }
    int rows(int c) const { return int(d.end[c] - d.begin[c]); }
    int par(int c) const { return int(d.parent[c]); }
    int pdeg(int lv) const { return d.p0 + (depth - lv) / 2; }
    int ipow(int p) const {
        int r = 1;
        for (int a = 0; a < dim; ++a) r *= p;
        return r;
    }

    void construct() {
        pts = R.alloc_n<double>(d.n * dim);
        H2F_CUDA(cudaMemcpyAsync(pts, d.points, sizeof(double) * d.n * dim, cudaMemcpyHostToDevice, st));
        if (top < 0) return;
        std::vector<GridTask> gt;
        for (int lv = depth; lv >= top; --lv)
            for (int c : levels[lv]) {
                GridTask g{};
                for (int a = 0; a < dim; ++a) {
                    g.lo[a] = d.box_lo[int64_t(c) * dim + a];
                    g.hi[a] = d.box_hi[int64_t(c) * dim + a];
                }
                g.p = pdeg(lv);
                rk[c] = ipow(g.p);
                grid[c] = g.out = R.alloc_n<double>(int64_t(rk[c]) * dim);
                gt.push_back(g);
            }
        launch_grid_tasks(upload(gt), int32_t(gt.size()), dim, st);
        std::vector<InterpTask> it;
        std::vector<int64_t> start{0};
        auto interp = [&](const double* p, int64_t np, int box, int pp, double* out) {
            InterpTask t{};
            t.pts = p;
            for (int a = 0; a < dim; ++a) {
                t.lo[a] = d.box_lo[int64_t(box) * dim + a];
                t.hi[a] = d.box_hi[int64_t(box) * dim + a];
            }
            t.out = out;
            t.ldo = ipow(pp);
            t.p = pp;
            it.push_back(t);
            start.push_back(start.back() + np);
        };
        for (int lv = depth; lv >= top; --lv)
            for (int c : levels[lv]) {
                if (leaf(c)) {
                    LB[c] = R.alloc_n<double>(int64_t(rows(c)) * rk[c]);
                    interp(pts + d.begin[c] * dim, rows(c), c, pdeg(lv), LB[c]);
                }
                if (lv > top) {
                    const int pu = pdeg(lv - 1);
                    T[c] = R.alloc_n<double>(int64_t(rk[c]) * ipow(pu));
                    interp(grid[c], rk[c], par(c), pu, T[c]);
                }
            }
        launch_interp_tasks(upload(it), upload(start), int32_t(it.size()), start.back(), dim, st);
        EvalBuild ev;
        for (int lv = 0; lv < nlev; ++lv)
            for (int64_t i = d.adm_ptr[lv]; i < d.adm_ptr[lv + 1]; ++i) {
                const int s = int(d.adm_pairs[2 * i]), t = int(d.adm_pairs[2 * i + 1]);
                if (rk[s] < 0 || rk[t] < 0) throw Error(H2F_E_ARG, "admissible pair above the top level");
                double* p = R.alloc_n<double>(int64_t(rk[s]) * rk[t]);
                ev.add(grid[s], grid[t], p, rk[t], -1, -1, rk[s], rk[t], 0);
                touch[s].push_back({int(cpl[lv].size()), false});
                if (t != s) touch[t].push_back({int(cpl[lv].size()), true});
                cpl[lv].push_back({s, t, p});
            }
        ev.launch(kparams());
    }

    KernelParams kparams() const {
        KernelParams k{};
        k.family = d.family;
        k.dim = dim;
        k.corr_length = d.corr_length;
        k.kappa = d.kappa;
        k.diag_base = d.family == KF_EXP_COV ? 1.0 : d.diag_value;
        k.alpha_r = d.alpha_r;
        return k;
    }

    struct EvalBuild {
        std::vector<EvalTask> tasks;
        std::vector<int64_t> start{0};
        void add(const double* X, const double* Y, double* out, int64_t ldo, int64_t row0, int64_t col0, int rows,
                 int cols, int diag) {
            if (rows <= 0 || cols <= 0) return;
            EvalTask t{};
            t.X = X;
            t.Y = Y;
            t.out = out;
            t.ldo = ldo;
            t.row0 = row0;
            t.col0 = col0;
            t.rows = rows;
            t.cols = cols;
            t.diag = diag;
            tasks.push_back(t);
            start.push_back(start.back() + cdiv(rows, 32) * cdiv(cols, 32));
        }
        void launch(const KernelParams& kp) {
            if (tasks.empty()) return;
            Context& X = ctx();
            auto* dt = X.up.put(tasks);
            auto* ds = X.up.put(start);
            X.up.flush(X.stream);
            launch_eval_tasks(dt, ds, int32_t(tasks.size()), start.back(), kp, X.stream);
        }
    };

    // h2core.py:201-215 (_qr_sweep): stacked basis = Q R, store Q, apply R
    // to the level's couplings and to the cluster's transfer
    void qr_sweep() {
        for (int lv = depth; lv >= top; --lv) {
            const auto& cl = levels[lv];
            std::vector<HhJob> jobs;
            std::vector<HhApply> xs;
            std::vector<RExtractTask> ex;
            std::vector<EyeTask> eye;
            CopyBuild cp, zero;
            std::vector<double*> Rc(N, nullptr);
            std::vector<int> newk(cl.size());
            int maxn = 1, maxe = 1;
            for (size_t i = 0; i < cl.size(); ++i) {
                const int c = cl[i], r = rk[c];
                int m;
                if (leaf(c)) {
                    m = rows(c);
                } else {
                    m = rk[d.child_left[c]] + rk[d.child_right[c]];
                }
                const int kq = std::min(m, r);
                newk[i] = kq;
                double* Q = R.alloc_n<double>(int64_t(m) * kq);
                Rc[c] = R.alloc_n<double>(int64_t(kq) * r);
                if (kq == 0) {
                    zero.zero(Rc[c], r, kq, r);
                } else {
                    double* Y = R.alloc_n<double>(int64_t(r) * m);  // S^T
                    if (leaf(c)) {
                        cp.add(Y, m, r, m, LB[c], r, 1, COPY_SET);
                    } else {
                        const int a = int(d.child_left[c]), b = int(d.child_right[c]);
                        cp.add(Y, m, r, rk[a], T[a], r, 1, COPY_SET);
                        cp.add(Y + rk[a], m, r, rk[b], T[b], r, 1, COPY_SET);
                    }
                    HhJob J;
                    J.M = Y;
                    J.ldm = m;
                    J.L = m;
                    J.ntot = r;
                    J.nfac = kq;
                    jobs.push_back(J);
                    xs.push_back(HhApply{Q, kq, kq});
                    ex.push_back(RExtractTask{Y, Rc[c], m, kq, r});
                    zero.zero(Q, kq, m, kq);
                    eye.push_back(EyeTask{Q, kq, 0, kq});
                    maxn = std::max(maxn, r);
                    maxe = std::max(maxe, kq);
                }
                if (leaf(c)) {
                    LB[c] = Q;
                } else {
                    const int a = int(d.child_left[c]), b = int(d.child_right[c]);
                    T[a] = Q;
                    T[b] = Q + int64_t(rk[a]) * kq;
                }
            }
            cp.launch();
            zero.launch();
            if (!eye.empty()) launch_set_eye(upload(eye), int32_t(eye.size()), maxe, st);
            if (!jobs.empty()) {
                hh_factor(jobs, R, true);
                launch_r_extract(upload(ex), int32_t(ex.size()), maxn, st);
                hh_apply_q(jobs, xs, R);
            }
            // couplings: C <- R_s C R_t^T ; transfer <- R T
            GemmBuild g1, g2, g3;
            for (auto& C : cpl[lv]) {
                const int ks = newk[pos(cl, C.s)], kt = newk[pos(cl, C.t)];
                double* tmp = R.alloc_n<double>(int64_t(rk[C.s]) * kt);
                g1.add1(tmp, kt, rk[C.s], kt, GEMM_STORE, contrib(C.p, rk[C.t], 0, Rc[C.t], rk[C.t], 1, rk[C.t]));
                double* np = R.alloc_n<double>(int64_t(ks) * kt);
                g2.add1(np, kt, ks, kt, GEMM_STORE, contrib(Rc[C.s], rk[C.s], 0, tmp, kt, 0, rk[C.s]));
                C.p = np;
            }
            if (lv > top)
                for (size_t i = 0; i < cl.size(); ++i) {
                    const int c = cl[i], kp = rk[par(c)];
                    double* nt = R.alloc_n<double>(int64_t(newk[i]) * kp);
                    g3.add1(nt, kp, newk[i], kp, GEMM_STORE, contrib(Rc[c], rk[c], 0, T[c], kp, 0, rk[c]));
                    T[c] = nt;
                }
            g1.launch(-1);
            g2.launch(-1);
            g3.launch(-1);
            for (size_t i = 0; i < cl.size(); ++i) rk[cl[i]] = newk[i];
        }
    }

    static size_t pos(const std::vector<int>& v, int c) {
        return size_t(std::lower_bound(v.begin(), v.end(), c) - v.begin());
    }

    // contiguous device copy, shaped as rows of 256 (+ one remainder row)
    static void copy_flat(CopyBuild& cb, double* dst, const double* src, int64_t cnt) {
        const int64_t full = cnt / 256, rem = cnt % 256;
        for (int64_t r0 = 0; r0 < full; r0 += int64_t(1) << 24) {
            const int64_t nr = std::min<int64_t>(full - r0, int64_t(1) << 24);
            cb.add(dst + r0 * 256, 256, int(nr), 256, src + r0 * 256, 256, 0, COPY_SET);
        }
        if (rem) cb.add(dst + full * 256, rem, 1, int(rem), src + full * 256, rem, 0, COPY_SET);
    }

    // state from an existing operator (copies: the input is not modified)
    void load(const H2Mat& A) {
        CopyBuild cb;
        for (int64_t c = 0; c < N; ++c) {
            rk[c] = int(A.rank[c]);
            if (A.leaf_basis_off[c] >= 0) {
                const int64_t cnt = int64_t(rows(int(c))) * rk[c];
                LB[c] = R.alloc_n<double>(cnt);
                copy_flat(cb, LB[c], A.vals + A.leaf_basis_off[c], cnt);
            }
        }
        for (int64_t c = 0; c < N; ++c)
            if (A.transfer_off[c] >= 0) {
                const int64_t cnt = int64_t(rk[c]) * A.rank[par(int(c))];
                T[c] = R.alloc_n<double>(cnt);
                copy_flat(cb, T[c], A.vals + A.transfer_off[c], cnt);
            }
        for (int lv = 0; lv < nlev; ++lv)
            for (int64_t i = d.adm_ptr[lv]; i < d.adm_ptr[lv + 1]; ++i) {
                const int s = int(d.adm_pairs[2 * i]), t = int(d.adm_pairs[2 * i + 1]);
                const int64_t cnt = int64_t(rk[s]) * rk[t];
                double* p = R.alloc_n<double>(cnt);
                copy_flat(cb, p, A.vals + A.coupling_list[size_t(i)], cnt);
                touch[s].push_back({int(cpl[lv].size()), false});
                if (t != s) touch[t].push_back({int(cpl[lv].size()), true});
                cpl[lv].push_back({s, t, p});
            }
        const int64_t nd = d.dense_ptr[nlev];
        dense_buf.assign(size_t(nd), nullptr);
        for (int64_t i = 0; i < nd; ++i) {
            const int s = int(d.dense_pairs[2 * i]), t = int(d.dense_pairs[2 * i + 1]);
            const int64_t cnt = int64_t(rows(s)) * rows(t);
            dense_buf[size_t(i)] = R.alloc_n<double>(cnt);
            copy_flat(cb, dense_buf[size_t(i)], A.vals + A.dense_list[size_t(i)], cnt);
        }
        cb.launch();
    }

    // h2core.py:342-392 (absorb_low_rank before its recompression): A + W W^T.
    // Dense blocks take W_s W_t^T; bottom-up, each cluster's basis is widened
    // by the significant range (sigma > 1e-12 |rows|_F) of its rows of W
    // outside the basis, so coef[c] = basis^T rows reproduces them exactly;
    // transfers gain zero rows; couplings take coef[s] coef[t]^T.
    void widen(const double* Wd, int rw) {
        GemmBuild gd;
        const int64_t nd = d.dense_ptr[nlev];
        for (int64_t i = 0; i < nd; ++i) {
            const int s = int(d.dense_pairs[2 * i]), t = int(d.dense_pairs[2 * i + 1]);
            gd.add1(dense_buf[size_t(i)], rows(t), rows(s), rows(t), GEMM_ADD,
                    contrib(Wd + d.begin[s] * rw, rw, 0, Wd + d.begin[t] * rw, rw, 1, rw));
        }
        gd.launch(-1);
        if (top < 0) return;
        const std::vector<int> rk0 = rk;
        std::vector<double*> coef(N, nullptr);
        for (int lv = depth; lv >= top; --lv) {
            const auto& cl = levels[lv];
            const size_t nc = cl.size();
            std::vector<const double*> rowsp(nc);
            std::vector<int> m(nc), rc(nc);
            std::vector<double*> inside(nc), fro(nc);
            CopyBuild c1;
            GemmBuild g1;
            for (size_t i = 0; i < nc; ++i) {
                const int c = cl[i];
                rc[i] = rk[c];
                if (leaf(c)) {
                    m[i] = rows(c);
                    rowsp[i] = Wd + d.begin[c] * rw;
                } else {
                    const int a = int(d.child_left[c]), b = int(d.child_right[c]);
                    m[i] = rk[a] + rk[b];
                    double* st_ = R.alloc_n<double>(int64_t(m[i]) * rw);
                    copy_flat(c1, st_, coef[a], int64_t(rk[a]) * rw);
                    copy_flat(c1, st_ + int64_t(rk[a]) * rw, coef[b], int64_t(rk[b]) * rw);
                    rowsp[i] = st_;
                }
                // inside = S^T rows (rk x rw)
                inside[i] = R.alloc_n<double>(int64_t(rc[i]) * rw);
                if (rc[i] > 0) {
                    if (leaf(c)) {
                        g1.add1(inside[i], rw, rc[i], rw, GEMM_STORE, contrib(LB[c], rc[i], 1, rowsp[i], rw, 0, m[i]));
                    } else {
                        const int a = int(d.child_left[c]), b = int(d.child_right[c]);
                        const GemmContrib cs[2] = {contrib(T[a], rc[i], 1, rowsp[i], rw, 0, rk[a]),
                                                   contrib(T[b], rc[i], 1, rowsp[i] + int64_t(rk[a]) * rw, rw, 0, rk[b])};
                        g1.add(inside[i], rw, rc[i], rw, GEMM_STORE, cs, 2);
                    }
                }
            }
            c1.launch();
            g1.launch(-1);
            // resid^T = rows^T - inside^T S^T (rw x m): the SVD input M (r = m rows of
            // left vectors... as M = resid (m x rw))
            CopyBuild c2;
            GemmBuild g2;
            std::vector<Svd> sv(nc);
            std::vector<RowNormOut> rn;
            std::vector<int64_t> rstart{0};
            for (size_t i = 0; i < nc; ++i) {
                const int c = cl[i];
                double* M = R.alloc_n<double>(int64_t(m[i]) * rw);
                copy_flat(c2, M, rowsp[i], int64_t(m[i]) * rw);
                if (rc[i] > 0) {
                    if (leaf(c)) {
                        g2.add1(M, rw, m[i], rw, GEMM_ADD, contrib(LB[c], rc[i], 0, inside[i], rw, 0, rc[i], -1.0));
                    } else {
                        const int a = int(d.child_left[c]), b = int(d.child_right[c]);
                        g2.add1(M, rw, rk[a], rw, GEMM_ADD, contrib(T[a], rc[i], 0, inside[i], rw, 0, rc[i], -1.0));
                        g2.add1(M + int64_t(rk[a]) * rw, rw, rk[b], rw, GEMM_ADD,
                                contrib(T[b], rc[i], 0, inside[i], rw, 0, rc[i], -1.0));
                    }
                }
                fro[i] = R.alloc_n<double>(1);
                rn.push_back(RowNormOut{rowsp[i], fro[i], 0, m[i] * rw, 0});
                rstart.push_back(rstart.back() + 1);
                sv[i].M = M;
                sv[i].r = m[i];
                sv[i].W = rw;
            }
            c2.launch();
            launch_row_norms(upload(rn), upload(rstart), int32_t(rn.size()), rstart.back(), st);
            g2.launch(-1);
            std::vector<double> fro_h(nc);
            {
                double* fd = R.alloc_n<double>(int64_t(nc));
                CopyBuild c3;
                for (size_t i = 0; i < nc; ++i) c3.add(fd + i, 1, 1, 1, fro[i], 1, 0, COPY_SET);
                c3.launch();
                H2F_CUDA(cudaMemcpyAsync(fro_h.data(), fd, sizeof(double) * nc, cudaMemcpyDeviceToHost, st));
            }
            svd_left(sv);  // syncs (fro_h is ready after it)
            std::vector<int> e(nc, 0);
            for (size_t i = 0; i < nc; ++i) {
                const double cut = 1e-12 * std::max(fro_h[i], 1e-300);
                for (double x : sv[i].sh) e[i] += x > cut;
            }
            // widened bases [S | extra], coef = [inside; extra^T rows]
            CopyBuild c4;
            GemmBuild g4;
            for (size_t i = 0; i < nc; ++i) {
                const int c = cl[i], k2 = rc[i] + e[i];
                const double* U = sv[i].U;  // rows 0..e-1: extra^T (e x m)
                auto widen_rows = [&](double*& B, int nrow, int row0) {
                    double* nb = R.alloc_n<double>(int64_t(nrow) * k2);
                    if (rc[i] > 0) c4.add(nb, k2, nrow, rc[i], B, rc[i], 0, COPY_SET);
                    if (e[i] > 0) c4.add(nb + rc[i], k2, nrow, e[i], U + row0, m[i], 1, COPY_SET);
                    B = nb;
                };
                if (leaf(c)) {
                    widen_rows(LB[c], m[i], 0);
                } else {
                    const int a = int(d.child_left[c]), b = int(d.child_right[c]);
                    widen_rows(T[a], rk[a], 0);
                    widen_rows(T[b], rk[b], rk[a]);
                }
                coef[c] = R.alloc_n<double>(int64_t(k2) * rw);
                if (rc[i] > 0) copy_flat(c4, coef[c], inside[i], int64_t(rc[i]) * rw);
                if (e[i] > 0)
                    g4.add1(coef[c] + int64_t(rc[i]) * rw, rw, e[i], rw, GEMM_STORE,
                            contrib(U, m[i], 0, rowsp[i], rw, 0, m[i]));
            }
            c4.launch();
            g4.launch(-1);
            // the cluster's own transfer gains e zero rows
            CopyBuild c5;
            for (size_t i = 0; i < nc; ++i) {
                const int c = cl[i];
                rk[c] = rc[i] + e[i];
                if (e[i] > 0 && T[c]) {
                    const int kp = rk[par(c)];
                    double* nt = R.alloc_n<double>(int64_t(rk[c]) * kp);
                    if (rc[i] > 0) copy_flat(c5, nt, T[c], int64_t(rc[i]) * kp);
                    c5.zero(nt + int64_t(rc[i]) * kp, kp, e[i], kp);
                    T[c] = nt;
                }
            }
            c5.launch();
        }
        // couplings: the old block in the leading corner (widening appends
        // coordinates), plus coef_s coef_t^T
        CopyBuild z6, c6;
        GemmBuild g6;
        for (int lv = 0; lv < nlev; ++lv)
            for (auto& C : cpl[lv]) {
                const int ks = rk[C.s], kt = rk[C.t], os = rk0[C.s], ot = rk0[C.t];
                double* np = R.alloc_n<double>(int64_t(ks) * kt);
                z6.zero(np, kt, ks, kt);
                c6.add(np, kt, os, ot, C.p, ot, 0, COPY_SET);
                g6.add1(np, kt, ks, kt, GEMM_ADD, contrib(coef[C.s], rw, 0, coef[C.t], rw, 1, rw));
                C.p = np;
            }
        z6.launch();
        c6.launch();
        g6.launch(-1);
    }

    // h2core.py:236-268: per cluster, SVD of [couplings | transfer * w_parent],
    // keep sigma > eps sigma_0, project basis, transfer and couplings
    // left singular vectors and singular values of a batch of r x W
    // matrices M (row-major, overwritten): R of the QR of M^T (shared-memory
    // TSQR for r <= 32, blocked Householder above, as factor.cpp's
    // augmentation), one-sided Jacobi of R keeping every vector (rows of U,
    // m = min(r, W), sorted by sigma), sigma_j = |R u_j| (GEMM + row norms).
    // Returns the host sigmas per item (one stream sync).
    struct Svd {
        double* M = nullptr;
        int r = 0, W = 0, m = 0;
        double *U = nullptr, *Rm = nullptr, *sig = nullptr;
        std::vector<double> sh;
    };
    void svd_left(std::vector<Svd>& v) {
        Context& X = ctx();
        std::vector<QrTask> qr_small, qr_big, qr_seg;
        std::vector<SvdTask> svd_small, svd_big;
        int max_small = 1;
        int* kept_d = R.alloc_n<int>(1);
        for (auto& it : v) {
            const int r = it.r, W = it.W;
            it.m = (r > 0 && W > 0) ? std::min(r, W) : 0;
            if (!it.m) continue;
            const int m = it.m;
            // both QR paths write a full r x r R (rows >= m zero), also when W < r
            it.Rm = R.alloc_n<double>(int64_t(r) * r);
            it.U = R.alloc_n<double>(int64_t(m) * r);
            it.sig = R.alloc_n<double>(m);
            if (r > 32) {
                qr_big.push_back(QrTask{it.M, it.Rm, W, r, W, 0, W, 0});
            } else {
                const int seg = std::max(256, 4 * r);
                const int nseg = int(cdiv(W, seg));
                if (nseg > 1) {
                    double* ST = R.alloc_n<double>(int64_t(r) * nseg * r);
                    for (int sg = 0; sg < nseg; ++sg)
                        qr_seg.push_back(QrTask{it.M, ST + int64_t(sg) * r, W, r, W, sg * seg,
                                                std::min(W, (sg + 1) * seg), int64_t(nseg) * r});
                    qr_small.push_back(QrTask{ST, it.Rm, int64_t(nseg) * r, r, nseg * r, 0, nseg * r, 0});
                } else {
                    qr_small.push_back(QrTask{it.M, it.Rm, W, r, W, 0, W, 0});
                }
            }
            SvdTask sv{it.Rm, it.U, m, r, kept_d, 0};
            if (r <= 64) {
                svd_small.push_back(sv);
                max_small = std::max(max_small, r);
            } else {
                svd_big.push_back(sv);
            }
        }
        if (!qr_seg.empty()) launch_qr_r_smem(upload(qr_seg), int32_t(qr_seg.size()), max_small, st);
        if (!qr_small.empty()) launch_qr_r_smem(upload(qr_small), int32_t(qr_small.size()), max_small, st);
        if (!qr_big.empty()) qr_r_blocked(qr_big, R);
        if (!svd_small.empty())
            launch_jacobi_smem(upload(svd_small), int32_t(svd_small.size()), max_small, 0.0, st);
        if (!svd_big.empty()) jacobi_multi_cta(svd_big, 0.0, R);
        GemmBuild gp;
        std::vector<RowNormOut> rn;
        std::vector<int64_t> rstart{0};
        int64_t total = 0;
        for (auto& it : v) {
            if (!it.m) continue;
            double* P = R.alloc_n<double>(int64_t(it.m) * it.m);
            gp.add1(P, it.m, it.m, it.m, GEMM_STORE, contrib(it.U, it.r, 0, it.Rm, it.r, 1, it.r));
            rn.push_back(RowNormOut{P, it.sig, it.m, it.m, 0});
            rstart.push_back(rstart.back() + it.m);
            total += it.m;
        }
        gp.launch(-1);
        if (!rn.empty()) launch_row_norms(upload(rn), upload(rstart), int32_t(rn.size()), rstart.back(), st);
        std::vector<double> sh(size_t(std::max<int64_t>(total, 1)));
        double* sdev = R.alloc_n<double>(std::max<int64_t>(total, 1));
        CopyBuild sc;
        int64_t off = 0;
        for (auto& it : v) {
            if (!it.m) continue;
            sc.add(sdev + off, it.m, 1, it.m, it.sig, it.m, 0, COPY_SET);
            off += it.m;
        }
        sc.launch();
        if (total) H2F_CUDA(cudaMemcpyAsync(sh.data(), sdev, sizeof(double) * total, cudaMemcpyDeviceToHost, st));
        X.sync();
        off = 0;
        for (auto& it : v) {
            it.sh.assign(sh.begin() + off, sh.begin() + off + it.m);
            off += it.m;
        }
    }

    void recompress(double eps) {
        for (int lv = top; lv <= depth; ++lv) {
            const auto& cl = levels[lv];
            const size_t nc = cl.size();
            // diag(w_parent) once per parent
            std::vector<double*> D(N, nullptr);
            std::vector<DiagTask> dt;
            if (lv > top)
                for (int p : levels[lv - 1])
                    if (rk[p] > 0 && w[p]) {
                        D[p] = R.alloc_n<double>(int64_t(rk[p]) * rk[p]);
                        dt.push_back(DiagTask{w[p], D[p], rk[p], 0});
                    }
            if (!dt.empty()) launch_set_diag(upload(dt), int32_t(dt.size()), st);
            CopyBuild gather;
            GemmBuild gw;
            std::vector<Svd> sv(nc);
            for (size_t i = 0; i < nc; ++i) {
                const int c = cl[i], r = rk[c];
                int W = 0;
                for (auto& tc : touch[c]) {
                    const Coupling& C = cpl[lv][tc.first];
                    W += tc.second ? rk[C.s] : rk[C.t];
                }
                const bool wt = lv > top && D[par(c)] != nullptr;
                if (wt) W += rk[par(c)];
                if (r <= 0 || W == 0) continue;
                double* M = R.alloc_n<double>(int64_t(r) * W);
                int off = 0;
                for (auto& tc : touch[c]) {
                    const Coupling& C = cpl[lv][tc.first];
                    if (tc.second) {  // c is the column cluster: C^T (r x rk[s])
                        gather.add(M + off, W, r, rk[C.s], C.p, r, 1, COPY_SET);
                        off += rk[C.s];
                    } else {
                        gather.add(M + off, W, r, rk[C.t], C.p, rk[C.t], 0, COPY_SET);
                        off += rk[C.t];
                    }
                }
                if (wt) {
                    const int kp = rk[par(c)];
                    gw.add1(M + off, W, r, kp, GEMM_STORE, contrib(T[c], kp, 0, D[par(c)], kp, 0, kp));
                }
                sv[i].M = M;
                sv[i].r = r;
                sv[i].W = W;
            }
            gather.launch();
            gw.launch(-1);
            svd_left(sv);
            std::vector<int> k(nc, 0);
            std::vector<double*> U(nc, nullptr), sig(nc, nullptr);
            for (size_t i = 0; i < nc; ++i) {
                U[i] = sv[i].U;
                sig[i] = sv[i].sig;
                if (!sv[i].m) continue;
                double smax = 0.0;
                for (double x : sv[i].sh) smax = std::max(smax, x);
                const double cut = eps * smax;
                int kk = 0;
                for (double x : sv[i].sh) kk += x > cut;
                k[i] = kk;
            }
            // projections: basis <- S U_k, transfer <- U_k^T T, C <- U_s^T C U_t
            GemmBuild gb, gt, gc1, gc2;
            auto proj_cols = [&](double*& B, int rows_, int r, double* Ui, int kk) {
                double* nb = R.alloc_n<double>(int64_t(rows_) * kk);
                if (kk > 0 && rows_ > 0) gb.add1(nb, kk, rows_, kk, GEMM_STORE, contrib(B, r, 0, Ui, r, 1, r));
                B = nb;
            };
            for (size_t i = 0; i < nc; ++i) {
                const int c = cl[i], r = rk[c], kk = k[i];
                if (leaf(c)) {
                    proj_cols(LB[c], rows(c), r, U[i], kk);
                } else {
                    const int a = int(d.child_left[c]), b = int(d.child_right[c]);
                    proj_cols(T[a], rk[a], r, U[i], kk);
                    proj_cols(T[b], rk[b], r, U[i], kk);
                }
                if (lv > top) {
                    const int kp = rk[par(c)];
                    double* nt = R.alloc_n<double>(int64_t(kk) * kp);
                    if (kk > 0 && kp > 0) gt.add1(nt, kp, kk, kp, GEMM_STORE, contrib(U[i], r, 0, T[c], kp, 0, r));
                    T[c] = nt;
                }
            }
            for (auto& C : cpl[lv]) {
                const size_t is = pos(cl, C.s), it = pos(cl, C.t);
                const int ks = k[is], kt = k[it], rs = rk[C.s], rt = rk[C.t];
                double* tmp = R.alloc_n<double>(int64_t(rs) * kt);
                double* np = R.alloc_n<double>(int64_t(ks) * kt);
                if (ks > 0 && kt > 0) {
                    gc1.add1(tmp, kt, rs, kt, GEMM_STORE, contrib(C.p, rt, 0, U[it], rt, 1, rt));
                    gc2.add1(np, kt, ks, kt, GEMM_STORE, contrib(U[is], rs, 0, tmp, kt, 0, rs));
                }
                C.p = np;
            }
            gb.launch(-1);
            gt.launch(-1);
            gc1.launch(-1);
            gc2.launch(-1);
            for (size_t i = 0; i < nc; ++i) {
                rk[cl[i]] = k[i];
                w[cl[i]] = k[i] > 0 ? sig[i] : nullptr;
            }
        }
    }
};


// final layout (leaf bases, transfers, couplings, dense blocks) in one new
// arena allocation; dense blocks are copied from the builder's buffers or,
// for a fresh construction, evaluated straight into it
H2Mat* pack_matrix(Builder& B, std::vector<int64_t>& rank) {
    const h2f_build_desc& d = B.d;
    const int64_t N = d.num_nodes;
    const int nlev = d.depth + 1;
    std::vector<int64_t> leaf_off(N, -1), trans_off(N, -1), coup_off, dense_off;
    rank.assign(N, -1);
    int64_t pos = 0;
    std::vector<std::pair<int64_t, std::pair<const double*, int64_t>>> pieces;  // (offset, (src, count))
    for (int64_t c = 0; c < N; ++c) {
        rank[c] = B.rk[c] < 0 ? -1 : B.rk[c];
        if (B.LB[c]) {
            leaf_off[c] = pos;
            pieces.push_back({pos, {B.LB[c], int64_t(B.rows(int(c))) * B.rk[c]}});
            pos += int64_t(B.rows(int(c))) * B.rk[c];
        }
    }
    for (int64_t c = 0; c < N; ++c)
        if (B.T[c]) {
            trans_off[c] = pos;
            const int64_t cnt = int64_t(B.rk[c]) * B.rk[B.par(int(c))];
            pieces.push_back({pos, {B.T[c], cnt}});
            pos += cnt;
        }
    for (int lv = 0; lv < nlev; ++lv)
        for (auto& C : B.cpl[lv]) {
            coup_off.push_back(pos);
            const int64_t cnt = int64_t(B.rk[C.s]) * B.rk[C.t];
            pieces.push_back({pos, {C.p, cnt}});
            pos += cnt;
        }
    const int64_t ndense = d.dense_ptr[nlev];
    for (int64_t i = 0; i < ndense; ++i) {
        dense_off.push_back(pos);
        const int s = int(d.dense_pairs[2 * i]), t = int(d.dense_pairs[2 * i + 1]);
        const int64_t cnt = int64_t(B.rows(s)) * B.rows(t);
        if (!B.dense_buf.empty()) pieces.push_back({pos, {B.dense_buf[size_t(i)], cnt}});
        pos += cnt;
    }
    double* vals = static_cast<double*>(dalloc(sizeof(double) * std::max<int64_t>(pos, 1)));
    CopyBuild pack;
    for (auto& pc : pieces) Builder::copy_flat(pack, vals + pc.first, pc.second.first, pc.second.second);
    pack.launch();
    if (B.dense_buf.empty()) {
        Builder::EvalBuild ev;
        for (int64_t i = 0; i < ndense; ++i) {
            const int s = int(d.dense_pairs[2 * i]), t = int(d.dense_pairs[2 * i + 1]);
            ev.add(B.pts + d.begin[s] * d.dim, B.pts + d.begin[t] * d.dim, vals + dense_off[i], B.rows(t),
                   d.begin[s], d.begin[t], B.rows(s), B.rows(t), 1);
        }
        ev.launch(B.kparams());
    }
    ctx().sync();
    h2f_matrix_desc md{};
    md.n = d.n;
    md.depth = d.depth;
    md.top_level = d.top_level;
    md.num_nodes = N;
    md.parent = d.parent;
    md.child_left = d.child_left;
    md.child_right = d.child_right;
    md.level = d.level;
    md.begin = d.begin;
    md.end = d.end;
    md.rank = rank.data();
    md.adm_pairs = d.adm_pairs;
    md.adm_ptr = d.adm_ptr;
    md.inner_pairs = d.inner_pairs;
    md.inner_ptr = d.inner_ptr;
    md.dense_pairs = d.dense_pairs;
    md.dense_ptr = d.dense_ptr;
    md.leaf_basis_off = leaf_off.data();
    md.transfer_off = trans_off.data();
    md.coupling_off = coup_off.data();
    md.dense_off = dense_off.data();
    md.nvals = pos;
    return h2mat_create_device(&md, vals);
}

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double>(b - a).count(); }

}  // namespace

H2Mat* h2mat_build(const h2f_build_desc* dp, int64_t* rank_out, double* seconds) {
    if (!dp || dp->n <= 0 || dp->num_nodes <= 0) throw Error(H2F_E_ARG, "empty H2 build description");
    const h2f_build_desc& d = *dp;
    if (d.dim < 1 || d.dim > 3) throw Error(H2F_E_ARG, "dim must be 1, 2 or 3");
    if (d.family < 0 || d.family > 2) throw Error(H2F_E_ARG, "unknown kernel family");
    if (d.top_level >= 0 && (d.p0 < 1 || d.p0 + d.depth / 2 > 32)) throw Error(H2F_E_ARG, "p0 out of range");
    const auto t0 = Clock::now();
    Region R(size_t(256) << 20);
    Builder B(d, R);
    B.construct();
    ctx().sync();
    const auto t1 = Clock::now();
    if (d.top_level >= 0 && d.eps > 0) {
        B.qr_sweep();
        B.recompress(d.eps);
        B.qr_sweep();
    }
    ctx().sync();
    const auto t2 = Clock::now();
    std::vector<int64_t> rank;
    H2Mat* m = pack_matrix(B, rank);
    const auto t3 = Clock::now();
    if (rank_out) std::memcpy(rank_out, rank.data(), sizeof(int64_t) * d.num_nodes);
    if (seconds) {
        // construction includes the dense near-field evaluation (done last,
        // straight into the operator's storage)
        seconds[0] = secs(t0, t1) + secs(t2, t3);
        seconds[1] = secs(t1, t2);
    }
    return m;
}

H2Mat* h2mat_absorb_low_rank(const H2Mat& A, const double* w_host, int rw, double eps, int64_t* rank_out,
                             double* seconds) {
    if (rw < 0) throw Error(H2F_E_ARG, "update rank must be >= 0");
    const auto t0 = Clock::now();
    // a build description over A's structure (no points: nothing is evaluated)
    const int nlev = A.depth + 1;
    std::vector<int64_t> adm, adm_ptr{0}, inner, inner_ptr{0}, dense, dense_ptr{0};
    for (int l = 0; l < nlev; ++l) {
        for (auto& p : A.adm[l]) adm.insert(adm.end(), {p.first, p.second});
        for (auto& p : A.inner[l]) inner.insert(inner.end(), {p.first, p.second});
        for (auto& p : A.dense[l]) dense.insert(dense.end(), {p.first, p.second});
        adm_ptr.push_back(int64_t(adm.size() / 2));
        inner_ptr.push_back(int64_t(inner.size() / 2));
        dense_ptr.push_back(int64_t(dense.size() / 2));
    }
    h2f_build_desc d{};
    d.n = A.n;
    d.dim = 1;
    d.depth = A.depth;
    d.top_level = A.top;
    d.num_nodes = A.nnodes;
    d.parent = A.parent.data();
    d.child_left = A.left.data();
    d.child_right = A.right.data();
    d.level = A.level.data();
    d.begin = A.begin.data();
    d.end = A.end.data();
    d.adm_pairs = adm.data();
    d.adm_ptr = adm_ptr.data();
    d.inner_pairs = inner.data();
    d.inner_ptr = inner_ptr.data();
    d.dense_pairs = dense.data();
    d.dense_ptr = dense_ptr.data();
    Region R(size_t(256) << 20);
    Builder B(d, R);
    B.load(A);
    double* Wd = R.alloc_n<double>(A.n * std::max(rw, 1));
    if (rw > 0) {
        H2F_CUDA(cudaMemcpyAsync(Wd, w_host, sizeof(double) * A.n * rw, cudaMemcpyHostToDevice, ctx().stream));
        B.widen(Wd, rw);
    }
    ctx().sync();
    const auto t1 = Clock::now();
    if (d.top_level >= 0 && eps > 0) {
        B.qr_sweep();
        B.recompress(eps);
        B.qr_sweep();
    }
    std::vector<int64_t> rank;
    H2Mat* m = pack_matrix(B, rank);
    const auto t2 = Clock::now();
    if (rank_out) std::memcpy(rank_out, rank.data(), sizeof(int64_t) * A.nnodes);
    if (seconds) {
        seconds[0] = secs(t0, t1);
        seconds[1] = secs(t1, t2);
    }
    return m;
}

}  // namespace h2f
