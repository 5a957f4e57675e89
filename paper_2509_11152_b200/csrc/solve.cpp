// Substitution against the factor (Alg. 3; solve.py:29-77).
//
// A SolvePlan is built once per (factor, nrhs): per batch, the cluster and
// edge descriptors, and the forward-scatter groups (products grouped by target
// span in reference order).  A solve is then a fixed launch sequence:
// forward over records (fwd_clusters + fwd_scatter per batch, then the
// up_index gather), the dense top solve, and the backward sweep in reverse
// (up_index scatter, bwd_clusters per batch).
#include <algorithm>
#include <map>

#include "builders.h"
#include "factor.h"

namespace h2f {

// multi-RHS substitution on the DMMA tile GEMM from this many columns on
// (below: the per-vector solve_tasks kernels)
constexpr int SOLVE_GEMM_MIN_RHS = 4;

namespace {

template <class T> T* to_dev(Region& r, const std::vector<T>& v) {
    T* d = r.alloc_n<T>(std::max<size_t>(v.size(), 1));
    if (!v.empty())
        H2F_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, ctx().stream));
    return d;
}

// a GEMM / copy / TRSM task list uploaded once with the plan
struct DevGemm {
    GemmTask* t = nullptr;
    GemmContrib* c = nullptr;
    int64_t *ts = nullptr, *cta = nullptr;
    int32_t nt = 0;
    int64_t ntiles = 0;
    double flops = 0, bytes = 0;
    void build(Region& mem, const GemmBuild& g) {
        if (g.tasks.empty()) return;
        t = to_dev(mem, g.tasks);
        c = to_dev(mem, g.contribs);
        ts = to_dev(mem, g.tile_start);
        ntiles = g.tile_start.back();
        if (ntiles > gemm_grid(ntiles)) cta = to_dev(mem, g.cta_ranges());
        nt = int32_t(g.tasks.size());
        flops = g.flops;
        bytes = g.bytes;
    }
    void launch(int kid, cudaStream_t st) const {
        if (!nt) return;
        ProfScope ps(kid, flops, bytes, double(ntiles));
        launch_gemm_tasks(t, c, ts, nt, ntiles, cta, nullptr, st);
    }
};

struct DevCopy {
    CopyTask* t = nullptr;
    int64_t* ts = nullptr;
    int32_t nt = 0;
    int64_t ntiles = 0;
    double bytes = 0;
    void build(Region& mem, const CopyBuild& c) {
        if (c.tasks.empty()) return;
        t = to_dev(mem, c.tasks);
        ts = to_dev(mem, c.tile_start);
        nt = int32_t(c.tasks.size());
        ntiles = c.tile_start.back();
        bytes = c.bytes;
    }
    void launch(int kid, cudaStream_t st) const {
        if (!nt) return;
        ProfScope ps(kid, 0.0, bytes);
        launch_copy_tasks(t, ts, nt, ntiles, st);
    }
};

struct DevTrsm {
    TrsmTask* t[2] = {};  // 32- and 16-column variants
    int32_t n[2] = {}, max_r[2] = {1, 1};
    double flops = 0;
    void build(Region& mem, const std::vector<TrsmTask> (&v)[2], const int (&mr)[2], double f) {
        for (int i = 0; i < 2; ++i) {
            n[i] = int32_t(v[i].size());
            if (n[i]) t[i] = to_dev(mem, v[i]);
            max_r[i] = mr[i];
        }
        flops = f;
    }
    void launch(int kid, cudaStream_t st) const {
        if (!n[0] && !n[1]) return;
        ProfScope ps(kid, flops, 0.0);
        if (n[0]) launch_trsm_dmma(t[0], n[0], max_r[0], 32, st);
        if (n[1]) launch_trsm_dmma(t[1], n[1], max_r[1], 16, st);
    }
};

}  // namespace

struct SolvePlan {
    struct Batch {
        SolveCluster* cl = nullptr;
        int32_t ncl = 0;
        SolveEdge* edges = nullptr;
        ScatterGroup* groups = nullptr;
        int32_t ngroups = 0;
        int64_t* list = nullptr;
        // task lists: forward rotation, forward products + L solves,
        // backward U solves + gathers, backward rotation
        SolveTask* tk[4] = {};
        int32_t ntk[4] = {};
        double fwd_flops = 0, fwd_bytes = 0, sc_bytes = 0;
        // multi-RHS path (nrhs >= SOLVE_GEMM_MIN_RHS): forward = rotation
        // GEMM, products GEMM, pivoted unit-lower TRSM, skeleton copy,
        // scatter; backward = upper TRSM, gather GEMM, add, rotation GEMM, copy
        bool gemm = false;
        DevGemm f_rot, f_prod, b_gather, b_rot;
        DevCopy f_copy, b_copy;
        std::vector<DevCopy> b_add;  // one launch per split-K partial of the gather
        DevTrsm f_trsm, b_trsm;
        int32_t scatter_split = 1;  // CTAs per scatter group (multi-RHS)
    };
    struct Level {
        int64_t total = 0;
        int64_t* up = nullptr;
        int64_t up_n = 0;
        std::vector<Batch> batches;
    };
    int nrhs = 1;
    std::vector<Level> levels;
    std::vector<double*> yv;   // per record level vectors
    double* ytop = nullptr;
    double* ttop = nullptr;   // top solve temporary
    int32_t* top_perm = nullptr;
    int32_t* top_sync = nullptr;
    double* scratch = nullptr;
    double* work = nullptr;
    int64_t last_use = 0;
    cudaGraphExec_t graph = nullptr;  // captured single-vector sweeps (solve_device)
    int64_t graph_launches = 0;
    int uses = 0;
    ~SolvePlan() {
        if (graph) cudaGraphExecDestroy(graph);
    }
    Region mem{size_t(16) << 20};
};

Factorization::~Factorization() = default;

namespace {

// plans are cached per nrhs; at most kMaxPlans stay alive (least recently
// used evicted -- each holds O(n nrhs) of vectors in its own region), so
// solves with many different column counts do not grow the arena
constexpr size_t kMaxPlans = 3;

SolvePlan& get_plan(Factorization& f, int nrhs) {
    static int64_t clock = 0;
    auto it = f.plans.find(nrhs);
    if (it != f.plans.end()) {
        it->second->last_use = ++clock;
        return *it->second;
    }
    while (f.plans.size() >= kMaxPlans) {
        auto victim = f.plans.begin();
        for (auto jt = f.plans.begin(); jt != f.plans.end(); ++jt)
            if (jt->second->last_use < victim->second->last_use) victim = jt;
        ctx().sync();  // no launch of the victim's task lists is in flight
        f.plans.erase(victim);
    }
    auto plan = std::make_shared<SolvePlan>();
    plan->last_use = ++clock;
    SolvePlan& P = *plan;
    P.nrhs = nrhs;
    int64_t scratch_rows = 0, work_max = 0;
    bool use_gemm = nrhs >= SOLVE_GEMM_MIN_RHS;
    for (auto& rec : f.recs)
        for (auto& cf : rec.factors)
            if (cf.r > 0 && trsm_dmma_cols(cf.r) == 0) use_gemm = false;
    const int q = nrhs;
    struct HostBatch {
        size_t level, batch;
        std::vector<SolveCluster> cls;
        std::vector<SolveEdge> edges;
    };
    std::vector<HostBatch> host_batches;
    for (auto& rec : f.recs) {
        SolvePlan::Level L;
        L.total = rec.total();
        L.up_n = int64_t(rec.up_index.size());
        L.up = to_dev(P.mem, rec.up_index);
        for (auto& batch : rec.batches) {
            std::vector<SolveCluster> cls;
            std::vector<SolveEdge> edges;
            // target lo -> (w, ordered scratch rows)
            std::map<int64_t, std::pair<int, std::vector<int64_t>>> groups;
            std::vector<int64_t> group_order;
            int64_t soff = 0, woff = 0;
            double flops_b = 0, bytes_b = 0;
            std::vector<SolveTask> tk[4];
            for (int c : batch) {
                const ClusterFactor& cf = rec.factors[rec.pos.at(c)];
                SolveCluster sc{};
                sc.q = cf.q;
                sc.lu = cf.lu;
                sc.piv = cf.piv;
                sc.off = cf.offset;
                sc.s = cf.s;
                sc.r = cf.r;
                sc.mw = cf.edges.empty() ? nullptr : cf.edges[0].mat;
                sc.W = 0;
                for (auto& e : cf.edges) sc.W += e.w;
                sc.soff = soff;
                sc.edge_begin = int64_t(edges.size());
                sc.woff = woff;
                if (cf.s + 256 > SOLVE_SMEM_VEC)
                    throw Error(H2F_E_INTERNAL, "assertion: cluster too large for the solve kernels");
                int64_t col = 0;
                for (auto& e : cf.edges) {
                    SolveEdge se{};
                    se.mat = e.mat;
                    se.ld = e.ld;
                    se.w = e.w;
                    if (e.mat != sc.mw + col || e.ld != sc.W)
                        throw Error(H2F_E_INTERNAL, "assertion: eliminator edges are not contiguous");
                    col += e.w;
                    // target span (solve.py:80-87)
                    if (e.kind == EDGE_SELF) {
                        se.lo = cf.offset + cf.r;
                    } else {
                        const ClusterFactor& of = rec.factors[rec.pos.at(e.other)];
                        se.lo = of.offset + (e.kind == EDGE_SKEL ? of.r : 0);
                    }
                    se.soff = soff;
                    auto g = groups.find(se.lo);
                    if (g == groups.end()) {
                        groups[se.lo] = {e.w, {soff}};
                        group_order.push_back(se.lo);
                    } else {
                        if (g->second.first != e.w) throw Error(H2F_E_INTERNAL, "assertion: scatter span mismatch");
                        g->second.second.push_back(soff);
                    }
                    soff += e.w;
                    edges.push_back(se);
                }
                sc.edge_end = int64_t(edges.size());
                sc.nch = cf.r > 0 ? int32_t(cdiv(std::max<int64_t>(sc.W, 1), SOLVE_GATHER_COLS)) : 0;
                woff += (int64_t(cf.s) + int64_t(sc.nch) * cf.r) * nrhs;
                const int ci = int(cls.size());
                cls.push_back(sc);
                for (int j = 0; j < cf.s; j += SOLVE_ROT_T_COLS)
                    tk[0].push_back({ci, ST_ROT_T, j, std::min(cf.s, j + SOLVE_ROT_T_COLS), 0, 0});
                for (int i = 0; i < cf.s; i += SOLVE_ROW_SLICE)
                    tk[3].push_back({ci, ST_ROT, i, std::min(cf.s, i + SOLVE_ROW_SLICE), 0, 0});
                if (cf.r > 0) {
                    tk[1].push_back({ci, ST_LSOLVE, 0, cf.r, 0, 0});
                    for (int64_t j = 0; j < sc.W; j += SOLVE_PROD_COLS)
                        tk[1].push_back({ci, ST_PROD, int32_t(j), int32_t(std::min<int64_t>(sc.W, j + SOLVE_PROD_COLS)),
                                         0, 0});
                    tk[2].push_back({ci, ST_USOLVE, 0, cf.r, 0, 0});
                    for (int64_t c0 = 0; c0 < std::max<int64_t>(sc.W, 1); c0 += SOLVE_GATHER_COLS) {
                        const int64_t c1 = std::min<int64_t>(sc.W, c0 + SOLVE_GATHER_COLS);
                        // the edges are consecutive column slices: only those
                        // overlapping [c0, c1) are scanned by the task
                        int64_t ea = sc.edge_begin, eb = sc.edge_begin;
                        while (ea < sc.edge_end && edges[ea].soff - sc.soff + edges[ea].w <= c0) ++ea;
                        eb = ea;
                        while (eb < sc.edge_end && edges[eb].soff - sc.soff < c1) ++eb;
                        for (int i = 0; i < cf.r; i += SOLVE_ROW_SLICE)
                            tk[2].push_back({ci, ST_GATHER, i, std::min(cf.r, i + SOLVE_ROW_SLICE), int32_t(c0),
                                             int32_t(c1), int32_t(ea), int32_t(eb)});
                    }
                } else {
                    // nothing eliminated: the rotated vector passes through
                    tk[1].push_back({ci, ST_LSOLVE, 0, 0, 0, 0});
                    tk[2].push_back({ci, ST_USOLVE, 0, 0, 0, 0});
                }
                double ew = double(sc.W);
                flops_b += (2.0 * cf.s * cf.s + 2.0 * cf.r * ew + double(cf.r) * cf.r) * nrhs;
                bytes_b += 8.0 * (double(cf.s) * cf.s + double(cf.r) * cf.r + cf.r * ew) +
                           16.0 * (cf.s + ew) * nrhs;
            }
            SolvePlan::Batch B;
            if (use_gemm) host_batches.push_back({P.levels.size(), L.batches.size(), cls, edges});
            std::vector<ScatterGroup> gs;
            std::vector<int64_t> list;
            for (int64_t lo : group_order) {
                auto& g = groups[lo];
                ScatterGroup sg{};
                sg.lo = lo;
                sg.w = g.first;
                sg.begin = int64_t(list.size());
                list.insert(list.end(), g.second.begin(), g.second.end());
                sg.end = int64_t(list.size());
                gs.push_back(sg);
            }
            B.ncl = int32_t(cls.size());
            B.cl = to_dev(P.mem, cls);
            B.edges = to_dev(P.mem, edges);
            B.ngroups = int32_t(gs.size());
            {
                int64_t wmax = 1;
                for (auto& g : gs) wmax = std::max<int64_t>(wmax, g.w);
                B.scatter_split = int32_t(std::min<int64_t>(64, cdiv(wmax * nrhs, 4096)));
            }
            B.groups = to_dev(P.mem, gs);
            B.list = to_dev(P.mem, list);
            for (int q = 0; q < 4; ++q) {
                B.tk[q] = to_dev(P.mem, tk[q]);
                B.ntk[q] = int32_t(tk[q].size());
            }
            B.fwd_flops = flops_b;
            B.fwd_bytes = bytes_b;
            B.sc_bytes = 16.0 * double(soff) * nrhs;
            L.batches.push_back(B);
            scratch_rows = std::max(scratch_rows, soff);
            work_max = std::max(work_max, woff);
        }
        P.levels.push_back(std::move(L));
    }
    for (auto& L : P.levels) P.yv.push_back(P.mem.alloc_n<double>(L.total * nrhs));
    P.ytop = P.mem.alloc_n<double>(std::max<int64_t>(f.top_size, 1) * nrhs);
    P.ttop = P.mem.alloc_n<double>(std::max<int64_t>(f.top_size, 1) * nrhs);
    P.top_perm = P.mem.alloc_n<int32_t>(std::max<int64_t>(f.top_size, 1));
    P.top_sync = P.mem.alloc_n<int32_t>(f.top_size / 64 + 2);
    launch_top_perm(f.top_piv, int32_t(f.top_size), P.top_perm, ctx().stream);
    P.scratch = P.mem.alloc_n<double>(std::max<int64_t>(scratch_rows, 1) * nrhs);
    P.work = P.mem.alloc_n<double>(std::max<int64_t>(work_max, 1));
    for (auto& hb : host_batches) {
        SolvePlan::Batch& B = P.levels[hb.level].batches[hb.batch];
        double* yv = P.yv[hb.level];
        GemmBuild frot, fprod, bgat, brot;
        CopyBuild fcopy, bcopy;
        std::vector<CopyBuild> badd;
        std::vector<TrsmTask> ft[2], bt[2];
        int mr[2] = {1, 1};
        double tf = 0;
        int64_t wo = 0;
        for (auto& sc : hb.cls) {
            const int s_ = sc.s, r_ = sc.r;
            double* yc = yv + sc.off * q;
            double* wk = P.work + wo;
            double* acc = wk + int64_t(s_) * q;
            const int nsplit = r_ > 0 ? int(std::max<int64_t>(1, cdiv(sc.W, SOLVE_GATHER_COLS))) : 0;
            wo += (int64_t(s_) + int64_t(nsplit) * r_) * q;
            // forward (solve.py:90-128): wk = Q~^T y_c
            frot.add1(wk, q, s_, q, GEMM_STORE, contrib(sc.q, s_, 1, yc, q, 0, s_));
            // skeleton rows pass through; redundant rows are solved below
            fcopy.add(yc + int64_t(r_) * q, q, s_ - r_, q, wk + int64_t(r_) * q, q, 0, COPY_SET);
            // backward (solve.py:131-164): y_c = Q~ y_c (after the TRSM and the gather-add)
            brot.add1(wk, q, s_, q, GEMM_STORE, contrib(sc.q, s_, 0, yc, q, 0, s_));
            bcopy.add(yc, q, s_, q, wk, q, 0, COPY_SET);
            if (r_ == 0) continue;
            // products (W x q) = (-W)^T y_R into the scatter scratch
            fprod.add1(P.scratch + sc.soff * q, q, int(sc.W), q, GEMM_STORE, contrib(sc.mw, sc.W, 1, wk, q, 0, r_));
            const int nc = trsm_dmma_cols(r_), vi = nc == 32 ? 0 : 1;
            mr[vi] = std::max(mr[vi], r_);
            tf += double(r_) * r_ * q;
            for (int c0 = 0; c0 < q; c0 += nc) {
                TrsmTask t{};
                t.LU = sc.lu;
                t.piv = sc.piv;
                t.r = r_;
                t.W = q;
                t.col0 = c0;
                t.ldg = t.ldw = q;
                t.G = wk;
                t.MW = yc;
                t.mode = TRSM_LOWER;
                ft[vi].push_back(t);
                t.G = yc;
                t.mode = TRSM_UPPER;
                bt[vi].push_back(t);
            }
            // gather acc = sum_e (-W_e) y[span_e], split-K: the concatenated
            // edge columns are cut into SOLVE_GATHER_COLS-wide ranges, each a
            // GEMM task into its own partial (r x q), the partials are added
            // to y_R in range order (deterministic)
            std::vector<std::vector<GemmContrib>> cs(nsplit);
            int64_t col = 0;
            for (int64_t e = sc.edge_begin; e < sc.edge_end; ++e) {
                const SolveEdge& E = hb.edges[e];
                for (int k0 = 0; k0 < E.w;) {
                    const int part = int(col / SOLVE_GATHER_COLS);
                    const int len = int(std::min<int64_t>(E.w - k0, (part + 1) * int64_t(SOLVE_GATHER_COLS) - col));
                    cs[part].push_back(contrib(E.mat + k0, E.ld, 0, yv + (E.lo + k0) * q, q, 0, len));
                    k0 += len;
                    col += len;
                }
            }
            if (int(badd.size()) < nsplit) badd.resize(nsplit);
            for (int part = 0; part < nsplit; ++part) {
                double* dst = acc + int64_t(part) * r_ * q;
                bgat.add(dst, q, r_, q, GEMM_STORE, cs[part].data(), cs[part].size());
                badd[part].add(yc, q, r_, q, dst, q, 0, COPY_ADD);
            }
        }
        B.f_rot.build(P.mem, frot);
        B.f_prod.build(P.mem, fprod);
        B.f_copy.build(P.mem, fcopy);
        B.f_trsm.build(P.mem, ft, mr, tf);
        B.b_trsm.build(P.mem, bt, mr, tf);
        B.b_gather.build(P.mem, bgat);
        B.b_add.resize(badd.size());
        for (size_t i = 0; i < badd.size(); ++i) B.b_add[i].build(P.mem, badd[i]);
        B.b_rot.build(P.mem, brot);
        B.b_copy.build(P.mem, bcopy);
        B.gemm = true;
    }
    ctx().sync();
    auto& ref = *plan;
    f.plans[nrhs] = std::move(plan);
    return ref;
}

}  // namespace

namespace {

// Dense top solve (solve.py:46-55) for a block of right-hand sides: row
// permutation, then blocked forward/backward substitution in 64-row steps --
// the diagonal block by the DMMA TRSM kernel, the rest of the column by one
// DMMA tile GEMM per step -- so the top LU is streamed twice per solve
// instead of once per right-hand side.
void top_solve_blocked(Factorization& f, SolvePlan& P, cudaStream_t st) {
    const int64_t n = f.top_size;
    const int q = P.nrhs;
    if (n == 0) return;
    constexpr int NB = 64;
    launch_permute_rows(P.ytop, P.top_perm, int32_t(n), q, P.ttop, st);
    const int nc = trsm_dmma_cols(NB);
    auto diag = [&](int64_t k0, int nb, int mode) {
        std::vector<TrsmTask> ts;
        for (int c0 = 0; c0 < q; c0 += nc) {
            TrsmTask t{};
            t.LU = f.top_lu + k0 * n + k0;
            t.ldlu = n;
            t.piv = nullptr;
            t.G = P.ttop + k0 * q;
            t.MW = P.ttop + k0 * q;
            t.ldg = t.ldw = q;
            t.r = nb;
            t.W = q;
            t.col0 = c0;
            t.mode = mode;
            ts.push_back(t);
        }
        launch_trsm_dmma(upload(ts), int32_t(ts.size()), nb, nc, st);
    };
    for (int64_t k0 = 0; k0 < n; k0 += NB) {  // L y = P b
        const int nb = int(std::min<int64_t>(NB, n - k0));
        diag(k0, nb, TRSM_LOWER);
        const int64_t rest = n - k0 - nb;
        if (rest <= 0) continue;
        GemmBuild g;
        g.add1(P.ttop + (k0 + nb) * q, q, int(rest), q, GEMM_ADD,
               contrib(f.top_lu + (k0 + nb) * n + k0, n, 0, P.ttop + k0 * q, q, 0, nb, -1.0));
        g.launch(-1);
    }
    for (int64_t k0 = ((n - 1) / NB) * NB; k0 >= 0; k0 -= NB) {  // U x = y
        const int nb = int(std::min<int64_t>(NB, n - k0));
        diag(k0, nb, TRSM_UPPER);
        if (k0 == 0) continue;
        GemmBuild g;
        g.add1(P.ttop, q, int(k0), q, GEMM_ADD,
               contrib(f.top_lu + k0, n, 0, P.ttop + k0 * q, q, 0, nb, -1.0));
        g.launch(-1);
    }
    H2F_CUDA(cudaMemcpyAsync(P.ytop, P.ttop, sizeof(double) * n * q, cudaMemcpyDeviceToDevice, st));
}

}  // namespace

namespace {

// the substitution proper on the plan's own buffers: P.yv[0] (b in, x out)
void solve_sweeps(Factorization& f, SolvePlan& P, int nrhs, cudaStream_t st) {
    const size_t R = P.levels.size();
    for (size_t li = 0; li < R; ++li) {
        auto& L = P.levels[li];
        for (auto& B : L.batches) {
            if (B.gemm) {
                B.f_rot.launch(K_SOLVE_FWD, st);
                B.f_prod.launch(K_SOLVE_FWD, st);
                B.f_trsm.launch(K_TRSM, st);
                B.f_copy.launch(K_COPY, st);
                ProfScope ps(K_SOLVE_SCATTER, 0.0, B.sc_bytes);
                launch_fwd_scatter(B.groups, B.ngroups, B.list, P.scratch, P.yv[li], nrhs, st, B.scatter_split);
                continue;
            }
            {
                ProfScope ps(K_SOLVE_FWD, B.fwd_flops, B.fwd_bytes);
                launch_solve_tasks(B.tk[0], B.ntk[0], B.cl, B.edges, P.yv[li], P.scratch, P.work, nrhs, st);
                launch_solve_tasks(B.tk[1], B.ntk[1], B.cl, B.edges, P.yv[li], P.scratch, P.work, nrhs, st);
            }
            ProfScope ps(K_SOLVE_SCATTER, 0.0, B.sc_bytes);
            launch_fwd_scatter(B.groups, B.ngroups, B.list, P.scratch, P.yv[li], nrhs, st);
        }
        double* next = (li + 1 < R) ? P.yv[li + 1] : P.ytop;
        launch_gather_rows(P.yv[li], L.up, L.up_n, nrhs, next, st);
    }
    {
        const double nt = double(f.top_size);
        ProfScope ps(K_SOLVE_TOP, 2.0 * nt * nt * nrhs, 8.0 * nt * nt);
        if (nrhs >= SOLVE_GEMM_MIN_RHS) top_solve_blocked(f, P, st);
        else launch_top_solve(f.top_lu, P.top_perm, int(f.top_size), P.ytop, nrhs, P.ttop, P.top_sync, st);
    }
    for (size_t li = R; li-- > 0;) {
        auto& L = P.levels[li];
        const double* src = (li + 1 < R) ? P.yv[li + 1] : P.ytop;
        launch_scatter_rows(src, L.up, L.up_n, nrhs, P.yv[li], st);
        for (size_t bi = L.batches.size(); bi-- > 0;) {
            auto& B = L.batches[bi];
            if (B.gemm) {
                B.b_trsm.launch(K_TRSM, st);
                B.b_gather.launch(K_SOLVE_BWD, st);
                for (auto& a : B.b_add) a.launch(K_COPY, st);
                B.b_rot.launch(K_SOLVE_BWD, st);
                B.b_copy.launch(K_COPY, st);
                continue;
            }
            ProfScope ps(K_SOLVE_BWD, B.fwd_flops, B.fwd_bytes);
            launch_solve_tasks(B.tk[2], B.ntk[2], B.cl, B.edges, P.yv[li], P.scratch, P.work, nrhs, st);
            launch_solve_tasks(B.tk[3], B.ntk[3], B.cl, B.edges, P.yv[li], P.scratch, P.work, nrhs, st);
        }
    }
}

}  // namespace

void solve_device(Factorization& f, const double* b_dev, double* x_dev, int nrhs) {
    SolvePlan& P = get_plan(f, nrhs);
    cudaStream_t st = ctx().stream;
    const size_t nb = sizeof(double) * f.n * nrhs;
    if (f.recs.empty()) {
        // solve.py:46-47
        H2F_CUDA(cudaMemcpyAsync(P.ytop, b_dev, nb, cudaMemcpyDeviceToDevice, st));
        launch_top_solve(f.top_lu, P.top_perm, int(f.top_size), P.ytop, nrhs, P.ttop, P.top_sync, st);
        H2F_CUDA(cudaMemcpyAsync(x_dev, P.ytop, nb, cudaMemcpyDeviceToDevice, st));
        return;
    }
    H2F_CUDA(cudaMemcpyAsync(P.yv[0], b_dev, nb, cudaMemcpyDeviceToDevice, st));
    // The single-vector sweeps (thousands of small launches, every task list
    // pre-uploaded into the plan) are captured once into a CUDA graph and
    // replayed: no per-launch host cost and no launch gaps on the device.
    // Not with the per-kernel profiler on (its events must stay per launch)
    // nor for the block path (its top solve uploads task lists per call).
    static const bool graphs = [] {
        const char* e = std::getenv("H2F_SOLVE_GRAPH");
        return !(e && std::atoi(e) == 0);
    }();
    // capturing + instantiating costs about one direct run, so a plan is
    // captured on its third use (a refined solve uses its plan twice)
    if (graphs && nrhs < SOLVE_GEMM_MIN_RHS && !ctx().prof.on && ++P.uses >= 3) {
        if (!P.graph) {
            const int64_t l0 = kernel_launch_count();
            cudaGraph_t g = nullptr;
            H2F_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            solve_sweeps(f, P, nrhs, st);
            H2F_CUDA(cudaStreamEndCapture(st, &g));
            H2F_CUDA(cudaGraphInstantiate(&P.graph, g, 0));
            cudaGraphDestroy(g);
            P.graph_launches = kernel_launch_count() - l0;
            add_launches(-P.graph_launches);  // counted when the graph runs
        }
        H2F_CUDA(cudaGraphLaunch(P.graph, st));
        add_launches(P.graph_launches);
    } else {
        solve_sweeps(f, P, nrhs, st);
    }
    H2F_CUDA(cudaMemcpyAsync(x_dev, P.yv[0], nb, cudaMemcpyDeviceToDevice, st));
}

void refined_solve_device(H2Mat& m, Factorization& f, const double* b_dev, double* x_dev, int steps, int nrhs) {
    // solve.py:63-77; nrhs > 1 refines every column at once (block matvec
    // and block substitution; the reference's refined_solve is single-vector)
    cudaStream_t st = ctx().stream;
    const int64_t n = f.n * int64_t(nrhs);
    // refinement temporaries: the factor's work region, rewound on every call
    Region& w = f.work;
    w.reset();
    double* tmp = w.alloc_n<double>(n);
    double* res = w.alloc_n<double>(n);
    double* dx = w.alloc_n<double>(n);
    solve_device(f, b_dev, x_dev, nrhs);
    for (int it = 0; it < steps; ++it) {
        matvec_device(m, x_dev, tmp, nrhs);
        launch_axpby(res, b_dev, 1.0, tmp, -1.0, n, st);
        solve_device(f, res, dx, nrhs);
        launch_axpby(x_dev, x_dev, 1.0, dx, 1.0, n, st);
    }
}

}  // namespace h2f
