// H2 operator upload, matvec plan and power-iteration norm estimate.
//
// matvec (h2core.py:285-315) becomes a fixed sequence of batched GEMV task
// launches built once per operator: leaf projections V^T x, the upward
// transfer sweep, couplings (both orientations), the downward sweep, and a
// final per-leaf gather of dense blocks (both orientations) plus V yhat.  Each
// output segment is owned by one CTA that sums its contributions in a fixed
// order, so there are no write conflicts and no atomics.
#include <cstring>
#include "h2mat.h"

#include <algorithm>
#include <cmath>

namespace h2f {

H2Mat::~H2Mat() {
    plans.clear();
    if (vals && ctx_ready()) dfree(vals);
}

namespace {

std::unique_ptr<H2Mat> h2mat_structure(const h2f_matrix_desc* d) {
    if (!d || d->n <= 0 || d->num_nodes <= 0) throw Error(H2F_E_ARG, "empty H2 matrix description");
    auto m = std::make_unique<H2Mat>();
    m->n = d->n;
    m->depth = d->depth;
    m->top = d->top_level;
    m->nnodes = d->num_nodes;
    const int64_t N = d->num_nodes;
    auto cp = [N](const int64_t* p) { return std::vector<int64_t>(p, p + N); };
    m->parent = cp(d->parent);
    m->left = cp(d->child_left);
    m->right = cp(d->child_right);
    m->level = cp(d->level);
    m->begin = cp(d->begin);
    m->end = cp(d->end);
    m->rank = cp(d->rank);
    m->leaf_basis_off = cp(d->leaf_basis_off);
    m->transfer_off = cp(d->transfer_off);
    const int nlev = m->depth + 1;
    m->levels.assign(nlev, {});
    for (int64_t c = 0; c < N; ++c) {
        if (m->level[c] < 0 || m->level[c] >= nlev) throw Error(H2F_E_ARG, "node level out of range");
        m->levels[m->level[c]].push_back(int(c));
    }
    auto read_pairs = [&](const int64_t* pairs, const int64_t* ptr, std::vector<std::vector<std::pair<int, int>>>& out) {
        out.assign(nlev, {});
        for (int l = 0; l < nlev; ++l)
            for (int64_t i = ptr[l]; i < ptr[l + 1]; ++i) out[l].push_back({int(pairs[2 * i]), int(pairs[2 * i + 1])});
    };
    read_pairs(d->adm_pairs, d->adm_ptr, m->adm);
    read_pairs(d->inner_pairs, d->inner_ptr, m->inner);
    read_pairs(d->dense_pairs, d->dense_ptr, m->dense);
    m->adm_set.assign(nlev, {});
    m->dense_set.assign(nlev, {});
    int64_t ia = 0, id = 0;
    for (int l = 0; l < nlev; ++l) {
        for (auto& p : m->adm[l]) {
            m->adm_set[l].insert(mkkey(p.first, p.second));
            m->coupling_off[mkkey(p.first, p.second)] = d->coupling_off[ia++];
        }
        for (auto& p : m->inner[l]) m->dense_set[l].insert(mkkey(p.first, p.second));
        for (auto& p : m->dense[l]) {
            m->dense_set[l].insert(mkkey(p.first, p.second));
            m->dense_off[mkkey(p.first, p.second)] = d->dense_off[id++];
        }
    }
    m->nvals = d->nvals;
    m->coupling_list.assign(d->coupling_off, d->coupling_off + d->adm_ptr[nlev]);
    m->dense_list.assign(d->dense_off, d->dense_off + d->dense_ptr[nlev]);
    return m;
}

}  // namespace

H2Mat* h2mat_create(const h2f_matrix_desc* d, const double* host_vals) {
    auto m = h2mat_structure(d);
    m->vals = static_cast<double*>(dalloc(sizeof(double) * std::max<int64_t>(d->nvals, 1)));
    if (d->nvals)
        H2F_CUDA(cudaMemcpyAsync(m->vals, host_vals, sizeof(double) * d->nvals, cudaMemcpyHostToDevice,
                                 ctx().stream));
    ctx().sync();
    return m.release();
}

H2Mat* h2mat_create_blocks(const h2f_matrix_desc* d, int64_t nblk, const double* const* ptrs, const int64_t* counts,
                           const int64_t* offs) {
    // the value array is assembled chunk by chunk in pinned staging memory
    // (OpenMP copies of the blocks overlapping the chunk) and shipped with
    // async copies, two staging buffers alternating: packing overlaps the
    // transfer, and no host-side copy of the whole operator is made
    for (int64_t i = 0; i < nblk; ++i)
        if (counts[i] < 0 || offs[i] < 0 || offs[i] + counts[i] > d->nvals || (i && offs[i] < offs[i - 1]))
            throw Error(H2F_E_ARG, "block list: offsets must be ascending and inside nvals");
    auto m = h2mat_structure(d);
    m->vals = static_cast<double*>(dalloc(sizeof(double) * std::max<int64_t>(d->nvals, 1)));
    cudaStream_t st = ctx().stream;
    constexpr int64_t CH = int64_t(32) << 20;  // doubles per chunk (256 MB)
    double* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    const int64_t nchunk = (d->nvals + CH - 1) / CH;
    const int nbuf = nchunk > 1 ? 2 : 1;
    try {
        for (int b = 0; b < nbuf; ++b) {
            H2F_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stage[b]), sizeof(double) * std::min(CH, std::max<int64_t>(d->nvals, 1)),
                                   cudaHostAllocDefault));
            H2F_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
        }
        int64_t first = 0;  // first block that may overlap the chunk
        for (int64_t k = 0; k < nchunk; ++k) {
            const int b = int(k % nbuf);
            const int64_t lo = k * CH, hi = std::min(d->nvals, lo + CH);
            if (k >= nbuf) H2F_CUDA(cudaEventSynchronize(done[b]));  // its previous transfer is complete
            while (first < nblk && offs[first] + counts[first] <= lo) ++first;
            int64_t last = first;
            while (last < nblk && offs[last] < hi) ++last;
            double* dst = stage[b];
            std::memset(dst, 0, sizeof(double) * size_t(hi - lo));  // gaps between blocks (none in practice)
#pragma omp parallel for schedule(dynamic, 64)
            for (int64_t i = first; i < last; ++i) {
                const int64_t a = std::max(lo, offs[i]), e = std::min(hi, offs[i] + counts[i]);
                if (e > a) std::memcpy(dst + (a - lo), ptrs[i] + (a - offs[i]), sizeof(double) * size_t(e - a));
            }
            H2F_CUDA(cudaMemcpyAsync(m->vals + lo, dst, sizeof(double) * size_t(hi - lo), cudaMemcpyHostToDevice, st));
            H2F_CUDA(cudaEventRecord(done[b], st));
        }
        ctx().sync();
    } catch (...) {
        for (int b = 0; b < 2; ++b) {
            if (done[b]) cudaEventDestroy(done[b]);
            if (stage[b]) cudaFreeHost(stage[b]);
        }
        throw;
    }
    for (int b = 0; b < 2; ++b) {
        if (done[b]) cudaEventDestroy(done[b]);
        if (stage[b]) cudaFreeHost(stage[b]);
    }
    return m.release();
}

H2Mat* h2mat_create_device(const h2f_matrix_desc* d, double* dev_vals) {
    std::unique_ptr<H2Mat> m;
    try {
        m = h2mat_structure(d);
    } catch (...) {
        dfree(dev_vals);
        throw;
    }
    m->vals = dev_vals;
    return m.release();
}

int sparsity_constant(const H2Mat& m, int level) {
    // structure.py:127-134
    std::unordered_map<int, int> cnt;
    for (Key k : m.dense_set[level]) {
        cnt[key_a(k)]++;
        if (key_a(k) != key_b(k)) cnt[key_b(k)]++;
    }
    int mx = 0;
    for (auto& kv : cnt) mx = std::max(mx, kv.second);
    return mx;
}

MatvecPlan& matvec_plan(H2Mat& m, int nrhs) {
    // cached per nrhs, at most 3 alive (least recently used evicted: each
    // holds O(n nrhs) of vectors in its own region)
    static int64_t clock = 0;
    auto it = m.plans.find(nrhs);
    if (it != m.plans.end()) {
        it->second->last_use = ++clock;
        return *it->second;
    }
    while (m.plans.size() >= 3) {
        auto victim = m.plans.begin();
        for (auto jt = m.plans.begin(); jt != m.plans.end(); ++jt)
            if (jt->second->last_use < victim->second->last_use) victim = jt;
        ctx().sync();  // no launch of the victim's task lists is in flight
        m.plans.erase(victim);
    }
    auto plan = std::make_unique<MatvecPlan>();
    plan->last_use = ++clock;
    MatvecPlan& P = *plan;
    P.nrhs = nrhs;
    const int64_t n = m.n;
    P.xin = P.mem.alloc_n<double>(n * nrhs);
    P.yout = P.mem.alloc_n<double>(n * nrhs);
    P.partial = P.mem.alloc_n<double>(256);
    P.est = P.mem.alloc_n<double>(64);
    // coefficient offsets for every node carrying a basis
    std::vector<int64_t> hoff(m.nnodes, -1);
    int64_t htot = 0;
    const bool has_h2 = m.top >= 0;
    if (has_h2)
        for (int l = m.top; l <= m.depth; ++l)
            for (int c : m.levels[l]) {
                hoff[c] = htot;
                htot += std::max<int64_t>(m.rank[c], 0);
            }
    P.xh = P.mem.alloc_n<double>(htot * nrhs);
    P.yh = P.mem.alloc_n<double>(htot * nrhs);

    struct Builder {
        std::vector<GemvTask> tasks;
        std::vector<GemvContrib> contribs;
    };
    std::vector<Builder> stages;
    auto task = [&](Builder& b, double* y, int rows, int mode) {
        GemvTask t{};
        t.y = y;
        t.rows = rows;
        t.mode = mode;
        t.contrib_begin = t.contrib_end = (int64_t)b.contribs.size();
        b.tasks.push_back(t);
    };
    auto contrib = [&](Builder& b, const double* A, int64_t lda, int cols, int trans, const double* x) {
        GemvContrib c{};
        c.A = A;
        c.lda = lda;
        c.cols = cols;
        c.trans = trans;
        c.x = x;
        c.alpha = 1.0;
        b.contribs.push_back(c);
        b.tasks.back().contrib_end = (int64_t)b.contribs.size();
    };
    auto xh = [&](int c) { return P.xh + hoff[c] * nrhs; };
    auto yh = [&](int c) { return P.yh + hoff[c] * nrhs; };

    if (has_h2) {
        // 1. leaf coefficients xhat = V^T x
        Builder b;
        for (int c : m.levels[m.depth]) {
            if (m.rank[c] <= 0 || m.leaf_basis_off[c] < 0) continue;
            task(b, xh(c), int(m.rank[c]), COPY_SET);
            contrib(b, m.leaf_basis(c), m.rank[c], int(m.rows(c)), 1, P.xin + m.begin[c] * nrhs);
        }
        stages.push_back(std::move(b));
        // 2. upward sweep
        for (int l = m.depth - 1; l >= m.top; --l) {
            Builder u;
            for (int p : m.levels[l]) {
                if (m.rank[p] <= 0) continue;
                task(u, xh(p), int(m.rank[p]), COPY_SET);
                for (int64_t ch : {m.left[p], m.right[p]}) {
                    if (ch < 0 || m.rank[ch] <= 0) continue;
                    contrib(u, m.transfer(int(ch)), m.rank[p], int(m.rank[ch]), 1, xh(int(ch)));
                }
            }
            stages.push_back(std::move(u));
        }
        // 3. couplings (both orientations)
        Builder cb;
        std::vector<std::vector<std::pair<Key, int>>> by_node(m.nnodes);
        for (int l = m.top; l <= m.depth; ++l)
            for (auto& pr : m.adm[l]) {
                by_node[pr.first].push_back({mkkey(pr.first, pr.second), 0});
                by_node[pr.second].push_back({mkkey(pr.first, pr.second), 1});
            }
        for (int l = m.top; l <= m.depth; ++l)
            for (int c : m.levels[l]) {
                if (m.rank[c] <= 0) continue;
                task(cb, yh(c), int(m.rank[c]), COPY_SET);
                for (auto& e : by_node[c]) {
                    const int s = key_a(e.first), t = key_b(e.first);
                    if (e.second == 0)
                        contrib(cb, m.coupling(e.first), m.rank[t], int(m.rank[t]), 0, xh(t));
                    else
                        contrib(cb, m.coupling(e.first), m.rank[t], int(m.rank[s]), 1, xh(s));
                }
            }
        stages.push_back(std::move(cb));
        // 4. downward sweep
        for (int l = m.top + 1; l <= m.depth; ++l) {
            Builder dn;
            for (int c : m.levels[l]) {
                if (m.rank[c] <= 0) continue;
                const int p = int(m.parent[c]);
                if (m.rank[p] <= 0) continue;
                task(dn, yh(c), int(m.rank[c]), COPY_ADD);
                contrib(dn, m.transfer(c), m.rank[p], int(m.rank[p]), 0, yh(p));
            }
            stages.push_back(std::move(dn));
        }
    }
    // 5. leaves: dense blocks (both orientations) + V yhat
    {
        Builder lb;
        std::vector<std::vector<std::pair<Key, int>>> by_leaf(m.nnodes);
        for (int l = 0; l <= m.depth; ++l)
            for (auto& pr : m.dense[l]) {
                by_leaf[pr.first].push_back({mkkey(pr.first, pr.second), 0});
                if (pr.first != pr.second) by_leaf[pr.second].push_back({mkkey(pr.first, pr.second), 1});
            }
        for (int64_t c = 0; c < m.nnodes; ++c) {
            if (!m.is_leaf(int(c))) continue;
            task(lb, P.yout + m.begin[c] * nrhs, int(m.rows(c)), COPY_SET);
            for (auto& e : by_leaf[c]) {
                const int s = key_a(e.first), t = key_b(e.first);
                const double* D = m.vals + m.dense_off.at(e.first);
                if (e.second == 0)
                    contrib(lb, D, m.rows(t), int(m.rows(t)), 0, P.xin + m.begin[t] * nrhs);
                else
                    contrib(lb, D, m.rows(t), int(m.rows(s)), 1, P.xin + m.begin[s] * nrhs);
            }
            if (has_h2 && m.rank[c] > 0 && m.leaf_basis_off[c] >= 0)
                contrib(lb, m.leaf_basis(int(c)), m.rank[c], int(m.rank[c]), 0, yh(int(c)));
        }
        stages.push_back(std::move(lb));
    }
    for (auto& b : stages) {
        if (b.tasks.empty()) continue;
        GemvLaunch L;
        L.ntasks = int32_t(b.tasks.size());
        for (auto& t : b.tasks) L.max_rows = std::max(L.max_rows, t.rows);
        for (auto& t : b.tasks)
            for (int64_t ci = t.contrib_begin; ci < t.contrib_end; ++ci) {
                const double e = double(t.rows) * b.contribs[ci].cols;
                L.flops += 2.0 * e * nrhs;
                L.bytes += 8.0 * e + 8.0 * b.contribs[ci].cols * nrhs;
            }
        L.tasks = P.mem.alloc_n<GemvTask>(b.tasks.size());
        L.contribs = P.mem.alloc_n<GemvContrib>(std::max<size_t>(b.contribs.size(), 1));
        H2F_CUDA(cudaMemcpyAsync(L.tasks, b.tasks.data(), sizeof(GemvTask) * b.tasks.size(),
                                 cudaMemcpyHostToDevice, ctx().stream));
        if (!b.contribs.empty())
            H2F_CUDA(cudaMemcpyAsync(L.contribs, b.contribs.data(), sizeof(GemvContrib) * b.contribs.size(),
                                     cudaMemcpyHostToDevice, ctx().stream));
        P.launches.push_back(L);
    }
    ctx().sync();
    auto& ref = *plan;
    m.plans[nrhs] = std::move(plan);
    return ref;
}

static void run_plan(MatvecPlan& P) {
    for (auto& L : P.launches) {
        ProfScope ps(K_MATVEC, L.flops, L.bytes);
        launch_gemv_tasks(L.tasks, L.ntasks, L.contribs, P.nrhs, ctx().stream, L.max_rows);
    }
}

void matvec_device(H2Mat& m, const double* x_dev, double* y_dev, int nrhs) {
    MatvecPlan& P = matvec_plan(m, nrhs);
    cudaStream_t st = ctx().stream;
    const size_t bytes = sizeof(double) * m.n * nrhs;
    H2F_CUDA(cudaMemcpyAsync(P.xin, x_dev, bytes, cudaMemcpyDeviceToDevice, st));
    run_plan(P);
    H2F_CUDA(cudaMemcpyAsync(y_dev, P.yout, bytes, cudaMemcpyDeviceToDevice, st));
}

double norm2_estimate(H2Mat& m, const double* v0_host, int iters) {
    // h2core.py:318-330; v0 already normalised on the host (Philox start)
    MatvecPlan& P = matvec_plan(m, 1);
    cudaStream_t st = ctx().stream;
    if (iters > 64) throw Error(H2F_E_ARG, "at most 64 power iterations");
    H2F_CUDA(cudaMemcpyAsync(P.xin, v0_host, sizeof(double) * m.n, cudaMemcpyHostToDevice, st));
    for (int it = 0; it < iters; ++it) {
        run_plan(P);
        launch_norm2(P.yout, m.n, P.partial, P.est + it, st);
        launch_scale_by_inv(P.xin, P.yout, m.n, P.est + it, st);
    }
    double* h = static_cast<double*>(ctx().pinned_buf(sizeof(double) * 64));
    if (iters > 0)
        H2F_CUDA(cudaMemcpyAsync(h, P.est, sizeof(double) * iters, cudaMemcpyDeviceToHost, st));
    ctx().sync();
    double est = 0.0;
    for (int it = 0; it < iters; ++it) {
        est = h[it];
        if (est == 0.0) return 0.0;
    }
    return est;
}

}  // namespace h2f
