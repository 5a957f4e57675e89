// RS-S factorization driver (Alg. 1/2; factorization.py:204-615) for B200.
//
// The host keeps only integer structure: the level's block maps (dense D, fill
// F), neighbour lists, the greedy colouring and the batch picker (all
// bit-exact with the reference), and the offsets of every block in the
// device arena.  Every floating-point operation of a batch runs as a handful
// of batched kernel launches over all clusters of the batch:
//
//   augment     copy(F-row gather) -> gemm(V^T Y) -> gemm(Y -= V C) -> qr_r ->
//               jacobi(svd, kept, vbar) -> complement(Q~)            [1 sync: kept]
//   project     gemm(Q~^T B | B Q~) (out of place, new arena views)
//   eliminate   copy(G panels) -> lu -> trsm(-W) -> gemm(Schur targets +=,
//               fill-candidate norms) -> reduce             [1 sync: norms, status]
//               -> gemm(create the surviving fill blocks, in reference order)
//   slice       host-only view arithmetic (factorization.py:513-523)
//
// Level transition and the dense top are batched copy launches plus a blocked
// partial-pivot LU whose trailing updates run on the DMMA tile GEMM.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <iterator>
#include <numeric>
#include <set>

#include <nvtx3/nvToolsExt.h>

#include "builders.h"
#include "coloring.h"
#include "dense.h"
#include "factor.h"

namespace h2f {

Replay& replay() {
    static Replay r;
    return r;
}

ShardStats& shard_stats() {
    static ShardStats st;
    return st;
}

std::vector<int> shard_owners_tree(int64_t nnodes, const int64_t* parent, const int64_t* level, int top,
                                   int world) {
    // contiguous subtrees: the top-level clusters (ascending id = left to
    // right) split into `world` equal runs; every descendant follows its
    // ancestor, so a parent and its children always share an owner and the
    // level transition (factorization.py:548-588) needs no exchange
    if (world < 1) throw Error(H2F_E_ARG, "world size must be >= 1");
    std::vector<int> own(size_t(nnodes), -1);
    if (world == 1) {
        std::fill(own.begin(), own.end(), 0);
        return own;
    }
    if (top < 0) throw Error(H2F_E_ARG, "sharded factorization needs a compressed level (dense-only operator)");
    std::vector<int> tops;
    for (int64_t c = 0; c < nnodes; ++c)
        if (level[c] == top) tops.push_back(int(c));
    if (int64_t(tops.size()) < world)
        throw Error(H2F_E_ARG, "sharded factorization: " + std::to_string(tops.size()) +
                                   " clusters at the top level for " + std::to_string(world) + " ranks");
    for (size_t i = 0; i < tops.size(); ++i) own[tops[i]] = int(int64_t(i) * world / int64_t(tops.size()));
    // node ids grow with depth (parents before children)
    for (int64_t c = 0; c < nnodes; ++c)
        if (level[c] > top) {
            if (parent[c] < 0 || parent[c] >= c) throw Error(H2F_E_ARG, "tree: parent after child");
            own[c] = own[parent[c]];
        }
    return own;
}

std::vector<int> shard_owners(const H2Mat& M, int world) {
    return shard_owners_tree(M.nnodes, M.parent.data(), M.level.data(), M.top, world);
}

namespace {

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double s() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

constexpr double PIVOT_RTOL = 1e-14;      // factorization.py:47
constexpr double FILL_DROP_FACTOR = 1e-2; // factorization.py:55

struct View {
    double* p = nullptr;
    int64_t ld = 0;
    int rows = 0, cols = 0;
    // Schur-target slot of the current batch (valid when stamp == the batch
    // number); written only by the one bucket thread that owns the view
    mutable int64_t stamp = -1;
    mutable int slot = -1;
};

struct CouplingW {    // coupling block with logical zero padding (factorization.py:396-403)
    const double* p = nullptr;
    int64_t ld = 0;
    int rows = 0, cols = 0;
};

struct TransferW {    // transfer with logical zero rows (factorization.py:404-407)
    const double* p = nullptr;
    int64_t ld = 0;
    int rows = 0, cols = 0;
    bool has = false;
};

struct Entry {
    Key key;
    bool dense;
    View* v;  // the block itself (std::map nodes are stable)
};

// neighbour list of one cluster: flat, sorted by partner id (the order the
// reference's sorted neighbour entries follow)
class Nbrs {
  public:
    using Item = std::pair<int, Entry>;
    void set(int o, const Entry& e) {
        auto it = std::lower_bound(v_.begin(), v_.end(), o, [](const Item& a, int b) { return a.first < b; });
        if (it != v_.end() && it->first == o) it->second = e;
        else v_.insert(it, {o, e});
    }
    const Entry* find(int o) const {
        auto it = std::lower_bound(v_.begin(), v_.end(), o, [](const Item& a, int b) { return a.first < b; });
        return (it != v_.end() && it->first == o) ? &it->second : nullptr;
    }
    // many new partners at once (none present yet): one sorted merge instead
    // of an O(size) vector insert each -- the same final list as set() calls
    void merge_new(std::vector<Item>& add) {
        auto lt = [](const Item& a, const Item& b) { return a.first < b.first; };
        std::sort(add.begin(), add.end(), lt);
        std::vector<Item> out;
        out.reserve(v_.size() + add.size());
        std::merge(v_.begin(), v_.end(), add.begin(), add.end(), std::back_inserter(out), lt);
        for (size_t i = 1; i < out.size(); ++i)
            if (out[i].first == out[i - 1].first) throw Error(H2F_E_INTERNAL, "assertion: fill partner linked twice");
        v_.swap(out);
    }
    std::vector<Item>::const_iterator begin() const { return v_.begin(); }
    std::vector<Item>::const_iterator end() const { return v_.end(); }
    size_t size() const { return v_.size(); }

  private:
    std::vector<Item> v_;
};

struct Lvl {
    int level = 0;
    std::vector<int> clusters;
    std::unordered_map<int, int> pos;
    std::vector<int64_t> offset, size;
    std::vector<int> live, red, k;
    std::vector<char> done;
    std::vector<View> basis;
    std::vector<double*> qv;  // [V_perp | V] per cluster, computed at level start
    std::map<Key, View> D, F;
    std::vector<View*> diag;  // D(c, c) per position
    std::vector<Nbrs> touch;
    std::unordered_map<Key, CouplingW> S;
    std::vector<TransferW> T;
    Region mem{size_t(256) << 20};
    std::vector<std::vector<int>> batches;
    std::vector<Key> fill_init;
    std::vector<std::vector<Key>> fill_created;
    std::vector<ClusterFactor> factors;

    int at(int c) const { return pos.at(c); }
    void link(Key key, bool dense) {
        View* v = &block(key, dense);
        touch[at(key_a(key))].set(key_b(key), {key, dense, v});
        touch[at(key_b(key))].set(key_a(key), {key, dense, v});
    }
    View& block(Key key, bool dense) { return dense ? D.at(key) : F.at(key); }
    View* find(Key key) {
        auto it = D.find(key);
        if (it != D.end()) return &it->second;
        auto jt = F.find(key);
        return jt != F.end() ? &jt->second : nullptr;
    }
    void init_common(const std::vector<int>& cl) {
        clusters = cl;
        const size_t n = cl.size();
        for (size_t i = 0; i < n; ++i) pos[cl[i]] = int(i);
        live.assign(n, 0);
        red.assign(n, 0);
        k.assign(n, 0);
        done.assign(n, 0);
        basis.assign(n, {});
        qv.assign(n, nullptr);
        touch.assign(n, {});
        diag.assign(n, nullptr);
        T.assign(n, {});
        factors.assign(n, {});
    }
    void build_touch() {
        for (auto& kv : D)
            if (key_a(kv.first) != key_b(kv.first)) link(kv.first, true);
            else diag[at(key_a(kv.first))] = &kv.second;
        for (auto& kv : F) link(kv.first, false);
    }
    View& dcc(int ci) {
        if (!diag[ci]) throw Error(H2F_E_INTERNAL, "assertion: cluster without a diagonal block");
        return *diag[ci];
    }
};

// phase accounting from CUDA events (sums to the device-side wall time); the
// same marks open NVTX ranges named after the reference's phase keys
// (factorization.py:130-193 phase_seconds), visible to nsys / ncu --nvtx
class PhaseClock {
  public:
    ~PhaseClock() {
        if (open_) nvtxRangePop();
        for (auto& e : marks_) cudaEventDestroy(e.first);
    }
    void mark(int phase) {
        static const char* names[PH_COUNT] = {"norm", "extract", "color", "augment", "project", "partial_lu",
                                              "transition", "top"};
        if (open_) nvtxRangePop();
        open_ = phase >= 0 && phase < PH_COUNT;
        if (open_) nvtxRangePushA(names[phase]);
        cudaEvent_t e;
        H2F_CUDA(cudaEventCreate(&e));
        H2F_CUDA(cudaEventRecord(e, ctx().stream));
        marks_.push_back({e, phase});
    }
    size_t size() const { return marks_.size(); }
    // call after a stream sync; returns seconds between mark i and j
    double between(size_t i, size_t j) const {
        float ms = 0.f;
        H2F_CUDA(cudaEventElapsedTime(&ms, marks_[i].first, marks_[j].first));
        return ms * 1e-3;
    }
    void accumulate(double* out) const {
        for (size_t i = 0; i + 1 < marks_.size(); ++i)
            if (marks_[i].second >= 0) out[marks_[i].second] += between(i, i + 1);
    }

  private:
    std::vector<std::pair<cudaEvent_t, int>> marks_;
    bool open_ = false;
};

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// Q~ for a set of clusters: one CTA per cluster up to H2F_HH_MIN_S rows,
// the blocked Householder with cooperative panels above
void complement(const std::vector<ComplementTask>& tasks, Region& scr) {
    const int min_s = env_int("H2F_HH_MIN_S", 224);
    int lim = min_s;
    if (const char* env = std::getenv("H2F_SMALL_N_MAX")) lim = std::min(lim, std::atoi(env));
    std::vector<ComplementTask> small, big;
    for (auto& t : tasks) {
        if (t.s > lim && t.kt > 0) big.push_back(t);  // plan-only tasks (Q == null) shape the waves
        else if (t.Q) small.push_back(t);
    }
    if (!small.empty()) launch_complement(upload(small), int32_t(small.size()), ctx().stream);
    if (!big.empty()) complement_blocked(big, scr);
}

class Factorizer {
  public:
    Factorizer(H2Mat& m, Factorization& f) : M(m), F(f) {}
    void run(double norm_estimate, const double* v0);
    void shard(const h2f_comm* c);

  private:
    H2Mat& M;
    Factorization& F;
    // ---- subtree sharding (h2f_factorize_sharded).  world
    // == 1: every predicate below is true and no collective is called.
    const h2f_comm* comm = nullptr;
    int rank = 0, world = 1;
    std::vector<int> owner;  // node -> rank
    bool sharded() const { return world > 1; }
    bool mine(int c) const { return world == 1 || owner[c] == rank; }
    // a block (a, b) lives on the owners of a and of b
    bool holds(Key k) const { return world == 1 || owner[key_a(k)] == rank || owner[key_b(k)] == rank; }
    // ranks other than c's owner that hold a block touching c (they need
    // c's Q~ and eliminator panels)
    std::vector<int> dests(const Lvl& L, int c) const;
    void coll_check(int rc, const char* what);
    void allreduce_max(double* buf, int64_t n);
    // one all-to-all of per-cluster device payloads: rows of `bytes` from
    // src[i] (owned here) to each rank of dests; returns the receive buffer
    // and, per payload received here, its address (recv_at[i], else null)
    double* exchange(const std::vector<int>& cl, const std::vector<std::vector<int>>& dst,
                     const std::vector<int64_t>& ndoubles, const std::vector<std::vector<std::pair<const double*, int64_t>>>& parts,
                     Region& scr, std::vector<double*>& recv_at);
    void gather_factors();
    void stats_tiles(const GemmBuild& g);
    double eps_fill = 0, drop = 0;
    PhaseClock clock;
    Region scratch[2] = {Region(size_t(64) << 20), Region(size_t(64) << 20)};
    int batch_counter = 0;
    std::vector<size_t> level_marks;
    std::vector<int> mark_node;  // node-indexed batch membership stamp
    std::vector<int> node_bi;    // node -> position in the current batch (valid where stamped)
    std::vector<int64_t> made_mark;  // node -> batch in which a fill key (node, .) was created
    int stamp = 0;
    bool level_prof = false;
    FILE* aug_log = nullptr;  // H2F_AUG_LOG=path: per-cluster augmentation shapes (development aid)
    double level_prev[K_COUNT] = {};
    std::chrono::steady_clock::time_point level_t0;
    // host wall time per section of process_batch (H2F_LEVEL_PROF); the two
    // sync entries are the host blocked on the device
    enum { HT_PICK, HT_AUG, HT_SYNC1, HT_AUG2, HT_PROJ, HT_ELIM, HT_S1, HT_S2A, HT_S2, HT_S3, HT_SCHUR, HT_SYNC2, HT_CREATE, HT_TRANS, HT_N };
    int64_t n_upd = 0, n_cand = 0, n_batches_lvl = 0;
    double ht[HT_N] = {};
    std::chrono::steady_clock::time_point ht_last = std::chrono::steady_clock::now();
    void tick(int i) {
        if (!level_prof) return;
        const auto now = std::chrono::steady_clock::now();
        ht[i] += std::chrono::duration<double>(now - ht_last).count();
        ht_last = now;
    }
    void dump_level_profile(int level);

    std::unique_ptr<Lvl> leaf_level(int level);
    void attach_couplings(Lvl& L);
    void level_complements(Lvl& L);
    void process_batch(Lvl& L, const std::vector<int>& batch);
    std::unique_ptr<Lvl> transition(Lvl& L);
    void finish_top(Lvl& L);
    void dense_only_top();
    void top_factor(double* A, int64_t n);
    std::vector<std::pair<int, int>> dense_pairs(int level) const;
};


std::vector<std::pair<int, int>> Factorizer::dense_pairs(int level) const {
    std::vector<std::pair<int, int>> out(M.inner[level]);
    out.insert(out.end(), M.dense[level].begin(), M.dense[level].end());
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    return out;
}

std::unique_ptr<Lvl> Factorizer::leaf_level(int level) {
    // factorization.py:288-327 (leaf: copies of the dense blocks)
    auto L = std::make_unique<Lvl>();
    L->level = level;
    L->init_common(M.levels[level]);
    const size_t n = L->clusters.size();
    L->offset.resize(n);
    L->size.resize(n);
    for (size_t i = 0; i < n; ++i) {
        const int c = L->clusters[i];
        L->offset[i] = M.begin[c];
        L->size[i] = M.rows(c);
        if (M.top >= 0 && M.leaf_basis_off[c] >= 0) {
            L->basis[i] = View{const_cast<double*>(M.leaf_basis(c)), M.rank[c], int(L->size[i]), int(M.rank[c])};
        } else {
            L->basis[i] = View{nullptr, 0, int(L->size[i]), 0};
        }
        L->k[i] = L->basis[i].cols;
    }
    CopyBuild cp;
    for (int l = 0; l <= M.depth; ++l)
        for (auto& pr : M.dense[l]) {
            if (M.level[pr.first] != level || M.level[pr.second] != level)
                throw Error(H2F_E_INTERNAL, "assertion: dense leaf block away from the leaf level");
            const int rs = int(M.rows(pr.first)), cs = int(M.rows(pr.second));
            if (!holds(mkkey(pr.first, pr.second))) {  // another rank's block: shape only
                L->D[mkkey(pr.first, pr.second)] = View{nullptr, cs, rs, cs};
                continue;
            }
            double* dst = L->mem.alloc_n<double>(int64_t(rs) * cs);
            cp.add(dst, cs, rs, cs, M.vals + M.dense_off.at(mkkey(pr.first, pr.second)), cs, 0, COPY_SET);
            L->D[mkkey(pr.first, pr.second)] = View{dst, cs, rs, cs};
        }
    cp.launch();
    L->build_touch();
    return L;
}

void Factorizer::attach_couplings(Lvl& L) {
    for (auto& pr : M.adm[L.level]) {
        const Key key = mkkey(pr.first, pr.second);
        CouplingW w;
        w.p = M.coupling(key);
        w.rows = int(M.rank[pr.first]);
        w.cols = int(M.rank[pr.second]);
        w.ld = w.cols;
        L.S[key] = w;
    }
    if (L.level > M.top)
        for (size_t i = 0; i < L.clusters.size(); ++i) {
            const int c = L.clusters[i];
            const int p = int(M.parent[c]);
            TransferW t;
            t.has = M.transfer_off[c] >= 0;
            if (t.has) {
                t.p = M.transfer(c);
                t.rows = int(M.rank[c]);
                t.cols = int(M.rank[p]);
                t.ld = t.cols;
            }
            L.T[i] = t;
        }
}

// [V_perp | V] (complete Householder QR of the basis V, factorization.py:88-99
// applied to V alone) for every cluster of the level at once: V is fixed for
// the whole level (the transition built it), so the complements leave the
// per-batch critical path and run as one wide launch instead of one small
// launch per batch.
void Factorizer::level_complements(Lvl& L) {
    CopyBuild gather;
    std::vector<ComplementTask> tasks;
    double cf = 0, cb = 0;
    for (size_t ci = 0; ci < L.clusters.size(); ++ci) {
        const int s = int(L.size[ci]);
        const View& V = L.basis[ci];
        const int k = V.cols;
        if (!mine(L.clusters[ci])) {  // shapes the blocked waves only (bit-identical plans on every rank)
            tasks.push_back(ComplementTask{nullptr, nullptr, nullptr, nullptr, s, k});
            continue;
        }
        double* bt = L.mem.alloc_n<double>(int64_t(std::max(k, 1)) * s);
        L.qv[ci] = L.mem.alloc_n<double>(int64_t(s) * s);
        gather.add(bt, s, k, s, V.p, V.ld, 1, COPY_SET);
        tasks.push_back(ComplementTask{bt, L.mem.alloc_n<double>(int64_t(s) * s), L.qv[ci],
                                       L.mem.alloc_n<double>(int64_t(16) * s), s, k});
        cf += 4.0 * double(s) * s * s;
        cb += 16.0 * double(s) * s;
    }
    gather.launch();
    ProfScope ps(K_COMPLEMENT_V, cf, cb);
    complement(tasks, L.mem);
}

void Factorizer::process_batch(Lvl& L, const std::vector<int>& batch) {
    Context& X = ctx();
    cudaStream_t st = X.stream;
    tick(HT_PICK);
    Region& scr = scratch[batch_counter++ & 1];
    scr.reset();
    const int nb = int(batch.size());
    ++stamp;
    for (int bi = 0; bi < nb; ++bi) {
        mark_node[batch[bi]] = stamp;
        node_bi[batch[bi]] = bi;
    }
    auto in_batch = [&](int c) { return mark_node[c] == stamp; };
    if (sharded()) {
        ShardStats& ss = shard_stats();
        ss.batches += 1;
        ss.total += nb;
        for (int c : batch) ss.local += mine(c);
    }

    // ------------------------------------------------------------- augment
    // factorization.py:62-99, 377-407.  The fill row is projected onto the
    // orthogonal complement of V first: Z = V_perp^T F has the singular values
    // of (I - V V^T) F, so the QR/SVD work on (s-k) instead of s rows.
    clock.mark(PH_AUGMENT);
    std::vector<double*> Q(nb);
    // kept counts [0, nb) and degenerate-sigma flags [nb, 2 nb)
    int* kept_d = scr.alloc_n<int>(2 * nb);
    struct Aug {
        int s, k, n, wf, m;
        bool skip;
        View V;
        double *BT, *QV, *U;
    };
    std::vector<Aug> aug(nb);
    {
        CopyBuild gather;
        GemmBuild gz;
        std::vector<QrTask> qr_small, qr_big, qr_seg;
        // block column pivoting of the blocked QR where the multi-CTA Jacobi
        // follows (fewer sweeps on a graded R): per qr_big task
        // its permutation, and the un-permutation of the Jacobi's vectors
        static const bool qr_pivot = env_int("H2F_QR_PIVOT", 1) != 0;

        std::vector<int32_t*> qr_big_perm;
        std::vector<UnpermTask> unperm;
        int max_unperm = 0;
        std::vector<SvdTask> svd_small, svd_big;
        int max_n_small = 1;
        // the Jacobi writes every singular vector (sorted); under a structure
        // replay the kept count then comes from the replayed run
        const double svd_thresh = drop;
        // H2F_SMALL_N_MAX (tests) lowers the shared-memory QR/SVD cut-off so
        // the large-n (blocked QR, multi-CTA Jacobi) path runs on small inputs
        int small_n_max = SMEM_DENSE_MAX_N;
        if (const char* env = std::getenv("H2F_SMALL_N_MAX"))
            small_n_max = std::min(SMEM_DENSE_MAX_N, std::atoi(env));
        // the shared-memory TSQR serves n <= hh_min_n; above, the blocked
        // Householder with cooperative panels (dense.cpp)
        const int hh_min_n = std::min(small_n_max, env_int("H2F_HH_MIN_N", 32));
        // one-CTA shared-memory Jacobi up to this n; above, the block-cyclic
        // multi-CTA Jacobi (n/16 CTAs per cluster) finishes a batch sooner
        const int svd_smem_max = std::min(small_n_max, env_int("H2F_SVD_SMEM_MAX", 64));
        // pivot where the Jacobi is large enough for its sweeps to matter
        // (default: every blocked-QR task, n > hh_min_n; measured 0.3 s better
        // on config 2 than the multi-CTA Jacobi only)
        const int qr_pivot_min_n = env_int("H2F_QR_PIVOT_MIN_N", hh_min_n);
        H2F_CUDA(cudaMemsetAsync(kept_d, 0, sizeof(int) * 2 * nb, st));
        for (int bi = 0; bi < nb; ++bi) {
            const int c = batch[bi], ci = L.at(c);
            Aug& A = aug[bi];
            A.s = int(L.size[ci]);
            A.V = L.basis[ci];
            A.k = A.V.cols;
            A.n = A.s - A.k;
            const int s = A.s, k = A.k, n = A.n;
            struct Part { View v; int trans; int w; };
            std::vector<Part> parts;
            A.wf = 0;
            for (auto& kv : L.touch[ci]) {  // sorted key order == sorted partner id
                if (kv.second.dense) continue;
                const View& B = *kv.second.v;
                const bool row = key_a(kv.second.key) == c;
                parts.push_back({B, row ? 0 : 1, row ? B.cols : B.rows});
                A.wf += parts.back().w;
            }
            A.skip = (A.wf == 0 || k == s);
            A.m = std::min(n, A.wf);
            if (!mine(c)) {
                // another rank's cluster: its QR / Jacobi shape the waves
                // (plans identical on every rank), nothing runs here
                Q[bi] = nullptr;
                if (A.skip) continue;
                if (n > hh_min_n) {
                    qr_big.push_back(QrTask{nullptr, nullptr, A.wf, n, A.wf, 0, A.wf, 0});
                    qr_big_perm.push_back(nullptr);
                }
                if (n <= svd_smem_max) max_n_small = std::max(max_n_small, n);
                else svd_big.push_back(SvdTask{nullptr, nullptr, A.m, n, nullptr, nb});
                continue;
            }
            Q[bi] = F.store.alloc_n<double>(int64_t(s) * s);
            A.QV = L.qv[ci];  // [V_perp | V], level_complements
            if (A.skip) {
                gather.add(Q[bi], s, s, s, A.QV, s, 0, COPY_SET);
                continue;
            }
            // BT rows 0..k-1 = V^T (rows k.. receive vbar^T below)
            A.BT = scr.alloc_n<double>(int64_t(s) * s);
            gather.add(A.BT, s, k, s, A.V.p, A.V.ld, 1, COPY_SET);
            const int wf = A.wf;
            double* Fb = scr.alloc_n<double>(int64_t(s) * wf);
            int off = 0;
            for (auto& p : parts) {
                gather.add(Fb + off, wf, s, p.w, p.v.p, p.v.ld, p.trans, COPY_SET);
                off += p.w;
            }
            double* Z = scr.alloc_n<double>(int64_t(n) * wf);
            gz.add1(Z, wf, n, wf, GEMM_STORE, contrib(A.QV, s, 1, Fb, wf, 0, s));
            double* R = scr.alloc_n<double>(int64_t(n) * n);
            A.U = scr.alloc_n<double>(int64_t(n) * n);
            const int m = std::min(n, wf);
            A.m = m;
            SvdTask sv{R, A.U, m, n, kept_d + bi, nb};
            if (n > hh_min_n) {
                qr_big.push_back(QrTask{Z, R, wf, n, wf, 0, wf, 0});
                int32_t* pv = nullptr;
                if (qr_pivot && n > qr_pivot_min_n) {
                    pv = scr.alloc_n<int32_t>(n);
                    unperm.push_back(UnpermTask{A.U, scr.alloc_n<double>(int64_t(m) * n), pv, m, n});
                    max_unperm = std::max(max_unperm, m * n);
                }
                qr_big_perm.push_back(pv);
            } else {
                // two-level TSQR: segments of <= seg columns fold into
                // their own R (written transposed side by side), then one
                // CTA folds the stacked R's
                const int seg = std::max(256, 4 * n);
                const int nseg = int(cdiv(wf, seg));
                if (nseg > 1) {
                    double* ST = scr.alloc_n<double>(int64_t(n) * nseg * n);
                    for (int sg = 0; sg < nseg; ++sg)
                        qr_seg.push_back(QrTask{Z, ST + int64_t(sg) * n, wf, n, wf, sg * seg,
                                                std::min(wf, (sg + 1) * seg), int64_t(nseg) * n});
                    qr_small.push_back(QrTask{ST, R, int64_t(nseg) * n, n, nseg * n, 0, nseg * n, 0});
                } else {
                    qr_small.push_back(QrTask{Z, R, wf, n, wf, 0, wf, 0});
                }
            }
            if (n <= svd_smem_max) {
                svd_small.push_back(sv);
                max_n_small = std::max(max_n_small, n);
            } else {
                svd_big.push_back(sv);
            }
        }
        gather.launch();
        gz.launch(K_GEMM_AUG);
        auto qr_work = [](const std::vector<QrTask>& v, double& f, double& b) {
            for (auto& t : v) {
                if (!t.Y) continue;
                const double n = t.s, w = t.wf;
                f += 2.0 * w * n * n - (w >= n ? 2.0 / 3.0 * n * n * n : 0.0);
                b += 8.0 * n * w + 8.0 * n * n;
            }
        };
        auto svd_work = [](const std::vector<SvdTask>& v, double& f, double& b) {
            for (auto& t : v) {
                if (!t.R) continue;
                f += 22.0 * double(t.m) * t.m * t.n;  // c_svd = 22 convention
                b += 16.0 * double(t.m) * t.n;
            }
        };
        if (!qr_small.empty()) {
            double f = 0, b = 0;
            qr_work(qr_small, f, b);
            ProfScope ps(K_QR, f, b);
            if (!qr_seg.empty()) launch_qr_r_smem(upload(qr_seg), int32_t(qr_seg.size()), max_n_small, st);
            launch_qr_r_smem(upload(qr_small), int32_t(qr_small.size()), max_n_small, st);
        }
        if (!qr_big.empty()) {
            double f = 0, b = 0;
            qr_work(qr_big, f, b);
            ProfScope ps(K_QR_BIG, f, b);
            qr_r_blocked(qr_big, scr, &qr_big_perm);
        }
        if (!svd_small.empty()) {
            double f = 0, b = 0;
            svd_work(svd_small, f, b);
            ProfScope ps(K_JACOBI, f, b);
            launch_jacobi_smem(upload(svd_small), int32_t(svd_small.size()), max_n_small, svd_thresh, st);
        }
        if (!svd_big.empty()) {
            double f = 0, b = 0;
            svd_work(svd_big, f, b);
            ProfScope ps(K_JACOBI_BIG, f, b);
            jacobi_multi_cta(svd_big, svd_thresh, scr);
        }
        // the Jacobi worked on R of the column-pivoted Z^T: its vectors are
        // in pivoted coordinates, u[perm[i]] = w[i]
        if (!unperm.empty()) launch_unpermute_rows(upload(unperm), int32_t(unperm.size()), max_unperm, st);
    }
    int* kept_h = static_cast<int*>(X.pinned_buf(sizeof(int) * 2 * nb));
    H2F_CUDA(cudaMemcpyAsync(kept_h, kept_d, sizeof(int) * 2 * nb, cudaMemcpyDeviceToHost, st));
    tick(HT_AUG);
    X.sync();
    tick(HT_SYNC1);
    std::vector<int> kept(kept_h, kept_h + nb);
    std::vector<int> degenerate(kept_h + nb, kept_h + 2 * nb);
    if (sharded()) {  // every rank's scheduler needs every cluster's kept count
        std::vector<double> kb(kept_h, kept_h + 2 * nb);
        allreduce_max(kb.data(), 2 * nb);
        for (int bi = 0; bi < nb; ++bi) {
            kept[bi] = int(kb[bi]);
            degenerate[bi] = int(kb[nb + bi]);
        }
    }
    if (replay().active) {
        Replay& R = replay();
        for (int bi = 0; bi < nb; ++bi) {
            if (aug[bi].skip) continue;
            auto it = R.kept.find((int64_t(L.level) << 32) | uint32_t(batch[bi]));
            if (it == R.kept.end())
                throw Error(H2F_E_ARG, "replay: no kept count for cluster " + std::to_string(batch[bi]) +
                                           " at level " + std::to_string(L.level));
            if (it->second > std::min(aug[bi].n, aug[bi].wf))
                throw Error(H2F_E_ARG, "replay: kept count exceeds the fill rank bound");
            ++R.kept_forced;
            R.kept_changed += kept[bi] != it->second;
            kept[bi] = it->second;
        }
    }
    if (aug_log) {
        for (int bi = 0; bi < nb; ++bi)
            std::fprintf(aug_log, "%d %d %d %d %d %d %d %d\n", L.level, batch_counter, nb, aug[bi].s, aug[bi].k,
                         aug[bi].wf, kept[bi], aug[bi].skip ? 1 : 0);
    }
    {
        // b_aug = [V, V_perp U_kept] re-orthogonalised, then Q~ = [complement | b_aug].
        // When the Jacobi produced a complete orthonormal U (m == n, no zero
        // sigma), the complement is V_perp U_rest: orthogonal to V (V_perp is)
        // and to vbar (U_rest is orthogonal to U_kept) -- an orthonormal
        // completion like the reference's Householder one (factorization.py:88-99;
        // the leading r columns are not unique), as one GEMM
        // instead of a second complete QR.  Otherwise: Householder complement.
        CopyBuild keep, place;
        GemmBuild gv;
        std::vector<ReorthTask> ro;
        std::vector<ComplementTask> cmp;
        const bool fast_ok = env_int("H2F_COMPLEMENT_QR", 0) == 0;
        for (int bi = 0; bi < nb; ++bi) {
            Aug& A = aug[bi];
            if (A.skip) continue;
            if (!mine(batch[bi])) {  // plan-only Householder complement (wave shapes)
                if (kept[bi] && !(fast_ok && A.m == A.n && !degenerate[bi]))
                    cmp.push_back(ComplementTask{nullptr, nullptr, nullptr, nullptr, A.s, A.k + kept[bi]});
                continue;
            }
            if (kept[bi] == 0) {
                keep.add(Q[bi], A.s, A.s, A.s, A.QV, A.s, 0, COPY_SET);
                continue;
            }
            const int s = A.s, k = A.k, n = A.n, kp = kept[bi];
            gv.add1(A.BT + int64_t(k) * s, s, kp, s, GEMM_STORE, contrib(A.U, n, 0, A.QV, s, 1, n));
            ro.push_back(ReorthTask{A.V.p, A.BT, scr.alloc_n<double>(int64_t(std::max(k, 1)) * kp), A.V.ld, s, k,
                                    kp, 0});
            if (fast_ok && A.m == n && !degenerate[bi]) {
                const int r = n - kp;
                if (r > 0) gv.add1(Q[bi], s, s, r, GEMM_STORE, contrib(A.QV, s, 0, A.U + int64_t(kp) * n, n, 1, n));
                place.add(Q[bi] + r, s, s, k + kp, A.BT, s, 1, COPY_SET);
            } else {
                cmp.push_back(ComplementTask{A.BT, scr.alloc_n<double>(int64_t(s) * s), Q[bi],
                                             scr.alloc_n<double>(int64_t(16) * s), s, k + kp});
            }
        }
        keep.launch();
        gv.launch(K_GEMM_AUG);
        double rf = 0, cf = 0, cb = 0;
        for (auto& t : ro) rf += 4.0 * double(t.s) * t.k * t.kept;
        for (auto& t : cmp) {
            if (!t.Q) continue;
            cf += 4.0 * double(t.s) * t.s * t.s;
            cb += 16.0 * double(t.s) * t.s;
        }
        {
            ProfScope ps(K_COMPLEMENT, rf + cf, cb);
            if (!ro.empty()) reorth_batched(ro, scr);
            if (!cmp.empty()) complement(cmp, scr);
        }
        place.launch();
    }
    if (env_int("H2F_CHECK_Q", 0)) {
        // development aid: orthogonality of every Q~ of the batch
        X.sync();
        for (int bi = 0; bi < nb; ++bi) {
            if (!mine(batch[bi])) continue;
            const int sz = aug[bi].s;
            std::vector<double> q(size_t(sz) * sz);
            H2F_CUDA(cudaMemcpy(q.data(), Q[bi], q.size() * 8, cudaMemcpyDeviceToHost));
            double worst = 0;
            for (int a = 0; a < sz; ++a)
                for (int b = 0; b < sz; ++b) {
                    double d = 0;
                    for (int i = 0; i < sz; ++i) d += q[size_t(i) * sz + a] * q[size_t(i) * sz + b];
                    worst = std::max(worst, std::fabs(d - (a == b ? 1.0 : 0.0)));
                }
            if (worst > 1e-10 && !aug[bi].skip && std::getenv("H2F_CHECK_Q_DUMP")) {
                const Aug& A = aug[bi];
                std::vector<double> u(size_t(A.n) * A.n), qv(size_t(sz) * sz);
                H2F_CUDA(cudaMemcpy(u.data(), A.U, u.size() * 8, cudaMemcpyDeviceToHost));
                H2F_CUDA(cudaMemcpy(qv.data(), A.QV, qv.size() * 8, cudaMemcpyDeviceToHost));
                FILE* f = std::fopen(std::getenv("H2F_CHECK_Q_DUMP"), "wb");
                std::fwrite(u.data(), 8, u.size(), f);
                std::fwrite(qv.data(), 8, qv.size(), f);
                std::fwrite(q.data(), 8, q.size(), f);
                std::fclose(f);
            }
            if (worst > 1e-10)
                std::fprintf(stderr, "[check_q] level %d cluster %d s %d k %d n %d m %d wf %d kept %d deg %d skip %d: %.3e\n",
                             L.level, batch[bi], sz, aug[bi].k, aug[bi].n, aug[bi].m, aug[bi].wf, kept[bi],
                             degenerate[bi], int(aug[bi].skip), worst);
        }
    }
    for (int bi = 0; bi < nb; ++bi) {
        const int c = batch[bi], ci = L.at(c);
        const int kt = L.k[ci] + kept[bi];
        if (kt > L.size[ci]) throw Error(H2F_E_INTERNAL, "assertion: augmented basis wider than the cluster");
        L.red[ci] = int(L.size[ci]) - kt;
        L.k[ci] = kt;
        // zero padding of couplings / transfer is logical: S and T keep their
        // stored extent and every consumer treats the added rows as zeros
    }
    if (sharded()) {
        // Q~ of every eliminated cluster to the ranks holding one of its
        // blocks (they project their copies, factorization.py:410-430)
        std::vector<std::vector<int>> dst(nb);
        std::vector<int64_t> nd(nb);
        std::vector<std::vector<std::pair<const double*, int64_t>>> parts(nb);
        for (int bi = 0; bi < nb; ++bi) {
            dst[bi] = dests(L, batch[bi]);
            nd[bi] = int64_t(aug[bi].s) * aug[bi].s;
            if (mine(batch[bi])) parts[bi] = {{Q[bi], nd[bi]}};
        }
        std::vector<double*> at;
        exchange(batch, dst, nd, parts, scr, at);
        for (int bi = 0; bi < nb; ++bi)
            if (!mine(batch[bi])) Q[bi] = at[bi];
    }

    tick(HT_AUG2);
    // ------------------------------------------------------------- project
    clock.mark(PH_PROJECT);
    {
        std::vector<std::pair<bool, Key>> items;  // (is_fill, key), dense first like the reference
        for (int c : batch) {
            items.push_back({false, mkkey(c, c)});
            for (auto& kv : L.touch[L.at(c)]) items.push_back({!kv.second.dense, kv.second.key});
        }
        std::sort(items.begin(), items.end());
        items.erase(std::unique(items.begin(), items.end()), items.end());
        GemmBuild p1, p2;
        for (auto& it : items) {
            if (!holds(it.second)) continue;  // another rank's block: shape unchanged
            View& B = L.block(it.second, !it.first);
            const int a = key_a(it.second), b = key_b(it.second);
            const bool ra = in_batch(a), rb = in_batch(b);
            double* out = L.mem.alloc_n<double>(int64_t(B.rows) * B.cols);
            if (ra && rb) {
                double* tmp = scr.alloc_n<double>(int64_t(B.rows) * B.cols);
                const int sa = B.rows, sb = B.cols;
                double* qa = Q[node_bi[a]];
                double* qb = Q[node_bi[b]];
                p1.add1(tmp, B.cols, B.rows, B.cols, GEMM_STORE, contrib(qa, sa, 1, B.p, B.ld, 0, sa));
                p2.add1(out, B.cols, B.rows, B.cols, GEMM_STORE, contrib(tmp, B.cols, 0, qb, sb, 0, sb));
            } else if (ra) {
                const int sa = B.rows;
                double* qa = Q[node_bi[a]];
                p1.add1(out, B.cols, B.rows, B.cols, GEMM_STORE, contrib(qa, sa, 1, B.p, B.ld, 0, sa));
            } else if (rb) {
                const int sb = B.cols;
                double* qb = Q[node_bi[b]];
                p1.add1(out, B.cols, B.rows, B.cols, GEMM_STORE, contrib(B.p, B.ld, 0, qb, sb, 0, sb));
            } else {
                throw Error(H2F_E_INTERNAL, "assertion: projected block touches no batch member");
            }
            B = View{out, B.cols, B.rows, B.cols};
        }
        p1.launch(K_GEMM_PROJECT);
        p2.launch(K_GEMM_PROJECT);
    }

    tick(HT_PROJ);
    // ------------------------------------------------------------- eliminate
    clock.mark(PH_PARTIAL_LU);
    struct Elim {
        int c, ci, r, kt, np;
        std::vector<int> ids, widths;
        std::vector<int64_t> offs;
        std::vector<Entry> ents;
        double* G;
        double* MW;
        int64_t W;
    };
    std::vector<Elim> el;
    int* status_d = scr.alloc_n<int>(nb);
    {
        CopyBuild panels, lu_copy;
        std::vector<LuTask> lus;
        struct BigLu {
            double* lu;
            int32_t* piv;
            int r;
            int* status;
        };
        std::vector<BigLu> lu_big;
        std::vector<TrsmTask> trs, trs32, trs16;
        int max_r_dmma[2] = {1, 1};
        const int lu_blocked_min = env_int("H2F_LU_BLOCKED_MIN", 192);
        const int trsm_dmma_min = env_int("H2F_TRSM_DMMA_MIN", 48);
        H2F_CUDA(cudaMemsetAsync(status_d, 0, sizeof(int) * nb, st));
        for (int bi = 0; bi < nb; ++bi) {
            const int c = batch[bi], ci = L.at(c);
            const int s = int(L.size[ci]), r = L.red[ci], kt = s - r;
            ClusterFactor& cf = L.factors[ci];
            cf.cluster = c;
            cf.s = s;
            cf.r = r;
            cf.offset = L.offset[ci];
            cf.q = mine(c) ? Q[bi] : nullptr;  // others' factors arrive in gather_factors
            if (r == 0) continue;
            Elim e;
            e.c = c;
            e.ci = ci;
            e.r = r;
            e.kt = kt;
            e.ids.push_back(c);
            e.widths.push_back(kt);
            for (auto& kv : L.touch[ci]) {
                e.ids.push_back(kv.first);
                e.ents.push_back(kv.second);
                const View& B = *kv.second.v;
                e.widths.push_back(key_a(kv.second.key) == c ? B.cols : B.rows);
            }
            e.np = int(e.ids.size());
            e.offs.assign(e.np + 1, 0);
            for (int i = 0; i < e.np; ++i) e.offs[i + 1] = e.offs[i] + e.widths[i];
            e.W = e.offs[e.np];
            const int nc = r >= trsm_dmma_min ? trsm_dmma_cols(r) : 0;
            if (nc) max_r_dmma[nc == 32 ? 0 : 1] = std::max(max_r_dmma[nc == 32 ? 0 : 1], r);
            if (!mine(c)) {
                // another rank eliminates c; its panels arrive below if a
                // block held here takes one of its Schur updates
                e.G = e.MW = nullptr;
                cf.edges.push_back({c, EDGE_SELF, nullptr, e.W, kt});
                for (int i = 1; i < e.np; ++i) {
                    const int o = e.ids[i];
                    cf.edges.push_back({o, L.done[L.at(o)] ? EDGE_SKEL : EDGE_FULL, nullptr, e.W, e.widths[i]});
                }
                el.push_back(std::move(e));
                continue;
            }
            e.G = scr.alloc_n<double>(int64_t(r) * e.W);
            e.MW = F.store.alloc_n<double>(int64_t(r) * e.W);
            cf.lu = F.store.alloc_n<double>(int64_t(r) * r);
            cf.piv = F.store.alloc_n<int32_t>(r);
            const View& Dcc = L.dcc(ci);
            // panel 0: d_cc[:r, r:]
            panels.add(e.G, e.W, r, kt, Dcc.p + r, Dcc.ld, 0, COPY_SET);
            for (int i = 1; i < e.np; ++i) {
                const Entry& en = e.ents[i - 1];
                const View& B = *en.v;
                if (key_a(en.key) == c)
                    panels.add(e.G + e.offs[i], e.W, r, B.cols, B.p, B.ld, 0, COPY_SET);
                else
                    panels.add(e.G + e.offs[i], e.W, r, B.rows, B.p, B.ld, 1, COPY_SET);
            }
            if (r > lu_blocked_min) {
                // large redundant blocks: cooperative-panel LU with DMMA updates
                lu_copy.add(cf.lu, r, r, r, Dcc.p, Dcc.ld, 0, COPY_SET);
                lu_big.push_back({cf.lu, cf.piv, r, status_d + bi});
            } else {
                LuTask lt{};
                lt.D = Dcc.p;
                lt.ldd = Dcc.ld;
                lt.LU = cf.lu;
                lt.piv = cf.piv;
                lt.r = r;
                lt.cluster = c;
                lt.status = status_d + bi;
                lus.push_back(lt);
            }
            for (int64_t c0 = 0; c0 < e.W; c0 += (nc ? nc : 128)) {
                TrsmTask tt{};
                tt.LU = cf.lu;
                tt.piv = cf.piv;
                tt.G = e.G;
                tt.MW = e.MW;
                tt.ldg = e.W;
                tt.ldw = e.W;
                tt.r = r;
                tt.W = int(e.W);
                tt.col0 = int(c0);
                tt.mode = TRSM_ELIMINATOR;
                (nc == 32 ? trs32 : nc == 16 ? trs16 : trs).push_back(tt);
            }
            // edges (factorization.py:453-456)
            cf.edges.push_back({c, EDGE_SELF, e.MW, e.W, kt});
            for (int i = 1; i < e.np; ++i) {
                const int o = e.ids[i];
                cf.edges.push_back({o, L.done[L.at(o)] ? EDGE_SKEL : EDGE_FULL, e.MW + e.offs[i], e.W,
                                    e.widths[i]});
            }
            el.push_back(std::move(e));
        }
        panels.launch();
        double lf = 0, lb = 0, tf = 0, tb = 0;
        for (auto& e : el) {
            if (!e.MW) continue;
            const double r = e.r, W = double(e.W);
            lf += 2.0 / 3.0 * r * r * r;
            lb += 16.0 * r * r;
            tf += 2.0 * r * r * W;
            tb += 16.0 * r * W + 8.0 * r * r;
        }
        {
            ProfScope ps(K_LU, lf, lb);
            if (!lus.empty()) launch_lu(upload(lus), int32_t(lus.size()), st);
            lu_copy.launch();
            for (auto& b : lu_big) {
                double* red = scr.alloc_n<double>(2);
                blocked_lu(b.lu, b.r, b.piv, scr, red, -1, -1, -1);
                launch_lu_status(red, b.r, b.status, st);
            }
        }
        {
            ProfScope ps(K_TRSM, tf, tb);
            if (!trs.empty()) launch_trsm(upload(trs), int32_t(trs.size()), st);
            if (!trs32.empty()) launch_trsm_dmma(upload(trs32), int32_t(trs32.size()), max_r_dmma[0], 32, st);
            if (!trs16.empty()) launch_trsm_dmma(upload(trs16), int32_t(trs16.size()), max_r_dmma[1], 16, st);
        }
    }

    if (sharded()) {
        // eliminator panels [G | -W] of every eliminated cluster to the ranks
        // holding a block it updates (factorization.py:122-126, 476-505)
        std::vector<int> cl(el.size());
        std::vector<std::vector<int>> dst(el.size());
        std::vector<int64_t> nd(el.size());
        std::vector<std::vector<std::pair<const double*, int64_t>>> parts(el.size());
        for (size_t i = 0; i < el.size(); ++i) {
            const Elim& e = el[i];
            cl[i] = e.c;
            dst[i] = dests(L, e.c);
            nd[i] = 2 * int64_t(e.r) * e.W;
            if (e.MW) parts[i] = {{e.G, int64_t(e.r) * e.W}, {e.MW, int64_t(e.r) * e.W}};
        }
        std::vector<double*> at;
        exchange(cl, dst, nd, parts, scr, at);
        for (size_t i = 0; i < el.size(); ++i)
            if (!el[i].MW && at[i]) {
                el[i].G = at[i];
                el[i].MW = at[i] + int64_t(el[i].r) * el[i].W;
            }
    }
    tick(HT_ELIM);
    // Schur updates (factorization.py:122-126) fused with the scatter into the
    // target blocks (factorization.py:476-505).  (target, contribution) pairs
    // are collected in reference order and grouped per target by a stable
    // counting sort; block lookups go through the per-cluster neighbour maps.
    struct THdr {
        double* C;
        int64_t ldc;
        int M, N;
        int64_t count;
    };
    // one (target, contribution) pair in compact form: elimination e, panel
    // pair (i, j); swap = the transposed (0, j) form -W_j^T g_0
    struct TCon {
        int32_t t, e, i, j;  // j < 0: swap, panel -j-1
    };
    struct Cand {
        Key key;
        int creator;
        int M, N;
        GemmContrib g;
        int64_t base, ntiles;
        bool here;  // this rank holds the would-be block and computes its norm
    };
    std::vector<Cand> cands;
    std::vector<size_t> lc;  // candidates whose norm is computed here (sharded: held here)
    int64_t npairs = 0;  // updates of the batch
    for (auto& e : el) npairs += int64_t(e.np) * (e.np + 1) / 2;
    // Target resolution in two passes: (1) per eliminated cluster, in
    // parallel, every update (i, j) is mapped to its target (sub)block -- the
    // neighbour-list walks and block lookups, i.e. the cache misses; (2)
    // slots per target and grouped contributions (bucket-parallel, below).
    struct Upd {
        const View* v;  // nullptr: fill candidate
        double* C;
        int64_t ldc;
        int32_t M, N, i, j;  // j < 0: swap form, panel -j-1
    };
    std::vector<std::vector<Upd>> upd(el.size());
    std::vector<std::vector<int64_t>> boff(el.size());  // per cluster: bucket segment offsets
    const int NBK = npairs > 20000 ? 16 : 1;
    auto bucket_of = [NBK](const View* v) {
        const uint64_t h = (reinterpret_cast<uintptr_t>(v) >> 4) * 0x9E3779B97F4A7C15ull;
        return int((h >> 40) % uint64_t(NBK));
    };
#pragma omp parallel for schedule(dynamic, 1) if (npairs > 20000)
    for (size_t ei = 0; ei < el.size(); ++ei) {
        const Elim& e = el[ei];
        const int c = e.c, r = e.r, kt = e.kt;
        std::vector<Upd>& out = upd[ei];
        out.reserve(size_t(e.np) * (e.np + 1) / 2);
        std::vector<int> opos(e.np);
        for (int i = 1; i < e.np; ++i) opos[i] = L.pos.at(e.ids[i]);
        std::vector<Nbrs::Item>::const_iterator walk{}, walk_end{};
        for (int i = 0; i < e.np; ++i)
            for (int j = i; j < e.np; ++j) {
                if (i == 0 && j == 0) {
                    const View& Dcc = *L.diag[e.ci];
                    if (!Dcc.p) continue;  // held by another rank (sharded)
                    out.push_back({&Dcc, Dcc.p + int64_t(r) * Dcc.ld + r, Dcc.ld, kt, kt, 0, 0});
                } else if (i == 0) {
                    const Entry& en = e.ents[j - 1];
                    const View* B = en.v;
                    if (!B->p) continue;
                    if (key_a(en.key) == c) out.push_back({B, B->p + int64_t(r) * B->ld, B->ld, kt, B->cols, 0, j});
                    else out.push_back({B, B->p + r, B->ld, B->rows, kt, 0, -j - 1});
                } else {
                    const View* B = nullptr;
                    if (i == j) {
                        B = L.diag[opos[i]];
                        walk = L.touch[opos[i]].begin();
                        walk_end = L.touch[opos[i]].end();
                    } else {
                        // ids[] ascending: merge-walk the neighbour list of ids[i]
                        while (walk != walk_end && walk->first < e.ids[j]) ++walk;
                        if (walk != walk_end && walk->first == e.ids[j]) B = walk->second.v;
                    }
                    if (B) {
                        if (B->p) out.push_back({B, B->p, B->ld, B->rows, B->cols, i, j});
                    } else {
                        out.push_back({nullptr, nullptr, 0, e.widths[i], e.widths[j], i, j});
                    }
                }
            }
        // stable counting sort of the targeted updates by bucket; candidates
        // (v == nullptr) go to the extra last segment
        std::vector<int64_t>& off = boff[ei];
        off.assign(NBK + 2, 0);
        for (const Upd& u : out) ++off[1 + (u.v ? bucket_of(u.v) : NBK)];
        for (int b = 0; b < NBK + 1; ++b) off[b + 1] += off[b];
        std::vector<Upd> sorted(out.size());
        std::vector<int64_t> pos(off.begin(), off.end() - 1);
        for (const Upd& u : out) sorted[pos[u.v ? bucket_of(u.v) : NBK]++] = u;
        out.swap(sorted);
    }
    tick(HT_S1);
    // (2) slots and grouped contributions, parallel over hash buckets of the
    // target view: a bucket scans all updates in reference order and keeps
    // its own targets, so the contributions of every target stay in
    // reference order (the only order the numerics depend on); the task order
    // is bucket-major, deterministic for a given arena layout.
    {
        // fill candidates in reference order (cluster, then pair order),
        // built per eliminated cluster in parallel at precomputed offsets
        std::vector<int64_t> cstart(el.size() + 1, 0);
#pragma omp parallel for schedule(dynamic, 4) if (npairs > 20000)
        for (size_t ei = 0; ei < el.size(); ++ei) {
            int64_t n = 0;
            for (int64_t k = boff[ei][NBK]; k < boff[ei][NBK + 1]; ++k) {
                const Upd& u = upd[ei][k];
                n += (u.M > 0 && u.N > 0);
            }
            cstart[ei + 1] = n;
        }
        for (size_t ei = 0; ei < el.size(); ++ei) cstart[ei + 1] += cstart[ei];
        cands.resize(size_t(cstart.back()));
#pragma omp parallel for schedule(dynamic, 4) if (npairs > 20000)
        for (size_t ei = 0; ei < el.size(); ++ei) {
            const Elim& e = el[ei];
            int64_t q = cstart[ei];
            for (int64_t k = boff[ei][NBK]; k < boff[ei][NBK + 1]; ++k) {
                const Upd& u = upd[ei][k];
                if (u.M <= 0 || u.N <= 0) continue;
                Cand& cd = cands[size_t(q++)];
                cd.key = mkkey(e.ids[u.i], e.ids[u.j]);
                cd.creator = e.c;
                cd.M = u.M;
                cd.N = u.N;
                cd.g = contrib(e.G + e.offs[u.i], e.W, 1, e.MW + e.offs[u.j], e.W, 0, e.r);
                cd.base = 0;
                cd.ntiles = GemmBuild::tiles(cd.M, cd.N);
                cd.here = holds(cd.key);
            }
        }
    }
    tick(HT_S2A);
    if (level_prof) {
        n_batches_lvl += 1;
        n_cand += int64_t(cands.size());
        for (auto& u : upd) n_upd += int64_t(u.size());
    }
    struct Bucket {
        std::vector<THdr> th;
        std::vector<TCon> tc;  // t = bucket-local slot
        std::vector<double> ksum;
        std::vector<int64_t> chunks;
        int64_t slot0 = 0, con0 = 0;
        bool bad = false;
    };
    std::vector<Bucket> bk(NBK);
#pragma omp parallel for schedule(static, 1) if (NBK > 1)
    for (int b = 0; b < NBK; ++b) {
        Bucket& B = bk[b];
        // slot per target view, first seen = first slot (reference order): the
        // view carries its slot, stamped with this batch's number
        const int64_t bstamp = batch_counter;
        for (size_t ei = 0; ei < el.size(); ++ei)
            for (int64_t k = boff[ei][b]; k < boff[ei][b + 1]; ++k) {
                const Upd& u = upd[ei][k];
                if (u.M <= 0 || u.N <= 0) continue;
                int t;
                if (u.v->stamp != bstamp) {
                    t = int(B.th.size());
                    u.v->stamp = bstamp;
                    u.v->slot = t;
                    B.th.push_back({u.C, u.ldc, u.M, u.N, 0});
                    B.ksum.push_back(0.0);
                    B.chunks.push_back(0);
                } else {
                    t = u.v->slot;
                    const THdr& th = B.th[t];
                    if (th.C != u.C || th.M != u.M || th.N != u.N || th.ldc != u.ldc) B.bad = true;
                }
                ++B.th[t].count;
                B.ksum[t] += el[ei].r;
                B.chunks[t] += cdiv(el[ei].r, GEMM_BK);
                B.tc.push_back({t, int32_t(ei), u.i, u.j});
            }
    }
    int64_t nslots = 0, ntc = 0;
    for (auto& B : bk) {
        if (B.bad) throw Error(H2F_E_INTERNAL, "assertion: Schur target shape mismatch");
        B.slot0 = nslots;
        B.con0 = ntc;
        nslots += int64_t(B.th.size());
        ntc += int64_t(B.tc.size());
    }
    tick(HT_S2);
    GemmBuild sch;
    // algorithmic bytes: panels G and -W read once per
    // cluster, every existing target element read+written once
    double schur_bytes = 0;
    for (auto& e : el) schur_bytes += 16.0 * e.r * double(e.W);
    {
        // contributions grouped per target (stable counting sort per bucket)
        // written straight into pinned upload memory
        const size_t ncon = size_t(ntc) + cands.size();
        GemmContrib* hc = nullptr;
        sch.ext = X.up.reserve<GemmContrib>(std::max<size_t>(ncon, 1), &hc);
        // contribution offsets per slot: a bucket's slots are contiguous and
        // its contributions start at con0
        std::vector<int64_t> tstart(size_t(nslots) + 1, 0);
        tstart[size_t(nslots)] = ntc;
#pragma omp parallel for schedule(static, 1) if (NBK > 1)
        for (int b = 0; b < NBK; ++b) {
            int64_t run = bk[b].con0;
            for (size_t t = 0; t < bk[b].th.size(); ++t) {
                tstart[size_t(bk[b].slot0) + t] = run;
                run += bk[b].th[t].count;
            }
        }
#pragma omp parallel for schedule(static, 1) if (NBK > 1)
        for (int b = 0; b < NBK; ++b) {
            Bucket& B = bk[b];
            std::vector<int64_t> fill(tstart.begin() + B.slot0, tstart.begin() + B.slot0 + int64_t(B.th.size()));
            for (const TCon& tc : B.tc) {
                const Elim& E = el[tc.e];
                GemmContrib& g = hc[fill[tc.t]++];
                if (tc.j >= 0) g = contrib(E.G + E.offs[tc.i], E.W, 1, E.MW + E.offs[tc.j], E.W, 0, E.r);
                else g = contrib(E.MW + E.offs[-tc.j - 1], E.W, 1, E.G + E.offs[0], E.W, 0, E.r);
            }
        }
        // target tasks (slot order = bucket-major), then the candidates'
        // norm tasks (reference order), built in bulk
        sch.tasks.reserve(size_t(nslots) + cands.size());
        std::vector<int64_t> slot0(NBK + 1, 0);
        for (int b = 0; b < NBK; ++b) slot0[b + 1] = slot0[b] + int64_t(bk[b].th.size());
        for (auto& B : bk)
            for (size_t t = 0; t < B.th.size(); ++t) schur_bytes += 16.0 * B.th[t].M * double(B.th[t].N);
        sch.add_ext_bulk(nslots, GEMM_ADD, [&](int64_t sl) {
            const int b = int(std::upper_bound(slot0.begin(), slot0.end(), sl) - slot0.begin()) - 1;
            const Bucket& B = bk[b];
            const size_t t = size_t(sl - slot0[b]);
            const THdr& h = B.th[t];
            return GemmBuild::BulkItem{h.C, h.ldc, h.M, h.N, tstart[size_t(sl)], h.count, B.ksum[t], B.chunks[t]};
        }, nullptr);
        if (sharded()) {
            for (size_t i = 0; i < cands.size(); ++i)
                if (cands[i].here) lc.push_back(i);
        } else {
            lc.resize(cands.size());
            std::iota(lc.begin(), lc.end(), size_t(0));
        }
        std::vector<int64_t> nbase(lc.size());
        sch.add_ext_bulk(int64_t(lc.size()), GEMM_NORM, [&](int64_t q) {
            const Cand& cd = cands[lc[size_t(q)]];
            hc[ntc + q] = cd.g;
            return GemmBuild::BulkItem{nullptr, 0, cd.M, cd.N, ntc + q, 1, double(cd.g.K), cdiv(cd.g.K, GEMM_BK)};
        }, nbase.data());
#pragma omp parallel for schedule(static) if (lc.size() > 4096)
        for (size_t q = 0; q < lc.size(); ++q) cands[lc[q]].base = nbase[q];
    }
    tick(HT_S3);
    double* norms_d = sch.norm_tiles ? scr.alloc_n<double>(sch.norm_tiles) : nullptr;
    double* cand_ss_d = lc.empty() ? nullptr : scr.alloc_n<double>(lc.size());
    sch.launch(K_GEMM_SCHUR, norms_d, schur_bytes);
    stats_tiles(sch);
    if (!lc.empty()) {
        // the candidates are the launch's only NORM tasks, their tiles
        // contiguous in candidate order: segment k = [base_k, base_k+1)
        std::vector<int64_t> seg(lc.size() + 1, 0);
#pragma omp parallel for schedule(static) if (lc.size() > 4096)
        for (size_t k = 0; k < lc.size(); ++k) seg[k] = cands[lc[k]].base;
        seg[lc.size()] = sch.norm_tiles;
        if (seg[0] != 0 || cands[lc.back()].base + cands[lc.back()].ntiles != sch.norm_tiles)
            throw Error(H2F_E_INTERNAL, "assertion: norm segments");
        ProfScope ps(K_REDUCE, 0.0, 8.0 * double(sch.norm_tiles));
        launch_sumsq_reduce(norms_d, upload(seg), int32_t(lc.size()), cand_ss_d, st);
    }
    tick(HT_SCHUR);
    // one sync: LU status + candidate norms
    const size_t nbytes_read = sizeof(int) * nb + sizeof(double) * lc.size() + 8;
    char* hbuf = static_cast<char*>(X.pinned_buf(nbytes_read + 64));
    int* status_h = reinterpret_cast<int*>(hbuf);
    double* ss_h = reinterpret_cast<double*>(hbuf + ((sizeof(int) * nb + 15) & ~size_t(15)));
    H2F_CUDA(cudaMemcpyAsync(status_h, status_d, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
    if (!lc.empty())
        H2F_CUDA(cudaMemcpyAsync(ss_h, cand_ss_d, sizeof(double) * lc.size(), cudaMemcpyDeviceToHost, st));
    X.sync();
    tick(HT_SYNC2);
    // candidate norms in reference order; sharded: max-reduced so that every
    // rank takes the same fill decisions (each candidate is computed, with
    // identical bits, by the owners of both of its clusters; -1 elsewhere)
    std::vector<double> cand_ss(cands.size(), -1.0);
    for (size_t k = 0; k < lc.size(); ++k) cand_ss[lc[k]] = ss_h[k];
    if (sharded()) {
        std::vector<double> red(size_t(nb) + cands.size());
        for (int bi = 0; bi < nb; ++bi) red[bi] = status_h[bi];
        std::copy(cand_ss.begin(), cand_ss.end(), red.begin() + nb);
        allreduce_max(red.data(), int64_t(red.size()));
        for (int bi = 0; bi < nb; ++bi) status_h[bi] = int(red[bi]);
        std::copy(red.begin() + nb, red.end(), cand_ss.begin());
    }
    for (int bi = 0; bi < nb; ++bi)
        if (status_h[bi]) {
            Error err(H2F_E_SINGULAR, "cluster " + std::to_string(batch[bi]) + " at level " +
                                          std::to_string(L.level) + ": vanishing pivot in redundant block");
            err.cluster = batch[bi];
            err.level = L.level;
            throw err;
        }
    // sequential fill-creation semantics (factorization.py:461-466, 492-505):
    // the first candidate whose own norm exceeds the drop tolerance creates
    // the block, earlier ones are dropped, later ones are added unconditionally
    {
        GemmBuild create;
        std::unordered_map<Key, int> made;
        std::vector<Key> linked;  // created fill keys, linked into the neighbour lists after the loop
        struct Target {
            double* C;
            int64_t ldc;
            int M, N;
            std::vector<GemmContrib> cs;
        };
        std::vector<Target> news;
        // made_mark[a] == this batch: some key (a, .) was created in it (a
        // cheap filter in front of the hash lookup)
        const int64_t mstamp = batch_counter;
        for (size_t i = 0; i < cands.size(); ++i) {
            const Cand& cd = cands[i];
            if (made_mark[key_a(cd.key)] == mstamp) {
                auto it = made.find(cd.key);
                if (it != made.end()) {
                    if (it->second >= 0) news[it->second].cs.push_back(cd.g);
                    continue;
                }
            }
            if (cand_ss[i] < 0) throw Error(H2F_E_INTERNAL, "assertion: fill candidate norm computed nowhere");
            bool create_it = std::sqrt(cand_ss[i]) > drop;
            if (replay().active) {
                Replay& R = replay();
                auto rt = R.created.find((int64_t(L.level) << 32) | uint32_t(cd.creator));
                const bool want = rt != R.created.end() &&
                                  std::find(rt->second.begin(), rt->second.end(), cd.key) != rt->second.end();
                if (want != create_it) {
                    ++R.fill_changed;
                    // how far this run's own norm is from the drop tolerance
                    const double lr = std::fabs(std::log10(std::max(std::sqrt(cand_ss[i]), 1e-300) / drop));
                    ++R.fill_margin_hist[lr < 0.01 ? 0 : lr < 0.1 ? 1 : lr < 0.5 ? 2 : lr < 1.0 ? 3 : 4];
                }
                create_it = want;
            }
            if (create_it) {
                made_mark[key_a(cd.key)] = mstamp;
                L.fill_created.back().push_back(cd.key);
                if (!cd.here) {  // another rank's block: structure only
                    L.F[cd.key] = View{nullptr, cd.N, cd.M, cd.N};
                    linked.push_back(cd.key);
                    made[cd.key] = -1;
                    continue;
                }
                double* blk = L.mem.alloc_n<double>(int64_t(cd.M) * cd.N);
                L.F[cd.key] = View{blk, cd.N, cd.M, cd.N};
                linked.push_back(cd.key);
                made[cd.key] = int(news.size());
                news.push_back({blk, cd.N, cd.M, cd.N, {cd.g}});
            }
        }
        if (!linked.empty()) {
            // (nothing in the loop reads the neighbour lists, and no created
            // block touches a batch cluster, so linking afterwards is the same)
            std::unordered_map<int, std::vector<Nbrs::Item>> add;
            for (Key k : linked) {
                const Entry e{k, false, &L.F.at(k)};
                add[L.at(key_a(k))].push_back({key_b(k), e});
                add[L.at(key_b(k))].push_back({key_a(k), e});
            }
            for (auto& kv : add) L.touch[kv.first].merge_new(kv.second);
        }
        for (auto& t : news) create.add(t.C, t.ldc, t.M, t.N, GEMM_STORE, t.cs.data(), t.cs.size());
        create.launch(K_GEMM_CREATE);
    }
    // slice to skeletons (views only) and mark done (factorization.py:513-523)
    for (int bi = 0; bi < nb; ++bi) {
        const int c = batch[bi], ci = L.at(c);
        const int r = L.red[ci];
        if (r) {
            View& Dcc = L.dcc(ci);
            if (Dcc.p) Dcc.p += int64_t(r) * Dcc.ld + r;
            Dcc.rows -= r;
            Dcc.cols -= r;
            for (auto& kv : L.touch[ci]) {
                View& B = *kv.second.v;
                if (key_a(kv.second.key) == c) {
                    if (B.p) B.p += int64_t(r) * B.ld;
                    B.rows -= r;
                } else {
                    if (B.p) B.p += r;
                    B.cols -= r;
                }
            }
            L.live[ci] -= r;
        }
        L.done[ci] = 1;
    }
    tick(HT_CREATE);
}

std::unique_ptr<Lvl> Factorizer::transition(Lvl& L) {
    // factorization.py:535-588
    const int nl = L.level - 1;
    auto N = std::make_unique<Lvl>();
    N->level = nl;
    N->init_common(M.levels[nl]);
    const size_t n = N->clusters.size();
    N->offset.resize(n);
    N->size.resize(n);
    CopyBuild zero, set, add;
    int64_t pos = 0;
    auto live_of = [&](int c) { return L.live[L.at(c)]; };
    for (size_t i = 0; i < n; ++i) {
        const int p = N->clusters[i];
        const int a = int(M.left[p]), b = int(M.right[p]);
        const int la = live_of(a), lb = live_of(b);
        N->size[i] = la + lb;
        N->offset[i] = pos;
        pos += N->size[i];
        const int kp = int(M.rank[p]);
        N->k[i] = kp;
        if (!mine(p)) {  // another rank's cluster: shape only
            N->basis[i] = View{nullptr, kp, int(N->size[i]), kp};
            continue;
        }
        double* bas = N->mem.alloc_n<double>(int64_t(N->size[i]) * std::max(kp, 1));
        zero.zero(bas, kp, int(N->size[i]), kp);
        const TransferW& ta = L.T[L.at(a)];
        const TransferW& tb = L.T[L.at(b)];
        if (ta.has) set.add(bas, kp, ta.rows, kp, ta.p, ta.ld, 0, COPY_SET);
        if (tb.has) set.add(bas + int64_t(la) * kp, kp, tb.rows, kp, tb.p, tb.ld, 0, COPY_SET);
        N->basis[i] = View{bas, kp, int(N->size[i]), kp};
        N->k[i] = kp;
    }
    auto nsize = [&](int c) { return int(N->size[N->at(c)]); };
    for (auto& pr : dense_pairs(nl)) {
        const int s = pr.first, t = pr.second;
        const int rs = nsize(s), cs = nsize(t);
        if (!holds(mkkey(s, t))) {
            N->D[mkkey(s, t)] = View{nullptr, cs, rs, cs};
            continue;
        }
        double* blk = N->mem.alloc_n<double>(int64_t(rs) * cs);
        zero.zero(blk, cs, rs, cs);
        N->D[mkkey(s, t)] = View{blk, cs, rs, cs};
        int ro = 0;
        for (int64_t ca : {M.left[s], M.right[s]}) {
            int co = 0;
            for (int64_t cb : {M.left[t], M.right[t]}) {
                const Key key = canon(int(ca), int(cb));
                const int tr = ca > cb ? 1 : 0;
                double* dst = blk + int64_t(ro) * cs + co;
                auto dit = L.D.find(key);
                if (dit != L.D.end()) {
                    const View& V = dit->second;
                    set.add(dst, cs, live_of(int(ca)), live_of(int(cb)), V.p, V.ld, tr, COPY_SET);
                } else {
                    auto sit = L.S.find(key);
                    if (sit == L.S.end()) throw Error(H2F_E_INTERNAL, "assertion: child pair neither dense nor coupled");
                    const CouplingW& S = sit->second;
                    set.add(dst, cs, tr ? S.cols : S.rows, tr ? S.rows : S.cols, S.p, S.ld, tr, COPY_SET);
                    auto fit = L.F.find(key);
                    if (fit != L.F.end())
                        add.add(dst, cs, live_of(int(ca)), live_of(int(cb)), fit->second.p, fit->second.ld, tr,
                                COPY_ADD);
                }
                co += live_of(int(cb));
            }
            ro += live_of(int(ca));
        }
    }
    for (auto& kv : L.F) {
        const int a = key_a(kv.first), b = key_b(kv.first);
        if (M.is_adm(L.level, a, b)) continue;
        const int p = int(M.parent[a]), q = int(M.parent[b]);
        if (!(p < q) || N->D.count(mkkey(p, q)))
            throw Error(H2F_E_INTERNAL, "assertion: fill block sweeps onto a dense parent pair");
        auto it = N->F.find(mkkey(p, q));
        if (it == N->F.end()) {
            const int rs = nsize(p), cs = nsize(q);
            double* blk = holds(mkkey(p, q)) ? N->mem.alloc_n<double>(int64_t(rs) * cs) : nullptr;
            if (blk) zero.zero(blk, cs, rs, cs);
            it = N->F.emplace(mkkey(p, q), View{blk, cs, rs, cs}).first;
        }
        if (!it->second.p) continue;  // held by other ranks
        if (!kv.second.p) throw Error(H2F_E_INTERNAL, "assertion: held parent fill block from a child held elsewhere");
        const int ro = (a == M.left[p]) ? 0 : live_of(int(M.left[p]));
        const int co = (b == M.left[q]) ? 0 : live_of(int(M.left[q]));
        View& dst = it->second;
        add.add(dst.p + int64_t(ro) * dst.ld + co, dst.ld, live_of(a), live_of(b), kv.second.p, kv.second.ld, 0,
                COPY_ADD);
    }
    zero.launch();
    set.launch();
    add.launch();
    N->build_touch();
    return N;
}

void Factorizer::finish_top(Lvl& L) {
    // factorization.py:591-615
    std::unordered_map<int, int64_t> offs;
    int64_t n = 0;
    for (size_t i = 0; i < L.clusters.size(); ++i) {
        offs[L.clusters[i]] = n;
        n += L.live[i];
    }
    for (auto& kv : L.F)
        if (!M.is_adm(L.level, key_a(kv.first), key_b(kv.first)))
            throw Error(H2F_E_INTERNAL, "assertion: fill above the shallowest compressed level");
    F.top_size = n;
    F.top_lu = F.store.alloc_n<double>(n * n);
    F.top_piv = F.store.alloc_n<int32_t>(n);
    CopyBuild zero, set, add;
    double* A = F.top_lu;
    zero.zero(A, n, int(n), int(n));
    auto live_of = [&](int c) { return L.live[L.at(c)]; };
    // sharded: each block is added by the owner of its first cluster (who
    // holds it), the other ranks' entries stay zero, and a sum-reduction
    // assembles the matrix exactly (x + 0 = x)
    for (auto& pr : dense_pairs(L.level)) {
        const int s = pr.first, t = pr.second;
        if (!mine(s)) continue;
        const View& V = L.D.at(mkkey(s, t));
        set.add(A + offs[s] * n + offs[t], n, V.rows, V.cols, V.p, V.ld, 0, COPY_SET);
        if (s != t) set.add(A + offs[t] * n + offs[s], n, V.cols, V.rows, V.p, V.ld, 1, COPY_SET);
    }
    for (auto& pr : M.adm[L.level]) {
        const int s = pr.first, t = pr.second;
        if (!mine(s)) continue;
        const Key key = mkkey(s, t);
        const CouplingW& S = L.S.at(key);
        set.add(A + offs[s] * n + offs[t], n, S.rows, S.cols, S.p, S.ld, 0, COPY_SET);
        if (s != t) set.add(A + offs[t] * n + offs[s], n, S.cols, S.rows, S.p, S.ld, 1, COPY_SET);
        auto fit = L.F.find(key);
        if (fit != L.F.end()) {
            const View& V = fit->second;
            add.add(A + offs[s] * n + offs[t], n, live_of(s), live_of(t), V.p, V.ld, 0, COPY_ADD);
            if (s != t) add.add(A + offs[t] * n + offs[s], n, live_of(t), live_of(s), V.p, V.ld, 1, COPY_ADD);
        }
    }
    zero.launch();
    set.launch();
    add.launch();
    if (sharded()) {
        ctx().sync();
        Timer t;
        coll_check(comm->allreduce_sum_dev(comm->user, A, n * n), "allreduce_sum_dev");
        shard_stats().calls += 1;
        shard_stats().seconds += t.s();
    }
}

void Factorizer::dense_only_top() {
    // factorization.py:274-285
    const int64_t n = M.n;
    F.top_size = n;
    F.top_lu = F.store.alloc_n<double>(n * n);
    F.top_piv = F.store.alloc_n<int32_t>(n);
    CopyBuild zero, set;
    zero.zero(F.top_lu, n, int(n), int(n));
    for (int l = 0; l <= M.depth; ++l)
        for (auto& pr : M.dense[l]) {
            const int s = pr.first, t = pr.second;
            const double* D = M.vals + M.dense_off.at(mkkey(s, t));
            const int rs = int(M.rows(s)), cs = int(M.rows(t));
            set.add(F.top_lu + M.begin[s] * n + M.begin[t], n, rs, cs, D, cs, 0, COPY_SET);
            if (s != t) set.add(F.top_lu + M.begin[t] * n + M.begin[s], n, cs, rs, D, cs, 1, COPY_SET);
        }
    zero.launch();
    set.launch();
}

void Factorizer::top_factor(double* A, int64_t n) {
    // factorization.py:259-263: pivoted LU + vanishing-pivot test
    Context& X = ctx();
    cudaStream_t st = X.stream;
    if (n == 0) return;
    if (const char* path = std::getenv("H2F_DUMP_TOP")) {
        // development aid: the assembled dense top matrix before its LU
        X.sync();
        std::vector<double> h(size_t(n) * n);
        H2F_CUDA(cudaMemcpy(h.data(), A, h.size() * 8, cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen(path, "wb")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    double* red = scratch[0].alloc_n<double>(2);
    blocked_lu(A, n, F.top_piv, scratch[0], red, K_TOP_PANEL, K_TOP_MISC, K_GEMM_TOP);
    double* h = static_cast<double*>(X.pinned_buf(16));
    H2F_CUDA(cudaMemcpyAsync(h, red, 16, cudaMemcpyDeviceToHost, st));
    X.sync();
    if (h[1] <= PIVOT_RTOL * std::max(h[0], 1e-300))
        throw Error(H2F_E_SINGULAR, "singular block at the final dense solve");
}

// H2F_LEVEL_PROF=1 (with the profiler on): per-level kernel seconds and host
// wall time on stderr (development aid)
void Factorizer::dump_level_profile(int level) {
    Profiler& P = ctx().prof;
    P.collect();
    const auto now = std::chrono::steady_clock::now();
    const double wall = std::chrono::duration<double>(now - level_t0).count();
    level_t0 = now;
    std::fprintf(stderr, "[level %d] wall %.4f s:", level, wall);
    double dev = 0;
    for (int k = 0; k < K_COUNT; ++k) {
        const double d = P.totals[k].seconds - level_prev[k];
        level_prev[k] = P.totals[k].seconds;
        dev += d;
        if (d > 1e-4) std::fprintf(stderr, " %s=%.4f", kernel_name(k), d);
    }
    std::fprintf(stderr, " | kernels %.4f\n", dev);
    static const char* names[HT_N] = {"pick", "aug", "sync1", "aug2", "proj", "elim", "s.resolve", "s.cands", "s.slots", "s.fill", "s.launch", "sync2", "create", "trans"};
    std::fprintf(stderr, "[level %d host]", level);
    for (int i = 0; i < HT_N; ++i) {
        std::fprintf(stderr, " %s=%.4f", names[i], ht[i]);
        ht[i] = 0;
    }
    std::fprintf(stderr, " | updates %lld candidates %lld batches %lld\n", (long long)n_upd, (long long)n_cand,
                 (long long)n_batches_lvl);
    n_upd = n_cand = n_batches_lvl = 0;
}


// ---------------------------------------------------------------- sharding

void Factorizer::shard(const h2f_comm* c) {
    comm = c;
    rank = c ? c->rank : 0;
    world = c ? c->world : 1;
    if (world < 1 || rank < 0 || rank >= world) throw Error(H2F_E_ARG, "comm: rank/world out of range");
    if (world > 1 && (!c->allreduce_max || !c->allreduce_sum_dev || !c->alltoallv_dev || !c->broadcast_dev))
        throw Error(H2F_E_ARG, "comm: missing collective callback");
    owner = shard_owners(M, world);
}

std::vector<int> Factorizer::dests(const Lvl& L, int c) const {
    std::vector<int> d;
    const int oc = owner[c];
    for (auto& kv : L.touch[L.at(c)]) {
        const int g = owner[kv.first];
        if (g != oc) d.push_back(g);
    }
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    return d;
}

void Factorizer::coll_check(int rc, const char* what) {
    if (rc != 0) throw Error(H2F_E_INTERNAL, std::string("sharded factorization: collective ") + what +
                                                 " failed with " + std::to_string(rc));
}

void Factorizer::allreduce_max(double* buf, int64_t n) {
    Timer t;
    coll_check(comm->allreduce_max(comm->user, buf, n), "allreduce_max");
    shard_stats().calls += 1;
    shard_stats().seconds += t.s();
}

void Factorizer::stats_tiles(const GemmBuild& g) {
    // Schur target tiles computed here vs the batch schedule's total
    // (identical on every rank: the host resolves all targets)
    shard_stats().tiles_here += double(g.tile_start.back());
}

// Per-cluster payloads (cl[i], payload of nd[i] doubles made of parts[i])
// from their owner to every rank in dst[i], as ONE all-to-all.  The send
// buffer is packed by destination rank then payload order; receivers see
// the payloads of each source rank in payload order, so recv_at[i] is the
// payload's address here (null where this rank is not a destination).
double* Factorizer::exchange(const std::vector<int>& cl, const std::vector<std::vector<int>>& dst,
                             const std::vector<int64_t>& nd,
                             const std::vector<std::vector<std::pair<const double*, int64_t>>>& parts, Region& scr,
                             std::vector<double*>& recv_at) {
    const size_t np = cl.size();
    std::vector<int64_t> sendc(world, 0), recvc(world, 0);
    for (size_t i = 0; i < np; ++i) {
        const int src = owner[cl[i]];
        for (int g : dst[i]) {
            if (src == rank) sendc[g] += nd[i];
            if (g == rank) recvc[src] += nd[i];
        }
    }
    int64_t stot = 0, rtot = 0;
    for (int g = 0; g < world; ++g) {
        stot += sendc[g];
        rtot += recvc[g];
    }
    double* sbuf = scr.alloc_n<double>(std::max<int64_t>(stot, 1));
    double* rbuf = scr.alloc_n<double>(std::max<int64_t>(rtot, 1));
    recv_at.assign(np, nullptr);
    // pack: contiguous ranges copied as rows of PACK_W doubles
    constexpr int PACK_W = 512;
    CopyBuild pack;
    auto copy_range = [&](double* d, const double* sp, int64_t cnt) {
        const int64_t rows = cnt / PACK_W, rest = cnt - rows * PACK_W;
        if (rows) pack.add(d, PACK_W, int(rows), PACK_W, sp, PACK_W, 0, COPY_SET);
        if (rest) pack.add(d + rows * PACK_W, rest, 1, int(rest), sp + rows * PACK_W, rest, 0, COPY_SET);
    };
    int64_t so = 0, ro = 0;
    for (int g = 0; g < world; ++g)
        for (size_t i = 0; i < np; ++i) {
            if (!std::binary_search(dst[i].begin(), dst[i].end(), g)) continue;
            const int src = owner[cl[i]];
            if (src == rank) {
                int64_t o = 0;
                for (auto& pt : parts[i]) {
                    copy_range(sbuf + so + o, pt.first, pt.second);
                    o += pt.second;
                }
                if (o != nd[i]) throw Error(H2F_E_INTERNAL, "assertion: exchange payload size");
                so += nd[i];
            }
        }
    // receive offsets: per source rank, payloads in order
    for (int g = 0; g < world; ++g)
        for (size_t i = 0; i < np; ++i)
            if (owner[cl[i]] == g && std::binary_search(dst[i].begin(), dst[i].end(), rank)) {
                recv_at[i] = rbuf + ro;
                ro += nd[i];
            }
    pack.launch();
    ctx().sync();
    std::vector<int64_t> sb(world), rb(world);
    for (int g = 0; g < world; ++g) {
        sb[g] = sendc[g] * 8;
        rb[g] = recvc[g] * 8;
    }
    Timer t;
    coll_check(comm->alltoallv_dev(comm->user, sbuf, sb.data(), rbuf, rb.data()), "alltoallv_dev");
    ShardStats& st = shard_stats();
    st.calls += 1;
    st.seconds += t.s();
    st.bytes_sent += 8.0 * double(stot);
    return rbuf;
}

// Every rank ends with every cluster's factor (q, lu, piv, eliminator): the
// owner packs its clusters of a record into one staging buffer, broadcasts
// it, and the others keep the broadcast buffer as their storage of those
// clusters (no unpack copy).  Layout per cluster: q (s*s), lu (r*r), the
// r x W eliminator, piv (r int32, padded to whole doubles).
void Factorizer::gather_factors() {
    Region stage(size_t(256) << 20);
    for (auto& rec : F.recs) {
        const size_t nc = rec.factors.size();
        std::vector<int64_t> W(nc, 0), sz(nc, 0);
        for (size_t i = 0; i < nc; ++i) {
            const ClusterFactor& cf = rec.factors[i];
            for (auto& e : cf.edges) W[i] += e.w;
            const int64_t r = cf.r;
            sz[i] = int64_t(cf.s) * cf.s + (r ? r * r + r * W[i] + (r + 1) / 2 : 0);
        }
        for (int g = 0; g < world; ++g) {
            int64_t tot = 0;
            for (size_t i = 0; i < nc; ++i)
                if (owner[rec.factors[i].cluster] == g) tot += sz[i];
            if (!tot) continue;
            stage.reset();
            double* buf = g == rank ? stage.alloc_n<double>(tot) : F.store.alloc_n<double>(tot);
            if (g == rank) {
                CopyBuild pack;
                int64_t o = 0;
                auto put = [&](const double* src, int64_t cnt) {
                    constexpr int PACK_W = 512;
                    const int64_t rows = cnt / PACK_W, rest = cnt - rows * PACK_W;
                    if (rows) pack.add(buf + o, PACK_W, int(rows), PACK_W, src, PACK_W, 0, COPY_SET);
                    if (rest) pack.add(buf + o + rows * PACK_W, rest, 1, int(rest), src + rows * PACK_W, rest, 0, COPY_SET);
                    o += cnt;
                };
                for (size_t i = 0; i < nc; ++i) {
                    const ClusterFactor& cf = rec.factors[i];
                    if (owner[cf.cluster] != g) continue;
                    const int64_t r = cf.r;
                    put(cf.q, int64_t(cf.s) * cf.s);
                    if (r) {
                        put(cf.lu, r * r);
                        put(cf.edges[0].mat, r * W[i]);
                        // int32 pivots read as whole doubles: the arena
                        // rounds every allocation up, so the pad is ours
                        put(reinterpret_cast<const double*>(cf.piv), (r + 1) / 2);
                    }
                }
                pack.launch();
            }
            ctx().sync();
            Timer t;
            coll_check(comm->broadcast_dev(comm->user, buf, tot * 8, g), "broadcast_dev");
            ShardStats& st = shard_stats();
            st.calls += 1;
            st.seconds += t.s();
            st.gather_bytes += 8.0 * double(tot);
            if (g == rank) continue;
            int64_t o = 0;
            for (size_t i = 0; i < nc; ++i) {
                ClusterFactor& cf = rec.factors[i];
                if (owner[cf.cluster] != g) continue;
                const int64_t r = cf.r;
                cf.q = buf + o;
                o += int64_t(cf.s) * cf.s;
                if (r) {
                    cf.lu = buf + o;
                    o += r * r;
                    double* mw = buf + o;
                    int64_t eo = 0;
                    for (auto& e : cf.edges) {
                        e.mat = mw + eo;
                        e.ld = W[i];
                        eo += e.w;
                    }
                    o += r * W[i];
                    cf.piv = reinterpret_cast<int32_t*>(buf + o);
                    o += (r + 1) / 2;
                }
            }
        }
    }
    ctx().sync();
}

void Factorizer::run(double norm_estimate, const double* v0) {
    if (owner.empty()) owner = shard_owners(M, 1);
    if (sharded()) shard_stats() = ShardStats{};
    level_prof = std::getenv("H2F_LEVEL_PROF") != nullptr && ctx().prof.on;
    if (level_prof) {
        ctx().prof.collect();
        for (int k = 0; k < K_COUNT; ++k) level_prev[k] = ctx().prof.totals[k].seconds;
        level_t0 = std::chrono::steady_clock::now();
    }
    mark_node.assign(M.nnodes, 0);
    node_bi.assign(M.nnodes, -1);
    made_mark.assign(M.nnodes, -1);
    if (const char* p = std::getenv("H2F_AUG_LOG")) aug_log = std::fopen(p, "a");
    clock.mark(PH_NORM);
    if (norm_estimate < 0) {
        if (!v0) throw Error(H2F_E_ARG, "norm estimate requested without a start vector");
        norm_estimate = norm2_estimate(M, v0, 30);
    }
    F.norm_estimate = norm_estimate;
    eps_fill = F.eps_lu * norm_estimate;
    F.eps_fill = eps_fill;
    drop = FILL_DROP_FACTOR * eps_fill;
    F.top_level = M.top;
    if (M.top < 0) {
        clock.mark(PH_TOP);
        dense_only_top();
    } else {
        std::unique_ptr<Lvl> L;
        for (int level = M.depth; level >= M.top; --level) {
            level_marks.push_back(clock.size());
            clock.mark(PH_EXTRACT);
            tick(HT_TRANS);
            if (!L) L = leaf_level(level);
            for (size_t i = 0; i < L->clusters.size(); ++i) L->live[i] = int(L->size[i]);
            attach_couplings(*L);
            level_complements(*L);
            L->fill_init.clear();
            for (auto& kv : L->F) L->fill_init.push_back(kv.first);
            clock.mark(PH_COLOR);
            // greedy colouring of the D+F graph in ascending id order
            // (factorization.py:330-337, structure.py:137-167)
            // (the routine h2f_greedy_coloring exports, coloring.h)
            const size_t nc = L->clusters.size();
            std::vector<size_t> order(nc);
            int degree = 0;
            for (size_t i = 0; i < nc; ++i) {
                order[i] = i;  // level clusters are in ascending id order
                degree = std::max(degree, int(L->touch[i].size()));
            }
            std::vector<int> color;
            const int ncolors = greedy_coloring(order, nc, [&](size_t i, auto visit) {
                for (auto& kv : L->touch[i]) visit(size_t(L->at(kv.first)));
            }, color);
            std::vector<std::vector<int>> groups(ncolors);
            for (size_t i = 0; i < nc; ++i) groups[color[i]].push_back(L->clusters[i]);
            for (auto& grp : groups) {
                std::vector<int> remaining = grp;
                while (!remaining.empty()) {
                    // greedy independent set in the live graph (factorization.py:353-362)
                    ++stamp;
                    std::vector<int> batch, rest;
                    for (int c : remaining) {
                        bool free_ = true;
                        for (auto& kv : L->touch[L->at(c)])
                            if (mark_node[kv.first] == stamp) { free_ = false; break; }
                        if (free_) {
                            batch.push_back(c);
                            mark_node[c] = stamp;
                        } else {
                            rest.push_back(c);
                        }
                    }
                    remaining.swap(rest);
                    L->batches.push_back(batch);
                    L->fill_created.emplace_back();
                    process_batch(*L, batch);
                    clock.mark(PH_COLOR);
                }
            }
            // level record
            LevelRecord rec;
            rec.level = level;
            rec.clusters = L->clusters;
            rec.offset = L->offset;
            rec.size = L->size;
            rec.batches = L->batches;
            rec.fill_init = L->fill_init;
            rec.fill_created = L->fill_created;
            rec.csp = sparsity_constant(M, level);
            rec.ncolors = ncolors;
            rec.graph_degree = degree;
            int mr = 0;
            for (size_t i = 0; i < nc; ++i) {
                mr = std::max(mr, L->live[i]);
                rec.pos[L->clusters[i]] = int(i);
                for (int64_t x = L->offset[i] + L->red[i]; x < L->offset[i] + L->size[i]; ++x) rec.up_index.push_back(x);
            }
            rec.max_rank = mr;
            rec.factors = std::move(L->factors);
            clock.mark(PH_TRANSITION);
            if (level > M.top) {
                auto N = transition(*L);
                ctx().sync();  // the old level's storage is released next
                L = std::move(N);
            } else {
                finish_top(*L);
                ctx().sync();
                L.reset();
            }
            F.recs.push_back(std::move(rec));
            tick(HT_TRANS);
            if (level_prof) dump_level_profile(level);
        }
    }
    if (sharded()) gather_factors();
    clock.mark(PH_TOP);
    top_factor(F.top_lu, F.top_size);
    clock.mark(-1);
    ctx().sync();
    clock.accumulate(F.phase);
    if (aug_log) std::fclose(aug_log);
    for (size_t i = 0; i < level_marks.size(); ++i) {
        const size_t j = (i + 1 < level_marks.size()) ? level_marks[i + 1] : clock.size() - 2;
        F.recs[i].time_s = clock.between(level_marks[i], j);
    }
    // nbytes (factorization.py:181-190)
    int64_t nb = F.top_size * F.top_size * 8 + F.top_size * 4;
    for (auto& rec : F.recs) {
        nb += int64_t(rec.up_index.size()) * 8;
        for (auto& cf : rec.factors) {
            nb += int64_t(cf.s) * cf.s * 8;
            if (cf.r) nb += int64_t(cf.r) * cf.r * 8 + int64_t(cf.r) * 4;
            for (auto& e : cf.edges) nb += int64_t(cf.r) * e.w * 8;
        }
    }
    F.nbytes = nb;
}

}  // namespace

Factorization* factorize(H2Mat& m, double eps_lu, double norm_estimate, const double* v0_host,
                         const h2f_comm* comm) {
    auto f = std::make_unique<Factorization>();
    f->mat = &m;
    f->n = m.n;
    f->eps_lu = eps_lu;
    Factorizer fz(m, *f);
    if (comm) fz.shard(comm);
    fz.run(norm_estimate, v0_host);
    return f.release();
}

}  // namespace h2f
