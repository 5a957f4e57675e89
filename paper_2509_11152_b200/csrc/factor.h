// Factor containers (factorization.py:130-193) and the factorization /
// substitution entry points of the runtime.
#pragma once
#include <map>
#include <memory>
#include <vector>

#include "h2mat.h"

namespace h2f {

enum EdgeKind : int32_t { EDGE_SELF = 0, EDGE_FULL = 1, EDGE_SKEL = 2 };

struct EdgeRec {        // (other, kind, mat) of ClusterFactor.edges, mat = r x w view
    int other;
    int kind;
    double* mat;
    int64_t ld;
    int w;
};

struct ClusterFactor {  // factorization.py:130-147
    int cluster = -1;
    int s = 0, r = 0;
    int64_t offset = 0;
    double* q = nullptr;       // s x s
    double* lu = nullptr;      // r x r (row-major)
    int32_t* piv = nullptr;    // r
    std::vector<EdgeRec> edges;
};

struct LevelRecord {    // factorization.py:150-164
    int level = 0;
    std::vector<int> clusters;
    std::vector<int64_t> offset, size;
    std::vector<std::vector<int>> batches;
    std::vector<int64_t> up_index;
    int csp = 0, ncolors = 0, graph_degree = 0, max_rank = 0;
    double time_s = 0.0;
    std::vector<ClusterFactor> factors;        // parallel to clusters
    // fill keys: present when the level started (swept up by the transition,
    // factorization.py:573-588) and created by each batch, in creation order
    // (factorization.py:502-505) -- the F-key set after batch b is the union
    std::vector<Key> fill_init;
    std::vector<std::vector<Key>> fill_created;  // parallel to batches
    std::unordered_map<int, int> pos;          // cluster -> index
    int64_t total() const {
        int64_t t = 0;
        for (auto s : size) t += s;
        return t;
    }
};

enum Phase : int { PH_NORM = 0, PH_EXTRACT, PH_COLOR, PH_AUGMENT, PH_PROJECT, PH_PARTIAL_LU,
                   PH_TRANSITION, PH_TOP, PH_COUNT };

struct SolvePlan;

struct Factorization {  // factorization.py:167-193
    H2Mat* mat = nullptr;
    int64_t n = 0;
    int top_level = -1;
    std::vector<LevelRecord> recs;
    double* top_lu = nullptr;
    int32_t* top_piv = nullptr;
    int64_t top_size = 0;
    double eps_lu = 0, eps_fill = 0, norm_estimate = 0;
    double phase[PH_COUNT] = {0};
    int64_t nbytes = 0;
    Region store{size_t(256) << 20};
    std::map<int, std::shared_ptr<SolvePlan>> plans;  // per nrhs
    Region work{size_t(16) << 20};
    ~Factorization();
};

// Structure replay (parity diagnostics, h2f_debug_replay_set): the threshold
// decisions of another run -- kept count per (level, cluster) and the created
// fill blocks per (level, creating cluster, key) -- replace this run's own,
// so the floating-point path can be compared on an identical structure.
struct Replay {
    std::unordered_map<int64_t, int> kept;            // (level << 32 | cluster) -> kept
    std::unordered_map<int64_t, std::vector<Key>> created;  // (level << 32 | creator) -> keys
    int64_t kept_forced = 0, kept_changed = 0, fill_changed = 0;
    // changed fill decisions by |log10(own norm / drop tolerance)|:
    // < 0.01, < 0.1, < 0.5, < 1, >= 1
    int64_t fill_margin_hist[5] = {0, 0, 0, 0, 0};
    bool active = false;
};
Replay& replay();

// subtree sharding (h2f_factorize_sharded): counters of the last run
struct ShardStats {
    double local = 0, total = 0;   // clusters eliminated here / in all
    double bytes_sent = 0, calls = 0;
    double tiles_here = 0, batches = 0;
    double seconds = 0;            // host wall time inside the collectives
    double gather_bytes = 0;       // factor broadcast at the end
};
ShardStats& shard_stats();
// node -> owner rank for a world-way split into contiguous subtrees of the
// top level (-1 above the top level)
std::vector<int> shard_owners(const H2Mat& m, int world);
std::vector<int> shard_owners_tree(int64_t nnodes, const int64_t* parent, const int64_t* level, int top,
                                   int world);

// throws Error(H2F_E_SINGULAR) with cluster/level set on a vanishing pivot;
// comm (world > 1): the subtree-sharded factorization, same result
Factorization* factorize(H2Mat& m, double eps_lu, double norm_estimate, const double* v0_host,
                         const h2f_comm* comm = nullptr);

void solve_device(Factorization& f, const double* b_dev, double* x_dev, int nrhs);
void refined_solve_device(H2Mat& m, Factorization& f, const double* b_dev, double* x_dev, int steps,
                          int nrhs = 1);

}  // namespace h2f
