// Device-resident H2 operator (the input of the path, h2core.py:97-125) and
// its matvec / power-iteration plan (h2core.py:272-330).
#pragma once
#include <map>
#include <memory>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "kernels.h"
#include "runtime.h"

namespace h2f {

using Key = uint64_t;
inline Key mkkey(int64_t a, int64_t b) { return (uint64_t(uint32_t(a)) << 32) | uint32_t(b); }
inline int key_a(Key k) { return int(k >> 32); }
inline int key_b(Key k) { return int(uint32_t(k)); }
inline Key canon(int a, int b) { return a <= b ? mkkey(a, b) : mkkey(b, a); }

struct GemvLaunch {
    GemvTask* tasks;
    GemvContrib* contribs;
    int32_t ntasks;
    int32_t max_rows = 0;  // largest output segment (shared-memory accumulator size)
    double flops = 0, bytes = 0;
};

struct MatvecPlan {
    int nrhs = 1;
    double* xin = nullptr;
    double* yout = nullptr;
    double* xh = nullptr;
    double* yh = nullptr;
    double* partial = nullptr;   // norm reduction scratch
    double* est = nullptr;       // power-iteration estimates
    std::vector<GemvLaunch> launches;
    Region mem;
    int64_t last_use = 0;
};

struct H2Mat {
    int64_t n = 0;
    int depth = 0, top = -1;
    int64_t nnodes = 0;
    std::vector<int64_t> parent, left, right, level, begin, end, rank;
    std::vector<std::vector<int>> levels;                  // node ids per level, ascending
    std::vector<std::vector<std::pair<int, int>>> adm, inner, dense;  // per level, sorted
    std::vector<std::unordered_set<Key>> adm_set, dense_set;          // dense = inner | leaves
    std::vector<int64_t> leaf_basis_off, transfer_off;     // per node, -1 absent
    std::unordered_map<Key, int64_t> coupling_off, dense_off;
    // offsets in the description's pair order (h2f_matrix_layout)
    std::vector<int64_t> coupling_list, dense_list;
    double* vals = nullptr;                                 // device
    int64_t nvals = 0;
    std::map<int, std::unique_ptr<MatvecPlan>> plans;

    int64_t rows(int c) const { return end[c] - begin[c]; }
    bool is_leaf(int c) const { return left[c] < 0; }
    const double* leaf_basis(int c) const { return vals + leaf_basis_off[c]; }
    const double* transfer(int c) const { return vals + transfer_off[c]; }
    const double* coupling(Key k) const { return vals + coupling_off.at(k); }
    bool is_adm(int lv, int a, int b) const { return adm_set[lv].count(canon(a, b)) != 0; }
    bool is_dense(int lv, int a, int b) const { return dense_set[lv].count(canon(a, b)) != 0; }

    ~H2Mat();
};

H2Mat* h2mat_create(const h2f_matrix_desc* d, const double* host_vals);
// values given as blocks (pointer, count, offset in the value array;
// offsets ascending): packed in pinned chunks overlapped with the upload
H2Mat* h2mat_create_blocks(const h2f_matrix_desc* d, int64_t nblk, const double* const* ptrs, const int64_t* counts,
                           const int64_t* offs);
// takes ownership of dev_vals (an arena allocation of d->nvals doubles)
H2Mat* h2mat_create_device(const h2f_matrix_desc* d, double* dev_vals);
// device construction + recompression from points, tree and partition (build.cpp)
H2Mat* h2mat_build(const h2f_build_desc* d, int64_t* rank_out, double* seconds);
// A + W W^T absorbed into a new operator, then recompressed at eps (build.cpp)
H2Mat* h2mat_absorb_low_rank(const H2Mat& A, const double* w_host, int rw, double eps, int64_t* rank_out,
                             double* seconds);
MatvecPlan& matvec_plan(H2Mat& m, int nrhs);
// y_dev = A x_dev (both n x nrhs row-major device buffers), stream-ordered
void matvec_device(H2Mat& m, const double* x_dev, double* y_dev, int nrhs);
// 30-step power iteration from a normalised host start vector
double norm2_estimate(H2Mat& m, const double* v0_host, int iters);
int sparsity_constant(const H2Mat& m, int level);

}  // namespace h2f
