// C ABI (include/h2f.h).  Never throws across the boundary: every entry point
// converts h2f::Error / std::exception into a status code + h2f_last_error().
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "builders.h"
#include "coloring.h"
#include "dense.h"
#include "factor.h"

using namespace h2f;

struct h2f_matrix_s {
    H2Mat* m;
};
struct h2f_factor_s {
    Factorization* f;
};

namespace {

thread_local std::string g_err;

// One context (arena, upload ring, plan cache, profiler) per process: every
// entry point runs under this lock, so concurrent callers (ctypes releases the
// GIL) serialise instead of racing on the host allocator state -- concurrent
// solves are safe as the reference promises.  Recursive because
// entry points may call each other.  The calling thread is also bound to the
// context's device, whatever cudaSetDevice it did itself.
std::recursive_mutex g_lock;

void bind_device() {
    if (ctx_ready()) H2F_CUDA(cudaSetDevice(ctx().device));
}

// a *_dev pointer must be device memory of the context's device
void check_dev_ptr(const void* p, const char* what) {
    if (!p) throw Error(H2F_E_ARG, std::string(what) + ": null device pointer");
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        throw Error(H2F_E_ARG, std::string(what) + ": not a CUDA pointer");
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
        throw Error(H2F_E_ARG, std::string(what) + ": host pointer passed to a _dev entry point");
    if (a.device != ctx().device)
        throw Error(H2F_E_ARG, std::string(what) + ": pointer on device " + std::to_string(a.device) +
                                   ", library context on device " + std::to_string(ctx().device));
}

template <class Fn> int guard(Fn&& fn) {
    std::lock_guard<std::recursive_mutex> hold(g_lock);
    try {
        bind_device();
        fn();
        return H2F_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return H2F_E_INTERNAL;
    }
}

// device buffer borrowed from the arena for a host-pointer call
struct DevBuf {
    double* p = nullptr;
    explicit DevBuf(size_t n) { p = static_cast<double*>(dalloc(sizeof(double) * std::max<size_t>(n, 1))); }
    ~DevBuf() {
        if (p) dfree(p);
    }
};

const LevelRecord& rec_at(h2f_factor f, int32_t rec) {
    if (!f || !f->f) throw Error(H2F_E_ARG, "null factor");
    if (rec < 0 || rec >= int32_t(f->f->recs.size())) throw Error(H2F_E_ARG, "record index out of range");
    return f->f->recs[rec];
}

const ClusterFactor& cf_at(h2f_factor f, int32_t rec, int32_t cluster) {
    const LevelRecord& r = rec_at(f, rec);
    auto it = r.pos.find(cluster);
    if (it == r.pos.end()) throw Error(H2F_E_ARG, "cluster not in record");
    return r.factors[it->second];
}

void d2h(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    H2F_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx().stream));
}

}  // namespace

extern "C" {

int h2f_init(int device, double arena_gb) {
    return guard([&] { ctx_init(device, arena_gb); });
}

const char* h2f_last_error(void) { return g_err.c_str(); }

int h2f_stream(void** stream_out) {
    return guard([&] { *stream_out = reinterpret_cast<void*>(ctx().stream); });
}

int h2f_device_count(int* count) {
    return guard([&] { H2F_CUDA(cudaGetDeviceCount(count)); });
}

int h2f_kernel_launches(int64_t* count) {
    *count = kernel_launch_count();
    return H2F_OK;
}

int h2f_memory_stats(int64_t* arena_bytes, int64_t* in_use, int64_t* peak) {
    return guard([&] {
        Context& X = ctx();
        *arena_bytes = int64_t(X.arena.capacity());
        *in_use = int64_t(X.arena.in_use());
        *peak = int64_t(X.arena.peak());
    });
}

int h2f_profile_enable(int on) {
    return guard([&] { ctx().prof.on = on != 0; });
}

int h2f_profile_reset(void) {
    return guard([&] { ctx().prof.reset(); });
}

int h2f_profile_count(int32_t* nkernels) {
    *nkernels = K_COUNT;
    return H2F_OK;
}

int h2f_profile_get(int32_t kid, h2f_kernel_profile* out) {
    return guard([&] {
        if (kid < 0 || kid >= K_COUNT) throw Error(H2F_E_ARG, "kernel id out of range");
        Profiler& P = ctx().prof;
        P.collect();
        std::memset(out, 0, sizeof(*out));
        std::strncpy(out->name, kernel_name(kid), sizeof(out->name) - 1);
        out->launches = P.totals[kid].launches;
        out->seconds = P.totals[kid].seconds;
        out->flops = P.totals[kid].flops;
        out->bytes = P.totals[kid].bytes;
    });
}

int h2f_bench_dmma(int64_t iters, double* tflops) {
    return guard([&] { *tflops = bench_dmma(iters, ctx().stream); });
}

namespace {

// events around a device section on the library stream
struct DevTimer {
    cudaEvent_t a, b;
    DevTimer() {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, ctx().stream);
    }
    double stop() {
        cudaEventRecord(b, ctx().stream);
        H2F_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return ms;
    }
};

void h2d(void* dst, const void* src, size_t bytes) {
    if (bytes) H2F_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx().stream));
}

}  // namespace

int h2f_dense_svd(const double* R, int32_t m, int32_t n, double thresh, int32_t path, double* U, int32_t* kept,
                  int32_t* sweeps, double* ms) {
    return guard([&] {
        if (m < 0 || n <= 0 || m > n || path < 0 || path > 2) throw Error(H2F_E_ARG, "bad svd arguments");
        Region scr(size_t(64) << 20);
        double* dR = scr.alloc_n<double>(int64_t(m) * n);
        double* dU = scr.alloc_n<double>(int64_t(n) * n);
        int32_t* dk = scr.alloc_n<int32_t>(1);
        h2d(dR, R, sizeof(double) * m * n);
        std::vector<SvdTask> t{SvdTask{dR, dU, m, n, dk, 0}};
        std::vector<int32_t*> flags;
        DevTimer tm;
        if (path == 0) {
            if (n > SMEM_DENSE_MAX_N) throw Error(H2F_E_ARG, "shared-memory Jacobi needs n <= 144");
            launch_jacobi_smem(upload(t), 1, n, thresh, ctx().stream);
        } else {
            jacobi_multi_cta(t, thresh, scr, path == 2, &flags);
        }
        *ms = tm.stop();
        int32_t k = 0, sw = -1;
        d2h(&k, dk, sizeof(int32_t));
        if (path != 0) d2h(&sw, flags[0] + 63, sizeof(int32_t));
        ctx().sync();
        d2h(U, dU, sizeof(double) * int64_t(k) * n);
        ctx().sync();
        *kept = k;
        *sweeps = sw;
    });
}

int h2f_dense_qr_r(const double* Y, int32_t n, int32_t wf, int32_t path, double* R, double* ms) {
    return guard([&] {
        if (n <= 0 || wf <= 0 || path < 0 || path > 1) throw Error(H2F_E_ARG, "bad qr arguments");
        if (path == 0 && n > SMEM_DENSE_MAX_N) throw Error(H2F_E_ARG, "shared-memory TSQR needs n <= 144");
        Region scr(size_t(64) << 20);
        double* dY = scr.alloc_n<double>(int64_t(n) * wf);
        const int m = std::min(n, wf);
        double* dR = scr.alloc_n<double>(int64_t(n) * n);
        h2d(dY, Y, sizeof(double) * int64_t(n) * wf);
        DevTimer tm;
        if (path == 0) {
            std::vector<QrTask> t{QrTask{dY, dR, wf, n, wf, 0, wf, 0}};
            launch_qr_r_smem(upload(t), 1, n, ctx().stream);
        } else {
            qr_r_blocked({QrTask{dY, dR, wf, n, wf, 0, wf, 0}}, scr);
        }
        *ms = tm.stop();
        d2h(R, dR, sizeof(double) * int64_t(m) * n);
        ctx().sync();
    });
}

int h2f_dense_complement(const double* BT, int32_t s, int32_t kt, int32_t path, double* Q, double* ms) {
    return guard([&] {
        if (s <= 0 || kt < 0 || kt > s || path < 0 || path > 1) throw Error(H2F_E_ARG, "bad complement arguments");
        Region scr(size_t(64) << 20);
        double* dB = scr.alloc_n<double>(int64_t(std::max(kt, 1)) * s);
        double* dW = scr.alloc_n<double>(int64_t(std::max(kt, 1)) * s);
        double* dQ = scr.alloc_n<double>(int64_t(s) * s);
        double* cs = scr.alloc_n<double>(int64_t(16) * s);
        h2d(dB, BT, sizeof(double) * int64_t(kt) * s);
        std::vector<ComplementTask> t{ComplementTask{dB, dW, dQ, cs, s, kt}};
        DevTimer tm;
        if (path == 0) launch_complement(upload(t), 1, ctx().stream);
        else complement_blocked(t, scr);
        *ms = tm.stop();
        d2h(Q, dQ, sizeof(double) * int64_t(s) * s);
        ctx().sync();
    });
}

int h2f_matrix_create(const h2f_matrix_desc* desc, const double* vals, h2f_matrix* out) {
    return guard([&] {
        if (!desc || !out) throw Error(H2F_E_ARG, "null argument");
        H2Mat* m = h2mat_create(desc, vals);
        *out = new h2f_matrix_s{m};
    });
}

int h2f_matrix_create_blocks(const h2f_matrix_desc* desc, int64_t num_blocks, const double* const* block_ptrs,
                             const int64_t* block_counts, const int64_t* block_offsets, h2f_matrix* out) {
    return guard([&] {
        if (!desc || !out || (num_blocks && (!block_ptrs || !block_counts || !block_offsets)))
            throw Error(H2F_E_ARG, "null argument");
        H2Mat* m = h2mat_create_blocks(desc, num_blocks, block_ptrs, block_counts, block_offsets);
        *out = new h2f_matrix_s{m};
    });
}

int h2f_matrix_destroy(h2f_matrix m) {
    return guard([&] {
        if (!m) return;
        ctx().sync();
        delete m->m;
        delete m;
    });
}

int h2f_matrix_build(const h2f_build_desc* desc, h2f_matrix* out, int64_t* rank, double* seconds) {
    return guard([&] {
        if (!desc || !out) throw Error(H2F_E_ARG, "null argument");
        H2Mat* m = h2mat_build(desc, rank, seconds);
        *out = new h2f_matrix_s{m};
    });
}

int h2f_matrix_absorb_low_rank(h2f_matrix m, const double* w, int32_t r, double eps, h2f_matrix* out,
                               int64_t* rank, double* seconds) {
    return guard([&] {
        if (!m || !out || (r > 0 && !w)) throw Error(H2F_E_ARG, "null argument");
        H2Mat* a = h2mat_absorb_low_rank(*m->m, w, r, eps, rank, seconds);
        *out = new h2f_matrix_s{a};
    });
}

int h2f_matrix_layout(h2f_matrix m, int64_t* leaf_basis_off, int64_t* transfer_off, int64_t* coupling_off,
                      int64_t* dense_off, int64_t* nvals) {
    return guard([&] {
        const H2Mat& M = *m->m;
        if (leaf_basis_off) std::copy(M.leaf_basis_off.begin(), M.leaf_basis_off.end(), leaf_basis_off);
        if (transfer_off) std::copy(M.transfer_off.begin(), M.transfer_off.end(), transfer_off);
        if (coupling_off) std::copy(M.coupling_list.begin(), M.coupling_list.end(), coupling_off);
        if (dense_off) std::copy(M.dense_list.begin(), M.dense_list.end(), dense_off);
        if (nvals) *nvals = M.nvals;
    });
}

int h2f_matrix_values(h2f_matrix m, double* vals) {
    return guard([&] {
        if (!vals) throw Error(H2F_E_ARG, "null argument");
        d2h(vals, m->m->vals, size_t(m->m->nvals) * 8);
        ctx().sync();
    });
}

int h2f_matrix_nbytes(h2f_matrix m, int64_t* bytes) {
    return guard([&] { *bytes = m->m->nvals * 8; });
}

int h2f_matvec_dev(h2f_matrix m, const double* x_dev, double* y_dev, int64_t nrhs) {
    return guard([&] {
        if (nrhs < 1) throw Error(H2F_E_ARG, "nrhs must be >= 1");
        check_dev_ptr(x_dev, "x_dev");
        check_dev_ptr(y_dev, "y_dev");
        matvec_device(*m->m, x_dev, y_dev, int(nrhs));
        ctx().sync();
    });
}

int h2f_matvec(h2f_matrix m, const double* x, double* y, int64_t nrhs) {
    return guard([&] {
        if (nrhs < 1) throw Error(H2F_E_ARG, "nrhs must be >= 1");
        const size_t n = size_t(m->m->n) * nrhs;
        DevBuf dx(n), dy(n);
        H2F_CUDA(cudaMemcpyAsync(dx.p, x, n * 8, cudaMemcpyHostToDevice, ctx().stream));
        matvec_device(*m->m, dx.p, dy.p, int(nrhs));
        d2h(y, dy.p, n * 8);
        ctx().sync();
    });
}

int h2f_norm2(h2f_matrix m, const double* v0, int32_t iters, double* est) {
    return guard([&] { *est = norm2_estimate(*m->m, v0, iters); });
}

static int factorize_entry(h2f_matrix m, double eps_lu, double norm_estimate, const double* v0,
                           const h2f_comm* comm, h2f_factor* out, h2f_status* status) {
    std::lock_guard<std::recursive_mutex> hold(g_lock);
    if (status) *status = {H2F_OK, -1, -1};
    try {
        bind_device();
        Factorization* f = factorize(*m->m, eps_lu, norm_estimate, v0, comm);
        *out = new h2f_factor_s{f};
        return H2F_OK;
    } catch (const Error& e) {
        g_err = e.what();
        if (status) *status = {e.code, e.cluster, e.level};
        try {
            ctx().sync();
        } catch (...) {
        }
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        if (status) *status = {H2F_E_INTERNAL, -1, -1};
        return H2F_E_INTERNAL;
    }
}

int h2f_factorize(h2f_matrix m, double eps_lu, double norm_estimate, const double* v0, h2f_factor* out,
                  h2f_status* status) {
    return factorize_entry(m, eps_lu, norm_estimate, v0, nullptr, out, status);
}

int h2f_factorize_sharded(h2f_matrix m, double eps_lu, double norm_estimate, const double* v0,
                          const h2f_comm* comm, h2f_factor* out, h2f_status* status) {
    if (!comm) {
        g_err = "h2f_factorize_sharded: null comm";
        if (status) *status = {H2F_E_ARG, -1, -1};
        return H2F_E_ARG;
    }
    return factorize_entry(m, eps_lu, norm_estimate, v0, comm, out, status);
}

int h2f_shard_stats(double* stats) {
    return guard([&] {
        const ShardStats& s = shard_stats();
        const double v[8] = {s.local, s.total, s.bytes_sent, s.calls, s.tiles_here, s.batches, s.seconds,
                             s.gather_bytes};
        std::memcpy(stats, v, sizeof(v));
    });
}

int h2f_shard_owners(int64_t num_nodes, const int64_t* parent, const int64_t* level, int32_t top_level,
                     int32_t world, int32_t* owner) {
    try {
        const std::vector<int> own = shard_owners_tree(num_nodes, parent, level, top_level, world);
        for (size_t i = 0; i < own.size(); ++i) owner[i] = own[i];
        return H2F_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    }
}

int h2f_factor_destroy(h2f_factor f) {
    return guard([&] {
        if (!f) return;
        ctx().sync();
        delete f->f;
        delete f;
    });
}

int h2f_solve_dev(h2f_factor f, const double* b_dev, double* x_dev, int64_t nrhs) {
    return guard([&] {
        if (nrhs < 1) throw Error(H2F_E_ARG, "nrhs must be >= 1");
        check_dev_ptr(b_dev, "b_dev");
        check_dev_ptr(x_dev, "x_dev");
        solve_device(*f->f, b_dev, x_dev, int(nrhs));
        ctx().sync();
    });
}

int h2f_solve(h2f_factor f, const double* b, double* x, int64_t nrhs) {
    return guard([&] {
        if (nrhs < 1) throw Error(H2F_E_ARG, "nrhs must be >= 1");
        const size_t n = size_t(f->f->n) * nrhs;
        DevBuf db(n), dx(n);
        H2F_CUDA(cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, ctx().stream));
        solve_device(*f->f, db.p, dx.p, int(nrhs));
        d2h(x, dx.p, n * 8);
        ctx().sync();
    });
}

int h2f_refined_solve_dev(h2f_matrix m, h2f_factor f, const double* b_dev, double* x_dev, int32_t steps) {
    return guard([&] {
        check_dev_ptr(b_dev, "b_dev");
        check_dev_ptr(x_dev, "x_dev");
        refined_solve_device(*m->m, *f->f, b_dev, x_dev, steps);
        ctx().sync();
    });
}

int h2f_refined_solve(h2f_matrix m, h2f_factor f, const double* b, double* x, int32_t steps) {
    return guard([&] {
        const size_t n = size_t(f->f->n);
        DevBuf db(n), dx(n);
        H2F_CUDA(cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, ctx().stream));
        refined_solve_device(*m->m, *f->f, db.p, dx.p, steps);
        d2h(x, dx.p, n * 8);
        ctx().sync();
    });
}

int h2f_refined_solve_multi(h2f_matrix m, h2f_factor f, const double* b, double* x, int64_t nrhs, int32_t steps) {
    return guard([&] {
        if (nrhs < 1) throw Error(H2F_E_ARG, "nrhs must be >= 1");
        const size_t n = size_t(f->f->n) * nrhs;
        DevBuf db(n), dx(n);
        H2F_CUDA(cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, ctx().stream));
        refined_solve_device(*m->m, *f->f, db.p, dx.p, steps, int(nrhs));
        d2h(x, dx.p, n * 8);
        ctx().sync();
    });
}

int h2f_refined_solve_multi_dev(h2f_matrix m, h2f_factor f, const double* b_dev, double* x_dev, int64_t nrhs,
                                int32_t steps) {
    return guard([&] {
        if (nrhs < 1) throw Error(H2F_E_ARG, "nrhs must be >= 1");
        check_dev_ptr(b_dev, "b_dev");
        check_dev_ptr(x_dev, "x_dev");
        refined_solve_device(*m->m, *f->f, b_dev, x_dev, steps, int(nrhs));
        ctx().sync();
    });
}

// ---- factor import (serialization) -------------------------

int h2f_factor_import_begin(int64_t n, int32_t top_level, int32_t num_records, int64_t top_size, double eps_lu,
                            double eps_fill, double norm_estimate, h2f_factor* out) {
    return guard([&] {
        if (n < 0 || num_records < 0 || top_size < 0) throw Error(H2F_E_ARG, "negative sizes");
        auto f = std::make_unique<Factorization>();
        f->n = n;
        f->top_level = top_level;
        f->recs.resize(size_t(num_records));
        f->top_size = top_size;
        f->eps_lu = eps_lu;
        f->eps_fill = eps_fill;
        f->norm_estimate = norm_estimate;
        f->top_lu = f->store.alloc_n<double>(top_size * top_size);
        f->top_piv = f->store.alloc_n<int32_t>(top_size);
        *out = new h2f_factor_s{f.release()};
    });
}

int h2f_factor_import_record(h2f_factor f, int32_t rec, int32_t level, int32_t num_clusters, const int64_t* clusters,
                             const int64_t* offsets, const int64_t* sizes, int32_t num_batches,
                             const int64_t* batch_ptr, const int64_t* batch_ids, int64_t up_size,
                             const int64_t* up_index, int32_t csp, int32_t ncolors, int32_t graph_degree,
                             int32_t max_rank, double time_s) {
    return guard([&] {
        if (!f || !f->f) throw Error(H2F_E_ARG, "null factor");
        if (rec < 0 || rec >= int32_t(f->f->recs.size())) throw Error(H2F_E_ARG, "record index out of range");
        LevelRecord& R = f->f->recs[rec];
        R.level = level;
        R.clusters.assign(clusters, clusters + num_clusters);
        R.offset.assign(offsets, offsets + num_clusters);
        R.size.assign(sizes, sizes + num_clusters);
        R.batches.assign(size_t(num_batches), {});
        for (int32_t b = 0; b < num_batches; ++b) R.batches[b].assign(batch_ids + batch_ptr[b], batch_ids + batch_ptr[b + 1]);
        R.up_index.assign(up_index, up_index + up_size);
        R.csp = csp;
        R.ncolors = ncolors;
        R.graph_degree = graph_degree;
        R.max_rank = max_rank;
        R.time_s = time_s;
        R.factors.assign(size_t(num_clusters), {});
        R.pos.clear();
        for (int32_t i = 0; i < num_clusters; ++i) R.pos[int(clusters[i])] = i;
    });
}

int h2f_factor_import_cluster(h2f_factor f, int32_t rec, int32_t cluster, int32_t s, int32_t r, const double* q,
                              const double* lu, const int32_t* piv, int32_t num_edges, const int64_t* edge_other,
                              const int32_t* edge_kind, const int64_t* edge_width, const double* mw) {
    return guard([&] {
        if (!f || !f->f) throw Error(H2F_E_ARG, "null factor");
        Factorization& F = *f->f;
        if (rec < 0 || rec >= int32_t(F.recs.size())) throw Error(H2F_E_ARG, "record index out of range");
        LevelRecord& R = F.recs[rec];
        auto it = R.pos.find(cluster);
        if (it == R.pos.end()) throw Error(H2F_E_ARG, "cluster not in record");
        ClusterFactor& cf = R.factors[it->second];
        if (s != R.size[it->second] || r < 0 || r > s) throw Error(H2F_E_ARG, "cluster shape mismatch");
        cudaStream_t st = ctx().stream;
        cf.cluster = cluster;
        cf.s = s;
        cf.r = r;
        cf.offset = R.offset[it->second];
        cf.q = F.store.alloc_n<double>(int64_t(s) * s);
        H2F_CUDA(cudaMemcpyAsync(cf.q, q, sizeof(double) * s * s, cudaMemcpyHostToDevice, st));
        cf.edges.clear();
        if (r == 0) return;
        int64_t W = 0;
        for (int32_t e = 0; e < num_edges; ++e) W += edge_width[e];
        cf.lu = F.store.alloc_n<double>(int64_t(r) * r);
        cf.piv = F.store.alloc_n<int32_t>(r);
        double* MW = F.store.alloc_n<double>(int64_t(r) * W);
        H2F_CUDA(cudaMemcpyAsync(cf.lu, lu, sizeof(double) * r * r, cudaMemcpyHostToDevice, st));
        H2F_CUDA(cudaMemcpyAsync(cf.piv, piv, sizeof(int32_t) * r, cudaMemcpyHostToDevice, st));
        H2F_CUDA(cudaMemcpyAsync(MW, mw, sizeof(double) * r * W, cudaMemcpyHostToDevice, st));
        int64_t col = 0;
        for (int32_t e = 0; e < num_edges; ++e) {
            cf.edges.push_back({int(edge_other[e]), int(edge_kind[e]), MW + col, W, int(edge_width[e])});
            col += edge_width[e];
        }
        ctx().sync();  // the host arrays may be released on return
    });
}

int h2f_factor_import_top(h2f_factor f, const double* top_lu, const int32_t* top_piv) {
    return guard([&] {
        if (!f || !f->f) throw Error(H2F_E_ARG, "null factor");
        Factorization& F = *f->f;
        const int64_t n = F.top_size;
        if (n) {
            H2F_CUDA(cudaMemcpyAsync(F.top_lu, top_lu, sizeof(double) * n * n, cudaMemcpyHostToDevice, ctx().stream));
            H2F_CUDA(cudaMemcpyAsync(F.top_piv, top_piv, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx().stream));
        }
        ctx().sync();
    });
}

int h2f_factor_import_end(h2f_factor f) {
    return guard([&] {
        if (!f || !f->f) throw Error(H2F_E_ARG, "null factor");
        Factorization& F = *f->f;
        // nbytes (factorization.py:181-190) and completeness
        int64_t nb = F.top_size * F.top_size * 8 + F.top_size * 4;
        for (auto& rec : F.recs) {
            nb += int64_t(rec.up_index.size()) * 8;
            for (auto& cf : rec.factors) {
                if (!cf.q) throw Error(H2F_E_ARG, "factor import: cluster " + std::to_string(cf.cluster) +
                                                      " of level " + std::to_string(rec.level) + " missing");
                nb += int64_t(cf.s) * cf.s * 8;
                if (cf.r) nb += int64_t(cf.r) * cf.r * 8 + int64_t(cf.r) * 4;
                for (auto& e : cf.edges) nb += int64_t(cf.r) * e.w * 8;
            }
        }
        F.nbytes = nb;
    });
}

int h2f_factor_info_get(h2f_factor f, h2f_factor_info* info) {
    return guard([&] {
        const Factorization& F = *f->f;
        info->n = F.n;
        info->top_level = F.top_level;
        info->num_records = int32_t(F.recs.size());
        info->top_size = F.top_size;
        info->eps_lu = F.eps_lu;
        info->eps_fill = F.eps_fill;
        info->norm_estimate = F.norm_estimate;
        info->nbytes = F.nbytes;
        for (int i = 0; i < 8; ++i) info->phase_seconds[i] = F.phase[i];
    });
}

int h2f_factor_level_info(h2f_factor f, int32_t rec, h2f_level_info* info) {
    return guard([&] {
        const LevelRecord& r = rec_at(f, rec);
        info->level = r.level;
        info->num_clusters = int32_t(r.clusters.size());
        info->num_batches = int32_t(r.batches.size());
        info->csp = r.csp;
        info->ncolors = r.ncolors;
        info->graph_degree = r.graph_degree;
        info->max_rank = r.max_rank;
        info->total_size = r.total();
        info->up_size = int64_t(r.up_index.size());
        int64_t be = 0;
        for (auto& b : r.batches) be += int64_t(b.size());
        info->batch_entries = be;
        info->time_s = r.time_s;
    });
}

int h2f_factor_level_arrays(h2f_factor f, int32_t rec, int64_t* clusters, int64_t* offsets, int64_t* sizes,
                            int64_t* batch_ptr, int64_t* batch_ids, int64_t* up_index) {
    return guard([&] {
        const LevelRecord& r = rec_at(f, rec);
        for (size_t i = 0; i < r.clusters.size(); ++i) {
            if (clusters) clusters[i] = r.clusters[i];
            if (offsets) offsets[i] = r.offset[i];
            if (sizes) sizes[i] = r.size[i];
        }
        int64_t k = 0;
        if (batch_ptr) batch_ptr[0] = 0;
        for (size_t b = 0; b < r.batches.size(); ++b) {
            for (int c : r.batches[b]) {
                if (batch_ids) batch_ids[k] = c;
                ++k;
            }
            if (batch_ptr) batch_ptr[b + 1] = k;
        }
        if (up_index) std::copy(r.up_index.begin(), r.up_index.end(), up_index);
    });
}

int h2f_factor_level_fills(h2f_factor f, int32_t rec, int64_t* num_init, int64_t* init_pairs,
                           int64_t* num_created, int64_t* created) {
    return guard([&] {
        const LevelRecord& r = rec_at(f, rec);
        if (num_init) *num_init = int64_t(r.fill_init.size());
        if (init_pairs)
            for (size_t i = 0; i < r.fill_init.size(); ++i) {
                init_pairs[2 * i] = key_a(r.fill_init[i]);
                init_pairs[2 * i + 1] = key_b(r.fill_init[i]);
            }
        int64_t k = 0;
        for (size_t b = 0; b < r.fill_created.size(); ++b)
            for (Key key : r.fill_created[b]) {
                if (created) {
                    created[3 * k] = int64_t(b);
                    created[3 * k + 1] = key_a(key);
                    created[3 * k + 2] = key_b(key);
                }
                ++k;
            }
        if (num_created) *num_created = k;
    });
}

int h2f_factor_cluster_info(h2f_factor f, int32_t rec, int32_t cluster, h2f_cluster_info* ci) {
    return guard([&] {
        const ClusterFactor& c = cf_at(f, rec, cluster);
        ci->cluster = c.cluster;
        ci->level = rec_at(f, rec).level;
        ci->size = c.s;
        ci->r = c.r;
        ci->num_edges = int32_t(c.edges.size());
        ci->offset = c.offset;
    });
}

int h2f_factor_cluster_arrays(h2f_factor f, int32_t rec, int32_t cluster, double* q, double* lu, int32_t* piv,
                              int64_t* edge_other, int32_t* edge_kind, int64_t* edge_width) {
    return guard([&] {
        const ClusterFactor& c = cf_at(f, rec, cluster);
        if (q) d2h(q, c.q, sizeof(double) * c.s * c.s);
        if (lu && c.r) d2h(lu, c.lu, sizeof(double) * c.r * c.r);
        if (piv && c.r) d2h(piv, c.piv, sizeof(int32_t) * c.r);
        for (size_t e = 0; e < c.edges.size(); ++e) {
            if (edge_other) edge_other[e] = c.edges[e].other;
            if (edge_kind) edge_kind[e] = c.edges[e].kind;
            if (edge_width) edge_width[e] = c.edges[e].w;
        }
        ctx().sync();
    });
}

int h2f_factor_cluster_edge(h2f_factor f, int32_t rec, int32_t cluster, int32_t e, double* mat) {
    return guard([&] {
        const ClusterFactor& c = cf_at(f, rec, cluster);
        if (e < 0 || e >= int32_t(c.edges.size())) throw Error(H2F_E_ARG, "edge index out of range");
        const EdgeRec& E = c.edges[e];
        if (c.r && E.w)
            H2F_CUDA(cudaMemcpy2DAsync(mat, sizeof(double) * E.w, E.mat, sizeof(double) * E.ld,
                                       sizeof(double) * E.w, c.r, cudaMemcpyDeviceToHost, ctx().stream));
        ctx().sync();
    });
}

int h2f_factor_top(h2f_factor f, double* top_lu, int32_t* top_piv) {
    return guard([&] {
        const Factorization& F = *f->f;
        if (top_lu) d2h(top_lu, F.top_lu, sizeof(double) * F.top_size * F.top_size);
        if (top_piv) d2h(top_piv, F.top_piv, sizeof(int32_t) * F.top_size);
        ctx().sync();
    });
}

int h2f_debug_replay_set(const int64_t* kept_rows, int64_t nkept, const int64_t* created_rows, int64_t ncreated) {
    return guard([&] {
        Replay& R = replay();
        R = Replay{};
        for (int64_t i = 0; i < nkept; ++i) {
            const int64_t* r = kept_rows + 3 * i;
            R.kept[(r[0] << 32) | uint32_t(r[1])] = int(r[2]);
        }
        for (int64_t i = 0; i < ncreated; ++i) {
            const int64_t* r = created_rows + 4 * i;
            R.created[(r[0] << 32) | uint32_t(r[1])].push_back(canon(int(r[2]), int(r[3])));
        }
        R.active = true;
    });
}

int h2f_debug_replay_clear(void) {
    return guard([&] { replay() = Replay{}; });
}

int h2f_debug_replay_stats(int64_t* stats) {
    return guard([&] {
        const Replay& R = replay();
        stats[0] = R.kept_forced;
        stats[1] = R.kept_changed;
        stats[2] = R.fill_changed;
        for (int i = 0; i < 5; ++i) stats[3 + i] = R.fill_margin_hist[i];
    });
}

int h2f_greedy_coloring(int64_t num_clusters, const int64_t* clusters, int64_t num_pairs, const int64_t* pairs,
                        int32_t* colors_out, int32_t* num_colors, int32_t* max_degree) {
    // structure.py:137-167 (same algorithm as the factorization's level colouring)
    return guard([&] {
        std::vector<int64_t> ids(clusters, clusters + num_clusters);
        std::vector<size_t> order(ids.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = i;
        std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ids[a] < ids[b]; });
        std::unordered_map<int64_t, size_t> pos;
        for (size_t i = 0; i < ids.size(); ++i) pos[ids[i]] = i;
        std::vector<std::vector<size_t>> adj(ids.size());
        for (int64_t p = 0; p < num_pairs; ++p) {
            const int64_t s = pairs[2 * p], t = pairs[2 * p + 1];
            if (s == t) continue;
            auto is = pos.find(s), it = pos.find(t);
            if (is == pos.end() || it == pos.end()) throw Error(H2F_E_ARG, "pair references unknown cluster");
            adj[is->second].push_back(it->second);
            adj[it->second].push_back(is->second);
        }
        int deg = 0;
        for (auto& a : adj) {
            std::sort(a.begin(), a.end());
            a.erase(std::unique(a.begin(), a.end()), a.end());
            deg = std::max(deg, int(a.size()));
        }
        std::vector<int> col;
        const int ncol = greedy_coloring(order, ids.size(), [&](size_t i, auto visit) {
            for (size_t j : adj[i]) visit(j);
        }, col);
        std::copy(col.begin(), col.end(), colors_out);
        *num_colors = ncol;
        *max_degree = deg;
    });
}

}  // extern "C"
