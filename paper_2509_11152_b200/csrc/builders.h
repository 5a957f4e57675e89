// Host-side builders of the batched task lists (GEMM, copy) shared by the
// factorization driver and the dense per-cluster orchestration.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "kernels.h"
#include "runtime.h"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace h2f {

#ifdef _OPENMP
inline int max_threads() { return omp_get_max_threads(); }
inline int thread_id() { return omp_get_thread_num(); }
#else
inline int max_threads() { return 1; }
inline int thread_id() { return 0; }
#endif

struct GemmBuild {
    std::vector<GemmTask> tasks;
    std::vector<GemmContrib> contribs;
    std::vector<int64_t> tile_start{0};
    std::vector<int64_t> tile_cost;  // per task: K chunks per tile + epilogue weight
    int64_t norm_tiles = 0;
    double flops = 0, bytes = 0;  // algorithmic work of the launch (profiler)

    static int64_t tiles(int M, int N) { return cdiv(M, GEMM_TILE) * cdiv(N, GEMM_TILE); }
    // returns the task's norm base (mode NORM) or -1
    int64_t add(double* C, int64_t ldc, int M, int N, int mode, const GemmContrib* cs, size_t nc) {
        if (M <= 0 || N <= 0) return -1;
        GemmTask t{};
        t.C = C;
        t.ldc = ldc;
        t.M = M;
        t.N = N;
        t.mode = mode;
        t.tiles_n = int(cdiv(N, GEMM_TILE));
        t.contrib_begin = int64_t(contribs.size());
        for (size_t i = 1; i < nc; ++i)  // the kernel applies alpha once per task
            if (cs[i].alpha != cs[0].alpha) throw Error(H2F_E_INTERNAL, "assertion: mixed alpha in one GEMM task");
        contribs.insert(contribs.end(), cs, cs + nc);
        t.contrib_end = int64_t(contribs.size());
        int64_t chunks = mode == GEMM_ADD ? 2 : 1;
        for (size_t i = 0; i < nc; ++i) {
            if (cs[i].K > 0) chunks += cdiv(cs[i].K, GEMM_BK);
            flops += 2.0 * M * N * cs[i].K;
            bytes += 8.0 * (double(M) * cs[i].K + double(cs[i].K) * N);
        }
        bytes += mode == GEMM_ADD ? 16.0 * M * N : (mode == GEMM_STORE ? 8.0 * M * N : 0.0);
        t.norm_base = -1;
        const int64_t nt = tiles(M, N);
        if (mode == GEMM_NORM) {
            t.norm_base = norm_tiles;
            norm_tiles += nt;
        }
        tasks.push_back(t);
        tile_start.push_back(tile_start.back() + nt);
        tile_cost.push_back(chunks);
        return t.norm_base;
    }
    // task whose `nc` contributions already sit at [begin, begin+nc) of an
    // external (pinned-uploaded) contribution array `ext`; kflops = sum of K,
    // chunks = sum of ceil(K / GEMM_BK), alpha uniform (the caller's duty)
    const GemmContrib* ext = nullptr;
    int64_t add_ext(double* C, int64_t ldc, int M, int N, int mode, int64_t begin, int64_t nc, double ksum,
                    int64_t chunks) {
        if (M <= 0 || N <= 0) return -1;
        GemmTask t{};
        t.C = C;
        t.ldc = ldc;
        t.M = M;
        t.N = N;
        t.mode = mode;
        t.tiles_n = int(cdiv(N, GEMM_TILE));
        t.contrib_begin = begin;
        t.contrib_end = begin + nc;
        flops += 2.0 * M * N * ksum;
        bytes += 8.0 * ksum * (double(M) + N);
        bytes += mode == GEMM_ADD ? 16.0 * M * N : (mode == GEMM_STORE ? 8.0 * M * N : 0.0);
        t.norm_base = -1;
        const int64_t nt = tiles(M, N);
        if (mode == GEMM_NORM) {
            t.norm_base = norm_tiles;
            norm_tiles += nt;
        }
        tasks.push_back(t);
        tile_start.push_back(tile_start.back() + nt);
        tile_cost.push_back(chunks + (mode == GEMM_ADD ? 2 : 1));
        return t.norm_base;
    }
    // n external-contribution tasks at once (all with M, N > 0), e.g. the
    // ~1e5 Schur targets / fill candidates of a leaf-level batch: get(i)
    // describes task i (called in parallel); tile offsets, norm bases and the
    // work sums are formed serially in task order, exactly as n add_ext calls
    // would, and the task records are written in parallel.
    struct BulkItem {
        double* C;
        int64_t ldc;
        int M, N;
        int64_t begin, nc;
        double ksum;
        int64_t chunks;
    };
    template <class F> void add_ext_bulk(int64_t n, int mode, F&& get, int64_t* norm_base_out) {
        if (n <= 0) return;
        const size_t t0 = tasks.size();
        std::vector<BulkItem> it(static_cast<size_t>(n));
        tasks.resize(t0 + size_t(n));
        tile_start.resize(t0 + 1 + size_t(n));
        tile_cost.resize(t0 + size_t(n));
        // two-pass parallel scan over contiguous thread ranges: items and
        // per-range sums, range offsets, then tile offsets / norm bases /
        // task records (the work sums feed the profiler and the kernel-variant
        // choice only, whose variants are bit-identical)
        const int nth = n > 4096 ? max_threads() : 1;
        std::vector<int64_t> tsum(size_t(nth) + 1, 0);
        std::vector<double> fsum(size_t(nth), 0.0), bsum(size_t(nth), 0.0);
        bool bad = false;
        const int64_t ts0 = tile_start[t0], nb0 = norm_tiles;
#pragma omp parallel num_threads(nth) if (nth > 1) reduction(|| : bad)
        {
            const int tid = thread_id();
            const int64_t lo = n * tid / nth, hi = n * (tid + 1) / nth;
            int64_t acc = 0;
            double f = 0, by = 0;
            for (int64_t i = lo; i < hi; ++i) {
                BulkItem& b = it[size_t(i)];
                b = get(i);
                if (b.M <= 0 || b.N <= 0) bad = true;
                acc += tiles(b.M, b.N);
                f += 2.0 * b.M * b.N * b.ksum;
                by += 8.0 * b.ksum * (double(b.M) + b.N) +
                      (mode == GEMM_ADD ? 16.0 * b.M * b.N : (mode == GEMM_STORE ? 8.0 * b.M * b.N : 0.0));
            }
            tsum[size_t(tid) + 1] = acc;
            fsum[size_t(tid)] = f;
            bsum[size_t(tid)] = by;
#pragma omp barrier
#pragma omp single
            for (int q = 0; q < nth; ++q) tsum[size_t(q) + 1] += tsum[size_t(q)];
            int64_t run = tsum[size_t(tid)];
            for (int64_t i = lo; i < hi; ++i) {
                const BulkItem& b = it[size_t(i)];
                const int64_t nt = tiles(b.M, b.N);
                GemmTask t{};
                t.C = b.C;
                t.ldc = b.ldc;
                t.M = b.M;
                t.N = b.N;
                t.mode = mode;
                t.tiles_n = int(cdiv(b.N, GEMM_TILE));
                t.contrib_begin = b.begin;
                t.contrib_end = b.begin + b.nc;
                t.norm_base = -1;
                if (mode == GEMM_NORM) {
                    t.norm_base = nb0 + run;
                    norm_base_out[i] = t.norm_base;
                }
                run += nt;
                tile_start[t0 + 1 + size_t(i)] = ts0 + run;
                tasks[t0 + size_t(i)] = t;
                tile_cost[t0 + size_t(i)] = b.chunks + (mode == GEMM_ADD ? 2 : 1);
            }
        }
        if (bad) throw Error(H2F_E_INTERNAL, "assertion: empty bulk GEMM task");
        for (int q = 0; q < nth; ++q) {
            flops += fsum[size_t(q)];
            bytes += bsum[size_t(q)];
        }
        if (mode == GEMM_NORM) norm_tiles += tsum[size_t(nth)];
    }
    int64_t add1(double* C, int64_t ldc, int M, int N, int mode, const GemmContrib& c) {
        return add(C, ldc, M, N, mode, &c, 1);
    }
    // per-CTA tile ranges with equal shares of the total chunk cost
    std::vector<int64_t> cta_ranges() const {
        const int64_t ntiles = tile_start.back();
        const int G = gemm_grid(ntiles);
        std::vector<int64_t> cta(size_t(G) + 1, ntiles);
        cta[0] = 0;
        double total = 0;
        for (size_t t = 0; t < tasks.size(); ++t) total += double(tile_start[t + 1] - tile_start[t]) * tile_cost[t];
        double acc = 0;
        int b = 1;
        for (size_t t = 0; t < tasks.size() && b < G; ++t) {
            const int64_t nt = tile_start[t + 1] - tile_start[t];
            const double c = double(tile_cost[t]), end = acc + double(nt) * c;
            while (b < G && total * b / G <= end) {
                int64_t off = int64_t(std::ceil((total * b / G - acc) / c));
                off = std::min<int64_t>(std::max<int64_t>(off, 0), nt);
                cta[b] = std::max(cta[b - 1], tile_start[t] + off);
                ++b;
            }
            acc = end;
        }
        return cta;
    }
    void launch(int kid, double* norms = nullptr, double bytes_override = -1.0) {
        if (tasks.empty()) return;
        Context& X = ctx();
        const int64_t ntiles = tile_start.back();
        auto* dt = X.up.put(tasks);
        const GemmContrib* dc = ext ? ext : X.up.put(contribs);
        auto* ds = X.up.put(tile_start);
        // short average K per tile: the C read-modify-write dominates, use
        // the variant that prefetches C during the tile's math
        static const double kmax = [] {
            // measured on config 2 (round 2): the C-prefetch variant is as
            // fast or faster at every K (Schur 5.43 -> 5.35 s), so it is used
            // throughout unless this caps it
            const char* e = std::getenv("H2F_GEMM_PREC_KMAX");
            return e ? std::atof(e) : 1e30;
        }();
        const double keff = flops / (double(ntiles) * 2.0 * GEMM_TILE * GEMM_TILE);
        // K_eff below this: the register-direct short-K kernel (one tile per
        // CTA, no cost-balanced CTA ranges needed)
        static const double kwarp = [] {
            const char* e = std::getenv("H2F_GEMM_WARP_KMAX");
            return e ? std::atof(e) : 40.0;
        }();
        const int64_t* dcta =
            keff >= kwarp && ntiles > gemm_grid(ntiles) ? X.up.put(cta_ranges()) : nullptr;
        X.up.flush(X.stream);
        ProfScope ps(kid, flops, bytes_override >= 0 ? bytes_override : bytes, double(ntiles));
        const int role = kid == K_GEMM_SCHUR ? 1 : 0;
        if (keff < kwarp)
            launch_gemm_warp(dt, dc, ds, int32_t(tasks.size()), ntiles, norms, X.stream, role);
        else
            launch_gemm_tasks(dt, dc, ds, int32_t(tasks.size()), ntiles, dcta, norms, X.stream, keff < kmax, role);
    }
};

inline GemmContrib contrib(const double* A, int64_t lda, int transA, const double* B, int64_t ldb,
                           int transB, int K, double alpha = 1.0) {
    GemmContrib c{};
    c.A = A;
    c.lda = lda;
    c.transA = transA;
    c.B = B;
    c.ldb = ldb;
    c.transB = transB;
    c.K = K;
    c.alpha = alpha;
    return c;
}

struct CopyBuild {
    std::vector<CopyTask> tasks;
    std::vector<int64_t> tile_start{0};
    double bytes = 0;
    void add(double* dst, int64_t ldd, int rows, int cols, const double* src, int64_t lds, int trans,
             int mode, double alpha = 1.0) {
        if (rows <= 0 || cols <= 0) return;
        CopyTask t{};
        t.dst = dst;
        t.ldd = ldd;
        t.rows = rows;
        t.cols = cols;
        t.src = src;
        t.lds = lds;
        t.trans = trans;
        t.mode = mode;
        t.alpha = alpha;
        tasks.push_back(t);
        tile_start.push_back(tile_start.back() + cdiv(rows, COPY_TILE) * cdiv(cols, COPY_TILE));
        bytes += double(rows) * cols * (mode == COPY_ZERO ? 8.0 : (mode == COPY_ADD ? 24.0 : 16.0));
    }
    void zero(double* dst, int64_t ldd, int rows, int cols) { add(dst, ldd, rows, cols, nullptr, 0, 0, COPY_ZERO); }
    void launch() {
        if (tasks.empty()) return;
        Context& X = ctx();
        auto* dt = X.up.put(tasks);
        auto* ds = X.up.put(tile_start);
        X.up.flush(X.stream);
        ProfScope ps(K_COPY, 0.0, bytes);
        launch_copy_tasks(dt, ds, int32_t(tasks.size()), tile_start.back(), X.stream);
    }
};

template <class T> inline T* upload(const std::vector<T>& v) {
    Context& X = ctx();
    T* d = X.up.put(v);
    X.up.flush(X.stream);
    return d;
}

}  // namespace h2f
