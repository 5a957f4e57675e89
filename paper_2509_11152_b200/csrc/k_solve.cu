// Substitution sweeps (solve.py:45-164), H2 matvec GEMV tasks
// (h2core.py:272-315) and vector utilities (power iteration, h2core.py:318-330).
//
// Forward sweep of one batch (solve.py:90-128) = fwd_clusters (rotation
// Q~^T y_c, eliminator products W^T y_R into a scratch area, pivots + unit
// lower TRSV) followed by fwd_scatter, which adds the products into each
// target span in a fixed order (per-target gather instead of the reference's
// sequential scatter: no atomics, bitwise deterministic).  The backward sweep
// (solve.py:131-164) is conflict-free and runs as one kernel per batch.
#include "common.cuh"
#include "kernels.h"

namespace h2f {

namespace {

constexpr int ST = 256;

__global__ void __launch_bounds__(ST)
fwd_clusters_kernel(const SolveCluster* __restrict__ cls, const SolveEdge* __restrict__ edges,
                    double* __restrict__ y, double* __restrict__ scratch, int nrhs,
                    double* __restrict__ work) {
    const SolveCluster C = cls[blockIdx.x];
    const int s = C.s, r = C.r;
    double* yc = y + C.off * nrhs;
    extern __shared__ double tmp[];  // s * nrhs when it fits, else the cluster's work slot
    double* t = ((int64_t)s * nrhs <= 6144) ? tmp : work + C.woff;
    // 1. rotate: t = Q^T y_c
    for (int64_t e = threadIdx.x; e < (int64_t)s * nrhs; e += ST) {
        const int j = (int)(e / nrhs), rh = (int)(e % nrhs);
        double acc = 0.0;
        for (int i = 0; i < s; ++i) acc += C.q[(int64_t)i * s + j] * yc[(int64_t)i * nrhs + rh];
        t[e] = acc;
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)s * nrhs; e += ST) yc[e] = t[e];
    __syncthreads();
    if (r == 0) return;
    // 2. products p_e = mat_e^T y_R
    for (int64_t ei = C.edge_begin; ei < C.edge_end; ++ei) {
        const SolveEdge E = edges[ei];
        double* out = scratch + E.soff * nrhs;
        for (int64_t e = threadIdx.x; e < (int64_t)E.w * nrhs; e += ST) {
            const int j = (int)(e / nrhs), rh = (int)(e % nrhs);
            double acc = 0.0;
            for (int k = 0; k < r; ++k) acc += E.mat[(int64_t)k * E.ld + j] * yc[(int64_t)k * nrhs + rh];
            out[e] = acc;
        }
    }
    __syncthreads();
    // 3. pivots + unit lower solve on y_R (one warp)
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (int k = 0; k < r; ++k) {
            const int p = C.piv[k];
            if (p != k)
                for (int rh = lane; rh < nrhs; rh += 32) {
                    const double a = yc[(int64_t)k * nrhs + rh];
                    yc[(int64_t)k * nrhs + rh] = yc[(int64_t)p * nrhs + rh];
                    yc[(int64_t)p * nrhs + rh] = a;
                }
            __syncwarp();
        }
        for (int k = 0; k < r; ++k) {
            for (int64_t e = lane; e < (int64_t)(r - k - 1) * nrhs; e += 32) {
                const int i = k + 1 + (int)(e / nrhs), rh = (int)(e % nrhs);
                yc[(int64_t)i * nrhs + rh] -= C.lu[(int64_t)i * r + k] * yc[(int64_t)k * nrhs + rh];
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(ST)
fwd_scatter_kernel(const ScatterGroup* __restrict__ groups, const int64_t* __restrict__ list,
                   const double* __restrict__ scratch, double* __restrict__ y, int nrhs) {
    const ScatterGroup G = groups[blockIdx.x];
    for (int64_t e = threadIdx.x; e < (int64_t)G.w * nrhs; e += ST) {
        double acc = y[G.lo * nrhs + e];
        for (int64_t l = G.begin; l < G.end; ++l) acc += scratch[list[l] * nrhs + e];
        y[G.lo * nrhs + e] = acc;
    }
}

__global__ void __launch_bounds__(ST)
bwd_clusters_kernel(const SolveCluster* __restrict__ cls, const SolveEdge* __restrict__ edges,
                    double* __restrict__ y, int nrhs, double* __restrict__ work) {
    const SolveCluster C = cls[blockIdx.x];
    const int s = C.s, r = C.r;
    double* yc = y + C.off * nrhs;
    extern __shared__ double tmp[];
    double* t = ((int64_t)s * nrhs <= 6144) ? tmp : work + C.woff;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = ST / 32;
    if (r > 0) {
        // 1. upper solve on y_R (one warp, column oriented)
        if (threadIdx.x < 32) {
            for (int k = r - 1; k >= 0; --k) {
                const double ukk = C.lu[(int64_t)k * r + k];
                for (int rh = lane; rh < nrhs; rh += 32) yc[(int64_t)k * nrhs + rh] /= ukk;
                __syncwarp();
                for (int64_t e = lane; e < (int64_t)k * nrhs; e += 32) {
                    const int i = (int)(e / nrhs), rh = (int)(e % nrhs);
                    yc[(int64_t)i * nrhs + rh] -= C.lu[(int64_t)i * r + k] * yc[(int64_t)k * nrhs + rh];
                }
                __syncwarp();
            }
        }
        __syncthreads();
        // 2. acc = sum_e mat_e y[span_e]  (warp per redundant row)
        for (int64_t e = warp; e < (int64_t)r * nrhs; e += nw) {
            const int k = (int)(e / nrhs), rh = (int)(e % nrhs);
            double acc = 0.0;
            for (int64_t ei = C.edge_begin; ei < C.edge_end; ++ei) {
                const SolveEdge E = edges[ei];
                const double* mk = E.mat + (int64_t)k * E.ld;
                for (int j = lane; j < E.w; j += 32) acc += mk[j] * y[(E.lo + j) * nrhs + rh];
            }
            acc = warp_sum(acc);
            if (lane == 0) t[e] = acc;
        }
        __syncthreads();
        for (int64_t e = threadIdx.x; e < (int64_t)r * nrhs; e += ST) yc[e] += t[e];
        __syncthreads();
    }
    // 3. y_c = Q y_c (warp per row)
    for (int64_t e = warp; e < (int64_t)s * nrhs; e += nw) {
        const int i = (int)(e / nrhs), rh = (int)(e % nrhs);
        const double* qi = C.q + (int64_t)i * s;
        double acc = 0.0;
        for (int j = lane; j < s; j += 32) acc += qi[j] * yc[(int64_t)j * nrhs + rh];
        acc = warp_sum(acc);
        if (lane == 0) t[e] = acc;
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)s * nrhs; e += ST) yc[e] = t[e];
}

__global__ void gather_rows_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx,
                                   int64_t n, int nrhs, double* __restrict__ dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nrhs) return;
    const int64_t i = e / nrhs, rh = e % nrhs;
    dst[e] = src[idx[i] * nrhs + rh];
}

__global__ void scatter_rows_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx,
                                    int64_t n, int nrhs, double* __restrict__ dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nrhs) return;
    const int64_t i = e / nrhs, rh = e % nrhs;
    dst[idx[i] * nrhs + rh] = src[e];
}

// dense LU solve (lu_solve semantics) by one CTA; x is n x nrhs
__global__ void __launch_bounds__(1024)
top_solve_kernel(const double* __restrict__ lu, const int* __restrict__ piv, int n,
                 double* __restrict__ x, int nrhs) {
    for (int k = 0; k < n; ++k) {
        const int p = piv[k];
        if (p != k)
            for (int rh = threadIdx.x; rh < nrhs; rh += blockDim.x) {
                const double a = x[(int64_t)k * nrhs + rh];
                x[(int64_t)k * nrhs + rh] = x[(int64_t)p * nrhs + rh];
                x[(int64_t)p * nrhs + rh] = a;
            }
        __syncthreads();
    }
    for (int k = 0; k < n; ++k) {
        for (int64_t e = threadIdx.x; e < (int64_t)(n - k - 1) * nrhs; e += blockDim.x) {
            const int i = k + 1 + (int)(e / nrhs), rh = (int)(e % nrhs);
            x[(int64_t)i * nrhs + rh] -= lu[(int64_t)i * n + k] * x[(int64_t)k * nrhs + rh];
        }
        __syncthreads();
    }
    for (int k = n - 1; k >= 0; --k) {
        const double ukk = lu[(int64_t)k * n + k];
        for (int rh = threadIdx.x; rh < nrhs; rh += blockDim.x) x[(int64_t)k * nrhs + rh] /= ukk;
        __syncthreads();
        for (int64_t e = threadIdx.x; e < (int64_t)k * nrhs; e += blockDim.x) {
            const int i = (int)(e / nrhs), rh = (int)(e % nrhs);
            x[(int64_t)i * nrhs + rh] -= lu[(int64_t)i * n + k] * x[(int64_t)k * nrhs + rh];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(128)
gemv_tasks_kernel(const GemvTask* __restrict__ tasks, const GemvContrib* __restrict__ contribs,
                  int nrhs) {
    const GemvTask T = tasks[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t e = warp; e < (int64_t)T.rows * nrhs; e += 4) {
        const int i = (int)(e / nrhs), rh = (int)(e % nrhs);
        double acc = 0.0;
        for (int64_t ci = T.contrib_begin; ci < T.contrib_end; ++ci) {
            const GemvContrib P = contribs[ci];
            double part = 0.0;
            if (P.trans) {
                for (int j = lane; j < P.cols; j += 32)
                    part += P.A[(int64_t)j * P.lda + i] * P.x[(int64_t)j * nrhs + rh];
            } else {
                const double* ai = P.A + (int64_t)i * P.lda;
                for (int j = lane; j < P.cols; j += 32) part += ai[j] * P.x[(int64_t)j * nrhs + rh];
            }
            acc += P.alpha * part;
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            double* d = T.y + e;
            if (T.mode == COPY_ADD) *d += acc; else *d = acc;
        }
    }
}

constexpr int NPART = 256;

__global__ void sumsq_partial_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += x[i] * x[i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sqrt_sum_kernel(const double* __restrict__ part, int np, double* __restrict__ out) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) *out = sqrt(s);
}

__global__ void scale_by_inv_kernel(double* __restrict__ x, const double* __restrict__ w, int64_t n,
                                    const double* __restrict__ s) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const double d = *s;
    if (i < n) x[i] = (d != 0.0) ? w[i] / d : w[i];
}

__global__ void axpby_kernel(double* __restrict__ y, const double* __restrict__ a, double alpha,
                             const double* __restrict__ b, double beta, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = alpha * a[i] + beta * b[i];
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_fwd_clusters(const SolveCluster* d_cl, int32_t ncl, const SolveEdge* d_edges, double* y,
                         double* scratch, int32_t nrhs, double* work, cudaStream_t st) {
    if (ncl <= 0) return;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(fwd_clusters_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             6144 * 8);
        configured = true;
    }
    fwd_clusters_kernel<<<ncl, ST, 6144 * sizeof(double), st>>>(d_cl, d_edges, y, scratch, nrhs, work);
    count_launch();
}

void launch_fwd_scatter(const ScatterGroup* d_groups, int32_t ngroups, const int64_t* d_list,
                        const double* scratch, double* y, int32_t nrhs, cudaStream_t st) {
    if (ngroups <= 0) return;
    fwd_scatter_kernel<<<ngroups, ST, 0, st>>>(d_groups, d_list, scratch, y, nrhs);
    count_launch();
}

void launch_bwd_clusters(const SolveCluster* d_cl, int32_t ncl, const SolveEdge* d_edges, double* y,
                         int32_t nrhs, double* work, cudaStream_t st) {
    if (ncl <= 0) return;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(bwd_clusters_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             6144 * 8);
        configured = true;
    }
    bwd_clusters_kernel<<<ncl, ST, 6144 * sizeof(double), st>>>(d_cl, d_edges, y, nrhs, work);
    count_launch();
}

void launch_gather_rows(const double* src, const int64_t* idx, int64_t n, int32_t nrhs, double* dst,
                        cudaStream_t st) {
    if (n <= 0) return;
    gather_rows_kernel<<<nblk(n * nrhs, 256), 256, 0, st>>>(src, idx, n, nrhs, dst);
    count_launch();
}

void launch_scatter_rows(const double* src, const int64_t* idx, int64_t n, int32_t nrhs, double* dst,
                         cudaStream_t st) {
    if (n <= 0) return;
    scatter_rows_kernel<<<nblk(n * nrhs, 256), 256, 0, st>>>(src, idx, n, nrhs, dst);
    count_launch();
}

void launch_top_solve(const double* lu, const int32_t* piv, int32_t n, double* x, int32_t nrhs,
                      double* work, cudaStream_t st) {
    (void)work;
    if (n <= 0) return;
    top_solve_kernel<<<1, 1024, 0, st>>>(lu, piv, n, x, nrhs);
    count_launch();
}

void launch_gemv_tasks(const GemvTask* d_tasks, int32_t ntasks, const GemvContrib* d_contribs,
                       int32_t nrhs, cudaStream_t st) {
    if (ntasks <= 0) return;
    gemv_tasks_kernel<<<ntasks, 128, 0, st>>>(d_tasks, d_contribs, nrhs);
    count_launch();
}

void launch_norm2(const double* x, int64_t n, double* partial, double* out, cudaStream_t st) {
    sumsq_partial_kernel<<<NPART, 256, 0, st>>>(x, n, partial);
    sqrt_sum_kernel<<<1, 256, 0, st>>>(partial, NPART, out);
    count_launch();
    count_launch();
}

void launch_scale_by_inv(double* x, const double* w, int64_t n, const double* s, cudaStream_t st) {
    if (n <= 0) return;
    scale_by_inv_kernel<<<nblk(n, 256), 256, 0, st>>>(x, w, n, s);
    count_launch();
}

void launch_axpby(double* y, const double* a, double alpha, const double* b, double beta, int64_t n,
                  cudaStream_t st) {
    if (n <= 0) return;
    axpby_kernel<<<nblk(n, 256), 256, 0, st>>>(y, a, alpha, b, beta, n);
    count_launch();
}

}  // namespace h2f
