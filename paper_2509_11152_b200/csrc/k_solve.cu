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
constexpr int STW = ST / 32;

// In-place triangular solve of one vector v (length r, stride vs) held in
// shared memory by the whole CTA: 64-row blocks, the off-block products by
// all warps, the 64x64 diagonal block by warp 0 through shuffles.
// LOWER: unit lower (L of LU); else upper with diagonal (U of LU).
template <bool LOWER>
__device__ void cta_trsv(const double* __restrict__ A, int r, double* v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nblk = (r + 63) / 64;
    for (int t = 0; t < nblk; ++t) {
        const int b = LOWER ? t : nblk - 1 - t;
        const int r0 = b * 64, rb = min(64, r - r0);
        // rows of block b minus the already solved part
        const int c0 = LOWER ? 0 : r0 + rb, c1 = LOWER ? r0 : r;
        if (c1 > c0) {
            // 4 rows per warp step, their loads in flight together (each
            // row's lane-strided sum and butterfly are the one-row form's)
            for (int i0 = warp * 4; i0 < rb; i0 += 4 * STW) {
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                const double* a0 = A + (int64_t)(r0 + i0) * r;
#pragma unroll 2
                for (int j = c0 + lane; j < c1; j += 32) {
                    const double vj = v[j];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (i0 + q < rb) acc[q] += a0[(int64_t)q * r + j] * vj;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double t = warp_sum(acc[q]);
                    if (lane == 0 && i0 + q < rb) v[r0 + i0 + q] -= t;
                }
            }
            __syncthreads();
        }
        if (warp == 0) {
            double v0 = lane < rb ? v[r0 + lane] : 0.0, v1 = lane + 32 < rb ? v[r0 + lane + 32] : 0.0;
            if (LOWER) {
                for (int k = 0; k < rb; ++k) {
                    const double xk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31);
                    const double* ak = A + (int64_t)r0 * r + r0 + k;
                    if (lane > k && lane < rb) v0 -= ak[(int64_t)lane * r] * xk;
                    if (lane + 32 > k && lane + 32 < rb) v1 -= ak[(int64_t)(lane + 32) * r] * xk;
                }
            } else {
                for (int k = rb - 1; k >= 0; --k) {
                    const double* ak = A + (int64_t)r0 * r + r0 + k;
                    if (lane == (k & 31)) {
                        const double d = ak[(int64_t)k * r];
                        if (k < 32) v0 /= d; else v1 /= d;
                    }
                    const double xk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31);
                    if (lane < k) v0 -= ak[(int64_t)lane * r] * xk;
                    if (lane + 32 < k) v1 -= ak[(int64_t)(lane + 32) * r] * xk;
                }
            }
            if (lane < rb) v[r0 + lane] = v0;
            if (lane + 32 < rb) v[r0 + lane + 32] = v1;
        }
        __syncthreads();
    }
}


__global__ void __launch_bounds__(ST)
solve_tasks_kernel(const SolveTask* __restrict__ tasks, const SolveCluster* __restrict__ cls,
                   const SolveEdge* __restrict__ edges, double* __restrict__ y, double* __restrict__ scratch,
                   double* __restrict__ work, int nrhs) {
    extern __shared__ double sv[];
    const SolveTask T = tasks[blockIdx.x];
    const SolveCluster C = cls[T.cl];
    const int s = C.s, r = C.r;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* yc = y + C.off * nrhs;
    double* wk = work + C.woff;                      // s x nrhs
    double* tb = work + C.woff + (int64_t)s * nrhs;  // nch x r x nrhs gather partials
    switch (T.kind) {
    case ST_ROT_T: {
        // 64 columns x 4 row groups, partial sums reduced through shared memory
        const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
        const int j = T.begin + tx;
        for (int rh = 0; rh < nrhs; ++rh) {
            for (int i = threadIdx.x; i < s; i += ST) sv[i] = yc[(int64_t)i * nrhs + rh];
            __syncthreads();
            double acc = 0.0;
            if (j < T.end)
                for (int i = ty; i < s; i += 4) acc += C.q[(int64_t)i * s + j] * sv[i];
            sv[s + ty * 64 + tx] = acc;
            __syncthreads();
            if (ty == 0 && j < T.end)
                wk[(int64_t)j * nrhs + rh] = ((sv[s + tx] + sv[s + 64 + tx]) + sv[s + 128 + tx]) + sv[s + 192 + tx];
            __syncthreads();
        }
        break;
    }
    case ST_PROD: {
        const int64_t j = T.begin + threadIdx.x;
        for (int rh = 0; rh < nrhs; ++rh) {
            for (int k = threadIdx.x; k < r; k += ST) sv[k] = wk[(int64_t)k * nrhs + rh];
            __syncthreads();
            if (j < T.end) {
                double acc = 0.0;
                const double* mj = C.mw + j;
                for (int k = 0; k < r; ++k) acc += mj[(int64_t)k * C.W] * sv[k];
                scratch[(C.soff + j) * nrhs + rh] = acc;
            }
            __syncthreads();
        }
        break;
    }
    case ST_LSOLVE: {
        for (int rh = 0; rh < nrhs; ++rh) {
            for (int i = threadIdx.x; i < r; i += ST) sv[i] = wk[(int64_t)i * nrhs + rh];
            __syncthreads();
            if (threadIdx.x == 0)
                for (int k = 0; k < r; ++k) {
                    const int p = C.piv[k];
                    if (p != k) { const double a = sv[k]; sv[k] = sv[p]; sv[p] = a; }
                }
            __syncthreads();
            cta_trsv<true>(C.lu, r, sv);
            for (int i = threadIdx.x; i < s; i += ST)
                yc[(int64_t)i * nrhs + rh] = i < r ? sv[i] : wk[(int64_t)i * nrhs + rh];
            __syncthreads();
        }
        break;
    }
    case ST_USOLVE: {
        for (int rh = 0; rh < nrhs; ++rh) {
            for (int i = threadIdx.x; i < r; i += ST) sv[i] = yc[(int64_t)i * nrhs + rh];
            __syncthreads();
            cta_trsv<false>(C.lu, r, sv);
            for (int i = threadIdx.x; i < s; i += ST)
                wk[(int64_t)i * nrhs + rh] = i < r ? sv[i] : yc[(int64_t)i * nrhs + rh];
            __syncthreads();
        }
        break;
    }
    case ST_GATHER: {
        // columns [c0, c1) of the eliminators: the edges are consecutive
        // column slices of mw (edge e starts at column soff_e - C.soff)
        const int ch = T.c0 / SOLVE_GATHER_COLS;
        double* part = tb + (int64_t)ch * r * nrhs;
        for (int k = T.begin + warp; k < T.end; k += STW)
            for (int rh = 0; rh < nrhs; ++rh) {
                double acc = 0.0;
                for (int64_t ei = T.e0; ei < T.e1; ++ei) {
                    const SolveEdge E = edges[ei];
                    const int e0 = (int)(E.soff - C.soff);
                    const int lo = max(e0, T.c0), hi = min(e0 + E.w, T.c1);
                    if (lo >= hi) continue;
                    const double* mk = E.mat + (int64_t)k * E.ld - e0;
                    const double* ys = y + (E.lo - e0) * nrhs + rh;
#pragma unroll 8
                    for (int j = lo + lane; j < hi; j += 32) acc += mk[j] * ys[(int64_t)j * nrhs];
                }
                acc = warp_sum(acc);
                if (lane == 0) part[(int64_t)k * nrhs + rh] = acc;
            }
        break;
    }
    case ST_ROT: {
        for (int rh = 0; rh < nrhs; ++rh) {
            for (int j = threadIdx.x; j < s; j += ST) {
                double t = 0.0;
                if (j < r)
                    for (int ch = 0; ch < C.nch; ++ch) t += tb[((int64_t)ch * r + j) * nrhs + rh];
                sv[j] = wk[(int64_t)j * nrhs + rh] + t;
            }
            __syncthreads();
            for (int i0 = T.begin + 4 * warp; i0 < T.end; i0 += 4 * STW) {
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                const double* q0 = C.q + (int64_t)i0 * s;
#pragma unroll 2
                for (int j = lane; j < s; j += 32) {
                    const double vj = sv[j];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (i0 + q < T.end) acc[q] += q0[(int64_t)q * s + j] * vj;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double t = warp_sum(acc[q]);
                    if (lane == 0 && i0 + q < T.end) yc[(int64_t)(i0 + q) * nrhs + rh] = t;
                }
            }
            __syncthreads();
        }
        break;
    }
    }
}

__global__ void __launch_bounds__(ST)
fwd_scatter_kernel(const ScatterGroup* __restrict__ groups, const int64_t* __restrict__ list,
                   const double* __restrict__ scratch, double* __restrict__ y, int nrhs) {
    const ScatterGroup G = groups[blockIdx.x];
    // gridDim.y CTAs share a group's element range (multi-RHS blocks)
    const int64_t tot = (int64_t)G.w * nrhs;
    const int64_t per = (tot + gridDim.y - 1) / gridDim.y;
    const int64_t e0 = (int64_t)blockIdx.y * per, e1 = min(tot, e0 + per);
    for (int64_t e = e0 + threadIdx.x; e < e1; e += ST) {
        double acc = y[G.lo * nrhs + e];
        for (int64_t l = G.begin; l < G.end; ++l) acc += scratch[list[l] * nrhs + e];
        y[G.lo * nrhs + e] = acc;
    }
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

// nrhs = 1 variant with coalesced loads in both orientations: the output
// segment is accumulated in shared memory, contribution by contribution (in
// order, one writer per element: deterministic); y += A x reads rows of A
// (a warp per output row, lanes along the row), y += A^T x reads columns of A
// as rows of the stored block (a thread per output element, consecutive
// threads on consecutive addresses) -- the one-warp-per-output form walked a
// column with lane stride lda, a quarter of every sector wasted.
constexpr int GV_T = 128;

__global__ void __launch_bounds__(GV_T)
gemv1_tasks_kernel(const GemvTask* __restrict__ tasks, const GemvContrib* __restrict__ contribs) {
    const GemvTask T = tasks[blockIdx.x];
    extern __shared__ double acc[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < T.rows; i += GV_T) acc[i] = 0.0;
    __syncthreads();
    for (int64_t ci = T.contrib_begin; ci < T.contrib_end; ++ci) {
        const GemvContrib P = contribs[ci];
        if (P.trans) {
            for (int i = threadIdx.x; i < T.rows; i += GV_T) {
                const double* a = P.A + i;
                double part = 0.0;
#pragma unroll 8
                for (int j = 0; j < P.cols; ++j) part += __ldg(a + (int64_t)j * P.lda) * __ldg(P.x + j);
                acc[i] += P.alpha * part;
            }
        } else {
            // GV_R rows per warp and step, their loads issued together (the
            // per-row sums -- lane-strided, then the warp butterfly -- are
            // the one-row form's, bit for bit; only more of them are in
            // flight before the reductions)
            constexpr int GV_R = 4;
            for (int i0 = warp * GV_R; i0 < T.rows; i0 += GV_R * (GV_T / 32)) {
                double part[GV_R];
#pragma unroll
                for (int r = 0; r < GV_R; ++r) part[r] = 0.0;
                const double* a0 = P.A + (int64_t)i0 * P.lda;
#pragma unroll 2
                for (int j = lane; j < P.cols; j += 32) {
                    const double xj = __ldg(P.x + j);
#pragma unroll
                    for (int r = 0; r < GV_R; ++r)
                        if (i0 + r < T.rows) part[r] += __ldg(a0 + (int64_t)r * P.lda + j) * xj;
                }
#pragma unroll
                for (int r = 0; r < GV_R; ++r) {
                    const double v = warp_sum(part[r]);
                    if (lane == 0 && i0 + r < T.rows) acc[i0 + r] += P.alpha * v;
                }
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < T.rows; i += GV_T) {
        double* d = T.y + i;
        if (T.mode == COPY_ADD) *d += acc[i]; else *d = acc[i];
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

void launch_solve_tasks(const SolveTask* d_tasks, int32_t ntasks, const SolveCluster* d_cl,
                        const SolveEdge* d_edges, double* y, double* scratch, double* work, int32_t nrhs,
                        cudaStream_t st) {
    if (ntasks <= 0) return;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(solve_tasks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SOLVE_SMEM_VEC * 8);
        configured = true;
    }
    solve_tasks_kernel<<<ntasks, ST, SOLVE_SMEM_VEC * sizeof(double), st>>>(d_tasks, d_cl, d_edges, y, scratch,
                                                                            work, nrhs);
    count_launch();
}

void launch_fwd_scatter(const ScatterGroup* d_groups, int32_t ngroups, const int64_t* d_list,
                        const double* scratch, double* y, int32_t nrhs, cudaStream_t st, int32_t ysplit) {
    if (ngroups <= 0) return;
    fwd_scatter_kernel<<<dim3(ngroups, max(1, ysplit)), ST, 0, st>>>(d_groups, d_list, scratch, y, nrhs);
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

void launch_gemv_tasks(const GemvTask* d_tasks, int32_t ntasks, const GemvContrib* d_contribs,
                       int32_t nrhs, cudaStream_t st, int32_t max_rows) {
    if (ntasks <= 0) return;
    static const bool v1 = [] {
        const char* e = std::getenv("H2F_GEMV1");
        return !(e && std::atoi(e) == 0);
    }();
    if (v1 && nrhs == 1 && max_rows > 0 && max_rows <= 6144) {
        const size_t smem = sizeof(double) * size_t(max_rows);
        if (smem > 48 * 1024) cudaFuncSetAttribute(gemv1_tasks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(smem));
        gemv1_tasks_kernel<<<ntasks, GV_T, smem, st>>>(d_tasks, d_contribs);
    } else {
        gemv_tasks_kernel<<<ntasks, 128, 0, st>>>(d_tasks, d_contribs, nrhs);
    }
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
