// Kernels of the device H2 construction: kernel-matrix
// entry evaluation (dense near-field blocks, coupling matrices), Chebyshev
// grids and tensor Lagrange interpolation (leaf bases, transfers), and the
// small helpers of the recompression (singular values as row norms, diagonal
// weights).  Reference: h2core.py:128-185 (build_h2), kernels.py:44-86
// (kernel families), geometry.py chebyshev helpers.
//
// All of it is HBM-write bound (a dense block entry costs one sqrt and one
// exp / cos / log and is written once), so the kernels are tile loops with
// the point coordinates staged in shared memory and coalesced row stores.
#include "common.cuh"
#include "kernels.h"

namespace h2f {

namespace {

int grid_for(int64_t ntiles, int per_sm) {
    const int64_t cap = int64_t(sm_count()) * per_sm;
    return int(ntiles < cap ? ntiles : cap);
}

constexpr double PI = 3.14159265358979323846;

__device__ __forceinline__ double kernel_of_r(const KernelParams& k, double r) {
    switch (k.family) {
        case KF_EXP_COV: return exp(-r / k.corr_length);
        case KF_LAPLACE2D: return -log(r) / (2.0 * PI);
        default: return cos(k.kappa * r) / r;  // KF_HELMHOLTZ3D
    }
}

constexpr int ET = 32;  // eval tile (rows x cols)

__global__ void __launch_bounds__(256)
eval_tasks_kernel(const EvalTask* __restrict__ tasks, const int64_t* __restrict__ tile_start, int ntasks,
                  int64_t ntiles, KernelParams kp) {
    __shared__ double xs[ET][3], ys[ET][3];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ti = find_segment(tile_start, ntasks, tile);
        const EvalTask T = tasks[ti];
        const int64_t local = tile - tile_start[ti];
        const int tn = (T.cols + ET - 1) / ET;
        const int r0 = int(local / tn) * ET, c0 = int(local % tn) * ET;
        __syncthreads();
        if (threadIdx.x < ET * kp.dim) {
            const int i = threadIdx.x / kp.dim, a = threadIdx.x % kp.dim;
            xs[i][a] = r0 + i < T.rows ? T.X[int64_t(r0 + i) * kp.dim + a] : 0.0;
        } else if (threadIdx.x >= 128 && threadIdx.x < 128 + ET * kp.dim) {
            const int e = threadIdx.x - 128, i = e / kp.dim, a = e % kp.dim;
            ys[i][a] = c0 + i < T.cols ? T.Y[int64_t(c0 + i) * kp.dim + a] : 0.0;
        }
        __syncthreads();
        const int c = c0 + tx;
        if (c >= T.cols) continue;
        for (int i = ty; i < ET; i += 8) {
            const int r = r0 + i;
            if (r >= T.rows) break;
            // scipy cdist order: sum over axes 0..dim-1, then sqrt
            double s = 0.0;
            for (int a = 0; a < kp.dim; ++a) {
                const double d = xs[i][a] - ys[tx][a];
                s += d * d;
            }
            double v;
            if (T.diag && int64_t(r) + T.row0 == int64_t(c) + T.col0)
                v = kp.diag_base + kp.alpha_r;
            else
                v = kernel_of_r(kp, sqrt(s));
            T.out[int64_t(r) * T.ldo + c] = v;
        }
    }
}

__device__ __forceinline__ double cheb_node(int p, int k, double lo, double hi) {
    const double t = cos((2 * k + 1) * PI / (2 * p));
    return 0.5 * (t + 1.0) * (hi - lo) + lo;
}

// tensor Chebyshev grid of one box: point (a, b, c) at index (a p + b) p + c
__global__ void grid_tasks_kernel(const GridTask* __restrict__ tasks, int ntasks, int dim) {
    const GridTask T = tasks[blockIdx.x];
    int npts = T.p;
    for (int a = 1; a < dim; ++a) npts *= T.p;
    for (int i = threadIdx.x; i < npts; i += blockDim.x) {
        int rem = i;
        for (int a = dim - 1; a >= 0; --a) {
            const int k = rem % T.p;
            rem /= T.p;
            T.out[int64_t(i) * dim + a] = cheb_node(T.p, k, T.lo[a], T.hi[a]);
        }
    }
}

constexpr int MAXP = 32;

// one warp per point: per-axis barycentric Lagrange weights of the point in
// the box's Chebyshev nodes (an exact node hit gives the unit row), then the
// tensor product written as one row of p^dim values
__global__ void __launch_bounds__(256)
interp_tasks_kernel(const InterpTask* __restrict__ tasks, const int64_t* __restrict__ pt_start, int ntasks,
                    int64_t npts_total, int dim) {
    __shared__ double wsh[8][3][MAXP];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t g = int64_t(blockIdx.x) * 8 + w; g < npts_total; g += int64_t(gridDim.x) * 8) {
        const int ti = find_segment(pt_start, ntasks, g);
        const InterpTask T = tasks[ti];
        const int64_t i = g - pt_start[ti];
        const int p = T.p;
        for (int a = 0; a < dim; ++a) {
            const double x = T.pts[i * dim + a];
            double q = 0.0;
            int hit = 0;
            if (lane < p) {
                const double node = cheb_node(p, lane, T.lo[a], T.hi[a]);
                const double bw = ((lane & 1) ? -1.0 : 1.0) * sin((2 * lane + 1) * PI / (2 * p));
                const double diff = x - node;
                hit = diff == 0.0;
                q = bw / diff;
            }
            const unsigned hits = __ballot_sync(0xffffffffu, hit);
            double s = warp_sum(lane < p && !hits ? q : 0.0);
            if (lane < p) {
                double v;
                if (hits) {
                    // numpy: the hit row is zeroed, then 1 at the (last) hit column
                    v = (lane == 31 - __clz(hits)) ? 1.0 : 0.0;
                } else {
                    v = q / s;
                }
                wsh[w][a][lane] = v;
            }
            __syncwarp();
        }
        int ncols = p;
        for (int a = 1; a < dim; ++a) ncols *= p;
        double* out = T.out + i * T.ldo;
        for (int col = lane; col < ncols; col += 32) {
            int rem = col;
            double v = 1.0;
            for (int a = dim - 1; a >= 0; --a) {
                v *= wsh[w][a][rem % p];
                rem /= p;
            }
            out[col] = v;
        }
        __syncwarp();
    }
}

// sig[j] = |row j of P| (one warp per row)
__global__ void __launch_bounds__(256) row_norms_kernel(const RowNormOut* __restrict__ tasks,
                                                        const int64_t* __restrict__ row_start, int ntasks,
                                                        int64_t nrows) {
    const int lane = threadIdx.x & 31;
    for (int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < nrows;
         g += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const int ti = find_segment(row_start, ntasks, g);
        const RowNormOut T = tasks[ti];
        const int64_t j = g - row_start[ti];
        const double* r = T.P + j * T.ldp;
        double a = 0.0;
        for (int c = lane; c < T.len; c += 32) a += r[c] * r[c];
        a = warp_sum(a);
        if (lane == 0) T.out[j] = sqrt(a);
    }
}

// D (n x n) = diag(w[0..n))
__global__ void set_diag_kernel(const DiagTask* __restrict__ tasks) {
    const DiagTask T = tasks[blockIdx.x];
    const int64_t nn = int64_t(T.n) * T.n;
    for (int64_t e = threadIdx.x; e < nn; e += blockDim.x) {
        const int i = int(e / T.n), j = int(e % T.n);
        T.D[e] = i == j ? T.w[i] : 0.0;
    }
}

}  // namespace

void launch_eval_tasks(const EvalTask* d_tasks, const int64_t* d_tile_start, int32_t ntasks, int64_t ntiles,
                       const KernelParams& kp, cudaStream_t st) {
    if (ntiles <= 0) return;
    eval_tasks_kernel<<<grid_for(ntiles, 8), 256, 0, st>>>(d_tasks, d_tile_start, ntasks, ntiles, kp);
    count_launch();
}

void launch_grid_tasks(const GridTask* d_tasks, int32_t ntasks, int32_t dim, cudaStream_t st) {
    if (ntasks <= 0) return;
    grid_tasks_kernel<<<ntasks, 128, 0, st>>>(d_tasks, ntasks, dim);
    count_launch();
}

void launch_interp_tasks(const InterpTask* d_tasks, const int64_t* d_pt_start, int32_t ntasks, int64_t npts,
                         int32_t dim, cudaStream_t st) {
    if (npts <= 0) return;
    interp_tasks_kernel<<<grid_for((npts + 7) / 8, 8), 256, 0, st>>>(d_tasks, d_pt_start, ntasks, npts, dim);
    count_launch();
}

void launch_row_norms(const RowNormOut* d_tasks, const int64_t* d_row_start, int32_t ntasks, int64_t nrows,
                      cudaStream_t st) {
    if (nrows <= 0) return;
    row_norms_kernel<<<grid_for((nrows + 7) / 8, 8), 256, 0, st>>>(d_tasks, d_row_start, ntasks, nrows);
    count_launch();
}

void launch_set_diag(const DiagTask* d_tasks, int32_t ntasks, cudaStream_t st) {
    if (ntasks <= 0) return;
    set_diag_kernel<<<ntasks, 256, 0, st>>>(d_tasks);
    count_launch();
}

}  // namespace h2f
