// Dense top of the factorization (factorization.py:259-263, solve.py:46-55):
//
//   coop_panel_lu   partial-pivot LU of one nb-column panel of the n_top x n_top
//                   top matrix by a cooperative grid (one CTA per SM).  Each CTA
//                   keeps its slice of panel rows in shared memory; one grid
//                   barrier per column (argmax candidates + candidate rows are
//                   exchanged through a small global table, double-buffered by
//                   column parity).  Same pivot rule as LAPACK idamax (first
//                   index of the largest |a|), same scale-by-reciprocal rule.
//   top_trsv        sync-free blocked triangular solve (unit lower / upper) of
//                   the row-major LU: CTAs take row blocks in ticket order and
//                   consume earlier blocks as their completion flags appear, so
//                   the matrix streams through all SMs in one launch and the
//                   critical path is one 64x64 block per step.
//   top_perm        composes LAPACK's sequential row swaps into one gather map.
#include <algorithm>
#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace h2f {

namespace {

constexpr int PT = 256;          // threads per panel CTA
constexpr int PNB = TOP_PANEL_NB; // max panel width
constexpr int PLD = PNB + 1;      // smem row stride (bank spread)

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nct) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nct - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(PT) coop_panel_lu_kernel(double* A, int64_t lda, int n, int k0, int nb,
                                                          int* piv, TopPanelScratch S) {
    extern __shared__ double P[];  // chunk x PLD
    __shared__ double prow[PNB];
    __shared__ double shv[PT / 32];
    __shared__ int shi[PT / 32];
    __shared__ int s_p, s_w;
    const int G = gridDim.x, b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = n - k0;
    const int chunk = (m + G - 1) / G;
    const int r0 = k0 + b * chunk;                      // first global row owned
    const int nr = max(0, min(n, r0 + chunk) - r0);     // rows owned
    for (int e = threadIdx.x; e < nr * nb; e += PT) {
        const int i = e / nb, j = e % nb;
        P[i * PLD + j] = A[(int64_t)(r0 + i) * lda + k0 + j];
    }
    __syncthreads();
    for (int c = 0; c < nb; ++c) {
        const int gk = k0 + c;
        const int par = c & 1;
        // local first-index argmax of |P[i][c]| over owned rows >= gk
        double v = -1.0;
        int idx = INT_MAX;
        for (int i = max(0, gk - r0) + threadIdx.x; i < nr; i += PT) {
            const double a = fabs(P[i * PLD + c]);
            if (a > v) { v = a; idx = r0 + i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
        if (lane == 0) { shv[warp] = v; shi[warp] = idx; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double bv = shv[0];
            int bi = shi[0];
            for (int w = 1; w < PT / 32; ++w)
                if (shv[w] > bv || (shv[w] == bv && shi[w] < bi)) { bv = shv[w]; bi = shi[w]; }
            S.val[par * G + b] = bv;
            S.idx[par * G + b] = bi;
            s_p = bi;
        }
        __syncthreads();
        // candidate row and (owner of gk) the current row gk go to the table
        if (s_p != INT_MAX && threadIdx.x < nb)
            S.rows[((int64_t)par * G + b) * PNB + threadIdx.x] = P[(s_p - r0) * PLD + threadIdx.x];
        if (gk >= r0 && gk < r0 + nr && threadIdx.x < nb)
            S.rowk[par * PNB + threadIdx.x] = P[(gk - r0) * PLD + threadIdx.x];
        __threadfence();
        grid_sync(S.bar, G);
        // global argmax (same fixed order in every CTA)
        if (warp == 0) {
            double bv = -1.0;
            int bi = INT_MAX, bw = -1;
            for (int w = lane; w < G; w += 32) {
                const double ov = __ldcg(S.val + par * G + w);
                const int oi = __ldcg(S.idx + par * G + w);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; bw = w; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const int ow = __shfl_xor_sync(0xffffffffu, bw, o);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; bw = ow; }
            }
            if (lane == 0) { s_p = bi; s_w = bw; }
        }
        __syncthreads();
        const int p = s_p, w = s_w;
        if (b == 0 && threadIdx.x == 0) piv[gk] = p;
        if (threadIdx.x < nb) prow[threadIdx.x] = __ldcg(S.rows + ((int64_t)par * G + w) * PNB + threadIdx.x);
        __syncthreads();
        if (p != gk) {
            if (p >= r0 && p < r0 + nr && threadIdx.x < nb)
                P[(p - r0) * PLD + threadIdx.x] = __ldcg(S.rowk + par * PNB + threadIdx.x);
            if (gk >= r0 && gk < r0 + nr && threadIdx.x < nb) P[(gk - r0) * PLD + threadIdx.x] = prow[threadIdx.x];
        }
        __syncthreads();
        const double pv = prow[c];
        const int i0 = max(0, gk + 1 - r0);
        if (pv != 0.0) {
            const bool recip = fabs(pv) >= DBL_MIN;
            const double inv = 1.0 / pv;
            for (int i = i0 + threadIdx.x; i < nr; i += PT) {
                double& a = P[i * PLD + c];
                a = recip ? a * inv : a / pv;
            }
        }
        __syncthreads();
        const int wd = nb - c - 1;
        if (wd > 0)
            for (int e = threadIdx.x; e < (nr - i0) * wd; e += PT) {
                const int i = i0 + e / wd, j = c + 1 + e % wd;
                P[i * PLD + j] -= P[i * PLD + c] * prow[j];
            }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < nr * nb; e += PT) {
        const int i = e / nb, j = e % nb;
        A[(int64_t)(r0 + i) * lda + k0 + j] = P[i * PLD + j];
    }
}

// ---- sync-free blocked triangular solve -------------------------------------
constexpr int TB = 64;   // row block
constexpr int TT = 256;  // threads
constexpr int TW = TT / 32;
constexpr int RPW = TB / TW;  // rows per warp (8)

template <bool UPPER>
__global__ void __launch_bounds__(TT) top_trsv_kernel(const double* __restrict__ lu, int n, double* x, int nrhs,
                                                      int* sync) {
    __shared__ double D[TB][TB + 1];
    __shared__ double y[TB];
    __shared__ int s_t;
    int* ticket = sync;
    volatile int* flag = sync + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nblk = (n + TB - 1) / TB;
    if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1);
    __syncthreads();
    const int ib = UPPER ? nblk - 1 - s_t : s_t;
    const int row0 = ib * TB;
    const int rb = min(TB, n - row0);
    // diagonal block into shared memory while earlier blocks finish
    for (int e = threadIdx.x; e < TB * TB; e += TT) {
        const int i = e / TB, j = e % TB;
        D[i][j] = (i < rb && j < rb) ? lu[(int64_t)(row0 + i) * n + row0 + j] : 0.0;
    }
    for (int rh = 0; rh < nrhs; ++rh) {
        double acc[RPW];
#pragma unroll
        for (int q = 0; q < RPW; ++q) acc[q] = 0.0;
        for (int s = 0; s < nblk - 1; ++s) {
            const int jb = UPPER ? nblk - 1 - s : s;
            if (UPPER ? jb <= ib : jb >= ib) break;
            if (threadIdx.x == 0)
            {
                while (flag[jb] <= rh) __nanosleep(20);
                __threadfence();
            }
            __syncthreads();
            const int c0 = jb * TB;
            const int cb = min(TB, n - c0);
            const double x0 = lane < cb ? __ldcg(x + (int64_t)(c0 + lane) * nrhs + rh) : 0.0;
            const double x1 = lane + 32 < cb ? __ldcg(x + (int64_t)(c0 + lane + 32) * nrhs + rh) : 0.0;
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int i = warp * RPW + q;
                if (i < rb) {
                    const double* li = lu + (int64_t)(row0 + i) * n + c0;
                    if (lane < cb) acc[q] += li[lane] * x0;
                    if (lane + 32 < cb) acc[q] += li[lane + 32] * x1;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
            const double a = warp_sum(acc[q]);
            const int i = warp * RPW + q;
            if (lane == 0 && i < rb) y[i] = __ldcg(x + (int64_t)(row0 + i) * nrhs + rh) - a;
        }
        __syncthreads();
        if (warp == 0) {
            double v0 = lane < rb ? y[lane] : 0.0, v1 = lane + 32 < rb ? y[lane + 32] : 0.0;
            if (!UPPER) {
                for (int k = 0; k < rb; ++k) {
                    const double xk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31);
                    if (lane > k) v0 -= D[lane][k] * xk;
                    if (lane + 32 > k) v1 -= D[lane + 32][k] * xk;
                }
            } else {
                for (int k = rb - 1; k >= 0; --k) {
                    if (lane == (k & 31)) {
                        if (k < 32) v0 /= D[k][k]; else v1 /= D[k][k];
                    }
                    const double xk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31);
                    if (lane < k) v0 -= D[lane][k] * xk;
                    if (lane + 32 < k) v1 -= D[lane + 32][k] * xk;
                }
            }
            if (lane < rb) x[(int64_t)(row0 + lane) * nrhs + rh] = v0;
            if (lane + 32 < rb) x[(int64_t)(row0 + lane + 32) * nrhs + rh] = v1;
            __threadfence();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicExch(sync + 1 + ib, rh + 1);
        }
    }
}

// perm[i] = source row of position i after LAPACK's sequential swaps
__global__ void top_perm_kernel(const int* __restrict__ piv, int n, int* __restrict__ perm) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < n; ++k) {
            const int p = piv[k];
            if (p != k) {
                const int t = perm[k];
                perm[k] = perm[p];
                perm[p] = t;
            }
        }
}

__global__ void permute_rows_kernel(const double* __restrict__ src, const int* __restrict__ perm, int n, int nrhs,
                                    double* __restrict__ dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)n * nrhs) return;
    const int i = (int)(e / nrhs), rh = (int)(e % nrhs);
    dst[e] = src[(int64_t)perm[i] * nrhs + rh];
}



}  // namespace

int top_panel_grid(int m) {
    // >= 32 rows per CTA, one CTA per SM, panel slice within shared memory
    int g = std::max(1, std::min(sm_count(), (m + 31) / 32));
    while (g < sm_count() && size_t((m + g - 1) / g) * PLD * sizeof(double) > TOP_PANEL_SMEM) ++g;
    return g;
}

bool launch_coop_panel_lu(double* A, int64_t lda, int32_t n, int32_t k0, int32_t nb, int32_t* piv,
                          TopPanelScratch S, cudaStream_t st) {
    const int m = n - k0;
    const int G = top_panel_grid(m);
    const size_t smem = size_t((m + G - 1) / G) * PLD * sizeof(double);
    if (smem > TOP_PANEL_SMEM || nb > PNB) return false;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(coop_panel_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TOP_PANEL_SMEM);
        configured = true;
    }
    cudaMemsetAsync(S.bar, 0, 2 * sizeof(unsigned), st);
    void* args[] = {(void*)&A, (void*)&lda, (void*)&n, (void*)&k0, (void*)&nb, (void*)&piv, (void*)&S};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)coop_panel_lu_kernel, dim3(G), dim3(PT), args, smem, st);
    if (e != cudaSuccess) {
        cudaGetLastError();  // handled: the caller falls back to the one-CTA panel; keep no sticky error
        return false;
    }
    count_launch();
    return true;
}

void launch_top_perm(const int32_t* piv, int32_t n, int32_t* perm, cudaStream_t st) {
    if (n <= 0) return;
    top_perm_kernel<<<1, 1024, 0, st>>>(piv, n, perm);
    count_launch();
}

void launch_permute_rows(const double* src, const int32_t* perm, int32_t n, int32_t nrhs, double* dst,
                         cudaStream_t st) {
    const int64_t tot = int64_t(n) * nrhs;
    if (tot <= 0) return;
    permute_rows_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(src, perm, n, nrhs, dst);
    count_launch();
}

void launch_top_solve(const double* lu, const int32_t* perm, int32_t n, double* x, int32_t nrhs, double* tmp,
                      int32_t* sync, cudaStream_t st) {
    if (n <= 0) return;
    const int nblk = (n + TB - 1) / TB;
    const int64_t tot = int64_t(n) * nrhs;
    permute_rows_kernel<<<unsigned((tot + 255) / 256), 256, 0, st>>>(x, perm, n, nrhs, tmp);
    cudaMemsetAsync(sync, 0, sizeof(int) * (nblk + 1), st);
    top_trsv_kernel<false><<<nblk, TT, 0, st>>>(lu, n, tmp, nrhs, sync);
    cudaMemsetAsync(sync, 0, sizeof(int) * (nblk + 1), st);
    top_trsv_kernel<true><<<nblk, TT, 0, st>>>(lu, n, tmp, nrhs, sync);
    cudaMemcpyAsync(x, tmp, sizeof(double) * tot, cudaMemcpyDeviceToDevice, st);
    count_launch();
    count_launch();
    count_launch();
}

}  // namespace h2f
