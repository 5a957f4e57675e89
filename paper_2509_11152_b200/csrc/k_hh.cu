// Blocked Householder QR with a cooperative multi-CTA panel (LAPACK geqrf
// conventions: dlarfg reflectors, dlarft forward/columnwise T).
//
// Used for the two tall QRs of the augmentation (factorization.py:78 and the
// complete QR of b_aug, :98) once the clusters outgrow one CTA.  One panel of
// HH_NB columns is spread over `ncta` co-resident CTAs, each holding a
// contiguous slice of the panel's rows in shared memory; every column costs
// one group barrier (norm and the dots with the rest of the panel travel
// together, the reflector's dots are recovered from the unscaled ones) and the
// partial sums are reduced in a fixed order, so the factor is bitwise
// reproducible.  The trailing update A -= V T^T (V^T A) runs on the DMMA tile
// GEMM (k_gemm.cu) between panels.
#include <algorithm>
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace h2f {

namespace {

constexpr int HT = 256;
constexpr int HW = HT / 32;

// LAPACK dlarfg-style reflector for x = [alpha, rest]; ss = ||rest||^2.
__device__ __forceinline__ void hh_reflector(double alpha, double ss, double& beta, double& tau, double& scal) {
    if (ss == 0.0) {
        beta = alpha;
        tau = 0.0;
        scal = 0.0;
    } else {
        beta = -copysign(hypot(alpha, sqrt(ss)), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
    }
}

// barrier over the `n` CTAs of one task (generation counter in bar[1])
__device__ __forceinline__ void group_barrier(uint32_t* bar, int n) {
    __syncthreads();
    if (threadIdx.x == 0) {
        // monotonic arrival counter (zeroed before the launch): the k-th
        // barrier completes when the counter reaches k * n -- one release
        // atomic per CTA, acquire polling, no reset round trip (the release /
        // acquire pair orders the CTA's writes, which bar.sync has ordered
        // before thread 0's atomic; H2F_BARRIER_FENCES keeps explicit fences)
#ifdef H2F_BARRIER_FENCES
        __threadfence();
#endif
        uint32_t old;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        const uint32_t target = (old / uint32_t(n) + 1u) * uint32_t(n);
        uint32_t cur;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
        } while (int32_t(cur - target) < 0);
#ifdef H2F_BARRIER_FENCES
        __threadfence();
#endif
    }
    __syncthreads();
}

__global__ void __launch_bounds__(HT, 1)
hh_panel_kernel(const HhPanelTask* __restrict__ tasks, const int32_t* __restrict__ cta_task) {
    const HhPanelTask T = tasks[cta_task[blockIdx.x]];
    const int g = blockIdx.x - T.cta0, G = T.ncta;
    const int nbp = T.nbp, lds = T.chunk + 4;
    const int64_t Lp = (int64_t)T.L - T.j0;
    const int64_t r0 = (int64_t)g * T.chunk;
    const int rows = (int)min((int64_t)T.chunk, Lp - r0);
    const int rows4 = (rows + 3) & ~3;
    extern __shared__ double S[];  // column jj of the slice at S[jj * lds]
    __shared__ double taus[HH_NB];
    __shared__ double red[HW];
    __shared__ double dsh[HH_NB + 2];
    __shared__ double wsh[HH_NB];
    __shared__ double Tm[HH_NB][HH_NB + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* M0 = T.M + (int64_t)T.j0 * T.ldm + T.j0 + r0;

    for (int jj = 0; jj < HH_NB; ++jj)
        for (int i = threadIdx.x; i < lds; i += HT)
            S[jj * lds + i] = (jj < nbp && i < rows) ? M0[(int64_t)jj * T.ldm + i] : 0.0;
    __syncthreads();

    // One group barrier per column: every CTA publishes, for the rows it owns
    // strictly below the diagonal, ss = |x|^2 and dx_c = x . a_c for the
    // panel columns c > jj (x = column jj before scaling); CTA 0, which owns
    // the panel's diagonal rows, adds alpha = a_jj[jj] and the head row a_c[jj].
    // With beta, tau, scal = 1/(alpha - beta) (dlarfg) the reflector is
    // v = [1; scal x], so v . a_c = a_c[jj] + scal dx_c and w_c = tau v . a_c.
    // Partials: (G + 1) x (HH_NB + 2) per buffer, double-buffered by column
    // parity (a CTA cannot reach column jj + 2 before every CTA has read jj).
    const int PW = HH_NB + 2;
    for (int jj = 0; jj < nbp; ++jj) {
        double* pp = T.part + (int64_t)(jj & 1) * (G + 1) * PW;
        const int lo = (int)max((int64_t)0, (int64_t)(jj + 1) - r0);  // local rows strictly below the diagonal
        // slot 0: ss; slots c (jj < c < nbp): dx_c
        for (int c = jj + warp; c < nbp; c += HW) {
            double d = 0.0;
            if (c == jj)
                for (int i = lo + lane; i < rows; i += 32) d += S[jj * lds + i] * S[jj * lds + i];
            else
                for (int i = lo + lane; i < rows; i += 32) d += S[jj * lds + i] * S[c * lds + i];
            d = warp_sum(d);
            if (lane == 0) pp[(int64_t)g * PW + (c == jj ? 0 : c)] = d;
        }
        if (g == 0)
            for (int c = jj + threadIdx.x; c < nbp; c += HT) pp[(int64_t)G * PW + (c == jj ? 0 : c)] = S[c * lds + jj];
        group_barrier(T.bar, G);
        // fixed-order sums over the CTAs (identical in every CTA)
        for (int c = jj + warp; c < nbp; c += HW) {
            double v = 0.0;
            for (int q = lane; q < G; q += 32) v += __ldcg(pp + (int64_t)q * PW + (c == jj ? 0 : c));
            v = warp_sum(v);
            if (lane == 0) dsh[c] = v;
        }
        if (threadIdx.x == 0) dsh[HH_NB] = __ldcg(pp + (int64_t)G * PW);  // alpha
        __syncthreads();
        double beta, tau, scal;
        hh_reflector(dsh[HH_NB], dsh[jj], beta, tau, scal);
        // w_c = tau (a_c[jj] + scal dx_c) for c > jj (tau is identical in every CTA)
        if (tau != 0.0) {
            for (int c = jj + 1 + threadIdx.x; c < nbp; c += HT)
                wsh[c] = tau * (__ldcg(pp + (int64_t)G * PW + c) + scal * dsh[c]);
            __syncthreads();
            // a_c -= w_c v on the owned rows below the diagonal (v = scal x),
            // then x -> v; CTA 0 also updates the head row
            const int w = nbp - jj - 1;
            for (int e = threadIdx.x; e < w * rows; e += HT) {
                const int c = jj + 1 + e / rows, i = e % rows;
                if (i >= lo) S[c * lds + i] -= wsh[c] * (scal * S[jj * lds + i]);
            }
            if (g == 0)
                for (int c = jj + 1 + threadIdx.x; c < nbp; c += HT) S[c * lds + jj] -= wsh[c];
            __syncthreads();
            for (int i = lo + threadIdx.x; i < rows; i += HT) S[jj * lds + i] *= scal;
        }
        if (threadIdx.x == 0) {
            taus[jj] = tau;
            if (g == 0) S[jj * lds + jj] = beta;
        }
        __syncthreads();
    }

    // write back (R on/above the diagonal, reflectors below) and the explicit
    // unit-lower V^T (HH_NB x Lp); S becomes the explicit V for the Gram
    for (int jj = 0; jj < nbp; ++jj)
        for (int i = threadIdx.x; i < rows; i += HT) {
            const double x = S[jj * lds + i];
            M0[(int64_t)jj * T.ldm + i] = x;
            const int64_t gi = r0 + i;
            const double v = gi < jj ? 0.0 : (gi == jj ? 1.0 : x);
            T.Vt[(int64_t)jj * Lp + gi] = v;
            S[jj * lds + i] = v;
        }
    __syncthreads();
    // partial Gram V^T V over the slice: 16 8x8 DMMA tiles, 2 per warp
    {
        const int gq = lane >> 2, t = lane & 3;
        double* gp = T.gram + (int64_t)g * HH_NB * HH_NB;
        for (int tile = warp; tile < 16; tile += HW) {
            const int ti = tile >> 2, tj = tile & 3;
            double c0 = 0.0, c1 = 0.0;
            const double* A = S + (ti * 8 + gq) * lds;
            const double* B = S + (tj * 8 + gq) * lds;
            for (int k0 = 0; k0 < rows4; k0 += 4) dmma_8x8x4(c0, c1, A[k0 + t], B[k0 + t]);
            gp[(ti * 8 + gq) * HH_NB + tj * 8 + 2 * t] = c0;
            gp[(ti * 8 + gq) * HH_NB + tj * 8 + 2 * t + 1] = c1;
        }
    }
    group_barrier(T.bar, G);
    if (g != 0) return;
    // CTA 0: Gram (fixed-order sum over the slices), then dlarft
    double* Gm = S;  // HH_NB x HH_NB, reuses the slice buffer
    for (int e = threadIdx.x; e < HH_NB * HH_NB; e += HT) {
        const int a = e / HH_NB, b = e % HH_NB;
        double v = 0.0;
        if (a < b && b < nbp)
            for (int q = 0; q < G; ++q) v += __ldcg(T.gram + (int64_t)q * HH_NB * HH_NB + e);
        Gm[e] = v;
    }
    __syncthreads();
    if (warp == 0) {
        for (int j = 0; j < HH_NB; ++j) {
            const double tj = j < nbp ? taus[j] : 0.0;
            double acc = 0.0;
            if (lane < j)
                for (int k = lane; k < j; ++k) acc += Tm[lane][k] * (-tj * Gm[k * HH_NB + j]);
            __syncwarp();
            Tm[lane][j] = lane < j ? acc : (lane == j ? tj : 0.0);
            __syncwarp();
        }
        for (int j = 0; j < HH_NB; ++j) T.T[lane * HH_NB + j] = Tm[lane][j];
    }
}


// ---- thread-block-cluster panel ----------------------------------------------
// The same panel factorization with the panel's CTAs forming ONE thread-block
// cluster (2..16 CTAs, one per SM): the per-column exchange of partial sums
// goes through distributed shared memory and the per-column barrier is the
// cluster barrier (barrier.cluster), instead of global-memory partials and a
// global atomic barrier -- the panel is latency bound (one exchange per
// column), so this is where its time goes.  Rows per CTA <= HH_CLUSTER_CHUNK
// (the slice stays in shared memory).  Clusters are independent, so a launch
// needs no co-residency of all its tasks (no cooperative launch, no waves),
// and a task's result depends only on its own (L, cluster size).
__global__ void __launch_bounds__(HT, 1) hh_panel_cluster_kernel(const HhPanelTask* __restrict__ tasks) {
    cg::cluster_group cluster = cg::this_cluster();
    const int G = int(cluster.num_blocks()), g = int(cluster.block_rank());
    const HhPanelTask T = tasks[blockIdx.x / G];
    const int nbp = T.nbp, lds = T.chunk + 4;
    const int64_t Lp = (int64_t)T.L - T.j0;
    const int64_t r0 = (int64_t)g * T.chunk;
    const int rows = (int)max((int64_t)0, min((int64_t)T.chunk, Lp - r0));
    const int rows4 = (rows + 3) & ~3;
    extern __shared__ double S[];  // column jj of the slice at S[jj * lds]
    __shared__ double taus[HH_NB];
    __shared__ double dsh[HH_NB + 2];
    __shared__ double wsh[HH_NB];
    __shared__ double Tm[HH_NB][HH_NB + 1];
    // this CTA's partials (column parity double buffer): slot 0 = |x|^2,
    // slot c = x . a_c; CTA 0 also publishes alpha (slot 0) and the head row
    __shared__ double cpart[2][HH_NB + 2];
    __shared__ double chead[2][HH_NB + 2];
    __shared__ double cgram[HH_NB * HH_NB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* M0 = T.M + (int64_t)T.j0 * T.ldm + T.j0 + r0;

    for (int jj = 0; jj < HH_NB; ++jj)
        for (int i = threadIdx.x; i < lds; i += HT)
            S[jj * lds + i] = (jj < nbp && i < rows) ? M0[(int64_t)jj * T.ldm + i] : 0.0;
    __syncthreads();

    for (int jj = 0; jj < nbp; ++jj) {
        const int par = jj & 1;
        const int lo = (int)max((int64_t)0, (int64_t)(jj + 1) - r0);  // local rows strictly below the diagonal
        for (int c = jj + warp; c < nbp; c += HW) {
            double d = 0.0;
            if (c == jj)
                for (int i = lo + lane; i < rows; i += 32) d += S[jj * lds + i] * S[jj * lds + i];
            else
                for (int i = lo + lane; i < rows; i += 32) d += S[jj * lds + i] * S[c * lds + i];
            d = warp_sum(d);
            if (lane == 0) cpart[par][c == jj ? 0 : c] = d;
        }
        if (g == 0)
            for (int c = jj + threadIdx.x; c < nbp; c += HT) chead[par][c == jj ? 0 : c] = S[c * lds + jj];
        cluster.sync();
        // fixed-order sums over the cluster's CTAs (identical in every CTA)
        for (int c = jj + warp; c < nbp; c += HW) {
            double v = 0.0;
            for (int q = lane; q < G; q += 32) v += cluster.map_shared_rank(&cpart[par][0], q)[c == jj ? 0 : c];
            v = warp_sum(v);
            if (lane == 0) dsh[c] = v;
        }
        const double* head = cluster.map_shared_rank(&chead[par][0], 0);
        if (threadIdx.x == 0) dsh[HH_NB] = head[0];  // alpha
        __syncthreads();
        double beta, tau, scal;
        hh_reflector(dsh[HH_NB], dsh[jj], beta, tau, scal);
        if (tau != 0.0) {
            for (int c = jj + 1 + threadIdx.x; c < nbp; c += HT) wsh[c] = tau * (head[c] + scal * dsh[c]);
            __syncthreads();
            const int w = nbp - jj - 1;
            for (int e = threadIdx.x; e < w * rows; e += HT) {
                const int c = jj + 1 + e / rows, i = e % rows;
                if (i >= lo) S[c * lds + i] -= wsh[c] * (scal * S[jj * lds + i]);
            }
            if (g == 0)
                for (int c = jj + 1 + threadIdx.x; c < nbp; c += HT) S[c * lds + jj] -= wsh[c];
            __syncthreads();
            for (int i = lo + threadIdx.x; i < rows; i += HT) S[jj * lds + i] *= scal;
        }
        if (threadIdx.x == 0) {
            taus[jj] = tau;
            if (g == 0) S[jj * lds + jj] = beta;
        }
        __syncthreads();
    }

    // write back (R on/above the diagonal, reflectors below) and the explicit
    // unit-lower V^T (HH_NB x Lp); S becomes the explicit V for the Gram
    for (int jj = 0; jj < nbp; ++jj)
        for (int i = threadIdx.x; i < rows; i += HT) {
            const double x = S[jj * lds + i];
            M0[(int64_t)jj * T.ldm + i] = x;
            const int64_t gi = r0 + i;
            const double v = gi < jj ? 0.0 : (gi == jj ? 1.0 : x);
            T.Vt[(int64_t)jj * Lp + gi] = v;
            S[jj * lds + i] = v;
        }
    __syncthreads();
    {
        const int gq = lane >> 2, t = lane & 3;
        for (int tile = warp; tile < 16; tile += HW) {
            const int ti = tile >> 2, tj = tile & 3;
            double c0 = 0.0, c1 = 0.0;
            const double* A = S + (ti * 8 + gq) * lds;
            const double* B = S + (tj * 8 + gq) * lds;
            for (int k0 = 0; k0 < rows4; k0 += 4) dmma_8x8x4(c0, c1, A[k0 + t], B[k0 + t]);
            cgram[(ti * 8 + gq) * HH_NB + tj * 8 + 2 * t] = c0;
            cgram[(ti * 8 + gq) * HH_NB + tj * 8 + 2 * t + 1] = c1;
        }
    }
    cluster.sync();
    if (g == 0) {
        double* Gm = S;  // HH_NB x HH_NB, reuses the slice buffer
        for (int e = threadIdx.x; e < HH_NB * HH_NB; e += HT) {
            const int a = e / HH_NB, b = e % HH_NB;
            double v = 0.0;
            if (a < b && b < nbp)
                for (int q = 0; q < G; ++q) v += cluster.map_shared_rank(cgram, q)[e];
            Gm[e] = v;
        }
        __syncthreads();
        if (warp == 0) {
            for (int j = 0; j < HH_NB; ++j) {
                const double tj = j < nbp ? taus[j] : 0.0;
                double acc = 0.0;
                if (lane < j)
                    for (int k = lane; k < j; ++k) acc += Tm[lane][k] * (-tj * Gm[k * HH_NB + j]);
                __syncwarp();
                Tm[lane][j] = lane < j ? acc : (lane == j ? tj : 0.0);
                __syncwarp();
            }
            for (int j = 0; j < HH_NB; ++j) T.T[lane * HH_NB + j] = Tm[lane][j];
        }
    }
    cluster.sync();  // the other CTAs' shared memory stays live until CTA 0 has read it
}


// ---- block column pivoting -------------------------------------------------
// (1) remaining squared norms of the trailing columns, one warp per column
__global__ void pivot_norms_kernel(const PivotTask* __restrict__ tasks) {
    const PivotTask P = tasks[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int c = P.j0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= P.ntot) return;
    const double* col = P.M + (int64_t)c * P.ldm;
    double s = 0.0;
#pragma unroll 8
    for (int i = P.j0 + lane; i < P.L; i += 32) s += col[i] * col[i];
    s = warp_sum(s);
    if (lane == 0) P.norms[c] = s;
}
// (2) rank sort (descending norm, ties by index): order[rank] = column;
// the permutation composes into perm
__global__ void pivot_rank_kernel(const PivotTask* __restrict__ tasks) {
    const PivotTask P = tasks[blockIdx.x];
    const int nc = P.ntot - P.j0;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        const double v = P.norms[P.j0 + i];
        int r = 0;
        for (int j = 0; j < nc; ++j) {
            const double w = P.norms[P.j0 + j];
            r += (w > v) || (w == v && j < i);
        }
        P.order[r] = i;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nc; i += blockDim.x) P.perm_tmp[i] = P.perm[P.j0 + P.order[i]];
    __syncthreads();
    for (int i = threadIdx.x; i < nc; i += blockDim.x) P.perm[P.j0 + i] = P.perm_tmp[i];
}
// (3) the job's matrix in its new column order into the other buffer (tmp,
// same ldm): trailing columns whole, in the new order; the factored columns
// [0, j0) only their R rows [0, j0) (their reflectors live in Vt) -- the
// caller then swaps the two buffers
__global__ void pivot_gather_kernel(const PivotTask* __restrict__ tasks) {
    const PivotTask P = tasks[blockIdx.z];
    const int c = blockIdx.y;
    if (c >= P.ntot) return;
    const bool done = c < P.j0;
    const double* src = P.M + (int64_t)(done ? c : P.j0 + P.order[c - P.j0]) * P.ldm;
    double* dst = P.tmp + (int64_t)c * P.ldm;
    const int rows = done ? P.j0 : P.L;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void iota_kernel(int32_t* p, int32_t n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}
__global__ void unpermute_rows_kernel(const UnpermTask* __restrict__ tasks, int phase) {
    const UnpermTask T = tasks[blockIdx.y];
    const int64_t tot = (int64_t)T.m * T.n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        if (phase == 0) {
            T.tmp[e] = T.U[e];
        } else {
            const int64_t j = e / T.n, i = e % T.n;
            T.U[j * T.n + T.perm[i]] = T.tmp[e];
        }
    }
}

// out[a][c] = sum_b op(T)[a][b] * (sum_ch P[ch][b][c]),  op(T) = T^T (trans) or T
// 32 columns per CTA, 8 row-threads: the split-K partial sums of the 32 x 32
// block S are formed with independent loads (4 rows per thread), then T (or
// T^T) is applied from shared memory
constexpr int TM_COLS = 32, TM_ROWS = 8;
__global__ void __launch_bounds__(TM_COLS * TM_ROWS) hh_tmul_kernel(const HhTmulTask* __restrict__ tasks) {
    const HhTmulTask R = tasks[blockIdx.y];
    __shared__ double Ssh[HH_NB][TM_COLS + 1];
    __shared__ double Tsh[HH_NB][HH_NB + 1];
    const int cx = threadIdx.x % TM_COLS, ty = threadIdx.x / TM_COLS;
    const int c0 = blockIdx.x * TM_COLS;
    if (c0 >= R.ncols) return;
    const int c = c0 + cx;
    for (int e = threadIdx.x; e < HH_NB * HH_NB; e += TM_COLS * TM_ROWS) Tsh[e / HH_NB][e % HH_NB] = R.T[e];
#pragma unroll
    for (int q = 0; q < HH_NB / TM_ROWS; ++q) {
        const int b = ty + q * TM_ROWS;
        double v = 0.0;
        if (c < R.ncols && b < R.nrows)
            for (int ch = 0; ch < R.nchunks; ++ch) v += R.P[((int64_t)ch * R.nrows + b) * R.ncols + c];
        Ssh[b][cx] = v;
    }
    __syncthreads();
    if (c >= R.ncols) return;
#pragma unroll
    for (int q = 0; q < HH_NB / TM_ROWS; ++q) {
        const int a = ty + q * TM_ROWS;
        if (a >= R.nrows) continue;
        double acc = 0.0;
        if (R.trans) {
            for (int b = 0; b <= a; ++b) acc += Tsh[b][a] * Ssh[b][cx];
        } else {
            for (int b = a; b < HH_NB; ++b) acc += Tsh[a][b] * Ssh[b][cx];
        }
        R.out[(int64_t)a * R.ncols + c] = acc;
    }
}

// X[kt + i][i] = 1 (the [0; I] seed of the complement columns); X pre-zeroed
__global__ void set_eye_kernel(const EyeTask* __restrict__ tasks) {
    const EyeTask E = tasks[blockIdx.y];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < E.n) E.X[(int64_t)(E.row0 + i) * E.ldx + i] = 1.0;
}

}  // namespace

size_t hh_panel_smem(int chunk) { return sizeof(double) * size_t(HH_NB) * (chunk + 4); }

int hh_panel_capacity(int chunk) {
    static int cached_chunk = -1, cached = 0;
    if (chunk == cached_chunk) return cached;
    const size_t smem = hh_panel_smem(chunk);
    cudaFuncSetAttribute(hh_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hh_panel_kernel, HT, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached_chunk = chunk;
    cached = per_sm * sms;
    return cached;
}

cudaError_t launch_hh_panel(const HhPanelTask* d_tasks, const int32_t* d_cta_task, int32_t total_ctas,
                            int32_t max_chunk, cudaStream_t st) {
    if (total_ctas <= 0) return cudaSuccess;
    const size_t smem = hh_panel_smem(max_chunk);
    cudaFuncSetAttribute(hh_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    void* args[] = {(void*)&d_tasks, (void*)&d_cta_task};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)hh_panel_kernel, dim3(total_ctas), dim3(HT), args,
                                                smem, st);
    count_launch();
    return e;  // never falls back to a plain launch: the group barriers need co-residency
}

cudaError_t launch_hh_panel_cluster(const HhPanelTask* d_tasks, int32_t ntasks, int32_t cluster, int32_t chunk,
                                    cudaStream_t st) {
    if (ntasks <= 0) return cudaSuccess;
    const size_t smem = hh_panel_smem(chunk);
    cudaFuncSetAttribute(hh_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(hh_panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(ntasks) * unsigned(cluster));
    cfg.blockDim = dim3(HT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(cluster);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, hh_panel_cluster_kernel, d_tasks);
    count_launch();
    return e;
}

void launch_pivot_panel(const PivotTask* d_tasks, int32_t ntasks, int32_t max_cols, int32_t max_l,
                        cudaStream_t st) {
    if (ntasks <= 0 || max_cols <= 0) return;
    pivot_norms_kernel<<<dim3((max_cols + 7) / 8, ntasks), 256, 0, st>>>(d_tasks);
    pivot_rank_kernel<<<ntasks, 512, 0, st>>>(d_tasks);
    const int gx = (max_l + 255) / 256;
    pivot_gather_kernel<<<dim3(gx, max_cols, ntasks), 256, 0, st>>>(d_tasks);
    for (int i = 0; i < 3; ++i) count_launch();
}

void launch_iota(int32_t* p, int32_t n, cudaStream_t st) {
    if (n <= 0) return;
    iota_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, n);
    count_launch();
}

void launch_unpermute_rows(const UnpermTask* d_tasks, int32_t ntasks, int32_t max_mn, cudaStream_t st) {
    if (ntasks <= 0 || max_mn <= 0) return;
    const dim3 grid(std::min(1024, (max_mn + 255) / 256), ntasks);
    unpermute_rows_kernel<<<grid, 256, 0, st>>>(d_tasks, 0);
    unpermute_rows_kernel<<<grid, 256, 0, st>>>(d_tasks, 1);
    count_launch();
    count_launch();
}

void launch_hh_tmul(const HhTmulTask* d_tasks, int32_t ntasks, int32_t max_cols, cudaStream_t st) {
    if (ntasks <= 0 || max_cols <= 0) return;
    dim3 grid((max_cols + TM_COLS - 1) / TM_COLS, ntasks);
    hh_tmul_kernel<<<grid, TM_COLS * TM_ROWS, 0, st>>>(d_tasks);
    count_launch();
}

void launch_set_eye(const EyeTask* d_tasks, int32_t ntasks, int32_t max_n, cudaStream_t st) {
    if (ntasks <= 0 || max_n <= 0) return;
    dim3 grid((max_n + 127) / 128, ntasks);
    set_eye_kernel<<<grid, 128, 0, st>>>(d_tasks);
    count_launch();
}

}  // namespace h2f
