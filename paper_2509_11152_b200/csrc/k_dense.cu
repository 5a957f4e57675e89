// Per-cluster dense linear algebra, batched: one CTA per cluster of a batch.
//
//   qr_r_smem   R of the reduced Householder QR of Y^T (Y = fill residual)   factorization.py:78
//   jacobi      one-sided Jacobi SVD of R^T, kept count, re-orthogonalised
//               new directions -> b_aug^T                                     factorization.py:79-84
//   complement  complete Householder QR of b_aug -> Q~ = [complement|b_aug]   factorization.py:88-99
//   lu          partial-pivot LU of D_RR + vanishing-pivot test              factorization.py:112-116
//   trsm        MW = -(LU)^-1 P G  (the stored eliminators -W)               factorization.py:117-121
//   panel LU / swaps / unit-lower TRSM for the blocked dense top LU          factorization.py:259-263
//
// Working matrices live in global memory (L1/L2 resident at these sizes) and
// are updated with CTA-wide barriers; reductions use a fixed order so the
// results are run-to-run deterministic.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace h2f {

namespace {

constexpr int DT = 512;  // threads per CTA for the dense kernels

// LAPACK dlarfg-style reflector for x = [alpha, rest]; ss = ||rest||^2.
__device__ __forceinline__ void reflector(double alpha, double ss, double& beta, double& tau,
                                          double& scal) {
    if (ss == 0.0) {
        beta = alpha;
        tau = 0.0;
        scal = 0.0;
    } else {
        const double xnorm = sqrt(ss);
        beta = -copysign(hypot(alpha, xnorm), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
    }
}

// ---- sequential TSQR in shared memory ---------------------------------------
// R of the QR of Z^T (Z is n x wf, row-major): R (n x n) stays in shared
// memory and absorbs Z^T 32 rows (= 32 columns of Z) at a time, one row per
// lane, by Householder reflectors of length 33 on the stacked [R; chunk].
constexpr int QB = 32;

__global__ void __launch_bounds__(DT) qr_r_smem_kernel(const QrTask* __restrict__ tasks) {
    const QrTask T = tasks[blockIdx.x];
    extern __shared__ double sm[];
    const int n = T.s, wf = T.c1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = DT / 32;
    double* R = sm;              // n x n
    double* Cc = sm + n * n;     // chunk, column c at Cc[c*QB + i]
    double* vt = Cc + n * QB;    // tau broadcast
    for (int e = threadIdx.x; e < n * n; e += DT) R[e] = 0.0;
    for (int col0 = T.c0; col0 < wf; col0 += QB) {
        __syncthreads();
        for (int e = threadIdx.x; e < n * QB; e += DT) {
            const int c = e / QB, i = e % QB;
            Cc[e] = (col0 + i < wf) ? T.Y[(int64_t)c * T.ldy + col0 + i] : 0.0;
        }
        __syncthreads();
        for (int j = 0; j < n; ++j) {
            if (warp == 0) {
                const double x = Cc[j * QB + lane];
                const double ss = warp_sum(x * x);
                double beta, tau, scal;
                reflector(R[j * n + j], ss, beta, tau, scal);
                if (tau != 0.0) Cc[j * QB + lane] = x * scal;
                if (lane == 0) {
                    R[j * n + j] = beta;
                    vt[0] = tau;
                }
            }
            __syncthreads();
            const double tau = vt[0];
            if (tau != 0.0) {
                const double v = Cc[j * QB + lane];
                for (int c = j + 1 + warp; c < n; c += nw) {
                    const double y = Cc[c * QB + lane];
                    double d = warp_sum(v * y) + R[j * n + c];
                    d *= tau;
                    Cc[c * QB + lane] = y - d * v;
                    if (lane == 0) R[j * n + c] -= d;
                }
            }
            __syncthreads();
        }
    }
    __syncthreads();
    if (T.ldrt > 0) {
        for (int e = threadIdx.x; e < n * n; e += DT) {
            const int j = e / n, c = e % n;
            T.R[(int64_t)c * T.ldrt + j] = R[e];
        }
    } else {
        for (int e = threadIdx.x; e < n * n; e += DT) T.R[e] = R[e];
    }
}

// A sweep whose rotations all had |cos angle(x_p, x_q)| <= 1e-7 leaves the rows
// orthogonal to O(1e-14) (quadratic convergence), below the rotation
// threshold tol = eps sqrt(n) of a further sweep: such a sweep ends the
// iteration instead of a final sweep that would rotate nothing.  The rotate
// helpers return 0 (no rotation), 1 (settling rotation) or 2 (rotation with
// |cos| > 1e-7, another sweep is needed).
#ifndef H2F_JAC_SETTLE2
#define H2F_JAC_SETTLE2 1e-14
#endif
constexpr double JAC_SETTLE2 = H2F_JAC_SETTLE2;

// Jacobi rotation annihilating the (p, q) inner product: a = |x_p|^2,
// b = |x_q|^2, g = x_p.x_q.  Rotate iff |g| > tol sqrt(a b) (tested
// squared); t = tan(theta) = sgn(d) 2g / (|d| + sqrt(d^2 + 4 g^2)), d = b - a
// (the Rutishauser formula without the zeta division): one sqrt, one
// division and one rsqrt per rotation.
__device__ __forceinline__ bool jac_rotation(double a, double b, double g, double tol, double& c, double& sn) {
    if (!(g != 0.0 && a > 0.0 && b > 0.0 && g * g > (tol * tol) * (a * b))) return false;
    const double d = b - a;
    const double t = (d >= 0.0 ? 2.0 * g : -2.0 * g) / (fabs(d) + sqrt(d * d + 4.0 * g * g));
    c = rsqrt(1.0 + t * t);
    sn = c * t;
    return true;
}

// Row pair rotation with cached squared norms (a = |x|^2, b = |y|^2 on entry,
// updated on exit): one dot product per pair instead of three.  After the
// rotation the exact identities a' = a - t g, b' = b + t g hold; a norm that
// shrinks below 1/64 of its old value is recomputed from the rotated row (the
// update would lose relative accuracy to cancellation, cf. LAPACK dgesvj).
// One warp per pair; a and b are warp-uniform.
__device__ __forceinline__ int jac_rotate_cached(double* __restrict__ x, double* __restrict__ y, int n, double tol,
                                                 double& a, double& b) {
    const int lane = threadIdx.x & 31;
    double g = 0.0;
    for (int i = lane; i < n; i += 32) g += x[i] * y[i];
    g = warp_sum(g);
    if (!(g != 0.0 && a > 0.0 && b > 0.0 && g * g > (tol * tol) * (a * b))) return 0;
    const int code = g * g > JAC_SETTLE2 * (a * b) ? 2 : 1;
    const double d = b - a;
    const double t = (d >= 0.0 ? 2.0 * g : -2.0 * g) / (fabs(d) + sqrt(d * d + 4.0 * g * g));
    const double c = rsqrt(1.0 + t * t), sn = c * t;
    for (int i = lane; i < n; i += 32) {
        const double u = x[i], v = y[i];
        x[i] = c * u - sn * v;
        y[i] = sn * u + c * v;
    }
    double a2 = a - t * g, b2 = b + t * g;
    // the FP64 pipe bounds this loop: the norms are recomputed from the rotated
    // rows (a second pass) only when the update formula loses accuracy
    const bool ra = !(a2 >= a * (1.0 / 64.0)), rb = !(b2 >= b * (1.0 / 64.0));
    if (ra | rb) {
        __syncwarp();
        double ax = 0.0, by = 0.0;
        for (int i = lane; i < n; i += 32) {
            ax += x[i] * x[i];
            by += y[i] * y[i];
        }
        if (ra) a2 = warp_sum(ax);
        if (rb) b2 = warp_sum(by);
    }
    a = a2;
    b = b2;
    return code;
}

// circle-method round robin: player list [0, rot...]; pair i of round st
__device__ __forceinline__ void rr_pair(int i, int st, int mm, int& p, int& q) {
    auto pos = [&](int j) { return j == 0 ? 0 : 1 + ((j - 1 + st) % (mm - 1)); };
    p = pos(i);
    q = pos(mm - 1 - i);
}

// one-sided (Hestenes) Jacobi on the m rows (length n) of A, in place
__device__ void jacobi_sweeps(double* A, int m, int n, int* flag, double* nrm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const double tol = 2.220446049250313e-16 * sqrt((double)n);
    const int mm = m + (m & 1);
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (threadIdx.x == 0) *flag = 0;
        // exact squared row norms at the start of every sweep (no drift)
        for (int i = warp; i < m; i += nw) {
            const double* ri = A + (int64_t)i * n;
            double v = 0.0;
            for (int c = lane; c < n; c += 32) v += ri[c] * ri[c];
            v = warp_sum(v);
            if (lane == 0) nrm[i] = v;
        }
        __syncthreads();
        for (int st = 0; st < mm - 1; ++st) {
            for (int pi = warp; pi < mm / 2; pi += nw) {
                int p, q;
                rr_pair(pi, st, mm, p, q);
                if (p >= m || q >= m) continue;
                double a = nrm[p], b = nrm[q];
                const int rc = jac_rotate_cached(A + (int64_t)p * n, A + (int64_t)q * n, n, tol, a, b);
                if (rc) {
                    __syncwarp();  // every lane has read nrm[p], nrm[q] before lane 0 rewrites them
                    if (lane == 0) {
                        nrm[p] = a;
                        nrm[q] = b;
                        if (rc == 2) *flag = 1;
                    }
                }
                __syncwarp();
            }
            __syncthreads();
        }
        const int any = *flag;
        __syncthreads();
        if (!any) break;
    }
}

// below this a singular value counts as zero: its row cannot be normalised
constexpr double JAC_TINY = 1e-290;
// Rows whose sigma is below JAC_RANK_REL * sigma_max carry rounding noise of R,
// not a direction: when R is numerically rank deficient (e.g. exact zero
// columns from structurally zero fill rows) such rows are not orthogonal to
// the others, so the sorted rows are not an orthonormal completion and the
// caller must fall back to the Householder complement (deg flag).
constexpr double JAC_RANK_REL = 1e-12;

// sigma_max over sig[0..m) (warp-reduced, every lane of every warp)
__device__ __forceinline__ double sig_max(const double* sig, int m) {
    double v = 0.0;
    for (int j = threadIdx.x & 31; j < m; j += 32) v = fmax(v, sig[j]);
    return warp_max(v);
}

// sigma = row norms, count sigma >= thresh, write all m rows normalised in
// descending sigma order (first index wins ties): rows 0..kept-1 are the kept
// left singular vectors, the rest complete them to an orthonormal basis when
// m == n and no sigma is ~0 (otherwise kept_out[deg_off] is set)
__device__ void jacobi_finish(const double* A, int m, int n, double thresh, double* sig, int* rnk,
                              int* kept_s, double* U, int* kept_out, int deg_off) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = warp; i < m; i += nw) {
        const double* ri = A + (int64_t)i * n;
        double a = 0.0;
        for (int c = lane; c < n; c += 32) a += ri[c] * ri[c];
        a = warp_sum(a);
        if (lane == 0) sig[i] = sqrt(a);
    }
    if (threadIdx.x == 0) *kept_s = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        int r = 0;
        const double si = sig[i];
        for (int j = 0; j < m; ++j) r += (sig[j] > si) || (sig[j] == si && j < i);
        rnk[i] = r;
        if (si >= thresh) atomicAdd(kept_s, 1);
    }
    __syncthreads();
    const int kept = *kept_s;
    if (threadIdx.x == 0) *kept_out = kept;
    (void)kept;
    const double smax = sig_max(sig, m);
    for (int i = warp; i < m; i += nw) {
        const int j = rnk[i];
        const double si = sig[i];
        if (!(si > JAC_TINY && si > JAC_RANK_REL * smax) && deg_off && lane == 0) kept_out[deg_off] = 1;
        const double inv = si > JAC_TINY ? 1.0 / si : 0.0;
        const double* ri = A + (int64_t)i * n;
        for (int c = lane; c < n; c += 32) U[(int64_t)j * n + c] = ri[c] * inv;
    }
}

__global__ void __launch_bounds__(DT) jacobi_smem_kernel(const SvdTask* __restrict__ tasks, double thresh) {
    const SvdTask T = tasks[blockIdx.x];
    extern __shared__ double dsh[];  // A[m*n], sig[m], rank[m]
    __shared__ int flag, kept_s;
    const int m = T.m, n = T.n;
    if (m == 0) {
        if (threadIdx.x == 0) *T.kept_out = 0;
        return;
    }
    double* A = dsh;
    for (int e = threadIdx.x; e < m * n; e += DT) A[e] = T.R[e];
    __syncthreads();
    jacobi_sweeps(A, m, n, &flag, A + m * n + 2 * m);  // after sig[m], rank[m]
    jacobi_finish(A, m, n, thresh, A + m * n, reinterpret_cast<int*>(A + m * n + m), &kept_s, T.U,
                  T.kept_out, T.deg_off);
}

// rows k..k+kept-1 of BT: re-orthogonalise against V and normalise
// (factorization.py:82-84)
__global__ void __launch_bounds__(DT) reorth_kernel(const ReorthTask* __restrict__ tasks) {
    const ReorthTask T = tasks[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = DT / 32;
    const int s = T.s, k = T.k, kept = T.kept;
    for (int64_t e = warp; e < (int64_t)k * kept; e += nw) {
        const int l = (int)(e / kept), j = (int)(e % kept);
        const double* u = T.BT + (int64_t)(k + j) * s;
        double d = 0.0;
        for (int i = lane; i < s; i += 32) d += T.V[(int64_t)i * T.ldv + l] * u[i];
        d = warp_sum(d);
        if (lane == 0) T.C[e] = d;
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)kept * s; e += DT) {
        const int j = (int)(e / s), i = (int)(e % s);
        double d = 0.0;
        for (int l = 0; l < k; ++l) d += T.V[(int64_t)i * T.ldv + l] * T.C[(int64_t)l * kept + j];
        T.BT[(int64_t)(k + j) * s + i] -= d;
    }
    __syncthreads();
    for (int j = warp; j < kept; j += nw) {
        double* u = T.BT + (int64_t)(k + j) * s;
        double a = 0.0;
        for (int i = lane; i < s; i += 32) a += u[i] * u[i];
        a = warp_sum(a);
        const double inv = 1.0 / sqrt(a);
        for (int i = lane; i < s; i += 32) u[i] *= inv;
    }
}

// u /= |u| per row, warp per row, fixed lane-strided summation order
__global__ void __launch_bounds__(256) normalize_rows_kernel(const RowNormTask* __restrict__ tasks, int nrows) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= nrows) return;
    const RowNormTask T = tasks[w];
    double a = 0.0;
    for (int i = lane; i < T.len; i += 32) a += T.p[i] * T.p[i];
    a = warp_sum(a);
    const double inv = 1.0 / sqrt(a);
    for (int i = lane; i < T.len; i += 32) T.p[i] *= inv;
}

__global__ void __launch_bounds__(DT) complement_kernel(const ComplementTask* __restrict__ tasks) {
    const ComplementTask T = tasks[blockIdx.x];
    extern __shared__ double taus[];  // [s]
    __shared__ double sh[DT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = DT / 32;
    const int s = T.s;
    const int kt = T.kt;
    const int r = s - kt;
    for (int64_t e = threadIdx.x; e < (int64_t)kt * s; e += DT) T.W[e] = T.BT[e];
    __syncthreads();
    for (int j = 0; j < kt; ++j) {
        double* wj = T.W + (int64_t)j * s;
        double ss = 0.0;
        for (int i = j + 1 + threadIdx.x; i < s; i += DT) ss += wj[i] * wj[i];
        ss = block_sum(ss, sh);
        double beta, tau, scal;
        reflector(wj[j], ss, beta, tau, scal);
        if (tau != 0.0)
            for (int i = j + 1 + threadIdx.x; i < s; i += DT) wj[i] *= scal;
        if (threadIdx.x == 0) taus[j] = tau;
        __syncthreads();
        if (tau != 0.0) {
            for (int c = j + 1 + warp; c < kt; c += nw) {
                double* wc = T.W + (int64_t)c * s;
                double d = 0.0;
                for (int i = j + 1 + lane; i < s; i += 32) d += wj[i] * wc[i];
                d = (warp_sum(d) + wc[j]) * tau;
                for (int i = j + 1 + lane; i < s; i += 32) wc[i] -= d * wj[i];
                __syncwarp();
                if (lane == 0) wc[j] -= d;
            }
        }
        __syncthreads();
    }
    // complement columns Q[:, kt + i] = H_0 ... H_{kt-1} e_{kt+i}
    double* q = T.scratch + (int64_t)warp * s;
    for (int i = warp; i < r; i += nw) {
        for (int l = lane; l < s; l += 32) q[l] = (l == kt + i) ? 1.0 : 0.0;
        __syncwarp();
        for (int j = kt - 1; j >= 0; --j) {
            const double tau = taus[j];
            if (tau == 0.0) continue;
            const double* wj = T.W + (int64_t)j * s;
            double d = 0.0;
            for (int l = j + 1 + lane; l < s; l += 32) d += wj[l] * q[l];
            d = (warp_sum(d) + q[j]) * tau;
            for (int l = j + 1 + lane; l < s; l += 32) q[l] -= d * wj[l];
            __syncwarp();
            if (lane == 0) q[j] -= d;
            __syncwarp();
        }
        for (int l = lane; l < s; l += 32) T.Q[(int64_t)l * s + i] = q[l];
        __syncwarp();
    }
    // trailing columns: b_aug itself
    for (int64_t e = threadIdx.x; e < (int64_t)kt * s; e += DT) {
        const int c = (int)(e / s), row = (int)(e % s);
        T.Q[(int64_t)row * s + r + c] = T.BT[e];
    }
}

__global__ void r_extract_kernel(const RExtractTask* __restrict__ tasks) {
    const RExtractTask X = tasks[blockIdx.y];
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)X.n * X.n) return;
    const int j = (int)(e / X.n), c = (int)(e % X.n);
    X.R[e] = (j < X.m && c >= j) ? X.Z[(int64_t)c * X.ldz + j] : 0.0;
}

// ---- multi-CTA Jacobi (large n) ---------------------------------------------
// CTAs [cta0, cta0+ncta) of the grid own one cluster; each round-robin step's
// pairs are spread over all their warps (one pair per warp), with a group
// barrier between steps.  A warp holds its pair's two rows in registers
// (NPL doubles per lane, all loads issued at once), so a rotation costs one
// L2 round trip; loads/stores bypass L1 (other SMs write the rows).  The
// arithmetic (lane-strided partial sums, butterfly reduction) is the same as
// the shared-memory kernel's.
__device__ __forceinline__ void cta_group_barrier(uint32_t* bar, int nct) {
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
        const uint32_t target = (old / uint32_t(nct) + 1u) * uint32_t(nct);
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

constexpr int JT = 256;  // threads per CTA of the multi-CTA Jacobi

__device__ __forceinline__ int jac_pair_loop(double* __restrict__ rp, double* __restrict__ rq, int n, double tol) {
    const int lane = threadIdx.x & 31;
    double a = 0.0, b = 0.0, g = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double x = __ldcg(rp + i), y = __ldcg(rq + i);
        a += x * x;
        b += y * y;
        g += x * y;
    }
    a = warp_sum(a);
    b = warp_sum(b);
    g = warp_sum(g);
    double c, sn;
    if (!jac_rotation(a, b, g, tol, c, sn)) return 0;
    for (int i = lane; i < n; i += 32) {
        const double x = __ldcg(rp + i), y = __ldcg(rq + i);
        __stcg(rp + i, c * x - sn * y);
        __stcg(rq + i, sn * x + c * y);
    }
    return g * g > JAC_SETTLE2 * (a * b) ? 2 : 1;
}

template <int NPL>
__device__ __forceinline__ int jac_pair_reg(double* __restrict__ rp, double* __restrict__ rq, int n, double tol) {
    if constexpr (NPL == 0) return jac_pair_loop(rp, rq, n, tol);
    const int lane = threadIdx.x & 31;
    double x[NPL > 0 ? NPL : 1], y[NPL > 0 ? NPL : 1];
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        const int i = lane + 32 * k;
        x[k] = i < n ? __ldcg(rp + i) : 0.0;
        y[k] = i < n ? __ldcg(rq + i) : 0.0;
    }
    double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        a += x[k] * x[k];
        b += y[k] * y[k];
        g += x[k] * y[k];
    }
    a = warp_sum(a);
    b = warp_sum(b);
    g = warp_sum(g);
    double c, sn;
    if (!jac_rotation(a, b, g, tol, c, sn)) return 0;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        const int i = lane + 32 * k;
        if (i < n) {
            __stcg(rp + i, c * x[k] - sn * y[k]);
            __stcg(rq + i, sn * x[k] + c * y[k]);
        }
    }
    return g * g > JAC_SETTLE2 * (a * b) ? 2 : 1;
}

template <int NPL>
__device__ __forceinline__ double row_norm_reg(const double* __restrict__ r, int n) {
    const int lane = threadIdx.x & 31;
    if constexpr (NPL == 0) {
        double a = 0.0;
        for (int i = lane; i < n; i += 32) {
            const double x = __ldcg(r + i);
            a += x * x;
        }
        return sqrt(warp_sum(a));
    }
    double x[NPL > 0 ? NPL : 1];
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
        const int i = lane + 32 * k;
        x[k] = i < n ? __ldcg(r + i) : 0.0;
    }
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < NPL; ++k) a += x[k] * x[k];
    return sqrt(warp_sum(a));
}

template <int NPL>
__global__ void __launch_bounds__(JT, 1) jacobi_coop_kernel(const CoopSvdTask* __restrict__ tasks,
                                                           const int* __restrict__ cta_task, double thresh) {
    const CoopSvdTask CT = tasks[cta_task[blockIdx.x]];
    const int rank = blockIdx.x - CT.cta0, nct = CT.ncta;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = JT / 32;
    const int m = CT.t.m, n = CT.t.n;
    double* A = CT.t.R;
    extern __shared__ double dsh[];  // sig[m]
    __shared__ int kept_s;
    if (m == 0) {
        if (rank == 0 && threadIdx.x == 0) *CT.t.kept_out = 0;
        return;
    }
    const double tol = 2.220446049250313e-16 * sqrt((double)n);
    const int mm = m + (m & 1);
    const int gw = rank * nw + warp, gnw = nct * nw;
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int st = 0; st < mm - 1; ++st) {
            for (int pi = gw; pi < mm / 2; pi += gnw) {
                int p, q;
                rr_pair(pi, st, mm, p, q);
                if (p >= m || q >= m) continue;
                rotated |= jac_pair_reg<NPL>(A + (int64_t)p * n, A + (int64_t)q * n, n, tol) == 2;
            }
            cta_group_barrier(CT.bar, nct);
        }
        if (rotated && lane == 0) CT.flags[sweep] = 1;
        cta_group_barrier(CT.bar, nct);
        const int any = __ldcg(CT.flags + sweep);
        if (rank == 0 && threadIdx.x == 0) CT.flags[63] = sweep + 1;
        if (!any) break;
    }
    // sigma (row norms) of this CTA's rows, shared through global memory
    for (int i = gw; i < m; i += gnw) {
        const double sg = row_norm_reg<NPL>(A + (int64_t)i * n, n);
        if (lane == 0) CT.sig[i] = sg;
    }
    cta_group_barrier(CT.bar, nct);
    for (int i = threadIdx.x; i < m; i += JT) dsh[i] = __ldcg(CT.sig + i);
    if (threadIdx.x == 0) kept_s = 0;
    __syncthreads();
    int cnt = 0;
    for (int i = threadIdx.x; i < m; i += JT) cnt += dsh[i] >= thresh;
    atomicAdd(&kept_s, cnt);
    __syncthreads();
    const int kept = kept_s;
    if (rank == 0 && threadIdx.x == 0) *CT.t.kept_out = kept;
    const double smax = sig_max(dsh, m);
    // all rows, normalised, in descending sigma order (first index wins ties)
    for (int i = gw; i < m; i += gnw) {
        const double si = dsh[i];
        int r = 0;
        for (int j = lane; j < m; j += 32) r += (dsh[j] > si) || (dsh[j] == si && j < i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        (void)kept;
        if (!(si > JAC_TINY && si > JAC_RANK_REL * smax) && CT.t.deg_off && lane == 0)
            CT.t.kept_out[CT.t.deg_off] = 1;
        const double inv = si > JAC_TINY ? 1.0 / si : 0.0;
        const double* ri = A + (int64_t)i * n;
        for (int c = lane; c < n; c += 32) CT.t.U[(int64_t)r * n + c] = __ldcg(ri + c) * inv;
    }
}

constexpr int JBT = 512;  // threads per CTA of the block-cyclic Jacobi

// jac_rotate_cached with the row pair split over W warps (a named barrier of
// 32*W threads per pair group, id 1 + grp): each warp owns a contiguous
// slice of the rows, the dot products are summed over the slices in a fixed
// order through `red` (double-buffered by the group's call parity `par`).
template <int W>
__device__ __forceinline__ int jac_rotate_split(double* __restrict__ x, double* __restrict__ y, int n, double tol,
                                                double& a, double& b, int grp, int sub, double* red, int& par) {
    if (W == 1) return jac_rotate_cached(x, y, n, tol, a, b);
    const int lane = threadIdx.x & 31;
    const int len = (n + W - 1) / W, i0 = sub * len, i1 = min(n, i0 + len);
    auto group_sum = [&](double v) {
        v = warp_sum(v);
        double* slot = red + (grp * 2 + par) * W;
        if (lane == 0) slot[sub] = v;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * W) : "memory");
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) t += slot[w];
        par ^= 1;
        return t;
    };
    double g = 0.0;
    for (int i = i0 + lane; i < i1; i += 32) g += x[i] * y[i];
    g = group_sum(g);
    if (!(g != 0.0 && a > 0.0 && b > 0.0 && g * g > (tol * tol) * (a * b))) return 0;
    const int code = g * g > JAC_SETTLE2 * (a * b) ? 2 : 1;
    const double d = b - a;
    const double t = (d >= 0.0 ? 2.0 * g : -2.0 * g) / (fabs(d) + sqrt(d * d + 4.0 * g * g));
    const double c = rsqrt(1.0 + t * t), sn = c * t;
    for (int i = i0 + lane; i < i1; i += 32) {
        const double u = x[i], v = y[i];
        x[i] = c * u - sn * v;
        y[i] = sn * u + c * v;
    }
    double a2 = a - t * g, b2 = b + t * g;
    // rare exact recompute (second pass over the slice), uniform over the group
    const bool ra = !(a2 >= a * (1.0 / 64.0)), rb = !(b2 >= b * (1.0 / 64.0));
    if (ra | rb) {
        __syncwarp();
        double ax = 0.0, by = 0.0;
        for (int i = i0 + lane; i < i1; i += 32) {
            ax += x[i] * x[i];
            by += y[i] * y[i];
        }
        if (ra) a2 = group_sum(ax);
        if (rb) b2 = group_sum(by);
    }
    a = a2;
    b = b2;
    return code;
}

// ---- block-cyclic multi-CTA Jacobi ----------------------------------------------
// The m rows are cut into 2P blocks of JB rows; P co-resident CTAs play a
// round-robin tournament over the blocks.  In one block step a CTA stages its
// two blocks in shared memory and applies all JB x JB cross rotations (JB
// inner steps of JB disjoint pairs, one warp per pair, __syncthreads between
// inner steps), plus, at the first block step of a sweep, the rotations
// inside each of its blocks; then the blocks go back to global memory and
// the CTAs meet at one group barrier.  Every pair of rows is visited once
// per sweep (a block-cyclic ordering), with one group barrier per JB^2
// rotations instead of one per row pair.
__device__ __forceinline__ bool jac_rotate_smem(double* __restrict__ x, double* __restrict__ y, int n, double tol) {
    const int lane = threadIdx.x & 31;
    double a = 0.0, b = 0.0, g = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double u = x[i], v = y[i];
        a += u * u;
        b += v * v;
        g += u * v;
    }
    a = warp_sum(a);
    b = warp_sum(b);
    g = warp_sum(g);
    double c, sn;
    if (!jac_rotation(a, b, g, tol, c, sn)) return false;
    for (int i = lane; i < n; i += 32) {
        const double u = x[i], v = y[i];
        x[i] = c * u - sn * v;
        y[i] = sn * u + c * v;
    }
    return true;
}

template <int JB>
__global__ void __launch_bounds__(JBT, 1) jacobi_block_kernel(const CoopSvdTask* __restrict__ tasks,
                                                            const int* __restrict__ cta_task, double thresh) {
    const CoopSvdTask CT = tasks[cta_task[blockIdx.x]];
    const int rank = blockIdx.x - CT.cta0, P = CT.ncta, NB2 = 2 * CT.ncta;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = JBT / 32;
    const int m = CT.t.m, n = CT.t.n;
    double* A = CT.t.R;
    extern __shared__ double bsm[];  // 2*JB rows of n; after the sweeps: sig[m]
    __shared__ int kept_s;
    __shared__ int rot_s;
    __shared__ double bn[2 * JB];  // squared norms of the staged rows
    constexpr int WPP = (JBT / 32) / JB;  // warps per row pair (JB pairs per round)
    __shared__ double red[JB * 2 * WPP];
    const int grp = warp / WPP, sub = warp % WPP;
    int par = 0;
    if (m == 0) {
        if (rank == 0 && threadIdx.x == 0) *CT.t.kept_out = 0;
        return;
    }
    const double tol = 2.220446049250313e-16 * sqrt((double)n);
    // rows of block j: [j*JB, min((j+1)*JB, m)); smem row r (0..2JB) <-> block (r < JB ? bp : bq)
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (threadIdx.x == 0) rot_s = 0;
        bool rotated = false;
        for (int st = 0; st < NB2 - 1; ++st) {
            int bp, bq;
            rr_pair(rank, st, NB2, bp, bq);
            const int p0 = bp * JB, q0 = bq * JB;
            const int np = max(0, min(JB, m - p0)), nq = max(0, min(JB, m - q0));
            // stage: 16 independent L2 loads in flight per thread (rows beyond
            // m are zero and never rotate); (r, i) advance without division
            {
                int r = threadIdx.x / n, i = threadIdx.x % n;
                while (r < 2 * JB) {
                    double v[16];
                    int rr[16], ii[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        rr[u] = r;
                        ii[u] = i;
                        const int row = r < JB ? p0 + r : q0 + r - JB;
                        const bool ok = r < 2 * JB && (r < JB ? r < np : r - JB < nq);
                        v[u] = ok ? __ldcg(A + (int64_t)row * n + i) : 0.0;
                        i += JBT;
                        while (i >= n) {
                            i -= n;
                            ++r;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (rr[u] < 2 * JB) bsm[(int64_t)rr[u] * n + ii[u]] = v[u];
                }
            }
            __syncthreads();
            for (int r = warp; r < 2 * JB; r += nw) {
                const double* rr = bsm + (int64_t)r * n;
                double v = 0.0;
                for (int i = lane; i < n; i += 32) v += rr[i] * rr[i];
                v = warp_sum(v);
                if (lane == 0) bn[r] = v;
            }
            __syncthreads();
            if (st == 0) {
                // rotations inside each block: round robin on JB rows, pair
                // groups [0, JB/2) on block p, [JB/2, JB) on block q
                const int half = JB / 2, blk = grp / half, wi = grp % half;
                const int jbe = JB + (JB & 1);
                for (int is = 0; is < jbe - 1; ++is) {
                    for (int pi = wi; pi < jbe / 2; pi += half) {
                        int a, b;
                        rr_pair(pi, is, jbe, a, b);
                        if (a >= JB || b >= JB) continue;
                        const int ra = blk * JB + a, rb = blk * JB + b;
                        double na = bn[ra], nb = bn[rb];
                        const int rc = jac_rotate_split<WPP>(bsm + (int64_t)ra * n, bsm + (int64_t)rb * n, n, tol,
                                                             na, nb, grp, sub, red, par);
                        if (rc) {
                            rotated |= rc == 2;
                            if (lane == 0 && sub == 0) {
                                bn[ra] = na;
                                bn[rb] = nb;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            // cross rotations: inner step s pairs p-row i with q-row (i + s) % JB
            for (int s = 0; s < JB; ++s) {
                const int i = grp;
                const int rq = JB + (i + s) % JB;
                double na = bn[i], nb = bn[rq];
                const int rc = jac_rotate_split<WPP>(bsm + (int64_t)i * n, bsm + (int64_t)rq * n, n, tol, na, nb, grp,
                                                     sub, red, par);
                if (rc) {
                    rotated |= rc == 2;
                    if (lane == 0 && sub == 0) {
                        bn[i] = na;
                        bn[rq] = nb;
                    }
                }
                __syncthreads();
            }
            for (int r = 0; r < 2 * JB; ++r) {
                const int row = r < JB ? p0 + r : q0 + r - JB;
                const bool v = r < JB ? r < np : r - JB < nq;
                if (!v) continue;
                double* dst = A + (int64_t)row * n;
                const double* src = bsm + (int64_t)r * n;
                for (int i = threadIdx.x; i < n; i += JBT) __stcg(dst + i, src[i]);
            }
            cta_group_barrier(CT.bar, P);
        }
        if (rotated && lane == 0) rot_s = 1;
        __syncthreads();
        if (rot_s && threadIdx.x == 0) CT.flags[sweep] = 1;
        cta_group_barrier(CT.bar, P);
        const int any = __ldcg(CT.flags + sweep);
        if (rank == 0 && threadIdx.x == 0) CT.flags[63] = sweep + 1;
        if (!any) break;
    }
    // sigma, kept count, sorted normalised rows (as jacobi_coop_kernel)
    const int gw = rank * nw + warp, gnw = P * nw;
    for (int i = gw; i < m; i += gnw) {
        const double sg = row_norm_reg<0>(A + (int64_t)i * n, n);
        if (lane == 0) CT.sig[i] = sg;
    }
    cta_group_barrier(CT.bar, P);
    double* dsh = bsm;
    for (int i = threadIdx.x; i < m; i += JBT) dsh[i] = __ldcg(CT.sig + i);
    if (threadIdx.x == 0) kept_s = 0;
    __syncthreads();
    int cnt = 0;
    for (int i = threadIdx.x; i < m; i += JBT) cnt += dsh[i] >= thresh;
    atomicAdd(&kept_s, cnt);
    __syncthreads();
    const int kept = kept_s;
    if (rank == 0 && threadIdx.x == 0) *CT.t.kept_out = kept;
    const double smax = sig_max(dsh, m);
    for (int i = gw; i < m; i += gnw) {
        const double si = dsh[i];
        int r = 0;
        for (int j = lane; j < m; j += 32) r += (dsh[j] > si) || (dsh[j] == si && j < i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        (void)kept;
        if (!(si > JAC_TINY && si > JAC_RANK_REL * smax) && CT.t.deg_off && lane == 0)
            CT.t.kept_out[CT.t.deg_off] = 1;
        const double inv = si > JAC_TINY ? 1.0 / si : 0.0;
        const double* ri = A + (int64_t)i * n;
        for (int c = lane; c < n; c += 32) CT.t.U[(int64_t)r * n + c] = __ldcg(ri + c) * inv;
    }
}

// first-index argmax of |x| across the CTA
__device__ __forceinline__ void block_argmax(double v, int idx, double* shv, int* shi, double& bv,
                                             int& bi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    __syncthreads();
    if (lane == 0) { shv[warp] = v; shi[warp] = idx; }
    __syncthreads();
    bv = shv[0];
    bi = shi[0];
    for (int w = 1; w < nw; ++w)
        if (shv[w] > bv || (shv[w] == bv && shi[w] < bi)) { bv = shv[w]; bi = shi[w]; }
}

__global__ void __launch_bounds__(DT) lu_kernel(const LuTask* __restrict__ tasks) {
    const LuTask T = tasks[blockIdx.x];
    __shared__ double shv[DT / 32];
    __shared__ int shi[DT / 32];
    const int r = T.r;
    double mx = 0.0;
    for (int64_t e = threadIdx.x; e < (int64_t)r * r; e += DT) {
        const int i = (int)(e / r), j = (int)(e % r);
        const double v = T.D[(int64_t)i * T.ldd + j];
        T.LU[e] = v;
        mx = fmax(mx, fabs(v));
    }
    const double scale = block_max(mx, shv);
    __syncthreads();
    double* A = T.LU;
    for (int k = 0; k < r; ++k) {
        double v = -1.0;
        int idx = r;
        for (int i = k + threadIdx.x; i < r; i += DT) {
            const double a = fabs(A[(int64_t)i * r + k]);
            if (a > v) { v = a; idx = i; }
        }
        double bv;
        int p;
        block_argmax(v, idx, shv, shi, bv, p);
        if (threadIdx.x == 0) T.piv[k] = p;
        if (p != k)
            for (int j = threadIdx.x; j < r; j += DT) {
                const double t0 = A[(int64_t)k * r + j];
                A[(int64_t)k * r + j] = A[(int64_t)p * r + j];
                A[(int64_t)p * r + j] = t0;
            }
        __syncthreads();
        const double pv = A[(int64_t)k * r + k];
        if (pv != 0.0) {
            const bool recip = fabs(pv) >= DBL_MIN;
            const double inv = 1.0 / pv;
            for (int i = k + 1 + threadIdx.x; i < r; i += DT) {
                double* a = A + (int64_t)i * r + k;
                *a = recip ? *a * inv : *a / pv;
            }
        }
        __syncthreads();
        const int rem = r - k - 1;
        for (int64_t e = threadIdx.x; e < (int64_t)rem * rem; e += DT) {
            const int i = k + 1 + (int)(e / rem), j = k + 1 + (int)(e % rem);
            A[(int64_t)i * r + j] -= A[(int64_t)i * r + k] * A[(int64_t)k * r + j];
        }
        __syncthreads();
    }
    double mn = DBL_MAX;
    for (int i = threadIdx.x; i < r; i += DT) mn = fmin(mn, fabs(A[(int64_t)i * r + i]));
    mn = -block_max(-mn, shv);
    if (threadIdx.x == 0)
        *T.status = (r > 0 && mn <= 1e-14 * fmax(scale, 1e-300)) ? 1 : 0;
}

constexpr int TRSM_T = 128;

__global__ void __launch_bounds__(TRSM_T) trsm_kernel(const TrsmTask* __restrict__ tasks) {
    const TrsmTask T = tasks[blockIdx.x];
    extern __shared__ int perm[];
    const int r = T.r;
    if (threadIdx.x == 0) {
        for (int i = 0; i < r; ++i) perm[i] = i;
        for (int k = 0; k < r; ++k) {
            const int p = T.piv[k];
            const int t0 = perm[k];
            perm[k] = perm[p];
            perm[p] = t0;
        }
    }
    __syncthreads();
    const int col = T.col0 + threadIdx.x;
    if (col >= T.W) return;
    const double* LU = T.LU;
    double* X = T.MW + col;
    const int64_t ldw = T.ldw;
    for (int i = 0; i < r; ++i) {
        double acc = T.G[(int64_t)perm[i] * T.ldg + col];
        const double* li = LU + (int64_t)i * r;
        for (int k = 0; k < i; ++k) acc -= li[k] * X[(int64_t)k * ldw];
        X[(int64_t)i * ldw] = acc;
    }
    for (int i = r - 1; i >= 0; --i) {
        double acc = X[(int64_t)i * ldw];
        const double* ui = LU + (int64_t)i * r;
        for (int k = i + 1; k < r; ++k) acc -= ui[k] * X[(int64_t)k * ldw];
        X[(int64_t)i * ldw] = acc / ui[i];
    }
    for (int i = 0; i < r; ++i) X[(int64_t)i * ldw] = -X[(int64_t)i * ldw];
}

// ---- blocked TRSM on DMMA: MW = -(U^-1 L^-1 P G), NC columns per CTA ---------
// The CTA keeps its NC-column slice X (r x NC) in shared memory; per 32-row
// block the update by the already solved rows is an 8x8x4 DMMA product with
// the L (U) block row streamed from L2, followed by a sequential in-block
// substitution (one thread per column) against the block staged in shared
// memory.  Same forward/backward substitution as getrs (factorization.py:120).
template <int NC>
__global__ void __launch_bounds__(256, 1) trsm_dmma_kernel(const TrsmTask* __restrict__ tasks) {
    constexpr int NCP = NC + 4;          // conflict-free B fragments
    constexpr int TN = NC / 8;           // 8x8 tiles across
    constexpr int TPW = (4 * TN) / 8;    // tiles per warp (8 warps, 32-row blocks)
    const TrsmTask T = tasks[blockIdx.x];
    const int r = T.r, r4 = (r + 3) & ~3;
    const int ncols = min(NC, T.W - T.col0);
    extern __shared__ double X[];        // r4 x NCP
    __shared__ double Lb[32][33];
    int* perm = reinterpret_cast<int*>(X + (int64_t)r4 * NCP);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const double* LU = T.LU;
    const int64_t ldl = T.ldlu ? T.ldlu : r;
    const int mode = T.mode;
    if (threadIdx.x == 0) {
        for (int i = 0; i < r; ++i) perm[i] = i;
        if ((mode & TRSM_LOWER) && T.piv)
            for (int k = 0; k < r; ++k) {
                const int p = T.piv[k];
                const int t0 = perm[k];
                perm[k] = perm[p];
                perm[p] = t0;
            }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < r4 * NC; e += 256) {
        const int i = e / NC, c = e % NC;
        X[i * NCP + c] = (i < r && c < ncols) ? T.G[(int64_t)perm[i] * T.ldg + T.col0 + c] : 0.0;
    }
    __syncthreads();
    const int nblk = (r + 31) / 32;
    for (int dir = 0; dir < 2; ++dir) {  // 0: unit lower, forward; 1: upper, backward
        if (!(mode & (dir == 0 ? TRSM_LOWER : TRSM_UPPER))) continue;
        for (int bb = 0; bb < nblk; ++bb) {
            const int blk = dir == 0 ? bb : nblk - 1 - bb;
            const int b0 = blk * 32, nb = min(32, r - b0);
            const int k_lo = dir == 0 ? 0 : b0 + nb, k_hi = dir == 0 ? b0 : r;
            if (k_hi > k_lo) {
                double c[TPW][2];
#pragma unroll
                for (int u = 0; u < TPW; ++u) c[u][0] = c[u][1] = 0.0;
                for (int k = k_lo; k < k_hi; k += 4) {
#pragma unroll
                    for (int u = 0; u < TPW; ++u) {
                        const int tid_ = warp * TPW + u, ti = tid_ / TN, tj = tid_ % TN;
                        const int row = ti * 8 + g;
                        const double a = (row < nb && k + t < k_hi) ? __ldg(LU + (int64_t)(b0 + row) * ldl + k + t) : 0.0;
                        const double bv = X[(k + t) * NCP + tj * 8 + g];
                        dmma_8x8x4(c[u][0], c[u][1], a, bv);
                    }
                }
                __syncthreads();
#pragma unroll
                for (int u = 0; u < TPW; ++u) {
                    const int tid_ = warp * TPW + u, ti = tid_ / TN, tj = tid_ % TN;
                    const int row = ti * 8 + g;
                    if (row < nb) {
                        X[(b0 + row) * NCP + tj * 8 + 2 * t] -= c[u][0];
                        X[(b0 + row) * NCP + tj * 8 + 2 * t + 1] -= c[u][1];
                    }
                }
            }
            for (int e = threadIdx.x; e < 32 * 32; e += 256) {
                const int i = e >> 5, k = e & 31;
                Lb[i][k] = (i < nb && k < nb) ? LU[(int64_t)(b0 + i) * ldl + b0 + k] : 0.0;
            }
            __syncthreads();
            if (threadIdx.x < NC) {
                double* xc = X + (int64_t)b0 * NCP + threadIdx.x;
                if (dir == 0) {
                    for (int i = 1; i < nb; ++i) {
                        double acc = xc[i * NCP];
                        for (int k = 0; k < i; ++k) acc -= Lb[i][k] * xc[k * NCP];
                        xc[i * NCP] = acc;
                    }
                } else {
                    for (int i = nb - 1; i >= 0; --i) {
                        double acc = xc[i * NCP];
                        for (int k = i + 1; k < nb; ++k) acc -= Lb[i][k] * xc[k * NCP];
                        xc[i * NCP] = acc / Lb[i][i];
                    }
                }
            }
            __syncthreads();
        }
    }
    const double sgn = (mode & TRSM_NEGATE) ? -1.0 : 1.0;
    for (int e = threadIdx.x; e < r * NC; e += 256) {
        const int i = e / NC, c = e % NC;
        if (c < ncols) T.MW[(int64_t)i * T.ldw + T.col0 + c] = sgn * X[i * NCP + c];
    }
}

__global__ void lu_status_kernel(const double* red, int r, int* status) {
    *status = (r > 0 && red[1] <= 1e-14 * fmax(red[0], 1e-300)) ? 1 : 0;
}

// ---- dense top LU pieces --------------------------------------------------------

__global__ void __launch_bounds__(DT) panel_lu_kernel(double* A, int64_t lda, int n, int k0, int nb,
                                                     int* piv) {
    __shared__ double shv[DT / 32];
    __shared__ int shi[DT / 32];
    const int cend = k0 + nb;
    for (int c = k0; c < cend; ++c) {
        double v = -1.0;
        int idx = n;
        for (int i = c + threadIdx.x; i < n; i += DT) {
            const double a = fabs(A[(int64_t)i * lda + c]);
            if (a > v) { v = a; idx = i; }
        }
        double bv;
        int p;
        block_argmax(v, idx, shv, shi, bv, p);
        if (threadIdx.x == 0) piv[c] = p;
        if (p != c)
            for (int j = k0 + threadIdx.x; j < cend; j += DT) {
                const double t0 = A[(int64_t)c * lda + j];
                A[(int64_t)c * lda + j] = A[(int64_t)p * lda + j];
                A[(int64_t)p * lda + j] = t0;
            }
        __syncthreads();
        const double pv = A[(int64_t)c * lda + c];
        if (pv != 0.0) {
            const bool recip = fabs(pv) >= DBL_MIN;
            const double inv = 1.0 / pv;
            for (int i = c + 1 + threadIdx.x; i < n; i += DT) {
                double* a = A + (int64_t)i * lda + c;
                *a = recip ? *a * inv : *a / pv;
            }
        }
        __syncthreads();
        const int w = cend - c - 1;
        if (w > 0) {
            const int rows = n - c - 1;
            for (int64_t e = threadIdx.x; e < (int64_t)rows * w; e += DT) {
                const int i = c + 1 + (int)(e / w), j = c + 1 + (int)(e % w);
                A[(int64_t)i * lda + j] -= A[(int64_t)i * lda + c] * A[(int64_t)c * lda + j];
            }
        }
        __syncthreads();
    }
}

// apply the panel's row swaps (rows k0..k0+nb-1, in order) to all columns
// outside [skip_c0, skip_c1)
__global__ void row_swaps_kernel(double* A, int64_t lda, int ncols, int k0, int nb, const int* piv,
                                 int skip_c0, int skip_c1) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncols || (j >= skip_c0 && j < skip_c1)) return;
    for (int c = k0; c < k0 + nb; ++c) {
        const int p = piv[c];
        if (p != c) {
            const double t0 = A[(int64_t)c * lda + j];
            A[(int64_t)c * lda + j] = A[(int64_t)p * lda + j];
            A[(int64_t)p * lda + j] = t0;
        }
    }
}

// A[k0:k0+nb, c0:c0+ncols] = L11^-1 A[...]  (L11 unit lower of the panel)
// X = L11^-1 X for the nb (<= TOP_PANEL_NB) panel rows of columns [c0, c0+ncols):
// L11 staged once per CTA in shared memory, the column's nb values in
// registers (fully unrolled), one thread per column
__global__ void __launch_bounds__(256) trsm_unit_lower_rows_kernel(double* A, int64_t lda, int k0, int nb, int c0,
                                                                   int ncols) {
    __shared__ double Ls[TOP_PANEL_NB][TOP_PANEL_NB + 1];
    for (int e = threadIdx.x; e < TOP_PANEL_NB * TOP_PANEL_NB; e += blockDim.x) {
        const int i = e / TOP_PANEL_NB, k = e % TOP_PANEL_NB;
        Ls[i][k] = (i < nb && k < i) ? A[(int64_t)(k0 + i) * lda + k0 + k] : 0.0;
    }
    __syncthreads();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncols) return;
    double* x = A + (int64_t)k0 * lda + c0 + j;
    double v[TOP_PANEL_NB];
#pragma unroll
    for (int i = 0; i < TOP_PANEL_NB; ++i) v[i] = i < nb ? x[(int64_t)i * lda] : 0.0;
#pragma unroll
    for (int i = 1; i < TOP_PANEL_NB; ++i) {
        double acc = v[i];
#pragma unroll
        for (int k = 0; k < i; ++k) acc -= Ls[i][k] * v[k];
        v[i] = acc;
    }
#pragma unroll
    for (int i = 1; i < TOP_PANEL_NB; ++i)
        if (i < nb) x[(int64_t)i * lda] = v[i];
}

// max |A| over all CTAs: per-CTA block max, then an integer atomicMax on the
// bit pattern (monotone for non-negative doubles, so the result is exact
// and order independent); *out must be 0 before the launch
__global__ void absmax_kernel(const double* A, int64_t lda, int rows, int cols, double* out) {
    __shared__ double sh[32];
    double m = 0.0;
    const int64_t tot = (int64_t)rows * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(A[(e / cols) * lda + (e % cols)]));
    m = block_max(m, sh);
    if (threadIdx.x == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(m));
}

__global__ void diag_absmin_kernel(const double* A, int64_t lda, int n, double* out) {
    __shared__ double sh[32];
    double m = DBL_MAX;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmin(m, fabs(A[(int64_t)i * lda + i]));
    m = -block_max(-m, sh);
    if (threadIdx.x == 0) *out = m;
}

}  // namespace

void launch_qr_r_smem(const QrTask* d_tasks, int32_t ntasks, int32_t max_n, cudaStream_t st) {
    if (ntasks <= 0) return;
    const size_t smem = sizeof(double) * (size_t(max_n) * max_n + size_t(max_n) * QB + 8);
    cudaFuncSetAttribute(qr_r_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qr_r_smem_kernel<<<ntasks, DT, smem, st>>>(d_tasks);
    count_launch();
}

void launch_jacobi_smem(const SvdTask* d_tasks, int32_t ntasks, int32_t max_n, double thresh,
                        cudaStream_t st) {
    if (ntasks <= 0) return;
    const size_t smem = sizeof(double) * (size_t(max_n) * max_n + 3 * size_t(max_n)) + 64;  // A, sig, rank, norms
    cudaFuncSetAttribute(jacobi_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    jacobi_smem_kernel<<<ntasks, DT, smem, st>>>(d_tasks, thresh);
    count_launch();
}

void launch_reorth(const ReorthTask* d_tasks, int32_t ntasks, cudaStream_t st) {
    if (ntasks <= 0) return;
    reorth_kernel<<<ntasks, DT, 0, st>>>(d_tasks);
    count_launch();
}

void launch_normalize_rows(const RowNormTask* d_tasks, int32_t nrows, cudaStream_t st) {
    if (nrows <= 0) return;
    normalize_rows_kernel<<<(nrows + 7) / 8, 256, 0, st>>>(d_tasks, nrows);
    count_launch();
}

void launch_r_extract(const RExtractTask* d_tasks, int32_t ntasks, int32_t max_n, cudaStream_t st) {
    if (ntasks <= 0) return;
    dim3 grid((unsigned)(((int64_t)max_n * max_n + 255) / 256), ntasks);
    r_extract_kernel<<<grid, 256, 0, st>>>(d_tasks);
    count_launch();
}

int jacobi_coop_npl(int n) {
    const int npl = (n + 31) / 32;
    for (int c : {2, 4, 8, 12, 16, 20, 24, 32, 40, 48})
        if (npl <= c) return c;
    return 0;  // generic loop version
}

template <int NPL>
static cudaError_t launch_jc(const CoopSvdTask* d_tasks, int32_t total_ctas, const int32_t* d_cta_task,
                             double thresh, size_t smem, cudaStream_t st) {
    cudaFuncSetAttribute(jacobi_coop_kernel<NPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    void* args[] = {(void*)&d_tasks, (void*)&d_cta_task, (void*)&thresh};
    return cudaLaunchCooperativeKernel((const void*)jacobi_coop_kernel<NPL>, dim3(total_ctas), dim3(JT), args,
                                       smem, st);
}

cudaError_t launch_jacobi_coop(const CoopSvdTask* d_tasks, int32_t total_ctas, const int32_t* d_cta_task,
                               int32_t max_n, int32_t max_m, double thresh, cudaStream_t st) {
    if (total_ctas <= 0) return cudaSuccess;
    const size_t smem = sizeof(double) * size_t(std::max(max_m, 1));
    cudaError_t e = cudaErrorInvalidValue;
    switch (jacobi_coop_npl(max_n)) {
    case 2: e = launch_jc<2>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 4: e = launch_jc<4>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 8: e = launch_jc<8>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 12: e = launch_jc<12>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 16: e = launch_jc<16>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 20: e = launch_jc<20>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 24: e = launch_jc<24>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 32: e = launch_jc<32>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 40: e = launch_jc<40>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    case 48: e = launch_jc<48>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    default: e = launch_jc<0>(d_tasks, total_ctas, d_cta_task, thresh, smem, st); break;
    }
    count_launch();
    return e;
}

int jacobi_coop_capacity(int max_n, int max_m) {
    const size_t smem = sizeof(double) * size_t(std::max(max_m, 1));
    int per_sm = 0, dev = 0, sms = 0;
    const void* fn = nullptr;
    switch (jacobi_coop_npl(max_n)) {
    case 2: fn = (const void*)jacobi_coop_kernel<2>; break;
    case 4: fn = (const void*)jacobi_coop_kernel<4>; break;
    case 8: fn = (const void*)jacobi_coop_kernel<8>; break;
    case 12: fn = (const void*)jacobi_coop_kernel<12>; break;
    case 16: fn = (const void*)jacobi_coop_kernel<16>; break;
    case 20: fn = (const void*)jacobi_coop_kernel<20>; break;
    case 24: fn = (const void*)jacobi_coop_kernel<24>; break;
    case 32: fn = (const void*)jacobi_coop_kernel<32>; break;
    case 40: fn = (const void*)jacobi_coop_kernel<40>; break;
    case 48: fn = (const void*)jacobi_coop_kernel<48>; break;
    default: fn = (const void*)jacobi_coop_kernel<0>; break;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, JT, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}


namespace {
const void* jacobi_block_fn(int jb) {
    return jb == 16 ? (const void*)jacobi_block_kernel<16>
                    : jb == 8 ? (const void*)jacobi_block_kernel<8> : (const void*)jacobi_block_kernel<4>;
}
}  // namespace

int jacobi_block_rows(int n) {
    // H2F_JACOBI_JB: force the rows per block (4, 8 or 16: one warp per row
    // pair, measured slower on config-2 shapes: the FP64 pipe of the fewer
    // CTAs saturates); default 8, 4 from H2F_JACOBI_JB4_MIN_N
    static const int forced = [] {
        const char* e = std::getenv("H2F_JACOBI_JB");
        return e ? std::atoi(e) : 0;
    }();
    static const int jb4_min = [] {
        const char* e = std::getenv("H2F_JACOBI_JB4_MIN_N");
        return e ? std::atoi(e) : 512;
    }();
    auto fits = [n](int jb) { return size_t(2 * jb) * n * 8 <= size_t(220) * 1024; };
    if ((forced == 16 || forced == 8 || forced == 4) && fits(forced)) return forced;
    if (n >= jb4_min) return 4;
    return fits(8) ? 8 : 4;
}



size_t jacobi_block_smem(int max_n, int max_m) {
    const int jb = jacobi_block_rows(max_n);
    return sizeof(double) * std::max<size_t>(size_t(2) * jb * max_n, size_t(max_m));
}

int jacobi_block_capacity(int max_n, int max_m) {
    const size_t smem = jacobi_block_smem(max_n, max_m);
    const void* fn = jacobi_block_fn(jacobi_block_rows(max_n));
    // a shared-memory request above the device limit means "cannot be
    // resident": capacity 0, and the caller takes the pairwise kernel --
    // checked here so no sticky launch error is left behind
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, JBT, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * sms;
}

cudaError_t launch_jacobi_block(const CoopSvdTask* d_tasks, int32_t total_ctas, const int32_t* d_cta_task,
                                int32_t max_n, int32_t max_m, double thresh, cudaStream_t st) {
    if (total_ctas <= 0) return cudaSuccess;
    const size_t smem = jacobi_block_smem(max_n, max_m);
    const void* fn = jacobi_block_fn(jacobi_block_rows(max_n));
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    void* args[] = {(void*)&d_tasks, (void*)&d_cta_task, (void*)&thresh};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(total_ctas), dim3(JBT), args, smem, st);
    count_launch();
    return e;
}


int trsm_dmma_cols(int r) {
    if (size_t(r + 4) * 36 * 8 + size_t(r) * 4 <= size_t(200) * 1024) return 32;
    if (size_t(r + 4) * 20 * 8 + size_t(r) * 4 <= size_t(200) * 1024) return 16;
    return 0;
}

void launch_trsm_dmma(const TrsmTask* d_tasks, int32_t ntasks, int32_t max_r, int32_t nc, cudaStream_t st) {
    if (ntasks <= 0) return;
    const int r4 = (max_r + 3) & ~3;
    if (nc == 32) {
        const size_t smem = size_t(r4) * 36 * 8 + size_t(max_r) * 4 + 16;
        cudaFuncSetAttribute(trsm_dmma_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        trsm_dmma_kernel<32><<<ntasks, 256, smem, st>>>(d_tasks);
    } else {
        const size_t smem = size_t(r4) * 20 * 8 + size_t(max_r) * 4 + 16;
        cudaFuncSetAttribute(trsm_dmma_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        trsm_dmma_kernel<16><<<ntasks, 256, smem, st>>>(d_tasks);
    }
    count_launch();
}

void launch_lu_status(const double* red, int32_t r, int32_t* status, cudaStream_t st) {
    lu_status_kernel<<<1, 1, 0, st>>>(red, r, status);
    count_launch();
}

void launch_complement(const ComplementTask* d_tasks, int32_t ntasks, cudaStream_t st) {
    if (ntasks <= 0) return;
    const size_t smem = 4096 * sizeof(double);
    cudaFuncSetAttribute(complement_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    complement_kernel<<<ntasks, DT, smem, st>>>(d_tasks);
    count_launch();
}

void launch_lu(const LuTask* d_tasks, int32_t ntasks, cudaStream_t st) {
    if (ntasks <= 0) return;
    lu_kernel<<<ntasks, DT, 0, st>>>(d_tasks);
    count_launch();
}

void launch_trsm(const TrsmTask* d_tasks, int32_t ntasks, cudaStream_t st) {
    if (ntasks <= 0) return;
    trsm_kernel<<<ntasks, TRSM_T, 4096 * sizeof(int), st>>>(d_tasks);
    count_launch();
}

void launch_panel_lu(double* A, int64_t lda, int32_t n, int32_t k0, int32_t nb, int32_t* piv,
                     cudaStream_t st) {
    panel_lu_kernel<<<1, DT, 0, st>>>(A, lda, n, k0, nb, piv);
    count_launch();
}

void launch_row_swaps(double* A, int64_t lda, int32_t ncols_total, int32_t k0, int32_t nb,
                      const int32_t* piv, int32_t skip_c0, int32_t skip_c1, cudaStream_t st) {
    row_swaps_kernel<<<(ncols_total + 127) / 128, 128, 0, st>>>(A, lda, ncols_total, k0, nb, piv,
                                                                skip_c0, skip_c1);
    count_launch();
}

void launch_trsm_unit_lower_rows(const double* A, int64_t lda, int32_t k0, int32_t nb, int32_t c0,
                                 int32_t ncols, cudaStream_t st) {
    if (ncols <= 0) return;
    trsm_unit_lower_rows_kernel<<<(ncols + 255) / 256, 256, 0, st>>>(const_cast<double*>(A), lda, k0,
                                                                      nb, c0, ncols);
    count_launch();
}

void launch_absmax(const double* A, int64_t lda, int32_t rows, int32_t cols, double* out,
                   cudaStream_t st) {
    cudaMemsetAsync(out, 0, sizeof(double), st);
    const int64_t tot = int64_t(rows) * cols;
    const int grid = int(std::min<int64_t>(int64_t(sm_count()) * 4, std::max<int64_t>(1, (tot + 1023) / 1024)));
    absmax_kernel<<<grid, 1024, 0, st>>>(A, lda, rows, cols, out);
    count_launch();
}

void launch_diag_absmin(const double* A, int64_t lda, int32_t n, double* out, cudaStream_t st) {
    diag_absmin_kernel<<<1, 1024, 0, st>>>(A, lda, n, out);
    count_launch();
}

}  // namespace h2f
