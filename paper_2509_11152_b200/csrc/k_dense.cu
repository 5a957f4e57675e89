// Per-cluster dense linear algebra, batched: one CTA per cluster of a batch.
//
//   qr_r        R of the reduced Householder QR of Y^T (Y = fill residual)   factorization.py:78
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
#include <cfloat>

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

__global__ void __launch_bounds__(DT) qr_r_kernel(const QrTask* __restrict__ tasks) {
    const QrTask T = tasks[blockIdx.x];
    __shared__ double sh[DT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = DT / 32;
    const int s = T.s, wf = T.wf;
    const int nref = s < wf ? s : wf;
    for (int j = 0; j < nref; ++j) {
        double* yj = T.Y + (int64_t)j * T.ldy;
        double ss = 0.0;
        for (int i = j + 1 + threadIdx.x; i < wf; i += DT) ss += yj[i] * yj[i];
        ss = block_sum(ss, sh);
        const double alpha = yj[j];
        double beta, tau, scal;
        reflector(alpha, ss, beta, tau, scal);
        if (tau != 0.0)
            for (int i = j + 1 + threadIdx.x; i < wf; i += DT) yj[i] *= scal;
        if (threadIdx.x == 0) {
            double* rj = T.R + (int64_t)j * s;
            rj[j] = beta;
            for (int c = 0; c < j; ++c) rj[c] = 0.0;
        }
        __syncthreads();
        for (int c = j + 1 + warp; c < s; c += nw) {
            double* yc = T.Y + (int64_t)c * T.ldy;
            double d = 0.0;
            for (int i = j + 1 + lane; i < wf; i += 32) d += yj[i] * yc[i];
            d = warp_sum(d) + yc[j];
            if (tau != 0.0) {
                d *= tau;
                for (int i = j + 1 + lane; i < wf; i += 32) yc[i] -= d * yj[i];
                __syncwarp();
                if (lane == 0) yc[j] -= d;
            }
            __syncwarp();
            if (lane == 0) T.R[(int64_t)j * s + c] = yc[j];
        }
        __syncthreads();
    }
}

// circle-method round robin: player list [0, rot...]; pair i of round st
__device__ __forceinline__ void rr_pair(int i, int st, int mm, int& p, int& q) {
    auto pos = [&](int j) { return j == 0 ? 0 : 1 + ((j - 1 + st) % (mm - 1)); };
    p = pos(i);
    q = pos(mm - 1 - i);
}

__global__ void __launch_bounds__(DT) jacobi_kernel(const SvdTask* __restrict__ tasks, double thresh) {
    const SvdTask T = tasks[blockIdx.x];
    extern __shared__ double dsh[];  // sig[m] then rank (int) [m]
    __shared__ double sh[DT / 32];
    __shared__ int rotated;
    __shared__ int kept_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = DT / 32;
    const int s = T.s, k = T.k, m = T.m;

    // b_aug^T rows 0..k-1 = V^T
    for (int64_t e = threadIdx.x; e < (int64_t)k * s; e += DT) {
        const int l = (int)(e / s), i = (int)(e % s);
        T.BT[(int64_t)l * s + i] = T.V[(int64_t)i * T.ldv + l];
    }
    if (T.skip || m == 0) {
        if (threadIdx.x == 0) *T.kept_out = 0;
        return;
    }
    const double tol = 2.220446049250313e-16 * sqrt((double)s);
    const int mm = m + (m & 1);
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int st = 0; st < mm - 1; ++st) {
            for (int pi = warp; pi < mm / 2; pi += nw) {
                int p, q;
                rr_pair(pi, st, mm, p, q);
                if (p >= m || q >= m) continue;
                double* rp = T.R + (int64_t)p * s;
                double* rq = T.R + (int64_t)q * s;
                double a = 0.0, b = 0.0, g = 0.0;
                for (int i = lane; i < s; i += 32) {
                    const double x = rp[i], y = rq[i];
                    a += x * x;
                    b += y * y;
                    g += x * y;
                }
                a = warp_sum(a);
                b = warp_sum(b);
                g = warp_sum(g);
                if (g != 0.0 && a > 0.0 && b > 0.0 && fabs(g) > tol * sqrt(a) * sqrt(b)) {
                    const double zeta = (b - a) / (2.0 * g);
                    const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
                    for (int i = lane; i < s; i += 32) {
                        const double x = rp[i], y = rq[i];
                        rp[i] = c * x - sn * y;
                        rq[i] = sn * x + c * y;
                    }
                    if (lane == 0) rotated = 1;
                }
            }
            __syncthreads();
        }
        const int any = rotated;
        __syncthreads();
        if (!any) break;
    }
    double* sig = dsh;
    int* rnk = reinterpret_cast<int*>(dsh + m);
    for (int i = warp; i < m; i += nw) {
        const double* ri = T.R + (int64_t)i * s;
        double a = 0.0;
        for (int c = lane; c < s; c += 32) a += ri[c] * ri[c];
        a = warp_sum(a);
        if (lane == 0) sig[i] = sqrt(a);
    }
    __syncthreads();
    if (threadIdx.x == 0) kept_s = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += DT) {
        int r = 0;
        const double si = sig[i];
        for (int j = 0; j < m; ++j) r += (sig[j] > si) || (sig[j] == si && j < i);
        rnk[i] = r;
        if (si >= thresh) atomicAdd(&kept_s, 1);
    }
    __syncthreads();
    const int kept = kept_s;
    if (threadIdx.x == 0) *T.kept_out = kept;
    if (kept == 0) return;
    // pass 1: u_j = rotated row / sigma  -> BT rows k..k+kept-1
    for (int i = warp; i < m; i += nw) {
        const int j = rnk[i];
        if (j >= kept) continue;
        const double inv = 1.0 / sig[i];
        const double* ri = T.R + (int64_t)i * s;
        double* dst = T.BT + (int64_t)(k + j) * s;
        for (int c = lane; c < s; c += 32) dst[c] = ri[c] * inv;
    }
    __syncthreads();
    // pass 2: C = V^T U (k x kept) stored in R (free now)
    double* C = T.R;
    for (int64_t e = warp; e < (int64_t)k * kept; e += nw) {
        const int l = (int)(e / kept), j = (int)(e % kept);
        const double* u = T.BT + (int64_t)(k + j) * s;
        double d = 0.0;
        for (int i = lane; i < s; i += 32) d += T.V[(int64_t)i * T.ldv + l] * u[i];
        d = warp_sum(d);
        if (lane == 0) C[e] = d;
    }
    __syncthreads();
    // pass 3: u_j -= V C[:, j]
    for (int64_t e = threadIdx.x; e < (int64_t)kept * s; e += DT) {
        const int j = (int)(e / s), i = (int)(e % s);
        double d = 0.0;
        for (int l = 0; l < k; ++l) d += T.V[(int64_t)i * T.ldv + l] * C[(int64_t)l * kept + j];
        T.BT[(int64_t)(k + j) * s + i] -= d;
    }
    __syncthreads();
    // pass 4: normalise columns
    for (int j = warp; j < kept; j += nw) {
        double* u = T.BT + (int64_t)(k + j) * s;
        double a = 0.0;
        for (int i = lane; i < s; i += 32) a += u[i] * u[i];
        a = warp_sum(a);
        const double inv = 1.0 / sqrt(a);
        for (int i = lane; i < s; i += 32) u[i] *= inv;
    }
}

__global__ void __launch_bounds__(DT) complement_kernel(const ComplementTask* __restrict__ tasks) {
    const ComplementTask T = tasks[blockIdx.x];
    extern __shared__ double taus[];  // [s]
    __shared__ double sh[DT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = DT / 32;
    const int s = T.s;
    const int kt = T.k + *T.kept;
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
__global__ void trsm_unit_lower_rows_kernel(double* A, int64_t lda, int k0, int nb, int c0, int ncols) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncols) return;
    double* x = A + c0 + j;
    for (int i = 1; i < nb; ++i) {
        const double* li = A + (int64_t)(k0 + i) * lda + k0;
        double acc = x[(int64_t)(k0 + i) * lda];
        for (int k = 0; k < i; ++k) acc -= li[k] * x[(int64_t)(k0 + k) * lda];
        x[(int64_t)(k0 + i) * lda] = acc;
    }
}

__global__ void absmax_kernel(const double* A, int64_t lda, int rows, int cols, double* out) {
    __shared__ double sh[32];
    double m = 0.0;
    for (int64_t e = threadIdx.x; e < (int64_t)rows * cols; e += blockDim.x)
        m = fmax(m, fabs(A[(e / cols) * lda + (e % cols)]));
    m = block_max(m, sh);
    if (threadIdx.x == 0) *out = m;
}

__global__ void diag_absmin_kernel(const double* A, int64_t lda, int n, double* out) {
    __shared__ double sh[32];
    double m = DBL_MAX;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmin(m, fabs(A[(int64_t)i * lda + i]));
    m = -block_max(-m, sh);
    if (threadIdx.x == 0) *out = m;
}

}  // namespace

void launch_qr_r(const QrTask* d_tasks, int32_t ntasks, cudaStream_t st) {
    if (ntasks <= 0) return;
    qr_r_kernel<<<ntasks, DT, 0, st>>>(d_tasks);
    count_launch();
}

void launch_jacobi(const SvdTask* d_tasks, int32_t ntasks, double thresh, cudaStream_t st) {
    if (ntasks <= 0) return;
    // sig[m] + rank[m] with m <= 2048
    const size_t smem = 2048 * (sizeof(double) + sizeof(int));
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    jacobi_kernel<<<ntasks, DT, smem, st>>>(d_tasks, thresh);
    count_launch();
}

void launch_complement(const ComplementTask* d_tasks, int32_t ntasks, cudaStream_t st) {
    if (ntasks <= 0) return;
    const size_t smem = 2048 * sizeof(double);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(complement_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
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
    trsm_unit_lower_rows_kernel<<<(ncols + 127) / 128, 128, 0, st>>>(const_cast<double*>(A), lda, k0,
                                                                      nb, c0, ncols);
    count_launch();
}

void launch_absmax(const double* A, int64_t lda, int32_t rows, int32_t cols, double* out,
                   cudaStream_t st) {
    absmax_kernel<<<1, 1024, 0, st>>>(A, lda, rows, cols, out);
    count_launch();
}

void launch_diag_absmin(const double* A, int64_t lda, int32_t n, double* out, cudaStream_t st) {
    diag_absmin_kernel<<<1, 1024, 0, st>>>(A, lda, n, out);
    count_launch();
}

}  // namespace h2f
