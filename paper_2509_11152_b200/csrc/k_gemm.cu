// Batched variable-size FP64 tile GEMM on DMMA tensor cores, and batched
// (transposing) block copies.
//
// These two kernels carry every block-level contraction of the path:
//   * basis augmentation residual  Y -= V (V^T Y)        factorization.py:77
//   * projection  Q~^T B, B Q~                           factorization.py:420-427
//   * Schur updates  -g_i^T W_j  fused with the scatter-add into the target
//     block and the fill-candidate Frobenius norm       factorization.py:122-126, 476-505
//   * fill creation and the dense-top trailing update   factorization.py:502-505, 259-261
// One CTA owns one 64x64 output tile and sums its ordered contribution list
// in registers before a single read-modify-write of the target, so a target
// shared by several clusters of a batch is updated without atomics and in a
// fixed order (run-to-run bitwise deterministic).
#include "common.cuh"
#include "kernels.h"

namespace h2f {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, PADS = 8, LDS = BM + PADS;
constexpr int GEMM_THREADS = 128;

struct Frag {
    double a[8];
    double b[8];
};

__device__ __forceinline__ void load_tile(const GemmContrib& P, int M, int N, int m0, int n0,
                                          int k0, Frag& f) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = tid + GEMM_THREADS * i;
        int k, m;
        if (P.transA) { k = e >> 6; m = e & 63; } else { k = e & 15; m = e >> 4; }
        const int gk = k0 + k, gm = m0 + m;
        double v = 0.0;
        if (gk < P.K && gm < M)
            v = P.transA ? __ldg(P.A + (int64_t)gk * P.lda + gm) : __ldg(P.A + (int64_t)gm * P.lda + gk);
        f.a[i] = v * P.alpha;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = tid + GEMM_THREADS * i;
        int k, n;
        if (P.transB) { k = e & 15; n = e >> 4; } else { k = e >> 6; n = e & 63; }
        const int gk = k0 + k, gn = n0 + n;
        double v = 0.0;
        if (gk < P.K && gn < N)
            v = P.transB ? __ldg(P.B + (int64_t)gn * P.ldb + gk) : __ldg(P.B + (int64_t)gk * P.ldb + gn);
        f.b[i] = v;
    }
}

__device__ __forceinline__ void store_tile(const GemmContrib& P, const Frag& f,
                                           double (*As)[LDS], double (*Bs)[LDS]) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = tid + GEMM_THREADS * i;
        int k, m;
        if (P.transA) { k = e >> 6; m = e & 63; } else { k = e & 15; m = e >> 4; }
        As[k][m] = f.a[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = tid + GEMM_THREADS * i;
        int k, n;
        if (P.transB) { k = e & 15; n = e >> 4; } else { k = e >> 6; n = e & 63; }
        Bs[k][n] = f.b[i];
    }
}

__global__ void __launch_bounds__(GEMM_THREADS)
gemm_tasks_kernel(const GemmTask* __restrict__ tasks, const GemmContrib* __restrict__ contribs,
                  const int64_t* __restrict__ tile_start, int ntasks, int64_t ntiles,
                  double* __restrict__ norms) {
    __shared__ __align__(16) double As[2][BK][LDS];
    __shared__ __align__(16) double Bs[2][BK][LDS];
    __shared__ double red[GEMM_THREADS / 32];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ti = find_segment(tile_start, ntasks, tile);
        const GemmTask T = tasks[ti];
        const int64_t local = tile - tile_start[ti];
        const int m0 = (int)(local / T.tiles_n) * BM;
        const int n0 = (int)(local % T.tiles_n) * BN;

        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (int64_t ci = T.contrib_begin; ci < T.contrib_end; ++ci) {
            const GemmContrib P = contribs[ci];
            const int nk = (P.K + BK - 1) / BK;
            if (nk == 0) continue;
            Frag f;
            load_tile(P, T.M, T.N, m0, n0, 0, f);
            store_tile(P, f, As[0], Bs[0]);
            __syncthreads();
            for (int kc = 0; kc < nk; ++kc) {
                const int cur = kc & 1;
                if (kc + 1 < nk) load_tile(P, T.M, T.N, m0, n0, (kc + 1) * BK, f);
#pragma unroll
                for (int kk = 0; kk < BK; kk += 4) {
                    double a[4], b[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i] = As[cur][kk + t][wm * 32 + i * 8 + g];
#pragma unroll
                    for (int j = 0; j < 4; ++j) b[j] = Bs[cur][kk + t][wn * 32 + j * 8 + g];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
                }
                if (kc + 1 < nk) store_tile(P, f, As[cur ^ 1], Bs[cur ^ 1]);
                __syncthreads();
            }
        }

        if (T.mode == GEMM_NORM) {
            double ss = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int row = m0 + wm * 32 + i * 8 + g;
                        const int col = n0 + wn * 32 + j * 8 + 2 * t + q;
                        if (row < T.M && col < T.N) ss += acc[i][j][q] * acc[i][j][q];
                    }
            ss = block_sum(ss, red);
            if (threadIdx.x == 0) norms[T.norm_base + local] = ss;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = m0 + wm * 32 + i * 8 + g;
                if (row >= T.M) continue;
                double* crow = T.C + (int64_t)row * T.ldc;
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int col = n0 + wn * 32 + j * 8 + 2 * t + q;
                        if (col < T.N) {
                            if (T.mode == GEMM_ADD) crow[col] += acc[i][j][q];
                            else crow[col] = acc[i][j][q];
                        }
                    }
            }
        }
        __syncthreads();
    }
}

constexpr int CT = 32;  // copy tile

__global__ void __launch_bounds__(256)
copy_tasks_kernel(const CopyTask* __restrict__ tasks, const int64_t* __restrict__ tile_start,
                  int ntasks, int64_t ntiles) {
    __shared__ double sh[CT][CT + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ti = find_segment(tile_start, ntasks, tile);
        const CopyTask T = tasks[ti];
        const int64_t local = tile - tile_start[ti];
        const int tn = (T.cols + CT - 1) / CT;
        const int r0 = (int)(local / tn) * CT, c0 = (int)(local % tn) * CT;
        if (T.mode == COPY_ZERO) {
            for (int i = ty; i < CT; i += 8) {
                const int r = r0 + i, c = c0 + tx;
                if (r < T.rows && c < T.cols) T.dst[(int64_t)r * T.ldd + c] = 0.0;
            }
            continue;
        }
        if (!T.trans) {
            for (int i = ty; i < CT; i += 8) {
                const int r = r0 + i, c = c0 + tx;
                if (r < T.rows && c < T.cols) {
                    const double v = T.alpha * T.src[(int64_t)r * T.lds + c];
                    double* d = T.dst + (int64_t)r * T.ldd + c;
                    if (T.mode == COPY_ADD) *d += v; else *d = v;
                }
            }
        } else {
            // dst(r, c) = src(c, r): read src rows c0.., columns r0..
            for (int i = ty; i < CT; i += 8) {
                const int sr = c0 + i, sc = r0 + tx;
                sh[i][tx] = (sr < T.cols && sc < T.rows) ? T.src[(int64_t)sr * T.lds + sc] : 0.0;
            }
            __syncthreads();
            for (int i = ty; i < CT; i += 8) {
                const int r = r0 + i, c = c0 + tx;
                if (r < T.rows && c < T.cols) {
                    const double v = T.alpha * sh[tx][i];
                    double* d = T.dst + (int64_t)r * T.ldd + c;
                    if (T.mode == COPY_ADD) *d += v; else *d = v;
                }
            }
            __syncthreads();
        }
    }
}

__global__ void sumsq_reduce_kernel(const double* __restrict__ parts, const int64_t* __restrict__ seg,
                                    int nseg, double* __restrict__ out) {
    // one warp per segment; fixed lane-strided order -> deterministic
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= nseg) return;
    double s = 0.0;
    for (int64_t i = seg[w] + lane; i < seg[w + 1]; i += 32) s += parts[i];
    s = warp_sum(s);
    if (lane == 0) out[w] = s;
}

__global__ void __launch_bounds__(128) dmma_peak_kernel(int64_t iters, double* out) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    double a = 1.0 + 1e-3 * threadIdx.x, b = 1.0 - 1e-3 * threadIdx.x;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;  // keeps the chain alive
}

int grid_for(int64_t ntiles, int per_sm) {
    const int64_t cap = (int64_t)148 * per_sm;
    return (int)(ntiles < cap ? ntiles : cap);
}

}  // namespace

void launch_gemm_tasks(const GemmTask* d_tasks, const GemmContrib* d_contribs,
                       const int64_t* d_tile_start, int32_t ntasks, int64_t ntiles,
                       double* d_norms, cudaStream_t st) {
    if (ntiles <= 0) return;
    gemm_tasks_kernel<<<grid_for(ntiles, 8), GEMM_THREADS, 0, st>>>(d_tasks, d_contribs, d_tile_start,
                                                                   ntasks, ntiles, d_norms);
    count_launch();
}

void launch_copy_tasks(const CopyTask* d_tasks, const int64_t* d_tile_start, int32_t ntasks,
                       int64_t ntiles, cudaStream_t st) {
    if (ntiles <= 0) return;
    copy_tasks_kernel<<<grid_for(ntiles, 16), 256, 0, st>>>(d_tasks, d_tile_start, ntasks, ntiles);
    count_launch();
}

double bench_dmma(int64_t iters, cudaStream_t st) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 8;
    double* out = nullptr;
    cudaMalloc(&out, 128 * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    dmma_peak_kernel<<<grid, 128, 0, st>>>(iters / 10 + 1, out);  // warm-up
    cudaEventRecord(a, st);
    dmma_peak_kernel<<<grid, 128, 0, st>>>(iters, out);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    const double flops = double(grid) * 4 /*warps*/ * double(iters) * 8 * 512.0;
    return flops / (ms * 1e-3) / 1e12;
}

void launch_sumsq_reduce(const double* d_parts, const int64_t* d_seg, int32_t nseg, double* d_out,
                         cudaStream_t st) {
    if (nseg <= 0) return;
    const int threads = 256, per = threads / 32;
    sumsq_reduce_kernel<<<(nseg + per - 1) / per, threads, 0, st>>>(d_parts, d_seg, nseg, d_out);
    count_launch();
}

}  // namespace h2f
