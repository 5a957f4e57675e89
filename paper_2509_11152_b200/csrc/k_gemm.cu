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
#include <cstdlib>

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
gemm_tasks_v1_kernel(const GemmTask* __restrict__ tasks, const GemmContrib* __restrict__ contribs,
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

// ---- v2: cp.async multi-stage pipeline over the concatenated K of all
// contributions of a tile (no pipeline restart between contributions); the
// operands are staged in their stored orientation with conflict-free padded
// strides, alpha (uniform per task) is applied in the epilogue.
constexpr int BK2 = 32, STAGES = 3;
constexpr int LDK2 = BK2 + 4;   // [m][k] / [n][k] layouts (k contiguous)
constexpr int LDM2 = BM + 4;    // [k][m] / [k][n] layouts
constexpr int STAGE_ELEMS = (BM * LDK2 > BK2 * LDM2 ? BM * LDK2 : BK2 * LDM2);
constexpr size_t GEMM2_SMEM = sizeof(double) * 2 * STAGES * STAGE_ELEMS;

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(valid ? src : nullptr), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// stage one BK2 chunk of contribution P (k offset k0) into As/Bs
__device__ __forceinline__ void stage_chunk(const GemmContrib& P, int M, int N, int m0, int n0, int k0,
                                            double* As, double* Bs) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < (BM * BK2) / GEMM_THREADS; ++i) {
        const int e = tid + GEMM_THREADS * i;
        if (P.transA) {  // stored K x M: [k][m]
            const int k = e / BM, m = e % BM;
            const bool v = (k0 + k < P.K) && (m0 + m < M);
            cp_async8(As + k * LDM2 + m, P.A + (int64_t)(k0 + k) * P.lda + m0 + m, v);
        } else {         // stored M x K: [m][k]
            const int m = e / BK2, k = e % BK2;
            const bool v = (k0 + k < P.K) && (m0 + m < M);
            cp_async8(As + m * LDK2 + k, P.A + (int64_t)(m0 + m) * P.lda + k0 + k, v);
        }
    }
#pragma unroll
    for (int i = 0; i < (BN * BK2) / GEMM_THREADS; ++i) {
        const int e = tid + GEMM_THREADS * i;
        if (P.transB) {  // stored N x K: [n][k]
            const int n = e / BK2, k = e % BK2;
            const bool v = (k0 + k < P.K) && (n0 + n < N);
            cp_async8(Bs + n * LDK2 + k, P.B + (int64_t)(n0 + n) * P.ldb + k0 + k, v);
        } else {         // stored K x N: [k][n]
            const int k = e / BN, n = e % BN;
            const bool v = (k0 + k < P.K) && (n0 + n < N);
            cp_async8(Bs + k * LDM2 + n, P.B + (int64_t)(k0 + k) * P.ldb + n0 + n, v);
        }
    }
}

template <bool TA, bool TB>
__device__ __forceinline__ void mma_chunk(const double* __restrict__ As, const double* __restrict__ Bs,
                                          double (&acc)[4][4][2], int wm, int wn, int g, int t) {
#pragma unroll
    for (int kk = 0; kk < BK2; kk += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int m = wm * 32 + i * 8 + g;
            a[i] = TA ? As[(kk + t) * LDM2 + m] : As[m * LDK2 + kk + t];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = wn * 32 + j * 8 + g;
            b[j] = TB ? Bs[n * LDK2 + kk + t] : Bs[(kk + t) * LDM2 + n];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
}

__global__ void __launch_bounds__(GEMM_THREADS, 2)
gemm_tasks_kernel(const GemmTask* __restrict__ tasks, const GemmContrib* __restrict__ contribs,
                  const int64_t* __restrict__ tile_start, int ntasks, int64_t ntiles,
                  double* __restrict__ norms) {
    extern __shared__ __align__(16) double gsm[];
    __shared__ double red[GEMM_THREADS / 32];
    __shared__ int chunk_contrib[STAGES], chunk_k0[STAGES];

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

        // producer cursor over (contribution, k0) chunks
        int64_t pc = T.contrib_begin;
        int pk = 0;
        auto advance = [&]() {
            pk += BK2;
            if (pk >= contribs[pc].K) {
                pk = 0;
                ++pc;
                while (pc < T.contrib_end && contribs[pc].K <= 0) ++pc;
            }
        };
        while (pc < T.contrib_end && contribs[pc].K <= 0) ++pc;
        // prologue: STAGES - 1 chunks in flight
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (pc < T.contrib_end) {
                const GemmContrib P = contribs[pc];
                double* As = gsm + (2 * s) * STAGE_ELEMS;
                stage_chunk(P, T.M, T.N, m0, n0, pk, As, As + STAGE_ELEMS);
                if (threadIdx.x == 0) {
                    chunk_contrib[s] = (int)(pc - T.contrib_begin);
                    chunk_k0[s] = pk;
                }
                advance();
            } else if (threadIdx.x == 0) {
                chunk_contrib[s] = -1;
            }
            cp_async_commit();
        }
        for (int it = 0;; ++it) {
            const int cur = it % STAGES;
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            const int cc = chunk_contrib[cur];
            if (cc < 0) break;
            // refill the stage consumed last iteration
            {
                const int nxt = (it + STAGES - 1) % STAGES;
                if (pc < T.contrib_end) {
                    const GemmContrib P = contribs[pc];
                    double* As = gsm + (2 * nxt) * STAGE_ELEMS;
                    stage_chunk(P, T.M, T.N, m0, n0, pk, As, As + STAGE_ELEMS);
                    if (threadIdx.x == 0) {
                        chunk_contrib[nxt] = (int)(pc - T.contrib_begin);
                        chunk_k0[nxt] = pk;
                    }
                    advance();
                } else if (threadIdx.x == 0) {
                    chunk_contrib[nxt] = -1;
                }
                cp_async_commit();
            }
            const GemmContrib P = contribs[T.contrib_begin + cc];
            const double* As = gsm + (2 * cur) * STAGE_ELEMS;
            const double* Bs = As + STAGE_ELEMS;
            // zero-filled tails add exact zeros: no k bound inside the chunk
            switch (P.transA * 2 + P.transB) {
            case 0: mma_chunk<false, false>(As, Bs, acc, wm, wn, g, t); break;
            case 1: mma_chunk<false, true>(As, Bs, acc, wm, wn, g, t); break;
            case 2: mma_chunk<true, false>(As, Bs, acc, wm, wn, g, t); break;
            default: mma_chunk<true, true>(As, Bs, acc, wm, wn, g, t); break;
            }
        }
        cp_async_wait<0>();
        const double alpha = (T.contrib_end > T.contrib_begin) ? contribs[T.contrib_begin].alpha : 1.0;

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
                        const double v = alpha * acc[i][j][q];
                        if (row < T.M && col < T.N) ss += v * v;
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
                            const double v = alpha * acc[i][j][q];
                            if (T.mode == GEMM_ADD) crow[col] += v; else crow[col] = v;
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
    static const bool v1 = std::getenv("H2F_GEMM_V1") != nullptr;
    if (v1) {
        gemm_tasks_v1_kernel<<<grid_for(ntiles, 8), GEMM_THREADS, 0, st>>>(d_tasks, d_contribs, d_tile_start,
                                                                          ntasks, ntiles, d_norms);
    } else {
        static bool configured = false;
        if (!configured) {
            cudaFuncSetAttribute(gemm_tasks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM2_SMEM);
            configured = true;
        }
        gemm_tasks_kernel<<<grid_for(ntiles, 2), GEMM_THREADS, GEMM2_SMEM, st>>>(d_tasks, d_contribs, d_tile_start,
                                                                                 ntasks, ntiles, d_norms);
    }
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
