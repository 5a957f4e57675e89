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

constexpr int BM = 64, BN = 64;
constexpr int GEMM_THREADS = 128;


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

// One CTA walks a contiguous range of tiles as a single stream of K chunks
// (tile -> contributions in order -> BK2 chunks): the producer issues cp.async
// STAGES-1 chunks ahead across contribution and tile boundaries, so the
// descriptor loads and the next tile's operand loads overlap the current
// tile's math and epilogue.  Per-stage metadata (contribution, tile origin,
// last-chunk-of-tile flag) travels with the stage through shared memory.
struct ChunkMeta {
    int contrib;  // global contribution index; -1: stream ended; -2: tile without contributions
    int ti;       // task
    int m0, n0;
    int last;     // last chunk of its tile: run the epilogue after it
    int pad_;
    int64_t local;  // tile index within the task
};

__global__ void __launch_bounds__(GEMM_THREADS, 2)
gemm_tasks_kernel(const GemmTask* __restrict__ tasks, const GemmContrib* __restrict__ contribs,
                  const int64_t* __restrict__ tile_start, int ntasks, int64_t ntiles,
                  double* __restrict__ norms) {
    extern __shared__ __align__(16) double gsm[];
    __shared__ double red[GEMM_THREADS / 32];
    __shared__ ChunkMeta meta[STAGES];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;

    const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_begin = (int64_t)blockIdx.x * per, t_end = min(ntiles, t_begin + per);
    if (t_begin >= t_end) return;

    // ---- producer cursor (uniform across the CTA) ----
    int64_t p_tile = t_begin;
    int p_ti = find_segment(tile_start, ntasks, t_begin);
    int64_t p_pc = 0, p_end = 0;
    int p_pk = 0, p_m0 = 0, p_n0 = 0, p_M = 0, p_N = 0;
    int64_t p_local = 0;
    auto open_tile = [&]() {
        while (p_ti + 1 < ntasks && p_tile >= tile_start[p_ti + 1]) ++p_ti;
        const GemmTask& T = tasks[p_ti];
        p_local = p_tile - tile_start[p_ti];
        p_m0 = (int)(p_local / T.tiles_n) * BM;
        p_n0 = (int)(p_local % T.tiles_n) * BN;
        p_M = T.M;
        p_N = T.N;
        p_pc = T.contrib_begin;
        p_end = T.contrib_end;
        p_pk = 0;
        while (p_pc < p_end && contribs[p_pc].K <= 0) ++p_pc;
    };
    open_tile();
    auto issue = [&](int stage) {
        ChunkMeta m{};
        if (p_tile >= t_end) {
            m.contrib = -1;
        } else if (p_pc >= p_end) {  // tile without contributions: epilogue only
            m.contrib = -2;
            m.ti = p_ti;
            m.m0 = p_m0;
            m.n0 = p_n0;
            m.local = p_local;
            m.last = 1;
            ++p_tile;
            if (p_tile < t_end) open_tile();
        } else {
            const GemmContrib P = contribs[p_pc];
            double* As = gsm + (2 * stage) * STAGE_ELEMS;
            stage_chunk(P, p_M, p_N, p_m0, p_n0, p_pk, As, As + STAGE_ELEMS);
            m.contrib = (int)p_pc;
            m.ti = p_ti;
            m.m0 = p_m0;
            m.n0 = p_n0;
            m.local = p_local;
            p_pk += BK2;
            if (p_pk >= P.K) {
                p_pk = 0;
                ++p_pc;
                while (p_pc < p_end && contribs[p_pc].K <= 0) ++p_pc;
            }
            m.last = p_pc >= p_end;
            if (m.last) {
                ++p_tile;
                if (p_tile < t_end) open_tile();
            }
        }
        if (threadIdx.x == 0) meta[stage] = m;
        cp_async_commit();
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) issue(st);
    for (int it = 0;; ++it) {
        const int cur = it % STAGES;
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const ChunkMeta m = meta[cur];
        if (m.contrib == -1) break;
        issue((it + STAGES - 1) % STAGES);  // refills the stage consumed last iteration
        if (m.contrib >= 0) {
            const GemmContrib P = contribs[m.contrib];
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
        if (!m.last) continue;
        // ---- epilogue of tile m ----
        const GemmTask T = tasks[m.ti];
        const double alpha = (T.contrib_end > T.contrib_begin) ? contribs[T.contrib_begin].alpha : 1.0;
        if (T.mode == GEMM_NORM) {
            double ss = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int row = m.m0 + wm * 32 + i * 8 + g;
                        const int col = m.n0 + wn * 32 + j * 8 + 2 * t + q;
                        const double v = alpha * acc[i][j][q];
                        if (row < T.M && col < T.N) ss += v * v;
                    }
            // block_sum's barriers are uniform: every thread reaches this epilogue
            ss = block_sum(ss, red);
            if (threadIdx.x == 0) norms[T.norm_base + m.local] = ss;
        } else {
            // all loads of the tile's C first (one memory round trip), then
            // the stores: the compiler cannot hoist loads over possibly
            // aliasing stores on its own
            double cv[4][4][2];
            if (T.mode == GEMM_ADD) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int row = m.m0 + wm * 32 + i * 8 + g;
                    const double* crow = T.C + (int64_t)row * T.ldc;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const int col = m.n0 + wn * 32 + j * 8 + 2 * t + q;
                            cv[i][j][q] = (row < T.M && col < T.N) ? crow[col] : 0.0;
                        }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = m.m0 + wm * 32 + i * 8 + g;
                if (row >= T.M) continue;
                double* crow = T.C + (int64_t)row * T.ldc;
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int col = m.n0 + wn * 32 + j * 8 + 2 * t + q;
                        if (col < T.N) {
                            const double v = alpha * acc[i][j][q];
                            crow[col] = T.mode == GEMM_ADD ? cv[i][j][q] + v : v;
                        }
                    }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    cp_async_wait<0>();
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
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(gemm_tasks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM2_SMEM);
        configured = true;
    }
    gemm_tasks_kernel<<<grid_for(ntiles, 2), GEMM_THREADS, GEMM2_SMEM, st>>>(d_tasks, d_contribs, d_tile_start,
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
