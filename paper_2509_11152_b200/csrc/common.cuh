// Small device helpers shared by the kernel files.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace h2f {

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).  On sm_100a this
// lowers to SASS DMMA.8x8x4 (tcgen05 has no f64 kind).
// Fragment ownership (lane = 4*g + t):  a = A[g][t], b = B[t][g],
// c0,c1 = C[g][2t], C[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// block-wide sum, result broadcast to all threads; `sh` needs blockDim/32 slots
__device__ __forceinline__ double block_sum(double v, double* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += sh[i];  // fixed order: deterministic
    return s;
}

__device__ __forceinline__ double block_max(double v, double* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = sh[0];
    for (int i = 1; i < nw; ++i) s = fmax(s, sh[i]);
    return s;
}

// largest i in [0, n) with start[i] <= t (start is a nondecreasing prefix)
__device__ __forceinline__ int find_segment(const int64_t* start, int n, int64_t t) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (start[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

}  // namespace h2f
