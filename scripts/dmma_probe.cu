// DMMA throughput probe: warps per SM x independent accumulator chains, with and without smem fragment loads
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int NI, int NJ, bool LDS>
__global__ void k(int iters, double* out) {
    __shared__ double sm[2][64 * 36];
    for (int i = threadIdx.x; i < 2 * 64 * 36; i += blockDim.x) (&sm[0][0])[i] = 1.0 + i * 1e-9;
    __syncthreads();
    double c[NI][NJ][2];
    for (int i = 0; i < NI; ++i) for (int j = 0; j < NJ; ++j) c[i][j][0] = c[i][j][1] = 0;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
    double a[NI], b[NJ];
    for (int i = 0; i < NI; ++i) a[i] = 1.0 + 1e-3 * i;
    for (int j = 0; j < NJ; ++j) b[j] = 1.0 - 1e-3 * j;
    for (int it = 0; it < iters; ++it) {
        for (int kk = 0; kk < 32; kk += 4) {
            if (LDS) {
#pragma unroll
                for (int i = 0; i < NI; ++i) a[i] = sm[0][(((w & 1) * 32 + i * 8 + g) & 63) * 36 + kk + t];
#pragma unroll
                for (int j = 0; j < NJ; ++j) b[j] = sm[1][(((w >> 1) * 16 + j * 8 + g) & 63) * 36 + kk + t];
            }
#pragma unroll
            for (int i = 0; i < NI; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(c[i][j][0], c[i][j][1], a[i], b[j]);
        }
    }
    double s = 0;
    for (int i = 0; i < NI; ++i) for (int j = 0; j < NJ; ++j) s += c[i][j][0] + c[i][j][1];
    if (s == 1.2345) out[threadIdx.x] = s;
}
template <int NI, int NJ, bool LDS>
void run(int ctas_per_sm, int threads, const char* name) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) { printf("attr fail\n"); return; }
    double* out = nullptr;
    if (cudaMalloc(&out, 1024 * 8) != cudaSuccess) { printf("malloc fail\n"); return; }
    int iters = 2000;
    k<NI, NJ, LDS><<<sms * ctas_per_sm, threads>>>(10, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<NI, NJ, LDS><<<sms * ctas_per_sm, threads>>>(iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaError_t err = cudaGetLastError(); if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); return; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = double(sms) * ctas_per_sm * (threads / 32) * iters * 8.0 * NI * NJ * 512.0;
    printf("%-34s ctas/sm %d threads %d warps/sm %2d: %6.2f TF/s\n", name, ctas_per_sm, threads, ctas_per_sm * threads / 32, flops / ms / 1e9);
}
int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    printf("start\n");
    run<4, 4, false>(2, 128, "4x4 chains, no lds");
    run<4, 4, true>(2, 128, "4x4 chains, lds (gemm-like)");
    run<4, 4, true>(3, 128, "4x4 chains, lds");
    run<4, 4, true>(4, 128, "4x4 chains, lds");
    run<4, 2, true>(2, 256, "4x2 chains, lds");
    run<4, 2, true>(4, 256, "4x2 chains, lds");
    run<4, 4, false>(4, 128, "4x4 chains, no lds");
    run<4, 4, false>(8, 128, "4x4 chains, no lds");
    run<2, 4, false>(2, 128, "2x4 chains, no lds");
    run<8, 4, true>(2, 128, "8x4 chains, lds");
    return 0;
}
