// Kernel micro-benchmark (development aid): the batched DMMA GEMM on the task
// shapes the factorization produces, checked against a naive FP64 kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_11152_b200/csrc -I include \
//        scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "kernels.h"

using namespace h2f;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

__global__ void naive_kernel(const GemmTask* tasks, const GemmContrib* cs, int ntasks, double* out_base,
                             const int64_t* out_off) {
    const GemmTask T = tasks[blockIdx.y];
    double* out = out_base + out_off[blockIdx.y];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)T.M * T.N;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = int(e / T.N), j = int(e % T.N);
        double acc = 0.0;
        for (int64_t c = T.contrib_begin; c < T.contrib_end; ++c) {
            const GemmContrib P = cs[c];
            double s = 0.0;
            for (int k = 0; k < P.K; ++k) {
                const double a = P.transA ? P.A[(int64_t)k * P.lda + i] : P.A[(int64_t)i * P.lda + k];
                const double b = P.transB ? P.B[(int64_t)j * P.ldb + k] : P.B[(int64_t)k * P.ldb + j];
                s += a * b;
            }
            acc += P.alpha * s;
        }
        out[e] = acc;
    }
}

struct Case {
    std::string name;
    int ntargets, M, N, ncontrib, K, transA, transB;
};

int main(int argc, char** argv) {
    const char* only = argc > 1 ? argv[1] : nullptr;
    std::vector<Case> cases = {
        {"schur_leaf_r13_47x47_x1", 8000, 47, 47, 1, 13, 1, 0},
        {"schur_leaf_r13_47x47_x3", 8000, 47, 47, 3, 13, 1, 0},
        {"schur_r24_60x60_x2", 8000, 60, 60, 2, 24, 1, 0},
        {"schur_r10_64x64_x6", 8000, 64, 64, 6, 10, 1, 0},
        {"schur_r8_48x48_x4", 8000, 48, 48, 4, 8, 1, 0},
        {"schur_r40_110x110_x2", 3000, 110, 110, 2, 40, 1, 0},
        {"schur_r150_300x300_x3", 60, 300, 300, 3, 150, 1, 0},
        {"schur_r60_120x120_x4", 400, 120, 120, 4, 60, 1, 0},
        {"schur_r300_500x500_x2", 12, 500, 500, 2, 300, 1, 0},
        {"proj_400x400_k400", 24, 400, 400, 1, 400, 1, 0},
        {"qr_splitk_32x358_k1024", 24, 32, 358, 1, 1024, 0, 1},
        {"qr_update_358x24000_k32", 1, 358, 24000, 1, 32, 1, 0},
    };
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    for (auto& cs : cases) {
        if (only && cs.name.find(only) == std::string::npos) continue;
        // operands: one A and B pool per contribution
        const int64_t asz = int64_t(cs.M) * cs.K, bsz = int64_t(cs.K) * cs.N;
        const int64_t npairs = int64_t(cs.ntargets) * cs.ncontrib;
        std::vector<double> h((asz + bsz) * npairs);
        for (auto& v : h) v = nd(rng);
        double *dAB, *dC, *dC0, *dRef;
        CK(cudaMalloc(&dAB, h.size() * 8));
        CK(cudaMemcpy(dAB, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
        const int64_t csz = int64_t(cs.M) * cs.N;
        CK(cudaMalloc(&dC, csz * cs.ntargets * 8));
        CK(cudaMalloc(&dC0, csz * cs.ntargets * 8));
        CK(cudaMalloc(&dRef, csz * cs.ntargets * 8));
        CK(cudaMemset(dC0, 0, csz * cs.ntargets * 8));
        std::vector<GemmTask> tasks;
        std::vector<GemmContrib> cons;
        std::vector<int64_t> start{0}, off;
        for (int t = 0; t < cs.ntargets; ++t) {
            GemmTask T{};
            T.C = dC + csz * t;
            T.ldc = cs.N;
            T.M = cs.M;
            T.N = cs.N;
            T.mode = GEMM_ADD;
            T.tiles_n = (cs.N + 63) / 64;
            T.contrib_begin = int64_t(cons.size());
            for (int c = 0; c < cs.ncontrib; ++c) {
                const int64_t p = int64_t(t) * cs.ncontrib + c;
                GemmContrib P{};
                P.A = dAB + p * (asz + bsz);
                P.B = P.A + asz;
                P.transA = cs.transA;
                P.transB = cs.transB;
                P.lda = cs.transA ? cs.M : cs.K;
                P.ldb = cs.transB ? cs.K : cs.N;
                P.K = cs.K;
                P.alpha = -1.0;
                cons.push_back(P);
            }
            T.contrib_end = int64_t(cons.size());
            tasks.push_back(T);
            start.push_back(start.back() + int64_t((cs.M + 63) / 64) * T.tiles_n);
            off.push_back(csz * t);
        }
        GemmTask* dT;
        GemmContrib* dCs;
        int64_t *dS, *dOff;
        CK(cudaMalloc(&dT, tasks.size() * sizeof(GemmTask)));
        CK(cudaMalloc(&dCs, cons.size() * sizeof(GemmContrib)));
        CK(cudaMalloc(&dS, start.size() * 8));
        CK(cudaMalloc(&dOff, off.size() * 8));
        CK(cudaMemcpy(dT, tasks.data(), tasks.size() * sizeof(GemmTask), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dCs, cons.data(), cons.size() * sizeof(GemmContrib), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dS, start.data(), start.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dOff, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
        // reference
        naive_kernel<<<dim3(64, cs.ntargets), 256>>>(dT, dCs, cs.ntargets, dRef, dOff);
        CK(cudaDeviceSynchronize());
        // timed: C = 0 + sum, each kernel variant (0: 3-stage smem pipeline,
        // 1: C-prefetch pipeline, 2: register-direct short-K)
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int reps = 20;
        std::vector<double> first;
        for (int variant = 0; variant < 3; ++variant) {
            float best = 1e30f;
            for (int r = 0; r < reps; ++r) {
                CK(cudaMemcpy(dC, dC0, csz * cs.ntargets * 8, cudaMemcpyDeviceToDevice));
                cudaEventRecord(e0);
                if (variant == 2)
                    launch_gemm_warp(dT, dCs, dS, int(tasks.size()), start.back(), nullptr, 0);
                else
                    launch_gemm_tasks(dT, dCs, dS, int(tasks.size()), start.back(), nullptr, nullptr, 0,
                                      variant == 1);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = std::min(best, ms);
            }
            std::vector<double> c(csz * cs.ntargets), ref(csz * cs.ntargets);
            CK(cudaMemcpy(c.data(), dC, c.size() * 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(ref.data(), dRef, ref.size() * 8, cudaMemcpyDeviceToHost));
            double err = 0, nrm = 0;
            for (size_t i = 0; i < c.size(); ++i) {
                err = std::max(err, std::fabs(c[i] - ref[i]));
                nrm = std::max(nrm, std::fabs(ref[i]));
            }
            bool same = true;
            if (variant == 0) first = c;
            else same = (c == first);
            const double flops = 2.0 * cs.M * cs.N * cs.K * double(npairs);
            const double bytes = 16.0 * csz * cs.ntargets;
            std::printf("%-28s v%d %8.3f ms  %7.2f TF/s  C-rmw %7.1f GB/s  rel.err %.2e  bits==v0 %d\n",
                        cs.name.c_str(), variant, best, flops / best / 1e9, bytes / best / 1e6, err / nrm,
                        int(same));
        }
        cudaFree(dAB);
        cudaFree(dC);
        cudaFree(dC0);
        cudaFree(dRef);
        cudaFree(dT);
        cudaFree(dCs);
        cudaFree(dS);
        cudaFree(dOff);
    }
    return 0;
}
