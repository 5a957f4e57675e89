// Batched per-cluster dense linear algebra, host orchestration (the large-n
// paths of the augmentation, factorization.py:62-99).
#pragma once
#include <vector>

#include "kernels.h"
#include "runtime.h"

namespace h2f {

// One matrix of a batched blocked Householder QR.  Column j lives at
// M + j*ldm with its L rows contiguous (e.g. the rows of a row-major Z are
// the columns of Z^T).  Columns [0, nfac) are factored; the trailing
// updates reach columns [0, ntot).  With keep=true the per-panel Vt / T are
// retained for hh_apply_q.
struct HhJob {
    double* M = nullptr;
    int64_t ldm = 0;
    int L = 0, ntot = 0, nfac = 0;
    std::vector<double*> Vt, T;  // per panel (keep=true)
    // non-null: block column pivoting -- before each panel the trailing
    // columns are reordered by their remaining norms; perm[c] = original
    // column now at position c (device, ntot entries)
    int32_t* perm = nullptr;
};

void hh_factor(std::vector<HhJob>& jobs, Region& scr, bool keep);

// X <- Q X with Q = H_0 ... H_{nfac-1} of job i; X_i is L x nx, row-major ld ldx
struct HhApply {
    double* X;
    int64_t ldx;
    int nx;
};
void hh_apply_q(const std::vector<HhJob>& jobs, const std::vector<HhApply>& xs, Region& scr);

// R of the QR of Y^T for the QrTasks (Y is n x wf, row-major; overwritten):
// written as a full n x n row-major block, rows >= min(n, wf) zero -- callers
// allocate n x n even when wf < n (as does the shared-memory TSQR)
void qr_r_blocked(const std::vector<QrTask>& tasks, Region& scr, const std::vector<int32_t*>* perms = nullptr);

// Q~ = [complement | b_aug] for each task (factorization.py:88-99), blocked
void complement_blocked(const std::vector<ComplementTask>& tasks, Region& scr);

// one-sided Jacobi SVD of large R's with several co-resident CTAs per cluster
// (block-cyclic; pairwise = one group barrier per round-robin step).  With
// flags_out, flags_out[i][63] receives the sweep count of task i (device).
void jacobi_multi_cta(const std::vector<SvdTask>& tasks, double thresh, Region& scr, bool pairwise = false,
                      std::vector<int32_t*>* flags_out = nullptr);

// factorization.py:82-84 for a batch: the kept rows u of BT (rows k..k+kept)
// get u -= V (V^T u) (two batched DMMA GEMMs) and u /= |u|
void reorth_batched(const std::vector<ReorthTask>& tasks, Region& scr);

// partial-pivot LU of the n x n row-major A in place (LAPACK getrf pivots,
// 0-based): cooperative panels + DMMA trailing updates.  red[0] = max|A|
// before, red[1] = min|diag(U)| after (device; the vanishing-pivot test).
void blocked_lu(double* A, int64_t n, int32_t* piv, Region& scr, double* red, int kid_panel, int kid_misc,
                int kid_gemm);

}  // namespace h2f
