// Device task descriptors and kernel launchers (sm_100a).
//
// Every batched kernel consumes a flat task list built on the host by the
// scheduler (factor.cpp / solve.cpp / matvec.cpp) and uploaded once per
// launch; variable-size work is mapped to CTAs through a tile prefix sum so
// one launch covers every cluster of a batch (the B200 replacement of the
// reference's WorkerPool.map, parallel.py:16-37).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace h2f {

// ---- batched FP64 tile GEMM (DMMA m8n8k4) --------------------------------
// C[M x N] (=|+=) sum_c alpha_c * op(A_c) * op(B_c); op(A) is M x K, op(B) K x N.
// mode NORM writes, per 64x64 tile, the sum of squares of the single
// contribution's tile to norms[norm_base + tile] instead of touching C.
enum GemmMode : int32_t { GEMM_STORE = 0, GEMM_ADD = 1, GEMM_NORM = 2 };

struct GemmTask {
    double* C;
    int64_t ldc;
    int32_t M, N;
    int32_t mode;
    int32_t tiles_n;
    int64_t contrib_begin, contrib_end;
    int64_t norm_base;
};

struct GemmContrib {
    const double* A;
    const double* B;
    int64_t lda, ldb;
    int32_t K;
    int32_t transA;  // 0: A stored M x K; 1: A stored K x M
    int32_t transB;  // 0: B stored K x N; 1: B stored N x K
    int32_t pad_;
    double alpha;
};

constexpr int GEMM_TILE = 64;
constexpr int GEMM_BK = 32;   // K chunk of the GEMM pipeline

// ---- batched copy / add / zero with optional transpose --------------------
enum CopyMode : int32_t { COPY_SET = 0, COPY_ADD = 1, COPY_ZERO = 2 };

struct CopyTask {
    const double* src;
    double* dst;
    int64_t lds, ldd;
    int32_t rows, cols;   // of dst region
    int32_t trans;        // dst(i,j) = src(j,i)
    int32_t mode;
    double alpha;
};

constexpr int COPY_TILE = 32;

// ---- per-cluster dense kernels ------------------------------------------------
struct QrTask {          // R of the reduced QR of Y^T, Y is s x wf (row-major, ld)
    double* Y;           // overwritten (global path) / read (smem path)
    double* R;           // min(s,wf) x s, row-major, ld = s
    int64_t ldy;
    int32_t s, wf;
    // smem path only: fold columns [c0, c1) of Y; if ldrt > 0 write R^T to
    // R + c*ldrt + j (the stacked-R input of a second TSQR level)
    int32_t c0, c1;
    int64_t ldrt;
};

struct SvdTask {         // one-sided Jacobi on the rows of R (m x n, ld n): writes the
    double* R;           // left singular vectors u_j (length n) of R^T with
    double* U;           // sigma_j >= thresh as rows of U, sorted by sigma desc
    int32_t m, n;
    int32_t* kept_out;   // device int
    int32_t deg_off;     // != 0: kept_out[deg_off] = 1 if some sigma_j is ~0 (all m
                         // sorted rows are written; rows kept.. complete U)
};

struct ReorthTask {      // rows k..k+kept-1 of BT: u -= V (V^T u); u /= |u|
    const double* V;     // s x k, row-major ld = ldv
    double* BT;          // (k+kept) x s
    double* C;           // k x kept scratch
    int64_t ldv;
    int32_t s, k, kept;
    int32_t pad_;
};

struct ComplementTask {  // Q~ = [complement | b_aug] from BT (kt x s rows = columns of b_aug)
    const double* BT;    // kt x s, row-major ld = s
    double* W;           // kt x s workspace (Householder vectors)
    double* Q;           // s x s row-major
    double* scratch;     // 16 * s warp workspace
    int32_t s, kt;
};

struct RExtractTask {    // R[j][c] = c >= j ? Z[c][j] : 0  (j < m, c < n)
    const double* Z;
    double* R;           // n x n
    int64_t ldz;
    int32_t m, n;
};

struct CoopSvdTask {     // multi-CTA Jacobi: CTAs [cta0, cta0+ncta) own one cluster
    SvdTask t;
    int32_t cta0, ncta;
    uint32_t* bar;       // [2] barrier counter + generation
    int32_t* flags;      // [64] per-sweep rotation flags (zeroed)
    double* sig;         // [m] singular values (scratch)
};

struct LuTask {          // partial-pivot LU of the r x r view of D_cc
    const double* D;
    int64_t ldd;
    double* LU;          // r x r row-major
    int32_t* piv;        // r
    int32_t r;
    int32_t cluster;     // for the status word
    int32_t* status;     // device: cluster index that failed (first), else -1
};

// TrsmTask.mode bits (trsm_dmma_kernel): which factors of LU = P^T L U to
// apply to the column block, and the sign of the result
constexpr int32_t TRSM_LOWER = 1;   // X = L^-1 P G (pivots, unit lower)
constexpr int32_t TRSM_UPPER = 2;   // X = U^-1 X
constexpr int32_t TRSM_NEGATE = 4;  // MW = -X
constexpr int32_t TRSM_ELIMINATOR = TRSM_LOWER | TRSM_UPPER | TRSM_NEGATE;  // -W = -(LU)^-1 P G

struct TrsmTask {        // MW = op((LU)^-1 P G) column block
    const double* LU;
    const int32_t* piv;
    const double* G;     // r x W row-major, ld
    double* MW;          // r x W row-major, ld (may alias G: the block is staged first)
    int64_t ldg, ldw;
    int32_t r, W;
    int32_t col0;        // first column of this CTA chunk
    int32_t mode;        // TRSM_* bits (trsm_dmma_kernel; trsm_kernel is TRSM_ELIMINATOR only)
    int64_t ldlu;        // row stride of LU (0: r); piv == nullptr: no row interchanges
};

// ---- blocked Householder QR with a cooperative panel (k_hh.cu) ---------------------
// Matrix column j at M + j*ldm (rows contiguous).  One task = one panel of
// nbp <= HH_NB columns starting at column/row j0, spread over CTAs
// [cta0, cta0+ncta) of the grid, `chunk` rows of [j0, L) each (chunk >= HH_NB,
// multiple of 4).  Outputs: R/reflectors in place, the explicit unit-lower
// reflectors Vt (HH_NB x (L-j0), row-major) and T (HH_NB x HH_NB, dlarft).
constexpr int HH_NB = 32;
constexpr int HH_CHUNK_MAX = 840;  // rows per CTA: 32 x 844 doubles of shared memory
struct HhPanelTask {
    double* M;
    int64_t ldm;
    double* Vt;
    double* T;
    double* part;        // 2 * (ncta + 1) * (HH_NB + 2) doubles (column-parity double buffer)
    double* gram;        // ncta * HH_NB * HH_NB doubles
    uint32_t* bar;       // 2 words, zeroed
    int32_t L, j0, nbp, chunk;
    int32_t cta0, ncta;
};
struct HhTmulTask {      // out = op(T) * sum_ch P[ch]   (nrows x ncols each)
    const double* P;
    const double* T;
    double* out;
    int32_t nchunks, nrows, ncols, trans;
};
struct EyeTask {         // X[row0 + i][i] = 1, i < n
    double* X;
    int64_t ldx;
    int32_t row0, n;
};

// ---- solve -----------------------------------------------------------------------
struct SolveCluster {
    const double* q;     // s x s
    const double* lu;    // r x r
    const int32_t* piv;
    const double* mw;    // r x W eliminators (-W), row-major ld W; edges are column slices
    int64_t off;         // offset in the level vector
    int32_t s, r;
    int64_t W;
    int64_t edge_begin, edge_end;
    int64_t woff;        // work slot: (s + nch * r) * nrhs doubles (rotated vector, gather partials)
    int32_t nch;         // column chunks of the backward gather
    int32_t pad2_;
    int64_t soff;        // forward products of column j of mw go to scratch row soff + j
};

struct SolveEdge {
    const double* mat;   // r x w, row-major, ld
    int64_t ld;
    int64_t lo;          // target span start in the level vector
    int64_t soff;        // scratch offset (forward products), in rows
    int32_t w;
    int32_t pad_;
};

// one CTA of a batched substitution launch (k_solve.cu)
enum SolveTaskKind : int32_t {
    ST_ROT_T = 0,  // work[j] = (Q^T y_c)[j], j in [begin, end)            forward
    ST_PROD,       // scratch[soff + j] = (mw^T work_R)[j], j in [begin,end)  forward
    ST_LSOLVE,     // y_c = [L^-1 P work_R ; work_S]                          forward
    ST_USOLVE,     // work = [U^-1 y_R ; y_S]                                 backward
    ST_GATHER,     // part[ch][k] = sum_e (mat_e y[span_e])[k] over columns [c0,c1) = chunk ch,
                   // k in [begin,end)                                         backward
    ST_ROT,        // y_c[i] = (Q (work + [sum_ch part[ch]; 0]))[i], i in [begin, end)  backward
};
struct SolveTask {
    int32_t cl, kind, begin, end;
    int32_t c0, c1;      // ST_GATHER: eliminator column range [c0, c1)
    int32_t e0, e1;      // ST_GATHER: the cluster's edges overlapping [c0, c1) (absolute edge indices)
};
constexpr int SOLVE_GATHER_COLS = 2048;  // column chunk of one ST_GATHER task
constexpr int SOLVE_ROT_T_COLS = 64;
constexpr int SOLVE_PROD_COLS = 256;
constexpr int SOLVE_ROW_SLICE = 16;
constexpr int SOLVE_SMEM_VEC = 8192;  // doubles of shared vector space per solve CTA

struct ScatterGroup {    // y[lo : lo+w] += sum of scratch rows listed in [begin,end)
    int64_t lo;
    int32_t w;
    int32_t pad_;
    int64_t begin, end;  // into a list of scratch offsets
};

// ---- GEMV tasks (matvec sweeps, small solves) -------------------------------------
struct GemvTask {
    double* y;
    int32_t rows;
    int32_t mode;        // COPY_SET / COPY_ADD
    int64_t contrib_begin, contrib_end;
};

struct GemvContrib {
    const double* A;
    const double* x;
    int64_t lda;
    int32_t cols;
    int32_t trans;       // 0: y += A x (A rows x cols); 1: y += A^T x (A cols x rows)
    double alpha;
};

// ---- launchers (defined in the .cu files) ----------------------------------------
// grid of launch_gemm_tasks for ntiles tiles (d_cta_tiles, when given, holds
// gemm_grid(ntiles)+1 tile boundaries, one range per CTA)
int gemm_grid(int64_t ntiles);
int sm_count();  // multiprocessors of the current device (cached)
// short-K GEMM (same task lists, same bits as launch_gemm_tasks): fragments
// straight from L2, one 64x64 tile per CTA, 4 CTAs per SM
void launch_gemm_warp(const GemmTask* d_tasks, const GemmContrib* d_contribs, const int64_t* d_tile_start,
                      int32_t ntasks, int64_t ntiles, double* d_norms, cudaStream_t st, int role = 0);
// role 1 = the Schur-complement launches (a separate kernel symbol, same code)
void launch_gemm_tasks(const GemmTask* d_tasks, const GemmContrib* d_contribs,
                       const int64_t* d_tile_start, int32_t ntasks, int64_t ntiles,
                       const int64_t* d_cta_tiles, double* d_norms, cudaStream_t st, bool short_k = false,
                       int role = 0);
void launch_copy_tasks(const CopyTask* d_tasks, const int64_t* d_tile_start, int32_t ntasks,
                       int64_t ntiles, cudaStream_t st);
void launch_qr_r_smem(const QrTask* d_tasks, int32_t ntasks, int32_t max_n, cudaStream_t st);
void launch_jacobi_smem(const SvdTask* d_tasks, int32_t ntasks, int32_t max_n, double thresh, cudaStream_t st);
void launch_reorth(const ReorthTask* d_tasks, int32_t ntasks, cudaStream_t st);
struct RowNormTask {      // row /= |row| (one warp per row)
    double* p;
    int32_t len;
    int32_t pad_;
};
void launch_normalize_rows(const RowNormTask* d_tasks, int32_t nrows, cudaStream_t st);
void launch_r_extract(const RExtractTask* d_tasks, int32_t ntasks, int32_t max_n, cudaStream_t st);
// block-cyclic multi-CTA Jacobi: JB-row blocks (jacobi_block_rows), 2 blocks per CTA
int jacobi_block_rows(int n);
int jacobi_block_capacity(int max_n, int max_m);
cudaError_t launch_jacobi_block(const CoopSvdTask* d_tasks, int32_t total_ctas, const int32_t* d_cta_task,
                                int32_t max_n, int32_t max_m, double thresh, cudaStream_t st);
// multi-CTA Jacobi for n <= 32 * 48 (jacobi_coop_npl(n) > 0); cooperative launch
int jacobi_coop_npl(int n);
int jacobi_coop_capacity(int max_n, int max_m);  // co-resident CTAs
cudaError_t launch_jacobi_coop(const CoopSvdTask* d_tasks, int32_t total_ctas, const int32_t* d_cta_task,
                               int32_t max_n, int32_t max_m, double thresh, cudaStream_t st);
constexpr int SMEM_DENSE_MAX_N = 144;  // n x n doubles resident in shared memory
void launch_complement(const ComplementTask* d_tasks, int32_t ntasks, cudaStream_t st);
void launch_lu(const LuTask* d_tasks, int32_t ntasks, cudaStream_t st);
void launch_trsm(const TrsmTask* d_tasks, int32_t ntasks, cudaStream_t st);
// blocked DMMA TRSM, nc (= trsm_dmma_cols(r), 0: too large) columns per task
int trsm_dmma_cols(int r);
void launch_trsm_dmma(const TrsmTask* d_tasks, int32_t ntasks, int32_t max_r, int32_t nc, cudaStream_t st);
// status = vanishing-pivot test from red = {max|D_RR|, min|diag U|}
void launch_lu_status(const double* red, int32_t r, int32_t* status, cudaStream_t st);
void launch_sumsq_reduce(const double* d_parts, const int64_t* d_seg, int32_t nseg,
                         double* d_out, cudaStream_t st);

size_t hh_panel_smem(int chunk);
int hh_panel_capacity(int chunk);  // co-resident CTAs of the panel kernel at this chunk
// ---- block column pivoting of the blocked Householder QR (augmentation):
// before each panel, the trailing columns [j0, ntot) of a job are reordered
// by their remaining norms (rows [j0, L)), descending (ties: lower index
// first).  Columns live at M + c*ldm with L contiguous rows.
struct PivotTask {
    double* M;
    int64_t ldm;
    int32_t L, j0, ntot;
    double* norms;       // ntot scratch
    int32_t* order;      // ntot scratch: new position -> old column (local, from j0)
    int32_t* perm;       // ntot: current column -> original column (updated)
    int32_t* perm_tmp;   // ntot scratch
    double* tmp;         // ntot * ldm: receives the reordered matrix (buffers swap)
};
// max_cols: the largest ntot of the launch (all columns are visited)
void launch_pivot_panel(const PivotTask* d_tasks, int32_t ntasks, int32_t max_cols, int32_t max_l,
                        cudaStream_t st);
void launch_iota(int32_t* p, int32_t n, cudaStream_t st);
// U[j][perm[i]] = W[j][i] for the first m rows of the n x n U (in place
// through scratch): un-permutes the Jacobi's vectors of a pivoted R
struct UnpermTask {
    double* U;
    double* tmp;         // m * n scratch
    const int32_t* perm;
    int32_t m, n;
};
void launch_unpermute_rows(const UnpermTask* d_tasks, int32_t ntasks, int32_t max_mn, cudaStream_t st);
// panels of ntasks tasks, each one thread-block cluster of `cluster` CTAs
// (2..16) holding `chunk` rows each (<= HH_CLUSTER_CHUNK); task.cta0/ncta,
// part, gram and bar are unused
constexpr int HH_CLUSTER_CHUNK = 800;
cudaError_t launch_hh_panel_cluster(const HhPanelTask* d_tasks, int32_t ntasks, int32_t cluster, int32_t chunk,
                                    cudaStream_t st);
cudaError_t launch_hh_panel(const HhPanelTask* d_tasks, const int32_t* d_cta_task, int32_t total_ctas,
                            int32_t max_chunk, cudaStream_t st);
void launch_hh_tmul(const HhTmulTask* d_tasks, int32_t ntasks, int32_t max_cols, cudaStream_t st);
void launch_set_eye(const EyeTask* d_tasks, int32_t ntasks, int32_t max_n, cudaStream_t st);

// top (dense) LU pieces
void launch_panel_lu(double* A, int64_t lda, int32_t n, int32_t k0, int32_t nb, int32_t* piv,
                     cudaStream_t st);
void launch_row_swaps(double* A, int64_t lda, int32_t ncols_total, int32_t k0, int32_t nb,
                      const int32_t* piv, int32_t skip_c0, int32_t skip_c1, cudaStream_t st);
void launch_trsm_unit_lower_rows(const double* A, int64_t lda, int32_t k0, int32_t nb,
                                 int32_t c0, int32_t ncols, cudaStream_t st);
// cooperative panel LU of the dense top (k_top.cu); false if the panel does
// not fit (caller falls back to launch_panel_lu)
constexpr int TOP_PANEL_NB = 64;
constexpr size_t TOP_PANEL_SMEM = 200 * 1024;
struct TopPanelScratch {
    double* val;     // 2 * grid
    int* idx;        // 2 * grid
    double* rows;    // 2 * grid * TOP_PANEL_NB
    double* rowk;    // 2 * TOP_PANEL_NB
    unsigned* bar;   // 2
};
int top_panel_grid(int m);
bool launch_coop_panel_lu(double* A, int64_t lda, int32_t n, int32_t k0, int32_t nb, int32_t* piv,
                          TopPanelScratch S, cudaStream_t st);
void launch_absmax(const double* A, int64_t lda, int32_t rows, int32_t cols, double* out,
                   cudaStream_t st);
void launch_diag_absmin(const double* A, int64_t lda, int32_t n, double* out, cudaStream_t st);

// solve
void launch_solve_tasks(const SolveTask* d_tasks, int32_t ntasks, const SolveCluster* d_cl,
                        const SolveEdge* d_edges, double* y, double* scratch, double* work, int32_t nrhs,
                        cudaStream_t st);
void launch_fwd_scatter(const ScatterGroup* d_groups, int32_t ngroups, const int64_t* d_list,
                        const double* scratch, double* y, int32_t nrhs, cudaStream_t st, int32_t ysplit = 1);
void launch_gather_rows(const double* src, const int64_t* idx, int64_t n, int32_t nrhs,
                        double* dst, cudaStream_t st);
void launch_scatter_rows(const double* src, const int64_t* idx, int64_t n, int32_t nrhs,
                         double* dst, cudaStream_t st);
// dense top solve: x <- (LU)^-1 P x through tmp (n x nrhs); sync holds
// 1 + ceil(n/64) ints; perm from launch_top_perm (k_top.cu)
void launch_top_perm(const int32_t* piv, int32_t n, int32_t* perm, cudaStream_t st);
// dst[i, :] = src[perm[i], :] for an n x nrhs row-major block
void launch_permute_rows(const double* src, const int32_t* perm, int32_t n, int32_t nrhs, double* dst,
                         cudaStream_t st);
void launch_top_solve(const double* lu, const int32_t* perm, int32_t n, double* x, int32_t nrhs,
                      double* tmp, int32_t* sync, cudaStream_t st);

// matvec / vectors
// max_rows > 0 (largest output segment of the launch) enables the
// shared-memory accumulating, coalesced nrhs = 1 kernel
void launch_gemv_tasks(const GemvTask* d_tasks, int32_t ntasks, const GemvContrib* d_contribs,
                       int32_t nrhs, cudaStream_t st, int32_t max_rows = 0);
void launch_norm2(const double* x, int64_t n, double* partial, double* out, cudaStream_t st);
void launch_scale_by_inv(double* x, const double* w, int64_t n, const double* s,
                         cudaStream_t st);
void launch_axpby(double* y, const double* a, double alpha, const double* b, double beta,
                  int64_t n, cudaStream_t st);

// ---- device H2 construction (k_build.cu) -----------------------------------------
enum KernelFamily : int32_t { KF_EXP_COV = 0, KF_LAPLACE2D = 1, KF_HELMHOLTZ3D = 2 };

struct KernelParams {     // kernels.py:44-86 families; diag_base = the entry at r = 0
    int32_t family, dim;
    double corr_length, kappa, diag_base, alpha_r;
};

struct EvalTask {         // out(i, j) = K(|X_i - Y_j|), row-major ldo
    const double* X;     // rows x dim
    const double* Y;     // cols x dim
    double* out;
    int64_t ldo;
    int64_t row0, col0;  // global point indices (diag: same index -> diag_base + alpha_r)
    int32_t rows, cols;
    int32_t diag, pad_;
};

struct GridTask {         // p^dim Chebyshev points of the box [lo, hi]
    double lo[3], hi[3];
    double* out;          // p^dim x dim
    int32_t p, pad_;
};

struct InterpTask {       // Lagrange interpolation of npts points in the box's p-grid
    const double* pts;    // npts x dim
    double lo[3], hi[3];
    double* out;          // npts x p^dim, row-major ldo
    int64_t ldo;
    int32_t p, pad_;
};

struct RowNormOut {       // out[j] = |P[j, 0:len]|
    const double* P;
    double* out;
    int64_t ldp;
    int32_t len, pad_;
};

struct DiagTask {         // D = diag(w), n x n
    const double* w;
    double* D;
    int32_t n, pad_;
};

void launch_eval_tasks(const EvalTask* d_tasks, const int64_t* d_tile_start, int32_t ntasks, int64_t ntiles,
                       const KernelParams& kp, cudaStream_t st);
void launch_grid_tasks(const GridTask* d_tasks, int32_t ntasks, int32_t dim, cudaStream_t st);
void launch_interp_tasks(const InterpTask* d_tasks, const int64_t* d_pt_start, int32_t ntasks, int64_t npts,
                         int32_t dim, cudaStream_t st);
void launch_row_norms(const RowNormOut* d_tasks, const int64_t* d_row_start, int32_t ntasks, int64_t nrows,
                      cudaStream_t st);
void launch_set_diag(const DiagTask* d_tasks, int32_t ntasks, cudaStream_t st);

double bench_dmma(int64_t iters, cudaStream_t st);
int64_t kernel_launch_count();
void count_launch();
void add_launches(int64_t n);  // kernels replayed inside a CUDA graph

}  // namespace h2f
