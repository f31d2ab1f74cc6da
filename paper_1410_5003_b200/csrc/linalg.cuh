// Batched complex FP64 dense linear algebra for sm_100a.
//   zgemm_batched : DMMA (mma.sync m8n8k4 f64) complex GEMM, 4 real MMAs per
//                   complex product, optional K-concatenation of two products
//   COD least squares (periodize.hpp:25-39): Eigen-semantics column-pivoted QR,
//                   rank at a threshold, RZ reduction, min-norm operator
//   LU with partial pivoting + triangular solves for block cyclic reduction
#pragma once

#include <atomic>

#include "hankel.cuh"
#include "qps_internal.h"

namespace qpsb {

// C = beta C + alpha * sum_s A_s B_s, A_s: M x K_s (lda), B_s: K_s x N (ldb).
struct GemmTask {
    const cplx* A[2];
    const cplx* B[2];
    int lda[2], ldb[2], K[2];
    int nseg;
    cplx* C;
    int ldc;
    int mlim;  // rows of C written: 0 = all M, > 0 = the first mlim, < 0 = none (device-built tasks)
};

struct Workspace;  // forward
extern std::atomic<uint64_t> g_zgemm_launches;

// family: profiling name (string literal); default by shape
void zgemm_batched(int M, int N, cplx alpha, cplx beta, const std::vector<GemmTask>& tasks, cudaStream_t s,
                   DBuf<GemmTask>& d_tasks, const char* family = nullptr);
// norms[t] = || alpha A_t B_t + beta C_t ||_F per task, C only read (the
// product is reduced in the GEMM epilogue, never stored); parts: scratch
void zgemm_residual_norms(int M, int N, cplx alpha, cplx beta, const std::vector<GemmTask>& tasks, cudaStream_t s,
                          DBuf<GemmTask>& d_tasks, DBuf<double>& parts, double* norms);

// ---- COD least squares -----------------------------------------------------
// Per problem b: Q_b (m x p, ld m).  Factor state lives in caller-provided
// device arrays sized for `count` problems.
struct CodBatch {
    int count = 0, m = 0, p = 0;
    const cplx* Q = nullptr;  // count x (m*p), column-major, ld m
    cplx* W = nullptr;        // factored CPQR (count x m*p)
    cplx* V = nullptr;        // RZ work copy (count x m*p)
    cplx* tau = nullptr;      // count x p
    cplx* zc = nullptr;       // count x p
    int* perm = nullptr;      // count x p
    int* nzp = nullptr;       // nonzero pivots per problem
    double* maxpiv = nullptr; // per problem
    int* rank = nullptr;      // per problem (current threshold)
    cplx* QH = nullptr;       // count x (p*m): Q_1^* (rows >= rank zero), ld p
    cplx* Wz = nullptr;       // count x (p*p): P Z^* [I_r; 0] (cols >= rank zero), ld p
    cplx* M1 = nullptr;       // count x (m*p) scratch
    cplx* Y = nullptr;        // count x (p*m) scratch
    GemmTask* trsm_tasks = nullptr;  // count x ceil(p/16) device-built tasks of the blocked cod_trsm
};
// rows 0..rank_b-1 of B_b (p x ncols, ld ldb, stride) <- T11_b^{-1} B_b, T11 in
// the RZ-reduced factor V_b (ld m): the backward-stable triangular step of the
// COD solve (never an explicit inverse)
void cod_trsm(const CodBatch& b, cplx* B, int ldb, size_t stride, int ncols, const int* d_flags, cudaStream_t s);
void cod_factor(const CodBatch& b, cudaStream_t s);
// same factorization with reciprocal-multiplies for the divisions (compression only)
void cod_factor_fast(const CodBatch& b, cudaStream_t s);
// rank at threshold th for problems whose flag is set (flags == nullptr: all)
void cod_rank(const CodBatch& b, double th, const int* d_flags, cudaStream_t s);
// forms QH and Wz for the current rank: X = Wz * T11^{-1} * (QH * RHS)
void cod_operator(const CodBatch& b, const int* d_flags, cudaStream_t s);

// ---- LU with partial pivoting (batched over pointer lists) ----------------
// n x n matrices A_b (ld) factored in place; ipiv_b[n] holds the row swapped
// with row k at step k (0-based, LAPACK-style sequential interchanges).
// d_singular[b] is set to 1 when a zero pivot is met.  Dinv_b (lu_dinv_elems(n)
// entries) receives the inverses of the 64x64 diagonal tiles of L and U so the
// triangular solves run as DMMA GEMMs.
size_t lu_dinv_elems(int n);
void lu_factor_batched(int n, int ld, const std::vector<cplx*>& A, const std::vector<int*>& ipiv,
                       const std::vector<cplx*>& Dinv, int* d_singular, cudaStream_t s, Workspace& ws);
// B_b <- A_b^{-1} B_b for n x nrhs right-hand sides (ldb) using those factors.
// factor + solve A X = B in one pass (A's factors are not reusable afterwards)
void lu_factor_solve_batched(int n, int ld, const std::vector<cplx*>& A, const std::vector<int*>& ipiv,
                             const std::vector<cplx*>& dinv, const std::vector<cplx*>& B, int ldb, int nrhs,
                             int* d_singular, cudaStream_t s, Workspace& ws);
void lu_solve_batched(int n, int ld, const std::vector<cplx*>& A, const std::vector<int*>& ipiv,
                      const std::vector<cplx*>& Dinv, const std::vector<cplx*>& B, int ldb, int nrhs,
                      cudaStream_t s, Workspace& ws);

// Reciprocal condition estimate of LU factors, the reference's
// PartialPivLU::rcond() test (tridiag.hpp:36-40): per block b (d_ptrs[b], or
// base + b * stride when d_ptrs is null) rcond(U_b) = 1 / (||U_b||_1
// est ||U_b^{-1}||_1) with LAPACK zlacn2's Hager/Higham estimator on the U
// factor left in the upper triangle, solving with the LU's inverse diagonal
// tiles (d_dinv[b] or dbase + b * dstride, lu_dinv_elems layout, U half
// filled); d_flag[b] = 1 when !(rcond > th); d_rcond / d_est (may be null)
// receive the estimates of rcond(U) and of ||U^{-1}||_1.
void lu_rcond_batched(int n, int ld, cplx* const* d_ptrs, const cplx* base, size_t stride, cplx* const* d_dinv,
                      const cplx* dbase, size_t dstride, int count, double th, int* d_flag, double* d_rcond,
                      cudaStream_t s, double* d_est = nullptr);
// ||A_b||_1 of count n x n blocks (base + b stride), as double bits (see rcond_screen)
void batched_norm1(const cplx* A, int n, int ld, size_t stride, int count, unsigned long long* d_out,
                   cudaStream_t s);
// rc_up_b = 1 / (||A_b||_1 max_k ||W_b[:, col0 + k]||_1 / rnorm1) for the nprobe
// solved probe columns of W_b (n x ..., ld n, base + b wstride): d_flag[b] = 1
// when rc_up <= th_def (certain), d_sus[b] = rc_up <= th_sus, d_est_lo[b] the
// lower bound of ||A_b^{-1}||_1
void rcond_screen(const cplx* W, size_t wstride, int n, int col0, int nprobe, const unsigned long long* d_anorm,
                  double rnorm1, int count, double th_def, double th_sus, int* d_flag, int* d_sus, double* d_est_lo,
                  cudaStream_t s);
constexpr double kRcondMin = 1e-15;  // tridiag.hpp:36
// dst_q[:, k] = src_q[:, cols[q * ncols + k]] (rows x ncols per problem q; src_q
// column-major with leading dimension ld[q]); pointer/ld tables staged in pbuf/lbuf
void gather_columns(const std::vector<const cplx*>& src, const std::vector<int>& ld, int rows, const int* d_cols,
                    int ncols, cplx* dst, int ldd, size_t dstride, DBuf<const cplx*>& pbuf, DBuf<int>& lbuf,
                    cudaStream_t s);

// ---- small utilities -------------------------------------------------------
// per problem max |X_ij| over an m x n block (ld), count problems with stride
void batched_maxabs(const cplx* X, int m, int n, int ld, size_t stride, int count, double* out, cudaStream_t s);
// per problem Frobenius norm
// y += x (n complex entries)
void axpy_blocks(cplx* y, const cplx* x, size_t n, cudaStream_t s);
void batched_fro(const cplx* X, int m, int n, int ld, size_t stride, int count, double* out, cudaStream_t s,
                 double* maxabs_out = nullptr);
void copy_blocks(const cplx* src, int lds, size_t sstride, cplx* dst, int ldd, size_t dstride, int m, int n,
                 int count, cudaStream_t s);
// y_b = beta y_b + alpha * sum_s A_s x_s  (batched complex GEMV, up to 2 terms)
struct GemvTask {
    const cplx* A[2];
    const cplx* x[2];
    int lda[2], n[2];
    int nseg;
    cplx* y;
};
void zgemv_batched(int M, cplx alpha, cplx beta, const std::vector<GemvTask>& tasks, cudaStream_t s,
                   DBuf<GemvTask>& d_tasks);
// FP64 peak microbenchmarks (same run as the solver): DFMA chain and DMMA loop
double measure_dfma_tflops(cudaStream_t s);
double measure_dmma_tflops(cudaStream_t s);

struct Workspace {
    DBuf<GemmTask> gemm_tasks;
    DBuf<GemvTask> gemv_tasks;
    DBuf<cplx*> ptrs, ptrs2, ptrs3;
    DBuf<int*> iptrs;
    DBuf<int> rl_map;  // right-looking LU: per matrix, the interchange map of the current panel
    DBuf<int> perm;    // gathered row permutations (row_permute_kernel)
    std::vector<GemmTask> h_gemm;
};

// Products on the right-hand sides of a block solve: m = 1 (one solve per
// system) runs them as batched GEMVs, m > 1 (several right-hand sides, e.g.
// the alpha-grouped sweep) as batched GEMMs with N = m.
struct RhsOps {
    int m;
    cudaStream_t s;
    Workspace& ws;
    inline void run(int M, cplx alpha, cplx beta, const std::vector<GemmTask>& t) {
        if (t.empty()) return;
        if (m > 1) {
            zgemm_batched(M, m, alpha, beta, t, s, ws.gemm_tasks, "wb_rhs");
            return;
        }
        std::vector<GemvTask> v(t.size());
        for (size_t q = 0; q < t.size(); ++q) {
            GemvTask g{};
            g.nseg = t[q].nseg;
            for (int k = 0; k < g.nseg; ++k) {
                g.A[k] = t[q].A[k];
                g.lda[k] = t[q].lda[k];
                g.x[k] = t[q].B[k];
                g.n[k] = t[q].K[k];
            }
            g.y = t[q].C;
            v[q] = g;
        }
        zgemv_batched(M, alpha, beta, v, s, ws.gemv_tasks);
    }
};

}  // namespace qpsb
