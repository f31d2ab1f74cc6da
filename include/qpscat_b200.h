/*
 * qpscat_b200.h — C-ABI drop-in boundary for the quasi-periodic multilayer
 * scattering hot path (Cho & Barnett, arXiv 1410.5003; reference library
 * `qpscat`, /root/reference/proj/include/qpscat).
 *
 * Plain pointers and sizes only; complex numbers are `qps_cplx` with the
 * memory layout of std::complex<double> (and CUDA double2).  All matrices
 * crossing the boundary are column-major, exactly like the reference's
 * Eigen::MatrixXcd (types.hpp:11).
 *
 * Two libraries implement this header:
 *   paper_1410_5003_b200/libqpscat_b200.so — the product: host C++ + sm_100a
 *       CUDA kernels (fill, Schur complements, block cyclic reduction, sweep);
 *   oracle/_ref/libqpscat_ref.so — test infrastructure only: the reference
 *       headers compiled unmodified on the CPU (oracle/ref_capi.cpp).
 *
 * Each entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/proj/include/qpscat/).  Error behaviour mirrors
 * the reference's exception taxonomy (errors.hpp:9-40): every call returns a
 * qps_status; qps_last_error() returns the message, the 1-based layer of a
 * SolverError and the byte count of a MemoryBudgetError.
 *
 * Threading: one context = one CUDA stream; a context is not thread-safe.
 * Calls are synchronous at the API level.
 */
#ifndef QPSCAT_B200_H
#define QPSCAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QPS_ABI_VERSION 4

typedef struct qps_ctx qps_ctx;
typedef struct {
    double re, im;
} qps_cplx;

/* errors.hpp:9-40, specfun.hpp:53-54 */
typedef enum {
    QPS_OK = 0,
    QPS_ERR_CONFIG = 1,        /* ConfigError          errors.hpp:9   */
    QPS_ERR_GEOMETRY = 2,      /* GeometryError        errors.hpp:14  */
    QPS_ERR_USAGE = 3,         /* UsageError           errors.hpp:19  */
    QPS_ERR_SINGULARITY = 4,   /* SingularityError     errors.hpp:24  */
    QPS_ERR_SOLVER = 5,        /* SolverError{layer}   errors.hpp:29  */
    QPS_ERR_MEMORY_BUDGET = 6, /* MemoryBudgetError    errors.hpp:36  */
    QPS_ERR_DOMAIN = 7,        /* std::domain_error    specfun.hpp:54 */
    QPS_ERR_CUDA = 8,          /* device failure (product only)        */
    QPS_ERR_INTERNAL = 9
} qps_status;

/* InterfaceSpec::Shape, geometry.hpp:274 */
typedef enum { QPS_SHAPE_SINE = 0, QPS_SHAPE_FOURIER = 1, QPS_SHAPE_POLYLINE = 2 } qps_shape;

/* InterfaceSpec, geometry.hpp:273-282 (offset = nominal height; shape
 * coordinates relative to it; vertices are x0,y0,x1,y1,...). */
typedef struct {
    int shape;
    double offset;
    double amplitude, phase;
    int n_cos;
    const double* cosc;
    int n_sin;
    const double* sinc;
    int n_vertices;
    const double* vertices;
    int n_nodes;
    const int* nodes;
    int grading_q;
} qps_interface_spec;

/* NumericsParams, geometry.hpp:405-414 */
typedef struct {
    int P, Mw, M, K;
    double R;
    int grading_q;
    double clearance;
    uint64_t memory_budget;
} qps_numerics;

/* Matrices that can be downloaded for parity checks.
 * Stage SYSTEM = BlockSystem (assembly.hpp:293-315);
 * stage PERIODIZED = PeriodizedSystem (periodize.hpp:44-56). */
typedef enum {
    QPS_BLK_A_DIAG = 0, QPS_BLK_A_SUPER, QPS_BLK_A_SUB, QPS_BLK_B_SELF, QPS_BLK_B_BELOW,
    QPS_BLK_C_SELF, QPS_BLK_C_ABOVE, QPS_BLK_Q, QPS_BLK_Z_U, QPS_BLK_Z_D, QPS_BLK_V_U, QPS_BLK_V_D,
    QPS_BLK_W_U, QPS_BLK_W_D, QPS_BLK_F, QPS_BLK_BP_FIRST, QPS_BLK_BP_LAST, QPS_BLK_CP_FIRST,
    QPS_BLK_CP_LAST, QPS_BLK_QP_FIRST, QPS_BLK_QP_LAST,
    /* PeriodizedSystem */
    QPS_BLK_AP_DIAG = 32, QPS_BLK_AP_SUPER, QPS_BLK_AP_SUB, QPS_BLK_X_FIRST, QPS_BLK_X_ABOVE,
    QPS_BLK_X_SELF, QPS_BLK_X_LAST
} qps_block_kind;

/* Per-phase timings, milliseconds of the last call of each phase
 * ("Matrix Filling / Schur / Block Solve"). */
typedef struct {
    double fill_ms, assemble_ms, schur_ms, solve_ms, recover_ms;
    double total_ms; /* device timeline of the last qps_solve, first to last event */
    /* inside solve_ms: the batched LU of every diagonal block with its
     * right-hand-side solves (level 0 of the Woodbury cyclic reduction); 0 when
     * the dense reduction ran or for the CPU oracle */
    double factor_ms;
} qps_phase_times;

/* How the last block solve ran (product diagnostics; the oracle reports
 * bcr_path = -1, the reference's sequential block Thomas):
 *   bcr_path        0 dense block cyclic reduction, 1 low-rank couplings in
 *                   Woodbury form (default), 2 low-rank with per-level LU
 *   lr_rank_max     largest numerical rank of a compressed coupling's sample
 *   lr_probe_worst  a-posteriori test of the compression: max over couplings
 *                   of ||(I - P P^*) C w2||_F / ||C w2||_F on an independent
 *                   probe block w2 (above 1e-12 -> dense reduction)
 *   refine_steps    iterative-refinement steps applied to the block solve
 *   refine_res0/1   ||f - A' eta||_2 / ||f||_2 before the first step and (when
 *                   QPS_REFINE_CHECK=1) after the last one; 0 when none ran
 *   lr_width        columns of the compressed coupling bases: the widest
 *                   accepted rank rounded up to 8 (48 at most; 0 when dense)
 *   lr_width_retry  1 when the truncated bases failed the probe and the solve
 *                   ran again at the full width */
typedef struct {
    int bcr_path;
    int lr_rank_max;
    double lr_probe_worst;
    int refine_steps;
    double refine_res0, refine_res1;
    int lr_width;
    int lr_width_retry;
} qps_solver_diag;

/* ---------------------------------------------------------------- context */
int qps_abi_version(void);
const char* qps_backend_name(void); /* "b200-cuda" or "reference-cpu" */
qps_ctx* qps_create(int device);
void qps_destroy(qps_ctx* ctx);
int qps_last_error(const qps_ctx* ctx, char* msg, size_t cap, int* solver_layer, uint64_t* required_bytes);
/* parallel.hpp:12-31 (CPU oracle thread count; ignored by the GPU library) */
int qps_set_num_threads(qps_ctx* ctx, int n);
/* periodize.hpp:15-18 qsolve_threshold() */
int qps_set_qsolve_threshold(qps_ctx* ctx, double th);
/* Product extension (no reference counterpart): steps of iterative refinement
 * of the block cyclic reduction (residual with the unfactored A', correction
 * through the kept factors).  -1 = default: 0 for qps_solve, 1 for the sweeps.
 * The oracle accepts and ignores it (its block Thomas needs none). */
int qps_set_refine(qps_ctx* ctx, int steps);

/* ----------------------------------------------------- geometry & problem */
/* LayerStack + build_geometry(stack, num), geometry.hpp:289-296,480-496 */
int qps_build_geometry(qps_ctx* ctx, double d, int n_layers, const double* epsilon, const double* mu,
                       int n_interfaces, const qps_interface_spec* ifaces, const qps_numerics* num);
/* make_problem(stack, geom, omega, theta, K), assembly.hpp:69-82 */
int qps_make_problem(qps_ctx* ctx, double omega, double theta, int K);
/* scalars of ScatteringProblem / StackGeometry (assembly.hpp:15-39, geometry.hpp:259-264):
 * n_nodes[I], k[I+1]; any pointer may be NULL */
int qps_problem_info(const qps_ctx* ctx, int* I, int* K, int* n_nodes, double* k, qps_cplx* alpha,
                     double* y_U, double* y_D);
/* nodes/normals (x,y interleaved, N each), weights, speeds of interface j
 * (InterfaceQuadrature, geometry.hpp:80-92) */
int qps_interface_nodes(const qps_ctx* ctx, int j, double* nodes_xy, double* normals_xy, double* weights,
                        double* speeds);

/* ------------------------------------------- step-wise hot path (cache) */
/* precompute_shift_blocks(p, num), assembly.hpp:212-287 (alpha-free cache) */
int qps_precompute_shift_blocks(qps_ctx* ctx);
/* assemble_system(p, cache, num), assembly.hpp:462-483 */
int qps_assemble_system(qps_ctx* ctx);
/* schur_complement(sys), periodize.hpp:124-126 */
int qps_schur_complement(qps_ctx* ctx);
/* block_lu_solve(ps), tridiag.hpp:23-46 (the product uses block cyclic
 * reduction; SolverError names the original 1-based layer of a singular
 * diagonal factor) */
int qps_block_lu_solve(qps_ctx* ctx);
/* block_lu_solve(ps) on a caller-built PeriodizedSystem (tridiag.hpp:23-46, as
 * the reference's own tests build one, proj/tests/test_tridiag.cpp:27-44):
 * I diagonal blocks n x n (Ad, I*n*n), I-1 super/sub blocks (Au, Al), RHS f
 * for block 0 (n); eta receives I*n.  SolverError names a singular layer. */
int qps_block_lu_solve_blocks(qps_ctx* ctx, int I, int n, const qps_cplx* Ad, const qps_cplx* Au,
                              const qps_cplx* Al, const qps_cplx* f, qps_cplx* eta);
/* recover_aux(ps, eta, sol), tridiag.hpp:50-66 */
int qps_recover_aux(qps_ctx* ctx);

/* ------------------------------------------------- one-shot hot path */
/* precompute_shift_blocks + assemble_system + solve_periodized
 * (assembly.hpp:212,462; tridiag.hpp:69-74).  The product fuses the alpha
 * recombination into the fill and never materialises the alpha-free cache. */
int qps_solve(qps_ctx* ctx);

/* Solution, tridiag.hpp:11-17: eta[sum 2N_j] (per interface tau then sigma),
 * c[(I+1)*P], aU[2K+1], aD[2K+1], lsq_residual[I+1]; NULL pointers skipped */
int qps_get_solution(const qps_ctx* ctx, qps_cplx* eta, qps_cplx* c, qps_cplx* aU, qps_cplx* aD,
                     double* lsq_residual, double* max_lsq_residual);
/* flux_error + reflection_transmission, postprocess.hpp:134-180.
 * Per-order arrays (2K+1 each, may be NULL): kappa, k^U_n, k^D_n, propagating flags. */
int qps_reflection_transmission(const qps_ctx* ctx, double* R, double* T, double* flux_error, double* kappa,
                                qps_cplx* kU, qps_cplx* kD, int* prop_up, int* prop_down);

/* Replace the current Solution (tridiag.hpp:11-17) by caller data -- the
 * reference's post-processing takes a Solution argument (evaluate_field,
 * residual_suite): eta[sum 2N_j], c[(I+1)*P], aU[2K+1], aD[2K+1].  Needs a
 * problem (make_problem) on this context. */
int qps_set_solution(qps_ctx* ctx, const qps_cplx* eta, const qps_cplx* c, const qps_cplx* aU, const qps_cplx* aD);

/* ---------------------------------------------------------- residual suite */
/* residual_suite(sol, p, num, interfaces), postprocess.hpp:369-399, of the
 * current solution: ResidualReport{wall_qp, radiation, interface}
 * (postprocess.hpp:186-190).  The product sums every potential on the device. */
int qps_residual_suite(qps_ctx* ctx, int n_interfaces, const int* interfaces, double* wall_qp, double* radiation,
                       double* interface_res);
/* interface_matching_residual(sol, p, num, j, n_probe), postprocess.hpp:263-365 */
int qps_interface_matching_residual(qps_ctx* ctx, int j, int n_probe, double* out);

/* ------------------------------------------------------ field evaluation */
/* evaluate_field(sol, p, points), postprocess.hpp:78-123, for the last solve:
 * xy[2n] interleaved points (any cell: x is mapped into the central cell and
 * the result phased by alpha^m).  Outputs (NULL skipped): scattered and total
 * field [n], region [n] (0 above y_U, 1 inside a layer, 2 below y_D) and the
 * 0-based layer [n].  GeometryError when a point lies on an interface
 * (classify_point, postprocess.hpp:27-39).  Plain Nystrom sums as the
 * reference (no close-evaluation correction). */
int qps_evaluate_field(qps_ctx* ctx, int n_points, const double* xy, qps_cplx* u_scattered, qps_cplx* u_total,
                       int* region, int* layer);

/* --------------------------------------------------------- angle sweep */
/* Multi-angle sweep (building blocks assembly.hpp:85-155,
 * periodize.hpp:58-126): the alpha-free cache is filled once and every angle
 * is assembled, periodized and solved from it (mode 0, "accelerated"), or the
 * cache is refilled per angle (mode 1, "independent").  K is fixed for all
 * angles.  Outputs per angle: R, T, flux_error [n]; aU, aD [n*(2K+1)];
 * status [n] (qps_status of that angle; a singular angle does not abort). */
int qps_sweep(qps_ctx* ctx, int n_angles, const double* theta, int K, int mode, double* R, double* T,
              double* flux_error, qps_cplx* aU, qps_cplx* aD, int* status);
/* plan_sweep(omega, n, theta_range), SPEC.md:505-512 (sweep module; the
 * reference has no code for it, proj/tests/test_sweep.cpp:1): angles on a grid
 * uniform in kappa_0 = k_1 cos(theta) with spacing 2 pi / (n d) inside
 * (theta_lo, theta_hi) (-pi < lo < hi < 0), so that alpha = exp(i d k_1 cos
 * theta) takes exactly n values.  k_1 and d from the last
 * make_problem.  Up to cap angles and their alpha-group index (j mod n) are
 * written; *n_angles receives the grid size. */
int qps_plan_sweep(qps_ctx* ctx, int n_alpha, double theta_lo, double theta_hi, int cap, double* theta,
                   int* alpha_group, int* n_angles);
/* The last qps_sweep: alpha group of every angle (SpectrumRow::alpha_group,
 * postprocess.hpp:155-161; -1 for an angle whose make_problem failed), number
 * of groups, interior eliminations (InteriorSchur, periodize.hpp:61-94) and
 * block factorizations performed.  Mode 0 computes both once per alpha group
 * of two or more angles (the product factors A(alpha) once and applies each
 * angle's corner terms as a rank-2P Woodbury correction; the reference
 * composition re-runs block_lu_solve per angle). */
int qps_sweep_info(const qps_ctx* ctx, int cap, int* alpha_group, int* n_groups, uint64_t* n_interior,
                   uint64_t* n_factorizations);

/* ------------------------------------------------- parity / diagnostics */
/* Copy block `kind` with index `i` (interface, layer or 0) into out
 * (column-major, rows x cols).  With out == NULL only the shape is returned. */
int qps_download_block(const qps_ctx* ctx, int kind, int i, qps_cplx* out, int* rows, int* cols);
/* ShiftBlockCache::fill_evals (assembly.hpp:285): `reference` = the reference
 * fill's Hankel-pair count for this geometry, `performed` = pairs evaluated by
 * this implementation in its last fill. */
int qps_fill_evals(const qps_ctx* ctx, uint64_t* reference, uint64_t* performed);
int qps_get_phase_times(const qps_ctx* ctx, qps_phase_times* t);
int qps_solver_diagnostics(const qps_ctx* ctx, qps_solver_diag* d);
/* hankel01 batch (specfun.hpp:69-73): h0[n], h1[n] for host x[n] */
int qps_hankel01(qps_ctx* ctx, int n, const double* x, qps_cplx* h0, qps_cplx* h1);
/* qsolve(Q, RHS), periodize.hpp:25-39: min-norm least squares through the
 * rank-revealing complete orthogonal decomposition with threshold escalation
 * (Q m x p, RHS m x n, X p x n; column-major).  *rank receives the rank used. */
int qps_qsolve(qps_ctx* ctx, int m, int p, int n, const qps_cplx* Q, const qps_cplx* RHS, qps_cplx* X, int* rank);
/* Diagnostics: C = A B (M x K times K x N, column-major) on the product's
 * batched DMMA GEMM (the oracle uses its BLAS). */
int qps_debug_zgemm(qps_ctx* ctx, int M, int N, int K, const qps_cplx* A, const qps_cplx* B, qps_cplx* C);
/* Kernel-family instrumentation: when enabled, every launch is bracketed by
 * CUDA events on its own stream and tagged with its algorithmic FLOPs, bytes
 * and kernel evaluations.  qps_prof_stats returns the number of families and
 * fills up to cap entries (names: cap x 64 chars).  The oracle reports 0. */
int qps_prof_enable(qps_ctx* ctx, int on);
int qps_prof_reset(qps_ctx* ctx);
int qps_prof_stats(qps_ctx* ctx, int cap, char* names, uint64_t* launches, double* ms, double* flops,
                   double* bytes, double* units);
/* number of kernels this library has launched (process lifetime) */
uint64_t qps_launch_count(void);
/* host<->device bytes moved since the last qps_prof_reset */
int qps_transfer_bytes(const qps_ctx* ctx, uint64_t* h2d, uint64_t* d2h);
/* FP64 peaks of this device measured by microbenchmarks (DFMA chain, DMMA
 * loop), TFLOP/s; the oracle returns 0 for both. */
int qps_measure_fp64_peaks(qps_ctx* ctx, double* dfma_tflops, double* dmma_tflops);

#ifdef __cplusplus
}
#endif

#endif /* QPSCAT_B200_H */
