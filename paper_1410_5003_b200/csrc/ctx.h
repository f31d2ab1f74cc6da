// Solver context: everything one qps_ctx owns on host and device.
#pragma once
#include <chrono>
#include <exception>

#include <array>
#include <string>
#include <vector>

#include "fill.cuh"
#include "linalg.cuh"

namespace qpsb {

struct Dims {
    int I = 0, nb = 0, P = 0, Mw = 0, M = 0, K = 0, nrb = 0;
    int mI = 0, mC = 0, pC = 0;  // interior Q rows, corner Q' rows / cols
    std::vector<int> N;
    bool padded = false;
    int nsys = 1;  // independent systems (incidence angles) held at once
    // per-system strides (complex elements); B blocks are alpha-free and shared
    size_t nb2() const { return size_t(nb) * nb; }
    size_t sA() const { return size_t(I) * nb2(); }
    size_t sU() const { return size_t(I > 1 ? I - 1 : 1) * nb2(); }
    size_t sQi() const { return size_t(I > 1 ? I - 1 : 1) * mI * P; }
    size_t sRi() const { return size_t(I > 1 ? I - 1 : 1) * mI * 2 * nb; }
    size_t sQc() const { return size_t(2) * mC * pC; }
    size_t sRc() const { return size_t(2) * mC * nb; }
    size_t sXi() const { return size_t(I > 1 ? I - 1 : 1) * P * 2 * nb; }
    size_t sXc() const { return size_t(2) * pC * nb; }
};

// COD least-squares state for one family of equal-shape problems
struct CodSet {
    int count = 0, m = 0, p = 0, ncols = 0;
    DBuf<cplx> W, V, tau, zc, M1, Y, QH, Wz, Tb;
    DBuf<int> perm, nzp, rank, flags;
    DBuf<double> maxpiv, xmax, rmax, enorm, rnorm, parts;
    DBuf<GemmTask> tasks1, tasks2;  // task tables of this family's GEMMs (families run on separate streams)
    DBuf<GemmTask> trsm_tasks;      // the blocked back substitution's device-built tasks
    HBuf<double> h_rmax, h_xmax, h_enorm, h_rnorm;  // pinned: read back without blocking the host
    cudaEvent_t ev = nullptr;                        // last read-back of this family
    ~CodSet() {
        if (ev) cudaEventDestroy(ev);
    }
    CodBatch batch(const cplx* Q) {
        CodBatch b;
        b.count = count; b.m = m; b.p = p; b.Q = Q;
        b.W = W.p; b.V = V.p; b.tau = tau.p; b.zc = zc.p; b.perm = perm.p; b.nzp = nzp.p;
        b.maxpiv = maxpiv.p; b.rank = rank.p; b.QH = QH.p; b.Wz = Wz.p; b.M1 = M1.p; b.Y = Y.p;
        b.trsm_tasks = trsm_tasks.p;
        return b;
    }
    void ensure(int cnt, int m_, int p_, int ncols_) {
        count = cnt; m = m_; p = p_; ncols = ncols_;
        const size_t mp = size_t(m) * p;
        W.ensure(cnt * mp); V.ensure(cnt * mp); M1.ensure(cnt * mp); Y.ensure(cnt * mp); QH.ensure(cnt * mp);
        Wz.ensure(size_t(cnt) * p * p); Tb.ensure(size_t(cnt) * p * ncols);
        tau.ensure(size_t(cnt) * p); zc.ensure(size_t(cnt) * p); perm.ensure(size_t(cnt) * p);
        nzp.ensure(cnt); rank.ensure(cnt); flags.ensure(cnt);
        trsm_tasks.ensure(size_t(cnt) * ((p + 15) / 16));
        maxpiv.ensure(cnt); xmax.ensure(cnt); rmax.ensure(cnt); enorm.ensure(cnt); rnorm.ensure(cnt);
        h_rmax.ensure(cnt); h_xmax.ensure(cnt); h_enorm.ensure(cnt); h_rnorm.ensure(cnt);
        if (!ev) QPS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
};

// Offsets (complex elements) of the alpha-free pieces inside Ctx::cache_pool:
// ShiftBlockCache (assembly.hpp:115-155).  Four-plane pieces hold the kinds
// D, S, T, D* as consecutive rows x cols planes.
struct CacheLayout {
    std::vector<std::array<size_t, 2>> self_c, band, nbr_m, nbr_p;  // [j][up k_j / down k_{j+1}]
    std::vector<std::array<size_t, 3>> cup, cdn;                     // [j][l + 1]
    std::vector<size_t> Csp, Csm, Cap, Cam, Qp, Qm;                  // [i], walls
    size_t ZU[3] = {0, 0, 0}, ZD[3] = {0, 0, 0}, VU = 0, VD = 0;
    size_t total = 0;
};

// out_a = sum_t coef(a, t) * piece_t over the planes of one cache piece group
struct CombineTask {
    int nplanes;  // 4 ([D S; T D*] stacking) or 1 (proxy block)
    int rows, cols;
    int npiece;
    int ident;
    size_t piece[6];
    int coef[6];
    cplx* out;
    size_t ostride;
    int ld, row_off, col_off;
};

// alpha^{+-1}-weighted out-of-period band of one smooth self block
struct BandTask {
    int N;
    size_t up, dn;
    cplx* out;
    size_t ostride;
    int ld;
};

// evaluate_field: one layer's sources and its range of the sorted point list
constexpr int kFieldTile = 32;  // points per CTA of the field kernel
struct FieldTask {
    double k;
    int nsrc;               // interfaces bounding the layer (0..2)
    int s_off[2], ns[2];    // pool offsets / node counts
    const cplx* tau[2];     // densities [tau; sigma] of those interfaces
    int p_off, P;           // layer proxies
    const cplx* c;          // proxy coefficients c_layer
    int pt0, npt;           // this layer's range of the sorted point list
};

// One block-tridiagonal system stored as pointer lists (block cyclic reduction)
struct BcrLevel {
    std::vector<int> idx;                 // original block index per active position
    std::vector<cplx*> D, L, U, F;        // per position (L/U may be null at the ends)
};
using BcrLevels = std::vector<BcrLevel>;  // one per system

// one position of the Woodbury block cyclic reduction (bcr_lr.cu): kept per
// level after a solve so that further right-hand sides (iterative refinement)
// replay the reduction without refactoring
struct WbPos {
    int idx;
    int j;  // a * I + idx: slot of the per-block buffers
    cplx* F;
    const cplx *PL, *RL, *PU, *RU;
    const cplx* Z;  // D^{-1} [P_L P_U] once eliminated (n x 2r, ld n)
    bool updated;   // S, g nonzero
};

struct Ctx {
    int device = 0;
    bool host_only = false;  // device == -1: geometry/problem logic only, every device call fails
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // second stream: work independent of the main stream (corner least squares)
    cudaStream_t side2 = nullptr; // third stream: the low-rank sample overlapping the Schur least squares
    cudaStream_t side3 = nullptr; // fourth stream (low priority): the early level-0 factorization
    cudaEvent_t ev_fork = nullptr, ev_fill = nullptr, ev_sample = nullptr;
    cudaEvent_t ev_anorm = nullptr;  // level-0 block norms done (side2)

    StackDesc stack;
    Numerics num;
    HostGeometry geo;
    bool have_geom = false;
    Problem prob;
    bool have_prob = false;
    double qsolve_th0 = 1e-14;

    // ---- device geometry pool (SoA) ----
    DBuf<double> px, py, pnx, pny, pw;
    std::vector<int> iface_off, wall_off, proxy_off;
    int U_off = 0, D_off = 0;
    DBuf<SegDesc> segs;
    std::vector<int> seg_first;
    DBuf<double> fourier;
    DBuf<double> aux_pool;         // host-computed Alpert auxiliary nodes of the open-arc interfaces
    std::vector<long long> aux_off;  // per interface offset into aux_pool (-1: smooth, evaluated on the device)
    DBuf<int> d_err;

    // ---- alpha-free shift-block cache (precompute_shift_blocks) ----
    CacheLayout cache;
    DBuf<cplx> cache_pool, coef_buf;
    std::vector<double> cache_k;  // wavenumbers the cache was filled for
    bool cache_valid = false;
    DBuf<CombineTask> d_comb;
    DBuf<int2> d_ctiles;
    DBuf<BandTask> d_band;
    DBuf<int> d_nodes2;
    DBuf<cplx> wtmp;  // staging of the radiation W blocks
    // ---- field evaluation ----
    DBuf<cplx> field_c, field_out;
    DBuf<double> field_qx, field_qy;
    DBuf<FieldTask> field_tasks;
    DBuf<int2> field_tiles;

    // ---- assembled system (BlockSystem, assembly.hpp:293-315) ----
    Dims dims;
    DBuf<cplx> Adiag, Asup, Asub, Bself, Bbelow, Qint, Rint, Qc, Rc, f;
    bool sys_valid = false;
    // ---- periodized system (PeriodizedSystem, periodize.hpp:44-56) ----
    DBuf<cplx> Apdiag, Apsup, Apsub;  // step-wise API keeps A and A' separately
    bool ps_separate = false, ps_valid = false;
    DBuf<cplx> Xint, Xc;
    std::vector<double> lsq;
    CodSet cod_int, cod_c;

    // ---- low-rank couplings (bcr_lr.cu) ----
    DBuf<cplx> lr_omega, lr_Y, lr_P, lr_PH, lr_R, lr_core, lr_T, lr_vec, lr_W, lr_G;
    DBuf<cplx> lr_L1i;                 // row ID: inverse unit-lower L1 = L[I, :] per coupling (r x r)
    DBuf<int> lr_sk_ptr, lr_sk_ent;    // sparse sign sketch (per 8-column slice: packed column/slot/sign)
    DBuf<const cplx*> lr_skp;          // sketch source pointers
    DBuf<int> lr_skl;                  // sketch source leading dimensions
    DBuf<int> lr_piv, lr_rank_d;       // row ID: skeleton rows I (r per coupling); sample ranks
    // adaptive basis width: the ID's first r' <= r columns repacked here, then swapped in
    DBuf<cplx> lr_Pc, lr_L1ic;
    DBuf<int> lr_pivc;
    cudaEvent_t ev_rank = nullptr;     // the ID's ranks are on the host
    DBuf<cplx> lr_V, lr_VH, lr_Tq, lr_THq, lr_W1, lr_W2, lr_R64, lr_Q2, lr_Q2H;  // blocked QR of the samples
    int lr_omega_n = 0, lr_r = 0;
    HBuf<double> geo_h;                // pinned staging of the geometry pool (upload_geometry)
    bool geo_h_ev_pending = false;
    cudaEvent_t ev_geo = nullptr;
    HBuf<int> lr_rank_h;               // sample ranks, read back without a stream sync
    DBuf<cplx> lr_G2, lr_Y2;           // probe: gathered R and X columns; C[:, J]
    DBuf<cplx> lr_Tall, lr_W1a, lr_W2a, lr_Gq;  // compact-WY T of the sample QR, V^* V, products
    DBuf<int> lr_probe_cols, lr_gld;   // probe column indices (nc x 16); gather leading dimensions
    DBuf<const cplx*> lr_gptr;         // gather source pointers
    int lr_probe_n = 0;
    DBuf<double> lr_pn, lr_parts;      // probe residual / probe norms per coupling; reduction scratch
    HBuf<double> lr_pn_h;
    double lr_probe_worst = 0;         // last compression: max ||(I - P P^*) C w2|| / ||C w2||
    int lr_rank_max = 0;               // last compression: largest sample rank
    int bcr_path = 0;                  // last block solve: 0 dense, 1 Woodbury low-rank, 2 low-rank per-level LU
    HBuf<int> bcr_flag_h;              // singular-factor flags of the level-0 batch (checked at the end)
    DBuf<int> rc_flag, rc_sus;         // level-0 rcond screen: certain flags (rcond <= 1e-15), suspects
    DBuf<double> rc_estlo;             // level-0 lower bounds of ||D_j^{-1}||_1 from the probes
    DBuf<unsigned long long> rc_anorm; // ||D_j^0||_1 (double bits)
    DBuf<cplx> rc_probe;               // the probe columns (nb x 4)
    int rc_probe_n = 0;
    bool anorm_pending = false;        // rc_anorm being computed on side2 (ev_anorm)
    // Woodbury level 0 factored on the side stream while the couplings are
    // compressed on the main stream (wb_factor_async); force_dense: the retry
    // after a compression that failed once that factorization had started
    bool factor_pending = false, force_dense = false;
    bool allow_early = false;          // set by callers that handle the kRetryDense re-run
    // lr_full_width: the kRetryWidth re-run (no adaptive basis width);
    // lr_width_retry: lr_compress failed its probe with a truncated width
    bool lr_full_width = false, lr_width_retry = false;
    bool lr_width_retried = false;     // diagnostics: the last solve needed the full-width re-run
    bool l0_async = false;             // level 0 solved on the factor stream (wb_level0_async, ev_l0)
    cudaEvent_t ev_l0 = nullptr;
    cudaStream_t factor_stream = nullptr;
    cplx* wb_Ad = nullptr;             // the diagonal blocks being factored early
    // QPS_TIMELINE=1: non-blocking timing events at phase boundaries on their
    // own streams, printed after qps_solve (critical-path study, no syncs)
    std::vector<std::pair<const char*, cudaEvent_t>> tl_marks;
    std::vector<cudaEvent_t> tl_pool;
    cudaEvent_t ev_factor = nullptr, ev_f0 = nullptr, ev_f1 = nullptr;
    DBuf<int> l0_flag;
    int nrhs = 1;                      // right-hand sides per block of the next block solve (> 1: caller fills F)
    bool skip_corners = false;         // schur(): interior elimination only (alpha-grouped sweep)
    bool xint_shared = false;          // recover(): every system uses system 0's interior X
    // alpha-grouped sweep: per-angle corner problems, multi-RHS solution, capacitance systems
    DBuf<cplx> ag_Q, ag_R, ag_X, ag_eta, ag_cap, ag_w, ag_dinv;
    DBuf<int> ag_piv, ag_flag;
    CodSet cod_ag;
    std::vector<int> sweep_group;      // last sweep: alpha group of every angle (-1: not solved)
    int sweep_ngroups = 0;
    // residual suite: private source pool and refined densities
    DBuf<double> res_px, res_py, res_pnx, res_pny, res_pw;
    DBuf<cplx> res_eta;
    uint64_t sweep_interior = 0, sweep_factorizations = 0;  // interior eliminations / block factorizations
    uint64_t n_factorizations = 0;     // block-solve factorizations performed (the sweep's per-group counter)
    DBuf<cplx> bcr_copy, bcr_cdinv;    // dense reduction: factored copies of the even blocks (rcond test)
    DBuf<int> bcr_cpiv;
    HBuf<int> rc_flag_h;
    // coupling Schur updates A'_{j,j+1} = A - B X left to the compression
    // (one-shot path): [system][j] tasks of A_super and A_sub
    std::vector<GemmTask> coupling_sup, coupling_sub;
    bool couplings_deferred = false;
    bool lr_sample_pending = false;
    DBuf<GemmTask> lr_tasks;  // task table of the side2 stream's GEMMs
    CodSet lr_cod;
    std::vector<DBuf<cplx>> lr_Z, lr_Rn;
    DBuf<cplx> lr_W0, lr_S, lr_g, lr_Cm, lr_Ci, lr_Cdinv, lr_a;  // Woodbury cyclic reduction
    DBuf<int> lr_Cpiv;

    // ---- block cyclic reduction ----
    std::vector<BcrLevels> levels;  // [level][system]
    std::vector<DBuf<cplx>> lvlL, lvlU;
    DBuf<cplx> F, eta, dinv;
    DBuf<int> ipiv, singular;
    DBuf<cplx*> dptrA, dptrB;
    DBuf<int*> dptrP;
    bool eta_valid = false;

    // ---- solution ----
    DBuf<cplx> csol, aUd, aDd;
    HBuf<cplx> h_eta;                                // system 0 densities (pinned: one DMA, no repack)
    size_t h_eta_n = 0;
    std::vector<cplx> h_c, h_aU, h_aD;               // system 0
    std::vector<cplx> h_aU_all, h_aD_all;            // nsys x (2K+1)
    std::vector<double> lsq_all;                     // nsys x (I+1)
    bool have_sol = false;
    double flux_error = 0.0, max_lsq = 0.0;

    // ---- bookkeeping ----
    qps_phase_times times{};
    uint64_t ref_evals = 0, performed_evals = 0;
    Workspace ws;
    Workspace ws2;                     // task tables of the early level-0 factorization (stream side)
    // the early level-0 batch split into chunks on their own streams, so the
    // latency-bound panels of one chunk overlap the GEMMs of another and a
    // chunk's solve starts as soon as its own factors exist
    static constexpr int kL0MaxChunks = 4;
    cudaStream_t l0_s[kL0MaxChunks] = {};
    cudaEvent_t l0_ev[kL0MaxChunks] = {};
    Workspace l0_ws[kL0MaxChunks];
    int l0_chunks = 1;
    // iterative refinement of the Woodbury block solve: steps (qps_set_refine,
    // QPS_REFINE; the sweeps default to one), the unfactored diagonal blocks
    // and right-hand sides it needs, the residual / correction buffer, and the
    // relative residuals ||f - A' eta|| / ||f|| before / after the last step
    int refine = -1;                   // -1: the default of the caller (refine_default)
    int refine_default = 0;            // 1 inside the sweeps
    int refine_used = 0;               // steps applied by the last block solve
    HBuf<double> ref_nrm_h;            // host copy of ref_nrm
    int ref_nrm_n = 0;                 // blocks per slot of ref_nrm
    bool refine_ready = false;         // ref_D / ref_F hold this solve's copies
    const cplx *ref_Au = nullptr, *ref_Al = nullptr;  // the couplings of the solve being refined
    DBuf<cplx> ref_D, ref_F, ref_R, ref_X, ref_A;
    DBuf<double> ref_nrm;              // per-block ||r_before||, ||r_after||, ||f|| of the last refinement
    std::vector<std::vector<std::vector<WbPos>>> wb_levels;
    std::chrono::steady_clock::time_point host_t0;  // QPS_HOST_TRACE
    DBuf<PairTask> d_pair;
    DBuf<ProxyTask> d_proxy;
    DBuf<AlpertTask> d_alpert;
    DBuf<int4> d_tiles;
    // one-shot solves split the fill: the wall / radiation blocks and the proxy
    // blocks that the Schur least squares read first on the main stream, the
    // couplings, self blocks and their Alpert corrections on side3, joined
    // before the A' update (fill_overlap; opt-in QPS_FILL_OVERLAP=1, no gain measured)
    bool fill_overlap = false, fill_pending = false, fill_err_pending = false;
    bool sketch_in_fill = false;   // one-shot solve: the fill launches the coupling sketch (set by qps_solve)
    bool sketch_launched = false;  // ... and did (lr_sample_async already queued)
    cudaEvent_t ev_fillB = nullptr;
    cudaEvent_t ev_rhs = nullptr;      // level fork/join of the Woodbury reduction's right-hand-side half
    // one-shot solves: the interior least squares' residual norms (reported
    // only) run on a low-priority stream beside the A' update and the block
    // solve; schur_finish joins them and fills lsq / max_lsq
    cudaStream_t lsq_stream = nullptr;
    bool lsq_pending = false, lsq_corners = false;
    std::vector<double> lsq_li, lsq_lc;
    cudaStream_t fill_stream = nullptr;
    DBuf<PairTask> d_pair2;
    DBuf<int4> d_tiles2;
    HBuf<int> fill_err_h;
    std::string err_msg;
    int err_layer = 0;
    uint64_t err_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

// geometry / problem
void upload_geometry(Ctx& c);
void setup_dims(Ctx& c, bool check_solvable = true);
// one-shot fused single-angle fill of the assembled system (alpha recombination fused)
void fill_system_fused(Ctx& c);
// Schur complements in place on (A_diag, A_super, A_sub) or on the A' copies,
// for all dims.nsys systems (system a at base + a * stride)
// defer_lsq: leave the per-layer LSQ residuals in flight (schur_finish)
void schur(Ctx& c, cplx* Ad, cplx* Au, cplx* Al, bool defer_couplings = false, bool defer_lsq = false);
// joins deferred LSQ residual norms into the main stream and fills lsq / max_lsq
void schur_finish(Ctx& c);
// a solve attempt threw e: true when the caller should run it once more
// (kRetryWidth -> full basis width, kRetryDense -> dense reduction; each once)
inline bool solve_retry(Ctx& c, const Error& e) {
    if (e.status != QPS_ERR_INTERNAL) return false;
    if (e.what() == std::string(kRetryWidth) && !c.lr_full_width) {
        c.lr_full_width = true;
        c.lr_width_retried = true;
        return true;
    }
    if (e.what() == std::string(kRetryDense) && !c.force_dense) {
        c.force_dense = true;
        return true;
    }
    return false;
}
// block cyclic reduction of all systems with RHS f (per system); eta in c.F
void bcr_solve(Ctx& c, cplx* Ad, cplx* Au, cplx* Al);
// allocate the per-system buffers of the assembled system for dims.nsys systems
void alloc_system(Ctx& c);
void recover(Ctx& c);
// low-rank couplings: compress A'_{j,j+1}, A'_{j+1,j} of every system (false if not low rank)
bool lr_compress(Ctx& c, cplx* Au, cplx* Al);
// start the A Omega part of the compression sample on the side2 stream (one-shot path, after the fill)
void lr_sample_async(Ctx& c);
// block cyclic reduction on the compressed couplings (after lr_compress)
void bcr_solve_lr(Ctx& c, cplx* Ad);
void bcr_solve_wb(Ctx& c, cplx* Ad);
void wb_anorm_async(Ctx& c, const cplx* Ad);
bool lr_eligible_pub(const Ctx& c);  // the low-rank reduction applies to these dims
// factor every diagonal block of the Woodbury reduction (level 0) on the side
// stream; bcr_solve_wb then only solves with the factors
void wb_factor_async(Ctx& c, cplx* Ad);
// level 0 solved on the factor stream once the compressed bases exist (called by lr_compress)
void wb_level0_async(Ctx& c);
void qsolve_family_public(Ctx& c, CodSet& cs, const cplx* Q, const cplx* R, int ldR, size_t Rstride, cplx* X,
                          int ldX, size_t Xstride, double* lsq_out);
void host_spectrum(const Ctx& c, double* R, double* T, double* fe, double* kappa, cplx* kU, cplx* kD, int* pu,
                   int* pd);
// flux_error + reflection_transmission of one angle's Bragg amplitudes
void spectrum_of(const Problem& p, double d, const cplx* aU, const cplx* aD, double* R, double* T, double* fe,
                 double* kappa, cplx* kU, cplx* kD, int* pu, int* pd);
// W blocks of Q' and the RHS f of every system of the batch (host, O(M K) + O(N))
// (Qdst: the corner Q' blocks to write W into, default c.Qc)
void write_radiation_and_rhs(Ctx& c, const std::vector<Problem>& probs, cplx* Qdst = nullptr);
// identity on the unused diagonal of padded A_jj blocks, every system
void pad_identity(Ctx& c, cudaStream_t s = nullptr);
// precompute_shift_blocks (assembly.hpp:212-287) into c.cache_pool
void cache_fill(Ctx& c);
// assemble_system (assembly.hpp:462-483) for dims.nsys angles from the cache
void assemble_from_cache(Ctx& c, const std::vector<Problem>& probs);
// evaluate_field (postprocess.hpp:78-123) for the last solution; region 0 above
// y_U, 1 inside a layer, 2 below y_D
void evaluate_field(Ctx& c, int n, const double* xy, cplx* u_scat, cplx* u_tot, int* region, int* layer);
// device sums of layer representations for explicit tasks (field.cu): points
// qx/qy grouped per task, tiles (task, first point) of kFieldTile points,
// sources and proxies at offsets of `pool`
void field_sums(Ctx& c, const std::vector<FieldTask>& tasks, const std::vector<int2>& tiles,
                const std::vector<double>& qx, const std::vector<double>& qy, const DevPool& pool,
                std::vector<cplx>& out);
// residual_suite / interface_matching_residual (postprocess.hpp:263-399) of the last solution
double interface_matching_residual(Ctx& c, int j, int n_probe);
void residual_suite(Ctx& c, const std::vector<int>& ifaces, double* wall_qp, double* radiation, double* iface);
// multi-angle sweep; mode 0 accelerated (cache once, angles batched), 1 independent
void run_sweep(Ctx& c, int n, const double* theta, int K, int mode, double* R, double* T, double* fe, cplx* aU,
               cplx* aD, int* status);
// plan_sweep: angles on the alpha grid of n distinct alphas in (th_lo, th_hi)
std::vector<double> plan_sweep_angles(double k1, double d, int n_alpha, double th_lo, double th_hi);
// alpha group of each listed problem (|alpha_a - alpha_b| <= 1e-12)
std::vector<int> group_by_alpha(const std::vector<Problem>& probs, const std::vector<int>& ids, int* ngroups);

inline bool timeline_on() {
    static const bool on = getenv("QPS_TIMELINE") != nullptr;
    return on;
}
inline void tl_mark(Ctx& c, const char* what, cudaStream_t s) {
    if (!timeline_on()) return;
    cudaEvent_t e;
    if (c.tl_pool.empty()) cudaEventCreate(&e);
    else { e = c.tl_pool.back(); c.tl_pool.pop_back(); }
    cudaEventRecord(e, s);
    c.tl_marks.push_back({what, e});
}
inline void tl_report(Ctx& c) {
    if (!timeline_on() || c.tl_marks.empty()) return;
    cudaDeviceSynchronize();
    fprintf(stderr, "timeline (ms from %s):", c.tl_marks.front().first);
    for (auto& m : c.tl_marks) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c.tl_marks.front().second, m.second);
        fprintf(stderr, " %s %.2f |", m.first, ms);
        c.tl_pool.push_back(m.second);
    }
    fprintf(stderr, "\n");
    c.tl_marks.clear();
}

struct Timer {
    Ctx& c;
    double* slot;
    Timer(Ctx& c_, double* s) : c(c_), slot(s) { QPS_CUDA(cudaEventRecord(c.ev0, c.stream)); }
    // noexcept: a destructor that threw while an exception (e.g. a sticky
    // CUDA error) is already unwinding would std::terminate the host process;
    // the C-ABI promises status codes, so timing is skipped on that path.
    ~Timer() noexcept {
        if (std::uncaught_exceptions() > 0) return;
        float ms = 0;
        if (cudaEventRecord(c.ev1, c.stream) != cudaSuccess || cudaEventSynchronize(c.ev1) != cudaSuccess ||
            cudaEventElapsedTime(&ms, c.ev0, c.ev1) != cudaSuccess)
            return;  // the next checked CUDA call reports the error
        *slot = ms;
    }
};

}  // namespace qpsb
