// Block cyclic reduction with low-rank couplings.
//
// The off-diagonal blocks of the periodized system, A'_{j,j+1} and A'_{j+1,j}
// (interface-to-interface interactions across one layer, minus the rank-P
// proxy correction), are numerically low rank: at config 4 (interfaces one
// period apart, k up to 30) their singular values fall below 1e-15 of the
// largest after ~35 of 600 (tools/coupling_rank.py).  Each coupling is
// compressed once, C ~= P (P^* C) with P an orthonormal n x r basis from a
// randomized range finder (C Omega, Omega n x 64) and column-pivoted QR of the
// sample (the Eigen-semantics CPQR kernel, rank at a relative 1e-15), r the
// fixed basis width (48 columns, more than any coupling's rank).
//
// Cyclic reduction then never forms a dense D^{-1} L or D^{-1} U: with
// L = P_L R_L and U = P_U R_U (R = P^* C, r x n) an odd elimination needs
//   Z = D_o^{-1} [P_L P_U]                   (n x 2r solve instead of n x 2n)
//   D_e -= P_L (R_L Z_U) R_U + P_U (R_U Z_L) R_L       (rank-r updates)
//   L'_e = P_L (-(R_L Z_L) R_L(o))  U'_e = P_U (-(R_U Z_U) R_U(o))
// so fill-in couplings keep the left factor of the even block and a new r x n
// right factor, and the work per elimination drops from 50.7 n^3 to about
// n^3 (8/3 + 32 r/n) real flops -- the LU of D_o dominates.  Back-substitution:
//   eta_o = z_o - Z_L (R_L(o) eta_{o-1}) - Z_U (R_U(o) eta_{o+1}).
// The truncation error (relative 1e-15 of each coupling) is far below the
// problem's own noise floor; systems whose couplings are not low rank
// (rank > 48 of a 64-column sample) take the dense cyclic reduction.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "ctx.h"
#include "prof.h"

namespace qpsb {

namespace {

constexpr int kLrSample = 64;    // columns of the random sample
constexpr int kLrMaxRank = 48;   // beyond this the dense reduction is used
constexpr double kLrTol = 1e-14; // relative pivot threshold of the sample's CPQR

// P_b = first r columns of Q (Q^* = H_{r-1} ... H_0 as applied by the CPQR, so
// Q e_c = H_0^* ... H_c^* e_c), and PH_b = P_b^*.  One warp per column.
__global__ void __launch_bounds__(256) lr_form_q_kernel(int m, int p, int r, const cplx* __restrict__ W,
                                                        const cplx* __restrict__ tau, cplx* __restrict__ P, int ldp,
                                                        size_t pstride, cplx* __restrict__ PH, size_t phstride) {
    extern __shared__ cplx lrv[];  // 8 warps x m
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const cplx* Wb = W + size_t(b) * m * p;
    const cplx* tb = tau + size_t(b) * p;
    cplx* v = lrv + size_t(warp) * m;
    for (int c = blockIdx.y * 8 + warp; c < r; c += gridDim.y * 8) {
        for (int i = lane; i < m; i += 32) v[i] = cplx{i == c ? 1.0 : 0.0, 0.0};
        __syncwarp();
        for (int k = min(c, p - 1); k >= 0; --k) {
            const cplx tk = tb[k];
            if (tk.re == 0.0 && tk.im == 0.0) continue;
            // t = w^* v, w = [0..0, 1, W[k+1.., k]]
            cplx t{0, 0};
            for (int i = k + 1 + lane; i < m; i += 32) {
                const cplx e = Wb[size_t(k) * m + i];
                const cplx a = v[i];
                t.re += e.re * a.re + e.im * a.im;
                t.im += e.re * a.im - e.im * a.re;
            }
            for (int o = 16; o > 0; o >>= 1) {
                t.re += __shfl_xor_sync(0xffffffffu, t.re, o);
                t.im += __shfl_xor_sync(0xffffffffu, t.im, o);
            }
            const cplx vk = v[k];
            t.re += vk.re;
            t.im += vk.im;
            // v -= conj(tau) w t
            const cplx ct{tk.re * t.re + tk.im * t.im, tk.re * t.im - tk.im * t.re};
            __syncwarp();
            if (lane == 0) {
                v[k].re -= ct.re;
                v[k].im -= ct.im;
            }
            for (int i = k + 1 + lane; i < m; i += 32) {
                const cplx e = Wb[size_t(k) * m + i];
                v[i].re -= e.re * ct.re - e.im * ct.im;
                v[i].im -= e.re * ct.im + e.im * ct.re;
            }
            __syncwarp();
        }
        cplx* pc = P + size_t(b) * pstride + size_t(c) * ldp;
        cplx* ph = PH + size_t(b) * phstride;
        for (int i = lane; i < m; i += 32) {
            const cplx x = v[i];
            pc[i] = x;
            ph[size_t(i) * r + c] = cplx{x.re, -x.im};
        }
        __syncwarp();
    }
}

GemmTask gemm1(const cplx* A, int lda, const cplx* B, int ldb, int K, cplx* C, int ldc) {
    GemmTask t{};
    t.nseg = 1;
    t.A[0] = A;
    t.lda[0] = lda;
    t.B[0] = B;
    t.ldb[0] = ldb;
    t.K[0] = K;
    t.C = C;
    t.ldc = ldc;
    return t;
}

GemvTask gemv1(const cplx* A, int lda, const cplx* x, int n, cplx* y) {
    GemvTask v{};
    v.nseg = 1;
    v.A[0] = A;
    v.lda[0] = lda;
    v.x[0] = x;
    v.n[0] = n;
    v.y = y;
    return v;
}

}  // namespace

namespace {
// random sample matrix (seeded, fixed), uploaded on stream s
void lr_omega_setup(Ctx& c, cudaStream_t s) {
    const int nb = c.dims.nb;
    if (c.lr_omega_n == nb) return;
    std::vector<cplx> om(size_t(nb) * kLrSample);
    uint64_t x = 0x9e3779b97f4a7c15ull;
    for (auto& z : om) {
        auto next = [&]() {
            x ^= x >> 12;
            x ^= x << 25;
            x ^= x >> 27;
            return double((x * 0x2545f4914f6cdd1dull) >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
        };
        z = cplx{next(), next()};
    }
    c.lr_omega.upload(om, s);
    c.lr_omega_n = nb;
}
bool lr_eligible(const Ctx& c) {
    static const bool dense_only = [] {
        const char* e = getenv("QPS_BCR");
        return e && !strcmp(e, "dense");
    }();
    return !dense_only && c.dims.I >= 2 && c.dims.nb >= 4 * kLrSample;
}
}  // namespace

// The sample's A Omega part needs only the assembled couplings: it runs on a
// second stream while the Schur least squares (latency-bound) run on the main
// one.  lr_compress adds the B (-X Omega) correction once X exists.
void lr_sample_async(Ctx& c) {
    c.lr_sample_pending = false;
    if (!lr_eligible(c)) return;
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys;
    const int nc = 2 * ns * (I - 1);
    QPS_CUDA(cudaEventRecord(c.ev_fill, c.stream));
    QPS_CUDA(cudaStreamWaitEvent(c.side2, c.ev_fill, 0));
    lr_omega_setup(c, c.side2);
    c.lr_Y.ensure(size_t(nc) * nb * kLrSample);
    std::vector<GemmTask> t(nc);
    for (int q = 0; q < nc; ++q) {
        const int a = q / (2 * (I - 1)), rem = q % (2 * (I - 1));
        const bool sup = rem >= I - 1;
        const int j = sup ? rem - (I - 1) : rem;
        const cplx* C = (sup ? c.Asup.p : c.Asub.p) + size_t(a) * D.sU() + size_t(j) * D.nb2();
        t[q] = gemm1(C, nb, c.lr_omega.p, nb, nb, c.lr_Y.p + size_t(q) * nb * kLrSample, nb);
    }
    {
        ProfPhase phase("lowrank");
        zgemm_batched(nb, kLrSample, cplx{1, 0}, cplx{0, 0}, t, c.side2, c.lr_tasks, "lr_compress");
    }
    QPS_CUDA(cudaEventRecord(c.ev_sample, c.side2));
    c.lr_sample_pending = true;
}

// Compress every coupling of every system: c.lr_P / c.lr_R (per coupling,
// n x r ld nb and r x n ld r), ordered [system][sub 0..I-2][super 0..I-2].
bool lr_compress(Ctx& c, cplx* Au, cplx* Al) {
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys;
    if (!lr_eligible(c)) return false;  // small blocks: dense is cheap
    cudaStream_t s = c.stream;
    ProfPhase phase("lowrank");
    const int nc = 2 * ns * (I - 1);
    lr_omega_setup(c, s);
    auto coupling = [&](int q) -> const cplx* {  // q in [0, nc)
        const int a = q / (2 * (I - 1)), rem = q % (2 * (I - 1));
        const bool sup = rem >= I - 1;
        const int j = sup ? rem - (I - 1) : rem;
        return (sup ? Au : Al) + size_t(a) * D.sU() + size_t(j) * D.nb2();
    };
    // deferred coupling Schur updates (one-shot path): C = A - Bc X, never formed
    const bool corr = c.couplings_deferred;
    auto corr_task = [&](int q) -> const GemmTask& {
        const int a = q / (2 * (I - 1)), rem = q % (2 * (I - 1));
        return rem >= I - 1 ? c.coupling_sup[size_t(a) * (I - 1) + rem - (I - 1)]
                            : c.coupling_sub[size_t(a) * (I - 1) + rem];
    };
    const int P = D.P;
    // Y = C Omega  (= A Omega + Bc (-X Omega) when deferred)
    c.lr_Y.ensure(size_t(nc) * nb * kLrSample);
    const bool early = c.lr_sample_pending && corr;  // Y already holds A Omega
    if (c.lr_sample_pending) QPS_CUDA(cudaStreamWaitEvent(s, c.ev_sample, 0));
    c.lr_sample_pending = false;
    {
        std::vector<GemmTask> t(nc);
        if (corr) {
            c.lr_W.ensure(size_t(nc) * P * kLrSample);
            std::vector<GemmTask> w(nc);
            for (int q = 0; q < nc; ++q) {
                const GemmTask& u = corr_task(q);
                w[q] = gemm1(u.B[0], u.ldb[0], c.lr_omega.p, nb, nb, c.lr_W.p + size_t(q) * P * kLrSample, P);
            }
            zgemm_batched(P, kLrSample, cplx{-1, 0}, cplx{0, 0}, w, s, c.ws.gemm_tasks, "lr_compress");
        }
        for (int q = 0; q < nc && early; ++q) {  // Y += Bc (-X Omega)
            const GemmTask& u = corr_task(q);
            t[q] = gemm1(u.A[0], u.lda[0], c.lr_W.p + size_t(q) * P * kLrSample, P, P,
                         c.lr_Y.p + size_t(q) * nb * kLrSample, nb);
        }
        if (early) zgemm_batched(nb, kLrSample, cplx{1, 0}, cplx{1, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        for (int q = 0; q < nc && !early; ++q) {
            t[q] = gemm1(coupling(q), nb, c.lr_omega.p, nb, nb, c.lr_Y.p + size_t(q) * nb * kLrSample, nb);
            if (corr) {
                const GemmTask& u = corr_task(q);
                t[q].nseg = 2;
                t[q].A[1] = u.A[0];
                t[q].lda[1] = u.lda[0];
                t[q].B[1] = c.lr_W.p + size_t(q) * P * kLrSample;
                t[q].ldb[1] = P;
                t[q].K[1] = P;
            }
        }
        if (!early) {
            if (getenv("QPS_TRACE_LAUNCH"))
                fprintf(stderr, "lr_compress sample GEMM is zgemm3m launch index %llu\n",
                        (unsigned long long)g_zgemm_launches.load());
            zgemm_batched(nb, kLrSample, cplx{1, 0}, cplx{0, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        }
    }
    // column-pivoted QR of each sample, numerical rank
    CodSet& cs = c.lr_cod;
    cs.ensure(nc, nb, kLrSample, 1);
    CodBatch b = cs.batch(c.lr_Y.p);
    cod_factor_fast(b, s);
    cod_rank(b, kLrTol, nullptr, s);
    std::vector<int> rk(nc);
    QPS_D2H(rk.data(), cs.rank.p, sizeof(int) * nc, s);
    QPS_CUDA(cudaStreamSynchronize(s));
    int r = 0;
    for (int v : rk) r = std::max(r, v);
    if (getenv("QPS_LR_TRACE")) {
        int mn = 1 << 30;
        double mean = 0;
        for (int v : rk) { mn = std::min(mn, v); mean += v; }
        fprintf(stderr, "low-rank couplings: %d blocks, rank min %d mean %.1f max %d (sample %d)\n", nc, mn,
                mean / nc, r, kLrSample);
    }
    if (r > kLrMaxRank) return false;
    // a fixed basis width keeps every system's factors independent of the batch
    // it is solved in (the sweep's batched and one-at-a-time results agree)
    r = kLrMaxRank;
    c.lr_r = r;
    // P (n x r) and P^* (r x n)
    c.lr_P.ensure(size_t(nc) * nb * r);
    c.lr_PH.ensure(size_t(nc) * r * nb);
    {
        ProfScope ps("lr_compress", s, 0.0);
        static size_t attr = 0;
        const size_t sm = size_t(8) * nb * sizeof(cplx);
        if (sm > attr) {
            QPS_CUDA(cudaFuncSetAttribute(lr_form_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(std::max<size_t>(sm, 48 * 1024))));
            attr = std::max<size_t>(sm, 48 * 1024);
        }
        lr_form_q_kernel<<<dim3(nc, (r + 7) / 8), 256, size_t(8) * nb * sizeof(cplx), s>>>(
            nb, kLrSample, r, cs.W.p, cs.tau.p, c.lr_P.p, nb, size_t(nb) * r, c.lr_PH.p, size_t(r) * nb);
        QPS_CUDA(cudaGetLastError());
    }
    // R = P^* C  (= P^* A + (-P^* Bc) X when deferred)
    c.lr_R.ensure(size_t(nc) * r * nb);
    {
        if (corr) {
            c.lr_G.ensure(size_t(nc) * r * P);
            std::vector<GemmTask> g(nc);
            for (int q = 0; q < nc; ++q) {
                const GemmTask& u = corr_task(q);
                g[q] = gemm1(c.lr_PH.p + size_t(q) * r * nb, r, u.A[0], u.lda[0], nb, c.lr_G.p + size_t(q) * r * P, r);
            }
            zgemm_batched(r, P, cplx{-1, 0}, cplx{0, 0}, g, s, c.ws.gemm_tasks, "lr_compress");
        }
        std::vector<GemmTask> t(nc);
        for (int q = 0; q < nc; ++q) {
            t[q] = gemm1(c.lr_PH.p + size_t(q) * r * nb, r, coupling(q), nb, nb, c.lr_R.p + size_t(q) * r * nb, r);
            if (corr) {
                const GemmTask& u = corr_task(q);
                t[q].nseg = 2;
                t[q].A[1] = c.lr_G.p + size_t(q) * r * P;
                t[q].lda[1] = r;
                t[q].B[1] = u.B[0];
                t[q].ldb[1] = u.ldb[0];
                t[q].K[1] = P;
            }
        }
        zgemm_batched(r, nb, cplx{1, 0}, cplx{0, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
    }
    return true;
}

void bcr_solve_lr(Ctx& c, cplx* Ad) {
    ProfPhase phase("bcr");
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys, r = c.lr_r;
    const size_t nb2 = D.nb2();
    cudaStream_t s = c.stream;
    const cplx one{1, 0}, mone{-1, 0}, zero{0, 0};
    c.F.ensure(size_t(ns) * I * nb);
    c.F.zero(s);
    for (int a = 0; a < ns; ++a)
        QPS_CUDA(cudaMemcpyAsync(c.F.p + size_t(a) * I * nb, c.f.p + size_t(a) * nb, sizeof(cplx) * nb,
                                 cudaMemcpyDeviceToDevice, s));
    c.ipiv.ensure(size_t(ns) * I * nb);
    const size_t dsz = lu_dinv_elems(nb);
    c.dinv.ensure(size_t(ns) * I * dsz);
    auto ipiv_of = [&](int a, int j) { return c.ipiv.p + (size_t(a) * I + j) * nb; };
    auto dinv_of = [&](int a, int j) { return c.dinv.p + (size_t(a) * I + j) * dsz; };
    // per-position state of one system at one level
    struct Pos {
        int idx;
        cplx *D, *F;
        const cplx *PL, *RL, *PU, *RU;  // couplings: L = PL RL (to the left), U = PU RU (to the right)
        cplx* Z;                        // odd positions: D^{-1} [PL PU]
    };
    using Level = std::vector<std::vector<Pos>>;  // [system][position]
    std::vector<Level> levels;
    {
        Level L0(ns);
        const size_t per = size_t(nb) * r;
        for (int a = 0; a < ns; ++a) {
            const size_t qa = size_t(a) * 2 * (I - 1);
            for (int j = 0; j < I; ++j) {
                Pos p{};
                p.idx = j;
                p.D = Ad + size_t(a) * D.sA() + j * nb2;
                p.F = c.F.p + (size_t(a) * I + j) * nb;
                if (j >= 1) {  // L_j = A'_{j,j-1} = Asub[j-1]
                    p.PL = c.lr_P.p + (qa + (j - 1)) * per;
                    p.RL = c.lr_R.p + (qa + (j - 1)) * per;
                }
                if (j + 1 < I) {  // U_j = A'_{j,j+1} = Asup[j]
                    p.PU = c.lr_P.p + (qa + (I - 1) + j) * per;
                    p.RU = c.lr_R.p + (qa + (I - 1) + j) * per;
                }
                L0[a].push_back(p);
            }
        }
        levels.push_back(std::move(L0));
    }
    int nlev = 0;
    {
        int n = I;
        while (n > 1) { n = (n + 1) / 2; ++nlev; }
    }
    c.lr_Z.resize(std::max(nlev, 1));
    c.lr_Rn.resize(std::max(nlev, 1));
    c.lr_core.ensure(size_t(ns) * I * 4 * r * r);
    c.lr_T.ensure(size_t(ns) * I * 2 * r * nb);
    c.lr_vec.ensure(size_t(ns) * I * 4 * r);
    DBuf<int> flag;
    auto factor = [&](const std::vector<cplx*>& fa, const std::vector<int*>& fp, const std::vector<cplx*>& fd,
                      const std::vector<int>& orig) {
        flag.ensure(fa.size());
        flag.zero(s);
        lu_factor_batched(nb, nb, fa, fp, fd, flag.p, s, c.ws);
        std::vector<int> hf(fa.size());
        QPS_D2H(hf.data(), flag.p, sizeof(int) * hf.size(), s);
        QPS_CUDA(cudaStreamSynchronize(s));
        int worst = -1;
        for (size_t q = 0; q < hf.size(); ++q)
            if (hf[q] && (worst < 0 || orig[q] < worst)) worst = orig[q];
        if (worst >= 0)
            throw Error(QPS_ERR_SOLVER,
                        "singular diagonal factor (resonant parameters?) at layer " + std::to_string(worst + 1),
                        worst + 1);
    };
    int lvl = 0;
    while (levels[lvl][0].size() > 1) {
        Level& cur = levels[lvl];
        const int sz = int(cur[0].size());
        const int nodd = sz / 2;
        // 1. factor the odd positions; Z = D^{-1} [PL PU], z_f = D^{-1} f
        DBuf<cplx>& Zb = c.lr_Z[lvl];
        Zb.ensure(size_t(ns) * nodd * nb * 2 * r);
        std::vector<cplx*> fa, fd, zb, vb;
        std::vector<int*> fp;
        std::vector<int> orig;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) {
                Pos& p = cur[a][o];
                fa.push_back(p.D);
                fp.push_back(ipiv_of(a, p.idx));
                fd.push_back(dinv_of(a, p.idx));
                orig.push_back(p.idx);
                p.Z = Zb.p + (size_t(a) * nodd + o / 2) * nb * 2 * r;
                zb.push_back(p.Z);
                vb.push_back(p.F);
            }
        factor(fa, fp, fd, orig);
        {  // stage [PL PU] (zeros where a coupling is absent), then solve in place
            QPS_CUDA(cudaMemsetAsync(Zb.p, 0, sizeof(cplx) * size_t(ns) * nodd * nb * 2 * r, s));
            for (int a = 0; a < ns; ++a)
                for (int o = 1; o < sz; o += 2) {
                    const Pos& p = cur[a][o];
                    if (p.PL)
                        QPS_CUDA(cudaMemcpyAsync(p.Z, p.PL, sizeof(cplx) * size_t(nb) * r, cudaMemcpyDeviceToDevice,
                                                 s));
                    if (p.PU)
                        QPS_CUDA(cudaMemcpyAsync(p.Z + size_t(nb) * r, p.PU, sizeof(cplx) * size_t(nb) * r,
                                                 cudaMemcpyDeviceToDevice, s));
                }
            lu_solve_batched(nb, nb, fa, fp, fd, zb, nb, 2 * r, s, c.ws);
            lu_solve_batched(nb, nb, fa, fp, fd, vb, nb, 1, s, c.ws);
        }
        // 2. even positions: cores, products, rank-r updates, new couplings, RHS
        const int nsz = (sz + 1) / 2;
        DBuf<cplx>& Rn = c.lr_Rn[lvl];
        Rn.ensure(size_t(ns) * nsz * 2 * r * nb);
        std::vector<GemmTask> cores, prods, newr, upd;
        std::vector<GemvTask> v1, v2;
        Level nxt(ns);
        const size_t rn = size_t(r) * nb, rr = size_t(r) * r;
        for (int a = 0; a < ns; ++a) {
            for (int e = 0; e < sz; e += 2) {
                const Pos& pe = cur[a][e];
                const int q = e / 2;
                const size_t slot = size_t(a) * nsz + q;
                cplx* core = c.lr_core.p + slot * 4 * rr;  // [LU, LL, UL, UU]
                cplx* T = c.lr_T.p + slot * 2 * rn;       // [T1; T2] as two r x n blocks
                cplx* vec = c.lr_vec.p + slot * 4 * r;
                Pos np{};
                np.idx = pe.idx;
                np.D = pe.D;
                np.F = pe.F;
                GemmTask u{};
                const bool hm = e >= 1, hp = e + 1 < sz;
                if (hm) {
                    const Pos& po = cur[a][e - 1];
                    const cplx* ZL = po.Z;
                    const cplx* ZU = po.Z + size_t(nb) * r;
                    cores.push_back(gemm1(pe.RL, r, ZU, nb, nb, core + 0 * rr, r));  // R_L(e) Z_U(o)
                    cores.push_back(gemm1(pe.RL, r, ZL, nb, nb, core + 1 * rr, r));  // R_L(e) Z_L(o)
                    prods.push_back(gemm1(core + 0 * rr, r, po.RU, r, r, T, r));     // T1 = (R_L Z_U) R_U(o)
                    u.A[u.nseg] = pe.PL; u.lda[u.nseg] = nb; u.B[u.nseg] = T; u.ldb[u.nseg] = r; u.K[u.nseg] = r;
                    ++u.nseg;
                    if (e - 2 >= 0) {  // L'_e = -P_L(e) (R_L Z_L) R_L(o)
                        cplx* Rl = Rn.p + slot * 2 * rn;
                        newr.push_back(gemm1(core + 1 * rr, r, po.RL, r, r, Rl, r));
                        np.PL = pe.PL;
                        np.RL = Rl;
                    }
                    v1.push_back(gemv1(pe.RL, r, po.F, nb, vec));  // t = R_L(e) z_f(o)
                    v2.push_back(gemv1(pe.PL, nb, vec, r, pe.F));  // f_e -= P_L t
                }
                if (hp) {
                    const Pos& po = cur[a][e + 1];
                    const cplx* ZL = po.Z;
                    const cplx* ZU = po.Z + size_t(nb) * r;
                    cores.push_back(gemm1(pe.RU, r, ZL, nb, nb, core + 2 * rr, r));  // R_U(e) Z_L(o)
                    cores.push_back(gemm1(pe.RU, r, ZU, nb, nb, core + 3 * rr, r));  // R_U(e) Z_U(o)
                    prods.push_back(gemm1(core + 2 * rr, r, po.RL, r, r, T + rn, r));  // T2 = (R_U Z_L) R_L(o)
                    u.A[u.nseg] = pe.PU; u.lda[u.nseg] = nb; u.B[u.nseg] = T + rn; u.ldb[u.nseg] = r;
                    u.K[u.nseg] = r;
                    ++u.nseg;
                    if (e + 2 < sz) {  // U'_e = -P_U(e) (R_U Z_U) R_U(o)
                        cplx* Ru = Rn.p + slot * 2 * rn + rn;
                        newr.push_back(gemm1(core + 3 * rr, r, po.RU, r, r, Ru, r));
                        np.PU = pe.PU;
                        np.RU = Ru;
                    }
                    v1.push_back(gemv1(pe.RU, r, po.F, nb, vec + r));
                    v2.push_back(gemv1(pe.PU, nb, vec + r, r, pe.F));
                }
                if (u.nseg) {
                    u.C = pe.D;
                    u.ldc = nb;
                    upd.push_back(u);
                }
                nxt[a].push_back(np);
            }
        }
        zgemm_batched(r, r, one, zero, cores, s, c.ws.gemm_tasks, "lr_core");
        zgemm_batched(r, nb, one, zero, prods, s, c.ws.gemm_tasks, "lr_core");
        zgemm_batched(r, nb, mone, zero, newr, s, c.ws.gemm_tasks, "lr_core");  // L' = P_L (-(core) R)
        zgemm_batched(nb, nb, mone, one, upd, s, c.ws.gemm_tasks, "bcr_update");
        zgemv_batched(r, one, zero, v1, s, c.ws.gemv_tasks);
        zgemv_batched(nb, mone, one, v2, s, c.ws.gemv_tasks);
        levels.push_back(std::move(nxt));
        ++lvl;
    }
    // final block of every system
    {
        std::vector<cplx*> fa, fd, vb;
        std::vector<int*> fp;
        std::vector<int> orig;
        for (int a = 0; a < ns; ++a) {
            const Pos& p = levels[lvl][a][0];
            fa.push_back(p.D);
            fd.push_back(dinv_of(a, p.idx));
            fp.push_back(ipiv_of(a, p.idx));
            vb.push_back(p.F);
            orig.push_back(p.idx);
        }
        factor(fa, fp, fd, orig);
        lu_solve_batched(nb, nb, fa, fp, fd, vb, nb, 1, s, c.ws);
    }
    // back substitution: eta_o = z_o - Z_L (R_L(o) eta_{o-1}) - Z_U (R_U(o) eta_{o+1})
    for (int l = lvl - 1; l >= 0; --l) {
        const Level& cur = levels[l];
        const int sz = int(cur[0].size());
        std::vector<GemvTask> t1, t2;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) {
                const Pos& p = cur[a][o];
                cplx* vec = c.lr_vec.p + (size_t(a) * I + p.idx) * 4 * r;
                GemvTask w{};
                if (p.RL) {
                    t1.push_back(gemv1(p.RL, r, cur[a][o - 1].F, nb, vec));
                    w.A[w.nseg] = p.Z; w.lda[w.nseg] = nb; w.x[w.nseg] = vec; w.n[w.nseg] = r; ++w.nseg;
                }
                if (p.RU && o + 1 < sz) {
                    t1.push_back(gemv1(p.RU, r, cur[a][o + 1].F, nb, vec + r));
                    w.A[w.nseg] = p.Z + size_t(nb) * r; w.lda[w.nseg] = nb; w.x[w.nseg] = vec + r;
                    w.n[w.nseg] = r;
                    ++w.nseg;
                }
                if (w.nseg) {
                    w.y = p.F;
                    t2.push_back(w);
                }
            }
        zgemv_batched(r, one, zero, t1, s, c.ws.gemv_tasks);
        zgemv_batched(nb, mone, one, t2, s, c.ws.gemv_tasks);
    }
    c.eta_valid = true;
}

}  // namespace qpsb
