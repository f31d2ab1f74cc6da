// The alpha-free shift-block cache (ShiftBlockCache, assembly.hpp:115-155,
// precompute_shift_blocks :212-287), assembly of any number of incidence
// angles from it in ONE pass over the cache (assemble_system :462-483), and
// the multi-angle sweep: cache filled once, angles batched
// through recombination, Schur complements, block cyclic reduction and
// recovery.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "ctx.h"
#include "prof.h"

namespace qpsb {

namespace {

using cd = std::complex<double>;
inline cplx C(cd z) { return cplx{z.real(), z.imag()}; }

// coefficient ids of the per-angle phase table
enum Coef : int { K_ONE = 0, K_AINV, K_A, K_MONE, K_MAINV, K_MA, K_AINV2, K_NCOEF };

// out_a = sum_t coef_{a, t} piece_t for every system a of the batch; each
// cache element is read once for all angles (HBM-bound recombination).
__global__ void __launch_bounds__(256) combine_kernel(const CombineTask* __restrict__ tasks,
                                                      const int2* __restrict__ tiles, const cplx* __restrict__ pool,
                                                      const cplx* __restrict__ coefs, int nsys) {
    const int2 tl = tiles[blockIdx.x];
    const CombineTask& T = tasks[tl.x];
    const size_t e = size_t(tl.y) * blockDim.x + threadIdx.x;
    const size_t plane = size_t(T.rows) * T.cols;
    if (e >= plane) return;
    const int i = int(e % T.rows), j = int(e / T.rows);
    for (int kd = 0; kd < T.nplanes; ++kd) {
        cplx v[6];
#pragma unroll
        for (int t = 0; t < 6; ++t) v[t] = t < T.npiece ? pool[T.piece[t] + kd * plane + e] : cplx{0, 0};
        const int ro = (kd >= 2) ? T.row_off : 0;                 // T, D* rows below
        const int co = (kd == 1 || kd == 3) ? T.col_off : 0;      // S, D* columns right
        const size_t o = size_t(j + co) * T.ld + i + ro;
        const bool diag = T.ident && i == j && (kd == 0 || kd == 3);
        for (int a = 0; a < nsys; ++a) {
            const cplx* cf = coefs + size_t(a) * K_NCOEF;
            cplx acc{0, 0};
#pragma unroll
            for (int t = 0; t < 6; ++t) {
                if (t >= T.npiece) break;
                const cplx c = cf[T.coef[t]];
                acc.re += c.re * v[t].re - c.im * v[t].im;
                acc.im += c.re * v[t].im + c.im * v[t].re;
            }
            if (diag) acc.re += (kd == 0) ? -1.0 : 1.0;  // -I value block, +I derivative block
            T.out[a * T.ostride + o] = acc;
        }
    }
}

// alpha^{+-1} wrap contributions of the self blocks (SelfQuadParts::assemble,
// kernels.hpp:147-153): up minus down, every system
__global__ void band_kernel(const BandTask* __restrict__ tasks, int ntasks, const cplx* __restrict__ pool,
                            const cplx* __restrict__ coefs, int nsys) {
    const int t = blockIdx.y;
    if (t >= ntasks) return;
    const BandTask& B = tasks[t];
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= B.N * 33) return;
    const int m = e / 33, c = e % 33;
    const int jraw = m + c - 16;
    if (jraw >= 0 && jraw < B.N) return;
    const int col = (jraw + B.N) % B.N;
    const bool minus = jraw < 0;
    for (int kd = 0; kd < 4; ++kd) {
        const cplx u = pool[B.up + (size_t(m) * 33 + c) * 4 + kd];
        const cplx d = pool[B.dn + (size_t(m) * 33 + c) * 4 + kd];
        const cplx v{u.re - d.re, u.im - d.im};
        if (v.re == 0.0 && v.im == 0.0) continue;
        const int ro = (kd >= 2) ? B.N : 0, co = (kd == 1 || kd == 3) ? B.N : 0;
        const size_t o = size_t(col + co) * B.ld + m + ro;
        for (int a = 0; a < nsys; ++a) {
            const cplx ph = coefs[size_t(a) * K_NCOEF + (minus ? K_AINV : K_A)];
            cplx* p = B.out + a * B.ostride + o;
            p->re += ph.re * v.re - ph.im * v.im;
            p->im += ph.re * v.im + ph.im * v.re;
        }
    }
}

__global__ void pad_identity_kernel(cplx* __restrict__ A, size_t sA, int nb, const int* __restrict__ n2, int I,
                                    int nsys) {
    const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= size_t(nsys) * I * nb) return;
    const int i = int(e % nb), j = int((e / nb) % I), a = int(e / (size_t(nb) * I));
    if (i < n2[j]) return;
    A[a * sA + size_t(j) * nb * nb + size_t(i) * nb + i] = cplx{1.0, 0.0};
}

}  // namespace

void pad_identity(Ctx& c, cudaStream_t s) {
    const Dims& D = c.dims;
    if (!s) s = c.stream;
    std::vector<int> n2(D.I);
    for (int j = 0; j < D.I; ++j) n2[j] = 2 * D.N[j];
    c.d_nodes2.upload(n2, s);
    const size_t tot = size_t(D.nsys) * D.I * D.nb;
    { QPS_NOTE_LAUNCH(); pad_identity_kernel<<<unsigned((tot + 255) / 256), 256, 0, s>>>(c.Adiag.p, D.sA(), D.nb, c.d_nodes2.p, D.I,
                                                                            D.nsys); }
    QPS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// precompute_shift_blocks: the alpha-free pieces, every layer in a handful of
// launches (same kernels as the fused fill, single-term tasks, plane outputs)
// ---------------------------------------------------------------------------
void cache_fill(Ctx& c) {
    const Dims& D = c.dims;
    const HostGeometry& g = c.geo;
    const int I = D.I, nb = D.nb, P = D.P, Mw = D.Mw, M = D.M;
    const double d = g.d;
    const auto& k = c.prob.k;
    cudaStream_t s = c.stream;
    CacheLayout& L = c.cache;
    L = CacheLayout{};
    size_t off = 0;
    auto take = [&](size_t n) {
        const size_t o = off;
        off += (n + 1) & ~size_t(1);
        return o;
    };
    L.self_c.assign(I, {0, 0});
    L.band.assign(I, {0, 0});
    L.nbr_m.assign(I, {0, 0});
    L.nbr_p.assign(I, {0, 0});
    L.cup.assign(I, {0, 0, 0});
    L.cdn.assign(I, {0, 0, 0});
    L.Csp.assign(I + 1, 0);
    L.Csm.assign(I + 1, 0);
    L.Cap.assign(I + 1, 0);
    L.Cam.assign(I + 1, 0);
    L.Qp.assign(I + 1, 0);
    L.Qm.assign(I + 1, 0);
    for (int j = 0; j < I; ++j) {
        const size_t N = D.N[j];
        for (int sd = 0; sd < 2; ++sd) {
            L.self_c[j][sd] = take(4 * N * N);
            L.band[j][sd] = take(N * 33 * 4);
            L.nbr_m[j][sd] = take(4 * N * N);
            L.nbr_p[j][sd] = take(4 * N * N);
        }
        for (int l = 0; l < 3; ++l) {
            if (j >= 1) L.cup[j][l] = take(4 * N * D.N[j - 1]);
            if (j + 1 < I) L.cdn[j][l] = take(4 * N * D.N[j + 1]);
        }
    }
    for (int i = 0; i <= I; ++i) {
        if (i < I) {
            L.Csp[i] = take(4 * size_t(Mw) * D.N[i]);
            L.Csm[i] = take(4 * size_t(Mw) * D.N[i]);
        }
        if (i >= 1) {
            L.Cap[i] = take(4 * size_t(Mw) * D.N[i - 1]);
            L.Cam[i] = take(4 * size_t(Mw) * D.N[i - 1]);
        }
        L.Qp[i] = take(2 * size_t(Mw) * P);
        L.Qm[i] = take(2 * size_t(Mw) * P);
    }
    for (int l = 0; l < 3; ++l) {
        L.ZU[l] = take(4 * size_t(M) * D.N[0]);
        L.ZD[l] = take(4 * size_t(M) * D.N[I - 1]);
    }
    L.VU = take(2 * size_t(M) * P);
    L.VD = take(2 * size_t(M) * P);
    L.total = off;
    c.cache_pool.ensure(off);
    c.cache_pool.zero(s);  // band entries are sparse
    cplx* base = c.cache_pool.p;
    // B blocks are alpha-free: filled straight into the system's shared B (B_below signed)
    c.Bself.ensure(size_t(I) * nb * P);
    c.Bbelow.ensure(size_t(I) * nb * P);
    if (D.padded) {
        c.Bself.zero(s);
        c.Bbelow.zero(s);
    }
    QPS_CUDA(cudaMemsetAsync(c.d_err.p, 0, sizeof(int), s));

    std::vector<PairTask> pt;
    std::vector<ProxyTask> xt;
    std::vector<AlpertTask> at;
    int alpert_rows = 0;
    auto planes = [&](PairTask& t, size_t o, int rows, int cols) {
        const size_t pl = size_t(rows) * cols;
        t.oD = base + o;
        t.oS = base + o + pl;
        t.oT = base + o + 2 * pl;
        t.oDs = base + o + 3 * pl;
        t.ld = rows;
    };
    auto single = [&](int toff, int nt, int soff, int ns, double kk, int l, double tdx) {
        PairTask t{};
        t.t_off = toff;
        t.nt = nt;
        t.s_off = soff;
        t.ns = ns;
        t.nk = 1;
        t.k[0] = kk;
        t.ksign[0] = 1.0;
        t.nterm = 1;
        t.lsh[0] = l;
        t.tdx[0] = tdx;
        t.sdx[0] = d * l;
        t.coef[0] = cplx{1.0, 0.0};
        return t;
    };
    for (int j = 0; j < I; ++j) {
        const int N = D.N[j];
        const auto& q = g.ifaces[j];
        for (int sd = 0; sd < 2; ++sd) {
            const double kk = k[j + sd];
            // central part of self_quad_parts (kernels.hpp:199-215)
            PairTask t = single(c.iface_off[j], N, c.iface_off[j], N, kk, 0, 0.0);
            t.self = q.smooth ? 1 : 2;
            t.nseg = int(q.segs.size());
            for (int sgi = 0; sgi < t.nseg; ++sgi) t.seg_start[sgi] = q.segs[sgi].offset;
            t.seg_start[t.nseg] = N;
            planes(t, L.self_c[j][sd], N, N);
            pt.push_back(t);
            AlpertTask a{};
            a.t_off = c.iface_off[j];
            a.N = N;
            a.smooth = q.smooth ? 1 : 0;
            a.nseg = int(q.segs.size());
            a.seg_first = c.seg_first[j];
            a.aux_off = c.aux_off[j];
            a.row_start = alpert_rows;
            a.nk = 1;
            a.k[0] = kk;
            a.ksign[0] = 1.0;
            a.mode = 1;
            a.oD = t.oD;
            a.oS = t.oS;
            a.oT = t.oT;
            a.oDs = t.oDs;
            a.ld = N;
            a.wrap = base + L.band[j][sd];
            at.push_back(a);
            alpert_rows += N;
            // plain l = -1, +1 neighbour blocks (assembly.hpp:246-247)
            PairTask tm = single(c.iface_off[j], N, c.iface_off[j], N, kk, -1, 0.0);
            planes(tm, L.nbr_m[j][sd], N, N);
            pt.push_back(tm);
            PairTask tp = single(c.iface_off[j], N, c.iface_off[j], N, kk, 1, 0.0);
            planes(tp, L.nbr_p[j][sd], N, N);
            pt.push_back(tp);
        }
        for (int l = -1; l <= 1; ++l) {  // couplings (assembly.hpp:249-255)
            if (j >= 1) {
                PairTask t = single(c.iface_off[j], N, c.iface_off[j - 1], D.N[j - 1], k[j], l, 0.0);
                planes(t, L.cup[j][l + 1], N, D.N[j - 1]);
                pt.push_back(t);
            }
            if (j + 1 < I) {
                PairTask t = single(c.iface_off[j], N, c.iface_off[j + 1], D.N[j + 1], k[j + 1], l, 0.0);
                planes(t, L.cdn[j][l + 1], N, D.N[j + 1]);
                pt.push_back(t);
            }
        }
        for (int side = 0; side < 2; ++side) {  // B_self, B_below (assembly.hpp:256-257)
            ProxyTask x{};
            x.t_off = c.iface_off[j];
            x.nt = N;
            x.p_off = c.proxy_off[j + side];
            x.P = P;
            x.k = k[j + side];
            x.nterm = 1;
            x.coef[0] = cplx{side == 0 ? 1.0 : -1.0, 0.0};
            x.drow = N;
            x.out = (side == 0 ? c.Bself.p : c.Bbelow.p) + size_t(j) * nb * P;
            x.ld = nb;
            xt.push_back(x);
        }
    }
    for (int i = 0; i <= I; ++i) {  // walls (assembly.hpp:260-275)
        for (int which = 0; which < 2; ++which) {
            const int src = which == 0 ? i : i - 1;
            if (src < 0 || src >= I) continue;
            PairTask tpp = single(c.wall_off[i], Mw, c.iface_off[src], D.N[src], k[i], 0, 2.0 * d);
            planes(tpp, which == 0 ? L.Csp[i] : L.Cap[i], Mw, D.N[src]);
            pt.push_back(tpp);
            PairTask tmm = single(c.wall_off[i], Mw, c.iface_off[src], D.N[src], k[i], 0, -d);
            planes(tmm, which == 0 ? L.Csm[i] : L.Cam[i], Mw, D.N[src]);
            pt.push_back(tmm);
        }
        for (int pm = 0; pm < 2; ++pm) {
            ProxyTask x{};
            x.t_off = c.wall_off[i];
            x.nt = Mw;
            x.p_off = c.proxy_off[i];
            x.P = P;
            x.k = k[i];
            x.nterm = 1;
            x.tdx[0] = pm == 0 ? d : 0.0;
            x.coef[0] = cplx{1.0, 0.0};
            x.drow = Mw;
            x.out = base + (pm == 0 ? L.Qp[i] : L.Qm[i]);
            x.ld = 2 * Mw;
            xt.push_back(x);
        }
    }
    for (int side = 0; side < 2; ++side) {  // U/D (assembly.hpp:277-284)
        const int src = side == 0 ? 0 : I - 1, layer = side == 0 ? 0 : I;
        const int toff = side == 0 ? c.U_off : c.D_off;
        for (int l = -1; l <= 1; ++l) {
            PairTask t = single(toff, M, c.iface_off[src], D.N[src], k[layer], l, 0.0);
            planes(t, side == 0 ? L.ZU[l + 1] : L.ZD[l + 1], M, D.N[src]);
            pt.push_back(t);
        }
        ProxyTask x{};
        x.t_off = toff;
        x.nt = M;
        x.p_off = c.proxy_off[layer];
        x.P = P;
        x.k = k[layer];
        x.nterm = 1;
        x.coef[0] = cplx{1.0, 0.0};
        x.drow = M;
        x.out = base + (side == 0 ? L.VU : L.VD);
        x.ld = 2 * M;
        xt.push_back(x);
    }
    const DevPool pool{c.px.p, c.py.p, c.pnx.p, c.pny.p, c.pw.p};
    launch_pair_fill(pt, pool, c.d_err.p, s, c.d_pair, c.d_tiles);
    launch_alpert(at, alpert_rows, pool, c.segs.p, c.fourier.p, c.aux_pool.p, c.d_err.p, s, c.d_alpert);
    launch_proxy_fill(xt, pool, c.d_err.p, s, c.d_proxy, c.d_tiles);
    int herr = 0;
    QPS_D2H(&herr, c.d_err.p, sizeof(int), s);
    QPS_CUDA(cudaStreamSynchronize(s));
    if (herr) fail(QPS_ERR_SINGULARITY, "kernel evaluated at coincident target/source pair");
    // the same evaluation set as the reference (incl. wrap-removal pairs)
    c.ref_evals = reference_fill_evals(g);
    c.performed_evals = c.ref_evals;
    c.cache_k = k;
    c.cache_valid = true;
}

// ---------------------------------------------------------------------------
// assemble_system for dims.nsys angles (alphas[a]) from the cache
// ---------------------------------------------------------------------------
void assemble_from_cache(Ctx& c, const std::vector<Problem>& probs) {
    const Dims& D = c.dims;
    const HostGeometry& g = c.geo;
    const int I = D.I, nb = D.nb, P = D.P, Mw = D.Mw, M = D.M, ns = D.nsys;
    const CacheLayout& L = c.cache;
    cudaStream_t s = c.stream;
    alloc_system(c);
    if (D.padded) {
        c.Adiag.zero(s);
        c.Asup.zero(s);
        c.Asub.zero(s);
        c.Rint.zero(s);
        c.Rc.zero(s);
    }
    c.Qc.zero(s);
    // per-angle phase table (reference expressions: 1.0 / alpha, 1.0 / (alpha * alpha))
    std::vector<cplx> coefs(size_t(ns) * K_NCOEF);
    for (int a = 0; a < ns; ++a) {
        const cd al(probs[a].ar, probs[a].ai);
        const cd ai = 1.0 / al;
        const cd vals[K_NCOEF] = {1.0, ai, al, -1.0, -ai, -al, 1.0 / (al * al)};
        for (int q = 0; q < K_NCOEF; ++q) coefs[size_t(a) * K_NCOEF + q] = C(vals[q]);
    }
    c.coef_buf.upload(coefs, s);
    std::vector<CombineTask> ct;
    auto task4 = [&](int rows, int cols, std::initializer_list<std::pair<size_t, int>> pcs, cplx* out,
                     size_t ostride, int ld, int ident) {
        CombineTask t{};
        t.nplanes = 4;
        t.rows = rows;
        t.cols = cols;
        t.npiece = 0;
        for (const auto& pc : pcs) {
            t.piece[t.npiece] = pc.first;
            t.coef[t.npiece] = pc.second;
            ++t.npiece;
        }
        t.ident = ident;
        t.out = out;
        t.ostride = ostride;
        t.ld = ld;
        t.row_off = rows;
        t.col_off = cols;
        ct.push_back(t);
    };
    auto task1 = [&](int rows, int cols, std::initializer_list<std::pair<size_t, int>> pcs, cplx* out,
                     size_t ostride, int ld) {
        task4(rows, cols, pcs, out, ostride, ld, 0);
        ct.back().nplanes = 1;
    };
    std::vector<BandTask> bt;
    for (int j = 0; j < I; ++j) {
        const int N = D.N[j];
        // A_jj = tilde_up - tilde_dn - I/+I (assembly.hpp:343-352)
        task4(N, N,
              {{L.self_c[j][0], K_ONE}, {L.nbr_m[j][0], K_AINV}, {L.nbr_p[j][0], K_A},
               {L.self_c[j][1], K_MONE}, {L.nbr_m[j][1], K_MAINV}, {L.nbr_p[j][1], K_MA}},
              c.Adiag.p + j * D.nb2(), D.sA(), nb, 1);
        if (g.ifaces[j].smooth)
            bt.push_back(BandTask{N, L.band[j][0], L.band[j][1], c.Adiag.p + j * D.nb2(), D.sA(), nb});
        if (j + 1 < I)  // A_{j,j+1} = -tilde(coupl_dn)
            task4(N, D.N[j + 1], {{L.cdn[j][1], K_MONE}, {L.cdn[j][0], K_MAINV}, {L.cdn[j][2], K_MA}},
                  c.Asup.p + j * D.nb2(), D.sU(), nb, 0);
        if (j >= 1)  // A_{j,j-1} = +tilde(coupl_up)
            task4(N, D.N[j - 1], {{L.cup[j][1], K_ONE}, {L.cup[j][0], K_AINV}, {L.cup[j][2], K_A}},
                  c.Asub.p + (j - 1) * D.nb2(), D.sU(), nb, 0);
    }
    for (int i = 0; i <= I; ++i) {
        cplx *R, *Qo;
        int ldR, ldQ, col_self = -1, col_above = -1;
        size_t sR, sQ;
        if (i == 0) {
            R = c.Rc.p; ldR = D.mC; col_self = 0; Qo = c.Qc.p; ldQ = D.mC; sR = D.sRc(); sQ = D.sQc();
        } else if (i == I) {
            R = c.Rc.p + size_t(D.mC) * nb; ldR = D.mC; col_above = 0; Qo = c.Qc.p + size_t(D.mC) * D.pC; ldQ = D.mC;
            sR = D.sRc(); sQ = D.sQc();
        } else {
            R = c.Rint.p + size_t(i - 1) * D.mI * 2 * nb; ldR = D.mI; col_above = 0; col_self = nb;
            Qo = c.Qint.p + size_t(i - 1) * D.mI * P; ldQ = D.mI; sR = D.sRi(); sQ = D.sQi();
        }
        // C = alpha^-2 K(wall + 2d) - alpha K(wall - d) (assembly.hpp:375-397)
        if (col_self >= 0 && i < I)
            task4(Mw, D.N[i], {{L.Csp[i], K_AINV2}, {L.Csm[i], K_MA}}, R + size_t(col_self) * ldR, sR, ldR, 0);
        if (col_above >= 0 && i >= 1)
            task4(Mw, D.N[i - 1], {{L.Cap[i], K_AINV2}, {L.Cam[i], K_MA}}, R + size_t(col_above) * ldR, sR, ldR, 0);
        // Q = alpha^-1 Q_p - Q_m (assembly.hpp:400-404)
        task1(2 * Mw, P, {{L.Qp[i], K_AINV}, {L.Qm[i], K_MONE}}, Qo, sQ, ldQ);
    }
    for (int side = 0; side < 2; ++side) {  // Z into C', V into Q' (assembly.hpp:408-413, 443-460)
        const int src = side == 0 ? 0 : I - 1;
        const auto& Z = side == 0 ? L.ZU : L.ZD;
        task4(M, D.N[src], {{Z[1], K_ONE}, {Z[0], K_AINV}, {Z[2], K_A}},
              c.Rc.p + size_t(side) * D.mC * nb + 2 * Mw, D.sRc(), D.mC, 0);
        task1(2 * M, P, {{side == 0 ? L.VU : L.VD, K_ONE}}, c.Qc.p + size_t(side) * D.mC * D.pC + 2 * Mw, D.sQc(),
              D.mC);
    }
    // launch: tiles of 256 elements over every task
    std::vector<int2> tiles;
    double bytes = 0;
    for (int t = 0; t < int(ct.size()); ++t) {
        const size_t plane = size_t(ct[t].rows) * ct[t].cols;
        for (size_t e = 0; e < plane; e += 256) tiles.push_back(make_int2(t, int(e / 256)));
        bytes += 16.0 * plane * ct[t].nplanes * (ct[t].npiece + ns);
    }
    c.d_comb.upload(ct, s);
    c.d_ctiles.upload(tiles, s);
    {
        ProfScope ps("assemble", s, 0.0, bytes);
        { QPS_NOTE_LAUNCH(); combine_kernel<<<unsigned(tiles.size()), 256, 0, s>>>(c.d_comb.p, c.d_ctiles.p, c.cache_pool.p, c.coef_buf.p,
                                                              ns); }
        QPS_CUDA(cudaGetLastError());
    }
    if (!bt.empty()) {
        c.d_band.upload(bt, s);
        int maxn = 0;
        for (const auto& b : bt) maxn = std::max(maxn, b.N);
        ProfScope ps("assemble", s, 0.0, 0.0);
        { QPS_NOTE_LAUNCH(); band_kernel<<<dim3((maxn * 33 + 127) / 128, unsigned(bt.size())), 128, 0, s>>>(
            c.d_band.p, int(bt.size()), c.cache_pool.p, c.coef_buf.p, ns); }
        QPS_CUDA(cudaGetLastError());
    }
    // W blocks and f per angle (assembly.hpp:414-441): O(M K) + O(N) on the host
    write_radiation_and_rhs(c, probs);
    if (D.padded) pad_identity(c);
    c.sys_valid = true;
}

// ---------------------------------------------------------------------------
// Multi-angle sweep.  mode 0 ("accelerated"): the cache is
// filled once and the angles go through recombination, Schur, cyclic
// reduction and recovery in batches of independent systems; mode 1
// ("independent"): every angle refills the cache and is solved alone.  A
// failing angle (make_problem error, singular layer) is reported in its
// status slot; a batch that fails is re-run angle by angle.
// ---------------------------------------------------------------------------
namespace {

size_t per_system_bytes(const Dims& D) {
    // A (diag, super, sub) + BCR level couplings + LU inverses, least-squares
    // right-hand sides + COD workspace, Schur solutions, corner blocks, RHS
    const size_t elems = 3 * D.sA() + 4 * D.sU() + 3 * D.sRi() + 2 * D.sXi() + D.sQi() + 2 * D.sRc() +
                         2 * D.sXc() + D.sQc() + 4 * size_t(D.I) * D.nb;
    return elems * sizeof(cplx);
}

}  // namespace

// ---------------------------------------------------------------------------
// Alpha grouping.  The system matrix
// depends on theta only through alpha = exp(i d k_1 cos theta); the Rayleigh-
// Bloch columns W of the corner blocks Q'_1, Q'_{I+1} (and the right-hand side
// f) depend on theta itself (kappa_n = k_1 cos theta + 2 pi n / d).  Angles
// whose alphas agree to kAlphaTol form a group.
// ---------------------------------------------------------------------------
constexpr double kAlphaTol = 1e-12;

std::vector<int> group_by_alpha(const std::vector<Problem>& probs, const std::vector<int>& ids, int* ngroups) {
    std::vector<int> g(ids.size(), -1);
    std::vector<std::pair<double, double>> reps;
    for (size_t q = 0; q < ids.size(); ++q) {
        const Problem& p = probs[ids[q]];
        for (size_t r = 0; r < reps.size(); ++r)
            if (std::hypot(p.ar - reps[r].first, p.ai - reps[r].second) <= kAlphaTol) {
                g[q] = int(r);
                break;
            }
        if (g[q] < 0) {
            g[q] = int(reps.size());
            reps.push_back({p.ar, p.ai});
        }
    }
    *ngroups = int(reps.size());
    return g;
}

std::vector<double> plan_sweep_angles(double k1, double d, int n_alpha, double th_lo, double th_hi) {
    // "a uniform grid ... with spacing 2 pi / (n d k_1)" so
    // that only n distinct alphas occur -- uniform in cos(theta) (i.e. in
    // kappa_0 = k_1 cos theta with spacing 2 pi / (n d)): alpha_j = alpha_0
    // exp(2 pi i j / n) repeats with period n.  Incidence from above:
    // theta in (-pi, 0), where cos is increasing.
    if (n_alpha < 1) fail(QPS_ERR_CONFIG, "plan_sweep: n >= 1 alpha values required");
    if (!(th_lo > -kPi && th_hi < 0.0 && th_lo < th_hi))
        fail(QPS_ERR_CONFIG, "plan_sweep: theta range must satisfy -pi < lo < hi < 0");
    const double klo = k1 * std::cos(th_lo), khi = k1 * std::cos(th_hi), dk = 2.0 * kPi / (n_alpha * d);
    std::vector<double> th;
    for (int j = 0;; ++j) {
        const double kap = klo + (j + 0.5) * dk;
        if (kap >= khi) break;
        th.push_back(-std::acos(kap / k1));
    }
    return th;
}

// One alpha group solved with a single interior elimination and a single
// block factorization ("periodized factorization computed exactly
// once per alpha group"): the corner eliminations are the only theta-dependent
// Schur terms and they change A'_{0,0} and A'_{I-1,I-1} by
//   -B_self[0] X_first[:P] and -B_below[I-1] X_last[:P]       (periodize.hpp:115,119),
// i.e. A(theta) = A_alpha - B V(theta)^* with B = [B_self[0] e_0 | B_below[I-1] e_{I-1}]
// theta-independent (alpha-free, cache) and V^* the corner X's first P rows.
// One block cyclic reduction of A_alpha with m = 2P + g right-hand sides gives
// Z = A_alpha^{-1} B and y_t = A_alpha^{-1} f_t; per angle the Woodbury identity
//   eta_t = y_t + Z (I - V_t^* Z)^{-1} V_t^* y_t          (2P x 2P capacitance)
// then recovery as usual.
void solve_alpha_group(Ctx& c, const std::vector<Problem>& gp, qps_phase_times& tm) {
    const int g = int(gp.size());
    c.prob = gp[0];
    c.dims.nsys = 1;
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, P = D.P, mC = D.mC, pC = D.pC;
    cudaStream_t s = c.stream;
    auto timed = [&](double* slot, auto&& f) {
        double ms = 0;
        {
            Timer t(c, &ms);
            f();
        }
        *slot += ms;
    };
    timed(&tm.assemble_ms, [&] { assemble_from_cache(c, {gp[0]}); });
    lr_sample_async(c);
    timed(&tm.schur_ms, [&] {
        c.skip_corners = true;
        try {
            schur(c, c.Adiag.p, c.Asup.p, c.Asub.p, true);
        } catch (...) {
            c.skip_corners = false;
            throw;
        }
        c.skip_corners = false;
        ++c.sweep_interior;
        // the corner problems of every angle: Q'(theta_t) = [[Q 0]; [V W(theta_t)]], C' shared
        c.ag_Q.ensure(size_t(g) * D.sQc());
        c.ag_R.ensure(size_t(g) * D.sRc());
        c.ag_X.ensure(size_t(g) * D.sXc());
        for (int t = 0; t < g; ++t) {
            QPS_CUDA(cudaMemcpyAsync(c.ag_Q.p + size_t(t) * D.sQc(), c.Qc.p, sizeof(cplx) * D.sQc(),
                                     cudaMemcpyDeviceToDevice, s));
            QPS_CUDA(cudaMemcpyAsync(c.ag_R.p + size_t(t) * D.sRc(), c.Rc.p, sizeof(cplx) * D.sRc(),
                                     cudaMemcpyDeviceToDevice, s));
        }
        c.dims.nsys = g;
        write_radiation_and_rhs(c, gp, c.ag_Q.p);  // W of each angle; f of each angle into c.f (g x nb)
        c.dims.nsys = 1;
        c.cod_ag.ensure(2 * g, mC, pC, nb);
        std::vector<double> lc(2 * size_t(g));
        qsolve_family_public(c, c.cod_ag, c.ag_Q.p, c.ag_R.p, mC, size_t(mC) * nb, c.ag_X.p, pC, size_t(pC) * nb,
                             lc.data());
        c.lsq_all.resize(size_t(g) * (I + 1));
        for (int t = g - 1; t >= 0; --t) {
            for (int i = 1; i < I; ++i) c.lsq_all[size_t(t) * (I + 1) + i] = c.lsq_all[i];
            c.lsq_all[size_t(t) * (I + 1)] = lc[2 * t];
            c.lsq_all[size_t(t) * (I + 1) + I] = lc[2 * t + 1];
        }
    });
    const int m = 2 * P + g;
    const size_t fs = size_t(nb) * m;
    timed(&tm.solve_ms, [&] {
        // right-hand sides [B_self[0] | B_below[I-1] | f_1 .. f_g] (blocks 0 and I-1)
        c.F.ensure(size_t(I) * fs);
        c.F.zero(s);
        QPS_CUDA(cudaMemcpyAsync(c.F.p, c.Bself.p, sizeof(cplx) * nb * P, cudaMemcpyDeviceToDevice, s));
        QPS_CUDA(cudaMemcpyAsync(c.F.p + size_t(I - 1) * fs + size_t(P) * nb, c.Bbelow.p + size_t(I - 1) * nb * P,
                                 sizeof(cplx) * nb * P, cudaMemcpyDeviceToDevice, s));
        QPS_CUDA(cudaMemcpyAsync(c.F.p + size_t(2 * P) * nb, c.f.p, sizeof(cplx) * nb * g, cudaMemcpyDeviceToDevice,
                                 s));
        c.nrhs = m;
        try {
            bcr_solve(c, c.Adiag.p, c.Asup.p, c.Asub.p);
        } catch (...) {
            c.nrhs = 1;
            throw;
        }
        c.nrhs = 1;
        ++c.sweep_factorizations;
        // capacitance C_t = I - V_t^* Z (2P x 2P) and w_t = V_t^* y_t per angle
        const int p2 = 2 * P;
        c.ag_cap.ensure(size_t(g) * p2 * p2);
        c.ag_w.ensure(size_t(g) * p2);
        {
            std::vector<cplx> eye(size_t(g) * p2 * p2, cplx{0, 0});
            for (int t = 0; t < g; ++t)
                for (int i = 0; i < p2; ++i) eye[size_t(t) * p2 * p2 + size_t(i) * p2 + i] = cplx{1, 0};
            c.ag_cap.upload(eye, s);
        }
        std::vector<GemmTask> ct;
        std::vector<GemvTask> wt;
        for (int t = 0; t < g; ++t) {
            const cplx* Xf = c.ag_X.p + size_t(t) * D.sXc();
            const cplx* Xl = Xf + size_t(pC) * nb;
            cplx* Ct = c.ag_cap.p + size_t(t) * p2 * p2;
            GemmTask a{};
            a.nseg = 1; a.A[0] = Xf; a.lda[0] = pC; a.B[0] = c.F.p; a.ldb[0] = nb; a.K[0] = nb; a.C = Ct; a.ldc = p2;
            ct.push_back(a);
            a.A[0] = Xl; a.B[0] = c.F.p + size_t(I - 1) * fs; a.C = Ct + P;
            ct.push_back(a);
            GemvTask v{};
            v.nseg = 1; v.A[0] = Xf; v.lda[0] = pC; v.x[0] = c.F.p + size_t(p2 + t) * nb; v.n[0] = nb;
            v.y = c.ag_w.p + size_t(t) * p2;
            wt.push_back(v);
            v.A[0] = Xl; v.x[0] = c.F.p + size_t(I - 1) * fs + size_t(p2 + t) * nb; v.y = c.ag_w.p + size_t(t) * p2 + P;
            wt.push_back(v);
        }
        zgemm_batched(P, p2, cplx{-1, 0}, cplx{1, 0}, ct, s, c.ws.gemm_tasks, "ag_cap");
        zgemv_batched(P, cplx{1, 0}, cplx{0, 0}, wt, s, c.ws.gemv_tasks);
        // s_t = C_t^{-1} w_t (LU with the rcond test: a singular capacitance is a
        // singular A(theta_t), reported by the caller's per-angle fallback)
        const size_t dsz = lu_dinv_elems(p2);
        c.ag_dinv.ensure(size_t(g) * dsz);
        c.ag_piv.ensure(size_t(g) * p2);
        c.ag_flag.ensure(g);
        c.ag_flag.zero(s);
        std::vector<cplx*> ca, cd, cw;
        std::vector<int*> cp;
        for (int t = 0; t < g; ++t) {
            ca.push_back(c.ag_cap.p + size_t(t) * p2 * p2);
            cd.push_back(c.ag_dinv.p + size_t(t) * dsz);
            cp.push_back(c.ag_piv.p + size_t(t) * p2);
            cw.push_back(c.ag_w.p + size_t(t) * p2);
        }
        lu_factor_batched(p2, p2, ca, cp, cd, c.ag_flag.p, s, c.ws);
        lu_rcond_batched(p2, p2, c.ws.ptrs.p, nullptr, 0, c.ws.ptrs3.p, nullptr, 0, g, kRcondMin, c.ag_flag.p,
                         nullptr, s);
        std::vector<int> hf(g);
        QPS_D2H(hf.data(), c.ag_flag.p, sizeof(int) * g, s);
        lu_solve_batched(p2, p2, ca, cp, cd, cw, p2, 1, s, c.ws);
        // eta_t = y_t + Z s_t, every block
        c.ag_eta.ensure(size_t(g) * I * nb);
        for (int t = 0; t < g; ++t)
            QPS_CUDA(cudaMemcpy2DAsync(c.ag_eta.p + size_t(t) * I * nb, sizeof(cplx) * nb,
                                       c.F.p + size_t(p2 + t) * nb, sizeof(cplx) * fs, sizeof(cplx) * nb, I,
                                       cudaMemcpyDeviceToDevice, s));
        std::vector<GemvTask> et;
        for (int t = 0; t < g; ++t)
            for (int j = 0; j < I; ++j) {
                GemvTask v{};
                v.nseg = 1; v.A[0] = c.F.p + size_t(j) * fs; v.lda[0] = nb; v.x[0] = c.ag_w.p + size_t(t) * p2;
                v.n[0] = p2; v.y = c.ag_eta.p + (size_t(t) * I + j) * nb;
                et.push_back(v);
            }
        zgemv_batched(nb, cplx{1, 0}, cplx{1, 0}, et, s, c.ws.gemv_tasks);
        QPS_CUDA(cudaStreamSynchronize(s));
        for (int t = 0; t < g; ++t)
            if (hf[t]) fail(QPS_ERR_SOLVER, "alpha group: singular corner capacitance");
    });
    timed(&tm.recover_ms, [&] {
        std::swap(c.F, c.ag_eta);
        std::swap(c.Xc, c.ag_X);
        c.dims.nsys = g;
        c.xint_shared = true;
        try {
            recover(c);
        } catch (...) {
            std::swap(c.F, c.ag_eta);
            std::swap(c.Xc, c.ag_X);
            c.dims.nsys = 1;
            c.xint_shared = false;
            throw;
        }
        std::swap(c.F, c.ag_eta);
        std::swap(c.Xc, c.ag_X);
        c.dims.nsys = 1;
        c.xint_shared = false;
    });
}

void run_sweep(Ctx& c, int n, const double* theta, int K, int mode, double* R, double* T, double* fe, cplx* aU,
               cplx* aD, int* status) {
    // one step of iterative refinement by default: a sweep crosses angles where
    // cyclic reduction is markedly less accurate than the reference's block
    // Thomas (qps_set_refine overrides)
    struct RefineDefault {
        Ctx& c;
        int old;
        ~RefineDefault() { c.refine_default = old; }
    } rd{c, c.refine_default};
    c.refine_default = 1;
    const Problem orig = c.prob;
    const double omega = orig.omega;
    c.sweep_interior = c.sweep_factorizations = 0;
    c.sweep_ngroups = 0;
    c.sweep_group.assign(n, -1);
    const int nrb = 2 * K + 1;
    const double nan = std::nan("");
    std::vector<Problem> probs(n);
    std::vector<int> todo;
    for (int a = 0; a < n; ++a) {
        if (status) status[a] = QPS_OK;
        if (R) R[a] = nan;
        if (T) T[a] = nan;
        if (fe) fe[a] = nan;
        try {
            probs[a] = make_problem(c.stack, c.geo, omega, theta[a], K);
            todo.push_back(a);
        } catch (const Error& e) {
            if (status) status[a] = e.status;
        }
    }
    qps_phase_times tm{};
    cudaEvent_t t0, t1;
    QPS_CUDA(cudaEventCreate(&t0));
    QPS_CUDA(cudaEventCreate(&t1));
    QPS_CUDA(cudaEventRecord(t0, c.stream));
    auto finish = [&]() {
        cudaEventRecord(t1, c.stream);
        cudaEventSynchronize(t1);
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        tm.total_ms = ms;
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        c.times = tm;
        c.prob = orig;
        c.dims.nsys = 1;
        c.sys_valid = c.ps_valid = c.eta_valid = c.have_sol = false;
    };
    try {
        if (!todo.empty()) {
            c.prob = probs[todo[0]];
            setup_dims(c);  // K is common: configuration errors apply to every angle
            auto timed = [&](double* slot, auto&& f) {
                double ms = 0;
                {
                    Timer t(c, &ms);
                    f();
                }
                *slot += ms;
            };
            if (mode == 0 && !(c.cache_valid && c.cache_k == c.prob.k)) timed(&tm.fill_ms, [&] { cache_fill(c); });
            int B = 1;
            if (mode == 0) {
                size_t fr = 0, tot = 0;
                QPS_CUDA(cudaMemGetInfo(&fr, &tot));
                const size_t per = per_system_bytes(c.dims);
                B = int(std::max<size_t>(1, std::min<size_t>(32, (fr / 2) / std::max<size_t>(per, 1))));
                B = std::min(B, int(todo.size()));
                if (const char* e = std::getenv("QPS_SWEEP_BATCH")) B = std::max(1, std::min(B, std::atoi(e)));
            }
            auto solve_batch = [&](const std::vector<int>& ids) {
                std::vector<Problem> bp;
                for (int id : ids) bp.push_back(probs[id]);
                c.prob = bp[0];
                c.dims.nsys = int(ids.size());
                if (mode != 0) timed(&tm.fill_ms, [&] { cache_fill(c); });
                for (int attempt = 0;; ++attempt) {
                    timed(&tm.assemble_ms, [&] { assemble_from_cache(c, bp); });
                    lr_sample_async(c);
                    timed(&tm.schur_ms, [&] { schur(c, c.Adiag.p, c.Asup.p, c.Asub.p, true); });
                    c.sys_valid = false;
                    try {
                        c.allow_early = true;
                        timed(&tm.solve_ms, [&] { bcr_solve(c, c.Adiag.p, c.Asup.p, c.Asub.p); });
                        c.allow_early = false;
                    } catch (const Error& e) {
                        c.allow_early = false;
                        if (solve_retry(c, e)) continue;  // the batch once more: full width / dense
                        c.force_dense = c.lr_full_width = false;
                        throw;
                    }
                    c.force_dense = c.lr_full_width = false;
                    break;
                }
                c.sweep_interior += ids.size();  // one independent system per angle
                c.sweep_factorizations += ids.size();
                timed(&tm.recover_ms, [&] { recover(c); });
                for (size_t q = 0; q < ids.size(); ++q) {
                    const int id = ids[q];
                    double r, t, f;
                    spectrum_of(bp[q], c.geo.d, c.h_aU_all.data() + q * nrb, c.h_aD_all.data() + q * nrb, &r, &t, &f,
                                nullptr, nullptr, nullptr, nullptr, nullptr);
                    if (R) R[id] = r;
                    if (T) T[id] = t;
                    if (fe) fe[id] = f;
                    for (int i = 0; i < nrb; ++i) {
                        if (aU) aU[size_t(id) * nrb + i] = c.h_aU_all[q * nrb + i];
                        if (aD) aD[size_t(id) * nrb + i] = c.h_aD_all[q * nrb + i];
                    }
                }
            };
            // alpha groups of two or more angles share one interior elimination and
            // one factorization (mode 0); the rest go through the batched pipeline
            std::vector<int> singles;
            c.sweep_group.assign(n, -1);
            {
                int ng = 0;
                const std::vector<int> gid = group_by_alpha(probs, todo, &ng);
                c.sweep_ngroups = ng;
                std::vector<std::vector<int>> members(ng);
                for (size_t q = 0; q < todo.size(); ++q) {
                    members[gid[q]].push_back(todo[q]);
                    c.sweep_group[todo[q]] = gid[q];
                }
                static const bool no_groups = [] {  // QPS_SWEEP_GROUPS=0: every angle through the batches
                    const char* e = std::getenv("QPS_SWEEP_GROUPS");
                    return e && !std::strcmp(e, "0");
                }();
                for (auto& mb : members) {
                    if (mode != 0 || mb.size() < 2 || no_groups) {
                        singles.insert(singles.end(), mb.begin(), mb.end());
                        continue;
                    }
                    std::vector<Problem> gp;
                    for (int id : mb) gp.push_back(probs[id]);
                    try {
                        solve_alpha_group(c, gp, tm);
                        for (size_t q = 0; q < mb.size(); ++q) {
                            const int id = mb[q];
                            double r, t, f;
                            spectrum_of(gp[q], c.geo.d, c.h_aU_all.data() + q * nrb, c.h_aD_all.data() + q * nrb,
                                        &r, &t, &f, nullptr, nullptr, nullptr, nullptr, nullptr);
                            if (R) R[id] = r;
                            if (T) T[id] = t;
                            if (fe) fe[id] = f;
                            for (int i = 0; i < nrb; ++i) {
                                if (aU) aU[size_t(id) * nrb + i] = c.h_aU_all[q * nrb + i];
                                if (aD) aD[size_t(id) * nrb + i] = c.h_aD_all[q * nrb + i];
                            }
                        }
                    } catch (const Error& e) {
                        if (e.status == QPS_ERR_CUDA || e.status == QPS_ERR_INTERNAL) throw;
                        singles.insert(singles.end(), mb.begin(), mb.end());  // per-angle solves name the failure
                    }
                }
                std::sort(singles.begin(), singles.end());
            }
            if (mode == 0) B = std::min(B, std::max(1, int(singles.size())));
            for (size_t b0 = 0; b0 < singles.size(); b0 += B) {
                const std::vector<int> ids(singles.begin() + b0, singles.begin() + std::min(singles.size(), b0 + B));
                try {
                    solve_batch(ids);
                } catch (const Error& e) {
                    if (e.status == QPS_ERR_CUDA || e.status == QPS_ERR_INTERNAL) throw;
                    if (ids.size() == 1) {
                        if (status) status[ids[0]] = e.status;
                        continue;
                    }
                    for (int id : ids) {
                        try {
                            solve_batch({id});
                        } catch (const Error& e2) {
                            if (e2.status == QPS_ERR_CUDA || e2.status == QPS_ERR_INTERNAL) throw;
                            if (status) status[id] = e2.status;
                        }
                    }
                }
            }
        }
    } catch (...) {
        finish();
        throw;
    }
    finish();
}

}  // namespace qpsb
