// Field evaluation on the device: evaluate_field (postprocess.hpp:78-123).
// For every point inside a layer the scattered field is the layer
// representation (eval_layer_representation, postprocess.hpp:46-63): the
// alpha-phased D and S potentials of the interfaces above and below the layer
// (neighbor_sum_block, kernels.hpp:123-129: shifts l = -1, 0, 1 with
// alpha^l) applied to the solved densities, plus the layer's proxy expansion
// phi_p = D + ik S (proxy_block, kernels.hpp:294-308) applied to c_layer.
// Points are mapped into the central cell (x - m d) and multiplied by alpha^m;
// points above y_U / below y_D use the Rayleigh-Bloch sums (rb_sum,
// postprocess.hpp:65-76).  Plain Nystrom sums, no close-evaluation
// correction, exactly as the reference.
#include <algorithm>
#include <cmath>
#include <complex>

#include "ctx.h"
#include "prof.h"

namespace qpsb {

namespace {

using cd = std::complex<double>;

constexpr int kFieldPts = kFieldTile, kFieldWarps = 4;

__global__ void __launch_bounds__(32 * kFieldWarps) field_kernel(const FieldTask* __restrict__ tasks,
                                                                 const int2* __restrict__ tiles,
                                                                 const double* __restrict__ qx,
                                                                 const double* __restrict__ qy, DevPool pool,
                                                                 const double* __restrict__ g_near, cplx alpha,
                                                                 cplx alpha_inv, double d, cplx* __restrict__ out,
                                                                 int* err) {
    __shared__ double2 s_near2[QPS_HANKEL_XB * QPS_HANKEL_NEAR_TERMS * 2];
    __shared__ cplx s_acc[kFieldWarps][kFieldPts];
    for (int e = threadIdx.x; e < QPS_HANKEL_XB * QPS_HANKEL_NEAR_TERMS * 2; e += blockDim.x) {
        const int half = e & 1, kk = (e >> 1) % QPS_HANKEL_NEAR_TERMS, i = (e >> 1) / QPS_HANKEL_NEAR_TERMS;
        const double* cc = g_near + i * QPS_NEAR_STRIDE;
        s_near2[e] = make_double2(cc[(2 * half) * QPS_HANKEL_NEAR_TERMS + kk],
                                  cc[(2 * half + 1) * QPS_HANKEL_NEAR_TERMS + kk]);
    }
    __syncthreads();
    const int2 tl = tiles[blockIdx.x];
    const FieldTask& T = tasks[tl.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pi = tl.y + lane;
    const bool live = pi < T.npt;
    const double x = live ? qx[T.pt0 + pi] : 0.0, y = live ? qy[T.pt0 + pi] : 0.0;
    const double k = T.k, ik = 1.0 / k, u_k = 64.0 * ik * ik, k4 = 0.25 * k;
    const double thr = 1e-13 * (1.0 + sqrt(x * x + y * y));
    cplx acc{0, 0};
    if (live) {
        // interface potentials, three shifts each, phase alpha^l
        for (int q = 0; q < T.nsrc; ++q) {
            const int n = T.ns[q];
            const cplx* tau = T.tau[q];
            const cplx* sig = tau + n;
            for (int j = warp; j < n; j += kFieldWarps) {
                const int g = T.s_off[q] + j;
                const double zx0 = pool.x[g], zy = pool.y[g], znx = pool.nx[g], zny = pool.ny[g], w = pool.w[g];
                const cplx tj = tau[j], sj = sig[j];
                cplx part{0, 0};
#pragma unroll
                for (int l = -1; l <= 1; ++l) {
                    const double rvx = x - (zx0 + l * d), rvy = y - zy;
                    const double r2 = rvx * rvx + rvy * rvy;
                    const double inv_r = rsqrt(r2);
                    const double r = r2 * inv_r;
                    if (r < thr) {
                        atomicOr(err, 1);
                        continue;
                    }
                    HankelOut h;
                    hankel01_dev(k * r, inv_r * ik, inv_r * inv_r * u_k, s_near2, h);
                    const double cdn = (rvx * znx + rvy * zny) * inv_r;
                    // S = (i/4) H0, D = (ik/4) H1 cdn
                    const cplx S{-0.25 * h.y0, 0.25 * h.j0};
                    const cplx D{-k4 * h.y1 * cdn, k4 * h.j1 * cdn};
                    cplx v{D.re * tj.re - D.im * tj.im + S.re * sj.re - S.im * sj.im,
                           D.re * tj.im + D.im * tj.re + S.re * sj.im + S.im * sj.re};
                    const cplx ph = l < 0 ? alpha_inv : (l > 0 ? alpha : cplx{1.0, 0.0});
                    part.re += ph.re * v.re - ph.im * v.im;
                    part.im += ph.re * v.im + ph.im * v.re;
                }
                acc.re += w * part.re;
                acc.im += w * part.im;
            }
        }
        // proxy expansion: phi_p = D + i k S with the proxy normal
        for (int p = warp; p < T.P; p += kFieldWarps) {
            const int g = T.p_off + p;
            const double rvx = x - pool.x[g], rvy = y - pool.y[g];
            const double r2 = rvx * rvx + rvy * rvy;
            const double inv_r = rsqrt(r2);
            const double r = r2 * inv_r;
            if (r < thr) {
                atomicOr(err, 1);
                continue;
            }
            HankelOut h;
            hankel01_dev(k * r, inv_r * ik, inv_r * inv_r * u_k, s_near2, h);
            const double cdn = (rvx * pool.nx[g] + rvy * pool.ny[g]) * inv_r;
            const cplx S{-0.25 * h.y0, 0.25 * h.j0};
            const cplx D{-k4 * h.y1 * cdn, k4 * h.j1 * cdn};
            const cplx phi{D.re - k * S.im, D.im + k * S.re};
            const cplx cp = T.c[p];
            acc.re += phi.re * cp.re - phi.im * cp.im;
            acc.im += phi.re * cp.im + phi.im * cp.re;
        }
    }
    s_acc[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && live) {
        cplx s = s_acc[0][lane];
        for (int w2 = 1; w2 < kFieldWarps; ++w2) {
            s.re += s_acc[w2][lane].re;
            s.im += s_acc[w2][lane].im;
        }
        out[T.pt0 + pi] = s;
    }
}

}  // namespace

void field_sums(Ctx& c, const std::vector<FieldTask>& tasks, const std::vector<int2>& tiles,
                const std::vector<double>& qx, const std::vector<double>& qy, const DevPool& pool,
                std::vector<cplx>& out) {
    const Problem& pb = c.prob;
    const std::complex<double> alpha(pb.ar, pb.ai), ainv = 1.0 / alpha;
    cudaStream_t s = c.stream;
    {  // this translation unit's copy of the far-field Hankel table (hankel.cuh)
        static bool uploaded = false;
        if (!uploaded) {
            QPS_CUDA(cudaMemcpyToSymbol(c_hankel_far, qps_hankel_far_coeffs, sizeof(qps_hankel_far_coeffs)));
            uploaded = true;
        }
    }
    const int n = int(qx.size());
    out.assign(n, cplx{0, 0});
    if (n == 0 || tiles.empty()) return;
    c.field_qx.upload(qx, s);
    c.field_qy.upload(qy, s);
    c.field_tasks.upload(tasks, s);
    c.field_tiles.upload(tiles, s);
    c.field_out.ensure(n);
    QPS_CUDA(cudaMemsetAsync(c.d_err.p, 0, sizeof(int), s));
    double evals = 0;
    for (const auto& t : tasks) {
        double per = t.P;
        for (int q = 0; q < t.nsrc; ++q) per += 3.0 * t.ns[q];
        evals += per * t.npt;
    }
    {
        ProfScope ps("field", s, 0.0, 0.0, evals);
        { QPS_NOTE_LAUNCH(); field_kernel<<<unsigned(tiles.size()), 32 * kFieldWarps, 0, s>>>(
            c.field_tasks.p, c.field_tiles.p, c.field_qx.p, c.field_qy.p, pool, device_near_table(),
            cplx{alpha.real(), alpha.imag()}, cplx{ainv.real(), ainv.imag()}, c.geo.d, c.field_out.p, c.d_err.p); }
        QPS_CUDA(cudaGetLastError());
    }
    int herr = 0;
    QPS_D2H(out.data(), c.field_out.p, sizeof(cplx) * n, s);
    QPS_D2H(&herr, c.d_err.p, sizeof(int), s);
    QPS_CUDA(cudaStreamSynchronize(s));
    if (herr) fail(QPS_ERR_SINGULARITY, "kernel evaluated at coincident target/source pair");
}

void evaluate_field(Ctx& c, int n, const double* xy, cplx* u_scat, cplx* u_tot, int* region, int* layer_out) {
    const HostGeometry& g = c.geo;
    const Problem& pb = c.prob;
    const Dims& D = c.dims;
    const double d = g.d;
    const int I = g.I;
    const cd alpha(pb.ar, pb.ai);
    cudaStream_t s = c.stream;
    // classification in the central cell (postprocess.hpp:85-95)
    std::vector<int> cell(n), reg(n), lay(n);
    for (int i = 0; i < n; ++i) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        const int m = int(std::floor((x + 0.5 * d) / d));
        cell[i] = m;
        reg[i] = classify_point(c.stack, g, x - m * d, y, &lay[i]);
    }
    // layer points sorted by layer
    std::vector<int> order;
    std::vector<int> start(I + 2, 0);
    for (int i = 0; i < n; ++i)
        if (reg[i] == 1) ++start[lay[i] + 1];
    for (int l = 0; l <= I; ++l) start[l + 1] += start[l];
    order.assign(start[I + 1], 0);
    {
        std::vector<int> fillp(start.begin(), start.end() - 1);
        for (int i = 0; i < n; ++i)
            if (reg[i] == 1) order[fillp[lay[i]]++] = i;
    }
    const int nl = int(order.size());
    std::vector<cplx> u_layer(nl);
    if (nl > 0) {
        std::vector<double> qx(nl), qy(nl);
        for (int t = 0; t < nl; ++t) {
            const int i = order[t];
            qx[t] = xy[2 * i] - cell[i] * d;
            qy[t] = xy[2 * i + 1];
        }
        // proxy coefficients of every layer (corners come from the host solution)
        c.field_c.upload(c.h_c, s);
        std::vector<FieldTask> tasks;
        std::vector<int2> tiles;
        for (int l = 0; l <= I; ++l) {
            const int cnt = start[l + 1] - start[l];
            if (cnt == 0) continue;
            FieldTask t{};
            t.k = pb.k[l];
            for (int which = 0; which < 2; ++which) {
                const int j = l - 1 + which;  // interface above (l-1) and below (l)
                if (j < 0 || j >= I) continue;
                t.s_off[t.nsrc] = c.iface_off[j];
                t.ns[t.nsrc] = D.N[j];
                t.tau[t.nsrc] = c.F.p + size_t(j) * D.nb;
                ++t.nsrc;
            }
            t.p_off = c.proxy_off[l];
            t.P = D.P;
            t.c = c.field_c.p + size_t(l) * D.P;
            t.pt0 = start[l];
            t.npt = cnt;
            const int ti = int(tasks.size());
            tasks.push_back(t);
            for (int p0 = 0; p0 < cnt; p0 += kFieldPts) tiles.push_back(make_int2(ti, p0));
        }
        const DevPool pool{c.px.p, c.py.p, c.pnx.p, c.pny.p, c.pw.p};
        field_sums(c, tasks, tiles, qx, qy, pool, u_layer);
    }
    std::vector<cd> us(n, cd(0.0, 0.0));
    for (int t = 0; t < nl; ++t) {
        const int i = order[t];
        us[i] = std::pow(alpha, cell[i]) * cd(u_layer[t].re, u_layer[t].im);
    }
    // Rayleigh-Bloch sums above / below (rb_sum, postprocess.hpp:65-76) and the
    // incident wave in the top layer (postprocess.hpp:113-121)
    const cd iu(0.0, 1.0);
    const double kx = pb.k.front() * std::cos(pb.theta), ky = pb.k.front() * std::sin(pb.theta);
    for (int i = 0; i < n; ++i) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        if (reg[i] != 1) {
            const bool upper = reg[i] == 0;
            cd u = 0.0;
            for (int m = -pb.K; m <= pb.K; ++m) {
                const cplx a = upper ? c.h_aU[m + pb.K] : c.h_aD[m + pb.K];
                const double kap = pb.kappa(m, d);
                const double kl = upper ? pb.k.front() : pb.k.back();
                const double t2 = kl * kl - kap * kap;
                const cd kv = t2 >= 0.0 ? cd(std::sqrt(t2), 0.0) : cd(0.0, std::sqrt(-t2));
                const double dy = upper ? y - g.y_U : g.y_D - y;
                u += cd(a.re, a.im) * std::exp(iu * kap * x) * std::exp(iu * kv * dy);
            }
            us[i] = u;
        }
        cd ut = us[i];
        if (reg[i] == 0 || (reg[i] == 1 && lay[i] == 0)) ut += std::exp(iu * (kx * x + ky * y));
        if (u_scat) u_scat[i] = cplx{us[i].real(), us[i].imag()};
        if (u_tot) u_tot[i] = cplx{ut.real(), ut.imag()};
        if (region) region[i] = reg[i];
        if (layer_out) layer_out[i] = lay[i];
    }
}

}  // namespace qpsb
