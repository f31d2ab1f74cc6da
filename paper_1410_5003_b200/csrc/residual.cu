// Post-solve residual suite: residual_suite / interface_matching_residual /
// ResidualReport (postprocess.hpp:186-399), the reference's a-posteriori
// accuracy certificate of a solution.
//
//   wall_qp    max |alpha^{-1} u(d/2, y) - u(-d/2, y)| at three heights of the
//              walls of layers 0, I/2, I (quasi-periodicity of the layer
//              representation, postprocess.hpp:375-383)
//   radiation  max |representation - Rayleigh-Bloch sum| at three points of
//              the U and D lines (postprocess.hpp:385-393)
//   interface  max over the probed interfaces of the one-sided value and
//              normal-derivative mismatch of the total field, extrapolated
//              to off-node interface points from both layers through a 4x
//              upsampled density (postprocess.hpp:263-365)
//
// Every potential is summed on the device by the field kernel (field.cu: the
// alpha-phased D/S potentials of the bounding interfaces, l = -1, 0, 1, plus
// the proxy expansion, one Hankel pair per source and shift), from a private
// source pool holding the coarse interfaces, the 4x refined interface and the
// proxies a call needs.  The host does what is O(N) per probe: the refined
// quadrature (geometry.hpp:423-447 with 4x the nodes), the density upsampling
// (trigonometric for periodic interfaces, order-12 Lagrange per segment on
// graded ones), the degree-8 least-squares fits of 10 standoff samples and
// their extrapolation to the interface, and the Rayleigh-Bloch sums.
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>

#include "ctx.h"
#include "prof.h"

namespace qpsb {

namespace {

using cd = std::complex<double>;
const cd iu(0.0, 1.0);

// A set of source point arrays assembled on the host and uploaded as one pool.
struct PoolBuilder {
    std::vector<double> x, y, nx, ny, w;
    int add_interface(const HostInterface& q) {
        const int off = int(x.size());
        x.insert(x.end(), q.x.begin(), q.x.end());
        y.insert(y.end(), q.y.begin(), q.y.end());
        nx.insert(nx.end(), q.nx.begin(), q.nx.end());
        ny.insert(ny.end(), q.ny.begin(), q.ny.end());
        w.insert(w.end(), q.w.begin(), q.w.end());
        return off;
    }
    int add_proxies(const HostGeometry& g, int layer) {
        const int off = int(x.size());
        x.insert(x.end(), g.px[layer].begin(), g.px[layer].end());
        y.insert(y.end(), g.py[layer].begin(), g.py[layer].end());
        nx.insert(nx.end(), g.pnx[layer].begin(), g.pnx[layer].end());
        ny.insert(ny.end(), g.pny[layer].begin(), g.pny[layer].end());
        w.insert(w.end(), g.px[layer].size(), 0.0);
        return off;
    }
};

// Layer representation (eval_layer_representation, postprocess.hpp:46-63) at
// points given with their layer; optionally interface `fine_j` replaced by a
// refined quadrature `fine` carrying the density `eta_fine` ([tau; sigma]).
std::vector<cd> layer_sums(Ctx& c, const std::vector<int>& layer, const std::vector<double>& px,
                           const std::vector<double>& py, int fine_j = -1, const HostInterface* fine = nullptr,
                           const std::vector<cplx>* eta_fine = nullptr) {
    const HostGeometry& g = c.geo;
    const Dims& D = c.dims;
    const int I = g.I, n = int(px.size());
    cudaStream_t s = c.stream;
    // points grouped by layer
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return layer[a] < layer[b]; });
    PoolBuilder pb;
    std::vector<int> ioff(I, -1), poff(I + 1, -1);
    int fine_off = -1;
    c.res_eta.ensure(eta_fine ? eta_fine->size() : 1);
    if (eta_fine) c.res_eta.upload(*eta_fine, s);
    c.field_c.upload(c.h_c, s);
    std::vector<FieldTask> tasks;
    std::vector<int2> tiles;
    std::vector<double> qx(n), qy(n);
    for (int t = 0; t < n; ++t) {
        qx[t] = px[order[t]];
        qy[t] = py[order[t]];
    }
    for (int t0 = 0; t0 < n;) {
        const int l = layer[order[t0]];
        int t1 = t0;
        while (t1 < n && layer[order[t1]] == l) ++t1;
        FieldTask t{};
        t.k = c.prob.k[l];
        for (int which = 0; which < 2; ++which) {
            const int j = l - 1 + which;
            if (j < 0 || j >= I) continue;
            if (j == fine_j) {
                if (fine_off < 0) fine_off = pb.add_interface(*fine);
                t.s_off[t.nsrc] = fine_off;
                t.ns[t.nsrc] = fine->N();
                t.tau[t.nsrc] = c.res_eta.p;
            } else {
                if (ioff[j] < 0) ioff[j] = pb.add_interface(g.ifaces[j]);
                t.s_off[t.nsrc] = ioff[j];
                t.ns[t.nsrc] = D.N[j];
                t.tau[t.nsrc] = c.F.p + size_t(j) * D.nb;
            }
            ++t.nsrc;
        }
        if (poff[l] < 0) poff[l] = pb.add_proxies(g, l);
        t.p_off = poff[l];
        t.P = D.P;
        t.c = c.field_c.p + size_t(l) * D.P;
        t.pt0 = t0;
        t.npt = t1 - t0;
        const int ti = int(tasks.size());
        tasks.push_back(t);
        for (int p0 = 0; p0 < t.npt; p0 += kFieldTile) tiles.push_back(make_int2(ti, p0));
        t0 = t1;
    }
    c.res_px.upload(pb.x, s);
    c.res_py.upload(pb.y, s);
    c.res_pnx.upload(pb.nx, s);
    c.res_pny.upload(pb.ny, s);
    c.res_pw.upload(pb.w, s);
    const DevPool pool{c.res_px.p, c.res_py.p, c.res_pnx.p, c.res_pny.p, c.res_pw.p};
    std::vector<cplx> raw;
    field_sums(c, tasks, tiles, qx, qy, pool, raw);
    std::vector<cd> out(n);
    for (int t = 0; t < n; ++t) out[order[t]] = cd(raw[t].re, raw[t].im);
    return out;
}

cd rb_sum(const Ctx& c, double x, double y, bool upper) {  // postprocess.hpp:65-76
    const Problem& p = c.prob;
    const HostGeometry& g = c.geo;
    cd u = 0.0;
    for (int m = -p.K; m <= p.K; ++m) {
        const cplx a = upper ? c.h_aU[m + p.K] : c.h_aD[m + p.K];
        const double kap = p.kappa(m, g.d);
        const double kl = upper ? p.k.front() : p.k.back();
        const double t2 = kl * kl - kap * kap;
        const cd kv = t2 >= 0.0 ? cd(std::sqrt(t2), 0.0) : cd(0.0, std::sqrt(-t2));
        const double dy = upper ? y - g.y_U : g.y_D - y;
        u += cd(a.re, a.im) * std::exp(iu * kap * x) * std::exp(iu * kv * dy);
    }
    return u;
}

// detail::upsample_smooth (postprocess.hpp:200-233): trigonometric upsampling of
// the quasi-periodic density psi_j e^{i w s_j / 2pi}
std::vector<cd> upsample_smooth(const std::vector<cd>& vals, double w, int fine) {
    const int N = int(vals.size()), NF = fine * N;
    std::vector<cd> psi(N), coef(N), out(NF);
    for (int j = 0; j < N; ++j) {
        const double s = 2.0 * kPi * (j + 0.5) / N;
        psi[j] = vals[j] * std::exp(-iu * w * s / (2.0 * kPi));
    }
    for (int m = 0; m < N; ++m) {
        const int mm = m <= N / 2 ? m : m - N;
        cd acc = 0.0;
        for (int j = 0; j < N; ++j) {
            const double s = 2.0 * kPi * (j + 0.5) / N;
            acc += psi[j] * std::exp(-iu * double(mm) * s);
        }
        coef[m] = acc / double(N);
    }
    for (int j = 0; j < NF; ++j) {
        const double s = 2.0 * kPi * (j + 0.5) / NF;
        cd acc = 0.0;
        for (int m = 0; m < N; ++m) {
            const int mm = m <= N / 2 ? m : m - N;
            acc += coef[m] * std::exp(iu * double(mm) * s);
        }
        out[j] = acc * std::exp(iu * w * s / (2.0 * kPi));
    }
    return out;
}

// detail::upsample_segmented (postprocess.hpp:236-258): order-12 Lagrange per
// segment, stencil clamped inside the segment
std::vector<cd> upsample_segmented(const std::vector<cd>& vals, const HostInterface& q, int fine) {
    constexpr int ord = 12;
    std::vector<cd> out(size_t(fine) * q.N());
    int fine_off = 0;
    for (const SegDesc& seg : q.segs) {
        const int n = seg.n, nf = fine * n;
        for (int j = 0; j < nf; ++j) {
            const double sx = (j + 0.5) / fine - 0.5;
            const int t0 = std::clamp(int(std::floor(sx)) - ord / 2 + 1, 0, n - ord);
            cd acc = 0.0;
            for (int r = 0; r < ord; ++r) {
                double L = 1.0;
                for (int qq = 0; qq < ord; ++qq) {
                    if (qq == r) continue;
                    L *= (sx - (t0 + qq)) / double(r - qq);
                }
                acc += L * vals[seg.offset + t0 + r];
            }
            out[fine_off + j] = acc;
        }
        fine_off += nf;
    }
    return out;
}

// least-squares solve of V c = b (V m x p real, full column rank) by Householder
// QR, the LAPACK/Eigen HouseholderQR::solve sequence: Q^T b, then R^{-1}
template <int M, int P>
std::array<cd, P> lsq_solve(std::array<std::array<double, P>, M> V, std::array<cd, M> b) {
    for (int k = 0; k < P; ++k) {
        double nrm = 0;
        for (int i = k; i < M; ++i) nrm += V[i][k] * V[i][k];
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) continue;
        const double alpha = V[k][k] > 0 ? -nrm : nrm;
        std::array<double, M> v{};
        for (int i = k; i < M; ++i) v[i] = V[i][k];
        v[k] -= alpha;
        double vn = 0;
        for (int i = k; i < M; ++i) vn += v[i] * v[i];
        if (vn == 0.0) continue;
        for (int j = k; j < P; ++j) {
            double dot = 0;
            for (int i = k; i < M; ++i) dot += v[i] * V[i][j];
            const double f = 2.0 * dot / vn;
            for (int i = k; i < M; ++i) V[i][j] -= f * v[i];
        }
        cd dot = 0;
        for (int i = k; i < M; ++i) dot += v[i] * b[i];
        const cd f = 2.0 * dot / vn;
        for (int i = k; i < M; ++i) b[i] -= f * v[i];
    }
    std::array<cd, P> x{};
    for (int k = P - 1; k >= 0; --k) {
        cd acc = b[k];
        for (int j = k + 1; j < P; ++j) acc -= V[k][j] * x[j];
        x[k] = acc / V[k][k];
    }
    return x;
}

}  // namespace

double interface_matching_residual(Ctx& c, int j, int n_probe) {
    const HostGeometry& g = c.geo;
    const Problem& p = c.prob;
    const Dims& D = c.dims;
    const int I = g.I;
    if (j < 0 || j >= I) fail(QPS_ERR_USAGE, "interface_matching_residual: interface index out of range");
    if (n_probe < 1) fail(QPS_ERR_USAGE, "interface_matching_residual: n_probe >= 1");
    // the 4x refined quadrature of interface j (build_interface_geometry with
    // every segment's node count times 4)
    qps_interface_spec fs = c.stack.ifaces[j];
    std::vector<int> nodes4(fs.nodes, fs.nodes + fs.n_nodes);
    for (int& v : nodes4) v *= 4;
    fs.nodes = nodes4.data();
    const HostInterface fq = build_interface_geometry(fs, g.d);
    const HostInterface& cq = g.ifaces[j];
    const int nc = cq.N();
    // the solved density of interface j (system 0) from the pinned host copy
    size_t off = 0;
    for (int q = 0; q < j; ++q) off += 2 * size_t(D.N[q]);
    std::vector<cd> tau(nc), sig(nc);
    for (int i = 0; i < nc; ++i) {
        tau[i] = cd(c.h_eta[off + i].re, c.h_eta[off + i].im);
        sig[i] = cd(c.h_eta[off + nc + i].re, c.h_eta[off + nc + i].im);
    }
    const double w = g.d * p.k.front() * std::cos(p.theta);
    std::vector<cd> tf, sf;
    if (cq.smooth) {
        tf = upsample_smooth(tau, w, 4);
        sf = upsample_smooth(sig, w, 4);
    } else {
        tf = upsample_segmented(tau, cq, 4);
        sf = upsample_segmented(sig, cq, 4);
    }
    const int nf = fq.N();
    std::vector<cplx> eta_f(2 * size_t(nf));
    for (int i = 0; i < nf; ++i) {
        eta_f[i] = cplx{tf[i].real(), tf[i].imag()};
        eta_f[nf + i] = cplx{sf[i].real(), sf[i].imag()};
    }
    const double h_phys = g.d / nc;  // InterfaceQuadrature::period / total
    constexpr int n_fit = 10, deg = 8;
    std::array<double, n_fit> ds{};
    for (int q = 0; q < n_fit; ++q) ds[q] = h_phys * (2.3 + std::cos(kPi * (q + 0.5) / n_fit));
    // every probe's 2 x 10 standoff points in one device evaluation
    std::vector<int> lay;
    std::vector<double> px, py;
    std::vector<int> probe_m(n_probe);
    for (int t = 0; t < n_probe; ++t) {
        const int m = int((0.2 + 0.6 * t / std::max(1, n_probe - 1)) * nf) | 1;
        probe_m[t] = m;
        const double zx = fq.x[m], zy = fq.y[m], nx = fq.nx[m], ny = fq.ny[m];
        for (int q = 0; q < n_fit; ++q) {
            lay.push_back(j);  // above: opposite the (downward) normal
            px.push_back(zx - nx * ds[q]);
            py.push_back(zy - ny * ds[q]);
            lay.push_back(j + 1);
            px.push_back(zx + nx * ds[q]);
            py.push_back(zy + ny * ds[q]);
        }
    }
    const std::vector<cd> u = layer_sums(c, lay, px, py, j, &fq, &eta_f);
    const double kx = p.k.front() * std::cos(p.theta), ky = p.k.front() * std::sin(p.theta);
    std::array<std::array<double, deg + 1>, n_fit> V{};
    for (int q = 0; q < n_fit; ++q) {
        const double x = ds[q] / h_phys - 2.3;
        for (int cc = 0; cc <= deg; ++cc) V[q][cc] = std::pow(x, cc);
    }
    auto horner = [&](const std::array<cd, deg + 1>& cf, double x, bool deriv) {
        cd acc = 0.0;
        if (!deriv) {
            for (int q = deg; q >= 0; --q) acc = acc * x + cf[q];
        } else {
            for (int q = deg; q >= 1; --q) acc = acc * x + double(q) * cf[q];
        }
        return acc;
    };
    double worst = 0.0;
    for (int t = 0; t < n_probe; ++t) {
        std::array<cd, n_fit> ua{}, ub{};
        for (int q = 0; q < n_fit; ++q) {
            ua[q] = u[size_t(t) * 2 * n_fit + 2 * q];
            ub[q] = u[size_t(t) * 2 * n_fit + 2 * q + 1];
        }
        const auto ca = lsq_solve<n_fit, deg + 1>(V, ua), cb = lsq_solve<n_fit, deg + 1>(V, ub);
        const double x0 = -2.3;
        const cd u_above = horner(ca, x0, false), u_below = horner(cb, x0, false);
        const cd dn_above = -horner(ca, x0, true) / h_phys, dn_below = horner(cb, x0, true) / h_phys;
        cd rv = u_above - u_below, rd = dn_above - dn_below;
        if (j == 0) {
            const int m = probe_m[t];
            const cd e = std::exp(iu * (kx * fq.x[m] + ky * fq.y[m]));
            rv += e;
            rd += iu * (kx * fq.nx[m] + ky * fq.ny[m]) * e;
        }
        worst = std::max({worst, std::abs(rv), std::abs(rd) / p.k[j]});
    }
    return worst;
}

void residual_suite(Ctx& c, const std::vector<int>& ifaces, double* wall_qp, double* radiation, double* iface) {
    const HostGeometry& g = c.geo;
    const Problem& p = c.prob;
    const int I = g.I;
    const double d = g.d;
    const cd alpha(p.ar, p.ai);
    std::vector<int> lay;
    std::vector<double> px, py;
    for (int layer : {0, I / 2, I})
        for (double f : {0.35, 0.5, 0.71}) {
            const double y = g.wall_lo[layer] + f * (g.wall_hi[layer] - g.wall_lo[layer]);
            for (double x : {0.5 * d, -0.5 * d}) {
                lay.push_back(layer);
                px.push_back(x);
                py.push_back(y);
            }
        }
    const int nwall = int(px.size());
    for (bool upper : {true, false})
        for (double x : {-0.37 * d, 0.021 * d, 0.44 * d}) {
            lay.push_back(upper ? 0 : I);
            px.push_back(x);
            py.push_back(upper ? g.y_U : g.y_D);
        }
    const std::vector<cd> u = layer_sums(c, lay, px, py);
    double wq = 0.0, rad = 0.0;
    for (int i = 0; i < nwall; i += 2) wq = std::max(wq, std::abs(u[i] / alpha - u[i + 1]));
    for (int i = nwall; i < int(px.size()); ++i) rad = std::max(rad, std::abs(u[i] - rb_sum(c, px[i], py[i], lay[i] == 0)));
    double ir = 0.0;
    for (int j : ifaces) ir = std::max(ir, interface_matching_residual(c, j, 4));
    if (wall_qp) *wall_qp = wq;
    if (radiation) *radiation = rad;
    if (iface) *iface = ir;
}

}  // namespace qpsb
