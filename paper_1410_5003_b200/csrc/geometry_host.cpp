// Host-side geometry and problem setup — a from-scratch restatement of the
// reference's discretisation so that node coordinates match it exactly
// (same formulas, same operation order):
//   build_smooth_quadrature   geometry.hpp:114-144
//   build_corner_quadrature   geometry.hpp:149-200 (Kress grading :37-65)
//   make_interface_segments   geometry.hpp:333-393
//   build_interface_geometry  geometry.hpp:423-447
//   build_frame               geometry.hpp:449-478 (Gauss-Legendre :229-251)
//   build_geometry            geometry.hpp:480-496 (proxy circles :213-226)
//   make_problem / choose_rb_order  assembly.hpp:43-82
// The Alpert auxiliary nodes are NOT built here: the segment descriptors
// (SegDesc) travel to the device, which evaluates them in the fill.
#include <algorithm>
#include <cmath>
#include <complex>
#include <exception>
#include <limits>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "alpert_table.h"
#include "qps_internal.h"

namespace qpsb {

namespace {

constexpr double pi = kPi;

struct V2 {
    double x, y;
};
inline double norm2(V2 v) { return std::hypot(v.x, v.y); }

double kress_v(double s, int q) {
    const double u = (pi - s) / pi;
    return (1.0 / q - 0.5) * u * u * u + (s - pi) / (pi * q) + 0.5;
}
double kress_vp(double s, int q) {
    const double u = (pi - s) / pi;
    return -3.0 * (1.0 / q - 0.5) * u * u / pi + 1.0 / (pi * q);
}
double kress_w(double s, int q) {
    if (s < 0.0 || s > 2.0 * pi) fail(QPS_ERR_DOMAIN, "kress_w: s outside [0, 2pi]");
    if (q < 2) fail(QPS_ERR_DOMAIN, "kress_w: q must be >= 2");
    const double vq = std::pow(kress_v(s, q), q);
    const double vr = std::pow(kress_v(2.0 * pi - s, q), q);
    return 2.0 * pi * vq / (vq + vr);
}
double kress_wp(double s, int q) {
    const double v1 = kress_v(s, q), v2 = kress_v(2.0 * pi - s, q);
    const double vq = std::pow(v1, q), vr = std::pow(v2, q);
    const double d1 = q * std::pow(v1, q - 1) * kress_vp(s, q);
    const double d2 = -q * std::pow(v2, q - 1) * kress_vp(2.0 * pi - s, q);
    const double den = vq + vr;
    return 2.0 * pi * (d1 * den - vq * (d1 + d2)) / (den * den);
}

// --- periodic smooth parametrisation (make_interface_segments, :359-390) ---
V2 smooth_Z(const qps_interface_spec& sp, double d, double s) {
    const double x = -0.5 * d + d * s / (2.0 * pi);
    double y = sp.offset;
    if (sp.shape == QPS_SHAPE_SINE) {
        y += sp.amplitude * std::sin(2.0 * pi * x / d + sp.phase);
    } else {
        for (int m = 0; m < sp.n_cos; ++m) y += sp.cosc[m] * std::cos(2.0 * pi * double(m + 1) * x / d);
        for (int m = 0; m < sp.n_sin; ++m) y += sp.sinc[m] * std::sin(2.0 * pi * double(m + 1) * x / d);
    }
    return {x, y};
}
V2 smooth_Zp(const qps_interface_spec& sp, double d, double s) {
    const double x = -0.5 * d + d * s / (2.0 * pi);
    const double dxds = d / (2.0 * pi);
    double dydx = 0.0;
    if (sp.shape == QPS_SHAPE_SINE) {
        dydx = sp.amplitude * (2.0 * pi / d) * std::cos(2.0 * pi * x / d + sp.phase);
    } else {
        for (int m = 0; m < sp.n_cos; ++m)
            dydx -= sp.cosc[m] * (2.0 * pi * double(m + 1) / d) * std::sin(2.0 * pi * double(m + 1) * x / d);
        for (int m = 0; m < sp.n_sin; ++m)
            dydx += sp.sinc[m] * (2.0 * pi * double(m + 1) / d) * std::cos(2.0 * pi * double(m + 1) * x / d);
    }
    return {dxds, dydx * dxds};
}

// spec_y_of_x, geometry.hpp:300-328
double spec_y_of_x(const qps_interface_spec& sp, double d, double x) {
    x -= d * std::floor((x + 0.5 * d) / d);
    switch (sp.shape) {
        case QPS_SHAPE_SINE:
            return sp.offset + sp.amplitude * std::sin(2.0 * pi * x / d + sp.phase);
        case QPS_SHAPE_FOURIER: {
            double y = sp.offset;
            for (int m = 0; m < sp.n_cos; ++m) y += sp.cosc[m] * std::cos(2.0 * pi * double(m + 1) * x / d);
            for (int m = 0; m < sp.n_sin; ++m) y += sp.sinc[m] * std::sin(2.0 * pi * double(m + 1) * x / d);
            return y;
        }
        default: {
            const double* v = sp.vertices;
            const int nv = sp.n_vertices;
            for (int l = 0; l + 1 < nv; ++l) {
                const double x0 = v[2 * l], y0 = v[2 * l + 1], x1 = v[2 * l + 2], y1 = v[2 * l + 3];
                if (x >= x0 && x <= x1) {
                    if (x1 - x0 < 1e-14) return sp.offset + std::max(y0, y1);
                    const double f = (x - x0) / (x1 - x0);
                    return sp.offset + y0 * (1.0 - f) + y1 * f;
                }
            }
            return sp.offset + v[2 * (nv - 1) + 1];
        }
    }
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    x.resize(n);
    w.resize(n);
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double t = std::cos(pi * (i + 0.75) / (n + 0.5));
        double pp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = 0.0;
            for (int k = 0; k < n; ++k) {
                const double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * k + 1.0) * t * p1 - k * p2) / (k + 1.0);
            }
            pp = n * (t * p0 - p1) / (t * t - 1.0);
            const double dt = -p0 / pp;
            t += dt;
            if (std::abs(dt) < 1e-15) break;
        }
        x[i] = -t;
        x[n - 1 - i] = t;
        w[i] = w[n - 1 - i] = 2.0 / ((1.0 - t * t) * pp * pp);
    }
}

void push_node(HostInterface& q, V2 z, V2 t_for_speed, V2 t_for_normal, double h) {
    q.x.push_back(z.x);
    q.y.push_back(z.y);
    const double sp = norm2(t_for_speed);
    q.speed.push_back(sp);
    q.w.push_back(h * sp);
    const double nn = norm2(t_for_normal);
    q.nx.push_back(t_for_normal.y / nn);
    q.ny.push_back(-t_for_normal.x / nn);
}

HostInterface build_interface(const qps_interface_spec& sp, double d, std::vector<double>& pool) {
    HostInterface g;
    {  // one allocation per array (the interfaces are built on concurrent host threads)
        size_t n = 0;
        for (int i = 0; i < sp.n_nodes; ++i) n += size_t(std::max(0, sp.nodes[i]));
        if (sp.shape != QPS_SHAPE_POLYLINE) n = sp.n_nodes > 0 ? size_t(std::max(0, sp.nodes[0])) : 70;
        if (sp.shape == QPS_SHAPE_POLYLINE && sp.n_nodes == 1) n *= size_t(std::max(1, sp.n_vertices - 1));
        for (auto* v : {&g.x, &g.y, &g.nx, &g.ny, &g.w, &g.speed}) v->reserve(n);
    }
    if (sp.shape == QPS_SHAPE_POLYLINE) {
        // make_interface_segments (:335-357) + build_corner_quadrature (:149-200)
        const int nv = sp.n_vertices;
        const double* v = sp.vertices;
        if (nv < 2) fail(QPS_ERR_CONFIG, "polyline interface needs >= 2 vertices");
        if (std::abs(v[0] + 0.5 * d) > 1e-12 || std::abs(v[2 * (nv - 1)] - 0.5 * d) > 1e-12)
            fail(QPS_ERR_CONFIG, "polyline must span x = -d/2 .. d/2");
        if (std::abs(v[1] - v[2 * (nv - 1) + 1]) > 1e-12)
            fail(QPS_ERR_CONFIG, "polyline endpoint heights must match (periodicity)");
        const int nseg = nv - 1;
        std::vector<int> npers(sp.nodes, sp.nodes + sp.n_nodes);
        if (npers.size() == 1) npers.assign(nseg, npers[0]);
        if (int(npers.size()) != nseg) fail(QPS_ERR_CONFIG, "interface node counts do not match segment count");
        // endpoint continuity checks hold by construction for polylines
        int offset = 0;
        for (int l = 0; l < nseg; ++l) {
            const V2 A{v[2 * l], v[2 * l + 1] + sp.offset};
            const V2 B{v[2 * l + 2], v[2 * l + 3] + sp.offset};
            const int n = npers[l];
            if (n < 8) fail(QPS_ERR_CONFIG, "build_corner_quadrature: n per segment must be >= 8");
            const int gq = sp.grading_q;  // build_interface_geometry passes sp.grading_q (> 0)
            const double h = 2.0 * pi / n;
            const V2 rawp{(B.x - A.x) / (2.0 * pi), (B.y - A.y) / (2.0 * pi)};
            for (int j = 0; j < n; ++j) {
                const double s = (j + 0.5) * h;
                const double wv = kress_w(s, gq);
                const double f = wv / (2.0 * pi);
                const V2 z{A.x + (B.x - A.x) * f, A.y + (B.y - A.y) * f};
                const double wp = kress_wp(s, gq);
                const V2 t{rawp.x * wp, rawp.y * wp};
                push_node(g, z, t, rawp, h);
            }
            // auxiliary Alpert nodes of this segment's rows (kernels.hpp:243-253 with
            // the QuadSegment maps of geometry.hpp:171-177 and the line segment
            // of geometry.hpp:345-353); rows the reference fills with the plain
            // rule (within a of a segment end, kernels.hpp:224) stay zero
            for (int j = 0; j < n; ++j) {
                for (int side = -1; side <= 1; side += 2)
                    for (int kk = 0; kk < QPS_ALPERT_NAUX; ++kk) {
                        double e[5] = {0, 0, 0, 0, 0};
                        if (std::min(j, n - 1 - j) >= QPS_ALPERT_A) {
                            const double xi = side * qps_alpert_nodes[kk];
                            const double s_aux = (j + 0.5 + xi) * h;
                            const double f = kress_w(s_aux, gq) / (2.0 * pi);
                            const V2 z{A.x + (B.x - A.x) * f, A.y + (B.y - A.y) * f};
                            const double wp = kress_wp(s_aux, gq);
                            const V2 t{rawp.x * wp, rawp.y * wp};
                            const double sp_ = std::hypot(t.x, t.y);
                            e[0] = z.x;
                            e[1] = z.y;
                            e[2] = t.y / sp_;
                            e[3] = -t.x / sp_;
                            e[4] = h * qps_alpert_weights[kk] * sp_;
                        }
                        g.aux.insert(g.aux.end(), e, e + 5);
                    }
            }
            SegDesc sd{};
            sd.kind = SEG_LINE;
            sd.n = n;
            sd.offset = offset;
            sd.periodic = 0;
            sd.q = gq;
            sd.d = d;
            sd.Ax = A.x;
            sd.Ay = A.y;
            sd.Bx = B.x;
            sd.By = B.y;
            g.segs.push_back(sd);
            offset += n;
        }
        g.smooth = false;
    } else {
        // build_smooth_quadrature (:114-144); normalize_direction is the identity
        // for these graphs since Z(2pi).x = Z(0).x + d
        const int N = sp.n_nodes > 0 ? sp.nodes[0] : 70;
        if (N < 8) fail(QPS_ERR_CONFIG, "build_smooth_quadrature: N must be >= 8");
        const double h = 2.0 * pi / N;
        for (int j = 0; j < N; ++j) {
            const double s = (j + 0.5) * h;
            const V2 z = smooth_Z(sp, d, s);
            const V2 t = smooth_Zp(sp, d, s);
            push_node(g, z, t, t, h);
        }
        SegDesc sd{};
        sd.kind = sp.shape == QPS_SHAPE_SINE ? SEG_SINE : SEG_FOURIER;
        sd.n = N;
        sd.offset = 0;
        sd.periodic = 1;
        sd.q = 0;
        sd.d = d;
        sd.y0 = sp.offset;
        sd.amp = sp.amplitude;
        sd.phase = sp.phase;
        sd.ncos = sp.n_cos;
        sd.nsin = sp.n_sin;
        sd.coef_off = int(pool.size());
        for (int m = 0; m < sp.n_cos; ++m) pool.push_back(sp.cosc[m]);
        for (int m = 0; m < sp.n_sin; ++m) pool.push_back(sp.sinc[m]);
        g.segs.push_back(sd);
        g.smooth = true;
    }
    // y range over the reference's 2049-point scan (geometry.hpp:449-460).  A
    // sine attains the scan's extremes at the grid points next to its peaks and
    // troughs (sin changes by ~1e-6 between neighbours there, far above
    // rounding), so only those points and the ends are evaluated -- with the
    // same expression, hence the same doubles as the full scan
    double ymin = std::numeric_limits<double>::infinity(), ymax = -ymin;
    auto probe = [&](int k) {
        const double x = -0.5 * d + d * k / 2048.0;
        const double y = spec_y_of_x(sp, d, x);
        ymin = std::min(ymin, y);
        ymax = std::max(ymax, y);
    };
    if (sp.shape == QPS_SHAPE_SINE) {
        probe(0);
        probe(2048);
        // theta_k = 2 pi (k / 2048 - 1/2) + phase; extremes of sin at pi/2 + pi m
        for (int m = -6; m <= 6; ++m) {
            const double kc = ((0.5 * pi + pi * m - sp.phase) / (2.0 * pi) + 0.5) * 2048.0;
            if (!(kc > -8.0 && kc < 2056.0)) continue;
            const int k0 = int(std::floor(kc));
            for (int k = k0 - 3; k <= k0 + 4; ++k)
                if (k >= 0 && k <= 2048) probe(k);
        }
    } else {
        for (int k = 0; k <= 2048; ++k) probe(k);
    }
    g.y_min = ymin;
    g.y_max = ymax;
    g.wall_y = spec_y_of_x(sp, d, -0.5 * d);
    return g;
}

}  // namespace

HostInterface build_interface_geometry(const qps_interface_spec& sp, double d) {
    std::vector<double> pool;  // Fourier coefficients stay on the host here
    return build_interface(sp, d, pool);
}

HostGeometry build_geometry(const StackDesc& st, const Numerics& num) {
    const int I = int(st.ifaces.size());
    if (int(st.eps.size()) != I + 1) fail(QPS_ERR_CONFIG, "stack needs exactly one more layer than interfaces");
    if (I < 1) fail(QPS_ERR_CONFIG, "stack needs at least one interface");
    HostGeometry g;
    g.d = st.d;
    g.I = I;
    g.P = num.P;
    g.Mw = num.Mw;
    g.M = num.M;
    g.R = num.R;
    static const bool htrace = getenv("QPS_HOST_TRACE") != nullptr;
    const auto tg0 = std::chrono::steady_clock::now();
    // interfaces are independent: built on host threads, each with its own
    // Fourier coefficient pool (concatenated afterwards in interface order);
    // the first failing interface (in order) raises, as the sequential reference
    {
        std::vector<HostInterface> ifs(I);
        std::vector<std::vector<double>> pools(I);
        std::vector<std::exception_ptr> errs(I);
        const int nt = std::max(1, std::min<int>(I, std::min(16u, std::max(1u, std::thread::hardware_concurrency()))));
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (int j = t; j < I; j += nt) {
                    try {
                        ifs[j] = build_interface(st.ifaces[j], st.d, pools[j]);
                    } catch (...) {
                        errs[j] = std::current_exception();
                    }
                }
            });
        for (auto& x : th) x.join();
        for (int j = 0; j < I; ++j)
            if (errs[j]) std::rethrow_exception(errs[j]);
        for (int j = 0; j < I; ++j) {
            const int base = int(g.fourier_pool.size());
            for (auto& sd : ifs[j].segs)
                if (sd.kind == SEG_FOURIER) sd.coef_off += base;
            g.fourier_pool.insert(g.fourier_pool.end(), pools[j].begin(), pools[j].end());
            g.ifaces.push_back(std::move(ifs[j]));
        }
    }
    const auto tg1 = std::chrono::steady_clock::now();
    if (htrace)
        fprintf(stderr, "build_geometry: interfaces %.3f ms\n", std::chrono::duration<double, std::milli>(tg1 - tg0).count());
    // build_frame (:449-478)
    g.y_U = g.ifaces.front().y_max + num.clearance * st.d;
    g.y_D = g.ifaces.back().y_min - num.clearance * st.d;
    std::vector<double> gx, gw;
    gauss_legendre(num.Mw, gx, gw);
    g.wall_lo.resize(I + 1);
    g.wall_hi.resize(I + 1);
    g.wall_ys.resize(I + 1);
    for (int i = 0; i <= I; ++i) {
        const double hi = (i == 0) ? g.y_U : g.ifaces[i - 1].wall_y;
        const double lo = (i == I) ? g.y_D : g.ifaces[i].wall_y;
        if (!(hi > lo))
            fail(QPS_ERR_GEOMETRY, "layer " + std::to_string(i + 1) +
                                       " has empty wall segment (interfaces cross at the wall?)");
        g.wall_hi[i] = hi;
        g.wall_lo[i] = lo;
        g.wall_ys[i].resize(num.Mw);
        for (int m = 0; m < num.Mw; ++m) g.wall_ys[i][m] = 0.5 * (lo + hi) + 0.5 * (hi - lo) * gx[m];
    }
    g.ud_x.resize(num.M);
    for (int m = 0; m < num.M; ++m) g.ud_x[m] = -0.5 * st.d + st.d * (m + 0.5) / num.M;
    // proxies (:489-494, build_proxy_circle :213-226)
    if (num.P < 1) fail(QPS_ERR_CONFIG, "build_proxy_circle: P must be >= 1");
    g.pc_x.resize(I + 1);
    g.pc_y.resize(I + 1);
    g.px.resize(I + 1);
    g.py.resize(I + 1);
    g.pnx.resize(I + 1);
    g.pny.resize(I + 1);
    // the circle's angles are the same for every layer: cos/sin once (the
    // values are bit-identical to evaluating them per layer)
    std::vector<double> pcos(num.P), psin(num.P);
    for (int p = 0; p < num.P; ++p) {
        const double ang = 2.0 * pi * p / num.P;
        pcos[p] = std::cos(ang);
        psin[p] = std::sin(ang);
    }
    for (int i = 0; i <= I; ++i) {
        const double hi = (i == 0) ? g.y_U : g.ifaces[i - 1].y_max;
        const double lo = (i == I) ? g.y_D : g.ifaces[i].y_min;
        const double cx = 0.0, cy = 0.5 * (lo + hi);
        g.pc_x[i] = cx;
        g.pc_y[i] = cy;
        g.pnx[i] = pcos;
        g.pny[i] = psin;
        g.px[i].resize(num.P);
        g.py[i].resize(num.P);
        for (int p = 0; p < num.P; ++p) {
            g.px[i][p] = cx + num.R * pcos[p];
            g.py[i][p] = cy + num.R * psin[p];
        }
    }
    return g;
}

double Problem::kappa(int n, double d) const { return k.front() * std::cos(theta) + 2.0 * pi * n / d; }

int choose_rb_order(const StackDesc& st, const HostGeometry& g, double omega, double theta) {
    const double k0 = omega * std::sqrt(st.eps.front() * st.mu.front());
    const double kb = omega * std::sqrt(st.eps.back() * st.mu.back());
    const double kap0 = k0 * std::cos(theta);
    const double cl_U = g.y_U - g.ifaces.front().y_max;
    const double cl_D = g.ifaces.back().y_min - g.y_D;
    const double kmax = std::max(k0, kb);
    for (int K = 4; K <= 400; ++K) {
        bool ok = true;
        for (int n : {K, -K}) {
            const double kap = kap0 + 2.0 * pi * n / g.d;
            if (std::abs(kap) <= kmax) {
                ok = false;
                break;
            }
            const double imU = std::sqrt(std::max(0.0, kap * kap - k0 * k0));
            const double imD = std::sqrt(std::max(0.0, kap * kap - kb * kb));
            ok = ok && imU * cl_U >= 30.0 && imD * cl_D >= 30.0;
        }
        if (ok) return K;
    }
    fail(QPS_ERR_CONFIG,
         "choose_rb_order: no K <= 400 decays the Rayleigh-Bloch tail; increase the U/D clearance");
}

Problem make_problem(const StackDesc& st, const HostGeometry& g, double omega, double theta, int K) {
    if (!(theta > -pi && theta < 0.0)) fail(QPS_ERR_CONFIG, "incidence angle must lie in (-pi, 0)");
    Problem p;
    p.omega = omega;
    p.theta = theta;
    for (size_t i = 0; i < st.eps.size(); ++i) p.k.push_back(omega * std::sqrt(st.eps[i] * st.mu[i]));
    const std::complex<double> iu{0.0, 1.0};
    const std::complex<double> a = std::exp(iu * (g.d * p.k.front() * std::cos(theta)));
    p.ar = a.real();
    p.ai = a.imag();
    p.K = K > 0 ? K : choose_rb_order(st, g, omega, theta);
    return p;
}

uint64_t reference_fill_evals(const HostGeometry& g) {
    // Loop structure of precompute_shift_blocks (assembly.hpp:239-284) and
    // self_quad_parts (kernels.hpp:199-270), counted in closed form per row.
    const int I = g.I, P = g.P, Mw = g.Mw, M = g.M;
    const int a = 10, naux = 15;
    uint64_t c = 0;
    for (int j = 0; j < I; ++j) {
        const auto& q = g.ifaces[j];
        const uint64_t N = q.N();
        uint64_t self = 0;
        if (q.smooth) {
            self = N * N + 11 * N + 180;  // central + wrap removal + aux
        } else {
            for (const auto& s : q.segs)
                for (int ml = 0; ml < s.n; ++ml) {
                    const bool corrected = std::min(ml, s.n - 1 - ml) >= a;
                    if (!corrected) {
                        self += N - 1;
                    } else {
                        const int lo = std::max(0, ml - (a - 1)), hi = std::min(s.n - 1, ml + (a - 1));
                        self += N - uint64_t(hi - lo + 1) + 2 * naux;
                    }
                }
        }
        c += 2 * (self + 2 * N * N);               // self_up/self_dn incl. nbr +-1
        if (j >= 1) c += 3 * N * g.ifaces[j - 1].N();  // coupl_up
        if (j + 1 < I) c += 3 * N * g.ifaces[j + 1].N();  // coupl_dn
        c += 2 * N * P;                              // B_self, B_below
    }
    for (int i = 0; i <= I; ++i) {
        if (i < I) c += 2 * uint64_t(Mw) * g.ifaces[i].N();
        if (i >= 1) c += 2 * uint64_t(Mw) * g.ifaces[i - 1].N();
        c += 2 * uint64_t(Mw) * P;  // Q_p, Q_m
    }
    c += 3 * uint64_t(M) * g.ifaces.front().N() + 3 * uint64_t(M) * g.ifaces.back().N();
    c += 2 * uint64_t(M) * P;
    return c;
}

// classify_point (postprocess.hpp:27-39).  The reference scans the interfaces
// top to bottom and returns the first one the point lies above; for a stack
// whose interfaces are ordered at this x (y_0(x) > y_1(x) > ...) the same
// answer comes from a binary search, checked against the scan's conditions
// at the boundary (and the scan itself is used where the order fails).
int classify_point(const StackDesc& st, const HostGeometry& g, double x, double y, int* layer) {
    if (y >= g.y_U) {
        *layer = 0;
        return 0;
    }
    if (y <= g.y_D) {
        *layer = g.I;
        return 2;
    }
    const int I = g.I;
    auto yj = [&](int j) { return spec_y_of_x(st.ifaces[j], st.d, x); };
    auto scan = [&]() {
        for (int j = 0; j < I; ++j) {
            const double v = yj(j);
            if (std::abs(y - v) < 1e-12 * st.d)
                fail(QPS_ERR_GEOMETRY, "field point lies on interface " + std::to_string(j + 1));
            if (y > v) return j;
        }
        return I;
    };
    int lo = 0, hi = I;  // first j in [lo, hi) with y > y_j(x), assuming decreasing y_j
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (y > yj(mid)) hi = mid;
        else lo = mid + 1;
    }
    // the scan's view: every j < lo has y <= y_j (and not within tolerance), lo has y > y_lo
    bool ok = true;
    for (int j = std::max(0, lo - 2); j < std::min(I, lo + 2) && ok; ++j) {
        const double v = yj(j);
        if (std::abs(y - v) < 1e-12 * st.d) ok = false;  // let the scan raise in reference order
        else if (j < lo && y > v) ok = false;
        else if (j == lo && !(y > v)) ok = false;
    }
    if (ok && lo >= 2) ok = yj(lo - 2) > yj(lo - 1);  // locally ordered
    *layer = ok ? lo : scan();
    return 1;
}

}  // namespace qpsb
