// qpscat_b200.hpp — C++ drop-in adapter for users of the reference library.
//
// Include AFTER the reference's own headers (it takes the reference's types):
//
//   #include "qpscat/postprocess.hpp"      // reference (Eigen, GSL)
//   #include "qpscat_b200.hpp"             // this adapter (links libqpscat_b200.so)
//
// and replace the reference's solve sequence (proj/tests/test_tridiag.cpp:112-126)
//
//   auto geom  = build_geometry(stack, num);
//   auto prob  = make_problem(stack, geom, omega, theta, K);
//   auto cache = precompute_shift_blocks(prob, num);
//   auto sys   = assemble_system(prob, cache, num);
//   Solution sol = solve_periodized(sys);
//   sol.flux_error = flux_error(sol, prob);
//
// by
//
//   qpscat::b200::Device dev;                       // one CUDA stream on GPU 0
//   Solution sol = dev.solve(stack, num, omega, theta, K);
//
// or keep the reference's step-wise sequence, each step on the device and its
// products resident in HBM (download any block with dev.block(kind, i)):
//
//   dev.setup(stack, num, omega, theta, K);         // build_geometry + make_problem
//   dev.precompute_shift_blocks();                  // assembly.hpp:212-287
//   dev.assemble_system();                          // assembly.hpp:462-483
//   dev.schur_complement();                         // periodize.hpp:124-126
//   std::vector<Vec> eta = dev.block_lu_solve();    // tridiag.hpp:23-46
//   Solution sol; dev.recover_aux(sol);             // tridiag.hpp:50-66
//
// Post-processing: spectrum() (reflection_transmission, postprocess.hpp:163-180),
// evaluate_field(), residual_suite() (postprocess.hpp:78-123, 369-399);
// angle sweeps: sweep() returns one SpectrumRow per angle with its orders and
// alpha_group, plan_sweep() the alpha grid.
//
// Errors are rethrown as the reference's exception types (errors.hpp:9-40).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "qpscat_b200.h"

namespace qpscat {
namespace b200 {

class Device {
public:
    explicit Device(int device = 0) : h_(qps_create(device)) {
        if (!h_) throw SolverError("qpscat_b200: no usable CUDA device", 0);
    }
    ~Device() { qps_destroy(h_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    // build_geometry + make_problem + precompute/assemble + solve_periodized + flux_error
    Solution solve(const LayerStack& stack, const NumericsParams& num, double omega, double theta, int K = 0) {
        setup(stack, num, omega, theta, K);
        check(qps_solve(h_));
        return solution();
    }

    // reflection_transmission (postprocess.hpp:163-180) of the last solve
    SpectrumRow spectrum(double theta) const {
        int I = 0, KK = 0;
        check(qps_problem_info(h_, &I, &KK, nullptr, nullptr, nullptr, nullptr, nullptr));
        const int nrb = 2 * KK + 1;
        std::vector<double> kappa(nrb);
        std::vector<qps_cplx> kU(nrb), kD(nrb), aU(nrb), aD(nrb);
        std::vector<int> pu(nrb), pd(nrb);
        SpectrumRow row;
        row.theta = theta;
        check(qps_reflection_transmission(h_, &row.R, &row.T, &row.flux_error, kappa.data(), kU.data(), kD.data(),
                                          pu.data(), pd.data()));
        check(qps_get_solution(h_, nullptr, nullptr, aU.data(), aD.data(), nullptr, nullptr));
        for (int i = 0; i < nrb; ++i) {
            row.up.push_back({i - KK, kappa[i], cd(kU[i].re, kU[i].im), cd(aU[i].re, aU[i].im), pu[i] != 0});
            row.down.push_back({i - KK, kappa[i], cd(kD[i].re, kD[i].im), cd(aD[i].re, aD[i].im), pd[i] != 0});
        }
        return row;
    }

    // build_geometry + make_problem (geometry.hpp:480-496, assembly.hpp:69-82)
    void setup(const LayerStack& stack, const NumericsParams& num, double omega, double theta, int K = 0) {
        std::vector<double> eps, mu;
        for (const auto& m : stack.materials) {
            eps.push_back(m.epsilon);
            mu.push_back(m.mu);
        }
        std::vector<qps_interface_spec> specs;
        std::vector<std::vector<double>> verts(stack.interfaces.size());
        for (size_t j = 0; j < stack.interfaces.size(); ++j) {
            const InterfaceSpec& sp = stack.interfaces[j];
            for (const auto& v : sp.vertices) {
                verts[j].push_back(v.x);
                verts[j].push_back(v.y);
            }
            qps_interface_spec s{};
            s.shape = sp.shape == InterfaceSpec::Shape::Sine      ? QPS_SHAPE_SINE
                      : sp.shape == InterfaceSpec::Shape::Fourier ? QPS_SHAPE_FOURIER
                                                                  : QPS_SHAPE_POLYLINE;
            s.offset = sp.offset;
            s.amplitude = sp.amplitude;
            s.phase = sp.phase;
            s.n_cos = int(sp.cosc.size());
            s.cosc = sp.cosc.data();
            s.n_sin = int(sp.sinc.size());
            s.sinc = sp.sinc.data();
            s.n_vertices = int(sp.vertices.size());
            s.vertices = verts[j].data();
            s.n_nodes = int(sp.nodes.size());
            s.nodes = sp.nodes.data();
            s.grading_q = sp.grading_q;
            specs.push_back(s);
        }
        const qps_numerics n{num.P, num.Mw, num.M, num.K, num.R, num.grading_q, num.clearance,
                             uint64_t(num.memory_budget)};
        check(qps_build_geometry(h_, stack.d, int(eps.size()), eps.data(), mu.data(), int(specs.size()),
                                 specs.data(), &n));
        P_ = num.P;
        period_ = stack.d;
        check(qps_make_problem(h_, omega, theta, K));
    }

    // ---- step-wise hot path (the reference's free functions, state on the device)
    void precompute_shift_blocks() { check(qps_precompute_shift_blocks(h_)); }
    void assemble_system() { check(qps_assemble_system(h_)); }
    void schur_complement() { check(qps_schur_complement(h_)); }
    std::vector<Vec> block_lu_solve() {
        check(qps_block_lu_solve(h_));
        check(qps_recover_aux(h_));  // eta is read back with the recovered solution
        return solution().eta;
    }
    void recover_aux(Solution& sol) {
        check(qps_recover_aux(h_));
        sol = solution();
    }
    Solution solve_periodized() {
        check(qps_schur_complement(h_));
        check(qps_block_lu_solve(h_));
        check(qps_recover_aux(h_));
        return solution();
    }
    // block_lu_solve on a caller-built PeriodizedSystem (tridiag.hpp:23-46)
    std::vector<Vec> block_lu_solve(const PeriodizedSystem& ps) {
        const int I = ps.I;
        const int n = int(ps.Ap_diag.at(0).rows());
        std::vector<qps_cplx> Ad(size_t(I) * n * n), Au(size_t(std::max(I - 1, 1)) * n * n),
            Al(size_t(std::max(I - 1, 1)) * n * n), f(n), eta(size_t(I) * n);
        auto put = [&](std::vector<qps_cplx>& dst, int j, const Mat& m) {
            for (int c = 0; c < n; ++c)
                for (int r = 0; r < n; ++r)
                    dst[(size_t(j) * n + c) * n + r] = qps_cplx{m(r, c).real(), m(r, c).imag()};
        };
        for (int j = 0; j < I; ++j) put(Ad, j, ps.Ap_diag[j]);
        for (int j = 0; j + 1 < I; ++j) {
            put(Au, j, ps.Ap_super[j]);
            put(Al, j, ps.Ap_sub[j]);
        }
        for (int r = 0; r < n; ++r) f[r] = qps_cplx{ps.f(r).real(), ps.f(r).imag()};
        check(qps_block_lu_solve_blocks(h_, I, n, Ad.data(), Au.data(), Al.data(), f.data(), eta.data()));
        std::vector<Vec> out(I, Vec(n));
        for (int j = 0; j < I; ++j)
            for (int r = 0; r < n; ++r) out[j](r) = cd(eta[size_t(j) * n + r].re, eta[size_t(j) * n + r].im);
        return out;
    }
    // any block of BlockSystem / PeriodizedSystem (qps_block_kind) as a matrix
    Mat block(int kind, int i = 0) const {
        int r = 0, c = 0;
        check(qps_download_block(h_, kind, i, nullptr, &r, &c));
        std::vector<qps_cplx> v(size_t(r) * c);
        if (r && c) check(qps_download_block(h_, kind, i, v.data(), &r, &c));
        Mat m(r, c);
        for (int cc = 0; cc < c; ++cc)
            for (int rr = 0; rr < r; ++rr) m(rr, cc) = cd(v[size_t(cc) * r + rr].re, v[size_t(cc) * r + rr].im);
        return m;
    }

    // evaluate_field(sol, p, points), postprocess.hpp:78-123: total field
    std::vector<cd> evaluate_field(const std::vector<Vec2>& points) {
        std::vector<double> xy;
        for (const auto& q : points) {
            xy.push_back(q.x);
            xy.push_back(q.y);
        }
        std::vector<qps_cplx> u(points.size());
        check(qps_evaluate_field(h_, int(points.size()), xy.data(), nullptr, u.data(), nullptr, nullptr));
        std::vector<cd> out;
        for (const auto& z : u) out.emplace_back(z.re, z.im);
        return out;
    }

    // residual_suite(sol, p, num, interfaces), postprocess.hpp:369-399
    ResidualReport residual_suite(const std::vector<int>& interfaces) {
        ResidualReport r;
        check(qps_residual_suite(h_, int(interfaces.size()), interfaces.data(), &r.wall_qp, &r.radiation,
                                 &r.interface));
        return r;
    }

    // plan_sweep: the alpha grid of n distinct alphas for the current k_1
    std::vector<double> plan_sweep(int n_alpha, double theta_lo, double theta_hi) {
        int cnt = 0;
        check(qps_plan_sweep(h_, n_alpha, theta_lo, theta_hi, 0, nullptr, nullptr, &cnt));
        std::vector<double> th(cnt);
        check(qps_plan_sweep(h_, n_alpha, theta_lo, theta_hi, cnt, th.data(), nullptr, &cnt));
        return th;
    }

    // multi-angle sweep: cache filled once, angles sharing
    // alpha eliminated and factored once, the rest batched; one SpectrumRow
    // per angle with its orders, flux error and alpha_group.  A failed angle
    // keeps NaN R/T and its qps_status in status (if given).
    std::vector<SpectrumRow> sweep(const LayerStack& stack, const NumericsParams& num, double omega,
                                   const std::vector<double>& thetas, int K, std::vector<int>* status = nullptr) {
        setup(stack, num, omega, thetas.at(0), K);
        return sweep(thetas, K, status);
    }
    std::vector<SpectrumRow> sweep(const std::vector<double>& thetas, int K, std::vector<int>* status = nullptr) {
        const int n = int(thetas.size()), nrb = 2 * K + 1;
        std::vector<double> R(n), T(n), fe(n);
        std::vector<qps_cplx> aU(size_t(n) * nrb), aD(size_t(n) * nrb);
        std::vector<int> st(n), grp(n);
        check(qps_sweep(h_, n, thetas.data(), K, 0, R.data(), T.data(), fe.data(), aU.data(), aD.data(), st.data()));
        int ng = 0;
        uint64_t ni = 0, nf = 0;
        check(qps_sweep_info(h_, n, grp.data(), &ng, &ni, &nf));
        const double d = period_;
        double k1 = 0, kl = 0;
        {
            int I = 0;
            check(qps_problem_info(h_, &I, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
            std::vector<double> k(I + 1);
            check(qps_problem_info(h_, nullptr, nullptr, nullptr, k.data(), nullptr, nullptr, nullptr));
            k1 = k.front();
            kl = k.back();
        }
        std::vector<SpectrumRow> rows(n);
        for (int a = 0; a < n; ++a) {
            SpectrumRow& row = rows[a];
            row.theta = thetas[a];
            row.R = R[a];
            row.T = T[a];
            row.flux_error = fe[a];
            row.alpha_group = grp[a];
            const double kref = std::max(k1, kl);
            for (int i = 0; i < nrb; ++i) {  // OrderAmplitude, postprocess.hpp:147-153, 166-176
                const int m = i - K;
                const double kap = k1 * std::cos(thetas[a]) + 2.0 * pi * m / d;
                auto vert = [&](double k) {
                    const double t2 = k * k - kap * kap;
                    return t2 >= 0.0 ? cd(std::sqrt(t2), 0.0) : cd(0.0, std::sqrt(-t2));
                };
                const cd ku = vert(k1), kd = vert(kl);
                const qps_cplx u = aU[size_t(a) * nrb + i], w = aD[size_t(a) * nrb + i];
                row.up.push_back({m, kap, ku, cd(u.re, u.im), ku.imag() == 0.0 && ku.real() > 1e-5 * kref});
                row.down.push_back({m, kap, kd, cd(w.re, w.im), kd.imag() == 0.0 && kd.real() > 1e-5 * kref});
            }
        }
        if (status) *status = st;
        return rows;
    }

    qps_ctx* handle() const { return h_; }

private:
    Solution solution() const {
        int I = 0, KK = 0;
        check(qps_problem_info(h_, &I, &KK, nullptr, nullptr, nullptr, nullptr, nullptr));
        std::vector<int> N(I);
        check(qps_problem_info(h_, nullptr, nullptr, N.data(), nullptr, nullptr, nullptr, nullptr));
        size_t ntot = 0;
        for (int v : N) ntot += 2 * size_t(v);
        std::vector<qps_cplx> eta(ntot), c(size_t(I + 1) * P_), aU(2 * KK + 1), aD(2 * KK + 1);
        std::vector<double> lsq(I + 1);
        double mx = 0;
        check(qps_get_solution(h_, eta.data(), c.data(), aU.data(), aD.data(), lsq.data(), &mx));
        Solution s;
        for (int i = 0; i <= I; ++i) {
            Vec ci(P_);
            for (int p = 0; p < P_; ++p) ci(p) = cd(c[size_t(i) * P_ + p].re, c[size_t(i) * P_ + p].im);
            s.c.push_back(ci);
        }
        size_t o = 0;
        for (int j = 0; j < I; ++j) {
            Vec e(2 * N[j]);
            for (int i = 0; i < 2 * N[j]; ++i) e(i) = cd(eta[o + i].re, eta[o + i].im);
            o += 2 * N[j];
            s.eta.push_back(e);
        }
        s.aU = Vec(2 * KK + 1);
        s.aD = Vec(2 * KK + 1);
        for (int i = 0; i < 2 * KK + 1; ++i) {
            s.aU(i) = cd(aU[i].re, aU[i].im);
            s.aD(i) = cd(aD[i].re, aD[i].im);
        }
        double R = 0, T = 0, fe = 0;
        check(qps_reflection_transmission(h_, &R, &T, &fe, nullptr, nullptr, nullptr, nullptr, nullptr));
        s.flux_error = fe;
        s.max_lsq_residual = mx;
        return s;
    }

    void check(int st) const {
        if (st == QPS_OK) return;
        char msg[1024];
        int layer = 0;
        uint64_t bytes = 0;
        qps_last_error(h_, msg, sizeof msg, &layer, &bytes);
        switch (st) {
            case QPS_ERR_CONFIG: throw ConfigError(msg);
            case QPS_ERR_GEOMETRY: throw GeometryError(msg);
            case QPS_ERR_USAGE: throw UsageError(msg);
            case QPS_ERR_SINGULARITY: throw SingularityError(msg);
            case QPS_ERR_SOLVER: throw SolverError(msg, layer);
            case QPS_ERR_MEMORY_BUDGET: throw MemoryBudgetError(msg, bytes);
            case QPS_ERR_DOMAIN: throw std::domain_error(msg);
            default: throw SolverError(std::string("qpscat_b200: ") + msg, layer);
        }
    }

    qps_ctx* h_;
    int P_ = 0;
    double period_ = 1.0;
};

}  // namespace b200
}  // namespace qpscat
