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

    // multi-angle sweep: cache filled once, angles batched on the device
    std::vector<SpectrumRow> sweep(const LayerStack& stack, const NumericsParams& num, double omega,
                                   const std::vector<double>& thetas, int K) {
        setup(stack, num, omega, thetas.at(0), K);
        const int n = int(thetas.size()), nrb = 2 * K + 1;
        std::vector<double> R(n), T(n), fe(n);
        std::vector<qps_cplx> aU(size_t(n) * nrb), aD(size_t(n) * nrb);
        std::vector<int> st(n);
        check(qps_sweep(h_, n, thetas.data(), K, 0, R.data(), T.data(), fe.data(), aU.data(), aD.data(), st.data()));
        std::vector<SpectrumRow> rows(n);
        for (int a = 0; a < n; ++a) {
            rows[a].theta = thetas[a];
            rows[a].R = R[a];
            rows[a].T = T[a];
            rows[a].flux_error = fe[a];
        }
        return rows;
    }

    qps_ctx* handle() const { return h_; }

private:
    void setup(const LayerStack& stack, const NumericsParams& num, double omega, double theta, int K) {
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
        check(qps_make_problem(h_, omega, theta, K));
    }

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
};

}  // namespace b200
}  // namespace qpscat
