// Drop-in demonstration: the reference's own end-to-end
// Fresnel case (proj/tests/test_postprocess.cpp:112-120, R = 0.0435607641)
// solved twice from the SAME reference types — once by the reference's CPU
// path, once through include/qpscat_b200.hpp on the B200.  Built against the
// reference headers + oracle shims; the GPU half needs a device.
#include <cstdio>

#include "qpscat/postprocess.hpp"
#include "qpscat_b200.hpp"

using namespace qpscat;

int main() {
    LayerStack stack;
    stack.d = 1.0;
    stack.materials = {{1.0, 1.0}, {2.0, 1.0}};
    InterfaceSpec sp;
    sp.shape = InterfaceSpec::Shape::Sine;
    sp.amplitude = 0.0;
    sp.nodes = {44};
    stack.interfaces = {sp};
    NumericsParams num;
    num.P = 64;
    num.Mw = 48;
    num.M = 36;
    num.R = 2.0;
    num.clearance = 0.4;
    const double omega = 5.0, theta = -pi / 3;

    auto geom = build_geometry(stack, num);
    auto prob = make_problem(stack, geom, omega, theta, 0);
    auto cache = precompute_shift_blocks(prob, num);
    auto sys = assemble_system(prob, cache, num);
    Solution ref = solve_periodized(sys);
    const SpectrumRow rr = reflection_transmission(ref, prob);
    std::printf("reference CPU : R = %.12f  T = %.12f  flux = %.2e\n", rr.R, rr.T, rr.flux_error);

    qpscat::b200::Device dev;
    Solution gpu = dev.solve(stack, num, omega, theta, 0);
    const SpectrumRow gr = dev.spectrum(theta);
    std::printf("qpscat_b200   : R = %.12f  T = %.12f  flux = %.2e  |aU0 diff| = %.2e\n", gr.R, gr.T,
                gr.flux_error, std::abs(gpu.aU(prob.K) - ref.aU(prob.K)));
    bool ok = std::abs(gr.R - 0.0435607641) < 1e-6 && std::abs(gr.R - rr.R) < 1e-8;

    // the reference's step-wise sequence on the device (assembly.hpp:212,462;
    // periodize.hpp:124; tridiag.hpp:23,50)
    dev.setup(stack, num, omega, theta, 0);
    dev.precompute_shift_blocks();
    dev.assemble_system();
    dev.schur_complement();
    const Mat a00 = dev.block(QPS_BLK_AP_DIAG, 0);  // A' is factored in place by the block solve
    const std::vector<Vec> eta = dev.block_lu_solve();
    Solution step;
    dev.recover_aux(step);
    const double dstep = std::abs(step.aU(prob.K) - ref.aU(prob.K));
    std::printf("step-wise     : |aU0 diff| = %.2e, eta blocks %zu, A'_00 %ldx%ld\n", dstep, eta.size(),
                long(a00.rows()), long(a00.cols()));
    ok = ok && dstep < 1e-8 && eta.size() == 1 && a00.rows() == 2 * 44;

    // residual suite (postprocess.hpp:369-399) of the device solution
    const ResidualReport rep = dev.residual_suite({0});
    std::printf("residual suite: wall %.2e radiation %.2e interface %.2e\n", rep.wall_qp, rep.radiation,
                rep.interface);
    ok = ok && rep.wall_qp < 1e-8 && rep.radiation < 1e-8;

    // alpha-grouped sweep: rows with orders and alpha_group
    const std::vector<double> grid = dev.plan_sweep(2, -2.8, -0.4);
    std::vector<int> st;
    const std::vector<SpectrumRow> rows = dev.sweep(stack, num, omega, grid, 10, &st);
    int groups = 0;
    for (const auto& r : rows) groups = std::max(groups, r.alpha_group + 1);
    std::printf("sweep         : %zu angles, %d alpha groups, R[0] = %.12f, %zu orders\n", rows.size(), groups,
                rows.at(0).R, rows.at(0).up.size());
    ok = ok && groups == 2 && rows.at(0).up.size() == 21;
    for (int s : st) ok = ok && s == QPS_OK;
    std::printf("%s\n", ok ? "DROP-IN OK" : "DROP-IN MISMATCH");
    return ok ? 0 : 1;
}
