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
    const bool ok = std::abs(gr.R - 0.0435607641) < 1e-6 && std::abs(gr.R - rr.R) < 1e-8;
    std::printf("%s\n", ok ? "DROP-IN OK" : "DROP-IN MISMATCH");
    return ok ? 0 : 1;
}
