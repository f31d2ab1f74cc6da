// FP64 Hankel functions H0^(1), H1^(1) and the four layer-potential kernels
// on the device.  Replaces hankel01 (specfun.hpp:52-66, four GSL calls per
// argument) and eval_kernels (kernels.hpp:35-52).
//
//   x < 8 : one interval lookup, four degree-13 polynomials (J0, J1 and the
//           log-free parts R0, R1 of Y0, Y1), one log, one reciprocal;
//   x >= 8: four degree-11 polynomials in u = 64/x^2 (P0, xQ0, P1, xQ1), one
//           sincos, one rsqrt, one reciprocal; H1's phase is H0's times -i.
// Tables: hankel_coeffs.h (tools/gen_hankel_coeffs.py, fitted with mpmath);
// max error vs 40-digit mpmath on [1e-8, 1e4]: 3.7e-16 * max(1, |f|).
#pragma once

#include <cuda_runtime.h>

#include "hankel_coeffs.h"

namespace qpsb {

struct cplx {
    double re, im;
};

__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return cplx{r, i}; }

#define QPS_NEAR_STRIDE (4 * QPS_HANKEL_NEAR_TERMS)

// Near-field coefficients must be staged (shared memory on the device);
// far-field ones are warp-uniform and live in constant memory.
#ifdef __CUDACC__
__constant__ double c_hankel_far[4 * QPS_HANKEL_FAR_TERMS];
#endif

struct HankelOut {
    double j0, y0, j1, y1;  // H0 = j0 + i y0, H1 = j1 + i y1
};

__host__ __device__ __forceinline__ void hankel01_eval(double x, const double* __restrict__ near,
                                                       const double* __restrict__ far, HankelOut& h) {
    constexpr double two_over_pi = 0.63661977236758134308;
    if (x < double(QPS_HANKEL_XB)) {
        int i = int(x);
        i = i > QPS_HANKEL_XB - 1 ? QPS_HANKEL_XB - 1 : i;
        const double t = x - (double(i) + 0.5);
        const double* c = near + i * QPS_NEAR_STRIDE;
        double a0 = c[0 * QPS_HANKEL_NEAR_TERMS + QPS_HANKEL_NEAR_TERMS - 1];
        double a1 = c[1 * QPS_HANKEL_NEAR_TERMS + QPS_HANKEL_NEAR_TERMS - 1];
        double a2 = c[2 * QPS_HANKEL_NEAR_TERMS + QPS_HANKEL_NEAR_TERMS - 1];
        double a3 = c[3 * QPS_HANKEL_NEAR_TERMS + QPS_HANKEL_NEAR_TERMS - 1];
#pragma unroll
        for (int k = QPS_HANKEL_NEAR_TERMS - 2; k >= 0; --k) {
            a0 = fma(a0, t, c[0 * QPS_HANKEL_NEAR_TERMS + k]);
            a1 = fma(a1, t, c[1 * QPS_HANKEL_NEAR_TERMS + k]);
            a2 = fma(a2, t, c[2 * QPS_HANKEL_NEAR_TERMS + k]);
            a3 = fma(a3, t, c[3 * QPS_HANKEL_NEAR_TERMS + k]);
        }
        const double lg = two_over_pi * log(x);
        h.j0 = a0;
        h.j1 = a1;
        h.y0 = fma(lg, a0, a2);
        h.y1 = fma(lg, a1, a3) - two_over_pi / x;
    } else {
        const double inv = 1.0 / x;
        const double u = (double(QPS_HANKEL_XB) * inv) * (double(QPS_HANKEL_XB) * inv);
        double p0 = far[0 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
        double q0 = far[1 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
        double p1 = far[2 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
        double q1 = far[3 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
#pragma unroll
        for (int k = QPS_HANKEL_FAR_TERMS - 2; k >= 0; --k) {
            p0 = fma(p0, u, far[0 * QPS_HANKEL_FAR_TERMS + k]);
            q0 = fma(q0, u, far[1 * QPS_HANKEL_FAR_TERMS + k]);
            p1 = fma(p1, u, far[2 * QPS_HANKEL_FAR_TERMS + k]);
            q1 = fma(q1, u, far[3 * QPS_HANKEL_FAR_TERMS + k]);
        }
        q0 *= inv;
        q1 *= inv;
        double s, c;
#ifdef __CUDA_ARCH__
        sincos(x, &s, &c);
        const double a = rsqrt(3.14159265358979323846 * x);
#else
        s = std::sin(x);
        c = std::cos(x);
        const double a = 1.0 / std::sqrt(3.14159265358979323846 * x);
#endif
        const double re0 = p0 * c - q0 * s, im0 = p0 * s + q0 * c;
        const double re1 = p1 * c - q1 * s, im1 = p1 * s + q1 * c;
        h.j0 = a * (re0 + im0);
        h.y0 = a * (im0 - re0);
        h.j1 = a * (im1 - re1);
        h.y1 = -a * (im1 + re1);
    }
}

#ifdef __CUDACC__
// Device evaluator for the fill kernels: the caller supplies 1/x and
// u = (8/x)^2 (from the shared 1/r of a pair), the far-field coefficients are read from constant
// memory at compile-time offsets (direct DFMA operands), the near-field table
// sits in shared memory as double2 pairs {J0, J1}, {R0, R1} per interval and
// term (two 16-byte loads per Horner step for four polynomials).
#define QPS_NEAR2_STRIDE (2 * QPS_HANKEL_NEAR_TERMS)
__device__ __forceinline__ void hankel01_dev(double x, double inv_x, double u, const double2* __restrict__ near2,
                                             HankelOut& h) {
    constexpr double two_over_pi = 0.63661977236758134308;
    if (x < double(QPS_HANKEL_XB)) {
        int i = int(x);
        i = i > QPS_HANKEL_XB - 1 ? QPS_HANKEL_XB - 1 : i;
        const double t = x - (double(i) + 0.5);
        const double2* c = near2 + i * QPS_NEAR2_STRIDE;
        double2 p = c[2 * (QPS_HANKEL_NEAR_TERMS - 1)], q = c[2 * (QPS_HANKEL_NEAR_TERMS - 1) + 1];
        double a0 = p.x, a1 = p.y, a2 = q.x, a3 = q.y;
#pragma unroll
        for (int k = QPS_HANKEL_NEAR_TERMS - 2; k >= 0; --k) {
            p = c[2 * k];
            q = c[2 * k + 1];
            a0 = fma(a0, t, p.x);
            a1 = fma(a1, t, p.y);
            a2 = fma(a2, t, q.x);
            a3 = fma(a3, t, q.y);
        }
        const double lg = two_over_pi * log(x);
        h.j0 = a0;
        h.j1 = a1;
        h.y0 = fma(lg, a0, a2);
        h.y1 = fma(lg, a1, a3) - two_over_pi * inv_x;
    } else {
        double p0 = c_hankel_far[0 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
        double q0 = c_hankel_far[1 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
        double p1 = c_hankel_far[2 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
        double q1 = c_hankel_far[3 * QPS_HANKEL_FAR_TERMS + QPS_HANKEL_FAR_TERMS - 1];
#pragma unroll
        for (int k = QPS_HANKEL_FAR_TERMS - 2; k >= 0; --k) {
            p0 = fma(p0, u, c_hankel_far[0 * QPS_HANKEL_FAR_TERMS + k]);
            q0 = fma(q0, u, c_hankel_far[1 * QPS_HANKEL_FAR_TERMS + k]);
            p1 = fma(p1, u, c_hankel_far[2 * QPS_HANKEL_FAR_TERMS + k]);
            q1 = fma(q1, u, c_hankel_far[3 * QPS_HANKEL_FAR_TERMS + k]);
        }
        // H0 = a (p0 + i Q0) e^{i(x - pi/4)}, H1 = a (p1 + i Q1) e^{i(x - 3pi/4)}, a = (pi x)^{-1/2},
        // Q = (x Q) / x, expanded with cos +- sin so that a and 1/x scale two shared factors
        double s, c;
        sincos(x, &s, &c);
        const double a = rsqrt(3.14159265358979323846 * x);
        const double A1 = a * (c + s), A2 = a * (c - s);
        const double A1q = A1 * inv_x, A2q = A2 * inv_x;
        h.j0 = fma(p0, A1, q0 * A2q);
        h.y0 = fma(q0, A1q, -p0 * A2);
        h.j1 = fma(q1, A1q, -p1 * A2);
        h.y1 = -fma(p1, A1, q1 * A2q);
    }
}
#endif

// eval_kernels (kernels.hpp:35-52) given the separation rv = x - z (r > 0):
//   S  = (i/4) H0(kr)
//   D  = (ik/4) H1(kr) (rhat . n')        n' = source normal
//   D* = -(ik/4) H1(kr) (rhat . n)        n  = target normal
//   T  = (ik/4) [ k H0 (rhat.n)(rhat.n') + H1/r (n.n' - 2 (rhat.n)(rhat.n')) ]
struct KVals {
    cplx S, D, Ds, T;
};

__host__ __device__ __forceinline__ void kernel_vals(double k, double rvx, double rvy, double r, double nxx,
                                                     double nxy, double nzx, double nzy, const HankelOut& h,
                                                     KVals& v) {
    const double inv_r = 1.0 / r;
    const double cn = (rvx * nxx + rvy * nxy) * inv_r;
    const double cdn = (rvx * nzx + rvy * nzy) * inv_r;
    const double nn = nxx * nzx + nxy * nzy;
    const double k4 = 0.25 * k;
    // S = (i/4)(j0 + i y0) = (-y0/4) + i (j0/4)
    v.S = cmk(-0.25 * h.y0, 0.25 * h.j0);
    // (ik/4) H1 = k4 * (-y1 + i j1)
    const double ih1r = -k4 * h.y1, ih1i = k4 * h.j1;
    v.D = cmk(ih1r * cdn, ih1i * cdn);
    v.Ds = cmk(-ih1r * cn, -ih1i * cn);
    // T = (ik/4)[k H0 cn cdn + H1 inv_r (nn - 2 cn cdn)]
    const double a = k * cn * cdn, b = inv_r * (nn - 2.0 * cn * cdn);
    const double br = a * h.j0 + b * h.j1, bi = a * h.y0 + b * h.y1;  // bracket
    v.T = cmk(-k4 * bi, k4 * br);
}

#ifdef __CUDACC__
// kernel_vals with the k-independent geometry of the pair precomputed:
// cn = rhat.n, cdn = rhat.n', nn = n.n', inv_r = 1/r
__device__ __forceinline__ void kernel_vals_geo(double k, double cn, double cdn, double nn, double inv_r,
                                                const HankelOut& h, KVals& v) {
    const double k4 = 0.25 * k;
    v.S = cmk(-0.25 * h.y0, 0.25 * h.j0);
    const double ih1r = -k4 * h.y1, ih1i = k4 * h.j1;
    v.D = cmk(ih1r * cdn, ih1i * cdn);
    v.Ds = cmk(-ih1r * cn, -ih1i * cn);
    const double a = k * cn * cdn, b = inv_r * (nn - 2.0 * cn * cdn);
    const double br = a * h.j0 + b * h.j1, bi = a * h.y0 + b * h.y1;
    v.T = cmk(-k4 * bi, k4 * br);
}
#endif

}  // namespace qpsb
