/* ORACLE TEST INFRASTRUCTURE — not product code.
 *
 * gsl_sf_bessel_{J0,J1,Y0,Y1}_e for the reference's hankel01
 * (proj/include/qpscat/specfun.hpp:52-66, calls at :58-61).  GSL (version
 * unpinned, proj/CMakeLists.txt:13) is absent from this container, so its
 * published contract — double results accurate to a few ulp, GSL_EDOM for
 * x <= 0 on Y0/Y1 — is restated with an independent extended-precision
 * (x87 long double, 64-bit mantissa) evaluation:
 *   x < 2        : ascending power series of J0, J1, Y0, Y1 (A&S 9.1.10-9.1.11)
 *   2 <= x < 25  : Miller backward recurrence for J_n normalised by
 *                  J0 + 2 sum J_2k = 1, with Neumann series for Y0 and its
 *                  derivative for Y1 (A&S 9.1.88 family)
 *   x >= 25      : Hankel asymptotic expansion (A&S 9.2.5-9.2.10) truncated
 *                  below 1e-21, phases from sinl/cosl(x) without subtracting pi/4.
 * Pinned against mpmath (tests/golden/hankel_mpmath.json) and the reference's
 * own specfun KATs (proj/tests/test_specfun.cpp:12-30).  The four calls the
 * reference makes per argument share one evaluation through a per-thread cache.
 */
#ifndef QPS_SHIM_GSL_SF_BESSEL_H
#define QPS_SHIM_GSL_SF_BESSEL_H

#include <cmath>

#include "gsl_errno.h"

typedef struct {
    double val;
    double err;
} gsl_sf_result;

namespace qps_gsl_shim {

typedef long double LD;
static const LD kPi = 3.141592653589793238462643383279502884L;
static const LD kEuler = 0.577215664901532860606512090082402431L;
static const LD kSqrtHalf = 0.707106781186547524400844362104849039L;

struct Bessel4 {
    double x = -1.0;
    double j0 = 0, j1 = 0, y0 = 0, y1 = 0;
};

inline void eval_series(LD x, LD& J0, LD& J1, LD& Y0, LD& Y1) {
    const LD q = x * x / 4;
    const LD lg = logl(x / 2);
    LD t = 1, s0 = 1, sy0 = 0, H = 0;
    for (int k = 1; k < 60; ++k) {
        t *= -q / (LD(k) * LD(k));
        H += 1.0L / k;
        s0 += t;
        sy0 -= t * H;
        if (fabsl(t) * (H + 1) < 1e-24L * fabsl(s0)) break;
    }
    J0 = s0;
    Y0 = (2 / kPi) * (lg + kEuler) * J0 + (2 / kPi) * sy0;
    LD u = x / 2, s1 = u, sy1 = u * (1 - 2 * kEuler);
    LD Hk = 0;
    for (int k = 1; k < 60; ++k) {
        u *= -q / (LD(k) * LD(k + 1));
        Hk += 1.0L / k;
        const LD Hk1 = Hk + 1.0L / (k + 1);
        s1 += u;
        sy1 += u * (-2 * kEuler + Hk + Hk1);
        if (fabsl(u) * (Hk1 + 2) < 1e-24L * fabsl(x)) break;
    }
    J1 = s1;
    Y1 = -2 / (kPi * x) + (2 / kPi) * lg * J1 - sy1 / kPi;
}

inline void eval_miller(LD x, LD& J0, LD& J1, LD& Y0, LD& Y1) {
    int N = int((x + 36 + 8 * cbrtl(x)) / 2) * 2;
    LD jp1 = 0, j = 1e-40L;
    LD norm = 0, y0s = 0, y1s = 0;
    LD jn0 = 0, jn1 = 0;
    const LD two_over_x = 2 / x;
    // index m carried by j; accumulate its contributions, then step down
    for (int m = N; m >= 0; --m) {
        if ((m & 1) == 0) {
            if (m == 0) {
                norm += j;
                jn0 = j;
            } else {
                norm += 2 * j;
                const int k = m / 2;
                y0s += ((k & 1) ? -j : j) / LD(k);
            }
        } else {
            const int kp = (m + 1) / 2;  // term (-1)^kp J_{2kp-1}/kp
            LD c = ((kp & 1) ? -1.0L : 1.0L) / LD(kp);
            if (m >= 3) {
                const int km = (m - 1) / 2;  // term -(-1)^km J_{2km+1}/km
                c -= ((km & 1) ? -1.0L : 1.0L) / LD(km);
            }
            y1s += c * j;
            if (m == 1) jn1 = j;
        }
        if (m == 0) break;
        const LD jm1 = LD(m) * two_over_x * j - jp1;
        jp1 = j;
        j = jm1;
    }
    J0 = jn0 / norm;
    J1 = jn1 / norm;
    const LD lg = logl(x / 2) + kEuler;
    Y0 = (2 / kPi) * lg * J0 - (4 / kPi) * (y0s / norm);
    Y1 = -(2 / kPi) * J0 / x + (2 / kPi) * lg * J1 + (2 / kPi) * (y1s / norm);
}

inline void asymp_pq(LD nu, LD x, LD& P, LD& Q) {
    const LD mu = 4 * nu * nu;
    LD term = 1, prev = 2;
    P = 1;
    Q = 0;
    for (int k = 1; k < 200; ++k) {
        term *= (mu - LD(2 * k - 1) * LD(2 * k - 1)) / (LD(8 * k) * x);
        const LD a = fabsl(term);
        if (a > prev) break;  // divergent tail
        prev = a;
        switch (k & 3) {
            case 1: Q += term; break;
            case 2: P -= term; break;
            case 3: Q -= term; break;
            default: P += term; break;
        }
        if (a < 1e-22L) break;
    }
}

inline void eval_asymp(LD x, LD& J0, LD& J1, LD& Y0, LD& Y1) {
    LD P0, Q0, P1, Q1;
    asymp_pq(0, x, P0, Q0);
    asymp_pq(1, x, P1, Q1);
    const LD sx = sinl(x), cx = cosl(x);
    const LD c0 = (cx + sx) * kSqrtHalf, s0 = (sx - cx) * kSqrtHalf;
    const LD c1 = (sx - cx) * kSqrtHalf, s1 = -(sx + cx) * kSqrtHalf;
    const LD amp = sqrtl(2 / (kPi * x));
    J0 = amp * (P0 * c0 - Q0 * s0);
    Y0 = amp * (P0 * s0 + Q0 * c0);
    J1 = amp * (P1 * c1 - Q1 * s1);
    Y1 = amp * (P1 * s1 + Q1 * c1);
}

inline const Bessel4& eval(double x) {
    thread_local Bessel4 cache;
    if (cache.x == x) return cache;
    LD J0, J1, Y0, Y1;
    const LD lx = x;
    if (x < 2.0) eval_series(lx, J0, J1, Y0, Y1);
    else if (x < 25.0) eval_miller(lx, J0, J1, Y0, Y1);
    else eval_asymp(lx, J0, J1, Y0, Y1);
    cache.x = x;
    cache.j0 = double(J0);
    cache.j1 = double(J1);
    cache.y0 = double(Y0);
    cache.y1 = double(Y1);
    return cache;
}

inline int finish(double v, gsl_sf_result* r) {
    r->val = v;
    r->err = 4.0 * 2.220446049250313e-16 * std::fabs(v);
    return GSL_SUCCESS;
}

}  // namespace qps_gsl_shim

inline int gsl_sf_bessel_J0_e(double x, gsl_sf_result* r) {
    const double ax = std::fabs(x);
    if (ax == 0.0) { r->val = 1.0; r->err = 0.0; return GSL_SUCCESS; }
    if (!std::isfinite(x)) { r->val = NAN; r->err = NAN; return GSL_EDOM; }
    return qps_gsl_shim::finish(qps_gsl_shim::eval(ax).j0, r);
}
inline int gsl_sf_bessel_J1_e(double x, gsl_sf_result* r) {
    const double ax = std::fabs(x);
    if (ax == 0.0) { r->val = 0.0; r->err = 0.0; return GSL_SUCCESS; }
    if (!std::isfinite(x)) { r->val = NAN; r->err = NAN; return GSL_EDOM; }
    const double v = qps_gsl_shim::eval(ax).j1;
    return qps_gsl_shim::finish(x < 0 ? -v : v, r);
}
inline int gsl_sf_bessel_Y0_e(double x, gsl_sf_result* r) {
    if (!(x > 0.0) || !std::isfinite(x)) { r->val = NAN; r->err = NAN; return GSL_EDOM; }
    return qps_gsl_shim::finish(qps_gsl_shim::eval(x).y0, r);
}
inline int gsl_sf_bessel_Y1_e(double x, gsl_sf_result* r) {
    if (!(x > 0.0) || !std::isfinite(x)) { r->val = NAN; r->err = NAN; return GSL_EDOM; }
    return qps_gsl_shim::finish(qps_gsl_shim::eval(x).y1, r);
}

#endif
