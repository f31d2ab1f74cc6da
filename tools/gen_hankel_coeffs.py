"""Generate paper_1410_5003_b200/csrc/hankel_coeffs.h — coefficient tables for the
device (and host) evaluator of H0^(1)(x), H1^(1)(x), x > 0.

Scheme (all tables fitted here with mpmath at 50 digits; nothing copied from a
third-party library):

  x < XB (= 8): piecewise on unit intervals [i, i+1], variable t = x - (i + 1/2):
      J0(x), J1(x), R0(x) = Y0(x) - (2/pi) ln(x) J0(x),
      R1(x) = Y1(x) - (2/pi) ln(x) J1(x) + 2/(pi x)
    are entire functions, so a degree-DEG_NEAR polynomial in t per interval
    (Chebyshev interpolant re-expanded in monomials) is accurate to ~1e-17.
    Then Y0 = R0 + (2/pi) ln x J0 and Y1 = R1 + (2/pi) ln x J1 - 2/(pi x).

  x >= XB: Hankel's modulus-free form
      H_nu(x) = sqrt(2/(pi x)) (P_nu(x) + i Q_nu(x)) exp(i(x - (2 nu + 1) pi/4)),
    with P_nu and x Q_nu smooth functions of u = (XB/x)^2 in (0, 1], fitted by
    Chebyshev interpolation in u (degree DEG_FAR) and re-expanded in monomials.

Run:  python tools/gen_hankel_coeffs.py   (prints max errors vs mpmath)
"""
import os

import mpmath as mp
import numpy as np

mp.mp.dps = 50

XB = 8
DEG_NEAR = 13
DEG_FAR = 11
TWO_OVER_PI = 2 / mp.pi


def near_funcs(x):
    x = mp.mpf(x)
    j0, j1 = mp.besselj(0, x), mp.besselj(1, x)
    y0, y1 = mp.bessely(0, x), mp.bessely(1, x)
    lg = mp.log(x)
    return [j0, j1, y0 - TWO_OVER_PI * lg * j0, y1 - TWO_OVER_PI * lg * j1 + TWO_OVER_PI / x]


def far_funcs(x):
    x = mp.mpf(x)
    out = []
    for nu in (0, 1):
        chi = x - (2 * nu + 1) * mp.pi / 4
        j, y = mp.besselj(nu, x), mp.bessely(nu, x)
        s = mp.sqrt(mp.pi * x / 2)
        P = s * (j * mp.cos(chi) + y * mp.sin(chi))
        Q = s * (-j * mp.sin(chi) + y * mp.cos(chi))
        out += [P, Q * x]
    return out


def cheb_to_monomial(f, a, b, deg, center):
    """Chebyshev interpolant of f on [a, b] at deg+1 nodes, re-expanded as a
    polynomial in (x - center); returns high-precision coefficients."""
    n = deg + 1
    nodes = [mp.cos(mp.pi * (k + mp.mpf(1) / 2) / n) for k in range(n)]
    xs = [(a + b) / 2 + (b - a) / 2 * t for t in nodes]
    vals = [f(x) for x in xs]
    nf = len(vals[0])
    out = []
    for q in range(nf):
        # Vandermonde solve in the shifted monomial basis (well conditioned on
        # half-width intervals, done in 50-digit arithmetic)
        V = mp.matrix(n, n)
        rhs = mp.matrix(n, 1)
        for i, x in enumerate(xs):
            t = x - center
            p = mp.mpf(1)
            for k in range(n):
                V[i, k] = p
                p *= t
            rhs[i] = vals[i][q]
        c = mp.lu_solve(V, rhs)
        out.append([c[k] for k in range(n)])
    return out


def main():
    near = []  # [interval][func][deg+1]
    for i in range(XB):
        near.append(cheb_to_monomial(near_funcs, mp.mpf(i), mp.mpf(i + 1), DEG_NEAR, mp.mpf(i) + mp.mpf(1) / 2))
    # far: functions of u = (XB/x)^2 on (0, 1]; fit on u in [0, 1]
    def far_u(u):
        u = mp.mpf(u)
        if u == 0:
            return [mp.mpf(1), mp.mpf(-1) / 8, mp.mpf(1), mp.mpf(3) / 8]
        return far_funcs(XB / mp.sqrt(u))
    far = cheb_to_monomial(far_u, mp.mpf(0), mp.mpf(1), DEG_FAR, mp.mpf(0))

    near_d = np.array([[[float(c) for c in fn] for fn in iv] for iv in near])
    far_d = np.array([[float(c) for c in fn] for fn in far])

    # ---------------- verify the double-precision evaluation formula -------
    def horner(c, t):
        acc = np.zeros_like(t) + c[-1]
        for k in range(len(c) - 2, -1, -1):
            acc = acc * t + c[k]
        return acc

    def eval_np(x):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros((4,) + x.shape)
        m = x < XB
        xn = x[m]
        i = np.minimum(np.floor(xn).astype(int), XB - 1)
        t = xn - (i + 0.5)
        vals = [np.array([horner(near_d[ii, q], tt) for ii, tt in zip(i, t)]) for q in range(4)]
        lg = np.log(xn) * (2 / np.pi)
        out[0][m] = vals[0]
        out[1][m] = vals[1]
        out[2][m] = vals[2] + lg * vals[0]
        out[3][m] = vals[3] + lg * vals[1] - (2 / np.pi) / xn
        xf = x[~m]
        inv = 1.0 / xf
        u = (XB * inv) ** 2
        P0, xQ0, P1, xQ1 = [horner(far_d[q], u) for q in range(4)]
        Q0, Q1 = xQ0 * inv, xQ1 * inv
        c, s = np.cos(xf), np.sin(xf)
        a = 1.0 / np.sqrt(np.pi * xf)
        # (P + iQ)(c + i s)(1 - i) a  and  (P + iQ)(c + i s)(-1 - i) a
        re0 = (P0 * c - Q0 * s)
        im0 = (P0 * s + Q0 * c)
        out[0][~m] = a * (re0 + im0)
        out[2][~m] = a * (im0 - re0)
        re1 = (P1 * c - Q1 * s)
        im1 = (P1 * s + Q1 * c)
        out[1][~m] = a * (-re1 + im1)
        out[3][~m] = a * (-im1 - re1)
        return out

    import json
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "hankel_mpmath.json")))
    rows = np.array(gold["rows"])
    xs = rows[:, 0]
    got = eval_np(xs)
    for q, name in enumerate(["J0", "J1", "Y0", "Y1"]):
        ref = rows[:, q + 1]
        err = np.abs(got[q] - ref) / np.maximum(1.0, np.abs(ref))
        k = np.argmax(err)
        print(f"{name}: max |err|/max(1,|f|) = {err[k]:.3g} at x = {xs[k]:.6g}")

    path = os.path.join(os.path.dirname(__file__), "..", "paper_1410_5003_b200", "csrc", "hankel_coeffs.h")
    with open(path, "w") as f:
        f.write("// GENERATED by tools/gen_hankel_coeffs.py (mpmath %s, %d digits) -- do not edit.\n" % (mp.__version__, mp.mp.dps))
        f.write("// Near (x < %d): per unit interval i, polynomials in t = x - (i + 1/2) of degree %d for\n" % (XB, DEG_NEAR))
        f.write("//   J0, J1, R0 = Y0 - (2/pi) ln(x) J0, R1 = Y1 - (2/pi) ln(x) J1 + 2/(pi x).\n")
        f.write("// Far (x >= %d): polynomials in u = (%d/x)^2 of degree %d for P0, x Q0, P1, x Q1.\n" % (XB, XB, DEG_FAR))
        f.write("#pragma once\n\n")
        f.write("#define QPS_HANKEL_XB %d\n#define QPS_HANKEL_NEAR_TERMS %d\n#define QPS_HANKEL_FAR_TERMS %d\n\n" % (XB, DEG_NEAR + 1, DEG_FAR + 1))
        f.write("// layout: [interval][function][term]\n")
        f.write("static const double qps_hankel_near_coeffs[%d] = {\n" % (XB * 4 * (DEG_NEAR + 1)))
        for i in range(XB):
            for q in range(4):
                f.write("    " + ", ".join("%.17e" % v for v in near_d[i, q]) + ",\n")
        f.write("};\n\n")
        f.write("// layout: [function][term]\n")
        f.write("static const double qps_hankel_far_coeffs[%d] = {\n" % (4 * (DEG_FAR + 1)))
        for q in range(4):
            f.write("    " + ", ".join("%.17e" % v for v in far_d[q]) + ",\n")
        f.write("};\n")
    print("wrote", os.path.normpath(path))


if __name__ == "__main__":
    main()
