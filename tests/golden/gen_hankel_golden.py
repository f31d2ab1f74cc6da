"""Generate tests/golden/hankel_mpmath.json: J0, J1, Y0, Y1 at 40 significant
digits (mpmath 1.3.0) on a log-spaced grid plus the reference's own KAT
arguments (proj/tests/test_specfun.cpp:18-22) and points straddling every
regime boundary used by the oracle shim and the device Hankel evaluator.

Run:  python tests/golden/gen_hankel_golden.py
"""
import json
import os

import mpmath as mp

mp.mp.dps = 40


def main():
    xs = set()
    n = 1500
    for i in range(n):
        xs.add(float(mp.mpf(10) ** (-8 + 12 * mp.mpf(i) / (n - 1))))
    # dense coverage of the fill's working range (k r in [1e-3, 200])
    for i in range(2000):
        xs.add(float(mp.mpf(10) ** (-3 + mp.mpf(5.3) * i / 1999)))
    for x in [0.5, 1.0, 8.0, 12.5, 1e4, 1e-12, 1e-8, 0.3, 1.7, 9.4, 55.0]:
        xs.add(float(x))
    for b in [1.0, 2.0, 4.0, 8.0, 12.0, 16.0, 25.0, 32.0]:
        for d in [-1e-12, -1e-9, 0.0, 1e-9, 1e-12]:
            xs.add(float(b + d))
    # zeros of J0, J1, Y0, Y1 (absolute-error regime)
    for k in range(1, 12):
        for f in (mp.besseljzero, mp.besselyzero):
            for nu in (0, 1):
                z = float(f(nu, k))
                for d in (-1e-6, 0.0, 1e-6):
                    xs.add(z + d)
    xs = sorted(x for x in xs if x > 0)
    rows = []
    for x in xs:
        X = mp.mpf(x)
        rows.append([
            x,
            float(mp.besselj(0, X)),
            float(mp.besselj(1, X)),
            float(mp.bessely(0, X)),
            float(mp.bessely(1, X)),
        ])
    out = {
        "generator": "tests/golden/gen_hankel_golden.py",
        "mpmath": mp.__version__,
        "dps": mp.mp.dps,
        "columns": ["x", "J0", "J1", "Y0", "Y1"],
        "rows": rows,
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "hankel_mpmath.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote {len(rows)} rows to {path}")


if __name__ == "__main__":
    main()
