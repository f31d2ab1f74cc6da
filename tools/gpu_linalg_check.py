"""GPU diagnostics for the dense building blocks: zgemm, qsolve vs numpy/oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1410_5003_b200.qpscat import Solver

rng = np.random.default_rng(1)
def rc(*s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)
g = Solver()
o = Solver(lib="oracle/_ref/libqpscat_ref.so")
for (M, N, K) in [(8, 8, 4), (64, 64, 8), (81, 160, 200), (600, 600, 80), (17, 3, 5)]:
    A, B = rc(M, K), rc(K, N)
    C = g.debug_zgemm(A, B)
    print("zgemm", M, N, K, np.abs(C - A @ B).max() / np.abs(A @ B).max())
for (m, p, n, defic) in [(8, 8, 3, 0), (40, 20, 5, 0), (80, 60, 30, 0), (12, 6, 2, 2), (80, 60, 50, 7), (200, 81, 40, 5)]:
    Q, R = rc(m, p), rc(m, n)
    for d in range(defic):
        Q[:, p - 1 - d] = Q[:, d] * (0.5 + 0.1j)
    Xg, rg = g.qsolve(Q, R)
    Xo, ro = o.qsolve(Q, R)
    Xl = np.linalg.lstsq(Q, R, rcond=1e-12)[0]
    print(f"qsolve m={m} p={p} n={n} defic={defic}: rank gpu {rg} ref {ro}; |Xg-Xo|/|Xo| {np.abs(Xg-Xo).max()/np.abs(Xo).max():.2e}"
          f"  |Xg-lstsq| {np.abs(Xg-Xl).max()/np.abs(Xl).max():.2e}  res gpu {np.linalg.norm(Q@Xg-R)/np.linalg.norm(R):.3e} ref {np.linalg.norm(Q@Xo-R)/np.linalg.norm(R):.3e}")
