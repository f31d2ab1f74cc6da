"""GPU COD least squares (qsolve) against numpy's pseudo-inverse on random full-rank and rank-deficient shapes, including the solver's 160 x 80 x 1216 case."""
import numpy as np, sys
sys.path.insert(0, ".")
from paper_1410_5003_b200.qpscat import Solver
g = Solver()
rng = np.random.default_rng(3)
def rc(*s): return rng.standard_normal(s) + 1j * rng.standard_normal(s)
for (m, p, n, defic) in [(20, 6, 50, 0), (40, 20, 100, 3), (160, 80, 1216, 0), (160, 80, 1216, 10), (280, 121, 608, 0), (280, 121, 608, 20), (80, 80, 1216, 33), (200, 121, 608, 18)]:
    Q = rc(m, p)
    if defic: Q[:, -defic:] = Q[:, :defic] @ rc(defic, defic)
    R = rc(m, n)
    X, r = g.qsolve(Q, R)
    ref = np.linalg.pinv(Q, rcond=1e-12) @ R
    print(m, p, n, defic, r, np.linalg.norm(X - ref) / np.linalg.norm(ref))
