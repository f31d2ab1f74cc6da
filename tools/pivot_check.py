"""How much pivoting do the periodized diagonal blocks need?  Row interchanges
of scipy's GEPP on A'_jj, and the growth of an unpivoted LU (max|U| / max|A|)."""
import os
import sys

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nif = int(sys.argv[2]) if len(sys.argv) > 2 else 8
st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
s = Solver()
s.build_geometry(st, num)
s.make_problem(om, th, K)
s.precompute_shift_blocks()
s.assemble_system()
s.schur_complement()
for j in range(0, nif, max(1, nif // 4)):
    A = s.download_block("Ap_diag", j)
    lu, piv = sl.lu_factor(A)
    swaps = int((piv != np.arange(len(piv))).sum())
    # unpivoted LU growth
    U = A.copy()
    n = len(U)
    minpiv = np.inf
    for k in range(n - 1):
        minpiv = min(minpiv, abs(U[k, k]) / np.abs(U[k:, k]).max())
        U[k + 1:, k] /= U[k, k]
        U[k + 1:, k + 1:] -= np.outer(U[k + 1:, k], U[k, k + 1:])
    growth = np.abs(np.triu(U)).max() / np.abs(A).max()
    print(f"j={j} n={n} GEPP swaps={swaps} unpivoted: growth={growth:.2e} min |a_kk|/max|col|={minpiv:.2e} "
          f"cond={np.linalg.cond(A):.2e}")
