"""Numerical rank of the inter-interface coupling blocks A_{j,j+1}, A'_{j,j+1}
(after the Schur update) and of the diagonal blocks, config 4 (first layers):
singular values relative to the largest, counts above 1e-8 / 1e-12 / 1e-15."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nif = int(sys.argv[2]) if len(sys.argv) > 2 else 12
st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
s = Solver()
s.build_geometry(st, num)
s.make_problem(om, th, K)
s.precompute_shift_blocks()
s.assemble_system()
s.schur_complement()
for name in ("A_super", "A_sub", "Ap_super", "Ap_sub", "A_diag"):
    for j in (1, 5, 9):
        b = s.download_block(name, j)
        sv = np.linalg.svd(b, compute_uv=False)
        r = sv / sv[0]
        print(f"{name:9s} j={j} {b.shape} rank@1e-8={int((r > 1e-8).sum())} @1e-12={int((r > 1e-12).sum())} "
              f"@1e-15={int((r > 1e-15).sum())}")
