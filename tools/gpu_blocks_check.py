"""At one alpha-grid angle of a config-5 prefix: the periodized blocks of the
GPU (step-wise path) vs the oracle's (norms of couplings and interior X), and
the GPU's own blocks solved by the GPU block solve and by the reference's
block Thomas.  usage: python tools/gpu_blocks_check.py [angle_index]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

ia = int(sys.argv[1]) if len(sys.argv) > 1 else 0
st, num, om, th0, K, _ = configs.config(5, n_interfaces=6)
o = Solver(lib="oracle/_ref/libqpscat_ref.so")
g = Solver(device=0)
o.build_geometry(st, num)
o.make_problem(om, th0, K)
th, _ = o.plan_sweep(3, -np.pi + 0.1, -0.1)
I = 6
blk = {}
for name, s in (("oracle", o), ("gpu", g)):
    s.build_geometry(st, num)
    s.make_problem(om, th[ia], K)
    s.precompute_shift_blocks()
    s.assemble_system()
    s.schur_complement()
    blk[name] = {k: [s.download_block(k, j) for j in range(n)] for k, n in
                 (("Ap_diag", I), ("Ap_super", I - 1), ("Ap_sub", I - 1), ("X_self", I), ("X_above", I))
                 if True}
    blk[name]["f"] = s.download_block("f", 0).ravel()
for k in ("Ap_super", "Ap_sub", "Ap_diag", "X_self"):
    a, b = blk["gpu"][k], blk["oracle"][k]
    print(k, "norm gpu", ["%.2e" % np.linalg.norm(x) for x in a], "oracle", ["%.2e" % np.linalg.norm(x) for x in b],
          "rel diff", ["%.1e" % (np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)) for x, y in zip(a, b)])
Ad, Au, Al, f = blk["gpu"]["Ap_diag"], blk["gpu"]["Ap_super"], blk["gpu"]["Ap_sub"], blk["gpu"]["f"]
n = Ad[0].shape[0]
f = np.r_[f, np.zeros(n - len(f))]
eo = o.block_lu_solve_blocks(Ad, Au, Al, f)
eg = np.array(g.block_lu_solve_blocks(Ad, Au, Al, f))
print("gpu blocks: gpu bcr vs reference thomas eta", np.linalg.norm(eg - eo) / np.linalg.norm(eo), g.solver_diagnostics())
for j in range(I - 1):
    sv = np.linalg.svd(Au[j], compute_uv=False)
    print("gpu coupling", j, "sv", ["%.1e" % (sv[i] / sv[0]) for i in (0, 20, 30, 40, 48, 60)], "|s0|", "%.1e" % sv[0])
A = np.zeros((I * n, I * n), complex)
for j in range(I):
    A[j * n:(j + 1) * n, j * n:(j + 1) * n] = Ad[j]
for j in range(I - 1):
    A[j * n:(j + 1) * n, (j + 1) * n:(j + 2) * n] = Au[j]
    A[(j + 1) * n:(j + 2) * n, j * n:(j + 1) * n] = Al[j]
x = np.linalg.solve(A, np.r_[f, np.zeros((I - 1) * n)]).reshape(I, n)
print("gpu blocks: cond", "%.2e" % np.linalg.cond(A), "diag conds", ["%.1e" % np.linalg.cond(a) for a in Ad])
print("numpy dense vs thomas", np.linalg.norm(x - eo) / np.linalg.norm(eo), "gpu bcr vs numpy",
      np.linalg.norm(eg - x) / np.linalg.norm(x))
# Thomas pivots' conditions (reference order)
At = Ad[0]
for j in range(1, I):
    At = Ad[j] - Al[j - 1] @ np.linalg.solve(At, Au[j - 1])
    print("thomas pivot", j, "cond %.1e" % np.linalg.cond(At))
