"""Feed the oracle's periodized blocks (Ap_diag/super/sub, f) at one angle to
the GPU block solve (bypassing fill and Schur) and compare eta against the
reference's block Thomas on the same blocks, with condition numbers.
usage: python tools/bcr_on_oracle_blocks.py [angle_index ...]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

st, num, om, th0, K, _ = configs.config(5, n_interfaces=6)
o = Solver(lib="oracle/_ref/libqpscat_ref.so")
g = Solver(device=0)
o.build_geometry(st, num)
o.make_problem(om, th0, K)
th, _ = o.plan_sweep(3, -np.pi + 0.1, -0.1)
for ia in [int(a) for a in sys.argv[1:]] or [0, 1, 3]:
    o.build_geometry(st, num)
    o.make_problem(om, th[ia], K)
    o.precompute_shift_blocks()
    o.assemble_system()
    o.schur_complement()
    I = 6
    Ad = [o.download_block("Ap_diag", j) for j in range(I)]
    Au = [o.download_block("Ap_super", j) for j in range(I - 1)]
    Al = [o.download_block("Ap_sub", j) for j in range(I - 1)]
    f = o.download_block("f", 0).ravel()
    n = Ad[0].shape[0]
    f = np.concatenate([f, np.zeros(n - len(f))]) if len(f) < n else f
    eo = o.block_lu_solve_blocks(Ad, Au, Al, f)
    for tag, pad in [("n=300", 0), ("n=304 (padded like the solver)", 4)]:
        m = n + pad
        P = lambda a: np.pad(a, ((0, pad), (0, pad)))  # noqa: E731
        Adp = [P(a) + (np.diag(np.r_[np.zeros(n), np.ones(pad)]) if pad else 0) for a in Ad]
        eg = g.block_lu_solve_blocks(Adp, [P(a) for a in Au], [P(a) for a in Al], np.r_[f, np.zeros(pad)])
        eg = np.array(eg)[:, :n]
        d = g.solver_diagnostics()
        print(f"angle {ia} theta {th[ia]:.6f} {tag}: eta rel diff {np.linalg.norm(eg - eo) / np.linalg.norm(eo):.2e}"
              f" block0 {np.linalg.norm(eg[0] - eo[0]) / np.linalg.norm(eo[0]):.2e} path {d['bcr_path']}", flush=True)
