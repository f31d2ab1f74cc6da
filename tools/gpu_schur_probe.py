"""Config 1: the GPU's periodization pieces (Qp, Cp, Schur complements) against the oracle's, block by block."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st, num, om, th, K, meta = configs.config(1)
o = Solver(lib="oracle/_ref/libqpscat_ref.so")
o.build_geometry(st, num); o.make_problem(om, th, K); o.precompute_shift_blocks(); o.assemble_system()
g = Solver()
g.build_geometry(st, num); g.make_problem(om, th, K); g.precompute_shift_blocks(); g.assemble_system()
for nm in ["Qp_first", "Qp_last"]:
    Q = o.download_block(nm); R = o.download_block(nm.replace("Qp", "Cp"))
    for thr in [1e-14, 1e-13, 1e-12, 1e-11, 1e-10]:
        o.set_qsolve_threshold(thr); g.set_qsolve_threshold(thr)
        Xo, ro = o.qsolve(Q, R); Xg, rg = g.qsolve(Q, R)
        print(nm, thr, "rank", ro, rg, "maxX", np.abs(Xo).max(), np.abs(Xg).max(), "res", np.linalg.norm(Q@Xo-R)/np.linalg.norm(R), np.linalg.norm(Q@Xg-R)/np.linalg.norm(R))
    sv = np.linalg.svd(Q, compute_uv=False); print("sv", sv[0], sv[-12:] / sv[0])
