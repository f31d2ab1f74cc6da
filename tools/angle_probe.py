"""One-shot GPU solve vs the oracle at alpha-grid angles of a config-5 prefix
(tools/alpha_sweep_diag.py found the standard path off at some angles).
usage: [env QPS_*=...] python tools/angle_probe.py"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

st, num, om, th0, K, _ = configs.config(5, n_interfaces=6)
g = Solver(device=0)
o = Solver(lib="oracle/_ref/libqpscat_ref.so")
g.build_geometry(st, num)
g.make_problem(om, th0, K)
th, grp = g.plan_sweep(3, -np.pi + 0.1, -0.1)
for t in th[:4]:
    out = []
    for s in (g, o):
        s.build_geometry(st, num)
        s.make_problem(om, t, K)
        s.solve()
        sol = s.solution()
        out.append((np.concatenate([sol["aU"], sol["aD"]]), sol["lsq_residual"], s.reflection_transmission()["flux_error"]))
    e = np.linalg.norm(out[0][0] - out[1][0]) / np.linalg.norm(out[1][0])
    print(f"theta {t:.6f} err {e:.2e} flux gpu {out[0][2]:.1e} oracle {out[1][2]:.1e} lsq_corner gpu "
          f"{out[0][1][0]:.1e},{out[0][1][-1]:.1e} oracle {out[1][1][0]:.1e},{out[1][1][-1]:.1e}", flush=True)
