"""Alpha-grouped sweep diagnostic: Bragg amplitudes of the GPU sweep (grouped and independent modes) against the oracle on a config-5 prefix at alpha-grid angles."""
import sys, os, numpy as np, json
sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st, num, om, th0, K, _ = configs.config(5, n_interfaces=6)
def run(s, mode, th):
    s.build_geometry(st, num); s.make_problem(om, th0, K)
    r = s.sweep(th, K, mode=mode)
    return np.concatenate([r["aU"], r["aD"]], 1)
g = Solver(device=0); g.build_geometry(st, num); g.make_problem(om, th0, K)
th, grp = g.plan_sweep(3, -np.pi + 0.1, -0.1); th = list(th[:9])
o = Solver(lib="oracle/_ref/libqpscat_ref.so")
res = {"oracle_m0": run(o, 0, th), "oracle_m1": run(o, 1, th), "gpu_m0": run(g, 0, th), "gpu_m1": run(g, 1, th)}
# gpu one-shot solve per angle
one = []
for t in th:
    g.build_geometry(st, num); g.make_problem(om, t, K); g.solve(); s = g.solution(); one.append(np.concatenate([s["aU"], s["aD"]]))
res["gpu_solve"] = np.array(one)
one = []
for t in th:
    o.build_geometry(st, num); o.make_problem(om, t, K); o.solve(); s = o.solution(); one.append(np.concatenate([s["aU"], s["aD"]]))
res["oracle_solve"] = np.array(one)
ref = res["oracle_m0"]
for k, v in res.items():
    print(k, ["%.1e" % x for x in np.linalg.norm(v - ref, axis=1) / np.linalg.norm(ref, axis=1)])
print("diag", g.solver_diagnostics())
