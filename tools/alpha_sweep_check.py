"""Alpha-grouped sweep accuracy report: GPU grouped (mode 0) vs GPU
independent (mode 1) vs the oracle's grouped composition, with the oracle's
1-ulp floor as the max over omega/theta +-1 ulp.  usage: python tools/alpha_sweep_check.py [cfg nif n_alpha count]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

cfg, nif, na, cnt = [int(a) for a in sys.argv[1:5]] if len(sys.argv) > 4 else (5, 6, 3, 9)
ORACLE = "oracle/_ref/libqpscat_ref.so"


def run(s, om, th_list, K, mode, st, num, th0):
    s.build_geometry(st, num)
    s.make_problem(om, th0, K)
    r = s.sweep(th_list, K, mode=mode)
    return np.concatenate([r["aU"], r["aD"]], 1), r["flux_error"]


st, num, om, th0, K, _ = configs.config(cfg, n_interfaces=nif)
g = Solver(device=0)
g.build_geometry(st, num)
g.make_problem(om, th0, K)
th, grp = g.plan_sweep(na, -np.pi + 0.1, -0.1)
th = th[:cnt]
ag, fg = run(g, om, th, K, 0, st, num, th0)
ai, fi = run(g, om, th, K, 1, st, num, th0)
o = Solver(lib=ORACLE)
ao, fo = run(o, om, th, K, 0, st, num, th0)
fl = np.zeros(len(th))
for o2, t2 in [(np.nextafter(om, np.inf), th), (np.nextafter(om, -np.inf), th),
               (om, np.nextafter(th, np.inf)), (om, np.nextafter(th, -np.inf))]:
    a1, _ = run(o, float(o2), list(t2), K, 0, st, num, th0)
    fl = np.maximum(fl, np.linalg.norm(a1 - ao, axis=1) / np.linalg.norm(ao, axis=1))
rel = lambda a, b: np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)  # noqa: E731
print(json.dumps({"grouped_vs_oracle": rel(ag, ao).tolist(), "independent_vs_oracle": rel(ai, ao).tolist(),
                  "grouped_vs_independent": rel(ag, ai).tolist(), "floor4": fl.tolist(),
                  "flux_gpu_grouped": fg.tolist(), "flux_oracle": fo.tolist()}, indent=1))
