"""Per-layer least-squares residuals of the periodization (solution()['lsq_residual'])
for one config prefix; prints max and the worst layers (QPS_* env selects variants)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1410_5003_b200 import Solver, configs
cfg = int(sys.argv[1]); nif = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
s = Solver(); s.build_geometry(st, num); s.make_problem(om, th, K); s.solve()
sol = s.solution(); l = sol["lsq_residual"]
print("max lsq", l.max(), "worst", np.argsort(l)[-5:], l[np.argsort(l)[-5:]], "R", s.reflection_transmission()["R"])
