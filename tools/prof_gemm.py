"""Small driver for ncu captures: a 64-layer cfg4 solve."""
import sys
sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st, num, om, th, K, _ = configs.config(4, n_interfaces=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
s = Solver()
s.build_geometry(st, num)
s.make_problem(om, th, K)
s.solve()
print("ok", s.phase_times())
