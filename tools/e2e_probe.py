"""End-to-end split of one config-4 call sequence through the public API: geometry, problem, solve (host and device time), solution readback."""
import time, sys
sys.path.insert(0, '.')
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st, num, om, th, K, meta = configs.config(4)
s = Solver()
sol = None
for r in range(4):
    t0 = time.perf_counter(); s.build_geometry(st, num); t1 = time.perf_counter()
    s.make_problem(om, th, K); t2 = time.perf_counter()
    s.solve(); t3 = time.perf_counter()
    sol = s.solution(out=sol); t4 = time.perf_counter()
    print(f"geom {1e3*(t1-t0):.1f} prob {1e3*(t2-t1):.1f} solve {1e3*(t3-t2):.1f} (device {s.phase_times()['total_ms']:.1f}) solution {1e3*(t4-t3):.1f} total {1e3*(t4-t0):.1f}", flush=True)
