"""Config-5 sweep time with 0 and 1 refinement steps per angle (the cost of the sweeps' default refinement)."""
import sys, time, math
sys.path.insert(0, '.')
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st, num, om, th, K, meta = configs.config(5)
g = Solver(device=0)
g.build_geometry(st, num); g.make_problem(om, th, K)
ta, grp = g.plan_sweep(40, -math.pi + 0.1, -0.1)
thetas = configs.sweep_angles(200)
g.sweep(list(ta)[:8], K, mode=0)
for steps in (0, 1, 0, 1):
    g.set_refine(steps)
    for name, angs in (("alpha-grid", list(ta)), ("uniform200", thetas)):
        g.build_geometry(st, num); g.make_problem(om, th, K)
        t0 = time.perf_counter(); r = g.sweep(angs, K, mode=0); dt = time.perf_counter() - t0
        print(f"refine {steps} {name}: {dt:.3f} s  phases {g.phase_times()}", flush=True)
