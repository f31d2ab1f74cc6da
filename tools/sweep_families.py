"""Kernel-family times of one config-5 accelerated sweep (200 angles).
usage: python tools/sweep_families.py"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

st, num, om, th, K, _ = configs.config(5)
thetas = configs.sweep_angles(200)
g = Solver(device=0)
g.build_geometry(st, num)
g.make_problem(om, th, K)
g.sweep(thetas[:2], K, mode=0)
g.prof_reset()
g.prof_enable(True)
t0 = time.perf_counter()
g.sweep(thetas, K, mode=0)
dt = time.perf_counter() - t0
g.prof_enable(False)
st_ = g.prof_stats()
print(json.dumps({"s": dt, "phases": g.phase_times(),
                  "families_ms": {k: round(v["ms"], 1) for k, v in sorted(st_.items(), key=lambda kv: -kv[1]["ms"])[:25]}},
                 indent=0))
