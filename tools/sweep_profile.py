"""Kernel-family breakdown of the config-5 accelerated sweep (QPS_PROF_PHASES=1)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
st, num, om, th, K, _ = configs.config(5)
s = Solver()
s.build_geometry(st, num)
s.make_problem(om, th, K)
thetas = configs.sweep_angles(200)[:n]
s.sweep(thetas, K)
s.prof_reset()
s.prof_enable(True)
s.sweep(thetas, K)
s.prof_enable(False)
print("phases", {k: round(v, 1) for k, v in s.phase_times().items()})
st_ = s.prof_stats()
tot = sum(v["ms"] for v in st_.values())
for k, v in sorted(st_.items(), key=lambda kv: -kv[1]["ms"])[:22]:
    print(f"  {k:24s} {v['launches']:6d} {v['ms']:9.2f} ms {100 * v['ms'] / tot:5.1f}%")
