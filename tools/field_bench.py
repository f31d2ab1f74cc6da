"""Field evaluation on a dense grid after a config solve (paper: 446 s for a
1000 x 1000 grid on the CPU).
usage: python tools/field_bench.py [cfg] [nx] [ny] [nif]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nx = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
ny = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
nif = int(sys.argv[4]) if len(sys.argv) > 4 else None
st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
s = Solver()
s.build_geometry(st, num)
s.make_problem(om, th, K)
s.solve()
info = s.problem_info()
xs = np.linspace(-0.5, 0.5, nx, endpoint=False) + 0.5 / nx
ys = np.linspace(info["y_D"] - 0.5, info["y_U"] + 0.5, ny)
X, Y = np.meshgrid(xs, ys)
pts = np.stack([X.ravel(), Y.ravel()], axis=1)
s.evaluate_field(pts[:1000])  # warm-up
s.prof_reset()
s.prof_enable(True)
t0 = time.perf_counter()
f = s.evaluate_field(pts)
wall = time.perf_counter() - t0
s.prof_enable(False)
st_ = s.prof_stats().get("field", {})
print(json.dumps({"config": cfg, "points": len(pts), "wall_s": wall, "kernel_ms": st_.get("ms"),
                  "kernel_evals": st_.get("units"),
                  "evals_per_s": st_.get("units", 0) / (st_["ms"] * 1e-3) if st_.get("ms") else None,
                  "finite": bool(np.isfinite(f["u_total"]).all())}))
