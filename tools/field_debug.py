"""Per-region field differences GPU vs oracle (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402
from conftest import ORACLE_LIB  # noqa: E402
from test_gpu_field import grid  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
st, num, om, th, K, _ = configs.config(cfg)
out = {}
for name, s in (("gpu", Solver()), ("ref", Solver(lib=ORACLE_LIB))):
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    s.solve()
    pts = grid(s, st)
    out[name] = s.evaluate_field(pts)
g, o = out["gpu"], out["ref"]
for r in (0, 1, 2):
    m = g["region"] == r
    if not m.any():
        continue
    e = np.abs(g["u_scattered"][m] - o["u_scattered"][m])
    i = np.argmax(e)
    print(f"region {r}: n={m.sum()} max|u_ref|={np.abs(o['u_scattered'][m]).max():.3e} max err={e.max():.3e} "
          f"at {pts[m][i]} gpu={g['u_scattered'][m][i]:.6e} ref={o['u_scattered'][m][i]:.6e}")
# error vs distance to the nearest interface (layer points)
from test_gpu_field import interface_y  # noqa: E402
m = g["region"] == 1
P = pts[m]
dist = np.min(np.stack([np.abs(P[:, 1] - interface_y(sp, P[:, 0])) for sp in st.interfaces]), axis=0)
e = np.abs(g["u_scattered"][m] - o["u_scattered"][m])
for lo, hi in ((0.1, 0.15), (0.15, 0.2), (0.2, 0.3), (0.3, 0.5), (0.5, 10)):
    sel = (dist >= lo) & (dist < hi)
    if sel.any():
        print(f"dist [{lo},{hi}): n={sel.sum()} max err {e[sel].max():.2e}")
