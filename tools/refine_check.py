"""Iterative refinement of the block cyclic reduction: Bragg amplitudes of the
GPU against the oracle with 0 / 1 / 2 refinement steps, on the alpha-grid
angles of a config-5 prefix (grouped sweep, mode 0, and one solve per angle,
mode 1) and on a config-4 prefix (one-shot solve).  Prints the relative
errors, the oracle's 1-ulp(omega, theta) floor and the relative residuals.
usage: python tools/refine_check.py [I5=6] [n_alpha=3] [I4=50]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

ORACLE = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libqpscat_ref.so")
I5 = int(sys.argv[1]) if len(sys.argv) > 1 else 6
NA = int(sys.argv[2]) if len(sys.argv) > 2 else 3
I4 = int(sys.argv[3]) if len(sys.argv) > 3 else 50


def setup(s, cfg, nif, du=0):
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
    if du:
        om = float(np.nextafter(om, np.inf if du > 0 else -np.inf))
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    return K, th


def amps(r):
    return np.concatenate([r["aU"], r["aD"]], axis=1)


g, o = Solver(device=0), Solver(lib=ORACLE)
K, _ = setup(g, 5, I5)
th, grp = g.plan_sweep(NA, -np.pi + 0.1, -0.1)
th = list(th)
setup(o, 5, I5)
ao = amps(o.sweep(th, K, mode=0))
floor = np.zeros(len(th))
for du, dt in [(1, 0), (-1, 0), (0, 1), (0, -1)]:
    setup(o, 5, I5, du)
    t2 = [float(np.nextafter(t, np.inf if dt > 0 else -np.inf)) if dt else t for t in th]
    a1 = amps(o.sweep(t2, K, mode=0))
    floor = np.maximum(floor, np.linalg.norm(a1 - ao, axis=1) / np.linalg.norm(ao, axis=1))
print(f"cfg5 I={I5}: {len(th)} alpha-grid angles, floor max {floor.max():.2e}")
for mode in (0, 1):
    for steps in (0, 1, 2):
        setup(g, 5, I5)
        g.set_refine(steps)
        ag = amps(g.sweep(th, K, mode=mode))
        err = np.linalg.norm(ag - ao, axis=1) / np.linalg.norm(ao, axis=1)
        ratio = err / np.maximum(floor, 1e-300)
        print(f"  mode {mode} refine {steps}: err max {err.max():.2e}  worst err/floor {ratio.max():.1f}  "
              f"angles > 3x floor {int((ratio > 3).sum())}")
g.set_refine(-1)
K4, th4 = setup(o, 4, I4)
o.solve()
so = o.solution()
a4 = np.concatenate([so["aU"], so["aD"]])
for steps in (0, 1, 2):
    setup(g, 4, I4)
    g.set_refine(steps)
    g.solve()
    sg = g.solution()
    e = np.linalg.norm(np.concatenate([sg["aU"], sg["aD"]]) - a4) / np.linalg.norm(a4)
    d = g.solver_diagnostics()
    print(f"cfg4 I={I4} refine {steps}: bragg_rel {e:.2e}  phases {g.phase_times()['solve_ms']:.1f} ms solve  "
          f"res0 {d['refine_res0']:.2e} res1 {d['refine_res1']:.2e}")
