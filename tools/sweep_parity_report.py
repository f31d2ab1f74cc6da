"""Per-angle Bragg-amplitude parity of the GPU sweep and the one-shot GPU solve
against the oracle, with the oracle's own 1-ulp(omega) noise floor."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402
from conftest import ORACLE_LIB  # noqa: E402

nif = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
th = configs.sweep_angles(200)
thetas = [th[i] for i in np.linspace(0, 199, n).astype(int)]
st, num, om, th0, K, _ = configs.config(5, n_interfaces=nif)
g, o = Solver(), Solver(lib=ORACLE_LIB)


def sw(s, omega):
    s.build_geometry(st, num)
    s.make_problem(omega, th0, K)
    return s.sweep(thetas, K, mode=0)


rg, ro = sw(g, om), sw(o, om)
r1 = sw(o, float(np.nextafter(om, 2 * om)))
for a, t in enumerate(thetas):
    v = lambda r: np.concatenate([r["aU"][a], r["aD"][a]])  # noqa: E731
    ao = v(ro)
    g.build_geometry(st, num)
    g.make_problem(om, t, K)
    g.solve()
    s = g.solution()
    af = np.concatenate([s["aU"], s["aD"]])
    nr = np.linalg.norm(ao)
    print(f"theta={t:+.4f} sweep_err={np.linalg.norm(v(rg)-ao)/nr:.2e} fused_err={np.linalg.norm(af-ao)/nr:.2e} "
          f"floor={np.linalg.norm(v(r1)-ao)/nr:.2e} dR={abs(rg['R'][a]-ro['R'][a]):.2e} "
          f"floorR={abs(r1['R'][a]-ro['R'][a]):.2e} fe={ro['flux_error'][a]:.1e}")
