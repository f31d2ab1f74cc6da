"""GPU one-shot solve vs the oracle over many angles of a config prefix, with
the oracle's 1-ulp(omega) floor: how often the GPU exceeds 3x floor.
usage: python tools/angle_scan.py cfg nif n_angles"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

cfg, nif, na = (int(a) for a in sys.argv[1:4])
st, num, om, th0, K, _ = configs.config(cfg, n_interfaces=nif)
g = Solver(device=0)
o = Solver(lib="oracle/_ref/libqpscat_ref.so")
ths = np.linspace(-np.pi + 0.1, -0.1, na)


def amp(s, om_, t):
    s.build_geometry(st, num)
    s.make_problem(om_, t, K)
    s.solve()
    sol = s.solution()
    return np.concatenate([sol["aU"], sol["aD"]])


bad = 0
ratios = []
for t in ths:
    ag, ao, a1 = amp(g, om, t), amp(o, om, t), amp(o, float(np.nextafter(om, np.inf)), t)
    e = np.linalg.norm(ag - ao) / np.linalg.norm(ao)
    fl = np.linalg.norm(a1 - ao) / np.linalg.norm(ao)
    ratios.append(e / max(fl, 1e-16))
    if e > max(1e-9, 3 * fl):
        bad += 1
        print(f"theta {t:.5f} err {e:.2e} floor {fl:.2e}", flush=True)
print(f"cfg{cfg} I={nif}: {bad}/{na} angles above max(1e-9, 3 x floor); median err/floor {np.median(ratios):.2f}")
