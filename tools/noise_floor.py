"""Noise-floor protocol: run the CPU oracle nominally and with
(a) every k_i perturbed by 1 ulp and (b) every interface node perturbed by
1 ulp in the offset, and with (c) a different BLAS/OpenMP thread count;
report the relative changes of the physics outputs ([aU; aD], R, T) and of
the raw densities eta.  Usage: python tools/noise_floor.py [cfg ...]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

ORACLE = "oracle/_ref/libqpscat_ref.so"


def solve(st, num, om, th, K, threads=None):
    s = Solver(lib=ORACLE)
    if threads:
        s.set_num_threads(threads)
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    s.solve()
    sol, rt = s.solution(), s.reflection_transmission()
    s.close()
    return np.concatenate([sol["aU"], sol["aD"]]), rt["R"], rt["T"], sol["eta_flat"], rt["flux_error"]


def floor(cfg, nif=None):
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
    a0, R0, T0, e0, f0 = solve(st, num, om, th, K, threads=8)
    out = {"cfg": cfg, "I": len(st.interfaces), "flux_error": f0}
    # (a) 1-ulp perturbation of omega (hence every k_i)
    a1, R1, T1, e1, _ = solve(st, num, np.nextafter(om, 2 * om), th, K, threads=8)
    # (b) 1-ulp perturbation of every interface offset
    import copy
    st2 = copy.deepcopy(st)
    for sp in st2.interfaces:
        sp.offset = float(np.nextafter(sp.offset, 1.0)) if sp.offset != 0 else 5e-324
    a2, R2, T2, e2, _ = solve(st2, num, om, th, K, threads=8)
    # (c) thread count
    a3, R3, T3, e3, _ = solve(st, num, om, th, K, threads=1)
    for tag, (a, R, T, e) in {"ulp_k": (a1, R1, T1, e1), "ulp_geometry": (a2, R2, T2, e2),
                               "threads_1_vs_8": (a3, R3, T3, e3)}.items():
        out[tag] = {"bragg_rel": float(np.linalg.norm(a - a0) / np.linalg.norm(a0)), "dR": abs(R - R0),
                    "dT": abs(T - T0), "eta_rel": float(np.linalg.norm(e - e0) / np.linalg.norm(e0))}
    return out


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2]
    res = [floor(c, 6 if c == 3 else None) for c in cfgs]
    print(json.dumps(res, indent=1))
