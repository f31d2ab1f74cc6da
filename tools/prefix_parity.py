"""Bragg-amplitude parity of the GPU against the oracle on config-4 prefixes
(the full 1000-layer oracle needs ~130 GB of host RAM and ~4 min on 16
cores): relative 2-norm error of [aU; aD], |dR|, |dT|, and the oracle's own
1-ulp(omega) floor.  usage: python tools/prefix_parity.py [I ...]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402
from conftest import ORACLE_LIB  # noqa: E402


def run(s, st, num, om, th, K):
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    t0 = time.perf_counter()
    s.solve()
    dt = time.perf_counter() - t0
    sol, rt = s.solution(), s.reflection_transmission()
    return np.concatenate([sol["aU"], sol["aD"]]), rt["R"], rt["T"], rt["flux_error"], dt


Is = [int(a) for a in sys.argv[1:]] or [50, 200]
cfg = int(os.environ.get("QPS_CFG", "4"))
for I in Is:
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=I)
    g = run(Solver(), st, num, om, th, K)
    o_s = Solver(lib=ORACLE_LIB)
    o = run(o_s, st, num, om, th, K)
    o1 = run(o_s, st, num, float(np.nextafter(om, 2 * om)), th, K)
    nr = np.linalg.norm(o[0])
    print(json.dumps({"config": cfg, "I": I, "bragg_rel_err": float(np.linalg.norm(g[0] - o[0]) / nr),
                      "oracle_floor": float(np.linalg.norm(o1[0] - o[0]) / nr),
                      "dR": abs(g[1] - o[1]), "dT": abs(g[2] - o[2]),
                      "floor_RT": max(abs(o1[1] - o[1]), abs(o1[2] - o[2])),
                      "flux_gpu": g[3], "flux_oracle": o[3], "gpu_s": g[4], "oracle_s": o[4]}), flush=True)
