"""Low-rank vs dense cyclic reduction on the same problem: Bragg amplitudes,
R, T, flux and the phase times of both (run once with each QPS_BCR setting in
separate processes; this script runs the current setting and prints JSON)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nif = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
out = sys.argv[3] if len(sys.argv) > 3 else None
st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
s = Solver()
s.build_geometry(st, num)
s.make_problem(om, th, K)
for _ in range(3):
    s.solve()
sol, rt = s.solution(), s.reflection_transmission()
a = np.concatenate([sol["aU"], sol["aD"]])
res = {"bcr": os.environ.get("QPS_BCR", "lowrank"), "phases": s.phase_times(), "R": rt["R"], "T": rt["T"],
       "flux": rt["flux_error"]}
if out:
    np.save(out, a)
print(json.dumps(res))
