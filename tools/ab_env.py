"""A/B of environment knobs on the config-4 one-shot solve: for each KEY=VAL[,KEY=VAL] argument, a fresh process
solves config 4 (2 warm-up + 5 timed solves) and prints the median device time and a hash of the solution
(densities, aU, aD), so that scheduling-only knobs can be checked for bitwise-identical results.

    python tools/ab_env.py "" QPS_SKETCH_EARLY=0 QPS_SAMPLE_PRIO=hi
"""
import hashlib
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ".")
    import numpy as np
    from paper_1410_5003_b200 import configs
    from paper_1410_5003_b200.qpscat import Solver
    st, num, om, th, K, meta = configs.config(4)
    s = Solver()
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    for _ in range(2):
        s.solve()
    t = []
    for _ in range(5):
        s.solve()
        t.append(s.phase_times()["total_ms"])
    sol = s.solution()
    h = hashlib.sha1()
    for k in ("eta_flat", "aU", "aD"):
        h.update(np.ascontiguousarray(sol[k]).tobytes())
    print(json.dumps({"ms": sorted(t)[2], "all": [round(x, 2) for x in t], "hash": h.hexdigest()[:16],
                      "phases": s.phase_times()}))
    sys.exit(0)

for arg in sys.argv[1:]:
    env = dict(os.environ)
    for kv in filter(None, arg.split(",")):
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
    print(f"[{arg or 'default'}] {line}", flush=True)
