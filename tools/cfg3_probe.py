"""Config-3 prefixes on the oracle or the GPU: which interface counts solve and which raise SingularityError. usage: python tools/cfg3_probe.py oracle|gpu I..."""
import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1410_5003_b200 import Solver, configs
from conftest import ORACLE_LIB
which = sys.argv[1]
for I in [int(a) for a in sys.argv[2:]]:
    st, num, om, th, K, _ = configs.config(3, n_interfaces=I)
    s = Solver(lib=ORACLE_LIB) if which == "oracle" else Solver()
    s.build_geometry(st, num); s.make_problem(om, th, K)
    try:
        s.solve(); print(which, I, "ok", s.reflection_transmission()["flux_error"], flush=True)
    except Exception as e:
        print(which, I, "ERR", type(e).__name__, e, flush=True)
