"""Run one BASELINE config on the product library and print phase times."""
import sys
import time
sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver

cfg = int(sys.argv[1])
nif = int(sys.argv[2]) if len(sys.argv) > 2 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
st, num, om, th, K, meta = configs.config(cfg, n_interfaces=nif)
s = Solver()
t0 = time.time()
s.build_geometry(st, num)
s.make_problem(om, th, K)
print("geometry", time.time() - t0, flush=True)
for r in range(reps):
    t0 = time.time()
    s.solve()
    t1 = time.time()
    rt = s.reflection_transmission()
    print(f"rep {r}: wall {t1 - t0:.3f}s phases {s.phase_times()} R {rt['R']:.12f} T {rt['T']:.12f} flux {rt['flux_error']:.3e} evals {s.fill_evals()}", flush=True)
