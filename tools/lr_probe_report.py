"""Report how the block solve ran (path, sample rank, a-posteriori probe) for
config 4 and config-5 sweeps; run with QPS_LR_TRACE=1 for per-compression lines.
usage: python tools/lr_probe_report.py"""
import json
import sys

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

g = Solver(device=0)
for cfg, nif in [(4, None), (4, 50), (5, 3), (5, None), (2, None)]:
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
    g.build_geometry(st, num)
    g.make_problem(om, th, K)
    g.solve()
    d = g.solver_diagnostics()
    print(json.dumps({"cfg": cfg, "I": len(st.interfaces), **d, "total_ms": g.phase_times()["total_ms"]}), flush=True)
st, num, om, th, K, _ = configs.config(5, n_interfaces=3)
g.build_geometry(st, num)
g.make_problem(om, th, K)
thetas = configs.sweep_angles(200)[::40]
for mode in (0, 1):
    r = g.sweep(thetas, K, mode=mode)
    print("sweep mode", mode, g.solver_diagnostics(), flush=True)
