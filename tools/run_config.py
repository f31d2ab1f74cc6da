"""Run one BASELINE config on the product library; print phase times and the
per-kernel-family breakdown.  Usage: python tools/run_config.py CFG [I] [reps]"""
import sys
import time
sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver

cfg = int(sys.argv[1])
nif = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
st, num, om, th, K, meta = configs.config(cfg, n_interfaces=nif)
s = Solver()
peaks = s.fp64_peaks()
print("peaks", peaks)
t0 = time.time()
s.build_geometry(st, num)
s.make_problem(om, th, K)
print("geometry", time.time() - t0, flush=True)
for r in range(reps):
    if r == reps - 1:
        s.prof_reset()
        s.prof_enable(True)
    t0 = time.time()
    s.solve()
    t1 = time.time()
    rt = s.reflection_transmission()
    print(f"rep {r}: wall {t1 - t0:.3f}s phases {s.phase_times()} R {rt['R']:.12f} flux {rt['flux_error']:.3e}", flush=True)
s.prof_enable(False)
stats = s.prof_stats()
tot = sum(v["ms"] for v in stats.values())
for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["ms"]):
    tf = v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["ms"] else 0
    gb = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] else 0
    print(f"  {k:14s} launches {v['launches']:7d}  {v['ms']:9.2f} ms ({100 * v['ms'] / tot:5.1f}%)  {tf:7.2f} TF/s  {gb:8.1f} GB/s")
