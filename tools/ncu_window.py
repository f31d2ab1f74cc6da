"""Aggregate an ncu launch list (CSV from --csv --metrics ...) over every
captured launch: total duration, executed FP64 flops (DMMA.8x8x4 = 512 flops,
DFMA = 2, DMUL = DADD = 1) and their rate against a given peak.

usage: python tools/ncu_window.py launches.csv PEAK_TFLOPS [nominal_flops]
Metrics expected: gpu__time_duration.sum, sm__inst_executed_pipe_tensor_subpipe_dmma.sum,
smsp__sass_thread_inst_executed_op_dfma_pred_on.sum, ..._dmul_..., ..._dadd_...,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active."""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[h.index("ID")], {"name": r[h.index("Kernel Name")]})
    try:
        d[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    except ValueError:
        pass
peak = float(sys.argv[2])
t = fl = tw = 0.0
fam = collections.defaultdict(lambda: [0, 0.0])
for d in L.values():
    dt = d.get("gpu__time_duration.sum", 0.0) * 1e-9
    f = 512.0 * d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0) \
        + 2.0 * d.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0) \
        + d.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0) \
        + d.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
    t += dt
    fl += f
    tw += dt * d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
    k = d["name"].split("(")[0].split("::")[-1][:40]
    fam[k][0] += 1
    fam[k][1] += dt
out = {"launches": len(L), "ms": t * 1e3, "executed_fp64_flops": fl, "executed_tflops": fl / t / 1e12,
       "frac_of_peak": fl / t / 1e12 / peak, "tensor_pipe_active_pct_time_weighted": tw / t,
       "families_ms": {k: round(v[1] * 1e3, 3) for k, v in sorted(fam.items(), key=lambda kv: -kv[1][1])}}
if len(sys.argv) > 3:
    nom = float(sys.argv[3])
    out["nominal_flops"] = nom
    out["nominal_tflops"] = nom / t / 1e12
    out["nominal_frac_of_peak"] = nom / t / 1e12 / peak
print(json.dumps(out, indent=1))
