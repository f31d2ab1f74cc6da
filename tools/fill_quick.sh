#!/bin/bash
# Quick FP64-rate check of the pair_fill kernels (config 4) under ncu:
# per launch and total duration, SASS FP64 flop rate (DFMA = 2, DMUL = DADD = 1)
# against the counters' peak, FP64 pipe utilisation, occupancy.
set -e
OUT=${1:-gpurun_out/fill_quick.csv}
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained,sm__cycles_elapsed.avg,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread
ncu --metrics $M --clock-control none -k regex:pair_fill -c 6 --csv python tools/run_config.py 4 - 1 2>/dev/null > $OUT
python - $OUT <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[h.index("ID")], {"name": r[h.index("Kernel Name")]})
    d[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
tt = tf = tp = 0.0
for d in L.values():
    fl = 2 * d["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] + d["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"] + d["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
    pk = 2 * d["sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained"] * d["sm__cycles_elapsed.avg"]
    t = d["gpu__time_duration.sum"]
    tt += t; tf += fl; tp += pk
    print(f"{d['name'][:40]:40s} grid {int(d['launch__grid_size']):7d} regs {int(d['launch__registers_per_thread'])} {t/1e6:7.3f} ms  frac {fl/pk:.4f}  pipe {d['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']:.1f}%  warps {d['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f}%")
print(f"TOTAL pair_fill {tt/1e6:.3f} ms  fp64 frac {tf/tp:.4f}")
PY
