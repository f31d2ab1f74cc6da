"""Summarise an ncu --set full capture of pair_fill_kernel: achieved FP64
FLOP/s from the SASS op counters (DFMA = 2, DMUL = DADD = 1) against the
FP64 peak of the same counters, FP64 pipe utilisation, DRAM traffic.
usage: python tools/ncu_fill_rate.py gpurun_out/<capture>.ncu-rep [evals]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
evals = float(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
for r in rows[2:]:
    d = dict(zip(rows[0], r))
    hz = float(d["sm__cycles_elapsed.avg.per_second"])
    hz = hz * 1e9 if hz < 1e3 else hz
    per_cyc = (2 * float(d["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed"])
               + float(d["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"])
               + float(d["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed"]))
    peak_cyc = 2 * float(d["sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained"])
    t_ms = float(d["gpu__time_duration.sum"])
    rw = float(d["dram__bytes_read.sum"]) * (1e6 if False else 1)
    res.append({"kernel": d["Kernel Name"][:60], "duration_ms": t_ms,
                "fp64_tflops_ncu": per_cyc * hz / 1e12, "fp64_peak_tflops_ncu": peak_cyc * hz / 1e12,
                "fp64_frac_of_peak": per_cyc / peak_cyc,
                "fp64_pipe_pct": float(d["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]),
                "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
                "registers": int(float(d["launch__registers_per_thread"])),
                "evals_per_s": (evals / (t_ms * 1e-3)) if evals else None})
if len(res) > 1:  # all captured kinds together: total flops over total time
    tt = sum(r["duration_ms"] for r in res)
    fl = sum(r["fp64_tflops_ncu"] * r["duration_ms"] for r in res)
    pk = sum(r["fp64_peak_tflops_ncu"] * r["duration_ms"] for r in res)
    res.append({"kernel": "all captured launches", "duration_ms": tt, "fp64_tflops_ncu": fl / tt,
                "fp64_peak_tflops_ncu": pk / tt, "fp64_frac_of_peak": fl / pk,
                "fp64_pipe_pct": sum(r["fp64_pipe_pct"] * r["duration_ms"] for r in res) / tt,
                "evals_per_s": (evals / (tt * 1e-3)) if evals else None})
print(json.dumps(res, indent=1))
