"""DRAM traffic of the level-0 LU batch's GEMMs (family lu_gemm) against their
algorithmic bytes, for profiles/ncu_summary.json's lu_gemm entry (bench.py's
roofline.traffic).

Inputs: an ncu launch list over the NVTX window bcr_level0 with
dram__bytes_read.sum and dram__bytes_write.sum, and the library's
QPS_TRACE_GEMM stderr lines of the same run (one per zgemm_batched call, in
launch order; the window's GEMM launches are exactly the lu_gemm calls).
Algorithmic bytes per launch: 16 (M K + K N + 2 M N) per task and segment
(A and B read once, C read and written).
usage: python tools/lu_gemm_traffic.py window.csv trace.err"""
import collections
import csv
import json
import re
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
gl = [d for d in L.values() if "zgemm3m" in d["name"]]
sh = [l for l in open(sys.argv[2]) if l.startswith("gemm lu_gemm ")]
assert len(gl) == len(sh), (len(gl), len(sh))
dram = alg = ns = 0.0
for d, l in zip(gl, sh):
    m = re.match(r"gemm (\S+) M=(\d+) N=(\d+) K=(\d+) nseg=(\d+) tasks=(\d+)", l)
    M, N, K, nseg, T = map(int, m.groups()[1:])
    alg += 16.0 * (M * K + K * N + 2 * M * N) * T * nseg
    dram += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    ns += d["gpu__time_duration.sum"]
n = len(gl)
print(json.dumps({"launches": n, "duration_ms_serialised": round(ns / 1e6, 3), "dram_bytes": dram / n,
                  "algorithmic_bytes": alg / n, "ratio": dram / alg}, indent=1))
