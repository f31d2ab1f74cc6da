"""Join an ncu launch list (--csv, gpu__time_duration.sum) with the library's
QPS_TRACE_GEMM stderr lines (one per zgemm_batched call, in launch order) and
print time and achieved rate per GEMM family / shape.
usage: python tools/gemm_shapes.py launches.csv trace.err [family]"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[h.index("ID")], {"name": r[h.index("Kernel Name")]})
    if r[h.index("Metric Name")] == "gpu__time_duration.sum":
        d["ns"] = float(r[h.index("Metric Value")].replace(",", ""))
gl = [d for d in L.values() if "zgemm3m" in d["name"] and not re.search(r", 1>\(", d["name"])]
sh = [l for l in open(sys.argv[2]) if l.startswith("gemm ")]
fam_only = sys.argv[3] if len(sys.argv) > 3 else None
assert len(gl) == len(sh), (len(gl), len(sh))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
per = []
for d, l in zip(gl, sh):
    m = re.match(r"gemm (\S+) M=(\d+) N=(\d+) K=(\d+) nseg=(\d+) tasks=(\d+)", l)
    fam, M, N, K, ns, T = m.group(1), *map(int, m.groups()[1:])
    fl = 6.0 * M * N * K * T * ns
    a = agg[fam]
    a[0] += 1
    a[1] += d["ns"] / 1e6
    a[2] += fl
    if fam_only is None or fam == fam_only:
        per.append((d["ns"] / 1e6, fam, M, N, K, ns, T, fl / (d["ns"] * 1e-9) / 1e12, d["name"].split("<")[1].split(">")[0]))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:14s} {v[0]:4d} launches {v[1]:8.2f} ms {v[2] / (v[1] * 1e-3) / 1e12:6.2f} TF/s")
print("top launches:")
for x in sorted(per, reverse=True)[:25]:
    print(f"  {x[0]:7.3f} ms {x[1]:12s} M={x[2]} N={x[3]} K={x[4]} nseg={x[5]} tasks={x[6]} {x[7]:6.2f} TF/s <{x[8]}>")
