"""Summarise an ncu launch list (--csv --nvtx --metrics gpu__time_duration.sum,
launch__grid_size,...): serialised time per kernel family, optionally only the
launches inside one NVTX push/pop range.

usage: python tools/launch_table.py launches.csv [NVTX_RANGE] [--shapes]"""
import collections
import csv
import sys

path = sys.argv[1]
rng = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
shapes = "--shapes" in sys.argv
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
rows = rows[next(i for i, r in enumerate(rows) if r and r[0] == "ID"):]  # skip program output before the CSV
h = rows[0]
iname, iid, imet, ival = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
inv = [i for i, c in enumerate(h) if "Push/Pop_Range" in c]
igrid = h.index("Grid Size")
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[iid], {"name": r[iname], "nvtx": r[inv[0]] if inv else "", "grid": r[igrid]})
    if r[imet] == "gpu__time_duration.sum":
        d["ns"] = float(r[ival].replace(",", ""))
fam = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for d in L.values():
    if rng and rng not in d["nvtx"]:
        continue
    k = d["name"].split("(")[0].split("::")[-1][:60]
    if shapes:
        k += " " + d["grid"]
    fam[k][0] += 1
    fam[k][1] += d.get("ns", 0) * 1e-6
    tot += d.get("ns", 0) * 1e-6
print(f"total {tot:.3f} ms over {sum(v[0] for v in fam.values())} launches" + (f" in range {rng}" if rng else ""))
for k, (n, ms) in sorted(fam.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"  {ms:9.3f} ms  {100 * ms / tot:5.1f}%  {n:5d}  {k}")
