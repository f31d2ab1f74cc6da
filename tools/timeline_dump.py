"""Per-scope device timeline of one config-4 solve (QPS_PROF_TIMELINE) after two warm-up solves.

Run as: QPS_PROF_TIMELINE=1 python tools/timeline_dump.py 2> timeline.txt
The TL lines on stderr give every profiled scope's [start, end] on its stream
relative to the first scope of the solve; tools/timeline_dump.py --summary FILE
prints the busy time of each stream and the scopes on the main stream's
critical path."""
import sys
import collections

if len(sys.argv) > 2 and sys.argv[1] == "--summary":
    rows = []
    for ln in open(sys.argv[2]):
        if not ln.startswith("TL "):
            continue
        p = ln.split()
        rows.append((p[1], p[3], float(p[5]), float(p[7])))
    # keep the last solve: scopes restart from ~0 after each prof_reset
    starts = [i for i, r in enumerate(rows) if r[2] < 1e-3]
    rows = rows[starts[-1]:] if starts else rows
    by_stream = collections.defaultdict(list)
    for r in rows:
        by_stream[r[1]].append(r)
    end = max(r[3] for r in rows)
    print(f"solve span {end:.2f} ms, {len(rows)} scopes")
    for s, rs in by_stream.items():
        rs.sort(key=lambda r: r[2])
        busy, cur0, cur1 = 0.0, None, None
        for r in rs:
            if cur1 is None or r[2] > cur1:
                if cur1 is not None:
                    busy += cur1 - cur0
                cur0, cur1 = r[2], r[3]
            else:
                cur1 = max(cur1, r[3])
        busy += cur1 - cur0
        fam = collections.defaultdict(float)
        for r in rs:
            fam[r[0]] += r[3] - r[2]
        top = ", ".join(f"{k} {v:.1f}" for k, v in sorted(fam.items(), key=lambda kv: -kv[1])[:8])
        print(f"stream {s}: busy {busy:.1f} ms [{rs[0][2]:.1f}, {max(r[3] for r in rs):.1f}]  {top}")
    sys.exit(0)

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

st, num, om, th, K, meta = configs.config(4)
s = Solver()
s.build_geometry(st, num)
s.make_problem(om, th, K)
s.prof_enable(True)
for _ in range(2):
    s.solve()
s.prof_reset()
print("=== timed solve ===", file=sys.stderr, flush=True)
s.solve()
s.prof_stats()
print(s.phase_times())
