"""Graded-corner self blocks (A_diag of polyline interfaces, config-3 prefix):
GPU vs oracle per entry against the oracle's own per-entry 1-ulp floor
(omega +- 1 ulp and every polyline offset +- 1 ulp), by region: rows/columns
within 13 nodes of a segment end (corner zone) and the rest.
usage: python tools/corner_floor_probe.py"""
import copy
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

ORACLE = "oracle/_ref/libqpscat_ref.so"
st, num, om, th, K, _ = configs.config(3, n_interfaces=4)


def blocks(lib, stack, omega):
    s = Solver(lib=lib) if lib else Solver()
    s.build_geometry(stack, num)
    s.make_problem(omega, th, K)
    s.precompute_shift_blocks()
    s.assemble_system()
    out = {j: s.download_block("A_diag", j) for j in range(len(stack.interfaces))}
    s.close()
    return out


g = blocks(None, st, om)
o = blocks(ORACLE, st, om)
pert = [blocks("oracle/_ref/libqpscat_ref_fma.so", st, om), blocks(ORACLE, st, float(np.nextafter(om, np.inf))), blocks(ORACLE, st, float(np.nextafter(om, -np.inf)))]
for sgn in (np.inf, -np.inf):
    s2 = copy.deepcopy(st)
    for sp in s2.interfaces:
        sp.offset = float(np.nextafter(sp.offset, sgn))
    pert.append(blocks(ORACLE, s2, om))
    # interior polyline vertices moved by one ulp (node spacings change, not just a shift)
    for comp in (0, 1):
        s3 = copy.deepcopy(st)
        for sp in s3.interfaces:
            if sp.shape == "polyline":
                sp.vertices = [v if i in (0, len(sp.vertices) - 1) else
                               tuple(float(np.nextafter(c, sgn)) if q == comp else c for q, c in enumerate(v))
                               for i, v in enumerate(sp.vertices)]
        pert.append(blocks(ORACLE, s3, om))
for j, sp in enumerate(st.interfaces):
    if sp.shape != "polyline":
        continue
    scale = np.abs(o[j]).max()
    d = np.abs(g[j] - o[j]) / scale
    fl = np.max([np.abs(p[j] - o[j]) for p in pert], axis=0) / scale
    N = g[j].shape[0] // 2
    ends = np.zeros(N, dtype=bool)
    off = 0
    for n in sp.nodes:
        ends[off:off + 13] = True
        ends[off + n - 13:off + n] = True
        off += n
    e2 = np.concatenate([ends, ends])
    mask = e2[:, None] | e2[None, :]
    for name, m in (("corner zone", mask), ("rest", ~mask)):
        ratio = d[m] / np.maximum(fl[m], 1e-16)
        print(f"iface {j} {name}: max err {d[m].max():.2e} max floor {fl[m].max():.2e} "
              f"err>3floor+1e-12: {(d[m] > 3 * fl[m] + 1e-12).sum()} of {m.sum()}  worst ratio {ratio.max():.1f}")
    bar = np.maximum(3 * fl, 1e-9)
    print(f"   entries above max(3 floor, 1e-9 scale): {(d > bar).sum()}")
    bad = np.argwhere((d > 3 * fl + 1e-12))
    if len(bad):
        i, k = bad[np.argmax(d[tuple(bad.T)])]
        print("   worst entry", (i, k), "err", d[i, k], "floor", fl[i, k], "oracle", o[j][i, k], "gpu", g[j][i, k])
