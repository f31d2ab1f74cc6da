"""Graded-corner self block (config-3 prefix): GPU vs oracle A_diag entries, split inside / outside the corner zones."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st, num, om, th, K, _ = configs.config(3, n_interfaces=4)
print([ (sp.shape, sp.vertices, sp.nodes) for sp in st.interfaces])
out = []
for lib in (None, "oracle/_ref/libqpscat_ref.so"):
    s = Solver(lib=lib); s.build_geometry(st, num); s.make_problem(om, th, K); s.precompute_shift_blocks(); s.assemble_system()
    out.append(s.download_block("A_diag", 3))
g, o = out
d = np.abs(g - o) / np.abs(o).max()
N = g.shape[0] // 2
for kind, (r0, c0) in {"D": (0, 0), "S": (0, N), "T": (N, 0), "Ds": (N, N)}.items():
    blk = d[r0:r0 + N, c0:c0 + N]
    i = np.unravel_index(np.argmax(blk), blk.shape)
    print(kind, blk.max(), i, "row max profile (top rows):", np.argsort(blk.max(axis=1))[-8:])
ends = np.zeros(N, dtype=bool)
for off, n in [(0, 100), (100, 100)]:
    ends[off:off + 10] = True; ends[off + n - 10:off + n] = True
e2 = np.concatenate([ends, ends]); mask = e2[:, None] | e2[None, :]
dd = np.where(mask, 0, d)
i = np.unravel_index(np.argmax(dd), dd.shape)
print("unmasked max", dd.max(), "at", i, "ref", o[i], "gpu", g[i])
print("top unmasked rows", np.argsort(dd.max(axis=1))[-10:], "cols", np.argsort(dd.max(axis=0))[-10:])
