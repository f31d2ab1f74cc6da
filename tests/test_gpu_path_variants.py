"""The round-2 fast paths and the slower paths they replaced (kept for A/B)
give the same physics: the row-ID compression vs the orthonormal P (P^* C)
(QPS_LR_ID=0), the sparse sign sketch vs the dense Gaussian sample
(QPS_LR_SKETCH=dense), 64-column LU leaves vs 16-column panels
(QPS_LU_WIDE=0), the levels' right-hand-side stream vs one stream
(QPS_WB_RHS_STREAM=0), the blocked interior back substitution vs the
one-kernel version (QPS_COD_TRSM=blk).  The switches are read once per process,
so each variant runs in its own subprocess (tools/lowrank_check.py) on the
config-4 prefix (50 interfaces, 608-point blocks, the low-rank Woodbury path);
Bragg amplitudes agree to 1e-10 relative (the problem's own floor is ~1e-11)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = {"QPS_LR_ID": "0", "QPS_LR_SKETCH": "dense", "QPS_LU_WIDE": "0", "QPS_WB_RHS_STREAM": "0",
            "QPS_COD_TRSM": "blk"}


def _run(tmp_path, name=None, value=None):
    out = str(tmp_path / f"a_{name or 'default'}.npy")
    env = dict(os.environ)
    for k in VARIANTS:
        env.pop(k, None)
    env.pop("QPS_BCR", None)
    if name:
        env[name] = value
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "lowrank_check.py"), "4", "50", out],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return np.load(out), json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_fast_paths_match_the_paths_they_replaced(tmp_path):
    a0, r0 = _run(tmp_path)
    assert abs(r0["flux"]) < 1e-9
    for name, value in VARIANTS.items():
        a, r = _run(tmp_path, name, value)
        err = np.linalg.norm(a - a0) / np.linalg.norm(a0)
        assert err < 1e-10, (name, err)
        assert abs(r["flux"]) < 1e-9, (name, r)
