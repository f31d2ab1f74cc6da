"""The command-line front end on the B200: `qpscat solve` writes the result
document of SPEC.md:597-606 (resolved config, per-order amplitudes, R, T,
flux error, residuals, per-phase timings, field CSV) with the same numbers the
library returns through the Python mirror; `qpscat sweep` writes spectra with
the alpha group of each angle."""
import csv
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_1410_5003_b200 import configs

pytestmark = pytest.mark.gpu
CLI = os.path.join(ROOT, "paper_1410_5003_b200", "qpscat")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_solve_writes_the_result_document(gpu, tmp_path):
    cfg = json.loads(run("example", "cfg2").stdout)
    cfg["outputs"] = {"residuals": True, "field_grid": {"x": [-0.5, 0.5, 7], "y": [-3.5, 0.9, 9]}}
    p = tmp_path / "run.json"
    p.write_text(json.dumps(cfg))
    r = run("solve", "--config", str(p), "--out", str(tmp_path / "o"))
    assert r.returncode == 0, r.stderr
    doc = json.loads((tmp_path / "o" / "result.json").read_text())
    st, num, om, th, K, _ = configs.config(2)
    gpu.build_geometry(st, num)
    gpu.make_problem(om, th, K)
    gpu.solve()
    rt, sol = gpu.reflection_transmission(), gpu.solution()
    assert doc["R"] == pytest.approx(rt["R"], rel=1e-12, abs=1e-14)
    assert doc["T"] == pytest.approx(rt["T"], rel=1e-12, abs=1e-14)
    aU = np.array([o["aU"][0] + 1j * o["aU"][1] for o in doc["orders"]])
    assert np.allclose(aU, sol["aU"], rtol=0, atol=1e-13 * np.abs(sol["aU"]).max())
    assert [o["n"] for o in doc["orders"]] == list(range(-K, K + 1))
    assert doc["config"]["numerics"]["K"] == K
    assert set(doc["timings_ms"]) >= {"matrix_filling", "schur_complement", "block_solve"}
    assert doc["residuals"]["wall_qp"] < 1e-6 and doc["residuals"]["radiation"] < 1e-6
    rows = list(csv.DictReader(open(tmp_path / "o" / "field.csv")))
    assert len(rows) == 63 and set(rows[0]) == {"x", "y", "re_u", "im_u", "layer"}


def test_sweep_writes_spectra_with_alpha_groups(gpu, tmp_path):
    cfg = json.loads(run("example", "cfg5", "--interfaces", "4").stdout)
    cfg["incidence"] = {"alpha_grid": {"n_alpha": 3, "lo": -3.0, "hi": -0.2}}
    p = tmp_path / "sweep.json"
    p.write_text(json.dumps(cfg))
    r = run("sweep", "--config", str(p), "--out", str(tmp_path / "s"))
    assert r.returncode == 0, r.stderr
    doc = json.loads((tmp_path / "s" / "sweep.json").read_text())
    rows = list(csv.DictReader(open(tmp_path / "s" / "spectra.csv")))
    assert len(rows) == doc["angles"] == doc["solved"]
    assert doc["alpha_groups"] == 3 and doc["factorizations"] == 3
    assert sorted({int(r_["alpha_group"]) for r_ in rows}) == [0, 1, 2]
    assert all(int(r_["status"]) == 0 for r_ in rows)
