"""The command-line front end (the reference's cli module is
a placeholder, proj/tools/main.cpp:1-2) on the host: built-in example
configurations reproduce paper_1410_5003_b200/configs.py exactly, validation
errors exit 2 naming the offending field, and compute commands
fail loudly without a device (no CPU fallback)."""
import json
import math
import os
import subprocess

import pytest

from conftest import ROOT
from paper_1410_5003_b200 import configs

CLI = os.path.join(ROOT, "paper_1410_5003_b200", "qpscat")


@pytest.fixture(scope="module")
def cli(product_lib):
    if not os.path.exists(CLI):
        pytest.fail("CLI missing: run __graft_entry__.build()")
    return CLI


def run(cli, *args, cwd=None):
    return subprocess.run([cli, *args], capture_output=True, text=True, cwd=cwd, timeout=120)


@pytest.mark.parametrize("cfg,nif", [(1, None), (2, None), (3, 6), (4, 7), (5, 4)])
def test_examples_match_configs_py(cli, cfg, nif):
    args = ["example", f"cfg{cfg}"] + (["--interfaces", str(nif)] if nif else [])
    r = run(cli, *args)
    assert r.returncode == 0, r.stderr
    doc = json.loads(r.stdout)
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
    assert doc["omega"] == om and doc["period"] == st.d
    assert [l["epsilon"] for l in doc["layers"]] == [m.epsilon for m in st.materials]
    assert len(doc["interfaces"]) == len(st.interfaces)
    for a, b in zip(doc["interfaces"], st.interfaces):
        assert a["shape"] == b.shape and a["offset"] == b.offset and a["nodes"] == list(b.nodes)
        if b.shape == "sine":
            assert a["amplitude"] == b.amplitude and a["phase"] == b.phase
        else:
            assert [tuple(v) for v in a["vertices"]] == [tuple(v) for v in b.vertices]
    n = doc["numerics"]
    assert (n["P"], n["Mw"], n["M"], n["K"], n["R"]) == (num.P, num.Mw, num.M, K, num.R)
    if cfg == 5:
        assert doc["incidence"]["uniform"]["n"] == 200
    else:
        assert doc["incidence"]["theta"] == th


def test_validate_accepts_and_rejects(cli, tmp_path):
    good = json.loads(run(cli, "example", "cfg2").stdout)
    p = tmp_path / "good.json"
    p.write_text(json.dumps(good))
    r = run(cli, "validate", "--config", str(p))
    assert r.returncode == 0 and "10 interfaces" in r.stdout, (r.stdout, r.stderr)
    bad = json.loads(json.dumps(good))
    del bad["layers"][3]["epsilon"]
    p.write_text(json.dumps(bad))
    r = run(cli, "validate", "--config", str(p))
    assert r.returncode == 2 and "layers[3].epsilon" in r.stderr, r.stderr
    bad = json.loads(json.dumps(good))
    bad["layers"].pop()  # one layer short of I + 1
    p.write_text(json.dumps(bad))
    assert run(cli, "validate", "--config", str(p)).returncode == 2
    bad = json.loads(json.dumps(good))
    bad["interfaces"][0] = {"shape": "polyline", "vertices": [[-0.4, 0], [0.5, 0]], "nodes": [40]}
    p.write_text(json.dumps(bad))
    r = run(cli, "validate", "--config", str(p))
    assert r.returncode == 2 and "span" in r.stderr, r.stderr
    p.write_text("{ not json")
    assert run(cli, "validate", "--config", str(p)).returncode == 2


def test_solve_needs_a_device(cli, tmp_path):
    p = tmp_path / "c.json"
    p.write_text(run(cli, "example", "cfg1").stdout)
    r = run(cli, "solve", "--config", str(p), "--out", str(tmp_path / "o"), "--device", "0")
    if "no usable CUDA device" not in r.stderr:
        pytest.skip("a device is present")
    assert r.returncode == 1
