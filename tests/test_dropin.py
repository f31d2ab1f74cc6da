"""The C++ drop-in adapter (include/qpscat_b200.hpp) compiles against the
reference's own headers and, on a GPU, reproduces the reference's Fresnel
end-to-end case from the same reference types (oracle/dropin_demo.cpp)."""
import os
import subprocess

import pytest

from conftest import REFERENCE, ROOT

DEMO = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")


def test_dropin_adapter_compiles(product_lib):
    if not os.path.isdir(REFERENCE):
        pytest.skip("reference headers not mounted")
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "dropin"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert os.path.exists(DEMO)


@pytest.mark.gpu
def test_dropin_demo_runs_on_gpu():
    if not os.path.exists(DEMO):
        pytest.skip("dropin_demo not built (needs /root/reference at build time)")
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROP-IN OK" in r.stdout
