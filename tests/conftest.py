"""Shared fixtures.  `-m gpu` tests need a B200 and the built product library;
everything else runs on CPU.  The CPU oracle (oracle/_ref/libqpscat_ref.so,
the reference headers compiled against oracle/shim) is test infrastructure:
tests load it explicitly as the checker."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ORACLE_LIB = os.path.join(ROOT, "oracle", "_ref", "libqpscat_ref.so")
PRODUCT_LIB = os.path.join(ROOT, "paper_1410_5003_b200", "libqpscat_b200.so")
REFERENCE = "/root/reference/proj"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built product library")


def _ensure_oracle():
    if not os.path.exists(ORACLE_LIB):
        if not os.path.isdir(REFERENCE):
            pytest.skip("oracle library not built and /root/reference absent")
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    return ORACLE_LIB


@pytest.fixture(scope="session")
def oracle_lib():
    return _ensure_oracle()


@pytest.fixture(scope="session")
def product_lib():
    if not os.path.exists(PRODUCT_LIB):
        pytest.fail("product library missing: run __graft_entry__.build()")
    return PRODUCT_LIB


@pytest.fixture()
def oracle(oracle_lib):
    from paper_1410_5003_b200.qpscat import Solver
    s = Solver(lib=oracle_lib)
    yield s
    s.close()


@pytest.fixture()
def host(product_lib):
    """Product library in host-only mode (device -1): host logic, no GPU."""
    from paper_1410_5003_b200.qpscat import Solver
    s = Solver(lib=product_lib, device=-1)
    yield s
    s.close()


@pytest.fixture()
def gpu(product_lib):
    from paper_1410_5003_b200.qpscat import Solver
    s = Solver(lib=product_lib, device=0)
    assert s.backend == "b200-cuda"
    yield s
    s.close()


_PARITY = []


@pytest.fixture()
def parity_report():
    """Record measured error vs the oracle's noise floor; printed in the
    terminal summary (visible under -q) as 'name: quantity err (floor f)'."""
    def rec(name, items):
        _PARITY.append((name, items))
    return rec


def pytest_terminal_summary(terminalreporter):
    if not _PARITY:
        return
    terminalreporter.section("parity vs oracle (measured error, oracle 1-ulp floor)")
    for name, items in _PARITY:
        parts = [f"{k} {v[0]:.3g} ({v[2] if len(v) > 2 else 'floor'} {v[1]:.3g})" for k, v in items.items()]
        terminalreporter.write_line(f"{name}: " + ", ".join(parts))
