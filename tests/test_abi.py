"""The C-ABI libraries load and export every symbol include/qpscat_b200.h declares."""
import ctypes
import os
import re

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "qpscat_b200.h")).read()
    return sorted(set(re.findall(r"\b(qps_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_hot_path_entry_points():
    syms = declared_symbols()
    for s in ["qps_build_geometry", "qps_make_problem", "qps_precompute_shift_blocks", "qps_assemble_system",
              "qps_schur_complement", "qps_block_lu_solve", "qps_recover_aux", "qps_solve", "qps_sweep",
              "qps_reflection_transmission", "qps_download_block", "qps_fill_evals", "qps_qsolve"]:
        assert s in syms


def test_product_exports_every_symbol(product_lib):
    lib = ctypes.CDLL(product_lib)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    lib.qps_backend_name.restype = ctypes.c_char_p
    assert lib.qps_backend_name() == b"b200-cuda"
    assert lib.qps_abi_version() == 4


def test_oracle_exports_every_symbol(oracle_lib):
    lib = ctypes.CDLL(oracle_lib)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    lib.qps_backend_name.restype = ctypes.c_char_p
    assert lib.qps_backend_name() == b"reference-cpu"


def test_product_has_no_cpu_fallback(product_lib):
    """Without a device the product refuses compute work loudly."""
    from paper_1410_5003_b200 import configs
    from paper_1410_5003_b200.qpscat import CudaError, Solver
    import pytest
    s = Solver(lib=product_lib, device=-1)
    st, num, om, th, K, _ = configs.config(1)
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    with pytest.raises(CudaError):
        s.solve()
    with pytest.raises(CudaError):
        s.hankel01([1.0])


def test_sm100a_code_in_library(product_lib):
    import shutil
    import subprocess
    import pytest
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "-lelf", product_lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([exe, "-sass", product_lib], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core path of the complex GEMM
