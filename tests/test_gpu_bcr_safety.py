"""Solver-error semantics and the low-rank safety net of the block solve, on
blocks wide enough (n = 320 >= 256) to enter the low-rank cyclic reduction.

* The reference throws SolverError(j + 1) when PartialPivLU::rcond() of a
  Thomas pivot is <= 1e-15 (tridiag.hpp:36-40).  A numerically singular (not
  exactly zero) diagonal block must be named by both implementations, on the
  low-rank path and on the dense fallback; the product estimates rcond of every
  LU factor it forms (LAPACK xTRCON on U, Hager/Higham) and of every Woodbury
  capacitance matrix (exact 1-norms of C and C^{-1}).
* Couplings that are not low rank (rank > 48 in the 64-column sample) must take
  the dense reduction automatically and still match the reference's block
  Thomas; low-rank couplings take the Woodbury path and pass the a-posteriori
  probe ||(I - P P^*) C w2|| <= 1e-12 ||C w2||; a failed probe (forced with
  QPS_LR_PROBE_TOL in a subprocess) falls back to the dense reduction."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1410_5003_b200 import SolverError

pytestmark = pytest.mark.gpu

N = 320


def rc(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def unitary(rng, n):
    q, r = np.linalg.qr(rc(rng, n, n))
    return q * (np.diag(r) / np.abs(np.diag(r)))


def stack(I, rank, seed, bad=None, smin=0.0):
    """Diagonally dominant blocks (4 I + 0.3 N(0,1)/sqrt(n) scale), couplings of
    the given rank (None: full rank).  Block `bad` is replaced by U diag(s) V^*
    with s_min = 0 (numerically singular, not exactly), and the couplings that
    enter its Thomas pivot avoid its left null vector so the reference's pivot
    stays singular too."""
    rng = np.random.default_rng(seed)
    n = N
    Ad = [4 * np.eye(n) + 0.3 * rc(rng, n, n) / np.sqrt(n) * 4 for _ in range(I)]

    def coupling():
        if rank is None:
            return 0.5 * rc(rng, n, n) / np.sqrt(n)
        return 0.5 * (rc(rng, n, rank) @ rc(rng, rank, n)) / n

    Au = [coupling() for _ in range(I - 1)]
    Al = [coupling() for _ in range(I - 1)]
    if bad is not None:
        U, V = unitary(rng, n), unitary(rng, n)
        s = np.linspace(2.0, 1.0, n)
        s[-1] = smin
        Ad[bad] = (U * s) @ V.conj().T
        u = U[:, -1:]
        if bad >= 1:
            Al[bad - 1] = Al[bad - 1] - u @ (u.conj().T @ Al[bad - 1])
    f = rc(rng, n)
    return Ad, Au, Al, f


def diag(s):
    return s.solver_diagnostics()


@pytest.mark.parametrize("rank,bad", [(12, 0), (12, 3), (None, 0), (None, 3)])
def test_numerically_singular_block_names_its_layer(gpu, oracle, rank, bad):
    Ad, Au, Al, f = stack(6, rank, 7 + bad, bad=bad)
    with pytest.raises(SolverError) as eo:
        oracle.block_lu_solve_blocks(Ad, Au, Al, f)
    with pytest.raises(SolverError) as eg:
        gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    assert eo.value.layer == bad + 1
    assert eg.value.layer == eo.value.layer


@pytest.mark.parametrize("rank", [12, None])
def test_ill_conditioned_block_is_not_rejected(gpu, oracle, rank):
    """rcond ~ 1e-12 (above the reference's 1e-15): the product's probe screen
    marks the block as a suspect, the full zlacn2 estimate clears it, and both
    implementations solve (to the conditioning of the problem)."""
    Ad, Au, Al, f = stack(6, rank, 21, bad=3, smin=2e-12)
    eo = oracle.block_lu_solve_blocks(Ad, Au, Al, f)
    eta = gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    assert np.linalg.norm(eta - eo) < 1e-3 * np.linalg.norm(eo)


def test_full_rank_couplings_take_the_dense_fallback(gpu, oracle):
    Ad, Au, Al, f = stack(9, None, 11)
    eta = gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    d = diag(gpu)
    assert d["bcr_path"] == 0 and d["lr_rank_max"] > 48, d
    eo = oracle.block_lu_solve_blocks(Ad, Au, Al, f)
    assert np.linalg.norm(eta - eo) < 1e-12 * np.linalg.norm(eo)


def test_low_rank_couplings_take_the_woodbury_path(gpu, oracle):
    Ad, Au, Al, f = stack(9, 20, 13)
    eta = gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    d = diag(gpu)
    assert d["bcr_path"] == 1 and d["lr_rank_max"] <= 48 and d["lr_probe_worst"] <= 1e-12, d
    eo = oracle.block_lu_solve_blocks(Ad, Au, Al, f)
    assert np.linalg.norm(eta - eo) < 1e-12 * np.linalg.norm(eo)


PROBE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from test_gpu_bcr_safety import stack
from paper_1410_5003_b200.qpscat import Solver
Ad, Au, Al, f = stack(9, 20, 13)
g = Solver(device=0)
eta = g.block_lu_solve_blocks(Ad, Au, Al, f)
o = Solver(lib={oracle!r})
eo = o.block_lu_solve_blocks(Ad, Au, Al, f)
d = g.solver_diagnostics()
print(d["bcr_path"], d["lr_rank_max"], d["lr_probe_worst"], np.linalg.norm(eta - eo) / np.linalg.norm(eo))
"""


def test_failed_probe_falls_back_to_dense(oracle_lib):
    here = os.path.dirname(os.path.abspath(__file__))
    code = PROBE_SCRIPT.format(root=os.path.dirname(here), tests=here, oracle=oracle_lib)
    env = dict(os.environ, QPS_LR_PROBE_TOL="1e-300")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    path, rank, worst, err = out.stdout.split()
    assert int(path) == 0 and int(rank) <= 48 and float(worst) > 1e-300
    assert float(err) < 1e-12
