"""GPU hot path vs the CPU oracle (the reference compiled unmodified) on the
same seeded inputs (paper_1410_5003_b200/configs.py).

Fill: every block of BlockSystem (assembly.hpp:293-315) element-wise.
Tolerances (max-norm, relative to the block's max entry):
  plain Nystrom / proxy / radiation blocks   1e-12
  A_diag (Alpert-corrected self blocks)      1e-9  (hypersingular T-kind
      corrections of size ~1e4-1e5 cancel in k_up - k_dn)
  A_diag of graded-corner interfaces: per entry max(3 x floor, 1e-9), floor =
      the largest change of the oracle's own entry under omega +- 1 ulp,
      every interface offset +- 1 ulp, the polyline vertices +- 1 ulp, and
      the reference compiled with FMA contraction (oracle/_ref/
      libqpscat_ref_fma.so).  Next to a corner the graded nodes are 1e-7 apart
      and an entry (k_up minus k_dn kernels) is the rounding residue of
      terms up to 1e10 times larger (a 40-digit mpmath evaluation of one such
      entry is 8 % away from the oracle's own value); the two builds of the
      reference differ there by up to 3e-5 of the block scale, and so does
      the GPU.  (Round 1 asserted 1e-3 inside 13-node corner zones; the
      residual it carried came from device-evaluated Alpert auxiliary nodes,
      now tabulated on the host, and a reference constant 1 ulp off.)
Solution: the raw densities eta are NOT compared: Q_i is numerically
rank-deficient at these sizes and equally valid residual minimizers differ by
O(1) in eta (proj/tests/test_periodize.cpp:119-126; the oracle moves eta by
~28 % under a 1-ulp change of omega, tools/noise_floor.py).  The physics
outputs are compared against the oracle's own noise floor measured here:
  ||[aU;aD]_gpu - [aU;aD]_ref|| / ||[aU;aD]_ref|| <= max(1e-8, 10 * floor)
  |R_gpu - R_ref|, |T_gpu - T_ref|                 <= max(1e-8, 10 * floor_RT)
where floor = change of the oracle's own outputs under a 1-ulp change of omega.
"""
import copy
import os

import numpy as np
import pytest

from conftest import ORACLE_LIB
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver

pytestmark = pytest.mark.gpu

CASES = [(1, None), (2, None), (3, 4), (5, 4), (4, 3)]
PLAIN_TOL = 1e-12
SELF_TOL = 1e-9


def rel(a, b):
    if b.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def setup(s, cfg, nif, omega_scale=None):
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
    if omega_scale:
        om = float(np.nextafter(om, 2 * om))
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    return st, num


ORACLE_FMA = os.path.join(os.path.dirname(ORACLE_LIB), "libqpscat_ref_fma.so")


def corner_floor(cfg, nif):
    """Per-entry rounding floor of the reference's graded-corner self blocks
    (see the module docstring), relative to each block's max entry."""
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)

    def fill(lib, stack, omega):
        s = Solver(lib=lib)
        s.build_geometry(stack, num)
        s.make_problem(omega, th, K)
        s.precompute_shift_blocks()
        s.assemble_system()
        out = {j: s.download_block("A_diag", j) for j, sp in enumerate(stack.interfaces) if sp.shape == "polyline"}
        s.close()
        return out

    base = fill(ORACLE_LIB, st, om)
    runs = [fill(ORACLE_FMA, st, om)] + [fill(ORACLE_LIB, st, float(np.nextafter(om, sgn))) for sgn in (np.inf, -np.inf)]
    for sgn in (np.inf, -np.inf):
        s2 = copy.deepcopy(st)
        for sp in s2.interfaces:
            sp.offset = float(np.nextafter(sp.offset, sgn))
        runs.append(fill(ORACLE_LIB, s2, om))
        for comp in (0, 1):
            s3 = copy.deepcopy(st)
            for sp in s3.interfaces:
                if sp.shape == "polyline":
                    sp.vertices = [v if q in (0, len(sp.vertices) - 1) else
                                   tuple(float(np.nextafter(x, sgn)) if c == comp else x for c, x in enumerate(v))
                                   for q, v in enumerate(sp.vertices)]
            runs.append(fill(ORACLE_LIB, s3, om))
    return {j: np.max([np.abs(r[j] - b) for r in runs], axis=0) / np.abs(b).max() for j, b in base.items()}


@pytest.mark.parametrize("cfg,nif", CASES)
def test_fill_blocks_match_oracle(gpu, oracle, cfg, nif):
    for s in (gpu, oracle):
        setup(s, cfg, nif)
        s.precompute_shift_blocks()
        s.assemble_system()
    I = gpu.problem_info()["I"]
    per = {"A_diag": range(I), "A_super": range(I - 1), "A_sub": range(I - 1), "B_self": range(I),
           "B_below": range(I), "C_self": range(I + 1), "C_above": range(I + 1), "Q": range(I + 1)}
    for name in ["Z_U", "Z_D", "V_U", "V_D", "W_U", "W_D", "f", "Bp_first", "Bp_last", "Cp_first", "Cp_last",
                 "Qp_first", "Qp_last"]:
        per[name] = [0]
    st = configs.config(cfg, n_interfaces=nif)[0]
    floors = corner_floor(cfg, nif) if any(sp.shape == "polyline" for sp in st.interfaces) else {}
    for name, idx in per.items():
        tol = SELF_TOL if name == "A_diag" else PLAIN_TOL
        for i in idx:
            g, o = gpu.download_block(name, i), oracle.download_block(name, i)
            assert g.shape == o.shape, (name, i)
            if name == "A_diag" and st.interfaces[i].shape == "polyline":
                floor = floors[i]
                scale = np.abs(o).max()
                d = np.abs(g - o) / scale
                bar = np.maximum(3 * floor, 1e-9)
                assert np.all(d <= bar), (name, i, d.max(), int((d > bar).sum()))
                continue
            assert rel(g, o) < tol, (name, i, rel(g, o))
    assert gpu.fill_evals()["reference"] == oracle.fill_evals()["reference"]


@pytest.mark.parametrize("cfg,nif", [(1, None), (2, None), (4, 3)])
def test_periodized_system_residuals(gpu, oracle, cfg, nif):
    """Per-layer LSQ residuals (periodize.hpp:84,113-118) agree: both solves
    reach the same least-squares optimum."""
    for s in (gpu, oracle):
        setup(s, cfg, nif)
        s.precompute_shift_blocks()
        s.assemble_system()
        s.schur_complement()
        s.block_lu_solve()
        s.recover_aux()
    lg, lo = gpu.solution()["lsq_residual"], oracle.solution()["lsq_residual"]
    assert np.all(lg < 10 * lo + 1e-13), (lg, lo)


def _phys(s):
    sol, rt = s.solution(), s.reflection_transmission()
    return np.concatenate([sol["aU"], sol["aD"]]), rt["R"], rt["T"], rt["flux_error"]


@pytest.mark.parametrize("cfg,nif", [(1, None), (2, None), (4, 4), (4, 50), (5, 6)])
def test_bragg_coefficients_at_oracle_noise_floor(gpu, oracle, cfg, nif):
    setup(gpu, cfg, nif)
    gpu.solve()
    ag, Rg, Tg, fg = _phys(gpu)
    setup(oracle, cfg, nif)
    oracle.solve()
    ao, Ro, To, fo = _phys(oracle)
    setup(oracle, cfg, nif, omega_scale=True)  # the oracle's own 1-ulp noise floor
    oracle.solve()
    a1, R1, T1, _ = _phys(oracle)
    floor = np.linalg.norm(a1 - ao) / np.linalg.norm(ao)
    floor_rt = max(abs(R1 - Ro), abs(T1 - To))
    err = np.linalg.norm(ag - ao) / np.linalg.norm(ao)
    assert err <= max(1e-8, 10 * floor), (err, floor)
    assert abs(Rg - Ro) <= max(1e-8, 10 * floor_rt) and abs(Tg - To) <= max(1e-8, 10 * floor_rt)
    assert abs(fg) <= max(1e-8, 10 * abs(fo))


def test_corner_wood_config_consistent(gpu, oracle):
    """Config 3 (graded corners, top layer 1e-10 from a Wood anomaly): the
    oracle itself is unresolved here (flux error ~4e-2 at P = 60), so parity is
    checked against its 1-ulp floor and finiteness (test_periodize.cpp:173-198)."""
    setup(gpu, 3, 4)
    gpu.solve()
    ag, Rg, Tg, fg = _phys(gpu)
    assert np.all(np.isfinite(ag))
    setup(oracle, 3, 4)
    oracle.solve()
    ao, Ro, To, fo = _phys(oracle)
    setup(oracle, 3, 4, omega_scale=True)
    oracle.solve()
    a1, _, _, _ = _phys(oracle)
    floor = np.linalg.norm(a1 - ao) / np.linalg.norm(ao)
    assert np.linalg.norm(ag - ao) / np.linalg.norm(ao) <= max(1e-8, 10 * floor)
