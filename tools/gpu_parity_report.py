"""Compare the product library with the CPU oracle block by block on small
configs and print relative max-norm errors (diagnostic companion of
tests/test_gpu_parity.py).  Usage: python tools/gpu_parity_report.py [cfg ...]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

ORACLE = "oracle/_ref/libqpscat_ref.so"


def rel(a, b):
    den = max(np.abs(b).max(), 1e-300) if b.size else 1.0
    return float(np.abs(a - b).max() / den) if a.size else 0.0


def run(cfg, n_if=None):
    st, num, om, th, K, meta = configs.config(cfg, n_interfaces=n_if)
    out = {}
    for name, lib in (("gpu", None), ("ref", ORACLE)):
        s = Solver(lib=lib)
        s.build_geometry(st, num)
        s.make_problem(om, th, K)
        t0 = time.time()
        s.precompute_shift_blocks()
        s.assemble_system()
        blocks = {}
        I = s.problem_info()["I"]
        for b in ["A_diag", "B_self", "B_below", "C_self", "C_above", "Q"]:
            rng = range(I + 1) if b in ("C_self", "C_above", "Q") else range(I)
            blocks[b] = [s.download_block(b, i) for i in rng]
        for b in ["A_super", "A_sub"]:
            blocks[b] = [s.download_block(b, i) for i in range(I - 1)]
        for b in ["Z_U", "Z_D", "V_U", "V_D", "W_U", "W_D", "f", "Qp_first", "Cp_first", "Qp_last", "Cp_last"]:
            blocks[b] = [s.download_block(b, 0)]
        s.schur_complement()
        for b in ["Ap_diag"]:
            blocks[b] = [s.download_block(b, i) for i in range(I)]
        blocks["X_first"] = [s.download_block("X_first")]
        blocks["X_last"] = [s.download_block("X_last")]
        s.block_lu_solve()
        s.recover_aux()
        t1 = time.time()
        out[name] = (blocks, s.solution(), s.reflection_transmission(), s.fill_evals(), t1 - t0)
    gb, gs, grt, gev, gt = out["gpu"]
    rb, rs, rrt, rev, rt = out["ref"]
    print(f"== config {cfg} (I={meta['I']}) gpu {gt:.3f}s  ref {rt:.3f}s  evals gpu {gev} ref {rev}")
    for b in gb:
        errs = [rel(x, y) for x, y in zip(gb[b], rb[b])] or [0.0]
        shapes_ok = all(x.shape == y.shape for x, y in zip(gb[b], rb[b]))
        print(f"  {b:10s} max rel err {max(errs):.3e}  shapes_ok={shapes_ok}")
    a_g = np.concatenate([gs["aU"], gs["aD"]])
    a_r = np.concatenate([rs["aU"], rs["aD"]])
    print(f"  [aU;aD] rel 2-norm err {np.linalg.norm(a_g - a_r) / np.linalg.norm(a_r):.3e}")
    print(f"  eta rel 2-norm err {np.linalg.norm(gs['eta_flat'] - rs['eta_flat']) / np.linalg.norm(rs['eta_flat']):.3e}")
    print(f"  R {grt['R']:.15f} vs {rrt['R']:.15f}  |dR| {abs(grt['R'] - rrt['R']):.2e}")
    print(f"  T {grt['T']:.15f} vs {rrt['T']:.15f}  |dT| {abs(grt['T'] - rrt['T']):.2e}")
    print(f"  flux gpu {grt['flux_error']:.3e} ref {rrt['flux_error']:.3e}; lsq gpu {gs['max_lsq_residual']:.2e} ref {rs['max_lsq_residual']:.2e}")


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2]
    for c in cfgs:
        run(c)
    s = Solver()
    print("fp64 peaks", s.fp64_peaks())
