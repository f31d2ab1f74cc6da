"""Config-5 angle sweep timing on the GPU: accelerated (cache once, angles
batched) vs independent (cache refilled per angle), plus one-shot solves.

usage: python tools/sweep_bench.py [--angles 200] [--nif N] [--independent]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1410_5003_b200 import Solver, configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--angles", type=int, default=200)
    ap.add_argument("--nif", type=int, default=None)
    ap.add_argument("--independent", action="store_true")
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args()
    if a.batch:
        os.environ["QPS_SWEEP_BATCH"] = str(a.batch)
    st, num, om, th, K, meta = configs.config(5, n_interfaces=a.nif)
    thetas = configs.sweep_angles(a.angles)
    s = Solver()
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    out = {"config": 5, "I": s.problem_info()["I"], "angles": a.angles, "K": K}
    s.sweep(thetas[:2], K, mode=0)  # warm-up (allocations, cache)
    s.build_geometry(st, num)       # drop the cache: the timed sweep fills it
    s.make_problem(om, th, K)
    t0 = time.perf_counter()
    r = s.sweep(thetas, K, mode=0)
    out["accelerated_s"] = time.perf_counter() - t0
    out["accelerated_phases_ms"] = s.phase_times()
    out["ok"] = int((r["status"] == 0).sum())
    out["mean_abs_flux_error"] = float(np.nanmean(np.abs(r["flux_error"])))
    if a.independent:
        t0 = time.perf_counter()
        r2 = s.sweep(thetas, K, mode=1)
        out["independent_s"] = time.perf_counter() - t0
        out["independent_phases_ms"] = s.phase_times()
        out["speedup"] = out["independent_s"] / out["accelerated_s"]
        out["max_rel_diff"] = float(np.abs(r2["aU"] - r["aU"]).max() / np.abs(r["aU"]).max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
