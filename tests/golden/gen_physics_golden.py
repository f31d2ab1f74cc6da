"""Generate the physics golden fixtures (TEST INFRASTRUCTURE — runs the CPU
oracle, i.e. the reference headers compiled unmodified against oracle/shim).

For each case the oracle solves the seeded configuration of
paper_1410_5003_b200/configs.py nominally and under eight perturbations of 1
and 2 ulp (omega up/down: every k_i moves; theta up/down: alpha and kappa_n
move), and stores
  * the Bragg amplitudes aU, aD (reflection_transmission's inputs,
    tridiag.hpp:11-17), R, T, flux_error (postprocess.hpp:134-180),
  * the total field u at fixed off-interface probes (evaluate_field,
    postprocess.hpp:82-123; one probe above y_U, below y_D and ~10 at
    mid-layer heights down the stack -- SURVEY §8(c)'s protocol),
  * the oracle's ulp-level noise floor = the largest change of those outputs
    under the eight perturbations (the outputs of a rank-deficient least-
    squares elimination are a random sample of equally valid minimisers; the
    maximum over eight samples bounds that spread more robustly than one).
The GPU tests (tests/test_gpu_golden.py) assert the product against these
numbers at <= max(1e-9, 3 x floor).

Cases: cfg1, cfg2 (full), cfg3 (I = 100, corners + Wood anomaly), cfg5 (the
sweep: I = 100, 20 of the 200 angles, through the oracle's qps_sweep = one
precompute_shift_blocks, then assemble/Schur/Thomas per angle), cfg4 (I =
1000; needs ~125 GB of host RAM and ~3 min per solve on 16 cores: run it on
the GPU box's host, `gpurun -- python tests/golden/gen_physics_golden.py cfg4`,
then copy gpurun_out/golden/physics_cfg4.json here).

usage: python tests/golden/gen_physics_golden.py [case ...] [--out DIR]
"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1410_5003_b200 import configs  # noqa: E402
from paper_1410_5003_b200.qpscat import Solver  # noqa: E402

ORACLE = os.path.join(ROOT, "oracle", "_ref", "libqpscat_ref.so")
CASES = {"cfg1": (1, None), "cfg2": (2, None), "cfg3": (3, None), "cfg4": (4, None), "cfg5": (5, None)}
SWEEP_STRIDE = 10  # cfg5: every 10th of the 200 angles -> 20 angles


def cx(a):
    return [[float(v.real), float(v.imag)] for v in np.ravel(a)]


def probes(st, info):
    """Off-interface probe points: above y_U, mid-layer heights, below y_D."""
    yU, yD = info["y_U"], info["y_D"]
    offs = [sp.offset for sp in st.interfaces]
    pts = [(0.15, yU + 0.3)]
    I = len(offs)
    if I == 1:
        pts += [(0.15, offs[0] + 0.6), (0.15, offs[0] - 0.6)]
    else:
        stride = max(1, (I - 1) // 10)
        for n, i in enumerate(range(0, I - 1, stride)):
            pts.append((0.15 if n % 2 == 0 else -0.35, 0.5 * (offs[i] + offs[i + 1])))
    pts.append((0.15, yD - 0.3))
    return np.array(pts)


def solve_once(s, st, num, om, th, K, pts):
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    t0 = time.perf_counter()
    s.solve()
    dt = time.perf_counter() - t0
    sol, rt = s.solution(), s.reflection_transmission()
    u = s.evaluate_field(pts)["u_total"]
    return {"a": np.concatenate([sol["aU"], sol["aD"]]), "aU": sol["aU"], "aD": sol["aD"], "R": rt["R"],
            "T": rt["T"], "flux_error": rt["flux_error"], "max_lsq": sol["max_lsq_residual"], "u": u,
            "seconds": dt}


def ulps(x, n):
    for _ in range(abs(n)):
        x = float(np.nextafter(x, np.inf if n > 0 else -np.inf))
    return x


def perturbations(om, th):
    out = {}
    for n in (1, -1, 2, -2):
        out[f"omega{n:+d}ulp"] = (ulps(om, n), th)
        out[f"theta{n:+d}ulp"] = (om, ulps(th, n))
    return out


def single(name, cfg, nif, threads):
    st, num, om, th, K, meta = configs.config(cfg, n_interfaces=nif)
    s = Solver(lib=ORACLE)
    s.set_num_threads(threads)
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    pts = probes(st, s.problem_info())
    nom = solve_once(s, st, num, om, th, K, pts)
    fl = {}
    for tag, (o2, t2) in perturbations(om, th).items():
        p = solve_once(s, st, num, o2, t2, K, pts)
        fl[tag] = {"bragg_rel": float(np.linalg.norm(p["a"] - nom["a"]) / np.linalg.norm(nom["a"])),
                   "dR": abs(p["R"] - nom["R"]), "dT": abs(p["T"] - nom["T"]),
                   "field_rel": float(np.abs(p["u"] - nom["u"]).max() / np.abs(nom["u"]).max())}
        print(name, tag, fl[tag], flush=True)
    s.close()
    floor = {k: max(v[k] for v in fl.values()) for k in ("bragg_rel", "dR", "dT", "field_rel")}
    return {"case": name, "cfg": cfg, "I": len(st.interfaces), "seed": meta["seed"], "omega": om, "theta": th,
            "K": K, "aU": cx(nom["aU"]), "aD": cx(nom["aD"]), "R": nom["R"], "T": nom["T"],
            "flux_error": nom["flux_error"], "max_lsq_residual": nom["max_lsq"], "probes": pts.tolist(),
            "u_total": cx(nom["u"]), "floor": floor, "floor_by_perturbation": fl,
            "oracle_seconds_per_solve": nom["seconds"]}


def sweep(name, cfg, threads):
    st, num, om, _, K, meta = configs.config(cfg)
    thetas = configs.sweep_angles(200)[::SWEEP_STRIDE]
    s = Solver(lib=ORACLE)
    s.set_num_threads(threads)

    def run(o2, ths):
        s.build_geometry(st, num)
        s.make_problem(o2, ths[0], K)
        t0 = time.perf_counter()
        r = s.sweep(ths, K, mode=0)
        r["seconds"] = time.perf_counter() - t0
        assert np.all(r["status"] == 0), r["status"]
        return r

    nom = run(om, thetas)
    a0 = np.concatenate([nom["aU"], nom["aD"]], axis=1)
    floors = []
    pert = []
    for n in (1, -1, 2, -2):
        pert.append((ulps(om, n), thetas))
        pert.append((om, [ulps(t, n) for t in thetas]))
    for o2, ths in pert:
        p = run(o2, ths)
        a = np.concatenate([p["aU"], p["aD"]], axis=1)
        floors.append({"bragg_rel": (np.linalg.norm(a - a0, axis=1) / np.linalg.norm(a0, axis=1)).tolist(),
                       "dR": np.abs(p["R"] - nom["R"]).tolist(), "dT": np.abs(p["T"] - nom["T"]).tolist()})
        print(name, "perturbation done", max(floors[-1]["bragg_rel"]), flush=True)
    s.close()
    n = len(thetas)
    floor = {k: [max(f[k][a] for f in floors) for a in range(n)] for k in ("bragg_rel", "dR", "dT")}
    return {"case": name, "cfg": cfg, "I": len(st.interfaces), "seed": meta["seed"], "omega": om, "K": K,
            "thetas": thetas, "angle_indices": list(range(0, 200, SWEEP_STRIDE)),
            "aU": [cx(v) for v in nom["aU"]], "aD": [cx(v) for v in nom["aD"]], "R": nom["R"].tolist(),
            "T": nom["T"].tolist(), "flux_error": nom["flux_error"].tolist(), "floor": floor,
            "oracle_seconds_sweep": nom["seconds"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["cfg1", "cfg2", "cfg3", "cfg5"])
    ap.add_argument("--out", default=os.path.dirname(os.path.abspath(__file__)))
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    for name in args.cases:
        cfg, nif = CASES[name]
        t0 = time.time()
        res = sweep(name, cfg, args.threads) if cfg == 5 else single(name, cfg, nif, args.threads)
        res["generator"] = "tests/golden/gen_physics_golden.py"
        res["host"] = {"cpu": platform.processor() or platform.machine(), "threads": args.threads}
        res["wall_seconds"] = time.time() - t0
        with open(os.path.join(args.out, f"physics_{name}.json"), "w") as f:
            json.dump(res, f, indent=0)
        print(name, "written", f"{res['wall_seconds']:.0f} s", flush=True)


if __name__ == "__main__":
    main()
