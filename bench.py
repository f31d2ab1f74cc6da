"""Benchmark: the 1000-layer quasi-periodic multilayer solve on B200.

Workload (BASELINE.json configs[3]): 1000 seeded sinusoidal
interfaces, N = 300 nodes each (6e5 density unknowns), k_i ~ U[10, 30],
P = 80, Mw = 40, M = 60, K = 20, theta = -pi/5.  One step = one full solve
through the product library: Nystrom fill -> Schur complements -> block
cyclic reduction -> recovery of proxies/Bragg amplitudes.

  value : layers/s = (I x ranks) / device step time (CUDA events on the
          solver's stream, barrier + synchronize around the timed region, max
          over ranks); the geometry is already resident in HBM.
  e2e   : the same metric through the public C-ABI from HOST data: geometry
          build + H2D, solve, D2H of eta/c/aU/aD, timed per step.
  roofline : dominant kernel family over the timed region (library
          CUDA-event instrumentation), achieved TFLOP/s vs the FP64 DMMA peak
          measured by a microbenchmark in the same run.
  cpu_baseline : the reference (oracle/_ref, the qpscat headers compiled
          unmodified against oracle/shim) on a bounded I-layer sample of the
          same per-layer sizes, all host threads, rank 0 only.

Multi-GPU (--gpus N under torchrun): replicas only — each rank solves its own
1000-layer stack (the north star keeps one solve on one GPU), no collective on
the data path; "scaling": "weak".
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "1000-layer solve wall time & layers/s; kernel evals/s; % of FP64 peak"
ORACLE = os.path.join(ROOT, "oracle", "_ref", "libqpscat_ref.so")
# ncu --set full summaries of the captured launches (profiles/README.md says how they were taken)
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")


def ncu_summary():
    try:
        with open(NCU_SUMMARY) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}
CFG = 4


def bcr_factor(phases, I, n, peak, width):
    """The block solve's factorization batch (Woodbury level 0: LU with partial
    pivoting of every n x n diagonal block and its 2r + 1 right-hand-side
    solves, r = the adaptive basis width: 40 at config 4) against the DMMA
    peak, at nominal complex flop counts (LU 8/3 n^3, forward + back
    substitution 8 n^2 per right-hand side; n = 2N, the padding to 608 not
    counted)."""
    ms = phases.get("factor_ms") or 0.0
    if ms <= 0 or width <= 0:
        return None
    rhs = 2 * width + 1
    fl = I * (8.0 / 3.0 * n ** 3 + 8.0 * n * n * rhs)
    tf = fl / (ms * 1e-3) / 1e12
    return {"ms": ms, "blocks": I, "n": n, "rhs": rhs, "nominal_flops": fl, "tflops": tf,
            "frac_of_dmma_peak": tf / peak}


def workload_config(I, N, num, K, theta, seed):
    return {"workload": f"cfg4: {I} seeded sinusoidal interfaces, N={N}, P={num.P}, Mw={num.Mw}, M={num.M}, "
                        f"K={K}, k~U[10,30], theta={theta:.6f}",
            "I": I, "N": N, "P": num.P, "Mw": num.Mw, "M": num.M, "K": K, "seed": seed,
            "density_unknowns": 2 * N * I, "parallelism": "replicas",
            "l2": "inputs larger than L2 (A' alone is 17.3 GB >> 126 MB), no flush needed"}


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        # NVML (nvidia-ml-py) samples every 20 ms; nvidia-smi (~0.2 s per call) as the fallback
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self.stop.is_set():
                r = get_reasons(h)
                self.samples.append([str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), str(mx)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self.stop.wait(0.02)
            return
        except Exception:
            pass
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return world, rank, local, dist


def barrier(dist):
    if dist is not None:
        dist.barrier()


def allmax(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(I_sample, threads, reps=1):
    """Time the reference (oracle/_ref) on a bounded sample of the same workload."""
    from paper_1410_5003_b200 import configs
    from paper_1410_5003_b200.qpscat import Solver
    st, num, om, th, K, meta = configs.config(CFG, n_interfaces=I_sample)
    s = Solver(lib=ORACLE)
    s.set_num_threads(threads)
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        s.solve()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    ph = s.phase_times()
    evals = s.fill_evals()["reference"]
    s.close()
    return {"value": I_sample / best, "unit": "layers/s", "cores": threads, "kind": "reference",
            "sample": f"{I_sample}-layer prefix of the cfg4 stack (same N={meta['N']}, P, Mw, M, K), "
                      f"one full solve (fill {ph['fill_ms'] + ph['assemble_ms']:.0f} ms, schur {ph['schur_ms']:.0f} ms, "
                      f"thomas {ph['solve_ms'] + ph['recover_ms']:.0f} ms)",
            "seconds": best, "kernel_evals_per_s": evals / ((ph["fill_ms"] + ph["assemble_ms"]) * 1e-3)}


def sweep_measure(device, ref_angles):
    """Config 5 (BASELINE configs[4]): 100 interfaces, N = 150, K = 20, 200
    angles uniform in [-pi + 0.1, -0.1].  GPU wall time (host clock around the
    C-ABI call, device synchronised inside it) of the accelerated sweep (cache
    filled once, angles batched; no two of these angles share alpha) and of
    independent per-angle solves; the same sweep on the paper's alpha grid
    (plan_sweep, n = 40 alphas over the same range: one interior elimination
    and one factorization per alpha group); and the reference's sweep
    composition (oracle/_ref: cache once, then assemble / Schur /
    Thomas per angle) on a bounded sample of the angles, all host threads."""
    from paper_1410_5003_b200 import configs
    from paper_1410_5003_b200.qpscat import Solver
    st, num, om, th, K, meta = configs.config(5)
    thetas = configs.sweep_angles(200)
    g = Solver(device=device)
    g.build_geometry(st, num)
    g.make_problem(om, th, K)
    g.sweep(thetas[:2], K, mode=0)  # warm-up: allocations
    out = {"workload": f"cfg5: {meta['I']} interfaces, N={meta['N']}, P={num.P}, K={K}, 200 angles in [-pi+0.1,-0.1]",
           "angles": len(thetas)}
    g.build_geometry(st, num)  # drop the cache: the timed sweep fills it
    g.make_problem(om, th, K)
    t0 = time.perf_counter()
    r = g.sweep(thetas, K, mode=0)
    out["accelerated_s"] = time.perf_counter() - t0
    out["accelerated_ms_per_angle"] = 1e3 * out["accelerated_s"] / len(thetas)
    out["converged"] = int((r["status"] == 0).sum())
    out["mean_abs_flux_error"] = float(statistics.fmean(abs(x) for x in r["flux_error"]))
    t0 = time.perf_counter()
    g.sweep(thetas, K, mode=1)
    out["independent_s"] = time.perf_counter() - t0
    out["speedup_vs_independent"] = out["independent_s"] / out["accelerated_s"]
    ta, grp = g.plan_sweep(40, -math.pi + 0.1, -0.1)
    t0 = time.perf_counter()
    ra = g.sweep(list(ta), K, mode=0)
    out["alpha_grid"] = {"angles": len(ta), "alpha_groups": 40, "s": time.perf_counter() - t0}
    info = g.sweep_info(len(ta))
    out["alpha_grid"].update({"n_groups": info["n_groups"], "n_factorizations": info["n_factorizations"],
                              "n_interior": info["n_interior"], "converged": int((ra["status"] == 0).sum())})
    t0 = time.perf_counter()
    g.sweep(list(ta), K, mode=1)
    out["alpha_grid"]["independent_s"] = time.perf_counter() - t0
    out["alpha_grid"]["speedup_vs_independent"] = out["alpha_grid"]["independent_s"] / out["alpha_grid"]["s"]
    g.close()
    if ref_angles > 0 and os.path.exists(ORACLE):
        o = Solver(lib=ORACLE)
        o.set_num_threads(os.cpu_count() or 1)
        o.build_geometry(st, num)
        o.make_problem(om, th, K)
        sample = thetas[::len(thetas) // ref_angles][:ref_angles]
        t0 = time.perf_counter()
        o.sweep(sample, K, mode=0)
        dt = time.perf_counter() - t0
        fill_s = o.phase_times()["fill_ms"] * 1e-3  # the oracle reports the whole sweep here
        o.build_geometry(st, num)
        o.make_problem(om, th, K)
        t1 = time.perf_counter()
        o.sweep(sample[:1], K, mode=0)
        one = time.perf_counter() - t1  # cache fill + one angle
        per_angle = (dt - one) / max(1, len(sample) - 1)
        cache = one - per_angle
        out["cpu_reference"] = {"kind": "reference", "cores": os.cpu_count() or 1,
                                "sample": f"{len(sample)} of the 200 angles (cache fill once + per angle assemble/"
                                          f"Schur/Thomas), extrapolated to 200 angles as cache + 200 x per-angle",
                                "sample_s": dt, "cache_fill_s": cache, "per_angle_s": per_angle,
                                "sweep_200_s_extrapolated": cache + 200 * per_angle, "sweep_reported_s": fill_s}
        out["speedup_vs_cpu_reference"] = out["cpu_reference"]["sweep_200_s_extrapolated"] / out["accelerated_s"]
        o.close()
    return out


def run_reference(args, world, rank):
    """The reference's own CPU implementation (oracle/_ref: the qpscat headers
    compiled unmodified) on all host threads.  A full config-4 solve takes
    ~195 s on 16 cores, so each step is a bounded sample of the workload: the
    first `--ref-layers` interfaces of the same seeded stack (same N, P, Mw,
    M, K); the line reports the I that ran and its measured time per step."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(args.ref_layers, threads)
        if i >= args.warmup:
            vals.append(cb)
    v = statistics.median(c["value"] for c in vals)
    step_s = statistics.median(c["seconds"] for c in vals)
    from paper_1410_5003_b200 import configs
    st, num, om, th, K, meta = configs.config(CFG, n_interfaces=args.ref_layers)
    cfg = workload_config(meta["I"], meta["N"], num, K, th, meta["seed"])
    cfg["workload"] = (f"cfg4 sample: the first {meta['I']} interfaces of the 1000-layer stack "
                       f"(N={meta['N']}, P={num.P}, Mw={num.Mw}, M={num.M}, K={K}, same seed)")
    cfg["sample_of"] = "cfg4, I=1000"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "layers/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64 complex)",
            "data": "synthetic (seeded, paper_1410_5003_b200/configs.py)",
            "config": cfg,
            "cpu_baseline": {k: vals[-1][k] for k in ("cores", "kind", "sample")} | {"value": v, "unit": "layers/s"},
            "e2e": {"value": v, "unit": "layers/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "kernel_evals_per_s": statistics.median(c["kernel_evals_per_s"] for c in vals)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--layers", type=int, default=None, help="override I (default: the config's 1000)")
    ap.add_argument("--ref-layers", type=int, default=8, help="I of the bounded CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 sweep measurement")
    ap.add_argument("--sweep-ref-angles", type=int, default=4, help="angles of the CPU reference sweep sample")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    from paper_1410_5003_b200 import configs
    from paper_1410_5003_b200.qpscat import Solver
    st, num, om, th, K, meta = configs.config(CFG, n_interfaces=args.layers)
    I, N = meta["I"], meta["N"]
    s = Solver(device=local)
    peaks = s.fp64_peaks()  # same-run FP64 microbenchmarks (north star)
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    for _ in range(args.warmup):
        s.solve()
    # ---- device-timed region (inputs resident in HBM) ----
    launches0 = s.launch_count()
    s.prof_reset()
    s.prof_enable(True)
    barrier(dist)
    totals = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            s.solve()
            totals.append(s.phase_times()["total_ms"])
        barrier(dist)
    s.prof_enable(False)
    launches = s.launch_count() - launches0
    stats = s.prof_stats()
    phases = s.phase_times()
    step_ms = allmax(dist, sum(totals) / len(totals))
    value = world * I / (step_ms * 1e-3)
    rt = s.reflection_transmission()
    diag = s.solver_diagnostics()
    evals = s.fill_evals()
    # dominant kernel family over the timed region (main-stream families: the
    # compression sample runs on a low-priority side stream and its events span
    # its overlap with the Schur chain, so its duration is not a kernel time)
    # the roofline family is the level-0 LU batch's GEMMs (lu_gemm), the
    # largest main-path tensor family; side-stream families (the compression
    # sample / sketch) span their overlap with other work and are excluded
    side = ("lr_sample", "lr_sketch", "zgemm_resid")
    dom = ("lu_gemm", stats["lu_gemm"]) if "lu_gemm" in stats else \
        max(((k, v) for k, v in stats.items() if k not in side and v["flops"] > 0), key=lambda kv: kv[1]["ms"])
    fams = {k: v for k, v in stats.items()}
    # zgemm_resid (the least squares' residual norms) runs on the low-priority
    # side stream: its event span covers its overlap with the A' update, so it
    # is kept out of the GEMM rate like the other side-stream families
    gemm_ms = sum(v["ms"] for k, v in fams.items() if k.startswith("zgemm") and k not in side)
    gemm_fl = sum(v["flops"] for k, v in fams.items() if k.startswith("zgemm") and k not in side)
    fill = {k: v for k, v in fams.items() if k.startswith("fill_")}
    fill_ms = sum(v["ms"] for v in fill.values())
    fill_units = sum(v["units"] for v in fill.values())
    peak = peaks["dmma_tflops"]
    dname, dv = dom
    d_tf = dv["flops"] / (dv["ms"] * 1e-3) / 1e12
    ncu = ncu_summary().get(dname, {})
    roofline = {"kernel": dname, "bound": "tensor", "achieved": d_tf, "peak": peak, "unit": "TFLOP/s",
                "frac": d_tf / peak,
                "traffic": ncu.get("dram_bytes"),
                "traffic_note": ncu.get("note"),
                "traffic_algorithmic_bytes": ncu.get("algorithmic_bytes") or
                (dv["bytes"] / max(1, dv["launches"]) if dv.get("bytes") else None),
                "peak_source": "FP64 DMMA (mma.sync m8n8k4 f64) microbenchmark in this run; bf16 peaks of "
                               "MEASURED_PEAKS.json do not apply to FP64",
                "algorithmic": "6*M*N*K real flops per complex GEMM task (3M Gauss product: three real DMMA "
                               "products per complex product), summed over the batched launches",
                "complex_equiv_tflops": d_tf * 8.0 / 6.0 if dv["flops"] else None,
                "launches": dv["launches"], "avg_launch_ms": dv["ms"] / max(1, dv["launches"])}
    fill_ncu = ncu_summary().get("fill_pair", {})
    # ---- end-to-end through the public API from host data ----
    sol = None
    for _ in range(args.warmup):  # untimed warm-up of the host path (first-touch of host buffers, thread pool)
        s.build_geometry(st, num)
        s.make_problem(om, th, K)
        s.solve()
        sol = s.solution(out=sol)
    barrier(dist)
    e2e_ms = []
    s.prof_reset()
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        s.build_geometry(st, num)
        s.make_problem(om, th, K)
        s.solve()
        sol = s.solution(out=sol)  # host result buffers reused across steps
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    xfer = s.transfer_bytes()
    e2e_step = allmax(dist, statistics.median(e2e_ms))
    e2e = {"value": world * I / (e2e_step * 1e-3), "unit": "layers/s",
           "h2d_bytes_per_step": xfer["h2d"] // max(1, len(e2e_ms)),
           "d2h_bytes_per_step": xfer["d2h"] // max(1, len(e2e_ms)), "ms_per_step": e2e_step}
    cb = None
    if rank == 0 and not args.no_cpu_baseline and os.path.exists(ORACLE):
        cb = cpu_baseline(args.ref_layers, os.cpu_count() or 1)
        cb = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    sweep = None
    if rank == 0 and not args.no_sweep:
        s.close()  # free the config-4 buffers: the sweep sizes its angle batches from free HBM
        sweep = sweep_measure(local, 0 if args.no_cpu_baseline else args.sweep_ref_angles)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "layers/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "c128 (f64 complex)",
                "data": "synthetic (seeded, paper_1410_5003_b200/configs.py)",
                "config": workload_config(I, N, num, K, th, meta["seed"]),
                "e2e": e2e, "roofline": roofline, "cpu_baseline": cb,
                "clocks": clk.summary(), "gpu_launches": launches,
                "phases_ms": {k: round(v, 3) for k, v in phases.items()},
                # reference fill_evals (assembly.hpp:285) per solve over the per-solve fill time
                "kernel_evals_per_s": evals["reference"] * args.steps / (fill_ms * 1e-3) if fill_ms else None,
                "fill_ms_per_step": fill_ms / args.steps,
                "fill_evals": evals, "fill_tflops_nominal": 200.0 * fill_units / (fill_ms * 1e-3) / 1e12
                if fill_ms else None,
                "fill_frac_of_dfma_peak": (200.0 * fill_units / (fill_ms * 1e-3) / 1e12) / peaks["dfma_tflops"]
                if fill_ms else None,
                "fill_fp64_frac_ncu": fill_ncu.get("fp64_frac_of_peak"),
                "fill_nominal_frac_ncu": fill_ncu.get("nominal_frac_of_peak"),
                "fill_fp64_ncu_note": fill_ncu.get("note"),
                "lr_basis_width": diag["lr_width"],
                "bcr_factor": dict(bcr_factor(phases, I, 2 * N, peak, diag["lr_width"]) or {},
                                   ncu={k: v for k, v in ncu_summary().get("bcr_level0", {}).items()
                                        if k not in ("command",)}),
                "gemm_tflops_issued": gemm_fl / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None,
                "gemm_tflops_complex_equiv": gemm_fl * 8.0 / 6.0 / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None,
                "fp64_peaks_tflops": peaks, "flux_error": rt["flux_error"], "R": rt["R"], "T": rt["T"],
                "sweep": sweep,
                "families_ms": {k: round(v["ms"] / args.steps, 3) for k, v in sorted(fams.items(),
                                                                                     key=lambda kv: -kv[1]["ms"])
                                if k not in side},
                "families_side_stream_span_ms": {k: round(v["ms"] / args.steps, 3) for k, v in fams.items()
                                                 if k in side},
                "families_note": "per-step event time of each main-stream kernel family; side-stream families "
                                 "(low-priority streams overlapping the main path) are listed separately because "
                                 "their event spans include the time they wait behind main-stream kernels and are "
                                 "not kernel durations (profiles/*_launches.csv has those)"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
