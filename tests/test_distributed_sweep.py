"""Angle sharding across ranks (paper_1410_5003_b200/sweep.py) on CPU with the
gloo backend, world size 2: the sharded sweep returns exactly the
single-process sweep (angles are independent; each rank refills its own
alpha-free cache with identical arithmetic).  The per-rank solver is the CPU
oracle library here (test infrastructure; the GPU product runs the same host
logic through libqpscat_b200.so)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.sweep import shard_bounds, sharded_sweep

THETAS = [-2.9, -2.2, -1.6, -0.9, -0.3]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(s, thetas):
    st, num, om, th, K, _ = configs.config(1)
    s.build_geometry(st, num)
    s.make_problem(om, th, K)
    return sharded_sweep(s, thetas, K, mode=0), K


def _worker(rank, world, port, lib, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1410_5003_b200.qpscat import Solver
        s = Solver(lib=lib)
        r, _ = _run(s, THETAS)
        if rank == 0:
            np.savez(out, **r)
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover():
    for n in (0, 1, 5, 200):
        for w in (1, 2, 3, 8):
            seen = []
            for r in range(w):
                lo, hi = shard_bounds(n, r, w)
                seen.extend(range(lo, hi))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def test_sharded_sweep_gloo_world2(oracle_lib, tmp_path):
    out = str(tmp_path / "r.npz")
    mp.start_processes(_worker, args=(2, _free_port(), oracle_lib, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    from paper_1410_5003_b200.qpscat import Solver
    ref, _ = _run(Solver(lib=oracle_lib), THETAS)
    for k in ("R", "T", "flux_error", "aU", "aD", "status"):
        assert np.array_equal(got[k], ref[k]), k
