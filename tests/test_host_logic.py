"""Host-side logic of the product (host-only context, no GPU) against the
reference's own host code in the oracle: discretisation bit-identity
(geometry.hpp:114-200,423-496), problem setup (assembly.hpp:43-82), the fill
count (assembly.hpp:285) and the error taxonomy (errors.hpp:9-40)."""
import math

import numpy as np
import pytest

from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.configs import MT19937_64
from paper_1410_5003_b200.qpscat import (ConfigError, GeometryError, InterfaceSpec, LayerStack, Material,
                                         MemoryBudgetError, NumericsParams)

CASES = [(1, None), (2, None), (3, 6), (4, 12), (5, 9)]


def test_mt19937_64_known_answer():
    r = MT19937_64(5489)
    for _ in range(9999):
        r.next()
    assert r.next() == 9981545732273789042  # C++11 [rand.predef]


@pytest.mark.parametrize("cfg,nif", CASES)
def test_geometry_bit_identical(host, oracle, cfg, nif):
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
    for s in (host, oracle):
        s.build_geometry(st, num)
        s.make_problem(om, th, K)
    gi, oi = host.problem_info(), oracle.problem_info()
    assert gi["N"] == oi["N"] and gi["K"] == oi["K"]
    assert gi["alpha"] == oi["alpha"] and np.array_equal(gi["k"], oi["k"])
    assert gi["y_U"] == oi["y_U"] and gi["y_D"] == oi["y_D"]
    for j in range(gi["I"]):
        for a, b in zip(host.interface_nodes(j), oracle.interface_nodes(j)):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg,nif", CASES)
def test_reference_fill_count(host, oracle, cfg, nif):
    st, num, om, th, K, _ = configs.config(cfg, n_interfaces=nif)
    for s in (host, oracle):
        s.build_geometry(st, num)
        s.make_problem(om, th, K)
        s.precompute_shift_blocks()
    assert host.fill_evals()["reference"] == oracle.fill_evals()["reference"]


def test_fill_counts_match_survey(host):
    # 108,520 (cfg 1), 1,541,600 (cfg 2), 1.189e9 (cfg 4)
    for cfg, want in [(1, 108520), (2, 1541600), (4, 1188944000)]:
        st, num, om, th, K, _ = configs.config(cfg)
        host.build_geometry(st, num)
        host.make_problem(om, th, K)
        host.precompute_shift_blocks()
        assert host.fill_evals()["reference"] == want


def test_auto_rb_order_matches(host, oracle):
    st, num, om, th, K, _ = configs.config(2)
    for s in (host, oracle):
        s.build_geometry(st, num)
    for theta in (-0.3, -math.pi / 5, -1.2, -2.9):
        assert host.make_problem(om, theta, 0)["K"] == oracle.make_problem(om, theta, 0)["K"]


def _expect_same_error(host, oracle, fn, exc):
    for s in (host, oracle):
        with pytest.raises(exc):
            fn(s)


def test_error_taxonomy(host, oracle):
    num = NumericsParams(P=40, Mw=30, M=24, R=1.8, clearance=0.25)
    two = [Material(1, 1), Material(2, 1)]
    few = LayerStack(1.0, two, [InterfaceSpec("sine", 0.0, 0.1, 0.0, nodes=[6])])
    _expect_same_error(host, oracle, lambda s: s.build_geometry(few, num), ConfigError)
    badpoly = LayerStack(1.0, two, [InterfaceSpec("polyline", 0.0, vertices=[(-0.4, 0), (0.5, 0)], nodes=[20])])
    _expect_same_error(host, oracle, lambda s: s.build_geometry(badpoly, num), ConfigError)
    uneven = LayerStack(1.0, two, [InterfaceSpec("polyline", 0.0, vertices=[(-0.5, 0), (0.5, 0.1)], nodes=[20])])
    _expect_same_error(host, oracle, lambda s: s.build_geometry(uneven, num), ConfigError)
    crossing = LayerStack(1.0, [Material(1, 1)] * 3,
                          [InterfaceSpec("sine", 0.0, 0.2, 0.0, nodes=[40]),
                           InterfaceSpec("sine", 0.3, 0.0, 0.0, nodes=[40])])
    _expect_same_error(host, oracle, lambda s: s.build_geometry(crossing, num), GeometryError)
    layers = LayerStack(1.0, [Material(1, 1)], [InterfaceSpec("sine", 0.0, 0.1, 0.0, nodes=[40])])
    _expect_same_error(host, oracle, lambda s: s.build_geometry(layers, num), ConfigError)
    ok = LayerStack(1.0, two, [InterfaceSpec("sine", 0.0, 0.1, 0.0, nodes=[40])])
    for s in (host, oracle):
        s.build_geometry(ok, num)
    _expect_same_error(host, oracle, lambda s: s.make_problem(3.0, 0.3, 8), ConfigError)
    _expect_same_error(host, oracle, lambda s: s.make_problem(3.0, -math.pi, 8), ConfigError)


def test_memory_budget_error_reports_same_bytes(host, oracle):
    st, num, om, th, K, _ = configs.config(2)
    num.memory_budget = 1 << 20
    got = []
    for s in (host, oracle):
        s.build_geometry(st, num)
        s.make_problem(om, th, K)
        with pytest.raises(MemoryBudgetError) as e:
            s.precompute_shift_blocks()
        got.append(e.value.required_bytes)
    assert got[0] == got[1] > (1 << 20)


def test_solvability_checks(host, oracle):
    """assembly.hpp:471-474 (2 Mw >= P) and alpert_min_nodes (kernels.hpp:183-185)."""
    two = [Material(1, 1), Material(2, 1)]
    ok = LayerStack(1.0, two, [InterfaceSpec("sine", 0.0, 0.1, 0.0, nodes=[40])])
    bad = NumericsParams(P=70, Mw=30, M=24, R=1.8, clearance=0.25)
    for s in (host, oracle):
        s.build_geometry(ok, bad)
        s.make_problem(3.0, -1.0, 8)
        s.precompute_shift_blocks()  # the reference checks solvability only at assembly
    with pytest.raises(ConfigError):
        oracle.assemble_system()
    with pytest.raises(ConfigError):
        host.solve()
    short = LayerStack(1.0, two, [InterfaceSpec("sine", 0.0, 0.1, 0.0, nodes=[30])])
    good = NumericsParams(P=40, Mw=30, M=24, R=1.8, clearance=0.25)
    for s in (host, oracle):
        s.build_geometry(short, good)
        s.make_problem(3.0, -1.0, 8)
        with pytest.raises(ConfigError):
            s.precompute_shift_blocks()


def test_plan_sweep_grid_matches_oracle(host, oracle):
    """plan_sweep: identical angle grids and alpha groups
    (j mod n) from the product's host code and the oracle; every group's
    angles share alpha = exp(i d k_1 cos theta) to 1e-12."""
    st, num, om, th, K, _ = configs.config(5, n_interfaces=3)
    for s in (host, oracle):
        s.build_geometry(st, num)
        s.make_problem(om, th, K)
    tg, gg = host.plan_sweep(4, -math.pi + 0.1, -0.1)
    to, go = oracle.plan_sweep(4, -math.pi + 0.1, -0.1)
    assert np.array_equal(tg, to) and np.array_equal(gg, go)
    assert len(tg) >= 8 and np.all(np.diff(tg) > 0) and np.all((tg > -math.pi) & (tg < 0))
    alpha = np.exp(1j * st.d * om * np.cos(tg))
    for g in range(4):
        a = alpha[gg == g]
        assert np.abs(a - a[0]).max() < 1e-12
    with pytest.raises(ConfigError):
        host.plan_sweep(0, -1.0, -0.5)
    with pytest.raises(ConfigError):
        oracle.plan_sweep(2, -0.5, -1.0)
