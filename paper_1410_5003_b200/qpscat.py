"""Host-side mirror of the reference's `qpscat` solver interface over the C-ABI
(include/qpscat_b200.h).

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/qpscat):
    LayerStack, Material, InterfaceSpec      geometry.hpp:273-296
    NumericsParams                           geometry.hpp:405-414
    build_geometry                           geometry.hpp:480-496
    make_problem                             assembly.hpp:69-82
    precompute_shift_blocks                  assembly.hpp:212-287
    assemble_system                          assembly.hpp:462-483
    schur_complement                         periodize.hpp:124-126
    block_lu_solve                           tridiag.hpp:23-46
    recover_aux / solve_periodized           tridiag.hpp:50-74
    flux_error / reflection_transmission     postprocess.hpp:134-180
and the exception taxonomy of errors.hpp:9-40.

`Solver()` binds the product library (paper_1410_5003_b200/libqpscat_b200.so,
host C++ + sm_100a CUDA).  There is no CPU fallback: if the library or a GPU
is missing, construction raises.  Tests bind the CPU oracle through the same
class by passing its path explicitly (`Solver(lib=...)`).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PRODUCT_LIB = os.environ.get("QPS_PRODUCT_LIB") or os.path.join(_HERE, "libqpscat_b200.so")  # override: dev A/B builds


# ---------------------------------------------------------------- errors
class QpscatError(RuntimeError):
    status = 9


class ConfigError(QpscatError):
    status = 1


class GeometryError(QpscatError):
    status = 2


class UsageError(QpscatError):
    status = 3


class SingularityError(QpscatError):
    status = 4


class SolverError(QpscatError):
    status = 5

    def __init__(self, msg, layer=0):
        super().__init__(msg)
        self.layer = layer


class MemoryBudgetError(QpscatError):
    status = 6

    def __init__(self, msg, required_bytes=0):
        super().__init__(msg)
        self.required_bytes = required_bytes


class DomainError(QpscatError, ValueError):
    status = 7


class CudaError(QpscatError):
    status = 8


_ERRS = {1: ConfigError, 2: GeometryError, 3: UsageError, 4: SingularityError, 5: SolverError,
         6: MemoryBudgetError, 7: DomainError, 8: CudaError, 9: QpscatError}

# ---------------------------------------------------------------- structs
SHAPES = {"sine": 0, "fourier": 1, "polyline": 2}


class _Cplx(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class _Spec(C.Structure):
    # qps_interface_spec; the array members are plain addresses (c_void_p has the
    # pointer ABI) so that the per-interface marshalling is integer arithmetic
    _fields_ = [("shape", C.c_int), ("offset", C.c_double), ("amplitude", C.c_double), ("phase", C.c_double),
                ("n_cos", C.c_int), ("cosc", C.c_void_p), ("n_sin", C.c_int),
                ("sinc", C.c_void_p), ("n_vertices", C.c_int), ("vertices", C.c_void_p),
                ("n_nodes", C.c_int), ("nodes", C.c_void_p), ("grading_q", C.c_int)]


class _Num(C.Structure):
    _fields_ = [("P", C.c_int), ("Mw", C.c_int), ("M", C.c_int), ("K", C.c_int), ("R", C.c_double),
                ("grading_q", C.c_int), ("clearance", C.c_double), ("memory_budget", C.c_uint64)]


class _Diag(C.Structure):
    _fields_ = [("bcr_path", C.c_int), ("lr_rank_max", C.c_int), ("lr_probe_worst", C.c_double),
                ("refine_steps", C.c_int), ("refine_res0", C.c_double), ("refine_res1", C.c_double),
                ("lr_width", C.c_int), ("lr_width_retry", C.c_int)]


class _Times(C.Structure):
    _fields_ = [("fill_ms", C.c_double), ("assemble_ms", C.c_double), ("schur_ms", C.c_double),
                ("solve_ms", C.c_double), ("recover_ms", C.c_double), ("total_ms", C.c_double),
                ("factor_ms", C.c_double)]


@dataclasses.dataclass
class Material:
    epsilon: float = 1.0
    mu: float = 1.0


@dataclasses.dataclass
class InterfaceSpec:
    shape: str = "sine"
    offset: float = 0.0
    amplitude: float = 0.0
    phase: float = 0.0
    cosc: List[float] = dataclasses.field(default_factory=list)
    sinc: List[float] = dataclasses.field(default_factory=list)
    vertices: List[tuple] = dataclasses.field(default_factory=list)
    nodes: List[int] = dataclasses.field(default_factory=list)
    grading_q: int = 6


@dataclasses.dataclass
class LayerStack:
    d: float = 1.0
    materials: List[Material] = dataclasses.field(default_factory=list)
    interfaces: List[InterfaceSpec] = dataclasses.field(default_factory=list)

    def n_interfaces(self):
        return len(self.interfaces)

    def n_layers(self):
        return len(self.materials)


@dataclasses.dataclass
class NumericsParams:
    P: int = 60
    Mw: int = 120
    M: int = 60
    K: int = 0
    R: float = 2.0
    grading_q: int = 6
    clearance: float = 0.05
    memory_budget: int = 4 << 30


BLOCKS = {name: i for i, name in enumerate(
    ["A_diag", "A_super", "A_sub", "B_self", "B_below", "C_self", "C_above", "Q", "Z_U", "Z_D", "V_U", "V_D",
     "W_U", "W_D", "f", "Bp_first", "Bp_last", "Cp_first", "Cp_last", "Qp_first", "Qp_last"])}
BLOCKS.update({name: 32 + i for i, name in enumerate(
    ["Ap_diag", "Ap_super", "Ap_sub", "X_first", "X_above", "X_self", "X_last"])})


def _bind(lib):
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "qps_abi_version": (C.c_int, []),
        "qps_backend_name": (C.c_char_p, []),
        "qps_create": (vp, [C.c_int]),
        "qps_destroy": (None, [vp]),
        "qps_last_error": (C.c_int, [vp, C.c_char_p, C.c_size_t, P(C.c_int), P(C.c_uint64)]),
        "qps_set_num_threads": (C.c_int, [vp, C.c_int]),
        "qps_set_qsolve_threshold": (C.c_int, [vp, C.c_double]),
        "qps_set_refine": (C.c_int, [vp, C.c_int]),
        "qps_build_geometry": (C.c_int, [vp, C.c_double, C.c_int, P(C.c_double), P(C.c_double), C.c_int,
                                         P(_Spec), P(_Num)]),
        "qps_make_problem": (C.c_int, [vp, C.c_double, C.c_double, C.c_int]),
        "qps_problem_info": (C.c_int, [vp, P(C.c_int), P(C.c_int), P(C.c_int), P(C.c_double), P(_Cplx),
                                       P(C.c_double), P(C.c_double)]),
        "qps_interface_nodes": (C.c_int, [vp, C.c_int, P(C.c_double), P(C.c_double), P(C.c_double),
                                          P(C.c_double)]),
        "qps_precompute_shift_blocks": (C.c_int, [vp]),
        "qps_assemble_system": (C.c_int, [vp]),
        "qps_schur_complement": (C.c_int, [vp]),
        "qps_block_lu_solve": (C.c_int, [vp]),
        "qps_recover_aux": (C.c_int, [vp]),
        "qps_block_lu_solve_blocks": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
        "qps_solve": (C.c_int, [vp]),
        "qps_get_solution": (C.c_int, [vp, vp, vp, vp, vp, P(C.c_double), P(C.c_double)]),
        "qps_reflection_transmission": (C.c_int, [vp, P(C.c_double), P(C.c_double), P(C.c_double),
                                                  P(C.c_double), vp, vp, P(C.c_int), P(C.c_int)]),
        "qps_evaluate_field": (C.c_int, [vp, C.c_int, P(C.c_double), vp, vp, P(C.c_int), P(C.c_int)]),
        "qps_sweep": (C.c_int, [vp, C.c_int, P(C.c_double), C.c_int, C.c_int, P(C.c_double), P(C.c_double),
                                P(C.c_double), vp, vp, P(C.c_int)]),
        "qps_set_solution": (C.c_int, [vp, vp, vp, vp, vp]),
        "qps_residual_suite": (C.c_int, [vp, C.c_int, P(C.c_int), P(C.c_double), P(C.c_double), P(C.c_double)]),
        "qps_interface_matching_residual": (C.c_int, [vp, C.c_int, C.c_int, P(C.c_double)]),
        "qps_plan_sweep": (C.c_int, [vp, C.c_int, C.c_double, C.c_double, C.c_int, P(C.c_double), P(C.c_int),
                                     P(C.c_int)]),
        "qps_sweep_info": (C.c_int, [vp, C.c_int, P(C.c_int), P(C.c_int), P(C.c_uint64), P(C.c_uint64)]),
        "qps_download_block": (C.c_int, [vp, C.c_int, C.c_int, vp, P(C.c_int), P(C.c_int)]),
        "qps_fill_evals": (C.c_int, [vp, P(C.c_uint64), P(C.c_uint64)]),
        "qps_get_phase_times": (C.c_int, [vp, P(_Times)]),
        "qps_solver_diagnostics": (C.c_int, [vp, P(_Diag)]),
        "qps_hankel01": (C.c_int, [vp, C.c_int, P(C.c_double), vp, vp]),
        "qps_measure_fp64_peaks": (C.c_int, [vp, P(C.c_double), P(C.c_double)]),
        "qps_prof_enable": (C.c_int, [vp, C.c_int]),
        "qps_prof_reset": (C.c_int, [vp]),
        "qps_prof_stats": (C.c_int, [vp, C.c_int, C.c_char_p, P(C.c_uint64), P(C.c_double), P(C.c_double),
                                     P(C.c_double), P(C.c_double)]),
        "qps_launch_count": (C.c_uint64, []),
        "qps_transfer_bytes": (C.c_int, [vp, P(C.c_uint64), P(C.c_uint64)]),
        "qps_qsolve": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, P(C.c_int)]),
        "qps_debug_zgemm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIBS = {}


def load_library(path: Optional[str] = None):
    """Load a library implementing include/qpscat_b200.h (default: the product)."""
    path = os.path.abspath(path or PRODUCT_LIB)
    if path not in _LIBS:
        if not os.path.exists(path):
            raise RuntimeError(
                f"qpscat_b200: native library {path} is missing; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        _LIBS[path] = _bind(C.CDLL(path))
    return _LIBS[path]


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Solver:
    """One solver context (one CUDA stream on the product library)."""

    def __init__(self, lib: Optional[str] = None, device: int = 0):
        self.lib = load_library(lib)
        self.backend = self.lib.qps_backend_name().decode()
        self.h = self.lib.qps_create(device)
        if not self.h:
            raise CudaError(f"qps_create failed on backend {self.backend} (no usable CUDA device {device}?)")
        self._keep = []
        self.stack = None
        self.num = None

    def close(self):
        if self.h:
            self.lib.qps_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -------------------------------------------------------------- errors
    def _check(self, st):
        if st == 0:
            return
        buf = C.create_string_buffer(1024)
        layer = C.c_int(0)
        nbytes = C.c_uint64(0)
        self.lib.qps_last_error(self.h, buf, 1024, C.byref(layer), C.byref(nbytes))
        msg = buf.value.decode(errors="replace")
        cls = _ERRS.get(st, QpscatError)
        if cls is SolverError:
            raise SolverError(msg, layer.value)
        if cls is MemoryBudgetError:
            raise MemoryBudgetError(msg, nbytes.value)
        raise cls(msg)

    # ------------------------------------------------------------ geometry
    def build_geometry(self, stack: LayerStack, num: NumericsParams):
        specs = (_Spec * len(stack.interfaces))()
        # every interface's arrays packed into one double and one int buffer
        dbl, ints, layout = [], [], []
        for sp in stack.interfaces:
            cos, sin = list(sp.cosc), list(sp.sinc)
            ver = [float(v) for xy in sp.vertices for v in (xy if hasattr(xy, "__len__") else (xy,))]
            nod = list(sp.nodes)
            layout.append((len(dbl), len(cos), len(sin), len(ver), len(ints), len(nod)))
            dbl += cos + sin + ver
            ints += nod
        dbuf = np.array(dbl + [0.0], dtype=np.float64)
        ibuf = np.array(ints + [0], dtype=np.int32)
        da, ia = dbuf.ctypes.data, ibuf.ctypes.data
        for s, sp, (d0, nc, ns_, nv, i0, nn) in zip(specs, stack.interfaces, layout):
            s.shape = SHAPES[sp.shape]
            s.offset, s.amplitude, s.phase = sp.offset, sp.amplitude, sp.phase
            s.n_cos, s.cosc = nc, da + 8 * d0
            s.n_sin, s.sinc = ns_, da + 8 * (d0 + nc)
            s.n_vertices, s.vertices = nv // 2, da + 8 * (d0 + nc + ns_)
            s.n_nodes, s.nodes = nn, ia + 4 * i0
            s.grading_q = sp.grading_q
        eps = np.array([m.epsilon for m in stack.materials], dtype=np.float64)
        mu = np.array([m.mu for m in stack.materials], dtype=np.float64)
        n = _Num(num.P, num.Mw, num.M, num.K, num.R, num.grading_q, num.clearance, num.memory_budget)
        self._check(self.lib.qps_build_geometry(self.h, stack.d, len(eps), _dptr(eps), _dptr(mu),
                                                len(stack.interfaces), specs, C.byref(n)))
        self.stack, self.num = stack, num
        return self

    def make_problem(self, omega: float, theta: float, K: int = 0):
        self._check(self.lib.qps_make_problem(self.h, omega, theta, K))
        return self.problem_info()

    def problem_info(self):
        nI = self.stack.n_interfaces()
        I = C.c_int()
        K = C.c_int()
        nn = np.zeros(nI, dtype=np.int32)
        k = np.zeros(nI + 1)
        alpha = _Cplx()
        yU = C.c_double()
        yD = C.c_double()
        self._check(self.lib.qps_problem_info(self.h, C.byref(I), C.byref(K), nn.ctypes.data_as(C.POINTER(C.c_int)),
                                              _dptr(k), C.byref(alpha), C.byref(yU), C.byref(yD)))
        return {"I": I.value, "K": K.value, "N": nn.tolist(), "k": k, "alpha": complex(alpha.re, alpha.im),
                "y_U": yU.value, "y_D": yD.value}

    def interface_nodes(self, j):
        N = self.problem_info()["N"][j]
        nodes = np.zeros((N, 2))
        normals = np.zeros((N, 2))
        w = np.zeros(N)
        sp = np.zeros(N)
        self._check(self.lib.qps_interface_nodes(self.h, j, _dptr(nodes), _dptr(normals), _dptr(w), _dptr(sp)))
        return nodes, normals, w, sp

    # ---------------------------------------------------------- hot path
    def precompute_shift_blocks(self):
        self._check(self.lib.qps_precompute_shift_blocks(self.h))

    def assemble_system(self):
        self._check(self.lib.qps_assemble_system(self.h))

    def schur_complement(self):
        self._check(self.lib.qps_schur_complement(self.h))

    def block_lu_solve(self):
        self._check(self.lib.qps_block_lu_solve(self.h))

    def block_lu_solve_blocks(self, Ad, Au, Al, f):
        """block_lu_solve on caller-built blocks (lists of n x n arrays); returns eta (I x n)."""
        I = len(Ad)
        n = Ad[0].shape[0]
        pack = lambda L: np.ascontiguousarray(np.stack([np.asfortranarray(a) for a in L]).transpose(0, 2, 1)
                                              if L else np.zeros((1, n, n)), dtype=np.complex128)
        A, U, Lo = pack(Ad), pack(Au), pack(Al)
        f = np.ascontiguousarray(f, dtype=np.complex128)
        eta = np.zeros((I, n), dtype=np.complex128)
        self._check(self.lib.qps_block_lu_solve_blocks(self.h, I, n, A.ctypes.data, U.ctypes.data, Lo.ctypes.data,
                                                       f.ctypes.data, eta.ctypes.data))
        return eta

    def recover_aux(self):
        self._check(self.lib.qps_recover_aux(self.h))

    def solve_periodized(self):
        self.schur_complement()
        self.block_lu_solve()
        self.recover_aux()

    def solve(self):
        """One-shot: fill + Schur + block solve + recovery."""
        self._check(self.lib.qps_solve(self.h))

    def set_num_threads(self, n):
        self._check(self.lib.qps_set_num_threads(self.h, n))

    def set_qsolve_threshold(self, th):
        self._check(self.lib.qps_set_qsolve_threshold(self.h, th))

    def set_refine(self, steps: int):
        """Iterative-refinement steps of the block solve (-1: default, 0 for
        solves and 1 for sweeps; the oracle ignores it)."""
        self._check(self.lib.qps_set_refine(self.h, int(steps)))

    # ------------------------------------------------------------ outputs
    def solution(self, out=None):
        """The last solve's Solution.  `out`: a previous result of this call
        whose arrays are overwritten in place (repeated solves of one
        configuration skip the allocation and first-touch of 10 MB)."""
        info = self.problem_info()
        ntot = 2 * sum(info["N"])
        nrb = 2 * info["K"] + 1
        if out is not None and out["eta_flat"].size == ntot and out["aU"].size == nrb and \
                out["c"].size == (info["I"] + 1) * self.num.P:
            eta, c, aU, aD, lsq = out["eta_flat"], out["c"], out["aU"], out["aD"], out["lsq_residual"]
        else:
            eta = np.zeros(ntot, dtype=np.complex128)
            c = np.zeros((info["I"] + 1) * self.num.P, dtype=np.complex128)
            aU = np.zeros(nrb, dtype=np.complex128)
            aD = np.zeros(nrb, dtype=np.complex128)
            lsq = np.zeros(info["I"] + 1)
        mx = C.c_double()
        self._check(self.lib.qps_get_solution(self.h, eta.ctypes.data, c.ctypes.data, aU.ctypes.data,
                                              aD.ctypes.data, _dptr(lsq), C.byref(mx)))
        offs = np.cumsum([0] + [2 * n for n in info["N"]])
        return {"eta": [eta[offs[j]:offs[j + 1]] for j in range(info["I"])], "eta_flat": eta,
                "c": c.reshape(info["I"] + 1, self.num.P), "aU": aU, "aD": aD, "lsq_residual": lsq,
                "max_lsq_residual": mx.value}

    def reflection_transmission(self):
        info = self.problem_info()
        nrb = 2 * info["K"] + 1
        R = C.c_double()
        T = C.c_double()
        fe = C.c_double()
        kappa = np.zeros(nrb)
        kU = np.zeros(nrb, dtype=np.complex128)
        kD = np.zeros(nrb, dtype=np.complex128)
        pu = np.zeros(nrb, dtype=np.int32)
        pd = np.zeros(nrb, dtype=np.int32)
        self._check(self.lib.qps_reflection_transmission(
            self.h, C.byref(R), C.byref(T), C.byref(fe), _dptr(kappa), kU.ctypes.data, kD.ctypes.data,
            pu.ctypes.data_as(C.POINTER(C.c_int)), pd.ctypes.data_as(C.POINTER(C.c_int))))
        return {"R": R.value, "T": T.value, "flux_error": fe.value, "kappa": kappa, "kU": kU, "kD": kD,
                "prop_up": pu.astype(bool), "prop_down": pd.astype(bool)}

    def flux_error(self):
        return self.reflection_transmission()["flux_error"]

    def sweep(self, thetas: Sequence[float], K: int, mode: int = 0):
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        n = len(th)
        nrb = 2 * K + 1
        R = np.zeros(n)
        T = np.zeros(n)
        fe = np.zeros(n)
        aU = np.zeros((n, nrb), dtype=np.complex128)
        aD = np.zeros((n, nrb), dtype=np.complex128)
        st = np.zeros(n, dtype=np.int32)
        self._check(self.lib.qps_sweep(self.h, n, _dptr(th), K, mode, _dptr(R), _dptr(T), _dptr(fe),
                                       aU.ctypes.data, aD.ctypes.data, st.ctypes.data_as(C.POINTER(C.c_int))))
        return {"R": R, "T": T, "flux_error": fe, "aU": aU, "aD": aD, "status": st}

    def set_solution(self, eta, c, aU, aD):
        """Load a Solution (tridiag.hpp:11-17) for post-processing: eta flat
        [tau_0; sigma_0; tau_1; ...], c (I+1, P), aU, aD (2K+1)."""
        arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.complex128).ravel()) for a in (eta, c, aU, aD)]
        self._check(self.lib.qps_set_solution(self.h, *[a.ctypes.data for a in arrs]))

    def residual_suite(self, interfaces):
        """ResidualReport of the current solution (residual_suite,
        postprocess.hpp:369-399): dict(wall_qp, radiation, interface)."""
        ifs = np.ascontiguousarray(interfaces, dtype=np.int32)
        w, r, i = C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.qps_residual_suite(self.h, len(ifs), ifs.ctypes.data_as(C.POINTER(C.c_int)),
                                                C.byref(w), C.byref(r), C.byref(i)))
        return {"wall_qp": w.value, "radiation": r.value, "interface": i.value}

    def interface_matching_residual(self, j: int, n_probe: int = 4):
        out = C.c_double()
        self._check(self.lib.qps_interface_matching_residual(self.h, j, n_probe, C.byref(out)))
        return out.value

    def plan_sweep(self, n_alpha: int, theta_lo: float, theta_hi: float):
        """plan_sweep(omega, n, theta_range): angles on the grid
        uniform in k_1 cos(theta) with n distinct alphas; returns (thetas,
        alpha_group) for the last make_problem's k_1."""
        cnt = C.c_int()
        self._check(self.lib.qps_plan_sweep(self.h, n_alpha, theta_lo, theta_hi, 0, None, None, C.byref(cnt)))
        th = np.zeros(cnt.value)
        grp = np.zeros(cnt.value, dtype=np.int32)
        self._check(self.lib.qps_plan_sweep(self.h, n_alpha, theta_lo, theta_hi, cnt.value, _dptr(th),
                                            grp.ctypes.data_as(C.POINTER(C.c_int)), C.byref(cnt)))
        return th, grp

    def sweep_info(self, n: int):
        """Last sweep: per-angle alpha_group (SpectrumRow::alpha_group), n_groups,
        interior eliminations and block factorizations performed."""
        grp = np.zeros(n, dtype=np.int32)
        ng = C.c_int()
        ni = C.c_uint64()
        nf = C.c_uint64()
        self._check(self.lib.qps_sweep_info(self.h, n, grp.ctypes.data_as(C.POINTER(C.c_int)), C.byref(ng),
                                            C.byref(ni), C.byref(nf)))
        return {"alpha_group": grp, "n_groups": ng.value, "n_interior": ni.value, "n_factorizations": nf.value}

    def evaluate_field(self, points):
        """evaluate_field(sol, p, points) (postprocess.hpp:78-123) for the last
        solve: points (n, 2) -> dict(u_scattered, u_total, region, layer);
        region 0 above y_U, 1 inside a layer, 2 below y_D."""
        xy = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 2))
        n = len(xy)
        us = np.zeros(n, dtype=np.complex128)
        ut = np.zeros(n, dtype=np.complex128)
        reg = np.zeros(n, dtype=np.int32)
        lay = np.zeros(n, dtype=np.int32)
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
        self._check(self.lib.qps_evaluate_field(self.h, n, _dptr(xy), us.ctypes.data, ut.ctypes.data, ip(reg),
                                                ip(lay)))
        return {"u_scattered": us, "u_total": ut, "region": reg, "layer": lay}

    def download_block(self, name: str, i: int = 0):
        kind = BLOCKS[name]
        r = C.c_int()
        c = C.c_int()
        self._check(self.lib.qps_download_block(self.h, kind, i, None, C.byref(r), C.byref(c)))
        out = np.zeros((c.value, r.value), dtype=np.complex128)  # column-major storage
        if r.value and c.value:
            self._check(self.lib.qps_download_block(self.h, kind, i, out.ctypes.data, C.byref(r), C.byref(c)))
        return out.T

    def fill_evals(self):
        a = C.c_uint64()
        b = C.c_uint64()
        self._check(self.lib.qps_fill_evals(self.h, C.byref(a), C.byref(b)))
        return {"reference": a.value, "performed": b.value}

    def phase_times(self):
        t = _Times()
        self._check(self.lib.qps_get_phase_times(self.h, C.byref(t)))
        return {f: getattr(t, f) for f, _ in _Times._fields_}

    def solver_diagnostics(self):
        """How the last block solve ran: bcr_path (-1 reference Thomas, 0 dense
        cyclic reduction, 1 low-rank Woodbury, 2 low-rank per-level LU),
        lr_rank_max, lr_probe_worst (a-posteriori compression test)."""
        d = _Diag()
        self._check(self.lib.qps_solver_diagnostics(self.h, C.byref(d)))
        return {f: getattr(d, f) for f, _ in _Diag._fields_}

    def hankel01(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        h0 = np.zeros(len(x), dtype=np.complex128)
        h1 = np.zeros(len(x), dtype=np.complex128)
        self._check(self.lib.qps_hankel01(self.h, len(x), _dptr(x), h0.ctypes.data, h1.ctypes.data))
        return h0, h1

    def prof_enable(self, on=True):
        self._check(self.lib.qps_prof_enable(self.h, int(on)))

    def prof_reset(self):
        self._check(self.lib.qps_prof_reset(self.h))

    def prof_stats(self):
        cap = 64
        names = C.create_string_buffer(64 * cap)
        la = (C.c_uint64 * cap)()
        arrs = [(C.c_double * cap)() for _ in range(4)]
        n = self.lib.qps_prof_stats(self.h, cap, names, la, *arrs)
        out = {}
        for i in range(min(n, cap)):
            nm = names.raw[64 * i:64 * (i + 1)].split(b"\0")[0].decode()
            out[nm] = {"launches": la[i], "ms": arrs[0][i], "flops": arrs[1][i], "bytes": arrs[2][i],
                       "units": arrs[3][i]}
        return out

    def launch_count(self):
        return int(self.lib.qps_launch_count())

    def transfer_bytes(self):
        a = C.c_uint64()
        b = C.c_uint64()
        self._check(self.lib.qps_transfer_bytes(self.h, C.byref(a), C.byref(b)))
        return {"h2d": a.value, "d2h": b.value}

    def qsolve(self, Q, rhs):
        """qsolve (periodize.hpp:25-39); returns (X, rank)."""
        Q = np.asfortranarray(Q, dtype=np.complex128)
        rhs = np.asfortranarray(rhs, dtype=np.complex128)
        m, p = Q.shape
        n = rhs.shape[1]
        X = np.zeros((p, n), dtype=np.complex128, order="F")
        r = C.c_int(0)
        self._check(self.lib.qps_qsolve(self.h, m, p, n, Q.ctypes.data, rhs.ctypes.data, X.ctypes.data, C.byref(r)))
        return X, r.value

    def debug_zgemm(self, A, B):
        A = np.asfortranarray(A, dtype=np.complex128)
        B = np.asfortranarray(B, dtype=np.complex128)
        M, K = A.shape
        N = B.shape[1]
        Cm = np.zeros((M, N), dtype=np.complex128, order="F")
        self._check(self.lib.qps_debug_zgemm(self.h, M, N, K, A.ctypes.data, B.ctypes.data, Cm.ctypes.data))
        return Cm

    def fp64_peaks(self):
        a = C.c_double()
        b = C.c_double()
        self._check(self.lib.qps_measure_fp64_peaks(self.h, C.byref(a), C.byref(b)))
        return {"dfma_tflops": a.value, "dmma_tflops": b.value}


def solve_stack(stack: LayerStack, num: NumericsParams, omega: float, theta: float, K: int = 0,
                lib: Optional[str] = None, solver: Optional[Solver] = None):
    """The reference test drivers' `solve_stack` (proj/tests/test_tridiag.cpp:112-126)."""
    s = solver or Solver(lib)
    s.build_geometry(stack, num)
    s.make_problem(omega, theta, K)
    s.solve()
    return s
