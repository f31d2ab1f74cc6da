"""B200-native (sm_100a) implementation of the quasi-periodic multilayer
scattering hot path of Cho & Barnett (arXiv 1410.5003): Nystrom fill ->
per-layer least-squares Schur complements -> block cyclic reduction ->
Rayleigh-Bloch coefficients, plus the multi-angle sweep.  See DESIGN.md."""
from .qpscat import (BLOCKS, ConfigError, CudaError, DomainError, GeometryError, InterfaceSpec, LayerStack,
                     Material, MemoryBudgetError, NumericsParams, QpscatError, SingularityError, Solver,
                     SolverError, UsageError, load_library, solve_stack)

__all__ = ["BLOCKS", "ConfigError", "CudaError", "DomainError", "GeometryError", "InterfaceSpec", "LayerStack",
           "Material", "MemoryBudgetError", "NumericsParams", "QpscatError", "SingularityError", "Solver",
           "SolverError", "UsageError", "load_library", "solve_stack"]
