"""paper_2403_01004_b200 -- B200-native PTL-cycled parabolic-operator advance.

Drop-in for the hot path of the reference ``paracycle`` package
(arXiv:2403.01004; SPEC.md ``operators``/``linsolve``/``schemes``/``ptl``):
the same entry points, arguments and returned fields / cycle reports, executed
by hand-written fp64 sm_100a kernels behind a C ABI (include/paracycle_b200.h).

Modules mirror the reference layout:
  mesh        Grid / Field / BoundaryCondition (+ spherical metric, 'axis' kind)
  operators   apply_scalar_diffusion, apply_aligned_conduction, estimate_euler_dt
  linsolve    pcg_solve, build_jacobi, SolveStats
  schemes     step_rkl2, step_rkg2, step_backward_euler, step_euler, coefficients
  ptl         compute_ptl, cycle_operator, split_advance, CycleReport
  device      Context / DeviceGrid / DeviceField (HBM-resident state)
  configs     seeded BASELINE C1-C5 inputs
"""
from . import mesh  # noqa: F401

__all__ = ["mesh", "operators", "linsolve", "schemes", "ptl", "device", "configs", "geometry"]
__version__ = "0.1.0"
