"""Jacobi-preconditioned conjugate gradient -- the SPEC ``linsolve`` API
 on the device.

  LinearOperatorAction   A = diag(a) - dt J, J the frozen operator's Jacobian
                         (a = 1 for the Backward-Euler system I - dt J)
  build_jacobi(A)        inverse diagonal, error if any entry <= 0
  pcg_solve(A, b, M, x0, tol, max_iter) -> (Field, SolveStats)

The inner product is the rho*V-weighted one in which A is symmetric
(SPEC.md:167, :186, :219); convergence ||b - A x||_w / ||b||_w <= tol is
tested after every iteration on the device (no per-iteration host sync).
ILU0 (PC2) is out of scope on the GPU.
"""
from __future__ import annotations

from ctypes import byref, c_double, c_int
from dataclasses import dataclass

import numpy as np

from . import _lib, device
from .errors import IndefiniteOperatorError
from .mesh import Field


@dataclass
class SolveStats:
    iterations: int
    final_relative_residual: float
    converged: bool


@dataclass
class LinearOperatorAction:
    """y = (a - dt J) x for a frozen DiffusionOperator (a: Field/array or None == 1)."""

    op: object
    dt: float
    a: object = None

    def apply(self, x: Field) -> Field:
        """Host convenience (device evaluation of a x - dt F(x))."""
        F = self.op.apply(x).values
        a = 1.0 if self.a is None else np.asarray(getattr(self.a, "values", self.a), float).reshape(x.values.shape[:-1] + (1,))
        return Field(x.grid, a * x.values - self.dt * F)


@dataclass
class Preconditioner:
    kind: str
    inv_diagonal: np.ndarray | None = None


def build_jacobi(A: LinearOperatorAction, grid=None, ncomp: int = 1) -> Preconditioner:
    """Point-Jacobi (PC1): stored inverse diagonal of A."""
    fs = getattr(A.op, "frozen_state", None)
    if grid is None and fs is not None:
        grid = fs.dgrid.grid if hasattr(fs, "dgrid") else fs.grid
    if grid is None:
        raise ValueError("build_jacobi needs the grid of the system")
    dop = A.op.device_op(grid, ncomp)
    dneg = dop.diagonal().download()[..., 0].reshape(tuple(grid.shape))
    a = 1.0 if A.a is None else np.asarray(getattr(A.a, "values", A.a), float).reshape(tuple(grid.shape))
    diag = a + A.dt * dneg
    if np.any(~(diag > 0)):
        raise IndefiniteOperatorError("non-positive diagonal entry in the Jacobi preconditioner")
    return Preconditioner("jacobi", 1.0 / diag)


def build_ilu0(*_a, **_k):
    raise NotImplementedError("ILU0 (PC2) is sequential by contract (SPEC.md:222) and out of scope on the GPU")


def pcg_solve(A: LinearOperatorAction, b: Field, M: Preconditioner | None, x0: Field, tol: float,
              max_iter: int):
    """SPEC.md:183-191.  M must be point-Jacobi (applied on the device)."""
    if M is not None and M.kind != "jacobi":
        raise NotImplementedError("only the point-Jacobi preconditioner runs on the device")
    if not (0.0 < tol < 1.0) or max_iter < 1:
        raise ValueError("need 0 < tol < 1 and max_iter >= 1")
    grid = b.grid
    nc = b.n_components
    dop = A.op.device_op(grid, nc)
    db = device.DeviceField.from_values(dop.dgrid, b.values)
    dx = device.DeviceField.from_values(dop.dgrid, x0.values)
    da = None
    if A.a is not None:
        av = np.asarray(getattr(A.a, "values", A.a), float).reshape(tuple(grid.shape))
        if np.any(~(av + A.dt * dop.diagonal().download()[..., 0].reshape(av.shape) > 0)):
            raise IndefiniteOperatorError("non-positive diagonal entry in the Jacobi preconditioner")
        da = device.DeviceField.from_values(dop.dgrid, av)
    it, rel, conv = c_int(), c_double(), c_int()
    _lib.check(_lib.lib().pc_pcg_solve(dop.handle, float(A.dt), da.handle if da is not None else None,
                                       db.handle, dx.handle, float(tol), int(max_iter), byref(it), byref(rel),
                                       byref(conv)), "pcg_solve")
    return dx.to_field(), SolveStats(it.value, rel.value, bool(conv.value))
