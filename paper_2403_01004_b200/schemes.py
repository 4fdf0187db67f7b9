"""Time integrators -- the SPEC ``schemes`` API.

  rkg2_iteration_count / rkl2_iteration_count    s formulas (host C, shared
                                                 with pc_cycle)
  rkg2_coefficients / rkl2_coefficients          StsCoefficients tables
  step_rkl2, step_rkg2, step_backward_euler, step_euler

RKL2 follows Meyer, Balsara & Aslam (2014) -- the "standard published
formulation" SPEC.md:279/:313 defers to; RKG2 is PAPER.md Appendix A with
alpha = 3/2.  Both share one fused stage kernel; the per-stage doubles
(mu, nu, 1-mu-nu, mu~ dt, gamma~ dt) come from ``pc_sts_table``.
"""
from __future__ import annotations

from ctypes import byref, c_double, c_int
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib, device
from .linsolve import SolveStats
from .mesh import Field


@dataclass
class SchemeConfig:
    """kind in {euler, backward_euler, rkl2, rkg2}."""

    kind: str = "rkl2"
    tol: float = 1e-10
    max_iter: int = 10000
    preconditioner: str = "jacobi"
    safety_factor: float = 1.0
    make_odd: bool = False  # RKL2 only: force odd s (RKG2 is always odd)

    def __post_init__(self):
        if self.kind not in ("euler", "backward_euler", "rkl2", "rkg2"):
            raise ValueError(f"unknown scheme {self.kind!r}")
        if self.kind == "backward_euler":
            if not (0.0 < self.tol < 1.0):
                raise ValueError("backward_euler needs 0 < tol < 1")
            if self.preconditioner not in ("jacobi", "line-r"):
                raise NotImplementedError("the device PCG implements point Jacobi (PC1) and the r-line "
                                          "block Jacobi ('line-r', the GPU substitute for PC2 ILU0)")

    @property
    def pc_code(self) -> int:
        return _lib.PC_LINE_R if self.preconditioner == "line-r" else _lib.PC_JACOBI

    @property
    def code(self) -> int:
        return {"rkl2": _lib.RKL2, "rkg2": _lib.RKG2, "backward_euler": _lib.BE, "euler": _lib.EULER}[self.kind]


@dataclass
class StsCoefficients:
    """s, w and per-stage arrays indexed 1..s (index 0 unused)."""

    kind: str
    s: int
    w: float
    mu: np.ndarray
    nu: np.ndarray
    mu_tilde: np.ndarray
    gamma: np.ndarray
    b: np.ndarray


def rkg2_iteration_count(dt: float, dt_euler: float) -> int:
    """s = ceil(sqrt(25 + 24 dt/dtE)/2 - 3/2), made odd, >= 3."""
    return int(_lib.lib().pc_sts_count(_lib.RKG2, float(dt), float(dt_euler), 0))


def rkl2_iteration_count(dt: float, dt_euler: float, make_odd: bool = False) -> int:
    """s = ceil((sqrt(9 + 16 dt/dtE) - 1)/2), >= 2 (stability |R| <= 1 for
    dt <= dtE (s^2+s-2)/4)."""
    return int(_lib.lib().pc_sts_count(_lib.RKL2, float(dt), float(dt_euler), int(make_odd)))


def sts_table(kind: str, s: int, dt: float) -> np.ndarray:
    """(s, 5) rows (mu, nu, 1-mu-nu, mu~ dt, gamma~ dt) exactly as the kernels use them."""
    out = np.empty(5 * s)
    code = _lib.RKL2 if kind == "rkl2" else _lib.RKG2
    _lib.check(_lib.lib().pc_sts_table(code, int(s), float(dt), _lib.dptr(out)), "sts_table")
    return out.reshape(s, 5)


def _b_rkg2(s):
    b = np.zeros(s + 1)
    b[0], b[1], b[2] = 1.0, 1.0 / 3.0, 1.0 / 15.0
    for k in range(3, s + 1):
        b[k] = ((4.0 * (k - 1.0)) * (k + 4.0)) / ((((3.0 * k) * (k + 1.0)) * (k + 2.0)) * (k + 3.0))
    return b


def _b_rkl2(s):
    b = np.zeros(s + 1)
    for j in range(s + 1):
        b[j] = 1.0 / 3.0 if j <= 2 else ((j * j + j) - 2.0) / ((2.0 * j) * (j + 1.0))
    return b


def _coefficients(kind, s):
    t = sts_table(kind, s, 1.0)
    pad = lambda col: np.concatenate([[0.0], t[:, col]])
    if kind == "rkg2":
        w = 6.0 / ((s + 4.0) * (s - 1.0))
        b = _b_rkg2(s)
    else:
        w = 4.0 / ((s * s + s) - 2.0)
        b = _b_rkl2(s)
    return StsCoefficients(kind, s, w, pad(0), pad(1), pad(3), pad(4), b)


def rkg2_coefficients(s: int) -> StsCoefficients:
    """PAPER.md Appendix A table; s must be odd and >= 3."""
    if s < 3 or s % 2 == 0:
        raise ValueError("RKG2 needs odd s >= 3")
    return _coefficients("rkg2", s)


def rkl2_coefficients(s: int) -> StsCoefficients:
    if s < 2:
        raise ValueError("RKL2 needs s >= 2")
    return _coefficients("rkl2", s)


# ---------------------------------------------------------------- steps

def _bind(op, u):
    if isinstance(u, device.DeviceField):
        raise TypeError("pass a mesh.Field, or use ptl.cycle_operator for device-resident fields")
    dop = op.device_op(u.grid, u.n_components)
    du = device.DeviceField.from_values(dop.dgrid, u.values)
    return dop, du


def _sts(op, u: Field, dt: float, dt_euler: float, kind: str) -> Field:
    if not dt > 0:
        raise ValueError("dt must be > 0")
    dop, du = _bind(op, u)
    s = rkl2_iteration_count(dt, dt_euler) if kind == "rkl2" else rkg2_iteration_count(dt, dt_euler)
    _lib.check(_lib.lib().pc_step_sts(dop.handle, du.handle, float(dt),
                                      _lib.RKL2 if kind == "rkl2" else _lib.RKG2, s, None), f"step_{kind}")
    return du.to_field()


def step_rkl2(op, u: Field, dt: float, dt_euler: float) -> Field:
    """One RKL2 step of dt."""
    return _sts(op, u, dt, dt_euler, "rkl2")


def step_rkg2(op, u: Field, dt: float, dt_euler: float) -> Field:
    """One RKG2 step of dt (Appendix A)."""
    return _sts(op, u, dt, dt_euler, "rkg2")


def step_euler(op, u: Field, dt: float) -> Field:
    """u + dt F(u)."""
    dop, du = _bind(op, u)
    _lib.check(_lib.lib().pc_step_euler(dop.handle, du.handle, float(dt)), "step_euler")
    return du.to_field()


def step_backward_euler(op, u: Field, dt: float, solver_cfg: SchemeConfig | None = None):
    """(I - dt J) u^{n+1} = u^n by PCG with x0 = u^n; point
    Jacobi, or the r-line preconditioner with SchemeConfig(preconditioner="line-r")."""
    cfg = solver_cfg or SchemeConfig("backward_euler")
    dop, du = _bind(op, u)
    it, rel, conv = c_int(), c_double(), c_int()
    _lib.check(_lib.lib().pc_op_set_preconditioner(dop.handle, cfg.pc_code), "preconditioner")
    _lib.check(_lib.lib().pc_step_be(dop.handle, du.handle, float(dt), float(cfg.tol), int(cfg.max_iter),
                                     byref(it), byref(rel), byref(conv)), "step_backward_euler")
    return du.to_field(), SolveStats(it.value, rel.value, bool(conv.value))
