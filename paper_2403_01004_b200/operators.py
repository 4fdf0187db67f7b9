"""Right-hand sides F(u) of the two parabolic operator families of Eq. 2 and
the explicit-Euler step estimate -- the SPEC ``operators`` API
 executed by the sm_100a kernels behind the C ABI.

  apply_scalar_diffusion(u, cfg) -> Field
  apply_aligned_conduction(T, cfg, T0) -> Field
  estimate_euler_dt(op, probe) -> float
  DiffusionOperator (scalar | aligned, frozen T0)

Discretisation: conservative rho-weighted 7-point finite
volumes with arithmetic face averages of nu*rho; the field-aligned operator is
the symmetric 19-point corner-tetrahedron stencil; on spherical grids a
3-component field with ``vector_metric`` gets the vector-Laplacian metric
terms (frame rotation).
"""
from __future__ import annotations

import math
from ctypes import byref, c_double, c_void_p
from dataclasses import dataclass, field as dc_field
from typing import Any

import numpy as np

from . import _lib, device, mesh
from .mesh import Field, BoundaryCondition


def _values(x, grid, name, ncomp=None):
    """Field / array / scalar -> grid-shaped ndarray (component axis kept if ncomp>1)."""
    if isinstance(x, (int, float)):
        return float(x)
    v = np.asarray(getattr(x, "values", x), dtype=float)
    shape = tuple(grid.shape)
    if ncomp is None:
        if v.shape == shape + (1,):
            v = v[..., 0]
        if v.shape != shape:
            raise ValueError(f"{name}: shape {v.shape} does not match grid {shape}")
    return v


def _positive_field(dg, values):
    """Upload a density and validate it on the device: ValueError if any node
    has !(rho > 0).  One counting pass over HBM instead of a
    host-side ``np.any(~(rho > 0))`` over the whole array (~0.5 s at C5)."""
    rd = device.DeviceField.from_values(dg, values)
    if rd.count_failing(_lib.TEST_POSITIVE):
        raise ValueError("rho must be > 0")
    return rd


@dataclass
class ScalarDiffusionConfig:
    """F = (1/rho) div(nu rho grad u).  ``nu`` and ``rho`` are
    Fields or constants (rho None == 1).  ``vector_metric`` applies the
    spherical vector-Laplacian metric terms to a 3-component field."""

    nu: Any
    rho: Any = None
    bc: BoundaryCondition | None = None
    vector_metric: bool = False


def tanh_cutoff(r0: float, width: float):
    """f_c preset ``tanh-cutoff(r0, width)`` = (1 - tanh((r - r0)/width))/2
    (our own preset; the paper gives no form)."""
    return ("tanh-cutoff", float(r0), float(width))


@dataclass
class AlignedConductionConfig:
    """F = ((gamma-1) m_p / (2 k rho)) div(f_c f_m(T0) kappa0 T0^{5/2} b b . grad T)
    (SPEC.md:94-99).  f_c: 'one', tanh_cutoff(r0, width), or a callable of the
    axis-0 coordinate; f_m: 'one'."""

    b_hat: Any
    kappa0: float = 1.0
    gamma: float = 5.0 / 3.0
    m_p: float = 1.0
    k_B: float = 1.0
    f_c: Any = "one"
    f_m: Any = "one"
    rho: Any = None
    bc: BoundaryCondition | None = None
    T_floor: float = 1e-10

    @property
    def prefactor(self) -> float:
        return (self.gamma - 1.0) * self.m_p / (2.0 * self.k_B)

    def fc_table(self, r: np.ndarray) -> np.ndarray | None:
        if isinstance(self.f_c, str):
            if self.f_c != "one":
                raise ValueError(f"unknown f_c preset {self.f_c!r}")
            return None
        if isinstance(self.f_c, tuple) and self.f_c[0] == "tanh-cutoff":
            _, r0, w = self.f_c
            return np.array([0.5 * (1.0 - math.tanh((x - r0) / w)) for x in r])
        if callable(self.f_c):
            return np.asarray([float(self.f_c(x)) for x in r])
        raise ValueError(f"unknown f_c preset {self.f_c!r}")


class DiffusionOperator:
    """Tagged union {scalar, aligned} plus the lagged state T0.

    The operator binds to a grid on first use; ``device_op(grid)`` returns the
    resident C-ABI operator for the current context."""

    def __init__(self, kind: str, config, frozen_state: Field | None = None, ncomp: int | None = None):
        if kind not in ("scalar", "aligned"):
            raise ValueError(f"unknown operator kind {kind!r}")
        self.kind = kind
        self.config = config
        self.frozen_state = frozen_state
        self.ncomp = ncomp
        self._dev = {}

    @classmethod
    def scalar(cls, cfg: ScalarDiffusionConfig, ncomp: int | None = None) -> "DiffusionOperator":
        return cls("scalar", cfg, ncomp=ncomp)

    @classmethod
    def aligned(cls, cfg: AlignedConductionConfig, T0: Field | None = None) -> "DiffusionOperator":
        return cls("aligned", cfg, T0, ncomp=1)

    @property
    def bc(self):
        return self.config.bc

    def freeze(self, T0):
        """Set the lagged state (aligned) and re-evaluate the device coefficients."""
        self.frozen_state = T0
        for dop in self._dev.values():
            dop.freeze(T0)
        return self

    def device_op(self, grid, ncomp: int = 1, ctx: device.Context | None = None) -> "DeviceOperator":
        ctx = ctx or device.default_context()
        key = (id(ctx), id(grid), ncomp)
        hit = self._dev.get(key)
        if hit is not None and hit.grid is grid:
            return hit
        dop = DeviceOperator(self, grid, ncomp, ctx)
        self._dev[key] = dop
        return dop

    def apply(self, u: Field) -> Field:
        dop = self.device_op(u.grid, u.n_components)
        du = device.DeviceField.from_values(dop.dgrid, u.values)
        F = device.DeviceField(dop.dgrid, u.n_components)
        dop.apply(du, F)
        return F.to_field()


class DeviceOperator:
    """A frozen linear operator resident on one rank (pc_op handle)."""

    def __init__(self, op: DiffusionOperator, grid, ncomp: int, ctx: device.Context):
        cfg = op.config
        if cfg.bc is None:
            raise ValueError("operator config needs a boundary condition (bc)")
        self.op = op
        self.grid = grid
        self.ncomp = ncomp
        self.ctx = ctx
        self.dgrid = device.device_grid(grid, cfg.bc, ctx)
        dg = self.dgrid
        L = _lib.lib()
        h = c_void_p()
        self._keep = []
        if op.kind == "scalar" and isinstance(cfg.rho, device.DeviceField):
            # device-resident density (C5-size inputs never visit the host)
            if not isinstance(cfg.nu, (int, float)):
                raise ValueError("a device-resident rho needs a constant nu")
            vm = bool(cfg.vector_metric) and ncomp == 3 and getattr(grid, "metric", "cartesian") == mesh.SPHERICAL
            _lib.check(L.pc_op_create_viscous(dg.handle, ncomp, int(vm), float(cfg.nu), cfg.rho.handle, byref(h)),
                       "pc_op_create_viscous")
            self._keep.append(cfg.rho)
        elif op.kind == "scalar":
            nu = _values(cfg.nu, grid, "nu")
            rho = None if cfg.rho is None else _values(cfg.rho, grid, "rho")
            if isinstance(rho, float) and rho == 1.0:
                rho = None
            viscous = isinstance(nu, float) and rho is not None and not isinstance(rho, float)
            if viscous:  # D = nu * rho formed per node on the device (no D array)
                Dc, Dd = nu, None
                if nu < 0:
                    raise ValueError("nu*rho must be >= 0")
            elif isinstance(nu, float) and (rho is None or isinstance(rho, float)):
                Dc = nu if rho is None else nu * rho
                Dd = None
                if rho is not None:  # constant rho != 1: F = (1/rho) div(nu rho grad u)
                    rho = np.full(tuple(grid.shape), rho)
            else:
                Dc = 1.0
                nu_a = nu if not isinstance(nu, float) else np.full(tuple(grid.shape), nu)
                if rho is None:
                    Darr = nu_a
                else:
                    rho_a = rho if not isinstance(rho, float) else np.full(tuple(grid.shape), rho)
                    Darr = nu_a * rho_a
                if np.any(Darr < 0):
                    raise ValueError("nu*rho must be >= 0")
                Dd = device.DeviceField.from_values(dg, Darr)
                self._keep.append(Dd)
            rd = None
            if rho is not None:
                rho_a = rho if not isinstance(rho, float) else np.full(tuple(grid.shape), rho)
                rd = _positive_field(dg, rho_a)
                self._keep.append(rd)
            vm = bool(cfg.vector_metric) and ncomp == 3 and getattr(grid, "metric", "cartesian") == mesh.SPHERICAL
            if cfg.vector_metric and ncomp != 3:
                raise ValueError("vector_metric needs a 3-component field")
            if viscous:
                _lib.check(L.pc_op_create_viscous(dg.handle, ncomp, int(vm), float(Dc), rd.handle, byref(h)),
                           "pc_op_create_viscous")
            else:
                _lib.check(L.pc_op_create_scalar(dg.handle, ncomp, int(vm), float(Dc),
                                                 Dd.handle if Dd is not None else None,
                                                 rd.handle if rd is not None else None, byref(h)),
                           "pc_op_create_scalar")
        else:
            if ncomp != 1:
                raise ValueError("aligned conduction acts on a scalar temperature")
            if isinstance(cfg.b_hat, device.DeviceField):
                bd = cfg.b_hat
                if bd.ncomp != 3:
                    raise ValueError("b_hat needs 3 components")
            else:
                b = np.asarray(getattr(cfg.b_hat, "values", cfg.b_hat), dtype=float)
                b = b.reshape(tuple(grid.shape) + (3,)) if b.size == 3 * grid.npoints else b
                if b.shape != tuple(grid.shape) + (3,):
                    raise ValueError("b_hat needs 3 components")
                bd = device.DeviceField.from_values(dg, b, 3)
            self._keep.append(bd)
            rd = None
            if isinstance(cfg.rho, device.DeviceField):
                rd = cfg.rho
                self._keep.append(rd)
            elif cfg.rho is not None and not (isinstance(cfg.rho, (int, float)) and float(cfg.rho) == 1.0):
                rho_a = _values(cfg.rho, grid, "rho")
                rho_a = rho_a if not isinstance(rho_a, float) else np.full(tuple(grid.shape), rho_a)
                rd = _positive_field(dg, rho_a)
                self._keep.append(rd)
            r = np.asarray(grid.coords[0], float)
            fc = cfg.fc_table(r)
            fcp = None
            if fc is not None:
                ext = np.zeros(dg.global_shape[0] + 2)
                ext[1:-1] = fc
                i0, n = dg.i0, dg.n0_local
                loc = np.zeros(n + 2)
                loc[:] = ext[i0:i0 + n + 2]
                if dg.ghost_lo and i0 == 0:
                    loc[0] = fc[-1]
                if dg.ghost_hi and i0 + n == dg.global_shape[0]:
                    loc[-1] = fc[0]
                fcp = np.ascontiguousarray(loc)
                self._keep.append(fcp)
            if cfg.f_m != "one":
                raise NotImplementedError("only the f_m = 'one' preset runs on the device")
            _lib.check(L.pc_op_create_aligned(dg.handle, bd.handle, rd.handle if rd is not None else None,
                                              float(cfg.prefactor), float(cfg.kappa0),
                                              _lib.dptr(fcp) if fcp is not None else None,
                                              float(cfg.T_floor), byref(h)), "pc_op_create_aligned")
        self.handle = h
        self.frozen = False
        if op.kind == "scalar":
            self.freeze(None)
        elif op.frozen_state is not None:
            self.freeze(op.frozen_state)

    def freeze(self, T0):
        """Aligned: conductivity from T0 (Field, array or DeviceField)."""
        L = _lib.lib()
        t = None
        if self.op.kind == "aligned":
            if T0 is None:
                raise ValueError("aligned operator needs T0")
            t = T0 if isinstance(T0, device.DeviceField) else device.DeviceField.from_values(
                self.dgrid, np.asarray(getattr(T0, "values", T0), float))
        _lib.check(L.pc_op_freeze(self.handle, t.handle if t is not None else None), "freeze")
        self.frozen = True
        return self

    @property
    def dt_euler(self) -> float:
        v = c_double()
        _lib.check(_lib.lib().pc_op_euler_dt(self.handle, byref(v)), "euler_dt")
        return v.value

    def apply(self, u: device.DeviceField, F: device.DeviceField):
        _lib.check(_lib.lib().pc_op_apply(self.handle, u.handle, F.handle), "apply")
        return F

    def diagonal(self) -> device.DeviceField:
        d = device.DeviceField(self.dgrid, 1)
        _lib.check(_lib.lib().pc_op_diagonal(self.handle, d.handle), "diagonal")
        return d

    def __del__(self):
        try:
            if _lib.alive() and self.handle is not None and self.ctx.handle is not None:
                _lib.lib().pc_op_destroy(self.handle)
        except Exception:
            pass


def apply_scalar_diffusion(u: Field, cfg: ScalarDiffusionConfig) -> Field:
    """SPEC.md:107-115."""
    return DiffusionOperator.scalar(cfg, u.n_components).apply(u)


def apply_aligned_conduction(T: Field, cfg: AlignedConductionConfig, T0: Field) -> Field:
    """SPEC.md:116-124 (diffusivity from the lagged T0)."""
    if np.any(~(np.asarray(getattr(T0, "values", T0)) > 0)):
        from .errors import DomainError
        raise DomainError("non-positive T0 (SPEC.md:120)")
    return DiffusionOperator.aligned(cfg, T0).apply(T)


def estimate_euler_dt(op: DiffusionOperator, probe: Field) -> float:
    """Gershgorin Delta t_Euler = 2 / max_i sum_j |J_ij|;
    +inf for a zero operator.  An unfrozen aligned operator is frozen at the
    probe."""
    if op.kind == "aligned" and op.frozen_state is None:
        op.freeze(probe)
    return op.device_op(probe.grid, probe.n_components).dt_euler
