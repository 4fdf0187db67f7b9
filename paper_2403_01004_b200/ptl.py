"""Practical time-step limit, the cycling controller and the split driver --
the SPEC ``ptl`` API on the device.

  compute_ptl(u, F, grid, cfg) -> float | UNLIMITED     PAPER.md Eq. 3-5
  cycle_operator(op, scheme, u, outer_dt, cfg)
      -> (u, CycleReport)     (u may be a mesh.Field or a resident DeviceField)
  split_advance(ops, state, outer_dt, cfgs) -> state

``cycle_operator`` is one C-ABI call (pc_cycle): per cycle one fused
F+argmax pass, the Eq. 5 pair kernel, a single 64-byte device->host read,
then s fused stage kernels (RKL2/RKG2) or a device-driven PCG solve.
"""
from __future__ import annotations

import csv
import math
from ctypes import byref, c_double, c_int, c_int64
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib, device, mesh
from .errors import CycleCapError, NotConvergedError
from .mesh import Field


class _Unlimited:
    def __repr__(self):
        return "UNLIMITED"

    def __bool__(self):
        return False


UNLIMITED = _Unlimited()


@dataclass
class PtlConfig:
    """SPEC.md:335-337."""

    eps_rel: float = 1e-12
    dt_floor_mode: str = "clamp-to-euler"  # or "clamp-to-fraction"
    floor_fraction: float = 1.0
    max_cycles: int = 10**6
    check_all_points: bool = False
    enabled: bool = True  # False: one cycle of the whole outer step (no PTL)
    # "dynamic": the PTL is re-evaluated every cycle;
    # "static": first-PTL cycling, the first cycle's PTL is reused by every
    # cycle (the comparison mode of SPEC.md:362 and acceptance 6)
    reevaluate: str = "dynamic"
    # lagged T0 of aligned operators: "outer" = refreshed once per outer step
    # (SPEC default); "cycle" = re-frozen at T0 := u at the start
    # of every cycle ("per-cycle refresh available via config")
    refresh_T0: str = "outer"

    def __post_init__(self):
        if not self.eps_rel > 0:
            raise ValueError("eps_rel must be > 0")
        if self.max_cycles < 1:
            raise ValueError("max_cycles must be >= 1")
        if self.dt_floor_mode not in ("clamp-to-euler", "clamp-to-fraction"):
            raise ValueError(f"unknown dt_floor_mode {self.dt_floor_mode!r}")
        if self.reevaluate not in ("dynamic", "static"):
            raise ValueError(f"unknown reevaluate mode {self.reevaluate!r}")
        if self.refresh_T0 not in ("outer", "cycle"):
            raise ValueError(f"unknown refresh_T0 cadence {self.refresh_T0!r}")

    @property
    def ptl_mode(self) -> int:
        """pc_cycle's use_ptl: 0 off, 1 dynamic, 2 static."""
        return 0 if not self.enabled else (2 if self.reevaluate == "static" else 1)


@dataclass
class CycleEntry:
    cycle: int
    dt: float
    ptl_raw: object  # float or UNLIMITED
    limited: bool
    iters: int
    relres: float = 0.0


@dataclass
class CycleReport:
    """Per-cycle records of one operator over one outer step."""

    entries: list = dc_field(default_factory=list)
    outer_step: int = 0
    dt_euler: float = float("nan")

    @property
    def n_cycles(self) -> int:
        return len(self.entries)

    @property
    def total_iters(self) -> int:
        return int(sum(e.iters for e in self.entries))

    @property
    def total_dt(self) -> float:
        return float(sum(e.dt for e in self.entries))

    def rows(self):
        for e in self.entries:
            yield (self.outer_step, e.cycle, repr(float(e.dt)),
                   "unlimited" if e.ptl_raw is UNLIMITED else repr(float(e.ptl_raw)), int(e.limited), e.iters)

    def write_csv(self, path: str, append: bool = False):
        """CSV ``outer_step,cycle,dt,ptl_raw,limited,iters``."""
        with open(path, "a" if append else "w", newline="") as fh:
            w = csv.writer(fh)
            if not append:
                w.writerow(["outer_step", "cycle", "dt", "ptl_raw", "limited", "iters"])
            for row in self.rows():
                w.writerow(row)


def _default_bc(grid):
    if getattr(grid, "metric", mesh.CARTESIAN) == mesh.SPHERICAL:
        return mesh.BoundaryCondition.spherical(mesh.FaceBC(mesh.NEUMANN), mesh.FaceBC(mesh.NEUMANN))
    return mesh.BoundaryCondition.neumann(len(grid.coords))


def compute_ptl(u: Field, F: Field, grid=None, cfg: PtlConfig | None = None, bc=None):
    """Eq. 5 at k = argmax |F| (ties -> lowest linear index); ``bc`` only
    decides which faces are periodic (defaults: spherical phi periodic,
    Cartesian non-periodic).  Returns the limit or ``UNLIMITED``."""
    cfg = cfg or PtlConfig()
    grid = grid or u.grid
    bc = bc or _default_bc(grid)
    dg = device.device_grid(grid, bc)
    du = device.DeviceField.from_values(dg, u.values)
    dF = device.DeviceField.from_values(dg, F.values)
    v, lim, k = c_double(), c_int(), c_int64()
    _lib.check(_lib.lib().pc_ptl(dg.handle, du.handle, dF.handle, float(cfg.eps_rel), int(cfg.check_all_points),
                                 byref(v), byref(lim), byref(k)), "compute_ptl")
    return v.value if lim.value else UNLIMITED


def _report(recs, n, dt_euler, outer_step=0):
    rep = CycleReport(outer_step=outer_step, dt_euler=dt_euler)
    for q in range(n):
        r = recs[q]
        rep.entries.append(CycleEntry(int(r.cycle), float(r.dt), float(r.ptl_raw) if r.limited else UNLIMITED,
                                      bool(r.limited), int(r.iters), float(r.relres)))
    return rep


_RECS = {}


def _record_buffer(cap: int):
    """A reused ctypes array of ``cap`` cycle records (the report copies the
    values out, so one buffer per size serves every call)."""
    buf = _RECS.get(cap)
    if buf is None:
        buf = _RECS[cap] = (_lib.CycleRecord * cap)()
    return buf


def cycle_operator(op, scheme, u, outer_dt: float, cfg: PtlConfig | None = None, *, dt_euler: float | None = None,
                   outer_step: int = 0, ctx: device.Context | None = None, record_cap: int = 1 << 16):
    """Advance ``u`` over ``outer_dt`` with PTL cycling.

    ``u``: mesh.Field (uploaded, returned as a new Field) or DeviceField
    (advanced in place on the device and returned)."""
    from .schemes import SchemeConfig

    cfg = cfg or PtlConfig()
    if isinstance(scheme, str):
        scheme = SchemeConfig(scheme)
    if not outer_dt > 0:
        raise ValueError("outer_dt must be > 0")
    if isinstance(u, device.DeviceField):
        dop = op.device_op(u.dgrid.grid, u.ncomp, ctx or u.dgrid.ctx)
        du = u
        host = False
    else:
        dop = op.device_op(u.grid, u.n_components, ctx)
        if dop.ctx.nranks > 1:
            device.require_gather_group()  # the result is gathered back to a global Field
        du = device.DeviceField.from_values(dop.dgrid, u.values)
        host = True
    recs = _record_buffer(record_cap)
    n = c_int64()
    floor_mode = _lib.FLOOR_EULER if cfg.dt_floor_mode == "clamp-to-euler" else _lib.FLOOR_FRACTION
    dtE = float(dt_euler) if dt_euler is not None else -1.0
    if scheme.kind == "backward_euler":
        _lib.check(_lib.lib().pc_op_set_preconditioner(dop.handle, scheme.pc_code), "preconditioner")
    if cfg.refresh_T0 == "cycle" and op.kind != "aligned":
        raise ValueError("refresh_T0='cycle' applies to aligned (lagged-T0) operators only")
    if op.kind == "aligned":
        _lib.check(_lib.lib().pc_op_set_refresh(dop.handle, int(cfg.refresh_T0 == "cycle")), "refresh_T0")
    rc = _lib.lib().pc_cycle(dop.handle, du.handle, float(outer_dt), scheme.code, int(scheme.make_odd),
                             float(scheme.tol), int(scheme.max_iter), float(cfg.eps_rel), int(cfg.check_all_points),
                             cfg.ptl_mode, floor_mode, float(cfg.floor_fraction), int(cfg.max_cycles), dtE,
                             recs, record_cap, byref(n))
    rep = _report(recs, min(n.value, record_cap), dop.dt_euler if dt_euler is None else float(dt_euler), outer_step)
    _lib.check(rc, "cycle_operator", report=rep)
    return (du.to_field() if host else du), rep


def _check_host_state(state, ops):
    """Host Fields on a multi-rank context are gathered back to global
    Fields at the end (device.DeviceField.to_field): that needs an
    initialised torch.distributed process group -- fail before any work."""
    if any(not isinstance(v, device.DeviceField) for n, v in state.items() if any(n == m for m, _ in ops)):
        ctx = device.default_context()
        if ctx.nranks > 1:
            device.require_gather_group()


class FieldSet(dict):
    """The state returned by ``split_advance``: a dict name -> Field /
    DeviceField (the SPEC's ``Field set``) that also carries the
    per-operator ``CycleReport`` list as ``.reports``."""

    reports: list

    def __init__(self, *a, reports=None, **k):
        super().__init__(*a, **k)
        self.reports = list(reports or [])


def split_advance(ops, state: dict, outer_dt: float, cfgs, *, outer_step: int = 0, refresh=None,
                  out_reports: list | None = None) -> FieldSet:
    """First-order (Lie) splitting over ``outer_dt`` in list order.

    ops:   list of (field_name, DiffusionOperator)
    state: dict name -> Field or DeviceField (advanced in place for DeviceFields)
    cfgs:  list of (SchemeConfig, PtlConfig) per operator
    refresh: optional {op_index: state_name}; aligned operators are re-frozen
             at the named state once per outer step before cycling begins
             (lagged T0; PtlConfig.refresh_T0 = "cycle" re-freezes
             every cycle instead).
    out_reports: optional list that receives the CycleReport of every operator.
    Returns the advanced state (SPEC.md:363 ``-> Field set``), a FieldSet whose
    ``.reports`` holds the same CycleReports.
    """
    refresh = refresh or {}
    _check_host_state(state, ops)
    # host Fields go to the device once per outer step and come back once at
    # the end.  The first operator's state and coefficients go first; the
    # other operators' states then move on the copy stream while the first
    # operator freezes and cycles (PCIe is not shared with its inputs); a
    # field no later operator touches starts its download as soon as its last
    # operator is done.
    host_names = {}
    dev = dict(state)
    for q, (name, op) in enumerate(ops):
        if name in dev and not isinstance(dev[name], device.DeviceField):
            f = dev[name]
            dg = device.device_grid(f.grid, op.config.bc)
            dev[name] = device.DeviceField.from_values(dg, f.values, async_=q > 0)
            host_names[name] = True
        if q == 0 and isinstance(dev.get(name), device.DeviceField):
            u = dev[name]  # the first operator's coefficients upload now, ahead of the later states
            op.device_op(u.dgrid.grid, u.ncomp, u.dgrid.ctx)
    for q, (name, op) in enumerate(ops):
        if op.kind == "aligned":
            src = dev.get(refresh.get(q, name), state.get(refresh.get(q, name)))
            op.freeze(src)
    reports = []
    pending = {}
    for q, ((name, op), (scheme, pcfg)) in enumerate(zip(ops, cfgs)):
        dev[name], rep = cycle_operator(op, scheme, dev[name], outer_dt, pcfg, outer_step=outer_step)
        reports.append(rep)
        last = all(n != name for n, _ in ops[q + 1:]) and all(refresh.get(p) != name for p in range(q + 1, len(ops)))
        if host_names.get(name) and last and dev[name].dgrid.ctx.nranks == 1:
            pending[name] = dev[name].download_async()
    out = dict(state)
    for name in dev:
        if not host_names.get(name):
            out[name] = dev[name]
        elif name in pending:
            dev[name].wait()
            grid = dev[name].dgrid.grid
            out[name] = mesh.Field(grid, pending[name].reshape(tuple(grid.shape) + (dev[name].ncomp,)))
        else:
            out[name] = dev[name].to_field()
    if out_reports is not None:
        out_reports.extend(reports)
    return FieldSet(out, reports=reports)
