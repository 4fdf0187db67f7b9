"""The reference harness over the B200 path: ``run``
(cmd_run), and ``ampfactor`` / ``speedup`` / ``convergence`` over
``analysis`` (Fig. 1).

    python -m paper_2403_01004_b200.cli run experiment.cfg

The config is a sectioned key/value document:

    [grid]        metric = cartesian | spherical
                  sizes  = n0, n1, n2                  (1-3 entries for cartesian)
                  extents = lo, hi [; lo, hi ...]      cartesian: one pair per axis;
                                                       spherical: the r range
                  r_spacing = uniform | geometric:<ratio> | stretched:<total ratio>
                  bc = dirichlet:<v> | neumann | periodic   (r / every non-spherical face)
    [operator.<name>]  (zero or more, applied in file order = Lie splitting order)
                  kind = scalar | aligned ; field = <state name>
                  scalar:  nu = <float>, rho = <float> | exp_r:<a>, vector = true|false, ncomp = 1|3
                  aligned: b = x | dipole | uniform:<bx>,<by>,<bz>, kappa0, m_p, k_B, gamma,
                           T_floor, rho = <float> | exp_r:<a>
    [initial]     <field> = step | gaussian | sinusoid | random | transition, with
                  <field>.<param> = value  (amp, width, centre, lo, hi, k, sigma, offset)
    [scheme]      kind = rkl2 | rkg2 | backward_euler | euler ; tol ; max_iter ; make_odd
    [ptl]         enabled ; eps_rel ; max_cycles ; check_all_points ; floor = euler | fraction:<f> ;
                  reevaluate = dynamic | static ; refresh_T0 = outer | cycle
    [run]         outer_dt = <float> | dt_over_dt_euler = <float> ; n_outer_steps ; seed ;
                  out_prefix (field CSVs <prefix>_<field>.csv + <prefix>_coords.csv) ;
                  out_report (CycleReport CSV, all operators and outer steps)

Outputs are the reference CSV formats (mesh.write_field_csv: repr() round
trip; CycleReport: outer_step,cycle,dt,ptl_raw,limited,iters).  Exit code 0
iff the run finished and every output was written; an invalid config exits 2
with a line-anchored message.  Results are bitwise deterministic (the device
path is), so two runs of one config write byte-identical files.
"""
from __future__ import annotations

import configparser
import re
import sys

import numpy as np

from . import configs, mesh

KNOWN = {
    "grid": {"metric", "sizes", "extents", "r_spacing", "bc"},
    "initial": None,
    "scheme": {"kind", "tol", "max_iter", "make_odd"},
    "ptl": {"enabled", "eps_rel", "max_cycles", "check_all_points", "floor", "reevaluate", "refresh_T0"},
    "run": {"outer_dt", "dt_over_dt_euler", "n_outer_steps", "seed", "out_prefix", "out_report"},
}
OP_KEYS = {"kind", "field", "nu", "rho", "vector", "ncomp", "b", "kappa0", "m_p", "k_B", "gamma", "T_floor"}


class ConfigError(ValueError):
    pass


class _Cfg:
    def __init__(self, path):
        self.path = path
        text = open(path).read()
        self.lines = {}
        sec = None
        for no, raw in enumerate(text.splitlines(), 1):
            s = raw.strip()
            m = re.match(r"^\[(.+)\]$", s)
            if m:
                sec = m.group(1).strip()
                self.lines[(sec, None)] = no
            elif sec and s and not s.startswith(("#", ";")) and ("=" in s or ":" in s):
                key = re.split(r"[=:]", s, maxsplit=1)[0].strip()
                self.lines[(sec, key.lower())] = no
        self.cp = configparser.ConfigParser(inline_comment_prefixes=("#",))
        self.cp.optionxform = str
        try:
            self.cp.read_string(text, source=path)
        except configparser.Error as e:
            raise ConfigError(f"{path}: {e}") from None

    def err(self, sec, key, msg):
        line = self.lines.get((sec, key.lower() if key else None), self.lines.get((sec, None), 0))
        return ConfigError(f"{self.path}:{line}: [{sec}]{' ' + key if key else ''}: {msg}")

    def get(self, sec, key, conv=str, default=None, required=False):
        if not self.cp.has_option(sec, key):
            if required:
                raise self.err(sec, None, f"missing key {key!r}")
            return default
        v = self.cp.get(sec, key)
        try:
            return conv(v)
        except Exception as e:  # noqa: BLE001
            raise self.err(sec, key, f"bad value {v!r} ({e})") from None


def _floats(s):
    return [float(x) for x in s.replace(";", ",").split(",") if x.strip()]


def _bool(s):
    t = s.strip().lower()
    if t in ("1", "true", "yes", "on"):
        return True
    if t in ("0", "false", "no", "off"):
        return False
    raise ValueError("expected a boolean")


def _face(spec):
    kind, _, val = spec.strip().partition(":")
    if kind not in (mesh.DIRICHLET, mesh.NEUMANN, mesh.PERIODIC):
        raise ValueError(f"unknown boundary kind {kind!r}")
    return mesh.FaceBC(kind, float(val) if val else 0.0)


def build_grid(c: _Cfg):
    metric = c.get("grid", "metric", default="cartesian")
    sizes = c.get("grid", "sizes", lambda s: [int(x) for x in _floats(s)], required=True)
    face = c.get("grid", "bc", _face, default=mesh.FaceBC(mesh.DIRICHLET, 0.0))
    if metric == "spherical":
        if len(sizes) != 3:
            raise c.err("grid", "sizes", "a spherical grid needs 3 sizes")
        lo, hi = c.get("grid", "extents", _floats, default=[1.0, 2.5])[:2]
        sp = c.get("grid", "r_spacing", default="uniform")
        if sp == "uniform":
            r = configs.r_uniform(sizes[0], lo, hi)
        elif sp.startswith("geometric:"):
            r = configs.r_geometric_ratio(sizes[0], lo, hi, float(sp.split(":")[1]))
        elif sp.startswith("stretched:"):
            r = configs.r_stretched_c3(sizes[0], lo, hi, float(sp.split(":")[1]))
        else:
            raise c.err("grid", "r_spacing", f"unknown spacing {sp!r}")
        try:
            grid = mesh.build_spherical_grid(r, sizes[1], sizes[2])
        except ValueError as e:
            raise c.err("grid", "sizes", str(e)) from None
        return grid, mesh.BoundaryCondition.spherical(face, face)
    if metric != "cartesian":
        raise c.err("grid", "metric", f"unknown metric {metric!r}")
    ext = c.get("grid", "extents", lambda s: [_floats(p) for p in s.split(";")], default=None)
    ext = ext or [[0.0, 1.0]] * len(sizes)
    if len(ext) != len(sizes) or any(len(e) != 2 for e in ext):
        raise c.err("grid", "extents", "one 'lo, hi' pair per axis")
    try:
        grid = mesh.build_grid(sizes, extents=[tuple(e) for e in ext])
    except ValueError as e:
        raise c.err("grid", "sizes", str(e)) from None
    faces = tuple((face, face) for _ in sizes)
    return grid, mesh.BoundaryCondition(faces)


def _radial(c, sec, key, grid):
    v = c.get(sec, key, default=None)
    if v is None:
        return None
    if v.startswith("exp_r:"):
        a = float(v.split(":")[1])
        r = np.asarray(grid.coords[0])
        return np.exp(-a * (r - r[0]))[:, None, None] * np.ones(grid.shape) if grid.dims == 3 else None
    try:
        return float(v)
    except ValueError:
        raise c.err(sec, key, f"bad density {v!r}") from None


def build_ops(c: _Cfg, grid, bc):
    from . import operators
    ops = []
    for sec in c.cp.sections():
        if not sec.startswith("operator."):
            continue
        for k in c.cp.options(sec):
            if k not in OP_KEYS:
                raise c.err(sec, k, "unknown key")
        kind = c.get(sec, "kind", required=True)
        field = c.get(sec, "field", required=True)
        rho = _radial(c, sec, "rho", grid)
        if kind == "scalar":
            nc = c.get(sec, "ncomp", int, default=1)
            cfg = operators.ScalarDiffusionConfig(nu=c.get(sec, "nu", float, default=1.0), rho=rho, bc=bc,
                                                  vector_metric=c.get(sec, "vector", _bool, default=False))
            ops.append((field, operators.DiffusionOperator.scalar(cfg, nc), nc))
        elif kind == "aligned":
            spec = c.get(sec, "b", default="x")
            shp = tuple(grid.shape) + (3,)
            if spec == "x":
                b = np.zeros(shp)
                b[..., 0] = 1.0
            elif spec == "dipole":
                if grid.metric != mesh.SPHERICAL:
                    raise c.err(sec, "b", "dipole needs a spherical grid")
                b = configs.dipole_bhat(grid, c.get("run", "seed", int, default=1), eps=0.0)
            elif spec.startswith("uniform:"):
                v = np.asarray(_floats(spec.split(":", 1)[1]), float)
                if v.size != 3 or not np.linalg.norm(v) > 0:
                    raise c.err(sec, "b", "uniform:<bx>,<by>,<bz> with a non-zero vector")
                b = np.broadcast_to(v / np.linalg.norm(v), shp).copy()
            else:
                raise c.err(sec, "b", f"unknown field direction {spec!r}")
            cfg = operators.AlignedConductionConfig(
                b_hat=b, kappa0=c.get(sec, "kappa0", float, default=1.0), gamma=c.get(sec, "gamma", float, default=5.0 / 3.0),
                m_p=c.get(sec, "m_p", float, default=1.0), k_B=c.get(sec, "k_B", float, default=1.0), rho=rho, bc=bc,
                T_floor=c.get(sec, "T_floor", float, default=1e-10))
            ops.append((field, operators.DiffusionOperator.aligned(cfg), 1))
        else:
            raise c.err(sec, "kind", f"unknown operator kind {kind!r}")
    return ops


def initial_state(c: _Cfg, grid, fields_nc):
    seed = c.get("run", "seed", int, default=None)
    X = [np.asarray(x) for x in np.meshgrid(*grid.coords, indexing="ij")]
    state = {}
    for name, nc in fields_nc.items():
        preset = c.get("initial", name, default=None)
        if preset is None:
            raise c.err("initial", None, f"no initial condition for field {name!r}")
        p = lambda k, d=None: c.get("initial", f"{name}.{k}", _floats, default=d)  # noqa: E731
        off = (p("offset", [0.0]) or [0.0])[0]
        if preset == "step":
            lo, hi = p("lo", [0.25]), p("hi", [0.5])
            amp = p("amp", [1.0])[0]
            m = (X[0] >= lo[0]) & (X[0] <= hi[0])
            v = np.where(m, amp, 0.0) + off
        elif preset == "gaussian":
            amp, width = p("amp", [1.0])[0], p("width", [0.2])[0]
            cen = p("centre", [float(np.mean(x)) for x in grid.coords])
            if grid.metric == mesh.SPHERICAL:
                v = amp * configs.gaussian_bump(grid, tuple(cen), width) + off
            else:
                d2 = sum((x - c0) ** 2 for x, c0 in zip(X, cen))
                v = amp * np.exp(-d2 / (width * width)) + off
        elif preset == "sinusoid":
            amp = p("amp", [1.0])[0]
            ks = p("k", [1.0] * grid.dims)
            v = amp * np.prod([np.sin(k * x) for k, x in zip(ks, X)], axis=0) + off
        elif preset == "random":
            if seed is None:
                raise c.err("initial", name, "a [run] seed is mandatory when randomness is used")
            v = off + p("sigma", [1.0])[0] * configs.block_noise(seed, 7, grid.shape)
        elif preset == "transition":
            if grid.metric != mesh.SPHERICAL:
                raise c.err("initial", name, "'transition' needs a spherical grid")
            v = configs.transition_profile(grid.coords[0])[:, None, None] * np.ones(grid.shape)
        else:
            raise c.err("initial", name, f"unknown preset {preset!r}")
        vals = np.repeat(np.asarray(v, float)[..., None], nc, axis=-1)
        state[name] = mesh.Field(grid, vals)
    return state


def cmd_run(path: str) -> int:
    from . import ptl, schemes
    c = _Cfg(path)
    for sec in c.cp.sections():
        allowed = KNOWN.get(sec, "op" if sec.startswith("operator.") else "bad")
        if allowed == "bad":
            raise c.err(sec, None, "unknown section")
        if isinstance(allowed, set):
            for k in c.cp.options(sec):
                if k not in allowed:
                    raise c.err(sec, k, "unknown key")
    grid, bc = build_grid(c)
    ops = build_ops(c, grid, bc)
    fields_nc = {}
    for f, _, nc in ops:
        fields_nc[f] = max(fields_nc.get(f, 1), nc)
    for k in (c.cp.options("initial") if c.cp.has_section("initial") else []):
        if "." not in k:
            fields_nc.setdefault(k, 1)
    state = initial_state(c, grid, fields_nc)
    kind = c.get("scheme", "kind", default="rkl2")
    try:
        sc = schemes.SchemeConfig(kind, tol=c.get("scheme", "tol", float, default=1e-10),
                                  max_iter=c.get("scheme", "max_iter", int, default=10000),
                                  make_odd=c.get("scheme", "make_odd", _bool, default=False))
    except (ValueError, NotImplementedError) as e:
        raise c.err("scheme", "kind", str(e)) from None
    floor = c.get("ptl", "floor", default="euler")
    fmode, frac = ("clamp-to-euler", 1.0) if floor == "euler" else ("clamp-to-fraction", float(floor.split(":")[1]))
    pcfg = ptl.PtlConfig(eps_rel=c.get("ptl", "eps_rel", float, default=1e-12), dt_floor_mode=fmode,
                         floor_fraction=frac, max_cycles=c.get("ptl", "max_cycles", int, default=10**6),
                         check_all_points=c.get("ptl", "check_all_points", _bool, default=False),
                         enabled=c.get("ptl", "enabled", _bool, default=True),
                         reevaluate=c.get("ptl", "reevaluate", default="dynamic"),
                         refresh_T0=c.get("ptl", "refresh_T0", default="outer"))
    nsteps = c.get("run", "n_outer_steps", int, default=1)
    outer_dt = c.get("run", "outer_dt", float, default=None)
    ratio = c.get("run", "dt_over_dt_euler", float, default=None)
    if (outer_dt is None) == (ratio is None) and ops:
        raise c.err("run", None, "give exactly one of outer_dt, dt_over_dt_euler")
    if ratio is not None and ops:
        from . import operators
        dts = []
        for f, op, nc in ops:
            dts.append(operators.estimate_euler_dt(op, state[f]))
        outer_dt = ratio * min(dts)
    prefix = c.get("run", "out_prefix", default="out")
    rpath = c.get("run", "out_report", default=f"{prefix}_report.csv")
    first = True
    for step in range(nsteps):
        if ops:
            import dataclasses  # (the per-cycle T0 refresh applies to the aligned operators only)
            cfgs = [(sc, pcfg if op.kind == "aligned" else dataclasses.replace(pcfg, refresh_T0="outer"))
                    for _, op, _ in ops]
            state = ptl.split_advance([(f, op) for f, op, _ in ops], state, outer_dt, cfgs, outer_step=step,
                                            refresh={q: f for q, (f, op, _) in enumerate(ops) if op.kind == "aligned"})
            reps = state.reports
            for rep in reps:
                rep.write_csv(rpath, append=not first)
                first = False
    if first:  # no operators: header-only report
        ptl.CycleReport().write_csv(rpath)
    mesh.write_coords_csv(grid, f"{prefix}_coords.csv")
    for f, fld in state.items():
        mesh.write_field_csv(fld if isinstance(fld, mesh.Field) else fld.to_field(), f"{prefix}_{f}.csv")
    return 0


USAGE = """usage:
  python -m paper_2403_01004_b200.cli run <config>
  python -m paper_2403_01004_b200.cli ampfactor --schemes be,rkl2,rkg2,exact --r 500 --out amp.csv
  python -m paper_2403_01004_b200.cli speedup --rmin 1 --rmax 1e4 --out speedup.csv
  python -m paper_2403_01004_b200.cli convergence --scheme rkg2 --problem sine
"""


def _flags(args, names):
    out, i = {}, 0
    while i < len(args):
        a = args[i]
        if not a.startswith("--") or a[2:] not in names or i + 1 >= len(args):
            raise ValueError(f"unexpected argument {a!r}")
        out[a[2:]] = args[i + 1]
        i += 2
    return out


def main(argv=None) -> int:
    from . import analysis
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv or argv[0] in ("-h", "--help"):
        sys.stderr.write(USAGE)
        return 0 if argv else 2
    cmd, rest = argv[0], argv[1:]
    try:
        if cmd == "run":
            if len(rest) != 1:
                raise ValueError("run takes one config path")
            return cmd_run(rest[0])
        if cmd == "ampfactor":
            f = _flags(rest, {"schemes", "r", "out"})
            kinds = [k for k in f.get("schemes", "").split(",") if k]
            if not kinds or any(k not in analysis.SCHEMES for k in kinds):
                raise ValueError(f"schemes must be a non-empty list of {','.join(analysis.SCHEMES)}")
            analysis.write_ampfactor_csv(f.get("out", "ampfactor.csv"), kinds, float(f.get("r", "500")))
            return 0
        if cmd == "speedup":
            f = _flags(rest, {"rmin", "rmax", "out"})
            analysis.write_speedup_csv(f.get("out", "speedup.csv"), float(f["rmin"]), float(f["rmax"]))
            return 0
        if cmd == "convergence":
            f = _flags(rest, {"scheme", "problem"})
            if f.get("problem", "sine") != "sine":
                raise ValueError(f"unknown problem preset {f.get('problem')!r} (available: sine)")
            kind = f.get("scheme", "rkg2")
            if kind not in ("be", "rkl2", "rkg2", "euler"):
                raise ValueError(f"unknown scheme {kind!r}")
            order, dts, errs = analysis.convergence_study(kind)
            print(f"{kind}: fitted order {order:.3f}")
            return 0
        raise ValueError(f"unknown command {cmd!r}")
    except ConfigError as e:
        sys.stderr.write(f"config error: {e}\n")
        return 2
    except (ValueError, KeyError) as e:
        sys.stderr.write(f"usage error: {e}\n{USAGE}")
        return 2
    except OSError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
