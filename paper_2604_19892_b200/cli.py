"""Scene configs, the frame driver and the penetration checker: the
reference's command-line surface (`pkg/src/ipcsim/cli.py`) on the device
solver.

* ``load_config(path) -> (Scene, SolverConfig, RunParams)`` -- the same INI
  schema and errors as `cli.py:145-228`: ``[scene]`` (h, d_hat, kappa,
  frames, gravity, output_dir, seed), ``[solver]`` (SolverConfig fields),
  ``[mesh:<name>]`` per object (kind box | tet | file (.node/.ele), cells,
  size, scale, translate, material arap | snh | neo-hookean, youngs,
  poisson, density, pinned all | none | x<v ...).
* ``simulate`` -- frames through ``solver.step`` writing ``frame_%05d.obj``,
  ``iters.csv`` and ``frames.csv`` with the reference's columns
  (`cli.py:235-294`).
* ``compare`` -- the update-strategy variants the device solver implements
  (mas+woodbury, mas+freeze, mas+fullrebuild; `cli.py:300-353`).
* ``check`` -- the penetration checker (`cli.py:360-422`) made scalable:
  minimum PT/EE distance through the solver's own broad phase on a
  surface-only context, triangle-triangle intersections by a uniform grid on
  the device (csrc/check.cuh).  Same exit codes.
* ``write_scene(path, objs, ...)`` -- emit a generated scene (C4 / C5) as
  INI + TetGen files the reference itself can load.
"""

from __future__ import annotations

import argparse
import configparser
import dataclasses
import os
import re
import sys
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import energy, geometry, scenes, solver
from .errors import ConfigError, PenetrationError, SimError

EXIT_OK, EXIT_CONFIG, EXIT_SOLVER, EXIT_CHECK = 0, 2, 3, 4
ITER_COLUMNS = "frame,iter,grad_norm,z_norm,r_k,restart,mu,nu,min_alpha,t_grad_ms,t_dir_ms,t_ccd_ms"
FRAME_COLUMNS = "frame,iterations,converged,min_alpha,wall_ms"
MATERIALS = {"arap": "arap", "snh": "snh", "neo-hookean": "snh"}
_PIN = re.compile(r"^([xyz])\s*([<>])\s*([-+0-9.eE]+)$")
_SOLVER_FIELDS = {"eps": float, "delta": float, "eps_rot": float, "alpha_l": float, "iter_max": int, "K": int,
                  "block_size": int, "levels": int, "coarse_block": int,
                  "ccd_per_subdomain": lambda s: s.strip().lower() in ("1", "true", "yes"),
                  "preconditioner": str, "direction_rule": str, "update_strategy": str}


@dataclass
class RunParams:
    gravity: np.ndarray
    h: float
    frames: int
    output_dir: Path
    seed: int


def _vec(text, n, where):
    parts = str(text).split()
    if len(parts) != n:
        raise ConfigError(f"{where}: expected {n} numbers, got {text!r}")
    try:
        return np.array(parts, dtype=float)
    except ValueError as e:
        raise ConfigError(f"{where}: {e}") from e


def _pinned(expr, rest, where):
    expr = expr.strip()
    if expr in ("none", "all"):
        return np.full(len(rest), expr == "all")
    m = _PIN.match(expr)
    if not m:
        raise ConfigError(f"{where}: cannot parse pinned selector {expr!r}")
    col = rest[:, "xyz".index(m.group(1))]
    return col < float(m.group(3)) if m.group(2) == "<" else col > float(m.group(3))


def _object(sec, name, root):
    where = f"[{name}]"
    kind = sec.get("kind", "box")
    if kind == "box":
        cells = [int(c) for c in sec.get("cells", "1 1 1").split()]
        mesh = geometry.make_box_mesh(*cells, tuple(_vec(sec.get("size", "1 1 1"), 3, where)))
    elif kind == "tet":
        mesh = geometry.make_single_tet(float(sec.get("scale", "1")))
    elif kind == "file":
        base = root / sec.get("path", "")
        if not Path(str(base) + ".node").exists():
            raise ConfigError(f"{where}: mesh file {base}.node not found")
        mesh = geometry.load_node_ele(base)
    else:
        raise ConfigError(f"{where}: unknown mesh kind {kind!r}")
    rest = mesh.rest_positions.copy()
    if "scale" in sec and kind != "tet":
        rest *= float(sec["scale"])
    if "translate" in sec:
        rest += _vec(sec["translate"], 3, where)
    material = sec.get("material", "arap").lower()
    if material not in MATERIALS:
        raise ConfigError(f"{where}: unknown material {material!r}")
    young, nu, rho = sec.getfloat("youngs", 1e4), sec.getfloat("poisson", 0.3), sec.getfloat("density", 1000.0)
    if young <= 0 or rho <= 0:
        raise ConfigError(f"{where}: {'youngs' if young <= 0 else 'density'} must be positive")
    if not 0 <= nu < 0.5:
        raise ConfigError(f"{where}: poisson must lie in [0, 0.5)")
    return {"mesh": geometry.TetMesh(rest_positions=rest, tets=mesh.tets), "material": MATERIALS[material],
            "young": young, "poisson": nu, "density": rho, "pin_mask": _pinned(sec.get("pinned", "none"), rest,
                                                                                  where)}


def load_config(path):
    """INI scene -> (Scene, SolverConfig, RunParams), `cli.py:145-228`."""
    path = Path(path)
    if not path.is_file():
        raise ConfigError(f"config file {path} not found")
    cp = configparser.ConfigParser(inline_comment_prefixes=("#", ";"))
    try:
        cp.read(path)
    except configparser.Error as e:
        raise ConfigError(str(e)) from e
    if "scene" not in cp:
        raise ConfigError("missing [scene] section")
    sc = cp["scene"]
    h, d_hat, kappa = sc.getfloat("h", 0.01), sc.getfloat("d_hat", 1e-3), sc.getfloat("kappa", 1e4)
    frames = sc.getint("frames", 1)
    for label, val in (("h", h), ("d_hat", d_hat), ("kappa", kappa)):
        if val <= 0:
            raise ConfigError(f"[scene] {label} must be positive")
    if frames < 0:
        raise ConfigError("[scene] frames must be >= 0")
    gravity = _vec(sc.get("gravity", "0 0 -9.81"), 3, "[scene] gravity")
    out = Path(sc.get("output_dir", "out"))
    run = RunParams(gravity=gravity, h=h, frames=frames, output_dir=out if out.is_absolute() else path.parent / out,
                    seed=sc.getint("seed", 0))
    kw = {}
    for key, raw in (cp["solver"].items() if "solver" in cp else []):
        field = "K" if key == "k" else key  # configparser lowercases keys
        if field not in _SOLVER_FIELDS:
            raise ConfigError(f"[solver] unknown key {key!r}")
        kw[field] = _SOLVER_FIELDS[field](raw)
    cfg = solver.SolverConfig(**kw).validate()
    objs = [_object(cp[s], s, path.parent) for s in cp.sections() if s.startswith("mesh")]
    if not objs:
        raise ConfigError("no [mesh:*] sections")
    scene = scenes.build_scene(objs, d_hat=d_hat, kappa=kappa, gravity=tuple(gravity))
    if np.any(scene.mass <= 0):
        raise ConfigError("every vertex needs positive lumped mass")
    return scene, cfg, run


def write_scene(path, objs, h=0.01, d_hat=1e-3, kappa=1e4, frames=1, gravity=(0.0, 0.0, -9.81), solver_cfg=None,
                output_dir="out"):
    """Emit objects (scenes.build_scene dicts) as an INI + one TetGen
    .node/.ele pair per distinct mesh, loadable by this module's and the
    reference's load_config."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    lines = ["[scene]", f"gravity = {' '.join(repr(float(g)) for g in gravity)}", f"h = {h!r}",
             f"d_hat = {d_hat!r}", f"kappa = {kappa!r}", f"frames = {frames}", f"output_dir = {output_dir}", ""]
    written = {}
    for i, ob in enumerate(objs):
        mid = id(ob["mesh"])
        if mid not in written:
            base = path.with_name(f"{path.stem}_mesh{len(written)}")
            geometry.save_node_ele(base, ob["mesh"])
            written[mid] = base.name
        t = ob.get("translate", (0.0, 0.0, 0.0))
        lines += [f"[mesh:obj{i:03d}]", "kind = file", f"path = {written[mid]}",
                  f"translate = {t[0]!r} {t[1]!r} {t[2]!r}", f"material = {ob.get('material', 'arap')}",
                  f"youngs = {float(ob.get('young', 1e5))!r}", f"poisson = {float(ob.get('poisson', 0.3))!r}",
                  f"density = {float(ob.get('density', 1000.0))!r}",
                  f"pinned = {'all' if ob.get('pinned') else 'none'}", ""]
    if solver_cfg:
        lines.append("[solver]")
        lines += [f"{k} = {v}" for k, v in solver_cfg.items()]
    path.write_text("\n".join(lines) + "\n")
    return path


# ---------------------------------------------------------------------------
# frame driver (`cli.py:235-294`)


def _g(x):
    return format(float(x), ".17g")


def _simulate(scene, cfg, run, curve=None, devices=None, x0=None, v0=None):
    out = Path(run.output_dir)
    out.mkdir(parents=True, exist_ok=True)
    x = scene.mesh.rest_positions.ravel().copy() if x0 is None else np.asarray(x0, float).ravel().copy()
    v = np.zeros_like(x) if v0 is None else np.asarray(v0, float).ravel().copy()
    tris = scene.surface.triangles
    geometry.save_obj(out / "frame_00000.obj", x.reshape(-1, 3), tris)
    ctx = scene.context(cfg, devices=devices) if devices else None
    total, ok = 0, True
    with open(out / "iters.csv", "w") as fi, open(out / "frames.csv", "w") as ff:
        fi.write(ITER_COLUMNS + "\n")
        ff.write(FRAME_COLUMNS + "\n")
        for frame in range(1, run.frames + 1):
            t0 = time.perf_counter()
            try:
                if ctx is None:
                    st, tr = solver.step(scene, x, v, run.h, cfg)
                    x, v = st.x, st.v
                else:
                    x, v, recs, conv, flags = ctx.step(x, v, run.h)
                    tr = solver._trace(recs, conv, flags)
            except SimError as e:
                print(f"solver failure at frame {frame}: {e}", file=sys.stderr)
                ok = False
                break
            wall = (time.perf_counter() - t0) * 1e3
            for r in tr.records:
                fi.write(f"{frame},{r.k},{_g(r.grad_norm)},{_g(r.z_norm)},{_g(r.r)},{int(r.restart)},{_g(r.mu)},"
                         f"{_g(r.nu)},{_g(r.min_alpha)},{_g(r.t_grad_ms)},{_g(r.t_dir_ms)},{_g(r.t_ccd_ms)}\n")
            ma = min([1.0] + [r.min_alpha for r in tr.records])
            ff.write(f"{frame},{tr.iterations},{int(tr.converged)},{_g(ma)},{_g(wall)}\n")
            total += tr.iterations
            if curve is not None and frame == 1 and tr.records:
                z0 = tr.records[0].z_norm or 1.0
                curve.extend((r.k, r.z_norm / z0) for r in tr.records)
            geometry.save_obj(out / f"frame_{frame:05d}.obj", x.reshape(-1, 3), tris)
    return ok, total


def run_simulation(config_path, devices=None) -> int:
    try:
        scene, cfg, run = load_config(config_path)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    ok, total = _simulate(scene, cfg, run, devices=devices)
    if not ok:
        return EXIT_SOLVER
    print(f"wrote {run.frames + 1} frames, {total} iterations -> {run.output_dir}")
    return EXIT_OK


VARIANTS = {"mas+woodbury": "Woodbury", "mas+freeze": "Freeze", "mas+fullrebuild": "FullRebuild"}


def compare_solvers(config_path, variants) -> int:
    """`cli.py:322-353` over the variants this backend implements."""
    try:
        _, base, run0 = load_config(config_path)
        cfgs = []
        for name in variants:
            if name.lower() not in VARIANTS:
                raise ConfigError(f"variant {name!r} is not on the device path (MAS + Subspace2D variants: "
                                  f"{', '.join(VARIANTS)})")
            cfgs.append((name, dataclasses.replace(base, update_strategy=VARIANTS[name.lower()])))
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    run0.output_dir.mkdir(parents=True, exist_ok=True)
    rows = []
    for name, cfg in cfgs:
        scene, _, run = load_config(config_path)
        slug = name.replace("+", "_").lower()
        run.output_dir = run0.output_dir / slug
        curve = []
        t0 = time.perf_counter()
        try:
            ok, total = _simulate(scene, cfg, run, curve=curve)
        except SimError:
            ok, total = False, 0
        rows.append((name, "ok" if ok else "failed", total, (time.perf_counter() - t0) * 1e3))
        with open(run0.output_dir / f"curve_{slug}.csv", "w") as f:
            f.write("iter,rel_z\n" + "".join(f"{k},{_g(v)}\n" for k, v in curve))
    with open(run0.output_dir / "comparison.csv", "w") as f:
        f.write("variant,status,total_iters,wall_ms\n" + "".join(f"{n},{s},{t},{_g(w)}\n" for n, s, t, w in rows))
    for n, s, t, w in rows:
        print(f"{n}: {s}, {t} iterations, {w:.1f} ms")
    return EXIT_OK


# ---------------------------------------------------------------------------
# the penetration checker (`cli.py:360-422`), scalable


class SurfaceChecker:
    """Min PT / EE distance over non-adjacent surface primitives through the
    device broad phase: a surface-only context whose d_hat is the search
    radius, doubled until a pair is found (every pair closer than the radius
    is a broad-phase candidate, so the minimum is exact)."""

    def __init__(self, positions, triangles, device=0):
        from types import SimpleNamespace

        x = np.asarray(positions, float).reshape(-1, 3)
        tris = np.asarray(triangles, np.int64).reshape(-1, 3)
        e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [0, 2]]])
        surf = SimpleNamespace(triangles=tris, edges=np.unique(np.sort(e, axis=1), axis=0), vertices=np.unique(tris))
        n = len(x)
        ext = float(np.ptp(x, axis=0).max()) if n else 1.0
        self.r0 = max(ext * 1e-4, 1e-12)
        mesh = SimpleNamespace(rest_positions=x, tets=np.zeros((0, 4), np.int64), n_vertices=n)
        elastic = SimpleNamespace(tets=np.zeros((0, 4), np.int64), kind_id=np.zeros(0, np.int8), mu=np.zeros(0),
                                  lam=np.zeros(0), Bm=np.zeros((0, 3, 3)), vol=np.zeros(0))
        self.scene = solver.Scene(mesh=mesh, surface=surf, elastic=elastic, mass=np.ones(n),
                                  dirichlet=np.zeros(n, bool), d_hat=self.r0, kappa=1.0, f_ext=np.zeros(3 * n))
        self.ctx = self.scene.context(solver.SolverConfig(levels=0), device=device)
        self.tris, self.device, self.ext = tris, device, ext

    def min_distance(self, positions):
        x = np.asarray(positions, float).ravel()
        r = self.r0
        while True:
            self.ctx.set_contact(r, 1.0)
            try:
                _, _, d, _, _ = self.ctx.constraint_set(x)
            except PenetrationError:
                return 0.0
            if len(d):
                return float(d.min())
            if r > 4.0 * self.ext:
                return float("inf")
            r *= 4.0

    def intersections(self, positions):
        return _intersections(positions, self.tris, self.device)


def _intersections(positions, triangles, device=0):
    from . import _native

    return _native.check_intersections(positions, triangles, device)


def run_check(output_dir, device=0) -> int:
    out = Path(output_dir)
    frames = sorted(out.glob("frame_*.obj"))
    if not frames:
        print(f"no frames found in {out}", file=sys.stderr)
        return EXIT_CONFIG
    worst, checker = float("inf"), None
    for path in frames:
        x, tris = geometry.load_obj(path)
        if checker is None or len(checker.tris) != len(tris) or not np.array_equal(checker.tris, tris):
            checker = SurfaceChecker(x, tris, device)
        d = checker.min_distance(x)
        worst = min(worst, d)
        if d <= 0.0 or checker.intersections(x)[0] > 0:
            print(f"penetration in {path.name}: min distance {d:g}", file=sys.stderr)
            return EXIT_CHECK
    print(f"{len(frames)} frames checked, min surface distance {worst:g}")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2604_19892_b200", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("simulate", help="run a scene config")
    p.add_argument("config")
    p.add_argument("--devices", default=None, help="comma-separated CUDA ordinals: the partitioned multi-GPU solver")
    p = sub.add_parser("compare", help="run solver variants on one scene")
    p.add_argument("config")
    p.add_argument("--variants", required=True)
    p = sub.add_parser("check", help="verify emitted frames are penetration-free")
    p.add_argument("output_dir")
    a = ap.parse_args(argv)
    if a.command == "simulate":
        devs = [int(d) for d in a.devices.split(",")] if a.devices else None
        return run_simulation(a.config, devs)
    if a.command == "compare":
        return compare_solvers(a.config, [v for v in a.variants.split(",") if v])
    return run_check(a.output_dir)


if __name__ == "__main__":
    sys.exit(main())
