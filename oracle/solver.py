"""Oracle solver: Alg. 1 (MAS-PNCG with Subspace2D directions, Woodbury /
Freeze / FullRebuild preconditioner strategies, per-subdomain CCD).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Reference: `pkg/src/ipcsim/solver.py` -- config `:48-77`, 2x2 subspace
`:147-161`, restart ratio `:164-168`, CCD clamp `:268-280`, advance_step
`:296-458`, step `:461-464`; `energy.prepare_step` `energy.py:77-94`.
The baseline preconditioner/direction rules (Jacobi, FR/PR/DK/CD) are
outside the hot path and not restated.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import ccd as occd
from . import physics as ophys
from . import precond as opre


@dataclass
class SolverConfig:
    eps: float = 1e-5
    delta: float = 0.3
    iter_max: int = 10000
    K: int = 8
    eps_rot: float = math.cos(math.radians(25.0))
    alpha_l: float = 2.0 ** -20
    update_strategy: str = "Woodbury"
    block_size: int = 32
    levels: int = 2
    coarse_block: int = 4
    ccd_per_subdomain: bool = True


@dataclass
class Scene:
    """Static scene arrays (the reference Scene + ElasticModel + SurfaceMesh
    fields the hot path reads)."""

    rest: np.ndarray
    tets: np.ndarray
    kind: np.ndarray
    mu: np.ndarray
    lam: np.ndarray
    Bm: np.ndarray
    vol: np.ndarray
    mass: np.ndarray
    dirichlet: np.ndarray
    f_ext: np.ndarray
    tris: np.ndarray
    edges: np.ndarray
    surf_verts: np.ndarray
    d_hat: float
    kappa: float
    _parts: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self.rest = np.asarray(self.rest, float).reshape(-1, 3)
        self.n = len(self.rest)
        self.tets = np.asarray(self.tets, np.int64).reshape(-1, 4)
        self.Bm = np.asarray(self.Bm, float).reshape(-1, 3, 3)
        self.dirichlet = np.asarray(self.dirichlet, bool)
        self.tris = np.asarray(self.tris, np.int64).reshape(-1, 3)
        self.edges = np.asarray(self.edges, np.int64).reshape(-1, 2)
        self.surf_verts = np.asarray(self.surf_verts, np.int64)
        self.mass3 = np.repeat(np.asarray(self.mass, float), 3)
        self.pinned3 = np.repeat(self.dirichlet, 3)

    @classmethod
    def from_scene(cls, s):
        """From a product Scene (or any object with the reference Scene's
        attribute layout)."""
        el, sf = s.elastic, s.surface
        return cls(rest=s.mesh.rest_positions, tets=el.tets, kind=el.kind_id, mu=el.mu, lam=el.lam, Bm=el.Bm,
                   vol=el.vol, mass=s.mass, dirichlet=s.dirichlet, f_ext=s.f_ext, tris=sf.triangles, edges=sf.edges,
                   surf_verts=sf.vertices, d_hat=float(s.d_hat), kappa=float(s.kappa))

    @classmethod
    def from_golden(cls, g):
        return cls(rest=g["rest"], tets=g["tets"], kind=g["kind"], mu=g["mu"], lam=g["lam"], Bm=g["Bm"],
                   vol=g["vol"], mass=g["mass"], dirichlet=g["dirichlet"], f_ext=g["f_ext"], tris=g["tris"],
                   edges=g["edges"], surf_verts=g["surf_verts"], d_hat=float(g["d_hat"]), kappa=float(g["kappa"]))

    def partition(self, block_size):
        if block_size not in self._parts:
            self._parts[block_size] = opre.partition_domain(self.rest, block_size)
        return self._parts[block_size]


def prepare_step(scene, x, v, h):
    """x_tilde = x + h v + h^2 M^-1 f_ext; pinned: x_tilde = x, v = 0."""
    x = np.array(x, float).ravel()
    v = np.array(v, float).ravel()
    m3 = scene.mass3
    acc = np.zeros_like(x)
    np.divide(np.asarray(scene.f_ext, float).ravel(), m3, out=acc, where=m3 > 0)
    xt = x + h * v + h * h * acc
    xt[scene.pinned3] = x[scene.pinned3]
    v[scene.pinned3] = 0.0
    return x, v, xt


def solve_2d(zHz, zHp, pHz, pHp, zg, pg):
    """`solver.py:147-161`: (mu, nu) of the 2x2 subspace model."""
    if zHz <= 0.0:
        raise ophys.NotSpdError("model-not-spd", "z.Hz <= 0 in subspace solve")
    A = np.array([[zHz, -zHp], [-pHz, pHp]])
    b = np.array([zg, -pg])
    if np.linalg.cond(A) > 1e12:
        return b[0] / zHz, 0.0
    mu, nu = np.linalg.solve(A, b)
    return float(mu), float(nu)


@dataclass
class Record:
    k: int
    grad_norm: float
    z_norm: float
    r: float
    restart: bool
    mu: float
    nu: float
    min_alpha: float
    energy: float = float("nan")
    certified: bool = True


@dataclass
class Trace:
    records: list = field(default_factory=list)
    converged: bool = False
    flags: list = field(default_factory=list)

    @property
    def iterations(self):
        return len(self.records)


def advance(scene, x, x_tilde, h, cfg: SolverConfig, deadline=None, with_energy=False):
    """`solver.advance_step` (`solver.py:296-458`) restricted to MAS +
    Subspace2D.  Returns (x, v, Trace).  ``deadline`` (perf_counter time)
    stops after the iteration that crosses it (bounded CPU samples)."""
    part = scene.partition(cfg.block_size)
    pin3 = scene.pinned3
    x_start = x.copy()
    x = x.copy()
    tr = Trace()
    restart = True
    z_prev = p_prev = Hp_prev = None
    best = (math.inf, x.copy())
    full = cfg.update_strategy == "FullRebuild"
    base = H = hier = None
    for k in range(cfg.iter_max):
        rebuild = restart or full
        cs = ophys.constraint_set(scene, x)
        if rebuild:
            base = cs
            H = ophys.assemble_base_hessian(scene, x, h, cs)
            hier = opre.build_hierarchy(H, part, cfg.levels, cfg.coarse_block)
            cands = opre.Candidates(np.zeros((0, 4), np.int64), np.zeros((0, 4, 3)), np.zeros(0))
            wb = None
        else:
            cands = opre.classify_all(cs, base, cfg.eps_rot)
            wb = None
            if cfg.update_strategy != "Freeze":
                wb = opre.build_update(hier, cands, opre.select_top_k(cands, part.subdomain_of, cfg.K), cfg.K)
        g = ophys.gradient(scene, x, x_tilde, h, cs)
        z = opre.apply_preconditioner(hier, wb, g)
        z[pin3] = 0.0
        z_norm = float(np.linalg.norm(z))
        g_norm = float(np.linalg.norm(g))
        if z_norm < best[0]:
            best = (z_norm, x.copy())
        v = ophys.hvp(H, cands.verts, cands.u, z)
        zg, zv = float(z @ g), float(z @ v)
        if z_norm == 0.0:
            mu = nu = 0.0
            p = np.zeros_like(z)
            Hp = np.zeros_like(z)
        elif restart or p_prev is None:
            if zv <= 0.0:
                raise ophys.NotSpdError("model-not-spd", "z.Hz <= 0 at restart")
            mu, nu = zg / zv, 0.0
            p, Hp = -mu * z, -mu * v
        else:
            mu, nu = solve_2d(zv, float(z @ Hp_prev), float(p_prev @ v), float(p_prev @ Hp_prev), zg,
                              float(p_prev @ g))
            p = -mu * z + nu * p_prev
            Hp = -mu * v + nu * Hp_prev
            if float(g @ p) >= 0.0:
                if zv <= 0.0:
                    raise ophys.NotSpdError("model-not-spd", "z.Hz <= 0 in fallback")
                mu, nu = zg / zv, 0.0
                p, Hp = -mu * z, -mu * v
        energy = ophys.incremental_potential(scene, x, x_tilde, h, cs) if with_energy else float("nan")
        cert = True
        if np.any(p):
            x, min_alpha, _, cert, _ = occd.clamp(scene, part, x, p, cfg.ccd_per_subdomain, cfg.alpha_l)
        else:
            min_alpha = 1.0
        rec = Record(k, g_norm, z_norm, 0.0, restart, float(mu), float(nu), float(min_alpha), energy, bool(cert))
        tr.records.append(rec)
        conv = z_norm <= cfg.eps
        if conv and (restart or full):
            tr.converged = True
            break
        if conv:
            restart = True
        else:
            r = 0.0
            if z_prev is not None:
                if zg <= 0.0:
                    raise ophys.NotSpdError("precond-not-spd", "g.z <= 0 in restart ratio")
                r = abs(float(g @ z_prev)) / zg
            rec.r = r
            restart = r > cfg.delta
        z_prev, p_prev, Hp_prev = z, p, Hp
        if deadline is not None and time.perf_counter() >= deadline:
            tr.flags.append("sample-deadline")
            return x, (x - x_start) / h, tr
    else:
        tr.flags.append("not-converged")
        x = best[1]
    v_new = (x - x_start) / h
    v_new[pin3] = 0.0
    return x, v_new, tr


def step(scene, x, v, h, cfg: SolverConfig, **kw):
    """`solver.step` (`solver.py:461-464`)."""
    x, v, xt = prepare_step(scene, x, v, h)
    return advance(scene, x, xt, h, cfg, **kw)


def timed_iterations(scene, x, v, h, cfg, budget_s=20.0, max_iters=None):
    """PNCG iterations of one frame within a wall-clock budget:
    (iterations, seconds).  The CPU baseline of bench.py."""
    if max_iters:
        cfg = SolverConfig(**{**cfg.__dict__, "iter_max": int(max_iters)})
    t0 = time.perf_counter()
    _, _, tr = step(scene, x, v, h, cfg, deadline=t0 + budget_s)
    return tr.iterations, time.perf_counter() - t0


def gradient_at(scene, x, x_tilde, h):
    """energy.gradient with the constraint set at x (smoke check)."""
    cs = ophys.constraint_set(scene, x)
    return ophys.gradient(scene, np.asarray(x, float), np.asarray(x_tilde, float), h, cs)
