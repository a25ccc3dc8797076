"""Drop-in solver API: same names, fields and defaults as the reference's
``ipcsim.solver`` (`pkg/src/ipcsim/solver.py:43-140, 296-464`), executed by
the sm_100a backend.

``step`` / ``advance_step`` run the whole MAS-PNCG loop (Alg. 1) inside the
native library (``csrc/maspncg.cu: advance_loop``); Python only marshals
arrays.  The device context (uploaded scene, partition, static BSR pattern,
all solver buffers) is created once per (Scene, block_size) and cached on the
Scene, like the reference caches its partition (`solver.py:92-97`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native
from .energy import SimState, lumped_masses, prepare_step
from .errors import ConfigError

PRECONDITIONERS = ("MAS", "Jacobi")
DIRECTION_RULES = ("Subspace2D", "FR", "PR", "DK", "CD")
UPDATE_STRATEGIES = ("Woodbury", "Freeze", "FullRebuild")
ALPHA_L_DEFAULT = 2.0 ** -20


@dataclass
class SolverConfig:
    eps: float = 1e-5
    delta: float = 0.3
    iter_max: int = 10000
    K: int = 8
    eps_rot: float = math.cos(math.radians(25.0))
    alpha_l: float = ALPHA_L_DEFAULT
    preconditioner: str = "MAS"
    direction_rule: str = "Subspace2D"
    update_strategy: str = "Woodbury"
    block_size: int = 32
    levels: int = 2
    coarse_block: int = 4
    ccd_per_subdomain: bool = True

    def validate(self):
        if not self.eps > 0:
            raise ConfigError("eps must be positive")
        if not 0 < self.delta < 1:
            raise ConfigError("delta must lie in (0, 1)")
        if self.iter_max < 1:
            raise ConfigError("iter_max must be >= 1")
        if self.preconditioner not in PRECONDITIONERS:
            raise ConfigError(f"unknown preconditioner {self.preconditioner!r}")
        if self.direction_rule not in DIRECTION_RULES:
            raise ConfigError(f"unknown direction rule {self.direction_rule!r}")
        if self.update_strategy not in UPDATE_STRATEGIES:
            raise ConfigError(f"unknown update strategy {self.update_strategy!r}")
        return self

    def to_native(self) -> _native.SolverConfigC:
        return _native.SolverConfigC(
            eps=self.eps, delta=self.delta, iter_max=int(self.iter_max), K=int(self.K),
            preconditioner=PRECONDITIONERS.index(self.preconditioner),
            direction_rule=DIRECTION_RULES.index(self.direction_rule),
            update_strategy=UPDATE_STRATEGIES.index(self.update_strategy),
            block_size=int(self.block_size), levels=int(self.levels), coarse_block=int(self.coarse_block),
            ccd_per_subdomain=int(bool(self.ccd_per_subdomain)), eps_rot=float(self.eps_rot),
            alpha_l=float(self.alpha_l),
        )


@dataclass
class Partition:
    """mas.Partition (`mas.py:53-60`)."""

    subdomain_of: np.ndarray
    selection: list
    D: int
    block_size: int


@dataclass
class Scene:
    mesh: object
    surface: object
    elastic: object
    mass: np.ndarray
    dirichlet: np.ndarray
    d_hat: float
    kappa: float
    f_ext: np.ndarray
    _partitions: dict = field(default_factory=dict, repr=False)
    _contexts: dict = field(default_factory=dict, repr=False)

    def partition(self, block_size):
        if block_size not in self._partitions:
            sub = _native.partition_host(self.mesh.rest_positions, block_size)
            D = int(sub.max()) + 1 if len(sub) else 1
            order = np.argsort(sub, kind="stable")
            bounds = np.searchsorted(sub[order], np.arange(D + 1))
            selection = [order[bounds[d]:bounds[d + 1]] for d in range(D)]
            self._partitions[block_size] = Partition(sub, selection, D, block_size)
        return self._partitions[block_size]

    @classmethod
    def build(cls, mesh, elastic, density, d_hat, kappa, gravity=(0.0, 0.0, -9.81)):
        from .geometry import SurfaceMesh

        mass = lumped_masses(mesh, density)
        f_ext = (mass[:, None] * np.asarray(gravity, dtype=float)).ravel()
        return cls(mesh=mesh, surface=SurfaceMesh.from_tet_mesh(mesh), elastic=elastic, mass=mass,
                   dirichlet=mesh.dirichlet, d_hat=d_hat, kappa=kappa, f_ext=f_ext)

    # ---- device context ----
    def native_arrays(self) -> dict:
        n = len(self.mass)
        el = self.elastic
        T = 0 if el is None else len(el.vol)
        surf = self.surface
        tris = np.zeros((0, 3), np.int64) if surf is None else np.asarray(surf.triangles, np.int64)
        edges = np.zeros((0, 2), np.int64) if surf is None else np.asarray(surf.edges, np.int64)
        sverts = np.zeros(0, np.int64) if surf is None else np.asarray(surf.vertices, np.int64)
        c = np.ascontiguousarray
        return {
            "rest": c(np.asarray(self.mesh.rest_positions, np.float64).reshape(-1, 3)),
            "mass": c(self.mass, np.float64),
            "dirichlet": c(np.asarray(self.dirichlet, bool).astype(np.uint8)),
            "f_ext": c(self.f_ext, np.float64),
            "tets": c(np.asarray(el.tets, np.int64).reshape(-1, 4) if T else np.zeros((0, 4), np.int64)),
            "kind": c(np.asarray(el.kind_id, np.int8) if T else np.zeros(0, np.int8)),
            "mu": c(np.asarray(el.mu, np.float64) if T else np.zeros(0)),
            "lam": c(np.asarray(el.lam, np.float64) if T else np.zeros(0)),
            "Bm": c(np.asarray(el.Bm, np.float64).reshape(-1, 9) if T else np.zeros((0, 9))),
            "vol": c(np.asarray(el.vol, np.float64) if T else np.zeros(0)),
            "tris": c(tris.reshape(-1, 3)), "edges": c(edges.reshape(-1, 2)), "surf_verts": c(sverts),
            "d_hat": float(self.d_hat), "kappa": float(self.kappa), "n": n,
        }

    def context(self, config: SolverConfig, device: int = 0, devices=None) -> _native.NativeContext:
        """The scene's device context (cached per block size and device set).
        ``devices`` (a list of CUDA ordinals, repeats allowed) gives the
        partitioned multi-GPU solver: one shard per entry, each owning a
        contiguous Morton range of level-1 aggregates (include/maspncg.h
        mp_create_multi); its results are bitwise the single-GPU ones."""
        devs = (int(device),) if devices is None else tuple(int(d) for d in devices)
        key = (int(config.block_size), devs)
        ctx = self._contexts.get(key)
        cfg = config.to_native()
        if ctx is None:
            ctx = _native.NativeContext(self.native_arrays(), cfg, devs[0] if len(devs) == 1 else list(devs))
            self._contexts[key] = ctx
        else:
            ctx.set_config(cfg)
        return ctx


@dataclass
class IterRecord:
    k: int
    grad_norm: float
    z_norm: float
    r: float
    restart: bool
    mu: float
    nu: float
    min_alpha: float
    t_grad_ms: float
    t_dir_ms: float
    t_ccd_ms: float
    n_contacts: int = 0
    n_candidates: int = 0
    n_ccd_pairs: int = 0
    ccd_certified: bool = True
    energy: float = float("nan")


@dataclass
class SolverTrace:
    records: list = field(default_factory=list)
    converged: bool = False
    flags: list = field(default_factory=list)

    @property
    def iterations(self):
        return len(self.records)


def _trace(recs, converged, flags) -> SolverTrace:
    out = SolverTrace(converged=converged)
    for r in recs:
        out.records.append(IterRecord(
            k=int(r.k), grad_norm=r.grad_norm, z_norm=r.z_norm, r=r.r, restart=bool(r.restart), mu=r.mu,
            nu=r.nu, min_alpha=r.min_alpha, t_grad_ms=r.t_grad_ms, t_dir_ms=r.t_dir_ms, t_ccd_ms=r.t_ccd_ms,
            n_contacts=int(r.n_contacts), n_candidates=int(r.n_candidates), n_ccd_pairs=int(r.n_ccd_pairs),
            ccd_certified=bool(r.ccd_certified), energy=float(r.energy),
        ))
    if flags & 1:
        out.flags.append("not-converged")
    return out


def advance_step(scene: Scene, state: SimState, config: SolverConfig):
    """One implicit time step on a prepared state (`solver.py:296-458`)."""
    config.validate()
    ctx = scene.context(config)
    x, v, recs, conv, flags = ctx.advance(state.x, state.v, state.x_tilde, state.h)
    return replace(state, x=x, v=v), _trace(recs, conv, flags)


def step(scene: Scene, x, v, h, config: SolverConfig):
    """prepare_step + advance_step (`solver.py:461-464`); the inertia target
    is formed on the device."""
    config.validate()
    ctx = scene.context(config)
    x_out, v_out, recs, conv, flags = ctx.step(x, v, h)
    state = prepare_step(x, v, scene.mass, h, scene.f_ext, scene.dirichlet)
    return replace(state, x=x_out, v=v_out), _trace(recs, conv, flags)


def total_energy(scene: Scene, state: SimState, x, config: SolverConfig = None):
    """Incremental potential at x with a fresh constraint set
    (`solver.py:262-265`), on the device."""
    ctx = scene.context(config or SolverConfig())
    return ctx.energy(x, state.x_tilde, state.h)
