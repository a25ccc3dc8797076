"""Per-scene elastic data and the per-step state container.

Setup-time host code.  The per-iteration physics (gradient, energy, PSD
projected Hessian, HVP) is evaluated on the device by
``csrc/elastic.cu``; this module only prepares the static per-tet arrays the
device context uploads once, with the reference's conventions:

* Lame parameters (`pkg/src/ipcsim/energy.py:34-38`);
* lumped masses, a quarter of each incident tet's rest mass (`energy.py:41-54`);
* ``ElasticModel``: inverse rest-shape matrices Bm (columns = rest edges) and
  rest volumes, rejected if non-positive (`energy.py:128-149`);
* ``SimState`` / ``prepare_step``: x_tilde = x + h v + h^2 M^-1 f_ext, pinned
  vertices keep x_tilde = x and v = 0 (`energy.py:61-94`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

KIND_NONE = 0
KIND_ARAP = 1
KIND_SNH = 2
_KINDS = {"none": KIND_NONE, "arap": KIND_ARAP, "snh": KIND_SNH}


def lame_parameters(youngs, poisson):
    mu = youngs / (2.0 * (1.0 + poisson))
    lam = youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
    return mu, lam


def lumped_masses(mesh, density):
    from .geometry import tet_volumes

    m = np.zeros(mesh.n_vertices)
    if mesh.tets.size:
        vol = tet_volumes(mesh.rest_positions, mesh.tets)
        share = np.broadcast_to(np.asarray(density, dtype=float), vol.shape) * vol / 4.0
        np.add.at(m, mesh.tets.ravel(), np.repeat(share, 4))
    return m


@dataclass
class SimState:
    x: np.ndarray
    v: np.ndarray
    mass: np.ndarray
    h: float
    x_tilde: np.ndarray
    f_ext: np.ndarray

    @property
    def mass3(self):
        return np.repeat(self.mass, 3)


def prepare_step(x, v, mass, h, f_ext, dirichlet):
    x = np.array(x, dtype=float).ravel()
    v = np.array(v, dtype=float).ravel()
    f_ext = np.asarray(f_ext, dtype=float).ravel()
    m3 = np.repeat(np.asarray(mass, dtype=float), 3)
    pin3 = np.repeat(np.asarray(dirichlet, dtype=bool), 3)
    acc = np.zeros_like(x)
    np.divide(f_ext, m3, out=acc, where=m3 > 0)
    x_tilde = x + h * v + h * h * acc
    x_tilde[pin3] = x[pin3]
    v[pin3] = 0.0
    return SimState(x=x, v=v, mass=np.asarray(mass, dtype=float), h=h, x_tilde=x_tilde, f_ext=f_ext)


def _kind_id(kind):
    key = str(kind).lower()
    if key not in _KINDS:
        raise ConfigError(f"unknown elastic model {kind!r}")
    return _KINDS[key]


@dataclass
class ElasticModel:
    tets: np.ndarray
    Bm: np.ndarray  # (T, 3, 3)
    vol: np.ndarray  # (T,)
    mu: np.ndarray
    lam: np.ndarray
    kind_id: np.ndarray

    @classmethod
    def from_mesh(cls, mesh, kind, youngs, poisson):
        T = len(mesh.tets)
        mu, lam = lame_parameters(youngs, poisson)
        return cls.from_arrays(mesh, np.full(T, _kind_id(kind), np.int8), np.full(T, mu), np.full(T, lam))

    @classmethod
    def from_arrays(cls, mesh, kind_id, mu, lam):
        p = mesh.rest_positions[mesh.tets]  # (T, 4, 3)
        Dm = np.transpose(p[:, 1:] - p[:, :1], (0, 2, 1))  # columns are rest edges
        vol = np.linalg.det(Dm) / 6.0
        if np.any(vol <= 0):
            raise ConfigError("non-positive rest volume")
        return cls(
            tets=mesh.tets, Bm=np.linalg.inv(Dm), vol=vol,
            mu=np.asarray(mu, dtype=float), lam=np.asarray(lam, dtype=float),
            kind_id=np.asarray(kind_id),
        )
