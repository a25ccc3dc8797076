"""Synthetic scene generators for parity tests and the benchmark.

Every builder takes an optional ``mods=(geometry, energy, solver)`` triple so
the same scene can be built with this package or -- in the golden-fixture
script only -- with the reference package, which has the same names
(`pkg/tests/test_acceptance.py:37-78` for the object-list convention).

Configs (BASELINE.json ``configs``):

* ``c1_cube``  -- floor slab + soft SNH cube ``cells^3`` (8^3: 737 V, 3,078 T)
* ``c2_stack`` -- floor + 8 cubes (17^3 cells each) stacked 2x2x2 with 1e-3 gaps
  (46,664 V, 235,830 T), SNH E=1e5, d_hat=2e-3, kappa=1e4, h=0.01
* ``c3_rod``   -- twisting soft SNH rod (8 x 8 x 2500 cells; 202,589 V / 960,006 T with the floor
  at full size) released above a pinned floor with a linear twist-rate
  field (``c3_rod_v0``): opposite ends spin in opposite senses, so the rod
  winds up and presses on itself; SURVEY.md 8.0 C3
* small reference-shaped scenes used by the golden fixtures: ``drop``
  (scenes/drop.ini), ``stacked_boxes`` (test_acceptance.py:369-388),
  ``locking`` (test_acceptance.py:488-499).
"""

from __future__ import annotations

import numpy as np


def _mods(mods):
    if mods is None:
        from . import energy, geometry, solver

        return geometry, energy, solver
    return mods


def build_scene(objs, d_hat, kappa, gravity=(0.0, 0.0, -9.81), mods=None):
    """Concatenate object meshes into one Scene.

    objs: dicts with mesh, translate, material ('arap'|'snh'), young, poisson,
    density, pinned (whole object) or pin_mask (per vertex)."""
    geo, en, sol = _mods(mods)
    verts, tets, pin, kinds, mus, lams, rhos = [], [], [], [], [], [], []
    off = 0
    for ob in objs:
        m = ob["mesh"]
        verts.append(m.rest_positions + np.asarray(ob.get("translate", (0.0, 0.0, 0.0))))
        tets.append(m.tets + off)
        pin.append(np.asarray(ob["pin_mask"], bool) if "pin_mask" in ob
                   else np.full(len(m.rest_positions), bool(ob.get("pinned", False))))
        T = len(m.tets)
        mu, lam = en.lame_parameters(ob.get("young", 1e5), ob.get("poisson", 0.3))
        kinds.append(np.full(T, 1 if ob.get("material", "arap") == "arap" else 2, dtype=np.int8))
        mus.append(np.full(T, mu))
        lams.append(np.full(T, lam))
        rhos.append(np.full(T, ob.get("density", 1000.0)))
        off += len(m.rest_positions)
    mesh = geo.TetMesh(rest_positions=np.vstack(verts), tets=np.vstack(tets), dirichlet=np.concatenate(pin))
    elastic = en.ElasticModel.from_arrays(mesh, np.concatenate(kinds), np.concatenate(mus), np.concatenate(lams))
    mass = en.lumped_masses(mesh, np.concatenate(rhos))
    return sol.Scene(
        mesh=mesh, surface=geo.SurfaceMesh.from_tet_mesh(mesh), elastic=elastic, mass=mass,
        dirichlet=mesh.dirichlet, d_hat=d_hat, kappa=kappa,
        f_ext=(mass[:, None] * np.asarray(gravity)).ravel(),
    )


def floor(size=(1.0, 1.0, 0.1), mods=None):
    geo, _, _ = _mods(mods)
    return {
        "mesh": geo.make_box_mesh(1, 1, 1, size),
        "translate": (-size[0] / 2, -size[1] / 2, -size[2]),
        "material": "arap", "young": 1e6, "pinned": True,
    }


def drop(mods=None):
    """scenes/drop.ini: one SNH tet over a pinned slab."""
    geo, _, _ = _mods(mods)
    objs = [floor((1.0, 1.0, 0.1), mods),
            {"mesh": geo.make_single_tet(0.2), "translate": (-0.05, -0.05, 0.05), "material": "snh",
             "young": 5e4, "poisson": 0.3, "density": 1000.0}]
    return build_scene(objs, d_hat=2e-3, kappa=1e4, mods=mods)


def stacked_boxes(mods=None):
    """test_acceptance.py:369-388 (three stiff 2x2x2 boxes pressing in)."""
    geo, _, _ = _mods(mods)
    box = geo.make_box_mesh(2, 2, 2, (0.3, 0.3, 0.3))
    objs = [floor((1.2, 1.2, 0.1), mods)]
    z = 0.0036
    for i, gap in enumerate((0.0036, 0.0036, 0.0040)):
        if i:
            z += 0.3 + gap
        objs.append({"mesh": box, "translate": (-0.15, -0.15, z), "material": "arap", "young": 1e7,
                     "density": 1000.0})
    return build_scene(objs, d_hat=4e-3, kappa=2e4, mods=mods)


def stacked_boxes_v0(scene):
    v0 = np.zeros((scene.mesh.n_vertices, 3))
    v0[8:, 2] = -0.05
    return v0.ravel()


def locking(mods=None):
    """test_acceptance.py:488-499."""
    geo, _, _ = _mods(mods)
    box = geo.make_box_mesh(1, 1, 1, (0.2, 0.2, 0.2))
    objs = [floor((1.2, 1.2, 0.1), mods),
            {"mesh": box, "translate": (-0.35, -0.35, 0.001), "material": "arap", "young": 2e5},
            {"mesh": box, "translate": (0.15, 0.15, 0.15), "material": "arap", "young": 2e5}]
    return build_scene(objs, d_hat=3e-3, kappa=1e4, mods=mods)


def c1_cube(cells=8, young=5e4, material="snh", gap=0.01, mods=None):
    """Config 1: pinned floor + soft cube of cells^3 (0.2 m), SURVEY 8(d) C1."""
    geo, _, _ = _mods(mods)
    cube = geo.make_box_mesh(cells, cells, cells, (0.2, 0.2, 0.2))
    objs = [floor((1.0, 1.0, 0.1), mods),
            {"mesh": cube, "translate": (-0.1, -0.1, gap), "material": material, "young": young,
             "poisson": 0.3, "density": 1000.0}]
    return build_scene(objs, d_hat=2e-3, kappa=1e4, mods=mods)


def c2_stack(cells=17, young=1e5, gap=1e-3, mods=None):
    """Config 2: 8 soft SNH cubes (cells^3, 0.2 m) stacked 2x2x2 above a pinned
    1.2 x 1.2 x 0.1 floor, 1e-3 gaps (46,664 V / 235,830 T at cells=17)."""
    geo, _, _ = _mods(mods)
    cube = geo.make_box_mesh(cells, cells, cells, (0.2, 0.2, 0.2))
    objs = [floor((1.2, 1.2, 0.1), mods)]
    for iz in range(2):
        for iy in range(2):
            for ix in range(2):
                objs.append({
                    "mesh": cube,
                    "translate": (-0.2 - 0.5 * gap + ix * (0.2 + gap), -0.2 - 0.5 * gap + iy * (0.2 + gap),
                                  gap + iz * (0.2 + gap)),
                    "material": "snh", "young": young, "poisson": 0.3, "density": 1000.0,
                })
    return build_scene(objs, d_hat=2e-3, kappa=1e4, mods=mods)


def c3_rod(cells=(2500, 8, 8), length=6.25, width=0.02, young=1e5, gap=2e-3, mods=None):
    """Config 3 surrogate: a soft SNH rod along x (cells = (nx, ny, nz)) held
    gap above a pinned floor; pair with ``c3_rod_v0`` for the twist."""
    geo, _, _ = _mods(mods)
    nx, ny, nz = cells
    rod = geo.make_box_mesh(nx, ny, nz, (length, width, width))
    objs = [floor((length + 0.4, 0.4, 0.1), mods),
            {"mesh": rod, "translate": (-0.5 * length, -0.5 * width, gap), "material": "snh", "young": young,
             "poisson": 0.3, "density": 1000.0}]
    return build_scene(objs, d_hat=2e-3, kappa=1e4, mods=mods)


def c3_rod_v0(scene, omega=5.0):
    """Twist field: angular velocity about the rod axis varying linearly from
    -omega at one end to +omega at the other; the pinned floor stays at rest.
    omega = 5 rad/s moves the rod's surface 0.5 mm per 10 ms step (a fifth
    of an element); round 1 used 20 rad/s (2 mm, 80% of an element per step,
    which turned every iteration into a 10^9-candidate CCD)."""
    x = scene.mesh.rest_positions
    rod = ~np.asarray(scene.dirichlet, dtype=bool)
    xr = x[rod]
    lo, hi = xr.min(axis=0), xr.max(axis=0)
    c = 0.5 * (lo + hi)
    w = omega * (2.0 * (xr[:, 0] - lo[0]) / max(hi[0] - lo[0], 1e-30) - 1.0)
    v = np.zeros_like(x)
    v[rod, 1] = -w * (xr[:, 2] - c[2])
    v[rod, 2] = w * (xr[:, 1] - c[1])
    return v.ravel()


SCENES = {
    "drop": drop,
    "stacked_boxes": stacked_boxes,
    "locking": locking,
    "c1_cube": c1_cube,
    "c2_stack": c2_stack,
    "c3_rod": c3_rod,
}


# ---------------------------------------------------------------------------
# C4 / C5: voxel (6-tet Kuhn) meshes of the paper's shapes, SURVEY.md 8(d)


def sphere_mesh(radius_cells=12, cell=0.05 / 12, mods=None):
    """Voxel ball: the cells of a (2R)^3 grid whose centres lie within R
    cells of the centre (R = 12: 7,153 V / 40,488 T -- SURVEY's ~7.8k V)."""
    geo, _, _ = _mods(mods)
    n = 2 * radius_cells
    c = geo.cell_centres((n, n, n), 1.0) - radius_cells
    mask = np.einsum("...k,...k->...", c, c) <= radius_cells ** 2
    return geo.voxel_tet_mesh(mask, cell, origin=(-radius_cells * cell,) * 3)


def bowl_mesh(inner=0.42, thickness=0.04, cell=0.02, mods=None):
    """Voxel hemispherical shell (the lower half, rim at z = 0) of inner
    radius ``inner``: the pinned bowl of config 4."""
    geo, _, _ = _mods(mods)
    R = inner + thickness
    n = int(np.ceil(2 * R / cell))
    nz = int(np.ceil(R / cell))
    org = (-0.5 * n * cell, -0.5 * n * cell, -nz * cell)
    c = geo.cell_centres((n, n, nz), cell, org)
    r = np.sqrt(np.einsum("...k,...k->...", c, c))
    return geo.voxel_tet_mesh((r >= inner) & (r <= R), cell, origin=org)


def c4_spheres_in_bowl(n_side=4, radius_cells=12, radius=0.05, gap=0.01, young=1e5, mods=None):
    """Config 4: n_side^3 soft SNH voxel balls (64 at n_side = 4, ~7.2k V
    each) in a cubic lattice falling into a pinned ARAP bowl; SNH E = 1e5,
    d_hat = 1e-3, kappa = 1e4."""
    ball = sphere_mesh(radius_cells, radius / radius_cells, mods)
    pitch = 2 * radius + gap
    half = 0.5 * (n_side - 1) * pitch
    objs = [{"mesh": bowl_mesh(inner=max(0.42, 1.5 * half + 2 * radius), mods=mods), "material": "arap",
             "young": 1e6, "pinned": True, "translate": (0.0, 0.0, 0.0)}]
    z0 = -0.5 * max(0.42, 1.5 * half + 2 * radius) + radius + 2 * gap
    for iz in range(n_side):
        for iy in range(n_side):
            for ix in range(n_side):
                objs.append({"mesh": ball, "material": "snh", "young": young, "poisson": 0.3, "density": 1000.0,
                             "translate": (-half + ix * pitch, -half + iy * pitch, z0 + iz * pitch)})
    return build_scene(objs, d_hat=1e-3, kappa=1e4, mods=mods)


def _fibonacci_dirs(n):
    k = np.arange(n) + 0.5
    phi = np.arccos(1.0 - 2.0 * k / n)
    theta = np.pi * (1.0 + 5.0 ** 0.5) * k
    return np.stack([np.cos(theta) * np.sin(phi), np.sin(theta) * np.sin(phi), np.cos(phi)], axis=1)


def puffer_mesh(core_cells=19, spike_cells=64, n_spikes=410, base_cells=0.84, tip_cells=0.55, cell=0.1 / 64,
                mods=None):
    """Puffer ball: a voxel sphere core of radius core_cells plus n_spikes
    thin conical spikes (Fibonacci directions) tapering from base_cells to
    tip_cells in radius out to spike_cells.  Defaults: 142,848 V / 342,960 T
    per ball (T/V = 2.40), eight balls 1.143M V / 2.744M T -- the paper's
    1.14M V / 2.72M T puffer-ball scene; 0.2 m across."""
    geo, _, _ = _mods(mods)
    n = 2 * spike_cells + 2
    c = geo.cell_centres((n, n, n), 1.0) - 0.5 * n
    r = np.sqrt(np.einsum("...k,...k->...", c, c))
    mask = r <= core_cells
    inside = r <= spike_cells
    cs, rs = c[inside], r[inside]
    spikes = np.zeros(len(cs), dtype=bool)
    for d in _fibonacci_dirs(n_spikes):
        t = cs @ d  # coordinate along the spike
        perp = np.sqrt(np.maximum(rs * rs - t * t, 0.0))
        frac = np.clip((t - core_cells) / (spike_cells - core_cells), 0.0, 1.0)
        spikes |= (t > 0.0) & (perp <= base_cells + (tip_cells - base_cells) * frac)
    mask[inside] |= spikes
    return geo.voxel_tet_mesh(mask, cell, origin=(-0.5 * n * cell,) * 3)


def c5_puffer_balls(young=1e5, gap=1e-3, mods=None, **puffer):
    """Config 5: eight puffer balls at the corners of a cube, flying at each
    other (``c5_puffer_v0``); SNH E = 1e5, h = 0.005, d_hat = 1e-4 (the
    paper's collision scene).  No floor, no gravity: the
    balls only meet each other."""
    ball = puffer_mesh(mods=mods, **puffer)
    ext = float(np.ptp(ball.rest_positions, axis=0).max())
    s = 0.5 * ext + 0.5 * gap  # corners: bounding boxes gap apart
    objs = [{"mesh": ball, "material": "snh", "young": young, "poisson": 0.3, "density": 1000.0,
             "translate": (sx * s, sy * s, sz * s)}
            for sz in (-1, 1) for sy in (-1, 1) for sx in (-1, 1)]
    return build_scene(objs, d_hat=1e-4, kappa=1e4, gravity=(0.0, 0.0, 0.0), mods=mods)


def c5_puffer_v0(scene, speed=0.1):
    """Each ball moves toward the scene centre at ``speed`` m/s."""
    x = scene.mesh.rest_positions
    n = len(x) // 8
    v = np.zeros_like(x)
    for b in range(8):
        sl = slice(b * n, (b + 1) * n)
        c = x[sl].mean(axis=0)
        v[sl] = -speed * c / max(np.linalg.norm(c), 1e-30)
    return v.ravel()


SCENES.update({"c4_spheres_in_bowl": c4_spheres_in_bowl, "c5_puffer_balls": c5_puffer_balls})
