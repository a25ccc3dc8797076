"""Scene-setup geometry: tet meshes, boundary extraction, builders and file IO.

This is host-side, once-per-scene data preparation feeding the device
context; nothing here runs inside the PNCG loop.  It reproduces the
reference's mesh conventions exactly so a scene built here is bit-identical
to one built by the reference:

* ``make_box_mesh`` -- Kuhn 6-tet split per cell with the orientation fix
  (`pkg/src/ipcsim/geometry.py:510-552`);
* ``SurfaceMesh.from_tet_mesh`` -- boundary faces = faces seen once, kept in
  the orientation of their tet, sorted; unique sorted edges
  (`pkg/src/ipcsim/geometry.py:386-405`);
* TetGen ``.node/.ele`` and OBJ readers/writers (`geometry.py:566-647`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

# faces of a positively oriented tet, outward (`geometry.py:330`)
TET_FACES = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]], dtype=np.int64)

# Kuhn subdivision of a cube into 6 tets, corner indices (`geometry.py:510-517`)
KUHN_TETS = np.array(
    [[0, 1, 3, 7], [0, 1, 7, 5], [0, 5, 7, 4], [0, 3, 2, 7], [0, 2, 6, 7], [0, 6, 4, 7]],
    dtype=np.int64,
)


def tet_volumes(positions, tets):
    """Signed tet volumes (det of edge rows / 6), as `geometry.py:333-336`."""
    p = np.asarray(positions, dtype=float)
    t = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    if len(t) == 0:
        return np.zeros(0)
    e = p[t[:, 1:]] - p[t[:, :1]]  # (T, 3, 3) rows are edges
    return np.linalg.det(e) / 6.0


@dataclass
class TetMesh:
    rest_positions: np.ndarray
    tets: np.ndarray
    positions: np.ndarray = None
    dirichlet: np.ndarray = None

    def __post_init__(self):
        self.rest_positions = np.asarray(self.rest_positions, dtype=float).reshape(-1, 3)
        self.tets = np.asarray(self.tets, dtype=np.int64).reshape(-1, 4)
        if self.positions is None:
            self.positions = self.rest_positions.copy()
        if self.dirichlet is None:
            self.dirichlet = np.zeros(len(self.rest_positions), dtype=bool)
        self.dirichlet = np.asarray(self.dirichlet, dtype=bool)
        self.validate()

    @property
    def n_vertices(self):
        return len(self.rest_positions)

    def validate(self):
        if self.tets.size:
            vols = tet_volumes(self.rest_positions, self.tets)
            if np.any(vols <= 0.0):
                bad = int(np.argmin(vols))
                raise ConfigError(f"tet {bad} has non-positive rest volume {vols[bad]:g}")
            if self.tets.min() < 0 or self.tets.max() >= self.n_vertices:
                raise ConfigError("tet index out of range")


@dataclass
class SurfaceMesh:
    triangles: np.ndarray  # (F, 3) oriented, sorted lexicographically
    edges: np.ndarray  # (E, 2) each row sorted, rows sorted
    vertices: np.ndarray  # (V,) surface vertex ids, ascending

    @classmethod
    def from_tet_mesh(cls, mesh) -> "SurfaceMesh":
        tets = np.asarray(mesh.tets, dtype=np.int64).reshape(-1, 4)
        if len(tets) == 0:
            z3 = np.zeros((0, 3), np.int64)
            return cls(triangles=z3, edges=np.zeros((0, 2), np.int64), vertices=np.zeros(0, np.int64))
        faces = tets[:, TET_FACES].reshape(-1, 3)  # oriented, tet-major order
        keys = np.sort(faces, axis=1)
        _, inv, counts = np.unique(keys, axis=0, return_inverse=True, return_counts=True)
        boundary = faces[counts[inv.ravel()] == 1]
        order = np.lexsort((boundary[:, 2], boundary[:, 1], boundary[:, 0]))
        tris = boundary[order]
        e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [0, 2]]])
        e = np.unique(np.sort(e, axis=1), axis=0)
        verts = np.unique(tris)
        return cls(triangles=tris, edges=e.reshape(-1, 2), vertices=verts)


def make_box_mesh(nx=1, ny=1, nz=1, size=(1.0, 1.0, 1.0)) -> TetMesh:
    """Box [0,sx]x[0,sy]x[0,sz], 6 Kuhn tets per cell, same ordering as the
    reference builder (`geometry.py:520-552`)."""
    sx, sy, sz = size
    gx, gy, gz = np.meshgrid(
        np.linspace(0.0, sx, nx + 1), np.linspace(0.0, sy, ny + 1), np.linspace(0.0, sz, nz + 1),
        indexing="ij",
    )
    verts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()

    def vid(a, b, c):
        return (a * (ny + 1) + b) * (nz + 1) + c

    corners = np.stack(
        [vid(i, j, k), vid(i + 1, j, k), vid(i, j + 1, k), vid(i + 1, j + 1, k),
         vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i, j + 1, k + 1), vid(i + 1, j + 1, k + 1)],
        axis=1,
    )  # (cells, 8)
    tets = corners[:, KUHN_TETS].reshape(-1, 4).copy()
    if len(tets):
        e = verts[tets[:, 1:]] - verts[tets[:, :1]]
        flip = np.linalg.det(e) < 0
        tets[flip, 2], tets[flip, 3] = tets[flip, 3].copy(), tets[flip, 2].copy()
    return TetMesh(rest_positions=verts, tets=tets)


def make_single_tet(scale=1.0) -> TetMesh:
    verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]) * scale
    return TetMesh(rest_positions=verts, tets=np.array([[0, 1, 2, 3]]))


# ---------------------------------------------------------------------------
# voxel tet meshes (the C4 / C5 generators)


def voxel_tet_mesh(mask, cell, origin=(0.0, 0.0, 0.0)) -> TetMesh:
    """Tet mesh of the occupied cells of a boolean grid ``mask`` (nx, ny, nz)
    of edge ``cell``: the used grid corners (in grid order) and the same
    6-tet Kuhn split with orientation fix as ``make_box_mesh`` -- a box mask
    gives make_box_mesh's mesh up to vertex numbering."""
    mask = np.asarray(mask, dtype=bool)
    nx, ny, nz = mask.shape
    i, j, k = np.nonzero(mask)

    def vid(a, b, c):
        return (a * (ny + 1) + b) * (nz + 1) + c

    corners = np.stack([vid(i, j, k), vid(i + 1, j, k), vid(i, j + 1, k), vid(i + 1, j + 1, k),
                        vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i, j + 1, k + 1), vid(i + 1, j + 1, k + 1)],
                       axis=1)
    used, inv = np.unique(corners, return_inverse=True)
    a = used // ((ny + 1) * (nz + 1))
    b = (used // (nz + 1)) % (ny + 1)
    c = used % (nz + 1)
    verts = np.stack([a, b, c], axis=1) * float(cell) + np.asarray(origin, dtype=float)
    tets = inv.reshape(-1, 8)[:, KUHN_TETS].reshape(-1, 4).copy()
    if len(tets):
        e = verts[tets[:, 1:]] - verts[tets[:, :1]]
        flip = np.linalg.det(e) < 0
        tets[flip, 2], tets[flip, 3] = tets[flip, 3].copy(), tets[flip, 2].copy()
    return TetMesh(rest_positions=verts, tets=tets)


def cell_centres(shape, cell, origin=(0.0, 0.0, 0.0)):
    """(nx, ny, nz, 3) centres of a voxel grid."""
    axes = [origin[d] + cell * (np.arange(shape[d]) + 0.5) for d in range(3)]
    return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)


# ---------------------------------------------------------------------------
# TetGen .node/.ele and OBJ (the reference's scene file formats,
# `geometry.py:566-647`): whole-array parsing, '#' comments, 0- or 1-based
# node ids (the smallest node id is the base), inverted tets repaired.


def _table(path):
    """Non-comment rows of a whitespace table as a list of token lists."""
    with open(path) as fh:
        text = fh.read()
    return [ln.split() for ln in (raw.partition("#")[0] for raw in text.splitlines()) if ln.strip()]


def load_node_ele(path_base) -> TetMesh:
    base = str(path_base)
    if base.endswith((".node", ".ele")):
        base = base[: base.rfind(".")]
    rows = _table(base + ".node")
    n, dim = int(rows[0][0]), int(rows[0][1])
    if dim != 3:
        raise ConfigError(f"{base}.node: expected 3-D points")
    body = np.array([r[:4] for r in rows[1:1 + n]], dtype=float).reshape(-1, 4)
    ids = body[:, 0].astype(np.int64)
    pts = body[np.argsort(ids, kind="stable"), 1:4]
    first = int(ids.min()) if n else 0
    rows = _table(base + ".ele")
    m, per = int(rows[0][0]), int(rows[0][1])
    if per != 4:
        raise ConfigError(f"{base}.ele: expected 4-node tets")
    tets = np.array([r[1:5] for r in rows[1:1 + m]], dtype=np.int64).reshape(-1, 4)
    if tets.size and tets.min() >= first:
        tets = tets - first
    if tets.size and (tets.min() < 0 or tets.max() >= n):
        raise ConfigError(f"{base}.ele: node index out of range")
    if tets.size:
        bad = tet_volumes(pts, tets) < 0
        tets[bad] = tets[bad][:, [0, 1, 3, 2]]
    return TetMesh(rest_positions=pts, tets=tets)


def save_node_ele(path_base, mesh: TetMesh):
    base = str(path_base)
    n, m = mesh.n_vertices, len(mesh.tets)
    idx = np.arange(n, dtype=np.int64)[:, None]
    with open(base + ".node", "w") as fh:
        fh.write(f"{n} 3 0 0\n")
        np.savetxt(fh, np.hstack([idx, mesh.rest_positions]), fmt=["%d", "%.17g", "%.17g", "%.17g"])
    with open(base + ".ele", "w") as fh:
        fh.write(f"{m} 4 0\n")
        np.savetxt(fh, np.hstack([np.arange(m, dtype=np.int64)[:, None], mesh.tets]), fmt="%d")


def save_obj(path, positions, triangles, groups=None):
    """Surface OBJ; ``groups`` = [(name, lo, hi)] triangle ranges as 'o' records."""
    with open(path, "w") as fh:
        np.savetxt(fh, np.asarray(positions, dtype=float).reshape(-1, 3), fmt="v %.17g %.17g %.17g")
        tri = np.asarray(triangles, dtype=np.int64).reshape(-1, 3) + 1
        for name, lo, hi in groups or [("surface", 0, len(tri))]:
            fh.write(f"o {name}\n")
            np.savetxt(fh, tri[lo:hi], fmt="f %d %d %d")


def load_obj(path):
    verts, tris = [], []
    for r in _table(path):
        if r[0] == "v":
            verts.append(r[1:4])
        elif r[0] == "f":
            tris.append([t.split("/", 1)[0] for t in r[1:4]])
    v = np.array(verts, dtype=float).reshape(-1, 3)
    f = np.array(tris, dtype=np.int64).reshape(-1, 3) - 1
    return v, f
