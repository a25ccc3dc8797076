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
# file formats (`geometry.py:566-647`)


def _rows(path):
    with open(path) as fh:
        for line in fh:
            body = line.split("#", 1)[0].split()
            if body:
                yield body


def load_node_ele(path_base) -> TetMesh:
    base = str(path_base)
    if base.endswith((".node", ".ele")):
        base = base.rsplit(".", 1)[0]
    nodes = list(_rows(base + ".node"))
    n = int(nodes[0][0])
    if int(nodes[0][1]) != 3:
        raise ConfigError(f"{base}.node: expected 3-D points")
    ids = np.array([int(r[0]) for r in nodes[1:1 + n]])
    pts = np.array([[float(c) for c in r[1:4]] for r in nodes[1:1 + n]]).reshape(-1, 3)
    first = int(ids.min()) if n else 0
    pts = pts[np.argsort(ids, kind="stable")]
    eles = list(_rows(base + ".ele"))
    m = int(eles[0][0])
    if int(eles[0][1]) != 4:
        raise ConfigError(f"{base}.ele: expected 4-node tets")
    tets = np.array([[int(c) for c in r[1:5]] for r in eles[1:1 + m]], dtype=np.int64).reshape(-1, 4)
    if tets.size and tets.min() >= first:
        tets -= first
    if tets.size and (tets.min() < 0 or tets.max() >= n):
        raise ConfigError(f"{base}.ele: node index out of range")
    if tets.size:
        flip = tet_volumes(pts, tets) < 0
        tets[flip, 2], tets[flip, 3] = tets[flip, 3].copy(), tets[flip, 2].copy()
    return TetMesh(rest_positions=pts, tets=tets)


def save_node_ele(path_base, mesh: TetMesh):
    base = str(path_base)
    with open(base + ".node", "w") as fh:
        fh.write(f"{mesh.n_vertices} 3 0 0\n")
        fh.writelines(f"{i} {p[0]:.17g} {p[1]:.17g} {p[2]:.17g}\n" for i, p in enumerate(mesh.rest_positions))
    with open(base + ".ele", "w") as fh:
        fh.write(f"{len(mesh.tets)} 4 0\n")
        fh.writelines(f"{i} {t[0]} {t[1]} {t[2]} {t[3]}\n" for i, t in enumerate(mesh.tets))


def save_obj(path, positions, triangles, groups=None):
    out = [f"v {p[0]:.17g} {p[1]:.17g} {p[2]:.17g}" for p in np.asarray(positions).reshape(-1, 3)]
    for name, lo, hi in groups or [("surface", 0, len(triangles))]:
        out.append(f"o {name}")
        out.extend(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}" for t in triangles[lo:hi])
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")


def load_obj(path):
    verts, tris = [], []
    for row in _rows(path):
        if row[0] == "v":
            verts.append([float(c) for c in row[1:4]])
        elif row[0] == "f":
            tris.append([int(tok.split("/", 1)[0]) - 1 for tok in row[1:4]])
    return np.array(verts, dtype=float).reshape(-1, 3), np.array(tris, dtype=np.int64).reshape(-1, 3)
