"""CPU-only checks: scene setup is bit-identical to the reference's, and the
C-ABI library loads and exports every entry point include/maspncg.h declares."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN_SCENES, ROOT, load_golden

from paper_2604_19892_b200 import _native, energy, geometry, scenes


def _build(name):
    if name == "drop":
        return scenes.drop()
    if name == "locking":
        return scenes.locking()
    if name.startswith("stacked"):
        return scenes.stacked_boxes()
    if name == "cube3_capped":
        return scenes.c1_cube(3, 1e6)
    raise KeyError(name)


@pytest.mark.parametrize("name", GOLDEN_SCENES)
def test_scene_builders_bit_identical_to_reference(name):
    g = load_golden(name)
    s = _build(name)
    assert np.array_equal(s.mesh.rest_positions, g["rest"])
    assert np.array_equal(s.elastic.tets, g["tets"])
    assert np.array_equal(s.elastic.Bm, g["Bm"])
    assert np.array_equal(s.elastic.vol, g["vol"])
    assert np.array_equal(s.mass, g["mass"])
    assert np.array_equal(s.f_ext, g["f_ext"])
    assert np.array_equal(s.dirichlet, g["dirichlet"])
    assert np.array_equal(s.surface.triangles, g["tris"])
    assert np.array_equal(s.surface.edges, g["edges"])
    assert np.array_equal(s.surface.vertices, g["surf_verts"])


def test_box_surface_counts():
    m = geometry.make_box_mesh(2, 1, 3)
    surf = geometry.SurfaceMesh.from_tet_mesh(m)
    assert len(surf.triangles) == 2 * 2 * (2 * 1 + 1 * 3 + 2 * 3)
    assert np.all(geometry.tet_volumes(m.rest_positions, m.tets) > 0)


def test_prepare_step_matches_definition():
    mass = np.array([1.0, 2.0])
    x = np.arange(6, dtype=float)
    v = np.ones(6)
    f = np.array([0, 0, -9.81, 0, 0, -19.62])
    st = energy.prepare_step(x, v, mass, 0.1, f, np.array([False, True]))
    assert np.allclose(st.x_tilde[:3], x[:3] + 0.1 + np.array([0, 0, -0.0981]))
    assert np.array_equal(st.x_tilde[3:], x[3:])
    assert np.all(st.v[3:] == 0.0)


def _declared_symbols():
    text = (ROOT / "include" / "maspncg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    names = _declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # status-code strings are the reference error codes (errors.py)
    lib.mp_status_code.restype = ctypes.c_char_p
    assert lib.mp_status_code(1) == b"penetration-detected"
    assert lib.mp_status_code(2) == b"non-spd-subdomain"
    assert lib.mp_status_code(3) == b"capacitance-not-spd"


def test_native_partition_is_morton_blocks():
    rng = np.random.default_rng(3)
    pts = rng.random((53, 3))
    sub = _native.partition_host(pts, 8)
    assert sub.max() == 6
    counts = np.bincount(sub)
    assert sorted(counts) == [5] + [8] * 6


def test_c2_bench_scene_bit_identical_to_reference():
    """Our config-2 builder gives the reference-built bench scene bit for bit
    (sha256 over every array, recorded by tests/golden/make_c2_golden.py)."""
    import hashlib

    import bench

    s = scenes.c2_stack(gap=bench.GAP)
    h = hashlib.sha256()
    el, sf = s.elastic, s.surface
    for a in (s.mesh.rest_positions, el.tets, el.Bm, el.vol, el.mu, el.lam, s.mass, s.dirichlet, s.f_ext,
              sf.triangles, sf.edges, sf.vertices):
        h.update(np.ascontiguousarray(a).tobytes())
    with np.load(ROOT / "tests" / "golden" / "c2_bench.npz") as z:
        assert h.hexdigest() == str(z["scene_sha256"])
