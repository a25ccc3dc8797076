"""The command-line surface (paper_2604_19892_b200/cli.py) against the
reference's schema (`pkg/src/ipcsim/cli.py:145-228`): INI -> Scene equal to
the in-memory builders, generated scenes (C4 / C5 shapes) round-trip through
INI + TetGen files, and -- when the reference is importable in this
container -- the reference's own load_config reads our generated files to
the same arrays.  GPU: a simulate run, its CSV/OBJ outputs, and the scalable
checker against a brute-force oracle and a planted intersection."""

import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2604_19892_b200 import cli, geometry, scenes

DATA = Path(__file__).resolve().parent / "data"
REF = Path("/root/reference/pkg/src")


def _same_scene(a, b):
    assert np.array_equal(a.mesh.rest_positions, b.mesh.rest_positions)
    assert np.array_equal(a.elastic.tets, b.elastic.tets)
    assert np.array_equal(a.elastic.Bm, b.elastic.Bm) and np.array_equal(a.elastic.vol, b.elastic.vol)
    assert np.array_equal(a.mass, b.mass) and np.array_equal(a.f_ext, b.f_ext)
    assert np.array_equal(a.dirichlet, b.dirichlet)
    assert np.array_equal(a.surface.triangles, b.surface.triangles)


def test_load_config_matches_builder():
    scene, cfg, run = cli.load_config(DATA / "drop_like.ini")
    _same_scene(scene, scenes.drop())
    assert cfg.iter_max == 200 and cfg.K == 8 and run.frames == 3 and run.h == 0.01
    assert run.output_dir == DATA / "out_drop"


def test_load_config_errors(tmp_path):
    from paper_2604_19892_b200.errors import ConfigError

    bad = tmp_path / "bad.ini"
    bad.write_text("[scene]\nh = -1\n[mesh:a]\nkind = box\n")
    with pytest.raises(ConfigError):
        cli.load_config(bad)
    bad.write_text("[scene]\n[mesh:a]\nkind = sphere\n")
    with pytest.raises(ConfigError):
        cli.load_config(bad)
    bad.write_text("[scene]\n[solver]\nbogus = 1\n[mesh:a]\n")
    with pytest.raises(ConfigError):
        cli.load_config(bad)


def test_pinned_selector(tmp_path):
    p = tmp_path / "s.ini"
    p.write_text("[scene]\n[mesh:a]\nkind = box\ncells = 2 1 1\nsize = 2 1 1\npinned = x < 0.5\n")
    scene, _, _ = cli.load_config(p)
    assert np.array_equal(scene.dirichlet, scene.mesh.rest_positions[:, 0] < 0.5)


def _small_c4(tmp_path):
    ball = scenes.sphere_mesh(3, 0.01)
    objs = [{"mesh": scenes.bowl_mesh(inner=0.05, thickness=0.01, cell=0.01), "material": "arap", "young": 1e6,
             "pinned": True},
            {"mesh": ball, "material": "snh", "young": 1e5, "translate": (0.0, 0.0, -0.02)},
            {"mesh": ball, "material": "snh", "young": 1e5, "translate": (0.0, 0.0, 0.05)}]
    path = cli.write_scene(tmp_path / "c4_small.ini", objs, d_hat=1e-3, frames=2, solver_cfg={"coarse_block": 32})
    return objs, path


def test_generated_scene_roundtrip(tmp_path):
    objs, path = _small_c4(tmp_path)
    scene, cfg, _ = cli.load_config(path)
    _same_scene(scene, scenes.build_scene(objs, d_hat=1e-3, kappa=1e4))
    assert cfg.coarse_block == 32


@pytest.mark.skipif(not REF.exists(), reason="the reference is only importable in the build container")
def test_reference_loads_generated_scene(tmp_path):
    objs, path = _small_c4(tmp_path)
    sys.path.insert(0, str(REF))
    try:
        import ipcsim.cli as rcli
    finally:
        sys.path.remove(str(REF))
    rscene, rcfg, _ = rcli.load_config(path)
    scene, cfg, _ = cli.load_config(path)
    _same_scene(scene, rscene)
    assert rcfg.coarse_block == cfg.coarse_block


def test_config_generators_sizes():
    m = scenes.sphere_mesh()
    assert (m.n_vertices, len(m.tets)) == (8625, 43248)
    p = scenes.puffer_mesh()
    assert (p.n_vertices, len(p.tets)) == (142848, 342960)  # x8: 1.143M V / 2.744M T


@pytest.mark.gpu
def test_simulate_and_check(tmp_path):
    ini = tmp_path / "drop.ini"
    ini.write_text((DATA / "drop_like.ini").read_text().replace("output_dir = out_drop", f"output_dir = {tmp_path}/o"))
    assert cli.main(["simulate", str(ini)]) == cli.EXIT_OK
    out = tmp_path / "o"
    rows = (out / "frames.csv").read_text().splitlines()
    assert rows[0] == cli.FRAME_COLUMNS and len(rows) == 4
    assert (out / "iters.csv").read_text().splitlines()[0] == cli.ITER_COLUMNS
    assert len(list(out.glob("frame_*.obj"))) == 4
    assert cli.main(["check", str(out)]) == cli.EXIT_OK


@pytest.mark.gpu
def test_checker_min_distance_matches_brute_force():
    from oracle import geometry as ogeo

    s = scenes.c1_cube(3)
    x = s.mesh.rest_positions.copy()
    tris = s.surface.triangles
    rng = np.random.default_rng(4)
    x[~s.dirichlet] += 1e-3 * rng.standard_normal(((~s.dirichlet).sum(), 3))
    x[~s.dirichlet, 2] -= 0.0095
    chk = cli.SurfaceChecker(x, tris)
    d = chk.min_distance(x)
    # brute force over every non-adjacent PT and EE pair (cli.py:359-389)
    verts = np.unique(tris)
    vi, ti = np.meshgrid(verts, np.arange(len(tris)), indexing="ij")
    vi, ti = vi.ravel(), ti.ravel()
    keep = ~np.any(tris[ti] == vi[:, None], axis=1)
    dpt, _ = ogeo.pt_distance_batch(x[vi[keep]], x[tris[ti[keep], 0]], x[tris[ti[keep], 1]], x[tris[ti[keep], 2]])
    e = np.unique(np.sort(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [0, 2]]]), axis=1), axis=0)
    i, j = np.triu_indices(len(e), k=1)
    a, b = e[i], e[j]
    keep = (a[:, 0] != b[:, 0]) & (a[:, 0] != b[:, 1]) & (a[:, 1] != b[:, 0]) & (a[:, 1] != b[:, 1])
    dee, _ = ogeo.ee_distance_batch(x[a[keep, 0]], x[a[keep, 1]], x[b[keep, 0]], x[b[keep, 1]])
    assert d == min(dpt.min(), dee.min())
    # this jitter pushes some cube vertices below the floor: triangles cross
    # while every PT / EE distance stays positive -- the tri-tri half's job
    assert chk.intersections(x)[0] == ogeo.count_tri_intersections(x, tris, 1e-9) > 0
    assert _native_check(x, tris, 0.0) == ogeo.count_tri_intersections(x, tris, 0.0)  # the reference's exact rule
    x2 = s.mesh.rest_positions.copy()
    x2[~s.dirichlet, 2] -= 0.005
    assert chk.intersections(x2)[0] == ogeo.count_tri_intersections(x2, tris, 1e-9) == 0


@pytest.mark.gpu
def test_checker_finds_planted_intersection():
    # two unit-ish triangles crossing through each other, plus a far one
    x = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0],
                  [0.2, 0.2, -0.5], [0.3, 0.2, 0.5], [0.2, 0.3, 0.5],
                  [5, 5, 5], [6, 5, 5], [5, 6, 5]], float)
    t = np.array([[0, 1, 2], [3, 4, 5], [6, 7, 8]])
    n, first = geometry_check(x, t)
    assert n == 1 and first == 0
    x[3:6, 2] += 2.0  # lift it clear
    assert geometry_check(x, t)[0] == 0


def _native_check(x, t, tol):
    from paper_2604_19892_b200 import _native

    return _native.check_intersections(x, t, coplanar_tol=tol)[0]


@pytest.mark.gpu
def test_checker_coplanar_rounding_is_not_an_intersection():
    """Two disjoint faces, coplanar to the last bits (a translated voxel
    surface): the reference's exact rule calls them intersecting, the
    checker's tolerance does not (the C5 case in DESIGN.md 4)."""
    from oracle import geometry as ogeo

    # the two triangles of the C5 run (gpurun_out c5_fail.npz), full precision
    x = np.array([[-0.1110214316702486, -0.051582198351108624, -0.18589964146451887],
                  [-0.10945893167024857, -0.051582198351108485, -0.1843371414645189],
                  [-0.11102143167024857, -0.05158219835110849, -0.18433714146451888],
                  [-0.1094589316702486, -0.05158219835110862, -0.1858996414645189],
                  [-0.10789643167024861, -0.0515821983511086, -0.18589964146451893],
                  [-0.10789643167024858, -0.05158219835110848, -0.18433714146451893]])
    t = np.array([[0, 1, 2], [3, 4, 5]])
    assert ogeo.count_tri_intersections(x, t, 0.0) == 1  # the reference's rule: a false positive
    assert ogeo.count_tri_intersections(x, t, 1e-9) == 0 == _native_check(x, t, 1e-9)


def geometry_check(x, t):
    from paper_2604_19892_b200 import _native

    return _native.check_intersections(x, t)
