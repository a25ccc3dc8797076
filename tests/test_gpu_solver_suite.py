"""The reference's solver-level test scenarios (`pkg/tests/test_solver.py:
263-431`), restated against the device backend through the drop-in API
(the reference package cannot travel to the GPU box; the scene builders and
every assertion are the reference tests' own): exact inertia-only steps,
drop-onto-box convergence and separation, update strategies / Jacobi /
FR-PR-DK-CD reaching the same minimum, the iter_max best-iterate flag, the
global CCD scope, step == prepare + advance, and multi-step settling."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2604_19892_b200 import energy as en
from paper_2604_19892_b200 import geometry as geo
from paper_2604_19892_b200 import solver
from paper_2604_19892_b200.errors import PenetrationError

pytestmark = pytest.mark.gpu


def _points_scene(points, masses, pinned=None, h=0.1):
    pts = np.asarray(points, dtype=float).reshape(-1, 3)
    n = len(pts)
    mesh = SimpleNamespace(rest_positions=pts.copy(), n_vertices=n)
    surface = geo.SurfaceMesh(triangles=np.zeros((0, 3), np.int64), edges=np.zeros((0, 2), np.int64),
                              vertices=np.zeros(0, np.int64))
    dirichlet = np.zeros(n, dtype=bool) if pinned is None else np.asarray(pinned, bool)
    mass = np.asarray(masses, dtype=float)
    f_ext = (mass[:, None] * np.array([0.0, 0.0, -9.81])).ravel()
    scene = solver.Scene(mesh=mesh, surface=surface, elastic=None, mass=mass, dirichlet=dirichlet, d_hat=0.01,
                         kappa=1.0, f_ext=f_ext)
    return scene, en.prepare_step(pts.ravel(), np.zeros(3 * n), mass, h, f_ext, dirichlet)


def _drop_scene(gap=0.05, h=0.02, young=200.0, kappa=50.0, d_hat=0.1):
    m = geo.make_box_mesh(1, 1, 1)
    n = m.n_vertices
    verts = np.vstack([m.rest_positions, m.rest_positions + np.array([0.0, 0.0, 1.0 + gap])])
    dirichlet = np.zeros(2 * n, dtype=bool)
    dirichlet[:n] = True
    mesh = geo.TetMesh(rest_positions=verts, tets=np.vstack([m.tets, m.tets + n]), dirichlet=dirichlet)
    scene = solver.Scene.build(mesh, en.ElasticModel.from_mesh(mesh, "arap", young, 0.3), density=1.0, d_hat=d_hat,
                               kappa=kappa)
    x0 = verts.ravel()
    return scene, en.prepare_step(x0, np.zeros_like(x0), scene.mass, h, scene.f_ext, dirichlet)


def _separated(scene, x):
    try:
        scene.context(solver.SolverConfig()).constraint_set(x)
    except PenetrationError:
        return False
    return True


@pytest.fixture
def rng():
    return np.random.default_rng(20260823)


def test_single_vertex_gravity_lands_inertia_target():
    scene, state = _points_scene([[0.0, 0.0, 1.0]], [2.0], h=0.1)
    new, tr = solver.advance_step(scene, state, solver.SolverConfig(eps=1e-10))
    assert tr.converged and tr.records[0].restart and abs(tr.records[0].mu - 1.0) <= 1e-12
    assert np.allclose(new.x, state.x_tilde, atol=1e-14) and tr.iterations <= 3
    assert np.allclose(new.v, (new.x - np.array([0.0, 0.0, 1.0])) / state.h)


def test_multi_point_inertia_single_subdomain_is_exact(rng):
    pts = rng.standard_normal((20, 3))
    scene, state = _points_scene(pts, rng.uniform(0.5, 2.0, 20), h=0.05)
    new, tr = solver.advance_step(scene, state, solver.SolverConfig(eps=1e-12, block_size=32))
    assert tr.converged and tr.iterations <= 3
    assert np.allclose(new.x, state.x_tilde, atol=1e-12)


def test_multi_subdomain_converges_on_quadratic(rng):
    pts = rng.standard_normal((16, 3))
    pinned = np.zeros(16, dtype=bool)
    pinned[[3, 7]] = True
    scene, state = _points_scene(pts, np.ones(16), pinned=pinned, h=0.05)
    new, tr = solver.advance_step(scene, state, solver.SolverConfig(eps=1e-10, block_size=4, levels=2,
                                                                      coarse_block=2))
    assert tr.converged
    free3 = ~np.repeat(pinned, 3)
    assert np.allclose(new.x[free3], state.x_tilde[free3], atol=1e-8)
    assert np.array_equal(new.x[~free3], pts.ravel()[~free3])


def test_velocity_update_and_pinned_velocity_zero(rng):
    pts = rng.standard_normal((6, 3))
    pinned = np.zeros(6, dtype=bool)
    pinned[0] = True
    scene, state = _points_scene(pts, np.ones(6), pinned=pinned, h=0.25)
    x0 = state.x.copy()
    new, _ = solver.advance_step(scene, state, solver.SolverConfig())
    assert np.allclose(new.v, (new.x - x0) / 0.25) and np.all(new.v[np.repeat(pinned, 3)] == 0.0)


def test_drop_step_converges_and_stays_separated():
    scene, state = _drop_scene()
    new, tr = solver.advance_step(scene, state, solver.SolverConfig())
    assert tr.converged and tr.records[0].restart and _separated(scene, new.x)
    pin3 = np.repeat(scene.dirichlet, 3)
    assert np.array_equal(new.x[pin3], state.x[pin3])
    for rec in tr.records:
        assert 0.0 < rec.min_alpha <= 1.0
        assert rec.t_grad_ms >= 0.0 and rec.t_dir_ms >= 0.0 and rec.t_ccd_ms >= 0.0


def test_drop_energy_decreases_over_step():
    scene, state = _drop_scene()
    e0 = solver.total_energy(scene, state, state.x)
    new, tr = solver.advance_step(scene, state, solver.SolverConfig())
    assert tr.converged and solver.total_energy(scene, state, new.x) < e0


def test_update_strategies_reach_same_minimum():
    res = {}
    for strategy in ("Woodbury", "Freeze", "FullRebuild"):
        scene, state = _drop_scene()
        new, tr = solver.advance_step(scene, state, solver.SolverConfig(update_strategy=strategy, eps=1e-7))
        assert tr.converged, strategy
        res[strategy] = new.x
    for strategy, x in res.items():
        assert np.linalg.norm(x - res["FullRebuild"], np.inf) <= 1e-4, strategy


def test_jacobi_reaches_same_minimum_as_mas():
    scene, state = _drop_scene()
    ref, tm = solver.advance_step(scene, state, solver.SolverConfig(eps=1e-7))
    scene2, state2 = _drop_scene()
    new, tj = solver.advance_step(scene2, state2, solver.SolverConfig(preconditioner="Jacobi", eps=1e-7))
    assert tm.converged and tj.converged and np.linalg.norm(new.x - ref.x, np.inf) <= 1e-4


@pytest.mark.parametrize("rule", ["FR", "PR", "DK", "CD"])
def test_baseline_rules_converge_to_same_minimum(rule):
    scene, state = _drop_scene()
    ref, _ = solver.advance_step(scene, state, solver.SolverConfig(eps=1e-7))
    scene2, state2 = _drop_scene()
    new, tr = solver.advance_step(scene2, state2, solver.SolverConfig(direction_rule=rule, eps=1e-6, iter_max=3000))
    assert tr.converged, rule
    assert np.linalg.norm(new.x - ref.x, np.inf) <= 5e-4, rule


def test_iter_max_returns_best_iterate_with_flag():
    scene, state = _drop_scene()
    _, tr = solver.advance_step(scene, state, solver.SolverConfig(iter_max=2))
    assert not tr.converged and "not-converged" in tr.flags and tr.iterations == 2


def test_global_ccd_scope_also_converges():
    scene, state = _drop_scene()
    new, tr = solver.advance_step(scene, state, solver.SolverConfig(ccd_per_subdomain=False))
    assert tr.converged and _separated(scene, new.x)


def test_step_wrapper_matches_manual_prepare():
    scene, state = _drop_scene(h=0.02)
    x0 = state.x.copy()
    a, _ = solver.advance_step(scene, state, solver.SolverConfig())
    scene2, _ = _drop_scene(h=0.02)
    b, _ = solver.step(scene2, x0, np.zeros_like(x0), 0.02, solver.SolverConfig())
    assert np.allclose(a.x, b.x, atol=1e-12)


def test_multiple_steps_settle_without_penetration():
    scene, state = _drop_scene(gap=0.12, h=0.02)
    x, v = state.x.copy(), np.zeros_like(state.x)
    for _ in range(6):
        new, tr = solver.step(scene, x, v, 0.02, solver.SolverConfig())
        assert tr.converged and _separated(scene, new.x)
        x, v = new.x, new.v
    upper = ~scene.dirichlet
    assert new.x.reshape(-1, 3)[upper, 2].mean() < scene.mesh.rest_positions[upper, 2].mean()
