"""Pin the CPU oracle (oracle/) before trusting it as the checker.

1. Known-answer values from the reference's own unit tests
   (`pkg/tests/test_contact.py:25-31`, `test_geometry.py:75-90`,
   `test_solver.py:56-65,108-113`, `test_woodbury.py:38-49`,
   `test_ccd.py:40-44,78-91,110-116,178-180,261-273`).
2. Every stage tap of every golden fixture (outputs of the reference run in
   the build container, tests/golden/make_golden.py): broad phase and
   constraint-set pairs/distances bit-exact, CCD candidate counts and the
   CCD-active subdomain set bit-exact, FP vectors within 1e-9 relative.
3. Closed-loop frames: per-frame iteration counts within +-5% of the
   reference's, convergence flags equal.
"""

import math

import numpy as np
import pytest

from conftest import golden_taps, load_golden, rel_err

from oracle import ccd as occd
from oracle import geometry as ogeo
from oracle import physics as oph
from oracle import precond as opre
from oracle import solver as osol

TOL = 1e-9
STAGE_SCENES = ("drop", "locking", "stacked_k8", "stacked_k256", "cube3_capped")


def _cfg(g):
    eps, delta, iter_max, K, bs, levels, cb, per_sub = g["cfg"]
    return osol.SolverConfig(eps=float(eps), delta=float(delta), iter_max=int(iter_max), K=int(K),
                             block_size=int(bs), levels=int(levels), coarse_block=int(cb),
                             ccd_per_subdomain=bool(per_sub), update_strategy=str(g["cfg_strategy"]))


# ---------------------------------------------------------------------------
# 1. known answers of the reference's unit tests


def test_barrier_known_values():
    b, b1, b2 = oph.barrier(np.array([0.5]), 1.0, 1.0)
    assert b[0] == pytest.approx(0.17328679513998632, abs=1e-12)
    assert b1[0] == pytest.approx(-1.1931471805599454, abs=1e-12)
    assert b2[0] == pytest.approx(6.386294361119891, abs=1e-12)
    assert oph.barrier_hess_scalar(0.5, 1.0, 1.0) == pytest.approx(6.386294361119891, abs=1e-12)
    assert [v[0] for v in oph.barrier(np.array([1.0]), 1.0, 10.0)] == [0.0, 0.0, 0.0]
    with pytest.raises(oph.PenetrationError):
        oph.barrier(np.array([0.0]), 1.0, 1.0)


def test_pt_distance_known_values():
    t0, t1, t2 = np.zeros((1, 3)), np.array([[1.0, 0, 0]]), np.array([[0.0, 1, 0]])
    d, _ = ogeo.pt_distance_batch(np.array([[2.0, 2.0, 0.0]]), t0, t1, t2)
    assert d[0] == pytest.approx(2.1213203435596424, abs=1e-12)
    d, _ = ogeo.pt_distance_batch(np.array([[-1.0, -1.0, 0.0]]), t0, t1, t2)
    assert d[0] == pytest.approx(math.sqrt(2.0), abs=1e-12)
    d, g = ogeo.pt_distance_batch(np.array([[0.0, 0.0, 1.0]]), t0, t1, t2)
    assert d[0] == pytest.approx(1.0, abs=1e-14)
    assert np.allclose(g[0, 0], [0, 0, 1]) and np.allclose(g[0, 1], [0, 0, -1])


def test_ee_distance_crossing_segments():
    d, g = ogeo.ee_distance_batch(np.array([[-1.0, 0, 0]]), np.array([[1.0, 0, 0]]), np.array([[0.0, -1, 1]]),
                                  np.array([[0.0, 1, 1]]))
    assert d[0] == pytest.approx(1.0)
    assert np.allclose(g[0].sum(axis=0), 0.0)


def test_subspace_and_restart_known_values():
    mu, nu = osol.solve_2d(1.0, 0.0, 0.0, 4.0, 2.0, 3.0)
    assert abs(mu - 2.0) <= 1e-14 and abs(nu + 0.75) <= 1e-14
    g, zp, z = np.array([1.0, 2.0]), np.array([3.0, -1.0]), np.array([2.0, 1.0])
    assert abs(abs(g @ zp) / (g @ z) - 0.25) <= 1e-15
    with pytest.raises(oph.NotSpdError):
        osol.solve_2d(-1.0, 0.0, 0.0, 1.0, 1.0, 1.0)


def test_woodbury_two_by_two():
    import scipy.linalg

    blk = opre.WoodburyBlock(U=np.array([[1.0], [0.0]]), W=np.array([[1.0], [0.0]]),
                             cap_chol=scipy.linalg.cho_factor(np.array([[2.0]])))
    z = opre.woodbury_apply(np.eye(2), blk, np.array([1.0, 1.0]))
    assert np.allclose(z, [0.5, 1.0], atol=1e-15)


def _floor_drop():
    x = np.array([[0.3, 0.3, 1.0], [0, 0, 0], [1.0, 0, 0], [0, 1.0, 0]])
    p = np.zeros((4, 3))
    p[0, 2] = -2.0
    return np.array([[0, 1, 2, 3]]), x.ravel(), p.ravel()


def test_ccd_known_values():
    verts, x, p = _floor_drop()
    co = occd.cubic_coeffs(verts, x, p)[0]
    assert co[0] == 0.0 and co[1] == 0.0 and co[2] != 0.0
    assert -co[3] / co[2] == pytest.approx(0.5, abs=1e-12)
    # relative-displacement lower bound 0.45 (test_ccd.py:178-180)
    d = occd.distances(verts, np.array([True]), x)
    sp = occd.rel_speed(verts, np.array([True]), p)
    assert min(1.0, 0.9 * d[0] / sp[0]) == pytest.approx(0.45, abs=1e-12)
    # bisection walkthrough f = 1 - 2a -> 0.25 in 3 evaluations
    a, ev, fl = occd.bisect(np.array([[0.0, 0.0, -2.0, 1.0]]), np.array([1.0]), 2.0 ** -20)
    assert a[0] == 0.25 and ev == 3 and not fl[0]
    # windows (test_ccd.py:78-91)
    w = occd.window(np.array([[1.0, -3.0, 0.0, 0.0], [-1.0, 0.0, 1.0, 5.0], [0.0, -1.0, 0.0, 1.0],
                              [0.0, 0.0, -2.0, 1.0]]))
    assert w[0] == pytest.approx(1.0)
    assert w[1] == pytest.approx(1.0 / math.sqrt(3.0))
    assert w[2] == np.inf and w[3] == np.inf


def test_per_subdomain_min_rule():
    verts, x, p = _floor_drop()
    x = np.r_[x, [50.0, 0, 0, 51.0, 0, 0]]
    p = np.r_[p, np.zeros(6)]
    ap = occd.pair_steps(verts, np.array([True]), x, p, 2.0 ** -20)
    sub = np.array([1, 2, 2, 2, 0, 0])
    alpha_d = np.ones(3)
    np.minimum.at(alpha_d, sub[verts].ravel(), np.repeat(ap, 4))
    assert ap[0] < 1.0 and alpha_d[1] == ap[0] and alpha_d[2] == ap[0] and alpha_d[0] == 1.0


def test_mas_identity_gives_one_plus_levels():
    """mas.py: H = I, levels built L -> z = (1 + L) g (test_mas.py:124-133)."""
    import scipy.sparse as sp

    rng = np.random.default_rng(1)
    rest = rng.random((64, 3))
    part = opre.partition_domain(rest, 4)
    hier = opre.build_hierarchy(sp.identity(192, format="csr"), part, levels=2, coarse_block=4)
    g = rng.standard_normal(192)
    z = opre.apply_preconditioner(hier, None, g)
    L = len(hier.coarsen)
    assert L == 2
    # coarse corrections C^T (C C^T)^-1 C g: projections onto aggregate means
    proj = sum(C.T @ np.linalg.solve((C @ C.T).toarray(), C @ g) for C in hier.coarsen)
    assert np.allclose(z, g + proj, atol=1e-12)


def test_partition_blocks_and_morton_order():
    rng = np.random.default_rng(3)
    pts = rng.random((53, 3))
    part = opre.partition_domain(pts, 8)
    assert part.D == 7
    assert sorted(np.bincount(part.subdomain_of)) == [5] + [8] * 6
    from paper_2604_19892_b200 import _native

    try:
        lib_sub = _native.partition_host(pts, 8)
    except ImportError:
        pytest.skip("native library not built")
    assert np.array_equal(lib_sub, part.subdomain_of)


# ---------------------------------------------------------------------------
# 2. stage taps of the reference run


@pytest.fixture(scope="module", params=STAGE_SCENES)
def golden(request):
    g = load_golden(request.param)
    return request.param, g, osol.Scene.from_golden(g), _cfg(g)


def test_broad_phase_bit_exact(golden):
    _, g, sc, _ = golden
    for t in golden_taps(g, "broad_phase"):
        pt, ee = ogeo.broad_phase(t["x"].reshape(-1, 3), sc.tris, sc.edges, sc.surf_verts, float(t["mb"]),
                                  float(t["d_hat"]))
        assert np.array_equal(pt, t["pt"].reshape(-1, 2))
        assert np.array_equal(ee, t["ee"].reshape(-1, 2))


@pytest.mark.parametrize("name", ["bp_cube8"])
def test_broad_phase_fixture_bit_exact(name):
    g = load_golden(name)
    sc = osol.Scene.from_golden(g)
    for t in golden_taps(g, "broad_phase"):
        pt, ee = ogeo.broad_phase(t["x"].reshape(-1, 3), sc.tris, sc.edges, sc.surf_verts, float(t["mb"]),
                                  float(t["d_hat"]))
        assert np.array_equal(pt, t["pt"].reshape(-1, 2))
        assert np.array_equal(ee, t["ee"].reshape(-1, 2))


def test_constraint_set_exact(golden):
    _, g, sc, _ = golden
    for t in golden_taps(g, "constraint_set"):
        cs = oph.constraint_set(sc, t["x"])
        assert np.array_equal(cs.verts, t["verts"].reshape(-1, 4))
        assert np.array_equal(cs.d, t["d"])
        assert rel_err(cs.grad, t["grad"]) <= 1e-14
        assert rel_err(cs.k, t["k"]) <= 1e-12


def test_gradient_and_energy(golden):
    _, g, sc, _ = golden
    for t in golden_taps(g, "gradient"):
        gr = osol.gradient_at(sc, t["x"], t["x_tilde"], float(t["h"]))
        assert rel_err(gr, t["g"]) <= TOL
        cs = oph.constraint_set(sc, t["x"])
        e = oph.incremental_potential(sc, t["x"], t["x_tilde"], float(t["h"]), cs)
        assert abs(e - float(t["energy"])) <= TOL * max(1.0, abs(float(t["energy"])))


def _snapshot(sc, cfg, t):
    base = oph.constraint_set(sc, t["x_base"])
    H = oph.assemble_base_hessian(sc, t["x_base"], float(t["h"]), base)
    hier = opre.build_hierarchy(H, sc.partition(cfg.block_size), cfg.levels, cfg.coarse_block)
    return base, H, hier


def test_hvp(golden):
    _, g, sc, cfg = golden
    for t in golden_taps(g, "hvp"):
        base, H, _ = _snapshot(sc, cfg, t)
        if bool(t["with_updates"]):
            c = opre.classify_all(oph.constraint_set(sc, t["x_cur"]), base, cfg.eps_rot)
            out = oph.hvp(H, c.verts, c.u, t["vec"])
        else:
            out = oph.hvp(H, np.zeros((0, 4), np.int64), np.zeros((0, 4, 3)), t["vec"])
        assert rel_err(out, t["out"]) <= TOL


def test_preconditioner(golden):
    _, g, sc, cfg = golden
    part = sc.partition(cfg.block_size)
    for t in golden_taps(g, "precond"):
        base, H, hier = _snapshot(sc, cfg, t)
        wb = None
        if bool(t["has_wb"]):
            c = opre.classify_all(oph.constraint_set(sc, t["x_cur"]), base, cfg.eps_rot)
            wb = opre.build_update(hier, c, opre.select_top_k(c, part.subdomain_of, cfg.K), cfg.K)
            assert len(wb) == int(t["n_touched"])
        assert rel_err(opre.apply_preconditioner(hier, wb, t["g"]), t["z"]) <= TOL


def test_ccd(golden):
    _, g, sc, cfg = golden
    part = sc.partition(cfg.block_size)
    for t in golden_taps(g, "ccd"):
        xn, ma, ad, cert, npairs = occd.clamp(sc, part, t["x"], t["p"], cfg.ccd_per_subdomain, cfg.alpha_l)
        assert npairs == int(t["n_pairs"])
        assert np.array_equal(ad < 1.0, t["alpha_d"] < 1.0)
        assert np.allclose(ad, t["alpha_d"], rtol=TOL, atol=1e-15)
        assert cert == bool(t["certified"])
        assert abs(ma - float(t["min_alpha"])) <= TOL
        assert rel_err(xn, t["x_new"]) <= TOL


# ---------------------------------------------------------------------------
# 3. closed-loop frames


@pytest.mark.parametrize("name", ["drop", "stacked_k256", "stacked_k8", "cube3_capped"])
def test_frames_iteration_counts(name):
    g = load_golden(name)
    sc, cfg = osol.Scene.from_golden(g), _cfg(g)
    x, v, h = g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"])
    for f in range(int(g["frames"])):
        x, v, tr = osol.step(sc, x, v, h, cfg)
        ref = int(g["iterations"][f])
        assert abs(tr.iterations - ref) <= max(1, round(0.05 * ref)), (f, tr.iterations, ref)
        assert tr.converged == bool(g["converged"][f])
        oph.constraint_set(sc, x)  # raises on penetration


def test_from_scene_matches_golden_arrays():
    from paper_2604_19892_b200 import scenes

    g = load_golden("drop")
    a, b = osol.Scene.from_scene(scenes.drop()), osol.Scene.from_golden(g)
    for k in ("rest", "tets", "Bm", "vol", "mass", "f_ext", "tris", "edges", "surf_verts"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k



def test_oracle_tri_tri_cases():
    """The checker oracle's tri-tri test (geometry.py:686-732 rules)."""
    from oracle.geometry import tri_tri_intersect

    a = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    assert tri_tri_intersect(a, [[0.2, 0.2, -0.5], [0.3, 0.2, 0.5], [0.2, 0.3, 0.5]])  # crossing
    assert not tri_tri_intersect(a, [[0.2, 0.2, 0.1], [0.3, 0.2, 0.5], [0.2, 0.3, 0.5]])  # above
    assert tri_tri_intersect(a, [[1, 0, 0], [2, 0, 1], [2, 0, -1]])  # touching at a vertex counts
    assert tri_tri_intersect(a, [[0.1, 0.1, 0], [0.5, 0.1, 0], [0.1, 0.5, 0]])  # coplanar, inside
    assert not tri_tri_intersect(a, [[2, 2, 0], [3, 2, 0], [2, 3, 0]])  # coplanar, apart
