"""Parity at BENCH scale (config 2: 46,664 V / 235,830 T, coarse orders 1095
and 276): every hot-path stage of the device against the REFERENCE's own
outputs at the state where bench.py's first timed frame starts
(tests/golden/make_c2_golden.py ran ipcsim on it; the state is the GPU's,
dumped by tools/c2_dump.py).

Bars (BASELINE north_star): contact pairs and the CCD-active subdomain set
bit-exact; gradient, preconditioned vectors, HVP, energy within 1e-9
relative (norm-wise, FP64)."""

from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err

GOLD = Path(__file__).resolve().parent / "golden"


def _load(name):
    with np.load(GOLD / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def c2():
    import bench
    from paper_2604_19892_b200 import scenes, solver

    g = _load("c2_bench.npz")
    scene = scenes.c2_stack(gap=bench.GAP)
    ctx = scene.context(solver.SolverConfig(iter_max=bench.ITER_MAX))
    return g, scene, ctx


def _sorted_pairs(verts, d, k):
    order = np.lexsort(verts.T[::-1])
    return verts[order], d[order], k[order]


@pytest.mark.gpu
def test_c2_constraint_set_bit_exact(c2):
    g, _, ctx = c2
    verts, is_pt, d, grad, k = ctx.constraint_set(g["x0"])
    assert len(d) == len(g["cs_d"])
    # both are in the reference's key order (contact.py:98-113)
    assert np.array_equal(verts, g["cs_verts"].astype(np.int64))
    assert np.array_equal(d, g["cs_d"])
    assert rel_err(k, g["cs_k"]) <= 1e-12


@pytest.mark.gpu
def test_c2_gradient_energy(c2):
    g, _, ctx = c2
    h = float(g["h"])
    assert rel_err(ctx.gradient(g["x0"], g["x_tilde"], h), g["g"]) <= 1e-9
    e = ctx.energy(g["x0"], g["x_tilde"], h)
    assert abs(e - float(g["energy"])) <= 1e-9 * abs(float(g["energy"]))


@pytest.mark.gpu
def test_c2_mas_build_apply_hvp(c2):
    """build_hierarchy (level-0 96x96 blocks, coarse 1095 / 276 through the
    persistent coarse kernel) + apply_preconditioner + HessianModel.hvp."""
    g, _, ctx = c2
    ctx.snapshot(g["x0"], float(g["h"]), build_mas=True)
    z = ctx.precond_apply(g["g"])
    assert rel_err(z, g["z"]) <= 1e-9
    hv = ctx.hvp(g["z"])
    assert rel_err(hv, g["hv"]) <= 1e-9
    # the restart step's scalars (solver.py:362-379)
    mu = float(z @ g["g"]) / float(z @ ctx.hvp(z))
    assert abs(mu - float(g["mu"])) <= 1e-9 * abs(float(g["mu"]))


@pytest.mark.gpu
def test_c2_ccd_restart_step(c2):
    g, _, ctx = c2
    ad, xn, ma, cert, n = ctx.ccd(g["x0"], g["p"], exact_set=True)
    assert n == int(g["ccd_pairs"])
    assert np.array_equal(ad < 1.0, g["alpha_d"] < 1.0)
    assert rel_err(ad, g["alpha_d"]) <= 1e-9
    assert cert == bool(g["ccd_certified"]) and abs(ma - float(g["ccd_min_alpha"])) <= 1e-9
    assert rel_err(xn, g["x1"]) <= 1e-12
    # the solver's tight enumeration: same alpha_d / minimum / certificate
    ad2, xn2, ma2, cert2, _ = ctx.ccd(g["x0"], g["p"], exact_set=False)
    assert np.array_equal(ad, ad2) and np.array_equal(xn, xn2) and ma == ma2 and cert == cert2


@pytest.mark.gpu
def test_c2_ccd_clamped(c2):
    """A 40x restart step: many subdomains clamp (alpha_d < 1)."""
    path = GOLD / "c2_bench_ccd.npz"
    if not path.exists():
        pytest.skip("c2_bench_ccd.npz not generated")
    g, _, ctx = c2
    r = _load("c2_bench_ccd.npz")
    p = float(r["scale"]) * g["p"]
    ad, xn, ma, cert, n = ctx.ccd(g["x0"], p, exact_set=True)
    assert n == int(r["n_pairs"])
    assert np.array_equal(ad < 1.0, r["alpha_d"] < 1.0)  # the CCD-active set, bit-exact
    assert rel_err(ad, r["alpha_d"]) <= 1e-9
    assert cert == bool(r["certified"]) and abs(ma - float(r["min_alpha"])) <= 1e-9 * max(1.0, abs(ma))
    assert rel_err(xn, r["x_new"]) <= 1e-9
    ad2, xn2, ma2, cert2, _ = ctx.ccd(g["x0"], p, exact_set=False)
    assert np.array_equal(ad, ad2) and np.array_equal(xn, xn2) and ma == ma2 and cert == cert2


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1.0, 40.0, 400.0])
def test_c2_ccd_bvh_vs_grid(c2, scale):
    """MP_OPT_CCD_BVH (14): the motion-aware BVH enumeration emits the grid's
    pair set (same count) and so the same alpha_d, minimum, certificate and
    x_new -- at bench scale, up to a 400x restart step (boxes ~ the scene)."""
    g, _, ctx = c2
    rng = np.random.default_rng(7)
    p0 = scale * g["p"]
    cases = [p0, p0 + 0.3 * np.abs(p0).max() * rng.standard_normal(p0.shape)]
    try:
        for p in cases:
            out = []
            for bvh in (0, 1):
                ctx.set_option(14, bvh)
                out.append(ctx.ccd(g["x0"], p, exact_set=False))
            a, b = out
            assert a[4] == b[4]  # reference pairs after the exact filters
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            assert a[2] == b[2] and a[3] == b[3]
    finally:
        ctx.set_option(14, 2)


@pytest.mark.gpu
def test_c2_ccd_bvh_task_overflow(c2):
    """MP_OPT_BVH_TASKS (15): with hand-on task lists far too small, threads
    finish their own traversals (fixed lists) or the queries are split into
    chunks rolled back and rerun (capped growth) -- the same pair count and
    results."""
    g, _, ctx = c2
    p = 400.0 * g["p"]
    try:
        ctx.set_option(14, 0)
        ref = ctx.ccd(g["x0"], p, exact_set=False)
        ctx.set_option(14, 1)
        for cap in (16384, -16384):  # fixed lists; grown lists capped low (query chunks)
            ctx.set_option(15, cap)
            out = ctx.ccd(g["x0"], p, exact_set=False)
            assert out[4] == ref[4]
            assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])
            assert out[2] == ref[2] and out[3] == ref[3]
    finally:
        ctx.set_option(15, 0)
        ctx.set_option(14, 2)


@pytest.mark.gpu
def test_c2_ccd_bvh_list_free(c2):
    """Past the one-pass list limit (lowered by MP_OPT_APPEND_LIMIT, 8) the
    BVH reruns list-free, working each pair where it is found, with the
    exact alpha prune (a near pass bounds alpha_d, then subtrees whose pairs
    cannot lower any bound are skipped): the same alpha_d, minimum,
    certificate and x_new; the count is the pairs worked (<= the set)."""
    g, _, ctx = c2
    p = 40.0 * g["p"]
    try:
        ctx.set_option(14, 0)
        ref = ctx.ccd(g["x0"], p, exact_set=False)
        ctx.set_option(14, 1)
        ctx.set_option(8, 4096)
        out = ctx.ccd(g["x0"], p, exact_set=False)
        assert ref[4] > 4096 and 0 < out[4] <= ref[4]
        assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])
        assert out[2] == ref[2] and out[3] == ref[3]
    finally:
        ctx.set_option(8, 0)
        ctx.set_option(14, 2)


@pytest.mark.gpu
def test_c2_update_branch(c2):
    """The non-rebuild branch at x1 against the x0 snapshot: classify_all,
    select_top_k (K=8), build_update (Sparse-Input Woodbury), then z and HVP
    with the candidates (solver.py:336-346)."""
    g, _, ctx = c2
    h = float(g["h"])
    ctx.snapshot(g["x0"], h, build_mas=True)
    nc, nt = ctx.update_at(g["x1"])
    assert nc == int(g["n_candidates"]) and nt == int(g["n_touched"])
    assert rel_err(ctx.gradient(g["x1"], g["x_tilde"], h), g["g1"]) <= 1e-9
    ctx.snapshot(g["x0"], h, build_mas=True)
    ctx.update_at(g["x1"])
    z1 = ctx.precond_apply(g["g1"], with_updates=True)
    assert rel_err(z1, g["z1"]) <= 1e-9
    assert rel_err(ctx.hvp(g["z1"], with_updates=True), g["hv1"]) <= 1e-9
