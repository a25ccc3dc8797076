"""Selectable implementation variants give the same bits.

- MP_OPT_BP_FUSED (6): broad-phase enumeration for the constraint set, CCD
  and certificate -- 1 one-pass unordered pair lists (default), 2 constraint-
  set pair work fused into the grid queries, 0 ordered count/scan/fill lists.
  All consumers are order-free (minima, flags, key-sorted contacts), so the
  constraint set, alpha_d, the certificate and x_new must be bit-identical.
- MP_OPT_APPLY_TMA (3): level-0 MAS apply -- 2 direct streaming loads
  (default), 1 TMA-staged, 0 cp.async-staged: the same sums in the same
  order, so z must be bit-identical.
"""

import numpy as np
import pytest

from conftest import golden_config, golden_taps, load_golden, scene_from_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["stacked_k256", "locking"])
def test_broad_phase_modes_same_bits(name):
    g = load_golden(name)
    scene = scene_from_golden(g)
    ctx = scene.context(golden_config(g))
    rng = np.random.default_rng(3)
    cases = [(t["x"], t["p"]) for t in golden_taps(g, "ccd")]
    for x, p in list(cases):
        cases.append((x, 4.0 * p + 0.5 * np.abs(p).max() * rng.standard_normal(p.shape)))
    for x, p in cases:
        out = []
        for mode in (1, 2, 0):
            ctx.set_option(6, mode)
            cs = ctx.constraint_set(x)
            ad, xn, ma, cert, n = ctx.ccd(x, p, exact_set=False)
            out.append((cs, ad, xn, ma, cert, n))
        ctx.set_option(6, 1)
        ref = out[0]
        for o in out[1:]:
            for a, b in zip(ref[0], o[0]):
                assert np.array_equal(np.asarray(a), np.asarray(b))
            assert np.array_equal(ref[1], o[1]) and np.array_equal(ref[2], o[2])
            assert ref[3] == o[3] and ref[4] == o[4] and ref[5] == o[5]


def test_apply_modes_same_bits():
    g = load_golden("stacked_k256")
    scene = scene_from_golden(g)
    ctx = scene.context(golden_config(g))
    x = g["rest"].ravel().copy()
    ctx.snapshot(x, float(g["h"]), build_mas=True)
    r = np.random.default_rng(5).standard_normal(x.size)
    zs = []
    for mode in (2, 1, 0):
        ctx.set_option(3, mode)
        zs.append(ctx.precond_apply(r))
    ctx.set_option(3, 2)
    assert np.array_equal(zs[0], zs[1]) and np.array_equal(zs[0], zs[2])


@pytest.mark.parametrize("name", ["stacked_k256", "locking"])
def test_append_overflow_rerun_same_bits(name):
    """MP_OPT_APPEND_LIMIT (8) lowers the one-pass list's counter limit so a
    small scene takes the >2^30-pairs path (list-free rerun with a 64-bit
    count): alpha_d, the global minimum (read back from the rerun), the
    certificate and x_new must equal the normal path's."""
    g = load_golden(name)
    scene = scene_from_golden(g)
    ctx = scene.context(golden_config(g))
    rng = np.random.default_rng(11)
    cases = [(t["x"], t["p"]) for t in golden_taps(g, "ccd")]
    for x, p in list(cases):
        cases.append((x, 4.0 * p + 0.5 * np.abs(p).max() * rng.standard_normal(p.shape)))
    try:
        for x, p in cases:
            ctx.set_option(8, 0)
            ref = ctx.ccd(x, p, exact_set=False)
            ctx.set_option(8, 64)
            low = ctx.ccd(x, p, exact_set=False)
            assert np.array_equal(ref[0], low[0]) and np.array_equal(ref[1], low[1])
            assert ref[2] == low[2] and ref[3] == low[3]
    finally:
        ctx.set_option(8, 0)


@pytest.mark.parametrize("name", ["stacked_k256", "locking", "cube3_capped"])
def test_gradient_fused_same_bits(name):
    """MP_OPT_GRAD_FUSED (9): the one-pass per-vertex gradient computes each
    corner force with the per-tet kernel's expression and sums them in the
    gather's order: the same values (bit-identical for SNH; the ARAP SVD
    path may contract FMAs differently: 1e-14)."""
    g = load_golden(name)
    scene = scene_from_golden(g)
    ctx = scene.context(golden_config(g))
    for t in golden_taps(g, "gradient"):
        out = []
        for mode in (1, 0):
            ctx.set_option(9, mode)
            out.append(ctx.gradient(t["x"], t["x_tilde"], float(t["h"])))
        ctx.set_option(9, 0)
        assert np.linalg.norm(out[0] - out[1]) <= 1e-14 * np.linalg.norm(out[1])


def test_apply_overlap_same_bits():
    """MP_OPT_APPLY_OVERLAP (10): level 0 on a side stream beside the coarse
    chain, then the prolongation pass -- the same sums as the fused kernel,
    with and without a Woodbury overlay."""
    g = load_golden("stacked_k256")
    scene = scene_from_golden(g)
    ctx = scene.context(golden_config(g))
    for t in golden_taps(g, "precond"):
        ctx.snapshot(t["x_base"], float(t["h"]), build_mas=True)
        wb = bool(t["has_wb"])
        if wb:
            ctx.update_at(t["x_cur"])
        zs = []
        for mode in (1, 0):
            ctx.set_option(10, mode)
            zs.append(ctx.precond_apply(t["g"], with_updates=wb))
        ctx.set_option(10, 1)
        assert np.array_equal(zs[0], zs[1])


@pytest.mark.parametrize("name", ["stacked_k256", "locking"])
def test_ccd_prefilter_and_bodies_same_results(name):
    """MP_OPT_CCD_PREFILTER (11, exact relative-motion pair prefilter),
    MP_OPT_CCD_BODIES (12, two-pass per-body enumeration) and
    MP_OPT_CCD_LOCAL (13, per-subdomain motion centres) and MP_OPT_CCD_BVH
    (14, motion-aware BVH instead of the grid): the same alpha_d, minimum,
    certificate and x_new as the plain tight enumeration, and the BVH the
    grid's pair count."""
    g = load_golden(name)
    scene = scene_from_golden(g)
    ctx = scene.context(golden_config(g))
    rng = np.random.default_rng(12)
    cases = [(t["x"], t["p"]) for t in golden_taps(g, "ccd")]
    for x, p in list(cases):
        cases.append((x, 4.0 * p + 0.5 * np.abs(p).max() * rng.standard_normal(p.shape)))
    try:
        for x, p in cases:
            out = {}
            for pre, bod, loc, bvh in ((0, 0, 0, 0), (1, 0, 0, 0), (0, 1, 0, 0), (1, 1, 0, 0), (0, 0, 1, 0),
                                       (1, 0, 1, 0), (0, 0, 0, 1), (1, 0, 0, 1), (1, 0, 1, 1)):
                ctx.set_option(11, pre)
                ctx.set_option(12, bod)
                ctx.set_option(13, loc)
                ctx.set_option(14, bvh)
                out[(pre, bod, loc, bvh)] = ctx.ccd(x, p, exact_set=False)
            ref = out[(0, 0, 0, 0)]
            for o in out.values():
                assert np.array_equal(ref[0], o[0]) and np.array_equal(ref[1], o[1])
                assert ref[2] == o[2] and ref[3] == o[3]
            assert out[(0, 0, 0, 1)][4] == out[(0, 0, 0, 0)][4]
            assert out[(1, 0, 0, 1)][4] == out[(1, 0, 0, 0)][4]
    finally:
        ctx.set_option(11, 1)
        ctx.set_option(12, 0)
        ctx.set_option(13, 0)
        ctx.set_option(14, 2)
