"""The partitioned multi-GPU solver (mp_create_multi, csrc/group.cuh) against
the single-GPU one: same bits.  Shards may share a device, so a world of 2
or 3 shards runs on the one B200 of the test box exactly as on 2-3 GPUs
(the exchanges are peer copies ordered by cross-device events; on one
device they are device-to-device copies).

Owner-computes splits the level-0 MAS build / apply, Woodbury, gradient and
HVP by Morton aggregate range; every PNCG scalar is a sum of per-chunk
partials in chunk order, so the discrete outputs (iteration counts, restart
flags, CCD certificates) AND every float (positions, velocities, z norms)
must be bitwise identical to the single-GPU run."""

import numpy as np
import pytest

from conftest import golden_config, load_golden, scene_from_golden

pytestmark = pytest.mark.gpu


def _same(a, b):
    xa, va, ra, ca, fa = a
    xb, vb, rb, cb, fb = b
    assert ca == cb and fa == fb and len(ra) == len(rb)
    for p, q in zip(ra, rb):
        assert (p.restart, p.z_norm, p.grad_norm, p.mu, p.nu, p.min_alpha, p.ccd_certified) == \
               (q.restart, q.z_norm, q.grad_norm, q.mu, q.nu, q.min_alpha, q.ccd_certified)
    assert np.array_equal(xa, xb) and np.array_equal(va, vb)


@pytest.mark.parametrize("name,frames", [("drop", 3), ("stacked_k8", 2), ("stacked_k256", 1), ("locking", 3)])
@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_group_equals_single_gpu(name, frames, devices):
    g = load_golden(name)
    scene = scene_from_golden(g)
    cfg = golden_config(g)
    one = scene.context(cfg)
    grp = scene.context(cfg, devices=devices)
    assert grp.shards == len(devices) and one.shards == 1
    x = g["rest"].ravel().copy()
    v = g["v0"].ravel().copy()
    h = float(g["h"])
    for _ in range(frames):
        a = one.step(x, v, h)
        b = grp.step(x, v, h)
        _same(a, b)
        x, v = a[0], a[1]


def test_group_equals_single_gpu_c2_bench_prefix():
    """Config 2 at bench scale (46,664 V; 365 level-1 aggregates split over
    the shards), the first 60 iterations of the bench's first timed frame."""
    import bench
    from paper_2604_19892_b200 import scenes, solver

    st = np.load("tests/golden/c2_bench.npz")
    scene = scenes.c2_stack(gap=bench.GAP)
    cfg = solver.SolverConfig(iter_max=60)
    one = scene.context(cfg)
    grp = scene.context(cfg, devices=[0, 0])
    _same(one.step(st["x0"], st["v0"], bench.H), grp.step(st["x0"], st["v0"], bench.H))


def test_group_device_resident_state():
    g = load_golden("stacked_k8")
    scene = scene_from_golden(g)
    cfg = golden_config(g)
    one = scene.context(cfg)
    grp = scene.context(cfg, devices=[0, 0])
    x = g["rest"].ravel().copy()
    v = g["v0"].ravel().copy()
    for c in (one, grp):
        c.set_state(x, v)
        c.step_device(float(g["h"]))
    xa, va = one.get_state()
    xb, vb = grp.get_state()
    assert np.array_equal(xa, xb) and np.array_equal(va, vb)
    with pytest.raises(Exception):
        grp.gradient(x, x, float(g["h"]))  # stage taps need a single-GPU context
