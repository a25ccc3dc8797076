"""The driver's entry points: smoke() on the GPU, and on CPU the checker
side of smoke (the oracle on the product's drop scene)."""

import numpy as np
import pytest


@pytest.mark.gpu
def test_smoke_runs():
    import __graft_entry__ as g

    g.smoke()


def test_smoke_checker_side_on_cpu():
    from oracle import solver as osol
    from paper_2604_19892_b200 import scenes

    scene = scenes.drop()
    osc = osol.Scene.from_scene(scene)
    x = scene.mesh.rest_positions.ravel().copy()
    _, _, xt = osol.prepare_step(osc, x, np.zeros_like(x), 0.01)
    g = osol.gradient_at(osc, x, xt, 0.01)
    assert g.shape == x.shape and np.linalg.norm(g) > 0.0
