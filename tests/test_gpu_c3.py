"""C3 (twisting rod) at a size the oracle finishes in seconds:
closed-loop per-iteration parity of the sm_100a solver against the CPU
oracle on the same twisting frames (same bar as the stacked-boxes frame in
test_gpu_vs_oracle.py)."""

import numpy as np
import pytest

from oracle import solver as osol

from test_gpu_vs_oracle import _ocfg, _track

pytestmark = pytest.mark.gpu


def test_c3_rod_small_tracks_oracle():
    from paper_2604_19892_b200 import scenes, solver

    scene = scenes.c3_rod(cells=(32, 2, 2), length=0.32)
    osc = osol.Scene.from_scene(scene)
    cfg = solver.SolverConfig(iter_max=60)
    x = scene.mesh.rest_positions.ravel().copy()
    v = scenes.c3_rod_v0(scene, omega=40.0)
    for f in range(3):
        st, tr = solver.step(scene, x, v, 0.01, cfg)
        ox, ov, otr = osol.step(osc, x, v, 0.01, _ocfg(cfg))
        _track(tr, otr, rtol=1e-6)
        if tr.converged and otr.converged:
            assert abs(tr.iterations - otr.iterations) <= max(1, round(0.05 * otr.iterations))
        assert np.all(np.isfinite(st.x))
        x, v = st.x, st.v
