"""Bitwise reproducibility of the sm_100a path.

Every floating-point reduction on the path has a fixed order: the elastic
gradient and Hessian sum per-element terms by static gather maps, contact
terms go through a vertex -> incidence CSR built by a stable sort, the coarse
levels gather the BSR by a static map and accumulate contact terms in 128-bit
fixed point, and the coarse matvec reduces its chunks in order.  So the same
inputs give the same bits run to run -- also on the contact-heavy frames whose
trajectories are chaotic, where any order-dependent
rounding would show up within a few iterations.
"""

import numpy as np
import pytest

from conftest import golden_config, load_golden, scene_from_golden

pytestmark = pytest.mark.gpu


def _run(name, frames, iter_max):
    from paper_2604_19892_b200 import solver

    g = load_golden(name)
    cfg = golden_config(g)
    cfg.iter_max = iter_max
    scene = scene_from_golden(g)
    x, v, h = g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"])
    out = []
    for _ in range(frames):
        st, tr = solver.step(scene, x, v, h, cfg)
        out.append((st.x.copy(), [(r.z_norm, r.mu, r.nu, r.min_alpha, r.restart) for r in tr.records]))
        x, v = st.x, st.v
    return out


@pytest.mark.parametrize("name,frames,iter_max", [("stacked_k256", 1, 60), ("drop", 12, 200)])
def test_same_bits_twice(name, frames, iter_max):
    a = _run(name, frames, iter_max)
    b = _run(name, frames, iter_max)
    for f, ((xa, ra), (xb, rb)) in enumerate(zip(a, b)):
        assert ra == rb, f"frame {f}: iteration records differ"
        assert np.array_equal(xa, xb), f"frame {f}: positions differ"


def test_same_bits_on_one_context():
    """Two solves of the same frame on one context (buffers reused, grown)."""
    from paper_2604_19892_b200 import solver

    g = load_golden("stacked_k256")
    cfg = golden_config(g)
    cfg.iter_max = 60
    scene = scene_from_golden(g)
    x, v, h = g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"])
    s1, t1 = solver.step(scene, x, v, h, cfg)
    s2, t2 = solver.step(scene, x, v, h, cfg)
    assert [r.z_norm for r in t1.records] == [r.z_norm for r in t2.records]
    assert np.array_equal(s1.x, s2.x)
