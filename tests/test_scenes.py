"""Synthetic generators for the BASELINE.json configs:
sizes at full scale and the C3 twist field."""

import numpy as np

from paper_2604_19892_b200 import scenes


def test_c3_rod_full_size():
    s = scenes.c3_rod()
    assert s.mesh.n_vertices == 9 * 9 * 2501 + 8
    assert len(s.mesh.tets) == 6 * 8 * 8 * 2500 + 6


def test_c3_rod_twist_field():
    s = scenes.c3_rod(cells=(24, 2, 2), length=0.24)
    v = scenes.c3_rod_v0(s, omega=20.0).reshape(-1, 3)
    pin = np.asarray(s.dirichlet, dtype=bool)
    assert np.all(v[pin] == 0.0)
    assert np.all(v[~pin, 0] == 0.0)  # spin about the rod's (x) axis only
    x = s.mesh.rest_positions[~pin]
    c = 0.5 * (x.min(axis=0) + x.max(axis=0))
    r = x[:, 1:] - c[1:]
    assert np.allclose(np.einsum("ij,ij->i", v[~pin, 1:], r), 0.0, atol=1e-15)  # tangential
    ends = np.isclose(x[:, 0], x[:, 0].min()), np.isclose(x[:, 0], x[:, 0].max())
    # opposite ends spin in opposite senses
    w0 = v[~pin][ends[0], 2] / np.where(r[ends[0], 0] == 0, np.inf, r[ends[0], 0])
    w1 = v[~pin][ends[1], 2] / np.where(r[ends[1], 0] == 0, np.inf, r[ends[1], 0])
    assert np.all(w0[np.isfinite(1 / w0)] < 0) and np.all(w1[np.isfinite(1 / w1)] > 0)
