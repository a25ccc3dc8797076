"""The coarse-level dense inverse (coarse.cuh k_coarse_sweep, one persistent
kernel; reference `_spd_inverse`, mas.py:84-90 used at mas.py:167) against
numpy on the sizes the scenes produce -- one tile (n <= 32), ragged tiles,
several 8-tile work-unit chunks -- and against the cho_factor decision on
non-SPD input."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _spd(n, rng, cond=1e6):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.geomspace(1.0, cond, n)
    return (q * w) @ q.T


@pytest.mark.parametrize("n", [3, 18, 32, 33, 96, 276, 300, 1095])
def test_spd_inverse_matches_numpy(n):
    from paper_2604_19892_b200 import _native

    rng = np.random.default_rng(n)
    A = _spd(n, rng)
    A = 0.5 * (A + A.T)
    inv, bad = _native.spd_inverse(A)
    assert not bad
    ref = np.linalg.inv(A)
    ref = 0.5 * (ref + ref.T)
    # forward error of any backward-stable inverse ~ cond * eps
    assert np.abs(inv - ref).max() <= 1e-9 * np.abs(ref).max()
    assert np.array_equal(inv, inv.T)


@pytest.mark.parametrize("n", [40, 300])
def test_spd_inverse_flags_indefinite(n):
    from paper_2604_19892_b200 import _native

    rng = np.random.default_rng(7)
    A = _spd(n, rng, cond=10.0)
    A[n // 2, n // 2] = -1.0  # a negative pivot: cho_factor raises
    _, bad = _native.spd_inverse(A)
    assert bad
