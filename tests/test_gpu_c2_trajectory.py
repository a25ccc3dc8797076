"""The bench's first timed frame (config 2, frame 6 from the committed start
state) against the CPU oracle's trajectory (tests/golden/c2_oracle_prefix.npz,
tools/c2_oracle_prefix.py: the reference's algorithm, first 60 PNCG
iterations).  The per-iteration records (‖z‖, ‖g‖, the CCD step, restart
flag) agree to 1e-9 until the first certify_mixed outcome that differs --
the documented rounding coin toss of the clamping pair (its
distance test holds with a ~1e-16 margin) -- after which both trajectories
are equally valid and diverge (chaotic contact frames).  Measured: identical
through iteration 5; the certificate of iteration 6 is where they part."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c2_frame_follows_oracle_until_a_certificate_coin_toss():
    import bench
    from paper_2604_19892_b200 import scenes, solver

    ref = np.load(Path(__file__).resolve().parent / "golden" / "c2_oracle_prefix.npz")["records"]
    scene = scenes.c2_stack(gap=bench.GAP)
    ctx = scene.context(solver.SolverConfig(iter_max=len(ref)))
    ctx.set_state(*bench.start_state())
    recs, _, _ = ctx.step_device(bench.H)
    matched = 0
    for r, q in zip(recs, ref):  # q: k, grad, z, r, restart, mu, nu, min_alpha, certified
        assert int(r.restart) == int(q[4])
        assert abs(r.z_norm - q[2]) <= 1e-9 * abs(q[2]) and abs(r.grad_norm - q[1]) <= 1e-9 * abs(q[1])
        assert abs(r.min_alpha - q[7]) <= 1e-9 * max(1.0, abs(q[7]))
        matched += 1
        if int(r.ccd_certified) != int(q[8]):
            break  # the coin toss: from here on the trajectories part
    assert matched >= 6, matched
