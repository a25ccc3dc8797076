"""BASELINE config 1 (a soft 8^3-cell SNH cube dropped on a pinned floor,
tests/golden/c1/c1.ini in the reference's INI schema) against the
UNMODIFIED reference's own run of the same file
(tests/golden/c1/make_c1_reference.sh): per-frame PNCG iteration counts
exact and every iteration's |g| and |z| within 1e-9 relative, frames 1-3
(the reference needs ~7 s per frame there and ~1.4 h per frame once the
cube rests on the floor -- frame 4 onwards runs into iter_max)."""

import csv
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "c1"


def _rows(name):
    with open(GOLD / name) as f:
        return list(csv.DictReader(f))


@pytest.mark.gpu
def test_c1_frames_match_reference():
    from paper_2604_19892_b200 import cli, solver

    scene, cfg, run = cli.load_config(GOLD / "c1.ini")
    ref_frames = _rows("reference_frames.csv")
    ref_iters = _rows("reference_iters.csv")
    x = scene.mesh.rest_positions.ravel().copy()
    v = np.zeros_like(x)
    for fr in ref_frames:
        f = int(fr["frame"])
        state, trace = solver.step(scene, x, v, run.h, cfg)
        x, v = state.x, state.v
        assert trace.iterations == int(fr["iterations"]), (f, trace.iterations, fr["iterations"])
        assert bool(trace.converged) == bool(int(fr["converged"]))
        rows = [r for r in ref_iters if int(r["frame"]) == f]
        assert len(rows) == len(trace.records)
        for rec, r in zip(trace.records, rows):
            for ours, key in ((rec.grad_norm, "grad_norm"), (rec.z_norm, "z_norm")):
                want = float(r[key])
                assert abs(ours - want) <= 1e-9 * max(abs(want), 1e-300), (f, rec.k, key, ours, want)
            assert int(rec.restart) == int(r["restart"])
