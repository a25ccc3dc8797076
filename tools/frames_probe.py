"""Runs a few config-2 frames (for an ncu launch list of the contact-phase
kernels): frames from rest, iter_max capped."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
scene = scenes.c2_stack(gap=5e-3)
ctx = scene.context(solver.SolverConfig(iter_max=iters))
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, np.zeros_like(x0))
for f in range(frames):
    recs, conv, _ = ctx.step_device(0.01)
    print(f"frame {f}: {len(recs)} iterations", flush=True)
