"""GPU check: two fresh contexts run the same config-2 frames from the same
state and must produce the same bits (iteration records and positions)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
scene = scenes.c2_stack(gap=5e-3)
cfg = solver.SolverConfig(iter_max=500)
runs = []
for rep in range(2):
    scene._contexts.clear()  # a fresh native context per run
    ctx = scene.context(cfg)
    x0 = scene.mesh.rest_positions.ravel().copy()
    ctx.set_state(x0, np.zeros_like(x0))
    recs = []
    for f in range(frames):
        r, conv, _ = ctx.step_device(0.01)
        recs.append([(q.z_norm, q.mu, q.min_alpha) for q in r])
    runs.append((recs, ctx.get_state()[0]))
same = runs[0][0] == runs[1][0] and np.array_equal(runs[0][1], runs[1][1])
print("iterations per frame:", [len(r) for r in runs[0][0]], "| identical:", same)
