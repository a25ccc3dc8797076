"""GPU A/B of the constraint-set broad phase at a contact state: fused query
pass vs stored pair list (MP_OPT_BP_FUSED), wall time per call."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

scene = scenes.c2_stack(gap=5e-3)
ctx = scene.context(solver.SolverConfig())
x = np.load("tools/_data/ccd_state.npz")["x"]
for fused in (1, 2, 0, 1, 2):
    ctx.set_option(6, fused)
    for _ in range(3):
        ctx.constraint_set(x)
    t0 = time.perf_counter()
    for _ in range(20):
        r = ctx.constraint_set(x)
    dt = (time.perf_counter() - t0) / 20
    print(f"fused={fused}: {1e3 * dt:.3f} ms per constraint set ({len(r[0])} contacts)", flush=True)
