"""GPU micro-benchmark of the MAS apply on the config-2 scene: level-0
kernel and whole stage, TMA vs cp.async staging (CUDA events)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

scene = scenes.c2_stack(gap=5e-3)
cfg = solver.SolverConfig()
ctx = scene.context(cfg)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.snapshot(x0, 0.01, build_mas=True)
g = np.random.default_rng(0).standard_normal(x0.size)
ref = None
for mode in (1, 0):
    for stages in (2, 3):
        for ctas in (1, 2, 3, 4):
            ctx.set_option(3, mode)
            ctx.set_option(4, stages)
            ctx.set_option(5, ctas)
            z = ctx.precond_apply(g)
            if ref is None:
                ref = z
            ctx.stage_timing(True)
            for _ in range(50):
                ctx.precond_apply(g)
            ms, cnt, b = ctx.stage_stats()["mas_apply_l0"]
            print(f"{'TMA     ' if mode else 'cp.async'} stages={stages} ctas/SM={ctas}: {1e3 * ms / cnt:7.2f} us "
                  f"{b / cnt / (ms / cnt * 1e-3) / 1e9:7.1f} GB/s  max|dz| = {np.abs(z - ref).max():.1e}", flush=True)
