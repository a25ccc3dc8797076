"""GPU micro-benchmark of the MAS apply on the config-2 scene: level-0
kernel and whole stage: direct streaming loads vs TMA vs cp.async staging
(CUDA events).  The apply reads 54 MB: note that back-to-back calls find
part of it in the 126 MB L2."""
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
runs = [(2, 2, 1)] + [(mode, stages, ctas) for mode in (1, 0) for stages in (2, 3) for ctas in (1, 2, 3, 4)]
flush = None
try:
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
except Exception:
    pass
for mode, stages, ctas in runs:
    if True:
        if True:
            ctx.set_option(3, mode)
            ctx.set_option(4, stages)
            ctx.set_option(5, ctas)
            z = ctx.precond_apply(g)
            if ref is None:
                ref = z
            ctx.stage_timing(True)
            for _ in range(50):
                if flush is not None:
                    flush.fill_(1)
                    torch.cuda.synchronize()
                ctx.precond_apply(g)
            ms, cnt, b = ctx.stage_stats()["mas_apply_l0"]
            print(f"{['cp.async', 'TMA     ', 'direct  '][mode]} stages={stages} ctas/SM={ctas}: {1e3 * ms / cnt:7.2f} us "
                  f"{b / cnt / (ms / cnt * 1e-3) / 1e9:7.1f} GB/s  max|dz| = {np.abs(z - ref).max():.1e}", flush=True)
