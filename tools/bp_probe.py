"""GPU probe: broad-phase / constraint-set / CCD call times on the config-2
scene at rest with synthetic directions of growing length."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

scene = scenes.c2_stack()
cfg = solver.SolverConfig()
ctx = scene.context(cfg)
x = scene.mesh.rest_positions.ravel().copy()
rng = np.random.default_rng(0)
free = np.repeat(~scene.dirichlet, 3)


def timed(name, fn, reps=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name:40s} {1e3 * dt:9.2f} ms", out if not isinstance(out, tuple) else tuple(
        len(o) if hasattr(o, '__len__') else o for o in out), flush=True)
    return out


timed("constraint_set", lambda: len(ctx.constraint_set(x)[0]))
timed("broad_phase(0, d_hat)", lambda: ctx.broad_phase(x, 0.0, scene.d_hat))
for scale in (1e-3, 3e-3, 1e-2):
    p = np.zeros_like(x)
    p[free] = scale * rng.standard_normal(free.sum()) * 0.3
    p[2::3][~scene.dirichlet] -= scale
    pinf = np.abs(p).max()
    timed(f"broad_phase(mb={pinf:.3g}, 0)", lambda: ctx.broad_phase(x, pinf, 0.0), reps=1)
    timed(f"ccd exact (|p|inf={pinf:.3g})", lambda: ctx.ccd(x, p, exact_set=True)[2:], reps=1)
    timed(f"ccd tight (|p|inf={pinf:.3g})", lambda: ctx.ccd(x, p, exact_set=False)[2:], reps=1)
    a1 = ctx.ccd(x, p, exact_set=True)
    a2 = ctx.ccd(x, p, exact_set=False)
    print("  tight == exact:", np.array_equal(a1[0], a2[0]), a1[2] == a2[2], a1[3] == a2[3], np.array_equal(a1[1], a2[1]))
