"""GPU probe: reproducible large-motion CCD on the config-2 scene.  Takes a
contact state (after frames 0-2; saved to tools/_data/ccd_state.npz on the
first run so later runs see the same x and p even though frames are
chaotic), forms the restart direction p = -mu P g and times mp_ccd on p
scaled by S (S ~ 37 reproduces the alpha ~ 0.027, Q ~ 1e9 iterations the
bench's chaotic frames hit), fused enumeration vs the stored pair list."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

EXACT = os.environ.get("EXACT", "0") == "1"
scales = [float(s) for s in sys.argv[1:]] or [1.0, 10.0, 37.0]
h = 0.01
scene = scenes.c2_stack(gap=5e-3)
cfg = solver.SolverConfig(iter_max=40)
ctx = scene.context(cfg)
path = "tools/_data/ccd_state.npz"
if os.path.exists(path):
    f = np.load(path)
    x, p0 = f["x"], f["p0"]
else:
    x0 = scene.mesh.rest_positions.ravel().copy()
    ctx.set_state(x0, np.zeros_like(x0))
    for _ in range(3):
        ctx.step_device(h)
    x, v = ctx.get_state()
    xt = x + h * v
    ctx.snapshot(x, h, build_mas=True)
    g = ctx.gradient(x, xt, h)
    z = ctx.precond_apply(g)
    hz = ctx.hvp(z)
    mu = float(z @ g) / float(z @ hz)
    p0 = -mu * z
    os.makedirs("tools/_data", exist_ok=True)
    np.savez(path, x=x, p0=p0)
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez("gpurun_out/ccd_state.npz", x=x, p0=p0)
ctx.constraint_set(x)
for S in scales:
    p = S * p0
    res = {}
    for fused in (1, 0):
        ctx.set_option(6, fused)
        best = 1e9
        for rep in range(3):
            t0 = time.perf_counter()
            ad, xn, ma, cert, q = ctx.ccd(x, p, exact_set=EXACT)
            best = min(best, time.perf_counter() - t0)
        res[fused] = (ad, xn, ma, cert, q)
        print(f"S={S:6.1f} fused={fused} Q={q:>11d} min_alpha={ma:.4e} certified={cert} "
              f"n_sub<1={(ad < 1).sum():5d} wall={1e3 * best:9.2f} ms", flush=True)
    a, b = res[1], res[0]
    same = np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2:] == b[2:]
    print(f"  fused == list: {same}", flush=True)
