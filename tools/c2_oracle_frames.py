"""The CPU oracle (oracle/, the reference's algorithm) on bench frames from
the GPU's own start states (tools/c2_dump.py): does the reference also cap
at iter_max = 500 on these frames, with the same restart pattern?

    python tools/c2_oracle_frames.py STATE.npz FRAME_INDEX OUT.npz

Writes the oracle's per-iteration records (k, grad_norm, z_norm, r, restart,
mu, nu, min_alpha, certified), converged flag and wall time.  One frame is
~15 min on one core."""

import sys
import time

import numpy as np

sys.path.insert(0, ".")
from threadpoolctl import threadpool_limits  # noqa: E402

import bench  # noqa: E402
from oracle import solver as osol  # noqa: E402
from paper_2604_19892_b200 import scenes  # noqa: E402

st = np.load(sys.argv[1])
f = int(sys.argv[2])
out = sys.argv[3]
scene = osol.Scene.from_scene(scenes.c2_stack(gap=bench.GAP))
cfg = osol.SolverConfig(iter_max=bench.ITER_MAX)
x, v = st[f"x{f}"], st[f"v{f}"]
t0 = time.time()
with threadpool_limits(limits=1):
    xn, vn, tr = osol.step(scene, x, v, bench.H, cfg)
dt = time.time() - t0
recs = np.array([[r.k, r.grad_norm, r.z_norm, r.r, float(r.restart), r.mu, r.nu, r.min_alpha, float(r.certified)]
                 for r in tr.records])
np.savez_compressed(out, records=recs, converged=tr.converged, seconds=dt, x_end=xn)
print(f"frame {f}: {len(recs)} iterations, {int(recs[:, 4].sum())} restarts, converged={tr.converged}, {dt:.0f}s")
