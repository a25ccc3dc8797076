"""The CPU oracle on the first ITERS PNCG iterations of bench frame 6 (the
committed start state): per-iteration records for the GPU comparison
(tests/golden/c2_oracle_prefix.npz)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from threadpoolctl import threadpool_limits  # noqa: E402

import bench  # noqa: E402
from oracle import solver as osol  # noqa: E402
from paper_2604_19892_b200 import scenes  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
scene = osol.Scene.from_scene(scenes.c2_stack(gap=bench.GAP))
cfg = osol.SolverConfig(iter_max=iters)
x, v = bench.start_state()
t0 = time.time()
with threadpool_limits(limits=1):
    _, _, tr = osol.step(scene, x, v, bench.H, cfg)
recs = np.array([[r.k, r.grad_norm, r.z_norm, r.r, float(r.restart), r.mu, r.nu, r.min_alpha, float(r.certified)]
                 for r in tr.records])
np.savez_compressed("tests/golden/c2_oracle_prefix.npz", records=recs, seconds=time.time() - t0, iter_max=iters)
print(f"{len(recs)} iterations, {int(recs[:, 4].sum())} restarts, {time.time() - t0:.0f} s")
