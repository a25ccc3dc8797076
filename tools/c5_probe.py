"""C5 penetration probe: step the puffer balls iteration by iteration
(iter_max = 1 frames would restart the frame, so: one frame, checking the
surface after every PNCG iteration through the record hook is not
available -- instead run frames of iter_max = k for k = 1, 2, 4, 8 from the
rest state) and run the checker after each; save the first failing state."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import cli, scenes, solver  # noqa: E402

scene = scenes.c5_puffer_balls()
v0 = scenes.c5_puffer_v0(scene)
x0 = scene.mesh.rest_positions.ravel().copy()
chk = cli.SurfaceChecker(scene.mesh.rest_positions, scene.surface.triangles)
for k in (1, 2, 3, 4, 6, 8, 10):
    ctx = scene.context(solver.SolverConfig(iter_max=k, coarse_block=32))
    ctx.set_state(x0, v0)
    recs, conv, _ = ctx.step_device(0.005)
    x, _ = ctx.get_state()
    n, first = chk.intersections(x)
    d = chk.min_distance(x)
    print(json.dumps({"iter_max": k, "iters": len(recs), "intersections": n, "min_distance": d,
                      "min_alpha": [r.min_alpha for r in recs], "cert": [int(r.ccd_certified) for r in recs],
                      "pairs": [int(r.n_ccd_pairs) for r in recs]}), flush=True)
    if n:
        np.savez_compressed("gpurun_out/c5_fail.npz", x=x, k=k, first=first)
        break
