"""C5 frame 1 from rest with stage timers: where do the seconds go?"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

scene = scenes.c5_puffer_balls()
v0 = scenes.c5_puffer_v0(scene)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx = scene.context(solver.SolverConfig(iter_max=int(sys.argv[1]) if len(sys.argv) > 1 else 20, coarse_block=32))
if os.environ.get("MP_CCD_BVH"):  # 0 grid, 1 BVH, 2 per call (default)
    ctx.set_option(14, int(os.environ["MP_CCD_BVH"]))
for rep in range(2):
    ctx.set_state(x0, v0)
    ctx.stage_timing(True)
    recs, conv, _ = ctx.step_device(0.005)
    st = ctx.stage_stats()
    ctx.stage_timing(False)
    print(json.dumps({"rep": rep, "iters": len(recs), "stages": {k: [round(v[0], 1), v[1]] for k, v in st.items()},
                      "t_ccd_ms": [round(r.t_ccd_ms, 1) for r in recs], "t_grad_ms": [round(r.t_grad_ms, 1) for r in recs],
                      "pairs": [int(r.n_ccd_pairs) for r in recs], "restart": [int(r.restart) for r in recs]}), flush=True)
