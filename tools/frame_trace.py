"""One frame of config 3/4/5 from rest with stage timers, twice (cold, warm):
where do the seconds go?  MP_CCD_BVH=0/1/2 selects the CCD enumeration
(MP_OPT_CCD_BVH); MP_CCD_TRACE=1 / MP_BP_TRACE=1 print per-call phases.

    python tools/frame_trace.py c3 ITERS"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

which = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
if which == "c3":
    scene = scenes.c3_rod()
    v0, h, cfg = scenes.c3_rod_v0(scene), 0.01, solver.SolverConfig(iter_max=iters)
elif which == "c4":
    scene = scenes.c4_spheres_in_bowl()
    v0, h = np.zeros(3 * scene.mesh.n_vertices), 0.01
    cfg = solver.SolverConfig(iter_max=iters, coarse_block=32)
else:
    scene = scenes.c5_puffer_balls()
    v0, h = scenes.c5_puffer_v0(scene), 0.005
    cfg = solver.SolverConfig(iter_max=iters, coarse_block=32)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx = scene.context(cfg)
if os.environ.get("MP_CCD_BVH"):
    ctx.set_option(14, int(os.environ["MP_CCD_BVH"]))
for rep in range(2):
    ctx.set_state(x0, v0)
    ctx.stage_timing(True)
    recs, conv, _ = ctx.step_device(h)
    st = ctx.stage_stats()
    ctx.stage_timing(False)
    print(json.dumps({"rep": rep, "iters": len(recs), "stages": {k: [round(v[0], 1), v[1]] for k, v in st.items()},
                      "t_ccd_ms": [round(r.t_ccd_ms, 1) for r in recs],
                      "pairs": [int(r.n_ccd_pairs) for r in recs], "restart": [int(r.restart) for r in recs]}),
          flush=True)
