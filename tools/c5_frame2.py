"""C5: frame 1 to convergence, then the first ITERS iterations of frame 2
(a fresh context capped at ITERS) -- for tracing frame 2's CCD calls.

    MP_CCD_TRACE=1 python tools/c5_frame2.py ITERS"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
scene = scenes.c5_puffer_balls()
v0 = scenes.c5_puffer_v0(scene)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx = scene.context(solver.SolverConfig(iter_max=500, coarse_block=32))
ctx.set_state(x0, v0)
t0 = time.time()
recs, conv, _ = ctx.step_device(0.005)
print(json.dumps({"frame": 1, "iters": len(recs), "converged": bool(conv), "s": round(time.time() - t0, 1)}), flush=True)
x, v = ctx.get_state()
print("=== frame 2", file=sys.stderr, flush=True)
if os.environ.get("FRAME2_BP_TRACE"):
    os.environ["MP_BP_TRACE"] = "1"  # read per call by the native layer
ctx2 = scene.context(solver.SolverConfig(iter_max=iters, coarse_block=32))
ctx2.set_state(x, v)
t0 = time.time()
recs, conv, _ = ctx2.step_device(0.005)
print(json.dumps({"frame": 2, "iters": len(recs), "s": round(time.time() - t0, 1),
                  "t_ccd_ms": [round(r.t_ccd_ms, 1) for r in recs], "pairs": [int(r.n_ccd_pairs) for r in recs]}),
      flush=True)
