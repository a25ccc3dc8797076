"""C3 (twisting rod, 202,589 V / 960,006 T) device-resident frames on one
B200: PNCG iterations/s per frame, CUDA events on the solver's stream, L2
flushed between frames.  Not the bench headline (bench.py measures C2);
a sizing/throughput probe for the next row of SURVEY.md 8."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iter_max = int(sys.argv[2]) if len(sys.argv) > 2 else 200
nx = int(sys.argv[3]) if len(sys.argv) > 3 else 2500
scene = scenes.c3_rod(cells=(nx, 8, 8), length=6.25 * nx / 2500)
cfg = solver.SolverConfig(iter_max=iter_max, **json.loads(os.environ.get("C3_CFG", "{}")))
ctx = scene.context(cfg, device=0)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, scenes.c3_rod_v0(scene))
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ctx.stage_timing(False)
out = []
for f in range(frames):
    flush.fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    recs, conv, _ = ctx.step_device(0.01)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out.append({"frame": f, "iters": len(recs), "ms": round(ms, 3), "iters_per_s": round(len(recs) / ms * 1e3, 1),
                "converged": bool(conv)})
print(json.dumps({"workload": f"c3_rod 8x8x{nx} cells SNH, omega=20 rad/s twist, h=0.01", "iter_max": iter_max,
                  "frames": out}))
