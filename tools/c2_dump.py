"""Dump the bench's (C2) device state at the start of each of the first
timed frames (after W warm-up frames, exactly bench.py's trajectory) and the
GPU's per-iteration records of those frames, for the CPU-side parity work
(tests/golden/make_c2_golden.py, tools/c2_oracle_frames.py)."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nframes = int(sys.argv[2]) if len(sys.argv) > 2 else 3
out_dir = os.environ.get("OUT", "gpurun_out")
os.makedirs(out_dir, exist_ok=True)
scene = scenes.c2_stack(gap=bench.GAP)
cfg = solver.SolverConfig(iter_max=bench.ITER_MAX)
ctx = scene.context(cfg, device=0)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, np.zeros_like(x0))
for _ in range(warm):
    ctx.step_device(bench.H)
out = {}
for f in range(nframes):
    x, v = ctx.get_state()
    out[f"x{f}"] = x
    out[f"v{f}"] = v
    recs, conv, _ = ctx.step_device(bench.H)
    out[f"recs{f}"] = np.array([[r.k, r.grad_norm, r.z_norm, r.r, r.restart, r.mu, r.nu, r.min_alpha,
                                 r.n_contacts, r.ccd_certified] for r in recs])
    out[f"conv{f}"] = np.array(conv)
    print(json.dumps({"frame": warm + f, "iters": len(recs), "restarts": int(sum(r.restart for r in recs)),
                      "converged": conv, "z_last": recs[-1].z_norm}), flush=True)
np.savez_compressed(os.path.join(out_dir, f"c2_state_w{warm}.npz"), **out)
