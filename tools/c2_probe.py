"""GPU probe: per-stage time breakdown and contact/CCD pair counts of the
config-2 scene over a few capped frames (diagnostics, not a bench)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iter_max = int(sys.argv[2]) if len(sys.argv) > 2 else 200
scene = scenes.c2_stack()
cfg = solver.SolverConfig(iter_max=iter_max)
ctx = scene.context(cfg)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, np.zeros_like(x0))
ctx.stage_timing(True)
for f in range(frames):
    t0 = time.perf_counter()
    recs, conv, _ = ctx.step_device(0.01)
    dt = time.perf_counter() - t0
    nc = [r.n_contacts for r in recs]
    nq = [r.n_ccd_pairs for r in recs]
    print(json.dumps({"frame": f, "iters": len(recs), "conv": conv, "s": round(dt, 3),
                      "ms_per_iter": round(1e3 * dt / max(1, len(recs)), 3),
                      "restarts": int(sum(r.restart for r in recs)),
                      "contacts": [int(min(nc)), int(np.mean(nc)), int(max(nc))],
                      "ccd_pairs": [int(min(nq)), int(np.mean(nq)), int(max(nq))],
                      "min_alpha": [float(min(r.min_alpha for r in recs)), float(np.mean([r.min_alpha for r in recs]))],
                      "z_norm_last": recs[-1].z_norm}), flush=True)
st = ctx.stage_stats()
tot = sum(v[0] for v in st.values())
for k, (ms, cnt, b) in st.items():
    if cnt:
        print(f"{k:15s} {ms:10.2f} ms {cnt:6d} calls {ms / cnt * 1e3:10.1f} us/call {100 * ms / tot:5.1f}%"
              + (f"  {b / cnt / (ms / cnt * 1e-3) / 1e9:8.1f} GB/s" if b else ""))
