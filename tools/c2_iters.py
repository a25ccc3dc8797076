"""GPU probe: per-iteration records of the config-2 scene (gap, frames and
iteration cap from argv) to see where time goes as contact develops."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

gap = float(sys.argv[1]) if len(sys.argv) > 1 else 5e-3
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
iter_max = int(sys.argv[3]) if len(sys.argv) > 3 else 20
budget = float(sys.argv[4]) if len(sys.argv) > 4 else 120.0
scene = scenes.c2_stack(gap=gap)
cfg = solver.SolverConfig(iter_max=iter_max)
ctx = scene.context(cfg)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, np.zeros_like(x0))
t_start = time.perf_counter()
for f in range(frames):
    t0 = time.perf_counter()
    recs, conv, _ = ctx.step_device(0.01)
    dt = time.perf_counter() - t0
    print(f"frame {f}: {len(recs)} iters conv={conv} {dt:.3f}s ({1e3 * dt / max(1, len(recs)):.2f} ms/iter), "
          f"restarts {sum(r.restart for r in recs)}", flush=True)
    for r in recs[:6] + recs[-3:]:
        print(f"   k={r.k:4d} z={r.z_norm:.3e} rs={r.restart} mu={r.mu:.3e} nu={r.nu:.3e} a={r.min_alpha:.3e} "
              f"C={r.n_contacts} cand={r.n_candidates} Q={r.n_ccd_pairs} t=({r.t_grad_ms:.2f},{r.t_dir_ms:.2f},"
              f"{r.t_ccd_ms:.2f})ms", flush=True)
    if time.perf_counter() - t_start > budget:
        break
