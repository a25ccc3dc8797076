"""GPU probe: where CCD time goes over the bench's frames (top iterations by
CCD wall time with their candidate counts)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 6
scene = scenes.c2_stack(gap=5e-3)
cfg = solver.SolverConfig(iter_max=500)
ctx = scene.context(cfg)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, np.zeros_like(x0))
rows = []
for f in range(frames):
    recs, conv, _ = ctx.step_device(0.01)
    for r in recs:
        rows.append((r.t_ccd_ms, r.n_ccd_pairs, f, r.k, r.min_alpha, r.restart, r.t_grad_ms, r.t_dir_ms))
    print(f"frame {f}: {len(recs)} iters, ccd {sum(r.t_ccd_ms for r in recs):.1f} ms, "
          f"grad+precond {sum(r.t_grad_ms for r in recs):.1f} ms", flush=True)
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"total ccd {tot:.1f} ms over {len(rows)} iterations")
for r in rows[:15]:
    print(f"  t_ccd={r[0]:9.2f} ms Q={r[1]:>11d} frame={r[2]} k={r[3]} alpha={r[4]:.3e} restart={r[5]}")
q = np.array([r[1] for r in rows], float)
t = np.array([r[0] for r in rows])
for lo, hi in ((0, 3e5), (3e5, 1e6), (1e6, 1e7), (1e7, 1e8), (1e8, 1e12)):
    s = (q >= lo) & (q < hi)
    if s.any():
        print(f"  Q in [{lo:.0e},{hi:.0e}): {s.sum():5d} iters, {t[s].sum():9.1f} ms, {t[s].mean():7.2f} ms/iter, "
              f"{1e6 * t[s].sum() / max(q[s].sum(), 1):.2f} ns/pair")
