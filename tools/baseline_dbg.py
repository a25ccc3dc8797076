"""First iterations of the stacked MAS+PR baseline frame vs the reference golden."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

G = np.load("tests/golden/baselines.npz")
for i in (6, 7):
    scene = scenes.stacked_boxes()
    v = scenes.stacked_boxes_v0(scene)
    x = scene.mesh.rest_positions.ravel().copy()
    name, pre, rule = [str(s) for s in G[f"v{i}_meta"]]
    st, tr = solver.step(scene, x, v, 0.01, solver.SolverConfig(preconditioner=pre, direction_rule=rule, iter_max=300))
    ref = G[f"v{i}_records"]
    print(pre, rule, "ours", tr.iterations, "ref", int(G[f"v{i}_iters"][0]))
    for r, q in zip(tr.records[:6], ref[:6]):
        print(f"k={r.k} z {r.z_norm:.15g} / {q[2]:.15g}  mu {r.mu:.15g} / {q[4]:.15g}  nu {r.nu:.15g} / {q[5]:.15g}  "
              f"alpha {r.min_alpha:.15g} / {q[6]:.15g}  restart {int(r.restart)}/{int(q[3])}")
