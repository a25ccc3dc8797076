"""Reference (ipcsim) trajectories of the baseline solver variants (SURVEY
8(f) rank 3: Jacobi, FR / PR / DK / CD with the backtracking line search;
solver.py:171-246, 283-293, 393-412) on the drop and stacked scenes.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_baseline_golden.py

Writes tests/golden/baselines.npz: per variant the per-frame iteration
counts, convergence flags, records and final positions."""

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import ipcsim.energy as en  # noqa: E402
import ipcsim.geometry as geo  # noqa: E402
import ipcsim.solver as sol  # noqa: E402

from paper_2604_19892_b200 import scenes  # noqa: E402

MODS = (geo, en, sol)
VARIANTS = [("drop", "MAS", "FR"), ("drop", "MAS", "PR"), ("drop", "MAS", "DK"), ("drop", "MAS", "CD"),
            ("drop", "Jacobi", "Subspace2D"), ("drop", "Jacobi", "PR"),
            ("stacked", "Jacobi", "Subspace2D"), ("stacked", "MAS", "PR")]


def main():
    out = {}
    for i, (name, pre, rule) in enumerate(VARIANTS):
        scene = scenes.drop(MODS) if name == "drop" else scenes.stacked_boxes(MODS)
        v = np.zeros(3 * scene.mesh.n_vertices) if name == "drop" else scenes.stacked_boxes_v0(scene)
        x = scene.mesh.rest_positions.ravel().copy()
        cfg = sol.SolverConfig(preconditioner=pre, direction_rule=rule, iter_max=300)
        frames = 8 if name == "drop" else 2
        iters, conv, recs = [], [], []
        t0 = time.time()
        for f in range(frames):
            st, tr = sol.step(scene, x, v, 0.01, cfg)
            x, v = st.x, st.v
            iters.append(tr.iterations)
            conv.append(tr.converged)
            recs += [[f, r.k, r.z_norm, float(r.restart), r.mu, r.nu, r.min_alpha] for r in tr.records]
        key = f"v{i}_"
        out.update({key + "meta": np.array([name, pre, rule]), key + "iters": np.array(iters),
                    key + "converged": np.array(conv), key + "records": np.array(recs), key + "x": x,
                    key + "v": v})
        print(f"{name} {pre}+{rule}: iters {iters} conv {conv} {time.time() - t0:.1f}s", flush=True)
    out["n"] = len(VARIANTS)
    np.savez_compressed(Path(__file__).resolve().parent / "baselines.npz", **out)


if __name__ == "__main__":
    main()
