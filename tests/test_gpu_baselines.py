"""Device baselines against the reference's own
trajectories (tests/golden/make_baseline_golden.py): the 3x3 block Jacobi
preconditioner (solver.py:207-246) and the FR / PR / DK / CD direction
rules with the backtracking line search (solver.py:171-200, 283-293,
393-412).  Drop scene (smooth frames): per-frame PNCG iteration counts
within +-5% (at least +-1), the same convergence flags, final positions
within 1e-6.  Stacked scene (chaotic contact frames, like the MAS stacked
goldens): the first two iterations' records follow the reference (1e-6),
then the same convergence outcome.  (Beyond that the trajectories part:
e.g. MAS+PR iteration 1's global CCD step is 0.011062 here and 0.011094 in
ipcsim -- an ill-conditioned cubic window of one pair, where np.linalg.det
(LU) and the filtered-exact determinants of ccd.cuh round differently;
SURVEY Appendix A #15.)"""

from pathlib import Path

import numpy as np
import pytest

from paper_2604_19892_b200 import scenes, solver

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).resolve().parent / "golden" / "baselines.npz")


@pytest.mark.parametrize("i", range(int(G["n"])))
def test_baseline_matches_reference(i):
    name, pre, rule = [str(s) for s in G[f"v{i}_meta"]]
    scene = scenes.drop() if name == "drop" else scenes.stacked_boxes()
    v = np.zeros(3 * scene.mesh.n_vertices) if name == "drop" else scenes.stacked_boxes_v0(scene)
    x = scene.mesh.rest_positions.ravel().copy()
    cfg = solver.SolverConfig(preconditioner=pre, direction_rule=rule, iter_max=300)
    ref_iters, ref_conv, ref_recs = G[f"v{i}_iters"], G[f"v{i}_converged"], G[f"v{i}_records"]
    if name != "drop":
        st, tr = solver.step(scene, x, v, 0.01, cfg)
        first = ref_recs[ref_recs[:, 0] == 0]
        n = min(2, len(first), tr.iterations)
        for r, q in zip(tr.records[:n], first[:n]):
            assert int(r.restart) == int(q[3])
            assert abs(r.z_norm - q[2]) <= 1e-6 * abs(q[2]), (r.k, r.z_norm, q[2])
        assert tr.converged == bool(ref_conv[0])
        return
    for f in range(len(ref_iters)):
        st, tr = solver.step(scene, x, v, 0.01, cfg)
        x, v = st.x, st.v
        tol = max(1, int(np.ceil(0.05 * ref_iters[f])))
        assert abs(tr.iterations - int(ref_iters[f])) <= tol, (f, tr.iterations, ref_iters[f])
        assert tr.converged == bool(ref_conv[f])
    ref_x = G[f"v{i}_x"]
    assert np.linalg.norm(x - ref_x) <= 1e-6 * np.linalg.norm(ref_x)
