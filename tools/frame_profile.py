"""One bench frame (C2, the first timed frame: start state from
tests/golden/c2_bench.npz) with per-iteration records: CCD time / pairs /
alpha / certificate, restart flags.  Run under ncu for a launch list of
exactly one frame, or plain for the per-iteration table."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2604_19892_b200 import scenes, solver  # noqa: E402

iter_max = int(sys.argv[1]) if len(sys.argv) > 1 else bench.ITER_MAX
g = np.load("tests/golden/c2_bench.npz")
scene = scenes.c2_stack(gap=bench.GAP)
ctx = scene.context(solver.SolverConfig(iter_max=iter_max))
ctx.set_state(g["x0"], g["v0"])
ctx.stage_timing(True)
recs, conv, _ = ctx.step_device(bench.H)
st = ctx.stage_stats()
rows = [[r.k, r.restart, r.min_alpha, r.ccd_certified, r.n_ccd_pairs, r.t_ccd_ms, r.t_grad_ms, r.t_dir_ms, r.z_norm,
         r.n_contacts] for r in recs]
np.save("gpurun_out/frame_profile_recs.npy", np.array(rows, float))
ccd = np.array([r[5] for r in rows])
clamped = np.array([r[2] < 1 for r in rows])
print(json.dumps({"iters": len(recs), "converged": conv, "restarts": int(sum(r.restart for r in recs)),
                  "ccd_ms_clamped_mean": float(ccd[clamped].mean()) if clamped.any() else None,
                  "ccd_ms_unclamped_mean": float(ccd[~clamped].mean()) if (~clamped).any() else None,
                  "n_clamped": int(clamped.sum()),
                  "stages_ms": {k: round(v[0], 2) for k, v in st.items()}}))
