"""C3 coarse-level SPD failure probe.

Runs the C3 rod (nx cells long, default 1000) with the default MAS depth on
the GPU until the build raises non-spd-subdomain, keeping every coarse
level's assembled Galerkin matrix (MP_OPT_KEEP_COARSE).  At the failing
iterate it then (1) reports the GPU coarse matrices' smallest eigenvalues and
whether numpy's Cholesky accepts them, (2) rebuilds the same hierarchy with
the CPU oracle (constraint set, H_base, C H C^T, cho_factor -- the
reference's algorithm) at the same x and reports whether IT fails, and the
relative difference of the two coarse matrices.  Writes the failing x to
gpurun_out/c3_fail_x.npy so the CPU side can replay it.
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import scenes, solver  # noqa: E402
from paper_2604_19892_b200.errors import NotSpdError  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
iter_max = int(sys.argv[3]) if len(sys.argv) > 3 else 200
out_dir = os.environ.get("OUT", "gpurun_out")
os.makedirs(out_dir, exist_ok=True)
H = 0.01
scene = scenes.c3_rod(cells=(nx, 8, 8), length=6.25 * nx / 2500)
cfg = solver.SolverConfig(iter_max=iter_max)
ctx = scene.context(cfg, device=0)
ctx.set_option(7, 1)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, scenes.c3_rod_v0(scene))
fail = None
for f in range(frames):
    try:
        recs, conv, _ = ctx.step_device(H)
        print(json.dumps({"frame": f, "iters": len(recs), "converged": conv}), flush=True)
    except NotSpdError as e:
        fail = (f, str(e))
        break
if fail is None:
    print("no failure")
    sys.exit(0)
print("failure in frame", fail, flush=True)
x_fail, _ = ctx.get_state()
np.save(os.path.join(out_dir, "c3_fail_x.npy"), x_fail)
rep = {"nx": nx, "frame": fail[0], "error": fail[1]}
gpu_M = []
for lvl in (1, 2):
    try:
        M = ctx.coarse_matrix(lvl)
    except Exception as e:  # noqa: BLE001
        rep[f"gpu_level{lvl}"] = repr(e)
        continue
    gpu_M.append(M)
    w = np.linalg.eigvalsh(0.5 * (M + M.T))
    try:
        np.linalg.cholesky(0.5 * (M + M.T))
        chol = True
    except np.linalg.LinAlgError:
        chol = False
    rep[f"gpu_level{lvl}"] = {"n": len(M), "eig_min": float(w[0]), "eig_max": float(w[-1]),
                              "n_neg": int((w <= 0).sum()), "numpy_cholesky_ok": chol,
                              "asym": float(np.abs(M - M.T).max() / np.abs(M).max())}
print(json.dumps(rep), flush=True)

# the oracle's hierarchy at the same iterate
from oracle import physics as ophys, precond as opre, solver as osol  # noqa: E402

t0 = time.time()
osc = osol.Scene.from_scene(scene)
cs = ophys.constraint_set(osc, x_fail)
Hb = ophys.assemble_base_hessian(osc, x_fail, H, cs)
part = osc.partition(32)
rep["oracle_contacts"] = len(cs)
units = list(part.selection)
n = Hb.shape[0]
import math  # noqa: E402
import scipy.linalg  # noqa: E402
import scipy.sparse as sp  # noqa: E402

for lvl in (1, 2):
    A_l = math.ceil(len(units) / 4)
    groups = [np.concatenate(units[a * 4:(a + 1) * 4]) for a in range(A_l)]
    rows = np.concatenate([np.repeat(3 * a + np.arange(3), len(g)) for a, g in enumerate(groups)])
    cols = np.concatenate([(3 * g[None, :] + np.arange(3)[:, None]).ravel() for g in groups])
    vals = np.concatenate([np.full(3 * len(g), 1.0 / len(g)) for g in groups])
    Cm = sp.csr_matrix((vals, (rows, cols)), shape=(3 * A_l, n))
    M = (Cm @ Hb @ Cm.T).toarray()
    M = 0.5 * (M + M.T)
    w = np.linalg.eigvalsh(M)
    try:
        scipy.linalg.cho_factor(M)
        ok = True
    except scipy.linalg.LinAlgError:
        ok = False
    r = {"n": len(M), "eig_min": float(w[0]), "eig_max": float(w[-1]), "n_neg": int((w <= 0).sum()),
         "cho_factor_ok": ok}
    # the GPU numbers its aggregates in renumbered order; the oracle's
    # aggregate a = the same subdomain range, so dof order matches
    if len(gpu_M) >= lvl and gpu_M[lvl - 1].shape == M.shape:
        G = gpu_M[lvl - 1]
        r["rel_diff_vs_gpu"] = float(np.abs(G - M).max() / np.abs(M).max())
    rep[f"oracle_level{lvl}"] = r
    units = groups
rep["oracle_s"] = round(time.time() - t0, 1)
print(json.dumps(rep), flush=True)
with open(os.path.join(out_dir, "c3_spd_probe.json"), "w") as fh:
    json.dump(rep, fh, indent=1)
