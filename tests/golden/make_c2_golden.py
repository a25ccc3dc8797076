"""Reference (ipcsim) stage taps at BENCH scale: config 2 (8 soft cubes on a
floor, 46,664 V / 235,830 T) at the state where bench.py's first timed frame
starts (after its 5 warm-up frames; GPU state dumped by tools/c2_dump.py --
the solver is bitwise deterministic, so every box reaches the same bits).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c2_golden.py STATE.npz

From (x0, v0) it runs the reference's own functions for the first PNCG
iteration of that frame exactly as advance_step does (solver.py:320-392,
rebuild branch) and then the non-rebuild branch at the CCD-clamped iterate
x1 (solver.py:336-346):

* prepare_step -> x_tilde; compute_constraint_set at x0 (pairs, d, k);
* gradient + incremental_potential at x0;
* assemble_base_hessian + build_hierarchy (levels 2, coarse_block 4: coarse
  orders 1095 and 276) -> z = apply_preconditioner(g), pinned rows zeroed;
* HessianModel.hvp(z); the restart step p = -(z.g / z.Hz) z;
* _apply_ccd -> alpha_d (per_subdomain_steps), certify_mixed, x1, min alpha;
* at x1 against the x0 base: classify_all, select_top_k (K=8), build_update,
  gradient g1, z1 = apply_preconditioner(wb, g1), HessianModel(H_base,
  candidates).hvp(z1).

Writes tests/golden/c2_bench.npz (inputs x0/v0 and the outputs above).  Takes
~8 minutes on one core (the reference's Python broad phase dominates).
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import ipcsim.ccd as ccdmod  # noqa: E402
import ipcsim.contact as con  # noqa: E402
import ipcsim.energy as en  # noqa: E402
import ipcsim.geometry as geo  # noqa: E402
import ipcsim.mas as masmod  # noqa: E402
import ipcsim.solver as sol  # noqa: E402
import ipcsim.woodbury as wbmod  # noqa: E402

import bench  # noqa: E402
from paper_2604_19892_b200 import scenes  # noqa: E402

OUT = Path(__file__).resolve().parent / "c2_bench.npz"


def scene_hash(scene):
    h = hashlib.sha256()
    el, s = scene.elastic, scene.surface
    for a in (scene.mesh.rest_positions, el.tets, el.Bm, el.vol, el.mu, el.lam, scene.mass, scene.dirichlet,
              scene.f_ext, s.triangles, s.edges, s.vertices):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    st = np.load(sys.argv[1] if len(sys.argv) > 1 else ROOT / "tools" / "_data" / "c2_state_w5.npz")
    x0, v0 = st["x0"], st["v0"]
    scene = scenes.c2_stack(gap=bench.GAP, mods=(geo, en, sol))
    cfg = sol.SolverConfig(iter_max=bench.ITER_MAX)
    h = bench.H
    T = {}
    t0 = time.time()

    def lap(msg):
        print(f"{time.time() - t0:7.1f}s {msg}", flush=True)

    state = en.prepare_step(x0, v0, scene.mass, h, scene.f_ext, scene.dirichlet)  # as solver.step does
    partition = scene.partition(cfg.block_size)
    pinned3 = np.repeat(scene.dirichlet, 3)
    x = state.x.copy()
    # ---- iteration 0: rebuild branch (solver.py:323-335) ----
    cs = sol._fresh_constraints(scene, x)
    verts, grad, d, k = cs.arrays()
    lap(f"constraint set: {len(d)} pairs")
    T.update(cs_verts=np.asarray(verts, np.int32), cs_d=d, cs_k=k)
    H_base = en.assemble_base_hessian(sol._state_at(state, x), scene.elastic, cs, scene.dirichlet)
    hier = masmod.build_hierarchy(H_base, partition, L=cfg.levels, coarse_block=cfg.coarse_block)
    lap(f"H_base + hierarchy (coarse {[m.shape[0] for m in hier.coarse_inv] if hasattr(hier, 'coarse_inv') else '?'})")
    g = en.gradient(sol._state_at(state, x), scene.elastic, cs, scene.dirichlet)
    e = en.incremental_potential(sol._state_at(state, x), scene.elastic, cs)
    z = masmod.apply_preconditioner(hier, None, g)
    z[pinned3] = 0.0
    hmodel = en.HessianModel(H_base=H_base, updates=[])
    v = hmodel.hvp(z)
    zg, zv = float(z @ g), float(z @ v)
    mu = zg / zv
    p = -mu * z
    lap("gradient / z / hvp")
    pairs = ccdmod.collect_pairs(x, scene.surface, p)
    alpha_d, info = ccdmod.per_subdomain_steps(pairs, partition, x, p, alpha_l=cfg.alpha_l)
    scale = alpha_d[partition.subdomain_of]
    p_mix = (scale[:, None] * p.reshape(-1, 3)).ravel()
    cert = bool(ccdmod.certify_mixed(pairs, x, p_mix))
    x1, min_alpha = sol._apply_ccd(scene, partition, x, p, cfg)
    lap(f"CCD: {len(pairs)} pairs, min alpha {min_alpha}, certified {cert}")
    T.update(x0=x0, v0=v0, x_tilde=state.x_tilde, h=h, g=g, energy=e, z=z, hv=v, mu=mu, p=p, alpha_d=alpha_d,
             ccd_min_alpha=min_alpha, ccd_certified=cert, ccd_pairs=len(pairs), x1=x1,
             z_norm=float(np.linalg.norm(z)), grad_norm=float(np.linalg.norm(g)))
    # ---- the non-rebuild branch at x1 (solver.py:336-346) ----
    cs1 = sol._fresh_constraints(scene, x1, base=cs.current)
    cands = con.classify_all(cs1, cfg.eps_rot)
    topk = con.select_top_k(cands, partition.subdomain_of, cfg.K)
    wb = wbmod.build_update(hier, topk, K=cfg.K)
    g1 = en.gradient(sol._state_at(state, x1), scene.elastic, cs1, scene.dirichlet)
    z1 = masmod.apply_preconditioner(hier, wb, g1)
    z1[pinned3] = 0.0
    hv1 = en.HessianModel(H_base=H_base, updates=cands).hvp(z1)
    lap(f"update branch: {len(cands)} candidates, {len(wb.per_subdomain)} touched subdomains")
    T.update(g1=g1, z1=z1, hv1=hv1, n_candidates=len(cands), n_touched=len(wb.per_subdomain))
    T["scene_sha256"] = scene_hash(scene)
    np.savez_compressed(OUT, **T)
    lap(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
