"""Generate golden fixtures by running the REFERENCE (ipcsim) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are frozen here
as small .npz files.  For every scene we store

* the scene arrays as the reference built them (rest, tets, masses, Bm, vol,
  surface, ...) so tests can check our builders bit-for-bit and feed the
  device identical inputs;
* the end-to-end trajectory: per-frame iteration counts, convergence flags,
  per-iteration records and the final positions of every frame;
* stage taps recorded by wrapping reference functions during the real run
  (open-loop parity): broad_phase,
  compute_constraint_set, gradient (+ incremental_potential at the same
  iterate), assemble_base_hessian + HessianModel.hvp, apply_preconditioner
  with the iterate the hierarchy was built at and the current iterate, and
  _apply_ccd (+ per_subdomain_steps alpha_d and certify_mixed).

Nothing in /root/reference is modified; wrappers are installed on the
imported modules only.
"""

from __future__ import annotations

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

from paper_2604_19892_b200 import scenes  # noqa: E402

OUT = Path(__file__).resolve().parent
MODS = (geo, en, sol)
MAX_TAPS = 6


class Tap:
    def __init__(self):
        self.rec = {}
        self.x_base = None
        self.x_cur = None
        self.h = None
        self.last_cs = None
        self.last_state = None

    def add(self, kind, item):
        lst = self.rec.setdefault(kind, [])
        lst.append(item)

    def install(self):
        tap = self
        orig = {}

        def wrap(mod, name, fn):
            orig[(mod, name)] = getattr(mod, name)
            setattr(mod, name, fn)

        o_fresh = sol._fresh_constraints

        def fresh(scene, x, base=None):
            tap.x_cur = np.array(x, copy=True)
            cs = o_fresh(scene, x, base)
            tap.last_cs = cs
            return cs

        wrap(sol, "_fresh_constraints", fresh)

        o_bp = geo.broad_phase

        def bp(x, surface, mb, d_hat):
            pt, ee = o_bp(x, surface, mb, d_hat)
            if len(tap.rec.get("broad_phase", [])) < 2 * MAX_TAPS:
                tap.add("broad_phase", dict(x=np.array(x, float).ravel(), mb=mb, d_hat=d_hat, pt=pt, ee=ee))
            return pt, ee

        wrap(geo, "broad_phase", bp)

        o_asm = en.assemble_base_hessian

        def asm(state, elastic, cs, dirichlet):
            tap.x_base = np.array(state.x, copy=True)
            tap.h = state.h
            H = o_asm(state, elastic, cs, dirichlet)
            if len(tap.rec.get("constraint_set", [])) < MAX_TAPS:
                verts, grad, d, k = cs.arrays()
                tap.add("constraint_set", dict(x=state.x.copy(), verts=verts, grad=grad, d=d, k=k))
            return H

        wrap(en, "assemble_base_hessian", asm)

        o_grad = en.gradient

        def grad(state, elastic, cs, dirichlet):
            g = o_grad(state, elastic, cs, dirichlet)
            if len(tap.rec.get("gradient", [])) < MAX_TAPS:
                e = en.incremental_potential(state, elastic, cs)
                tap.add("gradient", dict(x=state.x.copy(), x_tilde=state.x_tilde.copy(), h=state.h, g=g.copy(),
                                         energy=e))
            return g

        wrap(en, "gradient", grad)

        o_apply = masmod.apply_preconditioner

        def apply(hier, wb, g):
            z = o_apply(hier, wb, g)
            n = len(tap.rec.get("precond", []))
            has_wb = wb is not None and len(wb.per_subdomain) > 0
            n_wb = sum(1 for r in tap.rec.get("precond", []) if r["has_wb"])
            if n < MAX_TAPS or (has_wb and n_wb < MAX_TAPS // 2):
                tap.add("precond", dict(x_base=tap.x_base.copy(), x_cur=tap.x_cur.copy(), h=tap.h, g=g.copy(),
                                        z=z.copy(), has_wb=has_wb,
                                        n_touched=0 if wb is None else len(wb.per_subdomain)))
            return z

        wrap(masmod, "apply_preconditioner", apply)

        o_hvp = en.HessianModel.hvp

        def hvp(self, vec):
            out = o_hvp(self, vec)
            n = len(tap.rec.get("hvp", []))
            with_upd = len(self.updates) > 0
            n_upd = sum(1 for r in tap.rec.get("hvp", []) if r["with_updates"])
            if n < MAX_TAPS or (with_upd and n_upd < MAX_TAPS // 2):
                tap.add("hvp", dict(x_base=tap.x_base.copy(), x_cur=tap.x_cur.copy(), h=tap.h, vec=vec.copy(),
                                    out=out.copy(), with_updates=with_upd))
            return out

        en.HessianModel.hvp = hvp
        orig[(en.HessianModel, "hvp")] = o_hvp

        o_pss = ccdmod.per_subdomain_steps
        o_cert = ccdmod.certify_mixed

        def pss(pairs, partition, x, p, alpha_l=ccdmod.ALPHA_L_DEFAULT, s=ccdmod.S_DEFAULT):
            alpha_d, info = o_pss(pairs, partition, x, p, alpha_l=alpha_l, s=s)
            tap._pss = (alpha_d.copy(), info.min_alpha, len(pairs))
            return alpha_d, info

        def cert(pairs, x, p_mix, s=ccdmod.S_DEFAULT):
            ok = o_cert(pairs, x, p_mix, s=s)
            tap._cert = ok
            return ok

        wrap(ccdmod, "per_subdomain_steps", pss)
        wrap(ccdmod, "certify_mixed", cert)

        o_ccd = sol._apply_ccd

        def apply_ccd(scene, partition, x, p, config):
            tap._pss, tap._cert = None, None
            x_new, ma = o_ccd(scene, partition, x, p, config)
            if len(tap.rec.get("ccd", [])) < MAX_TAPS and tap._pss is not None:
                alpha_d, pair_min, npairs = tap._pss
                tap.add("ccd", dict(x=np.array(x).copy(), p=np.array(p).copy(), alpha_d=alpha_d,
                                    x_new=np.array(x_new).copy(), min_alpha=ma,
                                    certified=bool(tap._cert) if tap._cert is not None else True,
                                    n_pairs=npairs))
            return x_new, ma

        wrap(sol, "_apply_ccd", apply_ccd)
        self._orig = orig

    def uninstall(self):
        for (mod, name), fn in self._orig.items():
            setattr(mod, name, fn)


def scene_arrays(scene):
    el = scene.elastic
    s = scene.surface
    return dict(
        rest=scene.mesh.rest_positions, tets=el.tets, kind=el.kind_id, mu=el.mu, lam=el.lam, Bm=el.Bm, vol=el.vol,
        mass=scene.mass, dirichlet=scene.dirichlet, f_ext=scene.f_ext, tris=s.triangles, edges=s.edges,
        surf_verts=s.vertices, d_hat=scene.d_hat, kappa=scene.kappa,
    )


def flatten_taps(rec):
    out = {}
    for kind, items in rec.items():
        out[f"n_{kind}"] = len(items)
        for i, item in enumerate(items):
            for key, val in item.items():
                out[f"{kind}_{i}_{key}"] = np.asarray(val)
    return out


def run_scene(name, scene, frames, cfg, v0=None, h=0.01, taps=True):
    tap = Tap()
    if taps:
        tap.install()
    x = scene.mesh.rest_positions.ravel().copy()
    v = np.zeros_like(x) if v0 is None else np.asarray(v0, float).copy()
    iters, conv, xs, recs = [], [], [], []
    t0 = time.time()
    try:
        for f in range(frames):
            st, tr = sol.step(scene, x, v, h, cfg)
            x, v = st.x, st.v
            iters.append(tr.iterations)
            conv.append(tr.converged)
            xs.append(x.copy())
            for r in tr.records:
                recs.append([f, r.k, r.grad_norm, r.z_norm, r.r, float(r.restart), r.mu, r.nu, r.min_alpha])
    finally:
        if taps:
            tap.uninstall()
    dt = time.time() - t0
    data = dict(scene_arrays(scene))
    data.update(
        name=name, frames=frames, h=h, v0=np.zeros_like(x) if v0 is None else np.asarray(v0, float),
        iterations=np.array(iters), converged=np.array(conv), x_frames=np.array(xs), records=np.array(recs),
        ref_seconds=dt,
        cfg=np.array([cfg.eps, cfg.delta, cfg.iter_max, cfg.K, cfg.block_size, cfg.levels, cfg.coarse_block,
                      float(cfg.ccd_per_subdomain)]),
        cfg_strategy=cfg.update_strategy,
    )
    data.update(flatten_taps(tap.rec))
    np.savez_compressed(OUT / f"{name}.npz", **data)
    print(f"{name}: N={scene.mesh.n_vertices} T={len(scene.elastic.vol)} iters={iters} {dt:.1f}s "
          f"taps={ {k: len(v) for k, v in tap.rec.items()} }", flush=True)


def broad_phase_cases(name="bp_cube8", cells=8):
    """Broad-phase-only fixture at C1 size (the 8^3 soft cube on its floor):
    jittered iterates pushed into the floor's contact zone, several motion
    bounds, both the constraint-set (mb = 0, d_hat) and the CCD (mb, 0) calls."""
    scene = scenes.c1_cube(cells, mods=MODS)
    rng = np.random.default_rng(20260823)
    rest = scene.mesh.rest_positions
    free = ~scene.dirichlet
    data = dict(scene_arrays(scene))
    cases = []
    for i, (drop, jit, mb, dh) in enumerate([(0.0, 0.0, 0.0, 2e-3), (0.0095, 1e-4, 0.0, 2e-3),
                                              (0.0095, 1e-4, 3e-3, 0.0), (0.0099, 3e-4, 1e-2, 0.0),
                                              (0.0099, 3e-4, 0.0, 2e-3), (0.0, 2e-3, 0.0, 2e-2),
                                              (0.0099, 1e-3, 3e-2, 0.0), (0.0099, 1e-3, 0.0, 1e-2)]):
        x = rest.copy()
        x[free, 2] -= drop
        x[free] += jit * rng.standard_normal((free.sum(), 3))
        pt, ee = geo.broad_phase(x, scene.surface, mb, dh)
        cases.append(dict(x=x.ravel(), mb=mb, d_hat=dh, pt=pt, ee=ee))
        print(f"{name} case {i}: pt={len(pt)} ee={len(ee)}", flush=True)
    data.update(flatten_taps({"broad_phase": cases}))
    np.savez_compressed(OUT / f"{name}.npz", **data)


def main():
    if "--bp" in sys.argv:
        broad_phase_cases()
        return
    run_scene("drop", scenes.drop(MODS), 25, sol.SolverConfig())
    s = scenes.locking(MODS)
    nv = s.mesh.n_vertices
    v0 = np.zeros((nv, 3))
    v0[8:24, 2] = -1.0
    run_scene("locking", s, 10, sol.SolverConfig(block_size=8), v0=v0.ravel())
    s = scenes.stacked_boxes(MODS)
    run_scene("stacked_k8", s, 3, sol.SolverConfig(), v0=scenes.stacked_boxes_v0(s))
    s = scenes.stacked_boxes(MODS)
    run_scene("stacked_k256", s, 3, sol.SolverConfig(K=256), v0=scenes.stacked_boxes_v0(s))
    # C1-shaped soft cube: capped run (the reference stalls at first contact)
    run_scene("cube3_capped", scenes.c1_cube(3, 1e6, mods=MODS), 5, sol.SolverConfig(iter_max=60))


if __name__ == "__main__":
    main()
