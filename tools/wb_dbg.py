"""Debug: precond apply with Woodbury updates, GPU vs oracle, small block sizes."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from conftest import golden_config, load_golden, scene_from_golden, rel_err
from oracle import solver as osol, physics as oph, precond as opre
g = load_golden("stacked_k256")
for bs, K in ((32, 256), (16, 256), (16, 8), (8, 256), (16, 40), (16, 48), (16, 49)):
    cfg = golden_config(g); cfg.block_size = bs; cfg.K = K
    sc = osol.Scene.from_golden(g)
    ocfg = osol.SolverConfig(block_size=bs, K=K, iter_max=3)
    # states: x_base = rest + small push, x_cur = x_base + step
    xs = []
    orig = osol.ophys.constraint_set
    def cs_tap(scene, x):
        xs.append(np.array(x).copy()); return orig(scene, x)
    osol.ophys.constraint_set = cs_tap
    osol.step(sc, g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"]), ocfg)
    osol.ophys.constraint_set = orig
    xb, xc = xs[0], xs[1]
    h = float(g["h"])
    part = sc.partition(bs)
    base = oph.constraint_set(sc, xb)
    H = oph.assemble_base_hessian(sc, xb, h, base)
    hier = opre.build_hierarchy(H, part, 2, 4)
    cands = opre.classify_all(oph.constraint_set(sc, xc), base, ocfg.eps_rot)
    topk = opre.select_top_k(cands, part.subdomain_of, K)
    wb = opre.build_update(hier, cands, topk, K)
    rng = np.random.default_rng(0)
    gv = rng.standard_normal(xb.size)
    z = opre.apply_preconditioner(hier, wb, gv); z[sc.pinned3] = 0
    scene = scene_from_golden(g); ctx = scene.context(cfg)
    ctx.snapshot(xb, h, True)
    nc, nt = ctx.update_at(xc)
    zg = ctx.precond_apply(gv, True)
    maxk = max((len(v) for v in topk.values()), default=0)
    print(f"bs={bs} K={K}: cands {len(cands)} gpu {nc}, touched oracle {len(wb)} gpu {nt}, max K_d {maxk}, rel err {rel_err(zg, z):.2e}", flush=True)
