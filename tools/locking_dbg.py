import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from conftest import golden_config, load_golden, scene_from_golden
from oracle import solver as osol
from paper_2604_19892_b200 import solver
name = sys.argv[1] if len(sys.argv) > 1 else "locking"
g = load_golden(name); cfg = golden_config(g)
x, v, h = g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"])
sc = osol.Scene.from_golden(g)
ocfg = osol.SolverConfig(eps=cfg.eps, delta=cfg.delta, iter_max=60, K=cfg.K, block_size=cfg.block_size, levels=cfg.levels,
                         coarse_block=cfg.coarse_block, ccd_per_subdomain=cfg.ccd_per_subdomain, update_strategy=cfg.update_strategy)
_, _, otr = osol.step(sc, x, v, h, ocfg, with_energy=True)
out = {}
for exact in (0, 1):
    scene = scene_from_golden(g)
    ctx = scene.context(cfg)
    ctx.set_option(1, exact)
    ctx.set_option(2, 1)
    _, tr = solver.step(scene, x, v, h, cfg)
    out[exact] = tr.records
for k in range(min(20, len(otr.records))):
    o = otr.records[k]
    line = f"{k:3d} orc z={o.z_norm:.9e} a={o.min_alpha:.6e} cert={int(o.certified)} E={o.energy:.12e}"
    for e in (0, 1):
        if k < len(out[e]):
            r = out[e][k]
            line += f" | {'ex' if e else 'ti'} z={r.z_norm:.9e} a={r.min_alpha:.6e} cert={int(r.ccd_certified)} E={r.energy:.12e}"
    print(line)
