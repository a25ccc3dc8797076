import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from conftest import golden_config, load_golden, scene_from_golden
from oracle import solver as osol
from paper_2604_19892_b200 import solver
g = load_golden("stacked_k256")
bs = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = golden_config(g); cfg.block_size = bs; cfg.iter_max = 400
ocfg = osol.SolverConfig(block_size=bs, K=cfg.K, iter_max=400)
x, v, h = g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"])
_, _, otr = osol.step(osol.Scene.from_golden(g), x, v, h, ocfg)
_, tr = solver.step(scene_from_golden(g), x, v, h, cfg)
print("iters oracle", otr.iterations, "gpu", tr.iterations)
for k in range(min(60, otr.iterations, tr.iterations)):
    o, r = otr.records[k], tr.records[k]
    print(f"{k:3d} orc z={o.z_norm:.6e} rs={int(o.restart)} mu={o.mu:.4e} a={o.min_alpha:.3e} c={int(o.certified)} | gpu z={r.z_norm:.6e} rs={int(r.restart)} mu={r.mu:.4e} a={r.min_alpha:.3e} c={int(r.ccd_certified)}")
