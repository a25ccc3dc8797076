"""Compare per-iteration records of frame 0 (z_norm, restart, mu, nu,
min_alpha) of a golden scene: reference vs oracle (CPU) [vs GPU with --gpu]."""
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from conftest import golden_config, load_golden, scene_from_golden  # noqa: E402

from oracle import solver as osol  # noqa: E402

name = sys.argv[1]
use_gpu = "--gpu" in sys.argv
g = load_golden(name)
rec = g["records"]
ref = rec[rec[:, 0] == 0]
cfg = golden_config(g)
ocfg = osol.SolverConfig(eps=cfg.eps, delta=cfg.delta, iter_max=cfg.iter_max, K=cfg.K, block_size=cfg.block_size,
                         levels=cfg.levels, coarse_block=cfg.coarse_block, ccd_per_subdomain=cfg.ccd_per_subdomain,
                         update_strategy=cfg.update_strategy)
sc = osol.Scene.from_golden(g)
x, v, h = g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"])
_, _, otr = osol.step(sc, x, v, h, ocfg)
orows = [(r.z_norm, r.restart, r.mu, r.nu, r.min_alpha) for r in otr.records]
grows = []
if use_gpu:
    from paper_2604_19892_b200 import solver
    scene = scene_from_golden(g)
    _, tr = solver.step(scene, x, v, h, cfg)
    grows = [(r.z_norm, r.restart, r.mu, r.nu, r.min_alpha) for r in tr.records]
print("iters ref", len(ref), "oracle", len(orows), "gpu", len(grows))
for k in range(max(len(ref), len(orows), len(grows))):
    line = f"{k:4d}"
    if k < len(ref):
        line += f" | ref z={ref[k, 3]:.6e} rs={int(ref[k, 5])} mu={ref[k, 6]:.4e} a={ref[k, 8]:.4e}"
    if k < len(orows):
        z, rs, mu, nu, a = orows[k]
        line += f" | orc z={z:.6e} rs={int(rs)} mu={mu:.4e} a={a:.4e}"
    if k < len(grows):
        z, rs, mu, nu, a = grows[k]
        line += f" | gpu z={z:.6e} rs={int(rs)} mu={mu:.4e} a={a:.4e}"
    print(line)
