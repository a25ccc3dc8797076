import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from conftest import golden_config, load_golden, scene_from_golden, rel_err
from oracle import solver as osol, ccd as occd
from paper_2604_19892_b200 import solver
g = load_golden("drop")
cfg = golden_config(g); cfg.update_strategy = "FullRebuild"
ocfg = osol.SolverConfig(update_strategy="FullRebuild")
osc = osol.Scene.from_golden(g)
x, v, h = g["rest"].ravel().copy(), g["v0"].copy(), float(g["h"])
for f in range(9):
    x, v, _ = osol.step(osc, x, v, h, ocfg)
calls = []
orig = occd.clamp
def clamp(scene, part, xx, p, per, al):
    out = orig(scene, part, xx, p, per, al)
    calls.append((xx.copy(), p.copy(), out[1], out[3]))
    return out
occd.clamp = clamp
_, _, otr = osol.step(osc, x, v, h, ocfg)
occd.clamp = orig
scene = scene_from_golden(g)
ctx = scene.context(cfg)
_, tr = solver.step(scene, x, v, h, cfg)
for k in range(min(6, len(calls))):
    xx, p, ma, cert = calls[k]
    a1, xn1, m1, c1, n1 = ctx.ccd(xx, p, exact_set=True)
    a2, xn2, m2, c2, n2 = ctx.ccd(xx, p, exact_set=False)
    print(k, "oracle min", ma, cert, "| gpu exact", m1, c1, n1, "| gpu tight", m2, c2, n2,
          "| rec gpu", tr.records[k].min_alpha if k < tr.iterations else None, "| rec orc", otr.records[k].min_alpha)
