"""Debug helper: run every stage tap of one golden scene, print errors."""
import sys, traceback
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from conftest import golden_config, golden_taps, load_golden, rel_err, scene_from_golden
name = sys.argv[1]; stages = sys.argv[2].split(",") if len(sys.argv) > 2 else ["grad","hvp","precond","ccd","e2e"]
g = load_golden(name); cfg = golden_config(g); scene = scene_from_golden(g); ctx = scene.context(cfg)
pin3 = np.repeat(g["dirichlet"].astype(bool), 3)
def run(tag, fn):
    try: print(tag, fn(), flush=True)
    except Exception as e: print(tag, "EXC", repr(e)[:300], flush=True)
if "grad" in stages:
    for t in golden_taps(g, "gradient"):
        run("grad", lambda: (rel_err(ctx.gradient(t["x"], t["x_tilde"], float(t["h"])), t["g"]),
                             ctx.energy(t["x"], t["x_tilde"], float(t["h"])) - float(t["energy"]), float(t["energy"])))
if "hvp" in stages:
    for t in golden_taps(g, "hvp"):
        def f():
            ctx.snapshot(t["x_base"], float(t["h"]), True)
            u = bool(t["with_updates"])
            if u: ctx.update_at(t["x_cur"])
            return u, rel_err(ctx.hvp(t["vec"], u), t["out"])
        run("hvp", f)
if "precond" in stages:
    for t in golden_taps(g, "precond"):
        def f():
            ctx.snapshot(t["x_base"], float(t["h"]), True)
            u = bool(t["has_wb"]); nt = None
            if u: nt = ctx.update_at(t["x_cur"])
            z = ctx.precond_apply(t["g"], u); ref = t["z"].copy(); ref[pin3] = 0
            return u, nt, int(t["n_touched"]), rel_err(z, ref)
        run("precond", f)
if "ccd" in stages:
    for t in golden_taps(g, "ccd"):
        def f():
            a, xn, ma, cert, npairs = ctx.ccd(t["x"], t["p"])
            return npairs, int(t["n_pairs"]), np.abs(a - t["alpha_d"]).max(), cert, bool(t["certified"]), ma, float(t["min_alpha"]), rel_err(xn, t["x_new"])
        run("ccd", f)
if "e2e" in stages:
    from paper_2604_19892_b200 import solver
    x = g["rest"].ravel().copy(); v = g["v0"].copy(); h = float(g["h"])
    for fr in range(int(g["frames"])):
        try:
            st, tr = solver.step(scene, x, v, h, cfg)
        except Exception as e:
            print("e2e EXC", repr(e)[:300]); break
        x, v = st.x, st.v
        print("e2e frame", fr, tr.iterations, int(g["iterations"][fr]), tr.converged, rel_err(x, g["x_frames"][fr]), flush=True)
