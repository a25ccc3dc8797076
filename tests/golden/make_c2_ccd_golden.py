"""A second reference CCD tap at bench scale with clamping active: from the
c2_bench.npz state x0, the restart step scaled up, p2 = 40 p, so that many
subdomains get alpha_d < 1 (ccd.py:221-320, solver.py:268-280).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c2_ccd_golden.py

Writes tests/golden/c2_bench_ccd.npz (alpha_d, x_new, min alpha, certificate,
pair count).  ~5 minutes on one core."""

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import ipcsim.ccd as ccdmod  # noqa: E402
import ipcsim.energy as en  # noqa: E402
import ipcsim.geometry as geo  # noqa: E402
import ipcsim.solver as sol  # noqa: E402

import bench  # noqa: E402
from paper_2604_19892_b200 import scenes  # noqa: E402

SCALE = 40.0


def main():
    g = np.load(Path(__file__).resolve().parent / "c2_bench.npz")
    scene = scenes.c2_stack(gap=bench.GAP, mods=(geo, en, sol))
    cfg = sol.SolverConfig(iter_max=bench.ITER_MAX)
    part = scene.partition(cfg.block_size)
    x, p = g["x0"], SCALE * g["p"]
    t0 = time.time()
    pairs = ccdmod.collect_pairs(x, scene.surface, p)
    alpha_d, info = ccdmod.per_subdomain_steps(pairs, part, x, p, alpha_l=cfg.alpha_l)
    scale = alpha_d[part.subdomain_of]
    p_mix = (scale[:, None] * p.reshape(-1, 3)).ravel()
    cert = bool(ccdmod.certify_mixed(pairs, x, p_mix))
    x_new, min_alpha = sol._apply_ccd(scene, part, x, p, cfg)
    print(f"{time.time() - t0:.0f}s: {len(pairs)} pairs, {int((alpha_d < 1).sum())} clamped subdomains, "
          f"min alpha {min_alpha}, certified {cert}", flush=True)
    np.savez_compressed(Path(__file__).resolve().parent / "c2_bench_ccd.npz", scale=SCALE, alpha_d=alpha_d,
                        x_new=x_new, min_alpha=min_alpha, certified=cert, n_pairs=len(pairs),
                        pair_min=info.min_alpha)


if __name__ == "__main__":
    main()
