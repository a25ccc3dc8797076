import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"
GOLDEN_SCENES = ("drop", "locking", "stacked_k8", "stacked_k256", "cube3_capped")
BP_FIXTURES = ("bp_cube8",)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libmaspncg.so")


@pytest.fixture
def rng():
    return np.random.default_rng(20260823)


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_taps(g, kind):
    n = int(g.get(f"n_{kind}", 0))
    out = []
    for i in range(n):
        pre = f"{kind}_{i}_"
        out.append({k[len(pre):]: v for k, v in g.items() if k.startswith(pre)})
    return out


def golden_config(g):
    from paper_2604_19892_b200.solver import SolverConfig

    eps, delta, iter_max, K, bs, levels, cb, per_sub = g["cfg"]
    return SolverConfig(eps=float(eps), delta=float(delta), iter_max=int(iter_max), K=int(K), block_size=int(bs),
                        levels=int(levels), coarse_block=int(cb), ccd_per_subdomain=bool(per_sub),
                        update_strategy=str(g["cfg_strategy"]))


def scene_from_golden(g):
    """Scene fed with the reference-built arrays (identical device inputs)."""
    from paper_2604_19892_b200.solver import Scene

    mesh = SimpleNamespace(rest_positions=g["rest"], tets=g["tets"], n_vertices=len(g["rest"]))
    surface = SimpleNamespace(triangles=g["tris"], edges=g["edges"], vertices=g["surf_verts"])
    elastic = SimpleNamespace(tets=g["tets"], kind_id=g["kind"], mu=g["mu"], lam=g["lam"], Bm=g["Bm"], vol=g["vol"])
    return Scene(mesh=mesh, surface=surface, elastic=elastic, mass=g["mass"], dirichlet=g["dirichlet"],
                 d_hat=float(g["d_hat"]), kappa=float(g["kappa"]), f_ext=g["f_ext"])


def rel_err(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)
