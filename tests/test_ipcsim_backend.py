"""The INTEGRATION.md binding (paper_2604_19892_b200/ipcsim_backend.py):
installs into the reference's own solver module and restores it.  Where a
GPU is present the patched reference ``step`` must also run on it; in the
build container (reference importable, no GPU) only the wiring is checked."""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="the reference is only importable in the build container")
def test_install_patches_and_restores_reference_solver():
    sys.path.insert(0, str(REF))
    try:
        import ipcsim.solver as rsol
    finally:
        sys.path.remove(str(REF))
    from paper_2604_19892_b200 import ipcsim_backend

    cpu_step, cpu_adv = rsol.step, rsol.advance_step
    ipcsim_backend.install(rsol)
    try:
        assert rsol.step is not cpu_step and rsol.advance_step is not cpu_adv
        import torch

        if torch.cuda.is_available():
            import ipcsim.geometry as geo

            mesh = geo.make_single_tet(0.2)
            from paper_2604_19892_b200 import scenes

            scene = scenes.drop()
            x = scene.mesh.rest_positions.ravel().copy()
            st, tr = rsol.step(scene, x, np.zeros_like(x), 0.01, rsol.SolverConfig())
            assert isinstance(tr, rsol.SolverTrace) and tr.converged and mesh is not None
    finally:
        ipcsim_backend.uninstall(rsol)
    assert rsol.step is cpu_step and rsol.advance_step is cpu_adv
