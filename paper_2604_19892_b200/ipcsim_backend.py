"""The INTEGRATION.md binding as a module: route the reference package's
``solver.step`` / ``solver.advance_step`` (`pkg/src/ipcsim/solver.py:296-464`)
through the B200 path, keeping the reference's own types.

    import ipcsim.solver
    from paper_2604_19892_b200 import ipcsim_backend
    ipcsim_backend.install(ipcsim.solver)      # step / advance_step now run on the GPU

The reference Scene is converted once (its arrays, the same layout the C ABI
takes) and the device context is cached on the Scene; SimState comes back
through ``dataclasses.replace`` and SolverTrace / IterRecord are the
module's own classes.  ``uninstall`` restores the CPU functions."""

from __future__ import annotations

import dataclasses

from . import solver as dev

_SAVED = {}


def _device_scene(scene):
    ds = getattr(scene, "_b200_scene", None)
    if ds is None:
        ds = dev.Scene(mesh=scene.mesh, surface=scene.surface, elastic=scene.elastic, mass=scene.mass,
                       dirichlet=scene.dirichlet, d_hat=scene.d_hat, kappa=scene.kappa, f_ext=scene.f_ext)
        object.__setattr__(scene, "_b200_scene", ds)
    return ds


def _device_config(cfg):
    return dev.SolverConfig(**{f.name: getattr(cfg, f.name) for f in dataclasses.fields(dev.SolverConfig)})


def _module_trace(mod, tr):
    out = mod.SolverTrace(converged=tr.converged, flags=list(tr.flags))
    for r in tr.records:
        out.records.append(mod.IterRecord(k=r.k, grad_norm=r.grad_norm, z_norm=r.z_norm, r=r.r, restart=r.restart,
                                          mu=r.mu, nu=r.nu, min_alpha=r.min_alpha, t_grad_ms=r.t_grad_ms,
                                          t_dir_ms=r.t_dir_ms, t_ccd_ms=r.t_ccd_ms))
    return out


def install(mod):
    """Patch a reference-compatible solver module (ipcsim.solver)."""
    if mod in _SAVED:
        return
    _SAVED[mod] = (mod.step, mod.advance_step)

    def advance_step(scene, state, config):
        config.validate()
        ctx = _device_scene(scene).context(_device_config(config))
        x, v, recs, conv, flags = ctx.advance(state.x, state.v, state.x_tilde, state.h)
        return dataclasses.replace(state, x=x, v=v), _module_trace(mod, dev._trace(recs, conv, flags))

    def step(scene, x, v, h, config):
        state = mod.en.prepare_step(x, v, scene.mass, h, scene.f_ext, scene.dirichlet)
        return advance_step(scene, state, config)

    mod.advance_step = advance_step
    mod.step = step


def uninstall(mod):
    if mod in _SAVED:
        mod.step, mod.advance_step = _SAVED.pop(mod)
