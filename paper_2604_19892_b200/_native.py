"""ctypes binding of the C ABI declared in include/maspncg.h.

The shared library is built in-tree (``build_native.py``) and is the ONLY
compute path: if it is missing or a call fails, an exception is raised --
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from .errors import (
    CapacityError, ConfigError, CudaError, DegeneratePrimitiveError, NotSpdError, PenetrationError, SimError,
)

LIB_PATH = Path(__file__).resolve().parent / "libmaspncg.so"

_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class SceneDesc(C.Structure):
    _fields_ = [
        ("n_verts", C.c_int64), ("rest", _f64p), ("mass", _f64p), ("dirichlet", C.POINTER(C.c_uint8)),
        ("f_ext", _f64p), ("n_tets", C.c_int64), ("tets", _i64p), ("kind", C.POINTER(C.c_int8)),
        ("mu", _f64p), ("lam", _f64p), ("Bm", _f64p), ("vol", _f64p), ("n_tris", C.c_int64), ("tris", _i64p),
        ("n_edges", C.c_int64), ("edges", _i64p), ("n_surf_verts", C.c_int64), ("surf_verts", _i64p),
        ("d_hat", C.c_double), ("kappa", C.c_double),
    ]


class SolverConfigC(C.Structure):
    _fields_ = [
        ("eps", C.c_double), ("delta", C.c_double), ("iter_max", C.c_int64), ("K", C.c_int32),
        ("preconditioner", C.c_int32), ("direction_rule", C.c_int32), ("update_strategy", C.c_int32),
        ("block_size", C.c_int32), ("levels", C.c_int32), ("coarse_block", C.c_int32),
        ("ccd_per_subdomain", C.c_int32), ("eps_rot", C.c_double), ("alpha_l", C.c_double),
    ]


class IterRecordC(C.Structure):
    _fields_ = [
        ("k", C.c_int64), ("grad_norm", C.c_double), ("z_norm", C.c_double), ("r", C.c_double),
        ("restart", C.c_int32), ("n_contacts", C.c_int32), ("mu", C.c_double), ("nu", C.c_double),
        ("min_alpha", C.c_double), ("t_grad_ms", C.c_double), ("t_dir_ms", C.c_double),
        ("t_ccd_ms", C.c_double), ("n_candidates", C.c_int32), ("n_ccd_pairs", C.c_int32),
        ("ccd_certified", C.c_int32), ("pad_", C.c_int32), ("energy", C.c_double),
    ]


EXPORTS = (
    "mp_create", "mp_create_multi", "mp_shards", "mp_destroy", "mp_set_config", "mp_status_code", "mp_last_error", "mp_stream", "mp_partition",
    "mp_step", "mp_advance", "mp_broad_phase", "mp_constraint_set", "mp_gradient", "mp_energy", "mp_snapshot",
    "mp_hvp", "mp_precond_apply", "mp_update_at", "mp_ccd", "mp_coarse_matrix", "mp_spd_inverse", "mp_shard_range", "mp_check_intersections", "mp_set_contact", "mp_launch_count", "mp_stage_timing", "mp_stage_stats", "mp_set_option",
)

STAGES = ("gradient", "mas_apply", "hvp", "constraint_set", "hessian", "mas_build", "update", "ccd", "mas_apply_l0",
          "tet_grad", "host_wait", "loop", "mas_sweep0", "coarse_inv")

_lib = None


def load_library():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2604_19892_b200.build_native` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(str(LIB_PATH))
    vp = C.c_void_p
    lib.mp_create.argtypes = [C.POINTER(SceneDesc), C.POINTER(SolverConfigC), C.c_int, C.POINTER(vp)]
    lib.mp_create_multi.argtypes = [C.POINTER(SceneDesc), C.POINTER(SolverConfigC), C.c_int, C.POINTER(C.c_int),
                                    C.POINTER(vp)]
    lib.mp_shards.argtypes = [vp]
    lib.mp_destroy.argtypes = [vp]
    lib.mp_destroy.restype = None
    lib.mp_set_config.argtypes = [vp, C.POINTER(SolverConfigC)]
    lib.mp_status_code.argtypes = [C.c_int]
    lib.mp_status_code.restype = C.c_char_p
    lib.mp_last_error.argtypes = [vp]
    lib.mp_last_error.restype = C.c_char_p
    lib.mp_create_error.restype = C.c_char_p
    lib.mp_stream.argtypes = [vp]
    lib.mp_stream.restype = vp
    lib.mp_launch_count.argtypes = [vp]
    lib.mp_launch_count.restype = C.c_int64
    lib.mp_partition.argtypes = [vp, _i64p, _i64p]
    lib.mp_partition_host.argtypes = [_f64p, C.c_int64, C.c_int32, _i64p]
    lib.mp_check_intersections.argtypes = [C.c_int, C.c_int64, _f64p, C.c_int64, _i64p, C.c_double, _i64p, _i64p]
    lib.mp_set_contact.argtypes = [vp, C.c_double, C.c_double]
    lib.mp_shard_range.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i64p]
    lib.mp_spd_inverse.argtypes = [C.c_int, C.c_int64, _f64p, _f64p, C.POINTER(C.c_int32)]
    rec = C.POINTER(IterRecordC)
    step_tail = [_f64p, _f64p, rec, C.c_int64, _i64p, C.POINTER(C.c_int32), C.POINTER(C.c_uint32)]
    lib.mp_step.argtypes = [vp, _f64p, _f64p, C.c_double] + step_tail
    lib.mp_advance.argtypes = [vp, _f64p, _f64p, _f64p, C.c_double] + step_tail
    lib.mp_step_device.argtypes = [vp, C.c_double, rec, C.c_int64, _i64p, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_uint32)]
    lib.mp_set_state.argtypes = [vp, _f64p, _f64p]
    lib.mp_get_state.argtypes = [vp, _f64p, _f64p]
    lib.mp_broad_phase.argtypes = [vp, _f64p, C.c_double, C.c_double, _i64p, C.c_int64, _i64p, _i64p, C.c_int64,
                                   _i64p]
    lib.mp_constraint_set.argtypes = [vp, _f64p, C.c_int64, _i64p, _i64p, C.POINTER(C.c_uint8), _f64p, _f64p,
                                      _f64p]
    lib.mp_gradient.argtypes = [vp, _f64p, _f64p, C.c_double, _f64p]
    lib.mp_energy.argtypes = [vp, _f64p, _f64p, C.c_double, _f64p]
    lib.mp_snapshot.argtypes = [vp, _f64p, C.c_double, C.c_int]
    lib.mp_hvp.argtypes = [vp, _f64p, C.c_int, _f64p]
    lib.mp_precond_apply.argtypes = [vp, _f64p, C.c_int, _f64p]
    lib.mp_update_at.argtypes = [vp, _f64p, _i64p, _i64p]
    lib.mp_ccd.argtypes = [vp, _f64p, _f64p, _f64p, _f64p, _f64p, C.POINTER(C.c_int32), _i64p, C.c_int32]
    lib.mp_coarse_matrix.argtypes = [vp, C.c_int, _f64p, C.c_int64, _i64p]
    lib.mp_stage_timing.argtypes = [vp, C.c_int]
    lib.mp_set_option.argtypes = [vp, C.c_int, C.c_int64]
    lib.mp_stage_stats.argtypes = [vp, C.c_int, _f64p, _i64p, _f64p]
    _lib = lib
    return lib


_ERRORS = {1: PenetrationError, 7: DegeneratePrimitiveError, 8: ConfigError, 9: CapacityError, 10: CudaError}


def raise_status(status: int, message: str):
    if status == 0:
        return
    code = load_library().mp_status_code(status).decode()
    if status in (2, 3, 4, 5, 6):
        raise NotSpdError(code, message)
    raise _ERRORS.get(status, SimError)(message or code)


def _ptr(a, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def partition_host(rest, block_size):
    """Native Morton partition (no GPU needed): subdomain_of (N,) int64."""
    lib = load_library()
    rest = np.ascontiguousarray(rest, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(len(rest), dtype=np.int64)
    raise_status(lib.mp_partition_host(_ptr(rest), len(rest), int(block_size), _ptr(out, C.c_int64)), "")
    return out


def check_intersections(positions, triangles, device=0, coplanar_tol=1e-9):
    """(number of intersecting non-adjacent triangle pairs, first triangle
    index or -1) of a surface, on the device (mp_check_intersections);
    coplanar_tol = 0 is the reference's exact-coplanarity rule."""
    lib = load_library()
    x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, dtype=np.int64).reshape(-1, 3)
    n, first = C.c_int64(), C.c_int64()
    raise_status(lib.mp_check_intersections(int(device), len(x), _ptr(x), len(t), _ptr(t, C.c_int64),
                                            float(coplanar_tol), C.byref(n), C.byref(first)),
                 "mp_check_intersections")
    return int(n.value), int(first.value)


def shard_range(n_verts, block_size, levels, coarse_block, rank, nshards):
    """Host-only mirror of a group shard's owned ranges (mp_shard_range):
    dict of (lo, hi) for vertices, subdomains, aggregates and chunks."""
    lib = load_library()
    out = np.zeros(8, np.int64)
    raise_status(lib.mp_shard_range(int(n_verts), int(block_size), int(levels), int(coarse_block), int(rank),
                                    int(nshards), _ptr(out, C.c_int64)), "mp_shard_range")
    return {"verts": (int(out[0]), int(out[1])), "subdomains": (int(out[2]), int(out[3])),
            "aggregates": (int(out[4]), int(out[5])), "chunks": (int(out[6]), int(out[7]))}


def spd_inverse(A, device=0):
    """The device coarse-level inverse (mas.py:84-90) of a dense symmetric
    matrix: (sym(A^-1), not_spd)."""
    lib = load_library()
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    out = np.empty((n, n))
    flag = C.c_int32()
    st = lib.mp_spd_inverse(int(device), n, _ptr(A), _ptr(out), C.byref(flag))
    raise_status(st, "mp_spd_inverse failed")
    return out, bool(flag.value)


class NativeContext:
    """One device context = one uploaded scene on one GPU (mp_create)."""

    def __init__(self, arrays: dict, cfg: SolverConfigC, device: int = 0):
        lib = load_library()
        self._keep = arrays  # keep host arrays alive while the descriptor is used
        a = arrays
        desc = SceneDesc(
            n_verts=len(a["mass"]), rest=_ptr(a["rest"]), mass=_ptr(a["mass"]),
            dirichlet=_ptr(a["dirichlet"], C.c_uint8), f_ext=_ptr(a["f_ext"]),
            n_tets=len(a["tets"]), tets=_ptr(a["tets"], C.c_int64), kind=_ptr(a["kind"], C.c_int8),
            mu=_ptr(a["mu"]), lam=_ptr(a["lam"]), Bm=_ptr(a["Bm"]), vol=_ptr(a["vol"]),
            n_tris=len(a["tris"]), tris=_ptr(a["tris"], C.c_int64), n_edges=len(a["edges"]),
            edges=_ptr(a["edges"], C.c_int64), n_surf_verts=len(a["surf_verts"]),
            surf_verts=_ptr(a["surf_verts"], C.c_int64), d_hat=float(a["d_hat"]), kappa=float(a["kappa"]),
        )
        h = C.c_void_p()
        if isinstance(device, (list, tuple)):  # partitioned multi-GPU group
            ids = (C.c_int * len(device))(*[int(d) for d in device])
            st = lib.mp_create_multi(C.byref(desc), C.byref(cfg), len(device), ids, C.byref(h))
        else:
            st = lib.mp_create(C.byref(desc), C.byref(cfg), int(device), C.byref(h))
        if st != 0:
            raise_status(st, lib.mp_create_error().decode())
        self.h = h
        self.lib = lib
        self.n = len(a["mass"])
        self.cfg = cfg

    def close(self):
        if getattr(self, "h", None):
            self.lib.mp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            raise_status(st, self.lib.mp_last_error(self.h).decode())

    def set_config(self, cfg: SolverConfigC):
        self._check(self.lib.mp_set_config(self.h, C.byref(cfg)))
        self.cfg = cfg

    @property
    def stream(self):
        return self.lib.mp_stream(self.h)

    @property
    def shards(self):
        return int(self.lib.mp_shards(self.h))

    @property
    def launches(self):
        return int(self.lib.mp_launch_count(self.h))

    def partition(self):
        D = C.c_int64()
        sub = np.zeros(self.n, dtype=np.int64)
        self._check(self.lib.mp_partition(self.h, C.byref(D), _ptr(sub, C.c_int64)))
        return int(D.value), sub

    def _vec(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64).ravel()
        if v.size != 3 * self.n:
            raise ConfigError(f"expected a (3N,) vector, got {v.size}")
        return v

    def _run_step(self, fn, *args, cap=None):
        cap = int(cap or max(16, self.cfg.iter_max))
        cap = min(cap, 1 << 20)
        x_out = np.empty(3 * self.n)
        v_out = np.empty(3 * self.n)
        recs = (IterRecordC * cap)()
        n = C.c_int64()
        conv = C.c_int32()
        flags = C.c_uint32()
        self._check(fn(self.h, *args, _ptr(x_out), _ptr(v_out), recs, cap, C.byref(n), C.byref(conv),
                       C.byref(flags)))
        return x_out, v_out, [recs[i] for i in range(min(n.value, cap))], bool(conv.value), int(flags.value)

    def step(self, x, v, h):
        x, v = self._vec(x), self._vec(v)
        return self._run_step(self.lib.mp_step, _ptr(x), _ptr(v), C.c_double(h))

    def advance(self, x, v, x_tilde, h):
        x, v, xt = self._vec(x), self._vec(v), self._vec(x_tilde)
        return self._run_step(self.lib.mp_advance, _ptr(x), _ptr(v), _ptr(xt), C.c_double(h))

    # ---- device-resident stepping (bench) ----
    def set_state(self, x, v):
        x, v = self._vec(x), self._vec(v)
        self._check(self.lib.mp_set_state(self.h, _ptr(x), _ptr(v)))

    def get_state(self):
        x = np.empty(3 * self.n)
        v = np.empty(3 * self.n)
        self._check(self.lib.mp_get_state(self.h, _ptr(x), _ptr(v)))
        return x, v

    def step_device(self, h, cap=None):
        cap = int(cap or max(16, self.cfg.iter_max))
        cap = min(cap, 1 << 20)
        recs = (IterRecordC * cap)()
        n = C.c_int64()
        conv = C.c_int32()
        flags = C.c_uint32()
        self._check(self.lib.mp_step_device(self.h, C.c_double(h), recs, cap, C.byref(n), C.byref(conv),
                                            C.byref(flags)))
        return [recs[i] for i in range(min(n.value, cap))], bool(conv.value), int(flags.value)

    def set_option(self, option, value):
        """MP_OPT_* of include/maspncg.h (CCD_EXACT_SET 1, RECORD_ENERGY 2, APPLY_TMA 3,
        APPLY_STAGES 4, APPLY_CTAS 5, BP_FUSED 6, KEEP_COARSE 7)."""
        self._check(self.lib.mp_set_option(self.h, int(option), int(value)))

    # ---- per-stage CUDA-event timing ----
    def stage_timing(self, enable=True):
        self._check(self.lib.mp_stage_timing(self.h, int(enable)))

    def stage_stats(self):
        """{stage: (total_ms, count, algorithmic_bytes)} since stage_timing(True)."""
        out = {}
        for i, name in enumerate(STAGES):
            ms, cnt, b = C.c_double(), C.c_int64(), C.c_double()
            self._check(self.lib.mp_stage_stats(self.h, i, C.byref(ms), C.byref(cnt), C.byref(b)))
            out[name] = (ms.value, int(cnt.value), b.value)
        return out

    # ---- stage taps ----
    def broad_phase(self, x, motion_bound, d_hat):
        x = self._vec(x)
        npt, nee = C.c_int64(), C.c_int64()
        self._check(self.lib.mp_broad_phase(self.h, _ptr(x), motion_bound, d_hat, None, 0, C.byref(npt), None, 0,
                                            C.byref(nee)))
        pt = np.zeros((npt.value, 2), np.int64)
        ee = np.zeros((nee.value, 2), np.int64)
        self._check(self.lib.mp_broad_phase(self.h, _ptr(x), motion_bound, d_hat, _ptr(pt, C.c_int64), npt.value,
                                            C.byref(npt), _ptr(ee, C.c_int64), nee.value, C.byref(nee)))
        return pt[: npt.value], ee[: nee.value]

    def constraint_set(self, x):
        x = self._vec(x)
        n = C.c_int64()
        self._check(self.lib.mp_constraint_set(self.h, _ptr(x), 0, C.byref(n), None, None, None, None, None))
        m = n.value
        verts = np.zeros((m, 4), np.int64)
        is_pt = np.zeros(m, np.uint8)
        d = np.zeros(m)
        grad = np.zeros((m, 4, 3))
        k = np.zeros(m)
        self._check(self.lib.mp_constraint_set(self.h, _ptr(x), m, C.byref(n), _ptr(verts, C.c_int64),
                                               _ptr(is_pt, C.c_uint8), _ptr(d), _ptr(grad), _ptr(k)))
        return verts, is_pt.astype(bool), d, grad, k

    def gradient(self, x, x_tilde, h):
        out = np.empty(3 * self.n)
        self._check(self.lib.mp_gradient(self.h, _ptr(self._vec(x)), _ptr(self._vec(x_tilde)), h, _ptr(out)))
        return out

    def energy(self, x, x_tilde, h):
        e = C.c_double()
        self._check(self.lib.mp_energy(self.h, _ptr(self._vec(x)), _ptr(self._vec(x_tilde)), h, C.byref(e)))
        return e.value

    def snapshot(self, x, h, build_mas=True):
        self._check(self.lib.mp_snapshot(self.h, _ptr(self._vec(x)), h, int(build_mas)))

    def hvp(self, vec, with_updates=False):
        out = np.empty(3 * self.n)
        self._check(self.lib.mp_hvp(self.h, _ptr(self._vec(vec)), int(with_updates), _ptr(out)))
        return out

    def precond_apply(self, g, with_updates=False):
        out = np.empty(3 * self.n)
        self._check(self.lib.mp_precond_apply(self.h, _ptr(self._vec(g)), int(with_updates), _ptr(out)))
        return out

    def update_at(self, x):
        nc, nt = C.c_int64(), C.c_int64()
        self._check(self.lib.mp_update_at(self.h, _ptr(self._vec(x)), C.byref(nc), C.byref(nt)))
        return nc.value, nt.value

    def ccd(self, x, p, exact_set=True):
        D, _ = self.partition()
        alpha_d = np.empty(D)
        x_new = np.empty(3 * self.n)
        ma = C.c_double()
        cert = C.c_int32()
        npairs = C.c_int64()
        self._check(self.lib.mp_ccd(self.h, _ptr(self._vec(x)), _ptr(self._vec(p)), _ptr(alpha_d), _ptr(x_new),
                                    C.byref(ma), C.byref(cert), C.byref(npairs), int(bool(exact_set))))
        return alpha_d, x_new, ma.value, bool(cert.value), npairs.value

    def set_contact(self, d_hat, kappa):
        self._check(self.lib.mp_set_contact(self.h, float(d_hat), float(kappa)))

    def coarse_matrix(self, level):
        """Assembled Galerkin matrix of coarse level `level` (1-based) of the
        last MAS build (set_option(MP_OPT_KEEP_COARSE=7, 1) before it)."""
        n = C.c_int64()
        self._check(self.lib.mp_coarse_matrix(self.h, int(level), None, 0, C.byref(n)))
        out = np.empty((n.value, n.value))
        self._check(self.lib.mp_coarse_matrix(self.h, int(level), _ptr(out), out.size, C.byref(n)))
        return out

    def ccd_pairs(self):
        """(verts (Q,4) original ids, is_pt (Q,), alpha_pair (Q,)) of the last CCD."""
        lib = self.lib
        lib.mp_ccd_pairs.argtypes = [C.c_void_p, C.c_int64, _i64p, _i64p, C.POINTER(C.c_uint8), _f64p]
        n = C.c_int64()
        self._check(lib.mp_ccd_pairs(self.h, 0, C.byref(n), None, None, None))
        m = n.value
        verts = np.zeros((m, 4), np.int64)
        is_pt = np.zeros(m, np.uint8)
        alpha = np.zeros(m)
        self._check(lib.mp_ccd_pairs(self.h, m, C.byref(n), _ptr(verts, C.c_int64), _ptr(is_pt, C.c_uint8),
                                     _ptr(alpha)))
        return verts, is_pt.astype(bool), alpha
