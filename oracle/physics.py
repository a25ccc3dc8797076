"""Oracle physics: barrier, constraint set, incremental potential, gradient,
PSD-projected Hessian snapshot and the model-Hessian product.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Reference: `pkg/src/ipcsim/contact.py` (barrier `:34-64`, constraint set
`:116-165`) and `pkg/src/ipcsim/energy.py` (elastic models `:101-290`,
objective/gradient/Hessian `:346-440`).

Representation: instead of the reference's dict of ContactPair objects the
constraint set is a struct of arrays already in the reference's key order
(`contact.py:98-113`: all ("ee", (a0,a1), (b0,b1)) keys, then all
("pt", v, (t0,t1,t2)) keys, each lexicographic), plus a dict from key tuple
to row for the classification lookup.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import geometry as ogeo

KIND_ARAP = 1
KIND_SNH = 2


class PenetrationError(Exception):
    code = "penetration-detected"


class NotSpdError(Exception):
    def __init__(self, code, msg=""):
        super().__init__(msg or code)
        self.code = code


# ---------------------------------------------------------------------------
# barrier  (contact.py:34-64)


def barrier(d, d_hat, kappa):
    """kappa * (b, b', b'') for distances d; zero outside (0, d_hat)."""
    d = np.asarray(d, float)
    if np.any(d <= 0.0):
        raise PenetrationError("contact distance <= 0")
    inside = d < d_hat
    t = d - d_hat
    ln = np.log(np.where(inside, d / d_hat, 1.0))
    b = np.where(inside, -t * t * ln, 0.0)
    b1 = np.where(inside, -2.0 * t * ln - t * t / d, 0.0)
    b2 = np.where(inside, -2.0 * ln - 4.0 * t / d + t * t / (d * d), 0.0)
    return kappa * b, kappa * b1, kappa * b2


def barrier_hess_scalar(d, d_hat, kappa):
    """kappa * b''(d) for one active pair, as `_make_pair` computes it
    (`contact.py:168-175` via `barrier_derivatives` `:34-49`)."""
    t = d - d_hat
    ln = math.log(d / d_hat)
    return kappa * (-2.0 * ln - 4.0 * t / d + t * t / (d * d))


# ---------------------------------------------------------------------------
# constraint set  (contact.py:116-165)


@dataclass
class Contacts:
    """Active pairs at one iterate, rows in reference key order."""

    verts: np.ndarray  # (C,4) canonical vertex ids
    is_pt: np.ndarray  # (C,)
    d: np.ndarray
    grad: np.ndarray  # (C,4,3) pinned rows zeroed
    n: np.ndarray  # (C,4,3) grad / |grad| (0 when |grad| <= 1e-12)
    k: np.ndarray  # kappa b''(d)
    index: dict = field(default_factory=dict)  # key tuple -> row

    def __len__(self):
        return len(self.d)


def _empty_contacts():
    return Contacts(np.zeros((0, 4), np.int64), np.zeros(0, bool), np.zeros(0), np.zeros((0, 4, 3)),
                    np.zeros((0, 4, 3)), np.zeros(0), {})


def constraint_set(scene, x):
    x3 = np.asarray(x, float).reshape(-1, 3)
    pt, ee = ogeo.broad_phase(x3, scene.tris, scene.edges, scene.surf_verts, 0.0, scene.d_hat)
    rows = []  # (verts, is_pt, d, grad)
    if len(ee):
        ea, eb = scene.edges[ee[:, 0]], scene.edges[ee[:, 1]]
        d, g = ogeo.ee_distance_batch(x3[ea[:, 0]], x3[ea[:, 1]], x3[eb[:, 0]], x3[eb[:, 1]])
        if np.any(d <= 0.0):
            raise PenetrationError("edge-edge distance <= 0")
        s = d < scene.d_hat
        rows.append((np.concatenate([ea[s], eb[s]], axis=1), np.zeros(s.sum(), bool), d[s], g[s]))
    if len(pt):
        v = pt[:, 0]
        ts = np.sort(scene.tris[pt[:, 1]], axis=1)
        d, g = ogeo.pt_distance_batch(x3[v], x3[ts[:, 0]], x3[ts[:, 1]], x3[ts[:, 2]])
        if np.any(d <= 0.0):
            raise PenetrationError("point-triangle distance <= 0")
        s = d < scene.d_hat
        rows.append((np.concatenate([v[s, None], ts[s]], axis=1), np.ones(s.sum(), bool), d[s], g[s]))
    if not rows or sum(len(r[2]) for r in rows) == 0:
        return _empty_contacts()
    verts = np.concatenate([r[0] for r in rows]).astype(np.int64)
    is_pt = np.concatenate([r[1] for r in rows])
    d = np.concatenate([r[2] for r in rows])
    grad = np.concatenate([r[3] for r in rows])
    # key order: EE block before PT block, lexicographic inside each block
    order = np.lexsort((verts[:, 3], verts[:, 2], verts[:, 1], verts[:, 0], is_pt))
    verts, is_pt, d, grad = verts[order], is_pt[order], d[order], grad[order]
    grad = grad.copy()
    grad[scene.dirichlet[verts]] = 0.0
    nrm = np.array([np.linalg.norm(gr) for gr in grad])
    n = np.where(nrm[:, None, None] > 1e-12, grad / np.where(nrm > 1e-12, nrm, 1.0)[:, None, None], 0.0)
    k = np.array([barrier_hess_scalar(float(di), scene.d_hat, scene.kappa) for di in d])
    index = {_key(vv, ip): r for r, (vv, ip) in enumerate(zip(verts.tolist(), is_pt.tolist()))}
    return Contacts(verts, is_pt, d, grad, n, k, index)


def _key(v, is_pt):
    return ("pt", v[0], tuple(v[1:])) if is_pt else ("ee", tuple(v[:2]), tuple(v[2:]))


# ---------------------------------------------------------------------------
# elastic models  (energy.py:101-290)


def _bcoef(Bm):
    """(T,4,3): rows dF/dx_m -- vertex 0 = -sum of Bm rows, vertices 1..3 =
    Bm rows (the coefficients of the reference's G, `energy.py:151-162`)."""
    out = np.empty((len(Bm), 4, 3))
    out[:, 1:] = Bm
    out[:, 0] = -Bm.sum(axis=1)
    return out


def deformation_gradients(scene, x):
    xv = np.asarray(x, float).reshape(-1, 3)[scene.tets]
    Ds = np.stack([xv[:, 1] - xv[:, 0], xv[:, 2] - xv[:, 0], xv[:, 3] - xv[:, 0]], axis=2)
    return Ds @ scene.Bm


def signed_svd(F):
    """SVD with a reflection folded into the smallest singular value
    (`energy.py:184-191`)."""
    U, S, Vt = np.linalg.svd(F)
    S = S.copy()
    refl = np.linalg.det(U @ Vt) < 0
    U[refl, :, 2] = -U[refl, :, 2]
    S[refl, 2] = -S[refl, 2]
    return U, S, Vt


def cofactor(F):
    """Columns are crosses of the other two columns (`energy.py:230-235`)."""
    return np.stack([np.cross(F[:, :, 1], F[:, :, 2]), np.cross(F[:, :, 2], F[:, :, 0]),
                     np.cross(F[:, :, 0], F[:, :, 1])], axis=2)


def _psi(F, mu, lam, kind):
    psi = np.zeros(len(F))
    a = kind == KIND_ARAP
    if a.any():
        _, S, _ = signed_svd(F[a])
        psi[a] = 0.5 * mu[a] * ((S - 1.0) ** 2).sum(axis=1)
    s = kind == KIND_SNH
    if s.any():
        Fs = F[s]
        J = np.linalg.det(Fs)
        I2 = (Fs * Fs).sum(axis=(1, 2))
        psi[s] = 0.5 * mu[s] * (I2 - 3.0) - mu[s] * (J - 1.0) + 0.5 * lam[s] * (J - 1.0) ** 2
    return psi


def _piola(F, mu, lam, kind):
    P = np.zeros_like(F)
    a = kind == KIND_ARAP
    if a.any():
        U, _, Vt = signed_svd(F[a])
        P[a] = mu[a, None, None] * (F[a] - U @ Vt)
    s = kind == KIND_SNH
    if s.any():
        Fs = F[s]
        J = np.linalg.det(Fs)
        P[s] = mu[s, None, None] * Fs + (lam[s] * (J - 1.0) - mu[s])[:, None, None] * cofactor(Fs)
    return P


_EPS3 = np.zeros((3, 3, 3))
for _i, _j, _k in ((0, 1, 2), (1, 2, 0), (2, 0, 1)):
    _EPS3[_i, _j, _k] = 1.0
    _EPS3[_i, _k, _j] = -1.0


def _hess9(F, mu, lam, kind):
    """(T,9,9) d2 Psi / dvec(F)^2, row-major vec, PSD: ARAP analytically
    projected (`energy.py:208-224`), SNH eigen-clamped (`:262-290`)."""
    T = len(F)
    H = np.zeros((T, 9, 9))
    a = np.nonzero(kind == KIND_ARAP)[0]
    if len(a):
        U, S, Vt = signed_svd(F[a])
        m = mu[a]
        Ha = m[:, None, None] * np.eye(9)[None]
        for i, j in ((0, 1), (1, 2), (0, 2)):
            den = S[:, i] + S[:, j]
            den = np.where(np.abs(den) < 1e-8, np.copysign(1e-8, den + 1e-300), den)
            ev = np.maximum(m * (1.0 - 2.0 / den), 0.0)
            # twist mode U (e_i e_j^T - e_j e_i^T) V^T / sqrt(2)
            Q = (np.einsum("tr,tc->trc", U[:, :, i], Vt[:, j, :]) - np.einsum("tr,tc->trc", U[:, :, j], Vt[:, i, :]))
            q = Q.reshape(len(a), 9) / math.sqrt(2.0)
            Ha += (ev - m)[:, None, None] * q[:, :, None] * q[:, None, :]
        H[a] = Ha
    s = np.nonzero(kind == KIND_SNH)[0]
    if len(s):
        Fs = F[s]
        J = np.linalg.det(Fs)
        g = cofactor(Fs).reshape(len(s), 9)
        # d2 det / dF_ab dF_cd = eps_ace eps_bdf F_ef
        Hdet = np.einsum("ace,bdf,tef->tabcd", _EPS3, _EPS3, Fs).reshape(len(s), 9, 9)
        Hs = mu[s, None, None] * np.eye(9)[None] + lam[s, None, None] * g[:, :, None] * g[:, None, :]
        Hs += (lam[s] * (J - 1.0) - mu[s])[:, None, None] * Hdet
        w, Q = np.linalg.eigh(Hs)
        H[s] = np.einsum("tak,tk,tbk->tab", Q, np.maximum(w, 0.0), Q)
    return H


# ---------------------------------------------------------------------------
# objective, gradient, Hessian  (energy.py:346-440)


def incremental_potential(scene, x, x_tilde, h, cs):
    dx = x - x_tilde
    e = 0.5 * float(dx @ (scene.mass3 * dx))
    if len(scene.vol):
        F = deformation_gradients(scene, x)
        e += h * h * float((scene.vol * _psi(F, scene.mu, scene.lam, scene.kind)).sum())
    if len(cs):
        e += float(barrier(cs.d, scene.d_hat, scene.kappa)[0].sum())
    return e


def _scatter12(scene, verts, vals12, out):
    dof = (3 * verts[:, :, None] + np.arange(3)).reshape(-1)
    out += np.bincount(dof, weights=vals12.reshape(-1), minlength=len(out))


def gradient(scene, x, x_tilde, h, cs):
    g = scene.mass3 * (x - x_tilde)
    if len(scene.vol):
        F = deformation_gradients(scene, x)
        P = _piola(F, scene.mu, scene.lam, scene.kind)
        ge = scene.vol[:, None, None] * (_bcoef(scene.Bm) @ np.transpose(P, (0, 2, 1)))  # (T,4,3)
        el = np.zeros_like(g)
        _scatter12(scene, scene.tets, ge, el)
        g += h * h * el
    if len(cs):
        db = barrier(cs.d, scene.d_hat, scene.kappa)[1]
        _scatter12(scene, cs.verts, db[:, None, None] * cs.grad, g)
    g[scene.pinned3] = 0.0
    return g


def element_hessians(scene, x):
    """(T,12,12) vol * G^T H9 G, no h^2 (`energy.py:328-339`)."""
    F = deformation_gradients(scene, x)
    H9 = _hess9(F, scene.mu, scene.lam, scene.kind).reshape(-1, 3, 3, 3, 3)
    bc = _bcoef(scene.Bm)
    H12 = np.einsum("tmj,tijkl,tnl->tmink", bc, H9, bc).reshape(-1, 12, 12)
    return scene.vol[:, None, None] * H12


def assemble_base_hessian(scene, x, h, cs):
    """CSR H = M + h^2 sum H_e + sum k g g^T, pinned rows/cols -> identity
    (`energy.py:373-413`)."""
    n = 3 * scene.n
    r_l, c_l, v_l = [], [], []

    def add(verts, blocks):
        idx = (3 * verts[:, :, None] + np.arange(3)).reshape(len(verts), 12)
        r_l.append(np.repeat(idx, 12, axis=1).ravel())
        c_l.append(np.tile(idx, (1, 12)).ravel())
        v_l.append(blocks.reshape(-1))

    if len(scene.vol):
        add(scene.tets, h * h * element_hessians(scene, x))
    if len(cs):
        u = cs.grad.reshape(len(cs), 12)
        add(cs.verts, cs.k[:, None, None] * u[:, :, None] * u[:, None, :])
    pin = scene.pinned3
    if r_l:
        r, c, v = np.concatenate(r_l), np.concatenate(c_l), np.concatenate(v_l)
        keep = ~(pin[r] | pin[c])
        H = sp.coo_matrix((v[keep], (r[keep], c[keep])), shape=(n, n))
    else:
        H = sp.coo_matrix((n, n))
    return (H + sp.diags(np.where(pin, 1.0, scene.mass3))).tocsr()


def hvp(H, cand_verts, cand_u, vec):
    """H_base v + sum_c u_c (u_c . v) (`energy.py:435-440`)."""
    out = H @ vec
    if len(cand_u):
        idx = (3 * cand_verts[:, :, None] + np.arange(3)).reshape(len(cand_u), 12)
        u = cand_u.reshape(len(cand_u), 12)
        dots = (u * vec[idx]).sum(axis=1)
        out += np.bincount(idx.ravel(), weights=(u * dots[:, None]).ravel(), minlength=len(out))
    return out
