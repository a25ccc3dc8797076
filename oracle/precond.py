"""Oracle preconditioner: Morton partition, MAS hierarchy + apply, contact
classification, per-subdomain top-K and the Sparse-Input Woodbury update.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Reference: `pkg/src/ipcsim/mas.py` (partition `:30-77`, hierarchy
`:84-179`, apply `:182-205`), `pkg/src/ipcsim/contact.py` (classification
`:182-214`, top-K `:217-233`), `pkg/src/ipcsim/woodbury.py:46-87`.

Level-0 blocks are gathered from the COO triplets of H in one vectorised
pass and inverted as one batch (upper-triangular Cholesky, triangular
inverse, then B = R^-1 R^-T, symmetrised), instead of the reference's
per-subdomain CSR slicing + cho_solve; the math is the same.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from .physics import NotSpdError


# ---------------------------------------------------------------------------
# partition  (mas.py:30-77)


def _spread3(v):
    v = v.astype(np.uint64)
    for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                        (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def morton_codes(points, bits=10):
    lo = points.min(axis=0)
    ext = points.max(axis=0) - lo
    ext[ext == 0.0] = 1.0
    q = ((points - lo) / ext * (2 ** bits - 1)).astype(np.uint64)
    return _spread3(q[:, 0]) | (_spread3(q[:, 1]) << np.uint64(1)) | (_spread3(q[:, 2]) << np.uint64(2))


@dataclass
class Partition:
    subdomain_of: np.ndarray  # (N,)
    selection: list  # sorted vertex ids per subdomain
    D: int


def partition_domain(rest, block_size):
    order = np.argsort(morton_codes(np.asarray(rest, float)), kind="stable")
    n = len(order)
    D = max(1, math.ceil(n / block_size))
    sel = [np.sort(order[d * block_size:(d + 1) * block_size]) for d in range(D)]
    sub = np.empty(n, np.int64)
    for d, vs in enumerate(sel):
        sub[vs] = d
    return Partition(sub, sel, D)


# ---------------------------------------------------------------------------
# MAS hierarchy  (mas.py:84-179)


@dataclass
class Hierarchy:
    part: Partition
    dof_rows: np.ndarray  # (D, m) global dof of each block row (-1 = padding)
    B: np.ndarray  # (D, m, m) level-0 inverses (identity on padding)
    coarsen: list  # C_l (3A_l x 3N) csr
    coarse_inv: list  # dense (3A_l)^2


def _spd_inverse_batch(A, code):
    """sym(A^-1) per batch entry through the Cholesky factor."""
    try:
        L = np.linalg.cholesky(A)
    except np.linalg.LinAlgError as e:
        raise NotSpdError(code, str(e)) from e
    Li = np.linalg.inv(L)
    inv = np.transpose(Li, (0, 2, 1)) @ Li
    return 0.5 * (inv + np.transpose(inv, (0, 2, 1)))


def _spd_inverse(A, code):
    try:
        c = scipy.linalg.cho_factor(A)
    except scipy.linalg.LinAlgError as e:
        raise NotSpdError(code, str(e)) from e
    inv = scipy.linalg.cho_solve(c, np.eye(len(A)))
    return 0.5 * (inv + inv.T)


def build_hierarchy(H, part: Partition, levels=2, coarse_block=4):
    n = H.shape[0]
    nv = n // 3
    m = 3 * max(len(s) for s in part.selection)
    D = part.D
    # dof -> (subdomain, local row)
    local = np.empty(nv, np.int64)
    dof_rows = -np.ones((D, m), np.int64)
    for d, vs in enumerate(part.selection):
        local[vs] = np.arange(len(vs))
        dof_rows[d, :3 * len(vs)] = (3 * vs[:, None] + np.arange(3)).ravel()
    Hc = H.tocoo()
    r, c, v = Hc.row, Hc.col, Hc.data
    sr, sc = part.subdomain_of[r // 3], part.subdomain_of[c // 3]
    same = sr == sc
    r, c, v, sr = r[same], c[same], v[same], sr[same]
    lr = 3 * local[r // 3] + r % 3
    lc = 3 * local[c // 3] + c % 3
    A = np.zeros((D, m, m))
    np.add.at(A, (sr, lr, lc), v)
    pad = dof_rows < 0
    dd, ii = np.nonzero(pad)
    A[dd, ii, ii] = 1.0
    B = _spd_inverse_batch(A, "non-spd-subdomain")
    coarsen, coarse_inv = [], []
    units = list(part.selection)
    for _ in range(levels):
        A_l = math.ceil(len(units) / coarse_block)
        if A_l == len(units):
            break
        groups = [np.concatenate(units[a * coarse_block:(a + 1) * coarse_block]) for a in range(A_l)]
        rows = np.concatenate([np.repeat(3 * a + np.arange(3), len(g)) for a, g in enumerate(groups)])
        cols = np.concatenate([(3 * g[None, :] + np.arange(3)[:, None]).ravel() for g in groups])
        vals = np.concatenate([np.full(3 * len(g), 1.0 / len(g)) for g in groups])
        C = sp.csr_matrix((vals, (rows, cols)), shape=(3 * A_l, n))
        M = (C @ H @ C.T).toarray()
        coarse_inv.append(_spd_inverse(0.5 * (M + M.T), "non-spd-subdomain"))
        coarsen.append(C)
        units = groups
    return Hierarchy(part, dof_rows, B, coarsen, coarse_inv)


def block_rows(hier, g):
    """g gathered into (D, m) block order, zero on padding."""
    gg = np.where(hier.dof_rows >= 0, g[np.maximum(hier.dof_rows, 0)], 0.0)
    return gg


def apply_preconditioner(hier: Hierarchy, wb, g):
    """z = sum_d Btilde_d g_d + sum_l C_l^T Minv_l C_l g (`mas.py:182-205`);
    wb maps subdomain -> WoodburyBlock (or is None)."""
    gb = block_rows(hier, g)
    zb = np.einsum("dab,db->da", hier.B, gb)
    if wb:
        for d, blk in wb.items():
            zb[d] = woodbury_apply(hier.B[d], blk, gb[d])
    z = np.zeros_like(g)
    ok = hier.dof_rows >= 0
    z[hier.dof_rows[ok]] += zb[ok]
    for C, Minv in zip(hier.coarsen, hier.coarse_inv):
        z += C.T @ (Minv @ (C @ g))
    return z


# ---------------------------------------------------------------------------
# classification + top-K  (contact.py:182-233)


@dataclass
class Candidates:
    verts: np.ndarray  # (n,4)
    u: np.ndarray  # (n,4,3)
    delta_s: np.ndarray  # (n,)

    def __len__(self):
        return len(self.delta_s)


def classify_all(cur, base, eps_rot):
    """One rank-one candidate per current pair, in key order."""
    keep_v, keep_u, keep_s = [], [], []
    for r in range(len(cur)):
        g = cur.grad[r]
        if np.linalg.norm(g) <= 1e-12:
            continue
        k = float(cur.k[r])
        key = ("pt", int(cur.verts[r, 0]), tuple(int(t) for t in cur.verts[r, 1:])) if cur.is_pt[r] else \
            ("ee", tuple(int(t) for t in cur.verts[r, :2]), tuple(int(t) for t in cur.verts[r, 2:]))
        b = base.index.get(key)
        if b is not None and float((cur.n[r] * base.n[b]).sum()) >= eps_rot:
            delta = k - float(base.k[b])
            if delta <= 0.0:
                continue
            keep_u.append(math.sqrt(delta) * g)
            keep_s.append(delta)
        else:
            keep_u.append(math.sqrt(k) * g)
            keep_s.append(k)
        keep_v.append(cur.verts[r])
    if not keep_s:
        return Candidates(np.zeros((0, 4), np.int64), np.zeros((0, 4, 3)), np.zeros(0))
    return Candidates(np.array(keep_v), np.array(keep_u), np.array(keep_s))


def select_top_k(cands: Candidates, subdomain_of, K):
    """subdomain -> candidate rows ordered by (-delta_s, key), <= K each.
    A candidate belongs to every subdomain owning a vertex whose u-row is
    non-zero."""
    if len(cands) == 0:
        return {}
    nz = np.any(cands.u != 0.0, axis=2)  # (n,4)
    own = np.where(nz, subdomain_of[cands.verts], -1)
    ci, sub = [], []
    for c in range(len(cands)):
        for d in sorted(set(own[c][own[c] >= 0].tolist())):
            ci.append(c)
            sub.append(d)
    ci, sub = np.array(ci, np.int64), np.array(sub, np.int64)
    order = np.lexsort((ci, -cands.delta_s[ci], sub))  # candidate index = key order
    ci, sub = ci[order], sub[order]
    out = {}
    for d in np.unique(sub):
        out[int(d)] = ci[sub == d][:K]
    return out


# ---------------------------------------------------------------------------
# Sparse-Input Woodbury  (woodbury.py:46-87)


@dataclass
class WoodburyBlock:
    U: np.ndarray
    W: np.ndarray
    cap_chol: tuple


def build_update(hier: Hierarchy, cands: Candidates, topk, K):
    out = {}
    for d in sorted(topk):
        rows = topk[d][:K]
        if len(rows) == 0:
            continue
        dofs = hier.dof_rows[d]
        m = hier.B.shape[1]
        U = np.zeros((m, len(rows)))
        pos_of = {int(g): i for i, g in enumerate(dofs) if g >= 0}
        for col, c in enumerate(rows):
            gd = (3 * cands.verts[c][:, None] + np.arange(3)).ravel()
            uu = cands.u[c].ravel()
            for j, gdof in enumerate(gd):
                i = pos_of.get(int(gdof))
                if i is not None:
                    U[i, col] = uu[j]
        W = hier.B[d] @ U
        cap = np.eye(len(rows)) + U.T @ W
        cap = 0.5 * (cap + cap.T)
        try:
            ch = scipy.linalg.cho_factor(cap)
        except scipy.linalg.LinAlgError as e:
            raise NotSpdError("capacitance-not-spd", str(e)) from e
        out[d] = WoodburyBlock(U, W, ch)
    return out


def woodbury_apply(B_d, blk: WoodburyBlock, g_d):
    z = B_d @ g_d
    lam = scipy.linalg.cho_solve(blk.cap_chol, blk.U.T @ z)
    return z - blk.W @ lam
