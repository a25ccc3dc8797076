"""Oracle geometry: batched PT/EE distances and the exact broad-phase set.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Distances restate `pkg/src/ipcsim/geometry.py:209-323` with the same IEEE
expression order, so distances are bit-identical to the reference's.

The broad phase restates the *membership rule* of
`geometry.py:443-503`: a pair is returned iff

  1. the reference's uniform hash grid reaches it -- the query box's cell
     range overlaps the inserted box's cell range on every axis (cell =
     max(largest primitive-box diagonal, d_hat + mb), boxes padded by
     d_hat/2 + mb; `geometry.py:417-440, 465-475`), and
  2. it passes the AABB gap filter (gap = d_hat + 2 mb): PT keeps
     v not in tri and tri_lo - gap <= p_v <= tri_hi + gap componentwise
     (`:478-487`); EE keeps i < j, no shared vertex, lo_i <= hi_j + gap and
     lo_j <= hi_i + gap (`:489-499`).

Enumerating pairs through the reference's own grid is O(V F) when one
primitive is large (a floor slab makes the cell as big as the scene), so
the oracle enumerates a superset of rule 2 through a fine auxiliary grid
(oversized primitives are tested against everything) and then applies
rules 1 and 2 exactly.  The output equals the reference's sorted unique
arrays bit for bit.
"""

from __future__ import annotations

import numpy as np


def _dot(a, b):
    return (a * b).sum(1)


def pt_distance_batch(p, t0, t1, t2):
    """Point-triangle distance + raw stacked gradient (m,4,3)
    (`geometry.py:209-284`): Voronoi-region classification in the order
    vertex A, vertex B, vertex C, edge AB, edge AC, edge BC, interior."""
    ab, ac = t1 - t0, t2 - t0
    ap, bp, cp = p - t0, p - t1, p - t2
    d1, d2 = _dot(ab, ap), _dot(ac, ap)
    d3, d4 = _dot(ab, bp), _dot(ac, bp)
    d5, d6 = _dot(ab, cp), _dot(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    m = len(p)
    region = np.full(m, 6, dtype=np.int8)  # 6 = interior
    conds = [
        (d1 <= 0.0) & (d2 <= 0.0),
        (d3 >= 0.0) & (d4 <= d3),
        (d6 >= 0.0) & (d5 <= d6),
        (vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0),
        (vb <= 0.0) & (d2 >= 0.0) & (d6 <= 0.0),
        (va <= 0.0) & ((d4 - d3) >= 0.0) & ((d5 - d6) >= 0.0),
    ]
    for r in range(5, -1, -1):  # first matching region wins
        region[conds[r]] = r
    w = np.zeros((m, 3))
    w[region == 0, 0] = 1.0
    w[region == 1, 1] = 1.0
    w[region == 2, 2] = 1.0
    with np.errstate(divide="ignore", invalid="ignore"):
        s = region == 3
        v = d1[s] / (d1[s] - d3[s])
        w[s, 0], w[s, 1] = 1.0 - v, v
        s = region == 4
        v = d2[s] / (d2[s] - d6[s])
        w[s, 0], w[s, 2] = 1.0 - v, v
        s = region == 5
        num = d4[s] - d3[s]
        v = num / (num + (d5[s] - d6[s]))
        w[s, 1], w[s, 2] = 1.0 - v, v
        s = region == 6
        den = va[s] + vb[s] + vc[s]
        bv, bw = vb[s] / den, vc[s] / den
        w[s, 0], w[s, 1], w[s, 2] = 1.0 - bv - bw, bv, bw
    diff = p - (w[:, 0:1] * t0 + w[:, 1:2] * t1 + w[:, 2:3] * t2)
    d = np.sqrt(_dot(diff, diff))
    u = np.zeros_like(diff)
    pos = d > 0.0
    u[pos] = diff[pos] / d[pos, None]
    grad = np.empty((m, 4, 3))
    grad[:, 0] = u
    for k in range(3):
        grad[:, k + 1] = -w[:, k:k + 1] * u
    return d, grad


def ee_distance_batch(a0, a1, b0, b1):
    """Clamped segment-segment distance + raw stacked gradient
    (`geometry.py:287-323`)."""
    da, db, r = a1 - a0, b1 - b0, a0 - b0
    a, e = _dot(da, da), _dot(db, db)
    f, c, b = _dot(db, r), _dot(da, r), _dot(da, db)
    den = a * e - b * b
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(den > 0.0, np.clip((b * f - c * e) / np.where(den > 0, den, 1.0), 0.0, 1.0), 0.0)
        t = (b * s + f) / e
        below, above = t < 0.0, t > 1.0
        t = np.clip(t, 0.0, 1.0)
        s = np.where(below, np.clip(-c / a, 0.0, 1.0), s)
        s = np.where(above, np.clip((b - c) / a, 0.0, 1.0), s)
    diff = (a0 + s[:, None] * da) - (b0 + t[:, None] * db)
    d = np.sqrt(_dot(diff, diff))
    u = np.zeros_like(diff)
    pos = d > 0.0
    u[pos] = diff[pos] / d[pos, None]
    grad = np.empty((len(a0), 4, 3))
    grad[:, 0] = (1.0 - s)[:, None] * u
    grad[:, 1] = s[:, None] * u
    grad[:, 2] = -(1.0 - t)[:, None] * u
    grad[:, 3] = -t[:, None] * u
    return d, grad


# ---------------------------------------------------------------------------
# candidate enumeration helpers


def _ranges(starts, counts):
    """Concatenation of arange(s, s+c) for every (s, c)."""
    counts = np.asarray(counts, np.int64)
    tot = int(counts.sum())
    if tot == 0:
        return np.zeros(0, np.int64)
    ends = np.cumsum(counts)
    base = np.repeat(np.asarray(starts, np.int64) - (ends - counts), counts)
    return base + np.arange(tot, dtype=np.int64)


class _FineGrid:
    """Auxiliary uniform grid for enumerating box-overlap supersets."""

    MAX_CELLS = 64

    def __init__(self, lo, hi):
        ext = hi - lo
        size = np.median(ext.max(axis=1)) if len(ext) else 1.0
        self.h = max(float(size), 1e-12) * 1.5
        self.origin = lo.min(axis=0) if len(lo) else np.zeros(3)

    def cells(self, lo, hi):
        c0 = np.floor((lo - self.origin) / self.h).astype(np.int64)
        c1 = np.floor((hi - self.origin) / self.h).astype(np.int64)
        return c0, c1

    def entries(self, lo, hi):
        """(cell keys, prim ids) of boxes within MAX_CELLS cells; the ids of
        oversized boxes separately."""
        c0, c1 = self.cells(lo, hi)
        span = c1 - c0 + 1
        n = span.prod(axis=1)
        small = n <= self.MAX_CELLS
        big = np.nonzero(~small)[0]
        ids = np.nonzero(small)[0]
        cnt = n[ids]
        prim = np.repeat(ids, cnt)
        off = _ranges(np.zeros(len(ids), np.int64), cnt)
        sp = span[prim]
        i = c0[prim, 0] + off % sp[:, 0]
        j = c0[prim, 1] + (off // sp[:, 0]) % sp[:, 1]
        k = c0[prim, 2] + off // (sp[:, 0] * sp[:, 1])
        return self.key(i, j, k), prim, big

    @staticmethod
    def key(i, j, k):
        # cell indices are >= -1 relative to the grid origin and far below 2^20
        return ((i + 1) << 42) | ((j + 1) << 21) | (k + 1)


def _ref_cells(lo, hi, cell):
    """The reference hash grid's inclusive cell range (`geometry.py:421-423`)."""
    return np.floor(lo / cell).astype(np.int64), np.floor(hi / cell).astype(np.int64)


_CHUNK = 1 << 23  # candidate pairs per filtering pass (bounded memory)


def _chunks(per):
    """[start, stop) item ranges whose summed candidate counts stay near
    _CHUNK (at least one item each)."""
    cum = np.cumsum(per)
    start, n = 0, len(per)
    while start < n:
        base = cum[start - 1] if start else 0
        stop = max(int(np.searchsorted(cum, base + _CHUNK, "right")), start + 1)
        yield start, min(stop, n)
        start = stop


def _ee_filter(a, b, edges, e_lo, e_hi, gap, pad, cell):
    i, j = np.minimum(a, b), np.maximum(a, b)
    sel = i < j
    i, j = i[sel], j[sel]
    ei, ej = edges[i], edges[j]
    ok = ~np.any(ej[:, :, None] == ei[:, None, :], axis=(1, 2))
    ok &= np.all(e_lo[i] <= e_hi[j] + gap, axis=1) & np.all(e_lo[j] <= e_hi[i] + gap, axis=1)
    i, j = i[ok], j[ok]
    q0, q1 = _ref_cells(e_lo[i] - pad, e_hi[i] + pad, cell)
    i0, i1 = _ref_cells(e_lo[j] - pad, e_hi[j] + pad, cell)
    ok = np.all((q0 <= i1) & (i0 <= q1), axis=1)
    return np.stack([i[ok], j[ok]], axis=1).astype(np.int64)


def broad_phase(x, tris, edges, surf_verts, motion_bound, d_hat):
    """Sorted unique (v, tri) and (edge i, edge j) candidate pairs, exactly
    the reference's `broad_phase` output (`geometry.py:443-503`)."""
    x = np.asarray(x, float).reshape(-1, 3)
    empty = np.zeros((0, 2), np.int64)
    if len(tris) == 0:
        return empty, empty
    tp = x[tris]
    tri_lo, tri_hi = tp.min(axis=1), tp.max(axis=1)
    ep = x[edges]
    e_lo, e_hi = ep.min(axis=1), ep.max(axis=1)
    diag = np.linalg.norm(tri_hi - tri_lo, axis=1)
    if len(edges):
        diag = np.concatenate([diag, np.linalg.norm(e_hi - e_lo, axis=1)])
    cell = max(float(diag.max()), d_hat + motion_bound)
    pad = 0.5 * d_hat + motion_bound
    gap = d_hat + 2.0 * motion_bound

    # ---- point-triangle ----
    pv = x[surf_verts]
    fg = _FineGrid(tri_lo - gap, tri_hi + gap)
    keys, prim, big = fg.entries(tri_lo - gap, tri_hi + gap)
    order = np.argsort(keys, kind="stable")
    keys, prim = keys[order], prim[order]
    c0, _ = fg.cells(pv, pv)
    vkey = fg.key(c0[:, 0], c0[:, 1], c0[:, 2])
    lo_i = np.searchsorted(keys, vkey, "left")
    hi_i = np.searchsorted(keys, vkey, "right")
    cnt = hi_i - lo_i
    bigc = len(big)
    out = []
    for start, stop in _chunks(cnt + bigc):  # bounded-memory query batches
        qs = np.arange(start, stop)
        qi = np.repeat(qs, cnt[qs])
        ti = prim[_ranges(lo_i[qs], cnt[qs])]
        if bigc:
            qi = np.concatenate([qi, np.repeat(qs, bigc)])
            ti = np.concatenate([ti, np.tile(big, len(qs))])
        v = surf_verts[qi]
        p = x[v]
        ok = ~np.any(tris[ti] == v[:, None], axis=1)
        ok &= np.all(p >= tri_lo[ti] - gap, axis=1) & np.all(p <= tri_hi[ti] + gap, axis=1)
        v, ti, p = v[ok], ti[ok], p[ok]
        q0, q1 = _ref_cells(p - pad, p + pad, cell)
        i0, i1 = _ref_cells(tri_lo[ti] - pad, tri_hi[ti] + pad, cell)
        ok = np.all((q0 <= i1) & (i0 <= q1), axis=1)
        out.append(np.stack([v[ok], ti[ok]], axis=1).astype(np.int64))
    pt = np.unique(np.concatenate(out), axis=0) if out else np.zeros((0, 2), np.int64)

    # ---- edge-edge ----
    E = len(edges)
    if E < 2:
        return pt.reshape(-1, 2), empty
    blo, bhi = e_lo, e_hi + gap  # boxes overlap <=> the two gap inequalities
    fg = _FineGrid(blo, bhi)
    keys, prim, big = fg.entries(blo, bhi)
    order = np.lexsort((prim, keys))
    keys, prim = keys[order], prim[order]
    starts = np.flatnonzero(np.r_[True, keys[1:] != keys[:-1]])
    gsize = np.diff(np.r_[starts, len(keys)])
    pos = np.arange(len(keys))
    later = np.repeat(starts + gsize, gsize) - pos - 1  # partners after this entry in its cell
    out = []
    for start, stop in _chunks(later):
        es = np.arange(start, stop)
        a = np.repeat(prim[es], later[es])
        b = prim[_ranges(es + 1, later[es])]
        out.append(_ee_filter(a, b, edges, e_lo, e_hi, gap, pad, cell))
    for start, stop in _chunks(np.full(len(big), E)):  # oversized edges vs all
        bb = big[start:stop]
        out.append(_ee_filter(np.repeat(bb, E), np.tile(np.arange(E), len(bb)), edges, e_lo, e_hi, gap, pad,
                              cell))
    ee = np.unique(np.concatenate(out), axis=0) if out else np.zeros((0, 2), np.int64)
    return pt.reshape(-1, 2), ee.reshape(-1, 2)


# ---------------------------------------------------------------------------
# triangle-triangle intersection (`geometry.py:654-732`): the reference's
# decision rules, one pair at a time (test-size inputs only)


def _seg_seg_2d(p0, p1, q0, q1):
    d1, d2, r = p1 - p0, q1 - q0, q0 - p0
    den = d1[0] * d2[1] - d1[1] * d2[0]
    if den == 0.0:
        if r[0] * d1[1] - r[1] * d1[0] != 0.0:
            return False
        tt = d1 @ d1
        if tt == 0.0:
            return False
        t0 = (r @ d1) / tt
        t1 = t0 + (d2 @ d1) / tt
        return max(min(t0, t1), 0.0) <= min(max(t0, t1), 1.0)
    s = (r[0] * d2[1] - r[1] * d2[0]) / den
    t = (r[0] * d1[1] - r[1] * d1[0]) / den
    return 0.0 <= s <= 1.0 and 0.0 <= t <= 1.0


def _in_tri_2d(p, a, b, c):
    s = [(b[0] - a[0]) * (p[1] - a[1]) - (b[1] - a[1]) * (p[0] - a[0]),
         (c[0] - b[0]) * (p[1] - b[1]) - (c[1] - b[1]) * (p[0] - b[0]),
         (a[0] - c[0]) * (p[1] - c[1]) - (a[1] - c[1]) * (p[0] - c[0])]
    return not (min(s) < 0 and max(s) > 0)


def tri_tri_intersect(t1, t2, coplanar_tol=0.0):
    """Touching counts; the coplanar case in 2-D on the dominant axes.
    coplanar_tol = 0: the reference's exact rule; > 0: vertex-plane values
    within coplanar_tol x |n| x the longest edge count as coplanar (the GPU
    checker's default 1e-9)."""
    t1, t2 = np.asarray(t1, float), np.asarray(t2, float)
    n1 = np.cross(t1[1] - t1[0], t1[2] - t1[0])
    n2 = np.cross(t2[1] - t2[0], t2[2] - t2[0])
    d2 = t2 @ n1 - t1[0] @ n1
    if np.all(d2 > 0) or np.all(d2 < 0):
        return False
    d1 = t1 @ n2 - t2[0] @ n2
    if np.all(d1 > 0) or np.all(d1 < 0):
        return False
    L = max(np.linalg.norm(np.roll(t, -1, axis=0) - t, axis=1).max() for t in (t1, t2))
    cop2 = np.all(np.abs(d2) <= coplanar_tol * L * np.linalg.norm(n1)) if coplanar_tol else np.all(d2 == 0.0)
    cop1 = np.all(np.abs(d1) <= coplanar_tol * L * np.linalg.norm(n2)) if coplanar_tol else np.all(d1 == 0.0)
    if cop2 or cop1:
        keep = [i for i in range(3) if i != int(np.argmax(np.abs(n1)))]
        a, b = t1[:, keep], t2[:, keep]
        if any(_seg_seg_2d(a[i], a[(i + 1) % 3], b[j], b[(j + 1) % 3]) for i in range(3) for j in range(3)):
            return True
        return _in_tri_2d(a[0], *b) or _in_tri_2d(b[0], *a)
    ax = int(np.argmax(np.abs(np.cross(n1, n2))))

    def span(tri, dist):
        pts = [tri[i, ax] for i in range(3) if dist[i] == 0]
        pts += [tri[i, ax] + dist[i] / (dist[i] - dist[j]) * (tri[j, ax] - tri[i, ax])
                for i in range(3) if dist[i] > 0 for j in range(3) if dist[j] < 0]
        return min(pts), max(pts)

    lo1, hi1 = span(t1, d1)
    lo2, hi2 = span(t2, d2)
    return max(lo1, lo2) <= min(hi1, hi2)


def count_tri_intersections(x, tris, coplanar_tol=0.0):
    """Non-adjacent intersecting triangle pairs (`cli.py:393-401`), boxes
    first (O(F^2) box test, vectorised), exact test on overlapping boxes."""
    x = np.asarray(x, float).reshape(-1, 3)
    tris = np.asarray(tris, np.int64).reshape(-1, 3)
    p = x[tris]
    lo, hi = p.min(axis=1), p.max(axis=1)
    n = 0
    for i in range(len(tris)):
        ov = np.all((lo[i] <= hi[i + 1:]) & (lo[i + 1:] <= hi[i]), axis=1)
        for j in np.nonzero(ov)[0] + i + 1:
            if set(tris[i].tolist()) & set(tris[j].tolist()):
                continue
            n += bool(tri_tri_intersect(p[i], p[j], coplanar_tol))
    return n
