"""Oracle conservative CCD with the per-subdomain min-reduction.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Reference: `pkg/src/ipcsim/ccd.py` -- orientation cubic `:40-56` (same
`np.linalg.det` evaluation, so coefficients are bit-identical), monotone
window `:95-115`, sign bisection `:142-157`, relative-displacement bound
`:172-193`, pair collection `:212-241`, per-pair steps `:244-281`,
per-subdomain min `:284-294`, mixed-step certificate `:297-320`, and the
clamp in `solver.py:268-280`.
"""

from __future__ import annotations

import numpy as np

from . import geometry as ogeo

S = 0.1


def collect_pairs(scene, x, p):
    """(verts (Q,4), is_pt (Q,)): PT rows (v, t0, t1, t2) in surface order,
    EE rows (a0, a1, b0, b1); boxes inflated by max |p| (`ccd.py:221-241`)."""
    x3 = np.asarray(x, float).reshape(-1, 3)
    mb = float(np.abs(p).max()) if np.size(p) else 0.0
    pt, ee = ogeo.broad_phase(x3, scene.tris, scene.edges, scene.surf_verts, mb, 0.0)
    vp = np.column_stack([pt[:, 0], scene.tris[pt[:, 1]]]) if len(pt) else np.zeros((0, 4), np.int64)
    ve = np.column_stack([scene.edges[ee[:, 0]], scene.edges[ee[:, 1]]]) if len(ee) else np.zeros((0, 4), np.int64)
    verts = np.vstack([vp, ve]).astype(np.int64)
    is_pt = np.r_[np.ones(len(vp), bool), np.zeros(len(ve), bool)]
    return verts, is_pt


def cubic_coeffs(verts, x, p):
    """(Q,4) = (a3, a2, a1, a0) of det[q1-q0, q2-q0, q3-q0](alpha)."""
    x3, p3 = x.reshape(-1, 3), p.reshape(-1, 3)
    c = x3[verts[:, 1:]] - x3[verts[:, :1]]
    e = p3[verts[:, 1:]] - p3[verts[:, :1]]

    def det(u, v, w):  # columns u, v, w
        return np.linalg.det(np.stack([u, v, w], axis=2))

    c1, c2, c3 = c[:, 0], c[:, 1], c[:, 2]
    e1, e2, e3 = e[:, 0], e[:, 1], e[:, 2]
    return np.stack([
        det(e1, e2, e3),
        det(e1, e2, c3) + det(e1, c2, e3) + det(c1, e2, e3),
        det(e1, c2, c3) + det(c1, e2, c3) + det(c1, c2, e3),
        det(c1, c2, c3),
    ], axis=1)


def window(coeffs):
    """min(first positive root of f'', first positive root of f'), +inf if
    none (`ccd.py:95-115`)."""
    a3, a2, a1 = coeffs[:, 0], coeffs[:, 1], coeffs[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        infl = np.where(a3 != 0.0, -a2 / (3.0 * a3), np.inf)
        infl = np.where(infl > 0.0, infl, np.inf)
        A, B, Cc = 3.0 * a3, 2.0 * a2, a1
        lin = np.where(B != 0.0, -Cc / B, np.inf)
        disc = B * B - 4.0 * A * Cc
        q = -0.5 * (B + np.where(B != 0.0, np.sign(B), -1.0) * np.sqrt(np.maximum(disc, 0.0)))
        r1 = np.where((A != 0.0) & (q != 0.0), q / A, np.inf)
        r2 = np.where(q != 0.0, Cc / q, np.inf)
    r1 = np.where((disc >= 0.0) & (r1 > 0.0), r1, np.inf)
    r2 = np.where((disc >= 0.0) & (r2 > 0.0), r2, np.inf)
    ext = np.where(A != 0.0, np.minimum(r1, r2), np.where(lin > 0.0, lin, np.inf))
    return np.minimum(infl, ext)


def horner(coeffs, a):
    return ((coeffs[:, 0] * a + coeffs[:, 1]) * a + coeffs[:, 2]) * a + coeffs[:, 3]


def bisect(coeffs, alpha_hat, alpha_l):
    """Halve from alpha_hat until f(alpha) a0 > 0 or alpha <= alpha_l
    (`ccd.py:147-157`), all rows at once; returns (alpha, evals, flagged)."""
    alpha = alpha_hat.copy()
    live = np.ones(len(alpha), bool)
    flagged = np.zeros(len(alpha), bool)
    evals = 0
    while live.any():
        idx = np.nonzero(live)[0]
        evals += len(idx)
        good = horner(coeffs[idx], alpha[idx]) * coeffs[idx, 3] > 0.0
        floor = ~good & (alpha[idx] <= alpha_l)
        flagged[idx[floor]] = True
        live[idx[good | floor]] = False
        more = idx[~good & ~floor]
        alpha[more] = np.maximum(0.5 * alpha[more], alpha_l)
    return alpha, evals, flagged


def rel_speed(verts, is_pt, p):
    p4 = p.reshape(-1, 3)[verts]
    q = p4 - p4.mean(axis=1, keepdims=True)
    nr = np.linalg.norm(q, axis=2)
    return np.where(is_pt, nr[:, 0] + nr[:, 1:].max(axis=1), nr[:, :2].max(axis=1) + nr[:, 2:].max(axis=1))


def distances(verts, is_pt, x):
    x3 = x.reshape(-1, 3)
    d = np.empty(len(verts))
    a, b = np.nonzero(is_pt)[0], np.nonzero(~is_pt)[0]
    if len(a):
        v = verts[a]
        d[a] = ogeo.pt_distance_batch(x3[v[:, 0]], x3[v[:, 1]], x3[v[:, 2]], x3[v[:, 3]])[0]
    if len(b):
        v = verts[b]
        d[b] = ogeo.ee_distance_batch(x3[v[:, 0]], x3[v[:, 1]], x3[v[:, 2]], x3[v[:, 3]])[0]
    return d


def pair_steps(verts, is_pt, x, p, alpha_l):
    """Certified step per pair = min(max(lb, bisection), 1) (`ccd.py:255-281`)."""
    if len(verts) == 0:
        return np.ones(0)
    co = cubic_coeffs(verts, x, p)
    d = distances(verts, is_pt, x)
    sp = rel_speed(verts, is_pt, p)
    with np.errstate(divide="ignore", invalid="ignore"):
        lb = np.where(sp > 0.0, (1.0 - S) * d / sp, np.inf)
    lb = np.minimum(np.where(d > 0.0, lb, 0.0), 1.0)
    ahat = np.minimum(1.0, window(co))
    bis = np.zeros(len(verts))
    todo = np.nonzero((lb < ahat) & (co[:, 3] != 0.0))[0]
    if len(todo):
        bis[todo] = bisect(co[todo], ahat[todo], alpha_l)[0]
    return np.minimum(np.maximum(lb, bis), 1.0)


def certify_mixed(verts, is_pt, x, p_mix):
    if len(verts) == 0:
        return True
    d = distances(verts, is_pt, x)
    sp = rel_speed(verts, is_pt, p_mix)
    ok = (np.where(sp > 0.0, (1.0 - S) * d, np.inf) >= sp) & (d > 0.0)
    rest = np.nonzero(~ok)[0]
    if len(rest) == 0:
        return True
    co = cubic_coeffs(verts[rest], x, p_mix)
    ok2 = (window(co) >= 1.0) & (co[:, 3] != 0.0) & (co.sum(axis=1) * co[:, 3] > 0.0)
    return bool(ok2.all())


def clamp(scene, part, x, p, per_subdomain, alpha_l):
    """`solver._apply_ccd`: returns (x_new, min_alpha, alpha_d, certified, n_pairs)."""
    verts, is_pt = collect_pairs(scene, x, p)
    ap = pair_steps(verts, is_pt, x, p, alpha_l)
    amin = float(ap.min()) if len(ap) else 1.0
    if not per_subdomain:
        return x + amin * p, amin, None, True, len(verts)
    alpha_d = np.ones(part.D)
    if len(verts):
        np.minimum.at(alpha_d, part.subdomain_of[verts].ravel(), np.repeat(ap, 4))
    p_mix = (alpha_d[part.subdomain_of][:, None] * p.reshape(-1, 3)).ravel()
    if not certify_mixed(verts, is_pt, x, p_mix):
        return x + amin * p, amin, alpha_d, False, len(verts)
    return x + p_mix, float(alpha_d.min()), alpha_d, True, len(verts)
